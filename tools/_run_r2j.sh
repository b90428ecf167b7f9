O=gpurun_out/r2j; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_fullsize.py tests/test_gpu_hierarchy.py tests/test_gpu_checkpoint.py -q -x --timeout 300 -p no:cacheprovider > $O/pytest_tc.txt 2>&1; echo pytest rc=$?; tail -3 $O/pytest_tc.txt
for c in 3 4 5; do MLSK_SERIAL=1 timeout 600 python tools/level_probe.py --config $c > $O/levels${c}.txt 2>&1; done
for f in $O/levels*; do echo == $f; cut -c 1-75 $f; done
timeout 300 python tools/tc_accuracy.py > $O/acc.jsonl 2>&1; tail -30 $O/acc.jsonl | cut -c 1-200
