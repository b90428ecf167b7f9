O=gpurun_out/r2n; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_fullsize.py tests/test_gpu_hierarchy.py tests/test_gpu_edge.py -q -x --timeout 300 -p no:cacheprovider > $O/pytest_tc.txt 2>&1; echo pytest rc=$?; tail -3 $O/pytest_tc.txt
MLSK_SERIAL=1 timeout 600 python tools/level_probe.py --config 5 > $O/levels5.txt 2>&1; cut -c 1-80 $O/levels5.txt
MLSK_SERIAL=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"gemm_tf32x3" -s 2 -c 1 python tools/one_level.py --config 5 --level 1 > $O/ncu5.log 2>&1; grep -E "dram__|gpu__time" $O/ncu5.log
timeout 900 python tools/bench_configs.py --configs 5 --steps 3 --no-cpu-baseline > $O/cfg5.jsonl 2>&1; cut -c 1-300 $O/cfg5.jsonl
