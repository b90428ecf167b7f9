O=gpurun_out/r2e; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_negative_control.py tests/test_gpu_exact.py -q --timeout 600 -p no:cacheprovider > $O/pytest_neg.txt 2>&1; echo pytest rc=$?; tail -8 $O/pytest_neg.txt
