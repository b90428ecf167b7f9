O=gpurun_out/r2zc; mkdir -p $O
timeout 240 python -m pytest tests/test_gpu_tc.py -q -x -p no:cacheprovider > $O/pytest_tc.txt 2>&1; echo pytest_tc rc=$?; tail -5 $O/pytest_tc.txt
