O=gpurun_out/r2p; mkdir -p $O
timeout 2400 python -m pytest tests/test_gpu_debug_checks.py -q --timeout 2000 -p no:cacheprovider --durations=5 > $O/pytest_dbg.txt 2>&1; echo pytest rc=$?; tail -15 $O/pytest_dbg.txt
