O=gpurun_out/r2f; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_checkpoint.py -q --timeout 600 -p no:cacheprovider --durations=5 > $O/pytest_ckpt.txt 2>&1; echo pytest rc=$?; tail -30 $O/pytest_ckpt.txt
