O=gpurun_out/r2t; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider --durations=8 > $O/pytest_gpu.txt 2>&1; echo pytest rc=$?; tail -14 $O/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
