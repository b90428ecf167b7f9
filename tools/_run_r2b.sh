O=gpurun_out/r2b; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo pytest rc=$?; tail -5 $O/pytest_gpu.txt
timeout 300 python tools/bench_configs.py --configs 1 --steps 10 --no-cpu-baseline > $O/c1.jsonl 2>&1; echo rc=$?; cut -c 1-1500 $O/c1.jsonl
