O=gpurun_out/r02a; mkdir -p $O
python -m pytest tests -m gpu -q -x --durations=15 > $O/pytest_gpu.txt 2>&1; tail -30 $O/pytest_gpu.txt
python bench.py --steps 5 --warmup 3 > $O/bench.jsonl 2> $O/bench.err; tail -1 $O/bench.jsonl | cut -c 1-300
MLSK_DIST_BACKEND=gloo timeout 300 python bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench2.jsonl 2> $O/bench2.err; echo rc=$?; tail -1 $O/bench2.jsonl | cut -c 1-300; tail -5 $O/bench2.err
