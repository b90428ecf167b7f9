O=gpurun_out/r2a; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider --durations=20 > $O/pytest_gpu.txt 2>&1; echo pytest rc=$?; tail -40 $O/pytest_gpu.txt
timeout 600 python __graft_entry__.py smoke > $O/smoke.txt 2>&1; echo smoke rc=$?; tail -3 $O/smoke.txt
timeout 900 python bench.py > $O/bench.jsonl 2> $O/bench.err; echo bench rc=$?; tail -c 3000 $O/bench.jsonl; tail -5 $O/bench.err
