O=gpurun_out/r2x; mkdir -p $O
timeout 1500 python tools/run_adaptive.py --config 5 --budget-s 300 > $O/adaptive5.jsonl 2>&1; tail -1 $O/adaptive5.jsonl | cut -c 1-1200
