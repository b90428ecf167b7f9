O=gpurun_out/r2w; mkdir -p $O
timeout 600 python tools/run_adaptive.py --config 2 --eps-rel 1e-2 > $O/adaptive2.jsonl 2>&1; tail -1 $O/adaptive2.jsonl | cut -c 1-400
timeout 900 python tools/run_adaptive.py --config 4 --eps-rel 1e-2 > $O/adaptive4.jsonl 2>&1; tail -1 $O/adaptive4.jsonl | cut -c 1-400
timeout 900 python tools/run_adaptive.py --config 3 --eps-rel 5e-2 > $O/adaptive3.jsonl 2>&1; tail -1 $O/adaptive3.jsonl | cut -c 1-400
timeout 1200 python tools/run_adaptive.py --config 5 --budget-s 300 > $O/adaptive5.jsonl 2>&1; tail -1 $O/adaptive5.jsonl | cut -c 1-800
