O=gpurun_out/r02c; mkdir -p $O
python tools/tc_accuracy.py > $O/acc.jsonl 2>&1; cat $O/acc.jsonl | cut -c 1-120
MLSK_TC_SEG=0 timeout 600 python tools/bench_configs.py --configs 3,4,6 --reps 3 > $O/configs_seg0.jsonl 2>&1
timeout 600 python tools/bench_configs.py --configs 3,4,6 --reps 3 > $O/configs_seg16.jsonl 2>&1
python - <<'PY'
import json
for f in ["configs_seg0","configs_seg16"]:
    for l in open(f"gpurun_out/r02c/{f}.jsonl"):
        d=json.loads(l)
        if "config" in d: print(f, d["config"], round(d["ms_per_step"],2), round(d["frac_of_peak_step"],3))
PY
python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; tail -15 $O/pytest_gpu.txt
