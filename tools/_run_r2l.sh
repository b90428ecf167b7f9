O=gpurun_out/r2l; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo pytest rc=$?; tail -3 $O/pytest_gpu.txt
timeout 900 python tools/bench_configs.py --configs 1,3,4,5 --steps 3 --no-cpu-baseline > $O/cfg.jsonl 2>&1; echo rc=$?
python - $O/cfg.jsonl <<'PY'
import json,sys
for l in open(sys.argv[1]):
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    print(d["config"], round(d["ms_per_step"],3), d.get("step_frac_of_peak"), round(d["roofline"]["frac"],3), {k: round(v["ms"],1) for k,v in d["kernels"].items()}, d["clocks"])
PY
