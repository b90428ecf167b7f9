O=gpurun_out/r2za; mkdir -p $O
for v in pair single pair single; do
  if [ $v = single ]; then export MLSK_TC_PAIR=0; else unset MLSK_TC_PAIR; fi
  timeout 900 python tools/bench_configs.py --configs 3,4,5 --steps 3 --no-cpu-baseline > $O/cfg_$v.jsonl 2>&1
  python3 - $O/cfg_$v.jsonl $v <<'PY'
import json,sys
for l in open(sys.argv[1]):
    try: d=json.loads(l)
    except Exception: continue
    print(sys.argv[2], d["config"], round(d["ms_per_step"],2), round(d["step_frac_of_peak"],3), round(d["roofline"]["frac"],3), {k: round(v["ms"],1) for k,v in d["kernels"].items()}, d["clocks"]["sm_mhz"])
PY
done
