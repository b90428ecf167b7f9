O=gpurun_out/r2zd; mkdir -p $O
python tools/build_variant.py p7 -DMLSK_TC_PSTAGES=7 > /dev/null 2>&1
for v in base p7 base p7; do
  if [ $v = base ]; then unset MLSK_LIB_PATH; else export MLSK_LIB_PATH=$PWD/_exp/libmlsk_$v.so; fi
  timeout 900 python tools/bench_configs.py --configs 3,4,5 --steps 3 --no-cpu-baseline > $O/cfg_$v.jsonl 2>&1
  python3 - $O/cfg_$v.jsonl $v <<'PY'
import json,sys
for l in open(sys.argv[1]):
    try: d=json.loads(l)
    except Exception: continue
    print(sys.argv[2], d["config"], round(d["ms_per_step"],2), round(d["step_frac_of_peak"],3), round(d["roofline"]["frac"],3), d["clocks"]["sm_mhz"])
PY
done
