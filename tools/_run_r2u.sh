O=gpurun_out/r2u; mkdir -p $O
python tools/build_variant.py h1 -DMLSK_PANEL_HINT=1 > /dev/null 2>&1 &
python tools/build_variant.py h2 -DMLSK_PANEL_HINT=2 > /dev/null 2>&1 &
wait
for v in base h1 h2 base h1 h2; do
  if [ $v = base ]; then unset MLSK_LIB_PATH; else export MLSK_LIB_PATH=$PWD/_exp/libmlsk_$v.so; fi
  timeout 600 python tools/bench_configs.py --configs 3,5 --steps 3 --no-cpu-baseline > $O/cfg_$v.jsonl 2>&1
  python3 - $O/cfg_$v.jsonl $v <<'PY'
import json,sys
for l in open(sys.argv[1]):
    try: d=json.loads(l)
    except Exception: continue
    print(sys.argv[2], d["config"], round(d["ms_per_step"],2), round(d["step_frac_of_peak"],3), {k: round(v["ms"],1) for k,v in d["kernels"].items()}, d["clocks"]["sm_mhz"])
PY
done
