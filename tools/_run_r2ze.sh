O=gpurun_out/r2ze; mkdir -p $O
python tools/build_variant.py mel -DMLSK_MEAN_EVICT_LAST=1 > /dev/null 2>&1
for v in base mel base mel; do
  if [ $v = base ]; then unset MLSK_LIB_PATH; else export MLSK_LIB_PATH=$PWD/_exp/libmlsk_$v.so; fi
  timeout 600 python tools/bench_configs.py --configs 3 --steps 3 --no-cpu-baseline > $O/cfg_$v.jsonl 2>&1
  python3 - $O/cfg_$v.jsonl $v <<'PY'
import json,sys
for l in open(sys.argv[1]):
    try: d=json.loads(l)
    except Exception: continue
    print(sys.argv[2], d["config"], round(d["ms_per_step"],2), {k: round(v["ms"],1) for k,v in d["kernels"].items()})
PY
  MLSK_SERIAL=1 timeout 300 python tools/level_probe.py --config 3 2>&1 | head -2 | cut -c 1-90
done
