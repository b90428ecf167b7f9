O=gpurun_out/r2c; mkdir -p $O
python tools/build_variant.py lo0 -DMLSK_TC_LOSMEM=0 > $O/build.txt 2>&1 || tail -5 $O/build.txt
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_fullsize.py tests/test_gpu_hierarchy.py -q -x --timeout 300 -p no:cacheprovider > $O/pytest_tc.txt 2>&1; echo pytest rc=$?; tail -5 $O/pytest_tc.txt
for v in new old new old; do
  if [ $v = old ]; then export MLSK_LIB_PATH=$PWD/_exp/libmlsk_lo0.so; else unset MLSK_LIB_PATH; fi
  timeout 600 python tools/bench_configs.py --configs 3,4,5 --steps 3 --no-cpu-baseline > $O/cfg_$v.jsonl 2>&1
  python - $O/cfg_$v.jsonl $v <<'PY'
import json,sys
for l in open(sys.argv[1]):
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    print(sys.argv[2], d["config"], round(d["ms_per_step"],2), round(d["step_frac_of_peak"],3), round(d["roofline"]["frac"],3), {k: round(v["ms"],1) for k,v in d["kernels"].items()}, d["clocks"]["sm_mhz"])
PY
done
