O=gpurun_out/r2v; mkdir -p $O
python tools/build_variant.py f64h1 -DMLSK_F64_PANEL_HINT=1 > /dev/null 2>&1
for v in base f64h1 base f64h1; do
  if [ $v = base ]; then unset MLSK_LIB_PATH; else export MLSK_LIB_PATH=$PWD/_exp/libmlsk_$v.so; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --configs "" > $O/b_$v.jsonl 2>/dev/null
  python3 -c "
import json
d=json.loads(open('$O/b_$v.jsonl').read().strip().splitlines()[-1]); print('$v', round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['frac'],4))"
done
