O=gpurun_out/r2r; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo pytest rc=$?; tail -3 $O/pytest_gpu.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --configs 3,4,5 > $O/bench.jsonl 2> $O/bench.err; echo bench rc=$?
python3 - $O/bench.jsonl <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print('c2', d['value'], d['ms_per_step'], d['roofline']['frac'], {k:round(v['ms'],1) for k,v in d['kernels'].items()})
for k,v in d['configs'].items():
    print(k, round(v['ms_per_step'],3), v.get('step_frac_of_peak'), v['roofline']['frac'], {a:round(b['ms'],1) for a,b in v['kernels'].items()}, v['clocks']['sm_mhz'])
PY
