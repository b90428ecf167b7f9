O=gpurun_out/r02d; mkdir -p $O
python tools/tc_accuracy.py > $O/acc.jsonl 2>&1; python -c "
import json
for l in open('$O/acc.jsonl'):
    d=json.loads(l)
    if 'level' in d: print(d['config'], d['level'], '%.2e'%d['frob_rel'])
" | paste - - - - - - | head -8
for seg in 0 16 32; do MLSK_TC_SEG=$seg timeout 600 python tools/bench_configs.py --configs 3,4,6 --reps 3 > $O/configs_seg$seg.jsonl 2>&1; done
python - <<'PY'
import json
for f in ["configs_seg0","configs_seg16","configs_seg32"]:
    for l in open(f"gpurun_out/r02d/{f}.jsonl"):
        d=json.loads(l)
        if "config" in d: print(f, d["config"], round(d["ms_per_step"],2), round(d["frac_of_peak_step"],3), {k: round(v["ms"],1) for k,v in d["kernels"].items()})
PY
python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; tail -3 $O/pytest_gpu.txt
