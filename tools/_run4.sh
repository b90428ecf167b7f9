O=gpurun_out/r02e; mkdir -p $O
timeout 300 python tools/tc_accuracy.py > $O/acc.jsonl 2>&1; python -c "
import json
for l in open('$O/acc.jsonl'):
    d=json.loads(l)
    if 'level' in d: print(d['config'], d['level'], '%.2e'%d['frob_rel'])
" | paste - - - - - - | head -8
for seg in 0 32; do MLSK_TC_SEG=$seg timeout 300 python tools/bench_configs.py --configs 3,4,5 --steps 3 --no-cpu-baseline > $O/configs_seg$seg.jsonl 2>&1; done
python - <<'PY'
import json
for f in ["configs_seg0","configs_seg32"]:
    for l in open(f"gpurun_out/r02e/{f}.jsonl"):
        try: d=json.loads(l)
        except Exception: print(l[:300]); continue
        if "config" in d: print(f, d["config"], round(d["ms_per_step"],2), round(d["step_frac_of_peak"],3), {k: round(v["ms"],1) for k,v in d["kernels"].items()})
PY
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > $O/pytest_gpu.txt 2>&1; tail -15 $O/pytest_gpu.txt
