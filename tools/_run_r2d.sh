O=gpurun_out/r2d; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_statistics.py tests/test_gpu_negative_control.py -q --timeout 600 -p no:cacheprovider --durations=10 > $O/pytest_new.txt 2>&1; echo pytest rc=$?; tail -25 $O/pytest_new.txt
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py > $O/sanitizer_$tool.txt 2>&1; echo $tool rc=$?; tail -4 $O/sanitizer_$tool.txt
done
timeout 600 python tools/bench_configs.py --configs 3,4,5 --steps 3 --no-cpu-baseline > $O/cfg.jsonl 2>&1; echo rc=$?
python - $O/cfg.jsonl <<'PY'
import json,sys
for l in open(sys.argv[1]):
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    print(d["config"], round(d["ms_per_step"],2), round(d["step_frac_of_peak"],3), round(d["roofline"]["frac"],3), d["peaks_tf32"], d["clocks"])
PY
