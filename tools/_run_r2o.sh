O=gpurun_out/r2o; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_hierarchy.py tests/test_gpu_fullsize.py tests/test_gpu_tc.py tests/test_gpu_exact.py -q -x --timeout 300 -p no:cacheprovider > $O/pytest.txt 2>&1; echo pytest rc=$?; tail -3 $O/pytest.txt
MLSK_SERIAL=1 timeout 600 python tools/level_probe.py --config 5 > $O/levels5.txt 2>&1; cut -c 1-80 $O/levels5.txt
timeout 900 python tools/bench_configs.py --configs 5 --steps 3 --no-cpu-baseline > $O/cfg5.jsonl 2>&1
python3 -c "
import json
d=json.loads(open('$O/cfg5.jsonl').read().splitlines()[-1])
print(d['ms_per_step'], d['step_frac_of_peak'], d['roofline']['frac'], d['clocks'], {k:round(v['ms'],1) for k,v in d['kernels'].items()})"
