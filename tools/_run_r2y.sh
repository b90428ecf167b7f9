O=gpurun_out/r2y; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_exact.py tests/test_gpu_fused.py tests/test_gpu_targets.py tests/test_gpu_statistics.py tests/test_gpu_invariance.py tests/test_gpu_multidevice.py -q -x -p no:cacheprovider 2>&1 | tail -3
for i in 1 2; do timeout 300 python tools/bench_configs.py --configs 1 --steps 20 --no-cpu-baseline > $O/c1_$i.jsonl 2>&1
python3 -c "
import json
d=json.loads(open('$O/c1_$i.jsonl').read().splitlines()[-1])
print(round(d['ms_per_step'],4), round(d['roofline']['frac'],3), {k:round(v['ms'],3) for k,v in d['kernels'].items()})"; done
