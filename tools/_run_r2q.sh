O=gpurun_out/r2q; mkdir -p $O
python tools/build_variant.py minb1 -DMLSK_INNER_MINB=1 > /dev/null 2>&1 &
python tools/build_variant.py minb3 -DMLSK_INNER_MINB=3 > /dev/null 2>&1 &
python tools/build_variant.py minb5 -DMLSK_INNER_MINB=5 > /dev/null 2>&1 &
wait
for v in base minb1 minb3 minb5 base; do
  if [ $v = base ]; then unset MLSK_LIB_PATH; else export MLSK_LIB_PATH=$PWD/_exp/libmlsk_$v.so; fi
  timeout 300 python tools/bench_configs.py --configs 1 --steps 20 --no-cpu-baseline > $O/c1_$v.jsonl 2>&1
  python3 -c "
import json
d=json.loads(open('$O/c1_$v.jsonl').read().splitlines()[-1])
print('$v', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), {k:round(v['ms'],3) for k,v in d['kernels'].items()})"
done
unset MLSK_LIB_PATH
timeout 600 python -m pytest tests/test_gpu_exact.py tests/test_gpu_fused.py tests/test_gpu_targets.py tests/test_gpu_statistics.py -q -x -p no:cacheprovider 2>&1 | tail -2
