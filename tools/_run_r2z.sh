O=gpurun_out/r2z; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_hierarchy.py tests/test_gpu_fullsize.py tests/test_gpu_edge.py tests/test_gpu_checkpoint.py tests/test_gpu_invariance.py -q -x -p no:cacheprovider > $O/pytest2.txt 2>&1; echo pytest rc=$?; tail -4 $O/pytest2.txt
for c in 3 4 5; do
  MLSK_SERIAL=1 timeout 300 python tools/level_probe.py --config $c > $O/l${c}_pair.txt 2>&1
  MLSK_TC_PAIR=0 MLSK_SERIAL=1 timeout 300 python tools/level_probe.py --config $c > $O/l${c}_single.txt 2>&1
  paste <(cut -c 1-48 $O/l${c}_single.txt) <(cut -c 20-48 $O/l${c}_pair.txt)
done
timeout 300 python tools/tc_accuracy.py > $O/acc.jsonl 2>&1; python3 -c "
import json
for l in open('$O/acc.jsonl'):
    d=json.loads(l)
    if 'level' in d: print(d['config'], d['level'], '%.2e'%d['frob_rel'])
" | paste - - - - - - | head -8
