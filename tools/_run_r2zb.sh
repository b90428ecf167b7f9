O=gpurun_out/r2zb; mkdir -p $O
python tools/build_variant.py nolo -DMLSK_TC_ABL_NOLO > /dev/null 2>&1
for v in base nolo; do
  if [ $v = base ]; then unset MLSK_LIB_PATH; else export MLSK_LIB_PATH=$PWD/_exp/libmlsk_$v.so; fi
  for c in 3 4; do MLSK_SERIAL=1 timeout 300 python tools/level_probe.py --config $c > $O/l${c}_$v.txt 2>&1; done
done
for c in 3 4; do echo "== $c"; paste <(cut -c 1-48 $O/l${c}_base.txt) <(cut -c 20-48 $O/l${c}_nolo.txt); done
