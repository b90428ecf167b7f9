O=gpurun_out/r2m; mkdir -p $O
python tools/build_variant.py lo1 -DMLSK_TC_LOSMEM=1 > $O/b1.txt 2>&1 &
python tools/build_variant.py lo1a1 -DMLSK_TC_LOSMEM=1 -DMLSK_TC_LOSMEM_ABL=1 > $O/b2.txt 2>&1 &
python tools/build_variant.py lo1a2 -DMLSK_TC_LOSMEM=1 -DMLSK_TC_LOSMEM_ABL=2 > $O/b3.txt 2>&1 &
wait
for v in base lo1 lo1a1 lo1a2; do
  if [ $v = base ]; then unset MLSK_LIB_PATH; else export MLSK_LIB_PATH=$PWD/_exp/libmlsk_$v.so; fi
  MLSK_SERIAL=1 timeout 300 python tools/level_probe.py --config 3 > $O/l3_$v.txt 2>&1
  echo "== $v"; head -5 $O/l3_$v.txt | cut -c 1-80
done
