O=gpurun_out/r2s; mkdir -p $O
python tools/build_variant.py noepi -DMLSK_TC_ABL_NOEPI > /dev/null 2>&1 &
python tools/build_variant.py nosum -DMLSK_TC_ABL_NOSUM > /dev/null 2>&1 &
python tools/build_variant.py noload -DMLSK_TC_ABL_NOLD > /dev/null 2>&1 &
wait
for v in base noepi nosum noload; do
  if [ $v = base ]; then unset MLSK_LIB_PATH; else export MLSK_LIB_PATH=$PWD/_exp/libmlsk_$v.so; fi
  MLSK_SERIAL=1 timeout 300 python tools/level_probe.py --config 3 > $O/l3_$v.txt 2>&1
  echo "== $v"; head -4 $O/l3_$v.txt | cut -c 1-60
done
