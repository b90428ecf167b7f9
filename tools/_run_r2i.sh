O=gpurun_out/r2i; mkdir -p $O
for seg in 32 0; do
  MLSK_TC_SEG=$seg MLSK_SERIAL=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"gemm_tf32x3" -s 1 -c 1 -o $O/c3l4_seg$seg python tools/one_level.py --config 3 --level 4 > $O/ncu_c3l4_$seg.log 2>&1; tail -1 $O/ncu_c3l4_$seg.log
  MLSK_TC_SEG=$seg MLSK_SERIAL=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"gemm_tf32x3" -s 1 -c 1 -o $O/c5l2_seg$seg python tools/one_level.py --config 5 --level 2 > $O/ncu_c5l2_$seg.log 2>&1; tail -1 $O/ncu_c5l2_$seg.log
done
