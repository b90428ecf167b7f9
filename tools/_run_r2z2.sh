O=gpurun_out/r2z2; mkdir -p $O
MLSK_SERIAL=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"gemm_tf32x3" -s 1 -c 1 -o $O/pair_c3l4 python tools/one_level.py --config 3 --level 4 > $O/ncu.log 2>&1; tail -1 $O/ncu.log
