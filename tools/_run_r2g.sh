O=gpurun_out/r2g; mkdir -p $O
python tools/e2e_breakdown.py > $O/e2e_breakdown.json 2>&1; cat $O/e2e_breakdown.json
MLSK_SERIAL=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"gen_panels_f64" -s 3 -c 1 -o $O/gen64 python tools/level_probe.py --config 2 > $O/ncu_gen64.log 2>&1; tail -2 $O/ncu_gen64.log
