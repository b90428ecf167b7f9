O=gpurun_out/r2h; mkdir -p $O
for c in 4 5; do
  MLSK_SERIAL=1 timeout 600 python tools/level_probe.py --config $c > $O/levels${c}_seg32.txt 2>&1
  MLSK_SERIAL=1 MLSK_TC_SEG=0 timeout 600 python tools/level_probe.py --config $c > $O/levels${c}_seg0.txt 2>&1
done
for f in $O/levels[45]*; do echo == $f; cat $f; done
