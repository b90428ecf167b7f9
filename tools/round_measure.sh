# Full measurement pass for profiles/ (one B200): tests, bench line, reference arm,
# configs 1-5 (+ config 5 over all levels), ncu launch list and full captures.
set -x
O=gpurun_out/r01d
mkdir -p $O
python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; tail -2 $O/pytest_gpu.txt
python bench.py > $O/bench.jsonl 2> $O/bench.err; tail -1 $O/bench.jsonl | cut -c 1-200
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.jsonl 2> $O/bench_ref.err; tail -1 $O/bench_ref.jsonl | cut -c 1-200
timeout 900 python tools/bench_configs.py --configs 1,2,3,4,5,6 --reps 3 > $O/configs.jsonl 2>&1; tail -6 $O/configs.jsonl | cut -c 1-120
MLSK_SERIAL=1 python tools/level_probe.py > $O/levels.txt 2>&1; MLSK_SERIAL=1 python tools/level_probe.py --config 3 > $O/levels3.txt 2>&1
MLSK_BENCH_WARM_S=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1; tail -1 $O/ncu_launch.log
MLSK_BENCH_WARM_S=0 ncu --set full --import-source on --clock-control none -k regex:"gemm_f64|gen_panels_f64" -s 20 -c 4 -o $O/full_config2 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1; tail -1 $O/ncu_full.log
