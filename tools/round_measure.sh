# Full measurement pass for profiles/ (one B200): tests, bench line, reference arm,
# configs 1-5 (+ config 5 over all levels) with clocks, per-level kernel times of
# configs 2-5, ncu launch list and full captures (config 2 fp64 kernels, config 3
# 3xTF32 kernels, config 4 RFF generator), adaptive runs.
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash tools/round_measure.sh r01e'
set -x
O=gpurun_out/${1:-r01e}
mkdir -p $O
(nproc; lscpu | grep "Model name"; ldd --version | head -1; nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv) > $O/host.txt 2>&1
python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; tail -2 $O/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
python bench.py > $O/bench.jsonl 2> $O/bench.err; tail -1 $O/bench.jsonl | cut -c 1-200
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.jsonl 2> $O/bench_ref.err; tail -1 $O/bench_ref.jsonl | cut -c 1-200
timeout 1200 python tools/bench_configs.py --configs 1,2,3,4,5,6 --reps 3 > $O/configs.jsonl 2>&1; tail -6 $O/configs.jsonl | cut -c 1-120
for c in 2 3 4 5; do MLSK_SERIAL=1 timeout 600 python tools/level_probe.py --config $c > $O/levels$c.txt 2>&1; done
timeout 900 python tools/run_adaptive.py --config 2 --eps-rel 1e-2 > $O/adaptive2.jsonl 2>&1; tail -1 $O/adaptive2.jsonl | cut -c 1-200
timeout 900 python tools/run_adaptive.py --config 4 --eps-rel 1e-2 > $O/adaptive4.jsonl 2>&1; tail -1 $O/adaptive4.jsonl | cut -c 1-200
MLSK_BENCH_WARM_S=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1; tail -1 $O/ncu_launch.log
MLSK_BENCH_WARM_S=0 ncu --set full --import-source on --clock-control none -k regex:"gemm_f64|gen_panels_f64" -s 20 -c 4 -o $O/full_config2 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1; tail -1 $O/ncu_full.log
MLSK_SERIAL=1 ncu --set full --import-source on --clock-control none -k regex:"gemm_tf32x3|gen_panels_tf32" -s 12 -c 2 -o $O/full_config3 python tools/level_probe.py --config 3 > $O/ncu_full3.log 2>&1; tail -1 $O/ncu_full3.log
MLSK_SERIAL=1 ncu --set full --import-source on --clock-control none -k regex:"gen_panels_rff|gemm_tf32x3" -s 4 -c 2 -o $O/full_config4 python tools/level_probe.py --config 4 > $O/ncu_full4.log 2>&1; tail -1 $O/ncu_full4.log
