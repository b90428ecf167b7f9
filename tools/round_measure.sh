# Full measurement pass for profiles/ (one B200): tests, smoke, bench line (config 2 + per-config
# blocks with cpu baselines), reference arm, per-level kernel times of configs 2-5 (serialised),
# ncu launch list of the bench step and ncu full captures of every engine's kernels.
#   /usr/local/graft/bin/gpurun --timeout 3600 -- 'bash tools/round_measure.sh r02'
set -x
O=gpurun_out/${1:-r02}
mkdir -p $O
(nproc; lscpu | grep "Model name"; ldd --version | head -1; nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv) > $O/host.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; tail -2 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 1200 python bench.py > $O/bench.jsonl 2> $O/bench.err; tail -1 $O/bench.jsonl | cut -c 1-200
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.jsonl 2> $O/bench_ref.err; tail -1 $O/bench_ref.jsonl | cut -c 1-200
for c in 2 3 4 5; do MLSK_SERIAL=1 timeout 600 python tools/level_probe.py --config $c > $O/levels$c.txt 2>&1; done
# launch list of the bench step (serialised, cold): per-kernel share
MLSK_BENCH_WARM_S=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --configs "" > $O/ncu_launch.log 2>&1; tail -1 $O/ncu_launch.log
# full captures: config 2 in the pipelined bench step (gemm + generator), the others one level each
MLSK_BENCH_WARM_S=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gemm_f64|gen_panels_f64" -s 20 -c 2 -o $O/full_config2 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --configs "" > $O/ncu_full2.log 2>&1; tail -1 $O/ncu_full2.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"fused_inner" -s 1 -c 1 -o $O/full_config1 python tools/bench_configs.py --configs 1 --steps 1 --no-cpu-baseline > $O/ncu_full1.log 2>&1; tail -1 $O/ncu_full1.log
MLSK_SERIAL=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"gemm_tf32x3|gen_panels_tf32" -s 2 -c 2 -o $O/full_config3 python tools/one_level.py --config 3 --level 4 > $O/ncu_full3.log 2>&1; tail -1 $O/ncu_full3.log
MLSK_SERIAL=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"gen_panels_rff|gemm_tf32x3" -s 2 -c 2 -o $O/full_config4 python tools/one_level.py --config 4 --level 3 > $O/ncu_full4.log 2>&1; tail -1 $O/ncu_full4.log
MLSK_SERIAL=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"gemm_tf32x3|gen_panels_tf32" -s 2 -c 2 -o $O/full_config5 python tools/one_level.py --config 5 --level 1 > $O/ncu_full5.log 2>&1; tail -1 $O/ncu_full5.log
ls -la $O
