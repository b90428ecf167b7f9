set -x
mkdir -p gpurun_out/r01b
python -m pytest tests -m gpu -q > gpurun_out/r01b/pytest_gpu.txt 2>&1; tail -2 gpurun_out/r01b/pytest_gpu.txt
python bench.py > gpurun_out/r01b/bench.jsonl 2> gpurun_out/r01b/bench.err; tail -1 gpurun_out/r01b/bench.jsonl | cut -c 1-300
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r01b/bench_ref.jsonl 2> gpurun_out/r01b/bench_ref.err; tail -1 gpurun_out/r01b/bench_ref.jsonl | cut -c 1-300
timeout 600 python tools/bench_configs.py --reps 3 > gpurun_out/r01b/configs.jsonl 2>&1; tail -5 gpurun_out/r01b/configs.jsonl | cut -c 1-120
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01b/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r01b/ncu_launch.log 2>&1; tail -1 gpurun_out/r01b/ncu_launch.log
ncu --set full --import-source on --clock-control none -k regex:"gemm_f64|gen_panels_f64" -s 20 -c 4 -o gpurun_out/r01b/full_config2 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r01b/ncu_full.log 2>&1; tail -1 gpurun_out/r01b/ncu_full.log
