# Copy / condense a tools/round_measure.sh pass (gpurun_out/<tag>) into profiles/r02_*.
#   bash tools/collect_profiles.sh r02g
set -e
O=gpurun_out/${1:?tag}
P=profiles
cp $O/bench.jsonl $P/r02_bench.jsonl
cp $O/bench_ref.jsonl $P/r02_bench_reference_arm.jsonl
cp $O/pytest_gpu.txt $P/r02_pytest_gpu.txt
cp $O/host.txt $P/r02_host.txt
for c in 2 3 4 5; do cp $O/levels$c.txt $P/r02_levels_config${c}_final.txt; done
python tools/ncu_summary.py --launches $O/launches.csv > $P/r02_launches_config2.json
for c in 1 2 3 4 5; do python tools/ncu_summary.py $O/full_config$c.ncu-rep > $P/r02_ncu_full_config$c.json; done
