"""Small invocations of every engine for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck): the fused fp64 engine (config-2 shapes, few samples),
the config-1 inner path, the tcgen05 3xTF32 engine (gauss, Student-t, RFF
Gram incl. a K-split and a K-parallel sample), the exact (reference-stream)
engine and a multi-round session.  Run as
  compute-sanitizer --tool memcheck python tools/sanitize_cases.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_00429_b200 import mlsketch as g  # noqa: E402

S = 20260823
idf = g.target_identity()
fused = g.EstimatorOptions(device=0, engine="fused")
exact = g.EstimatorOptions(device=0, engine="exact")

m2 = g.gaussian_mean_matrix_model(256, 4096, 256, sd=0.5, data_seed=g.RngStream.derive_seed(S, 0xD47A0002, 0))
g.mlmc_matmul(m2, idf, g.LevelPlan(2, 2, [4, 2, 1], c0=32), S, fused)
g.mlmc_matmul(m2, g.target_f2(), g.LevelPlan(2, 1, [2, 1], c0=32), S, fused)
m1 = g.gaussian_mean_model(4096, sd=1.0, data_seed=g.RngStream.derive_seed(S, 0xD47A0001, 0))
g.mlmc_inner(m1, idf, g.LevelPlan(2, 5, [64, 32, 16, 8, 4, 2], c0=8), S, fused)
m3 = g.gaussian_mean_matrix_model(256, 2048, 256, sd=1.0, data_seed=3, dtype=1)
g.mlmc_matmul(m3, idf, g.LevelPlan(2, 1, [2, 1], c0=64), S, fused)
m5 = g.student_t_matrix_model(256, 4096, 256, data_seed=5)
g.mlmc_matmul(m5, idf, g.LevelPlan(2, 1, [2, 1], c0=64), S, fused)
m4 = g.rff_gram_model(512, 4096, dim=64, sigma=4.0, data_seed=4)
g.mlmc_matmul(m4, idf, g.LevelPlan(2, 1, [2, 1], c0=128), S, fused)
os.environ["MLSK_SPLIT_MB"] = "1"  # force K-split samples
g.mlmc_matmul(m3, idf, g.LevelPlan(2, 0, [1], c0=1024), S, fused)
pm = g.paper_matrix_model()
g.mlmc_matmul(pm, g.target_f2(), g.LevelPlan(10, 1, [3, 2]), S, exact)
vm = g.paper_inner_model()
g.mlmc_inner(vm, g.target_f1(), g.LevelPlan(7, 2, [5, 3, 2]), S, exact)
sess = g.MlmcSession(m2, idf, 2, 2, S, c0=32, options=fused)
sess.run_round([3, 2, 1])
sess.run_round([2, 1, 1])
sess.stats()
sess.close()
print("sanitize cases done")
