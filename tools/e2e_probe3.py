"""Per-call breakdown of the public-API path (bench.py's e2e leg)."""
import sys, time, ctypes as C
sys.path.insert(0, ".")
import numpy as np
import torch
import bench
from paper_1904_00429_b200 import mlsketch as g
seeded = g.gaussian_mean_matrix_model(256, 4096, 256, sd=0.5, data_seed=bench.data_seed())
ma, mb = g.model_data(seeded, 0), g.model_data(seeded, 1)
pa = torch.from_numpy(ma).pin_memory().numpy()
pb = torch.from_numpy(mb).pin_memory().numpy()
host = g.gaussian_mean_matrix_model(256, 4096, 256, sd=0.5, mean_a=pa, mean_b=pb)
plan = g.LevelPlan(2, 6, bench.STEP_N, c0=32)
opts = g.EstimatorOptions(engine="fused")
r1 = g.mlmc_matmul(seeded, g.target_identity(), plan, 5, opts)
r2 = g.mlmc_matmul(host, g.target_identity(), plan, 5, opts)
print("host means == seeded means result:", np.array_equal(r1.value, r2.value))
for i in range(6):
    t0 = time.perf_counter()
    r = g.mlmc_matmul(host, g.target_identity(), plan, 7 + i, opts)
    t1 = time.perf_counter()
    print(f"call {1e3*(t1-t0):.2f} ms  inside {1e3*r.wall_time_seconds:.2f} ms")
