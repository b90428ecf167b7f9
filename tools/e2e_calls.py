"""Per-call wall times of the bench's e2e leg (diagnostics)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1904_00429_b200 import mlsketch as g  # noqa: E402

seeded = g.gaussian_mean_matrix_model(256, 4096, 256, sd=0.5, data_seed=bench.data_seed())
ma, mb = g.model_data(seeded, 0), g.model_data(seeded, 1)
pa = torch.from_numpy(ma).pin_memory().numpy()
pb = torch.from_numpy(mb).pin_memory().numpy()
model = g.gaussian_mean_matrix_model(256, 4096, 256, sd=0.5, mean_a=pa, mean_b=pb)
plan = g.LevelPlan(2, 6, bench.STEP_N, c0=32)
opts = g.EstimatorOptions(device=0, engine="fused")
ts = []
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    t0 = time.perf_counter()
    g.mlmc_matmul(model, g.target_identity(), plan, 100 + i, opts)
    ts.append(1e3 * (time.perf_counter() - t0))
print(" ".join(f"{t:.1f}" for t in ts))
