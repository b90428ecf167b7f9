"""Where does the end-to-end (public API, host buffers) time go? (diagnostics)"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from oracle import pyoracle as po  # noqa: E402
from paper_1904_00429_b200 import _abi as abi, mlsketch as g  # noqa: E402

om = po.OracleModel(po.model_desc(abi.MODEL_GAUSS_MEAN, n=4096, m=256, p=256, sd=0.5, mean_lo=-1, mean_hi=1,
                                  data_seed=bench.data_seed()))
ma, mb = om.means()
pa = torch.from_numpy(ma).pin_memory().numpy()
pb = torch.from_numpy(mb).pin_memory().numpy()
plan = g.LevelPlan(2, 6, bench.STEP_N, c0=32)
for label, model in [("host-means", g.gaussian_mean_matrix_model(256, 4096, 256, sd=0.5, mean_a=pa, mean_b=pb)),
                     ("device-means", g.gaussian_mean_matrix_model(256, 4096, 256, sd=0.5, data_seed=bench.data_seed()))]:
    g.mlmc_matmul(model, g.target_identity(), plan, 1)
    ts = []
    for i in range(5):
        t0 = time.perf_counter()
        r = g.mlmc_matmul(model, g.target_identity(), plan, 2 + i)
        ts.append(time.perf_counter() - t0)
    print(label, "per call ms", [round(t * 1e3, 1) for t in ts], "reported wall", round(r.wall_time_seconds * 1e3, 1))
# tiny call: fixed overhead
small = g.LevelPlan(2, 0, [1], c0=32)
m2 = g.gaussian_mean_matrix_model(256, 4096, 256, sd=0.5, data_seed=1)
g.mlmc_matmul(m2, g.target_identity(), small, 1)
t0 = time.perf_counter()
for i in range(10):
    g.mlmc_matmul(m2, g.target_identity(), small, 1)
print("tiny call ms", (time.perf_counter() - t0) * 100)
