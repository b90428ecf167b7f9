import sys, time, ctypes as C
sys.path.insert(0, ".")
import numpy as np
import bench
from paper_1904_00429_b200 import mlsketch as g, _abi as abi
from paper_1904_00429_b200._lib import lib
plan = g.LevelPlan(2, 6, bench.STEP_N, c0=32)
model = g.gaussian_mean_matrix_model(256, 4096, 256, sd=0.5, data_seed=bench.data_seed())
L = lib()
for i in range(8):
    t0 = time.perf_counter()
    desc = model.desc(); cpl = plan._c(); buf = g._Buffers(7, 65536); o = g.EstimatorOptions()._c()
    t1 = time.perf_counter()
    rc = L.mlsk_mlmc_matmul(C.byref(desc), 0, 0.0, C.byref(cpl), 3 + i, C.byref(o), C.byref(buf.c))
    t2 = time.perf_counter()
    rep = g._report(buf, model, 7, False)
    t3 = time.perf_counter()
    print(f"prep {1e3*(t1-t0):.1f} call {1e3*(t2-t1):.1f} (inside {1e3*buf.c.wall_time_s:.1f}) report {1e3*(t3-t2):.1f}")
