import time, sys, numpy as np
sys.path.insert(0,'/root/repo')
from paper_1904_00429_b200 import mlsketch as g
model = g.gaussian_mean_matrix_model(256, 4096, 256, sd=0.5, data_seed=5)
for c0, N in [(32, 4096), (256, 1024), (2048, 256)]:
    plan = g.LevelPlan(2, 0, [N], c0=c0)
    g.mlmc_matmul(model, g.target_identity(), plan, 1)
    t=time.time(); r=g.mlmc_matmul(model, g.target_identity(), plan, 2); dt=time.time()-t
    fl = 2*256*256*c0*N
    print(f"c={c0} N={N}: {dt*1e3:.1f} ms  {fl/dt/1e12:.2f} TFLOP/s  {N/dt:.0f} samples/s")
