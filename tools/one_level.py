"""One level of a BASELINE configuration, for ncu captures of a single
GEMM / generator launch:  python tools/one_level.py --config 3 --level 4
(the level's step count N_l from bench_configs_lib, one warm-up round + --reps)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench_configs_lib  # noqa: E402
from paper_1904_00429_b200 import mlsketch as g  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--level", type=int, default=0)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--n", type=int, default=0, help="replications (default: the bench step's N_l)")
a = ap.parse_args()
cf = bench_configs_lib.configs(g)[a.config]
LV = len(cf["N"]) - 1
N = [0] * (LV + 1)
N[a.level] = a.n or cf["N"][a.level]
opts = g.EstimatorOptions(engine="fused")
sess = g.MlmcSession(cf["model"], g.target_identity(), 2, LV, 1, c0=cf["c0"], options=opts)
for _ in range(1 + a.reps):
    sess.run_round(N)
torch.cuda.synchronize()
sess.close()
print("done", a.config, a.level, N[a.level])
