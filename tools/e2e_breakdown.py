"""Where the e2e call time goes (config 2): the public-API call with host means,
the same call with device-generated means (no H2D), and a session round
(the bench `value` step), each median of 15 after warm-up; plus the
library's event-timed kernel sum per call."""
import ctypes as C
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1904_00429_b200 import mlsketch as g  # noqa: E402
from paper_1904_00429_b200._lib import lib  # noqa: E402

L = lib()
seeded = g.gaussian_mean_matrix_model(256, 4096, 256, sd=0.5, data_seed=bench.data_seed())
ma, mb = g.model_data(seeded, 0), g.model_data(seeded, 1)
pa = torch.from_numpy(ma).pin_memory().numpy()
pb = torch.from_numpy(mb).pin_memory().numpy()
host = g.gaussian_mean_matrix_model(256, 4096, 256, sd=0.5, mean_a=pa, mean_b=pb)
plan = g.LevelPlan(2, 6, bench.STEP_N, c0=32)
opts = g.EstimatorOptions(device=0, engine="fused")


def timed(fn, n=15):
    for _ in range(3):
        fn(0)
    ts = []
    for i in range(n):
        t = time.perf_counter()
        fn(i + 1)
        ts.append(1e3 * (time.perf_counter() - t))
    return statistics.median(ts)


out = {}
out["call_host_means_ms"] = timed(lambda i: g.mlmc_matmul(host, g.target_identity(), plan, 100 + i, opts))
out["call_device_means_ms"] = timed(lambda i: g.mlmc_matmul(seeded, g.target_identity(), plan, 100 + i, opts))
sess = g.MlmcSession(seeded, g.target_identity(), 2, 6, 7, c0=32, options=opts)
out["session_round_ms"] = timed(lambda i: sess.run_round(bench.STEP_N))
L.mlsk_profile_reset()
L.mlsk_profile_enable(1)
g.mlmc_matmul(host, g.target_identity(), plan, 999, opts)
L.mlsk_profile_enable(0)
name = C.create_string_buffer(64)
nl, ms = C.c_int64(), C.c_double()
n = L.mlsk_profile_read(0, name, 64, C.byref(nl), C.byref(ms))
kern = {}
for i in range(n):
    L.mlsk_profile_read(i, name, 64, C.byref(nl), C.byref(ms))
    kern[name.value.decode()] = round(ms.value, 3)
out["kernels_one_call_ms"] = kern
print(json.dumps(out))
