"""Run a few bench-like rounds and print the per-kernel timeline (diagnostics)."""
import ctypes as C
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1904_00429_b200 import mlsketch as g  # noqa: E402
from paper_1904_00429_b200._lib import lib  # noqa: E402

L = lib()
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
opts = g.EstimatorOptions(stream=stream.cuda_stream, engine="fused")
if len(sys.argv) > 1 and sys.argv[1] == "3":  # config 3 (fp32, 3xTF32 engine)
    model = g.gaussian_mean_matrix_model(1024, 16384, 1024, sd=1.0, data_seed=3, dtype=1)
    sess = g.MlmcSession(model, g.target_identity(), 2, 8, 1, c0=64, options=opts)
    STEP = [8 * 2 ** (8 - l) for l in range(9)]
elif len(sys.argv) > 1 and sys.argv[1] in ("4", "5"):  # as tools/bench_configs.py defines them
    import bench_configs_lib  # noqa: E402
    cf = bench_configs_lib.configs(g)[int(sys.argv[1])]
    model, STEP = cf["model"], cf["N"]
    sess = g.MlmcSession(model, g.target_identity(), 2, len(STEP) - 1, 1, c0=cf["c0"], options=opts)
else:
    model = g.gaussian_mean_matrix_model(256, 4096, 256, sd=0.5, data_seed=bench.data_seed())
    sess = g.MlmcSession(model, g.target_identity(), 2, 6, 1, c0=32, options=opts)
    STEP = bench.STEP_N
for _ in range(3):
    sess.run_round(STEP)
torch.cuda.synchronize()
L.mlsk_profile_reset()
L.mlsk_profile_enable(1)
sess.run_round(STEP)
torch.cuda.synchronize()
L.mlsk_profile_enable(0)
name = C.create_string_buffer(64)
t0, t1 = C.c_double(), C.c_double()
n = L.mlsk_profile_timeline(0, name, 64, C.byref(t0), C.byref(t1))
rows = []
for i in range(n):
    L.mlsk_profile_timeline(i, name, 64, C.byref(t0), C.byref(t1))
    rows.append((t0.value, t1.value, name.value.decode()))
rows.sort()
for a, b, nm in rows:
    print(f"{a:8.3f} {b:8.3f} {b - a:7.3f}  {nm}")
