"""Per-level kernel times of the config-2 round (diagnostics): each level of the
bench step alone, serialised generator / GEMM, event-timed per kernel."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1904_00429_b200 import mlsketch as g  # noqa: E402
from paper_1904_00429_b200._lib import lib  # noqa: E402

import argparse  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2, choices=[2, 3, 4, 5])
args = ap.parse_args()
L = lib()
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
opts = g.EstimatorOptions(stream=stream.cuda_stream, engine="fused")
if args.config == 2:
    model = g.gaussian_mean_matrix_model(256, 4096, 256, sd=0.5, data_seed=bench.data_seed())
    m = p = 256
    c0, LV, STEP = 32, 6, bench.STEP_N
    gemm_name = "gemm_f64"
elif args.config == 3:
    model = g.gaussian_mean_matrix_model(1024, 16384, 1024, sd=1.0, data_seed=3, dtype=1)
    m = p = 1024
    c0, LV, STEP = 64, 8, [8 * 2 ** (8 - l) for l in range(9)]
    gemm_name = "gemm_tf32x3"
else:  # configs 4 and 5 as tools/bench_configs.py defines them
    import bench_configs_lib  # noqa: E402
    cf = bench_configs_lib.configs(g)[args.config]
    model, m, p, c0, STEP = cf["model"], cf["m"], cf["p"], cf["c0"], cf["N"]
    LV = len(STEP) - 1
    gemm_name = "gemm_tf32x3"
name = C.create_string_buffer(64)
nl, ms = C.c_int64(), C.c_double()
for lvl in range(LV + 1):
    N = [0] * (LV + 1)
    N[lvl] = STEP[lvl]
    sess = g.MlmcSession(model, g.target_identity(), 2, LV, 1, c0=c0, options=opts)
    sess.run_round(N)
    torch.cuda.synchronize()
    L.mlsk_profile_reset()
    L.mlsk_profile_enable(1)
    for _ in range(3):
        sess.run_round(N)
    torch.cuda.synchronize()
    L.mlsk_profile_enable(0)
    out = {}
    for i in range(L.mlsk_profile_read(0, name, 64, C.byref(nl), C.byref(ms))):
        L.mlsk_profile_read(i, name, 64, C.byref(nl), C.byref(ms))
        out[name.value.decode()] = round(ms.value / 3, 3)
    c = c0 * 2 ** lvl
    flops = 2.0 * m * p * c * N[lvl]
    gemm = out.get(gemm_name, 0)
    print(f"level {lvl} c={c:5d} N={N[lvl]:6d}  " + "  ".join(f"{k} {v:.3f} ms" for k, v in out.items()) +
          f"  gemm {flops / (gemm * 1e-3) / 1e12 if gemm else 0:.1f} TFLOP/s")
    sess.close()
