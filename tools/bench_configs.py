"""Per-configuration throughput of the B200 engines (BASELINE.json configs 1-5).

bench.py reports the metric on config 2 (the metric's single-GPU config); this
tool measures the other configurations the same way (device-resident inputs,
CUDA-event timing on the launching stream, per-kernel event timing) at a
bounded level mix per config, and prints one JSON line per config:
level-samples/s, sampled-GEMM TFLOP/s (2 m p c per level-sample; config 1:
2 c), the dominant kernel's achieved rate and its fraction of the measured
peak (fp64 DMMA, or dense TF32 / 3 for the 3xTF32 engine).

  python tools/bench_configs.py [--configs 1,3,4,5] [--reps 3]
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1904_00429_b200 import mlsketch as g  # noqa: E402
from paper_1904_00429_b200._lib import lib  # noqa: E402

MASTER = 20260823


def configs():
    ds = lambda i: g.RngStream.derive_seed(MASTER, 0xD47A0000 + i, 0)  # noqa: E731
    return {
        1: dict(model=g.gaussian_mean_model(4096, sd=1.0, mean_lo=0.0, mean_hi=1.0, data_seed=ds(1)),
                c0=8, N=[8192, 4096, 2048, 1024, 512, 256], m=1, p=1, inner=True,
                desc="x,y in R^4096 fp64, c0=8, L=5, N_l = BASELINE fixed counts"),
        2: dict(model=g.gaussian_mean_matrix_model(256, 4096, 256, sd=0.5, data_seed=ds(2)),
                c0=32, N=[256 * 2 ** (6 - l) for l in range(7)], m=256, p=256,
                desc="256x4096x256 fp64, c0=32, L=6, N_l = 256*2^(6-l)"),
        3: dict(model=g.gaussian_mean_matrix_model(1024, 16384, 1024, sd=1.0, data_seed=ds(3), dtype=1),
                c0=64, N=[8 * 2 ** (8 - l) for l in range(9)], m=1024, p=1024,
                desc="1024x16384x1024 fp32 (3xTF32), c0=64, L=8, N_l = 8*2^(8-l)"),
        4: dict(model=g.rff_gram_model(4096, 2 ** 16, dim=64, sigma=4.0, data_seed=ds(4)),
                c0=128, N=[max(1, 2 ** (6 - l)) for l in range(10)], m=4096, p=4096,
                desc="RFF Gram 4096 points, n=2^16 features, D=64, c0=128, L=9, N_l = max(1, 2^(6-l))"),
        5: dict(model=g.student_t_matrix_model(8192, 2 ** 20, 8192, data_seed=ds(5)),
                c0=256, N=[8, 4, 2, 1, 1], m=8192, p=8192,
                desc="8192x2^20x8192 fp32 Student-t(3), c0=256, levels 0-4 (c <= 4096) of L=10, N_l = 8,4,2,1,1"),
        # config 5's whole hierarchy: levels 5-10 (c = 8192 .. 262144, up to 34 GB of panels per sample) run as
        # K-segments of one sample with the partial Y carried in device memory
        6: dict(model=g.student_t_matrix_model(8192, 2 ** 20, 8192, data_seed=ds(5)),
                c0=256, N=[8, 4, 2, 1, 1, 1, 1, 1, 1, 1, 1], m=8192, p=8192,
                desc="config 5, all levels 0-10 (c = 256 .. 262144), N_l = 8,4,2,1,...,1"),
    }


def profile_read(L):
    name = C.create_string_buffer(64)
    nl, ms = C.c_int64(), C.c_double()
    out = {}
    n = L.mlsk_profile_read(0, name, 64, C.byref(nl), C.byref(ms))
    for i in range(n):
        L.mlsk_profile_read(i, name, 64, C.byref(nl), C.byref(ms))
        out[name.value.decode()] = {"launches": nl.value, "ms": ms.value}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    L = lib()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    fp64_peak = L.mlsk_measure_fp64_peak(0)
    tf32_peak = L.mlsk_measure_tf32_peak(0, 256)
    print(json.dumps({"peaks": {"fp64_dmma_tflops": fp64_peak, "tf32_dense_tflops": tf32_peak,
                                "tf32x3_effective_tflops": tf32_peak / 3}}), flush=True)
    cfgs = configs()
    for cid in [int(x) for x in args.configs.split(",")]:
        c = cfgs[cid]
        opts = g.EstimatorOptions(stream=stream.cuda_stream, engine="fused")
        L_ = len(c["N"]) - 1
        sess = g.MlmcSession(c["model"], g.target_identity(), 2, L_, MASTER, c0=c["c0"], options=opts)
        sess.run_round(c["N"])  # warm-up
        torch.cuda.synchronize()
        L.mlsk_profile_reset()
        L.mlsk_profile_enable(1)
        times = []
        with bench.ClockSampler(0) as clk:  # SM clocks / throttle reasons while the timed rounds run
            for _ in range(args.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                sess.run_round(c["N"])
                e1.record(stream)
                e1.synchronize()
                times.append(e0.elapsed_time(e1))
        L.mlsk_profile_enable(0)
        kern = profile_read(L)
        ms = sum(times) / len(times)
        samples = sum(c["N"])
        cl = [c["c0"] * 2 ** l for l in range(L_ + 1)]
        flops = sum(2.0 * c["m"] * c["p"] * cl[l] * n for l, n in enumerate(c["N"]))
        # SURVEY 8(d) algorithmic work: config 4 is a SYRK (P (P + 1) c) plus the
        # feature generation (2 P D c); the others the full 2 m p c product
        alg = (sum((c["p"] * (c["p"] + 1) + 2.0 * c["p"] * 64) * cl[l] * n for l, n in enumerate(c["N"]))
               if cid == 4 else flops)
        dom = max(kern.items(), key=lambda kv: kv[1]["ms"]) if kern else (None, {"ms": 0})
        f32 = cid >= 3
        peak = tf32_peak / 3 if f32 else fp64_peak
        dom_rate = flops * args.reps / (dom[1]["ms"] * 1e-3) / 1e12 if dom[1]["ms"] else None
        print(json.dumps({
            "config": cid, "desc": c["desc"], "ms_per_step": ms, "level_samples_per_s": samples / (ms * 1e-3),
            "sampled_gemm_tflops": flops / (ms * 1e-3) / 1e12,
            "algorithmic_tflops": alg / (ms * 1e-3) / 1e12, "kernels": kern,
            "dominant_kernel": dom[0], "dominant_achieved_tflops": dom_rate,
            "peak_tflops": peak, "peak_kind": "3xTF32 = measured dense TF32 / 3" if f32 else "measured fp64 DMMA",
            "frac_of_peak_step": alg / (ms * 1e-3) / 1e12 / peak if peak > 0 else None,
            "clocks": clk.summary(),
        }), flush=True)
        sess.close()


if __name__ == "__main__":
    main()
