"""Per-configuration measurement blocks for bench.py (BASELINE.json configs
1, 3, 4 and 5; config 2 is the headline line itself).

Each block times one STEP of the configuration -- one round of the MLMC
driver at a fixed level mix, inputs (means, RFF data) resident in HBM, the
per-sample noise generated in-kernel -- with CUDA events on the stream the
library launches on, after a warm-up round, and reports:

  value        level-samples / s
  roofline     the dominant kernel against its bound:
               configs 3-5: algorithmic flops (2 m p c per level-sample;
               config 4: P (P + 1) c + 2 P D c, the SYRK and the feature
               generation) / the kernel's event time, against the dense TF32
               tcgen05 peak measured in this run / 3 (3xTF32);
               config 1: index-samples / s against the RNG roofline measured
               in this run (mlsk_measure_index_rate: the per-index Philox,
               Box-Muller and mean gathers alone, no launch or reduction)
  cpu_baseline the reference's CPU implementation (compiled from
               /root/reference into oracle/_ref) on this host:
               config 1: the full per-replication body (draw, realization,
               sketch fine + coarse) on all cores, ref_throughput;
               configs 3-5: the reference cannot draw these models in
               bounded time (config 3: 33.5 M normals per replication,
               config 5: 17 G), so the time per level-sample is composed
               from its own measured components on one core (BASELINE.md
               section 2): RngStream::normal throughput x the normals one
               replication draws (config 4: the feature evaluations, timed
               with the oracle's fp64 RFF entry), plus sketch_matmul at the
               config's (m, p) for c_l + c_l / 2 indices (linear in c, timed
               at a small c on pre-drawn data)
"""
from __future__ import annotations

import ctypes as C
import os
import time

MASTER = 20260823


def _ds(i):
    import bench
    return bench.derive_seed(MASTER, 0xD47A0000 + i, 0)


def configs(g):
    return {
        1: dict(model=g.gaussian_mean_model(4096, sd=1.0, mean_lo=0.0, mean_hi=1.0, data_seed=_ds(1)),
                c0=8, N=[8192 * 64 // 2 ** l for l in range(6)], m=1, p=1, n=4096, inner=True,
                workload="config1: x,y in R^4096 fp64 N(U(0,1) means, 1); c0=8, M=2, L=5; step = 64 x the "
                         "BASELINE counts N_l = {8192 ... 256} in one round (64 estimators' samples; one "
                         "estimator alone is launch-bound: see single_estimator_ms)"),
        3: dict(model=g.gaussian_mean_matrix_model(1024, 16384, 1024, sd=1.0, data_seed=_ds(3), dtype=1),
                c0=64, N=[8 * 2 ** (8 - l) for l in range(9)], m=1024, p=1024, n=16384,
                workload="config3: A 1024x16384, B 16384x1024 fp32 N(U(-1,1) means, 1); c0=64, M=2, L=8; "
                         "step = N_l = 8*2^(8-l) (standard-allocation shape: every level costs the same)"),
        4: dict(model=g.rff_gram_model(4096, 2 ** 16, dim=64, sigma=4.0, data_seed=_ds(4)),
                c0=128, N=[max(1, 2 ** (6 - l)) for l in range(10)], m=4096, p=4096, n=2 ** 16,
                workload="config4: RFF Gram of 4096 points in R^64, n=2^16 features, sigma=4; c0=128, M=2, L=9; "
                         "step = N_l = max(1, 2^(6-l))"),
        5: dict(model=g.student_t_matrix_model(8192, 2 ** 20, 8192, data_seed=_ds(5)),
                c0=256, N=[8, 4, 2, 1, 1, 1, 1, 1, 1, 1, 1], m=8192, p=8192, n=2 ** 20,
                workload="config5: A 8192x2^20, B 2^20x8192 fp32 Student-t(3) + U(-0.5,0.5) means; c0=256, M=2, "
                         "L=10; step = N_l = 8,4,2,1,...,1 (all levels; c_10 = 262144: K-split samples)"),
    }


def alg_flops(cid, c, levels_c):
    if cid == 4:  # SYRK + feature generation
        return sum((c["p"] * (c["p"] + 1) + 2.0 * c["p"] * 64) * cl * n for cl, n in zip(levels_c, c["N"]))
    return sum(2.0 * c["m"] * c["p"] * cl * n for cl, n in zip(levels_c, c["N"]))


TRAFFIC_JSON = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "tc_traffic.json")


def attach_traffic(cid, blk):
    """roofline.traffic (DRAM bytes per launch of the dominant kernel) and the
    step's DRAM bytes against its algorithmic bytes, from the ncu pass
    tools/traffic_probe.py committed under profiles/ (same step, same kernels)."""
    try:
        import json as _json
        t = _json.load(open(TRAFFIC_JSON))[str(cid)]
    except (OSError, KeyError, ValueError):
        return
    kname = "k_fused_inner_multi" if cid == 1 else "k_gemm_tf32x3"
    k = t["kernels"].get(kname)
    if k and "roofline" in blk:
        blk["roofline"]["traffic"] = k["dram_bytes_per_launch"]
        blk["roofline"]["traffic_source"] = t["source"]
    blk["step_traffic"] = {"dram_bytes_per_step": t["dram_bytes_per_step"],
                           "algorithmic_bytes_per_step": t["algorithmic_bytes_per_step"], "ratio": t["ratio"],
                           "per_kernel_dram_bytes_per_step": {
                               n: v["dram_bytes_per_launch"] * v["launches_per_step"]
                               for n, v in t["kernels"].items()},
                           "source": t["source"]}


def profile_read(L):
    name = C.create_string_buffer(64)
    nl, ms = C.c_int64(), C.c_double()
    out = {}
    n = L.mlsk_profile_read(0, name, 64, C.byref(nl), C.byref(ms))
    for i in range(n):
        L.mlsk_profile_read(i, name, 64, C.byref(nl), C.byref(ms))
        out[name.value.decode()] = {"launches": nl.value, "ms": ms.value}
    return out


# ------------------------------------------------------------ CPU baselines


def _cpu_component_baseline(cid, c, levels_c):
    """Reference CPU time per level-sample from its measured components (one core)."""
    from oracle import pyoracle as po
    R = po.ref_lib()
    # RngStream::normal throughput (rng.hpp:55-65, glibc)
    import numpy as np
    cnt = 2_000_000
    buf = np.zeros(cnt)
    t0 = time.perf_counter()
    R.ref_normals(12345, cnt, buf.ctypes.data_as(C.POINTER(C.c_double)))
    t_normal = (time.perf_counter() - t0) / cnt
    # sketch_matmul (sketch.cpp:45-77) per sampled index at (m, p): pre-drawn data, n = 64 (cost is linear in c
    # and independent of n)
    cs = 16 if c["m"] * c["p"] >= 8192 * 8192 else 64
    reps = 1 if c["m"] * c["p"] >= 4096 * 4096 else 3
    t_sk = R.ref_time_sketch_matmul(c["m"], 64, c["p"], cs, 7, reps) / cs
    if cid == 4:
        # the reference draws the whole feature matrix Z (P x n, B = Z^T) per replication: time the
        # oracle's fp64 entry (dot of 64 + glibc cos, the reference model's arithmetic) on a sample
        om = po.OracleModel(c["model"].desc())
        cc = 256
        t0 = time.perf_counter()
        om.draw(1, 0, 0, cc)  # P x cc entries of A and the same again for B = A^T
        t_entry = (time.perf_counter() - t0) / (2 * c["m"] * cc)
        t_draw = t_entry * c["m"] * c["n"]
        draw_desc = f"feature evaluations {c['m']}x{c['n']} at {t_entry * 1e9:.1f} ns (oracle fp64 RFF entry)"
    else:
        draws = c["m"] * c["n"] + c["n"] * c["p"]
        t_draw = draws * t_normal
        draw_desc = f"{draws:.3g} normals at {t_normal * 1e9:.1f} ns (RngStream::normal)"
    per_level = [t_draw + (cl + (cl // 2 if l > 0 else 0)) * t_sk for l, cl in enumerate(levels_c)]
    total = sum(n * t for n, t in zip(c["N"], per_level))
    return {"value": sum(c["N"]) / total, "unit": "level-samples/s", "cores": 1, "kind": "reference",
            "sample": f"composed per level-sample (one core): draw = {draw_desc}; sketch_matmul fine + coarse at "
                      f"{t_sk * 1e6:.1f} us per index ({c['m']}x{c['p']}, timed at c={cs}); level mix N_l={c['N']}",
            "seconds_per_level_sample": per_level}


def _cpu_config1_baseline(c):
    from oracle import pyoracle as po
    from paper_1904_00429_b200 import _abi as abi
    threads = os.cpu_count() or 1
    desc = po.model_desc(abi.MODEL_GAUSS_MEAN, n=4096, sd=1.0, mean_lo=0.0, mean_hi=1.0, stream=abi.STREAM_REF,
                         data_seed=_ds(1))
    om = po.OracleModel(desc)
    ma, mb = om.means()
    rdesc = po.model_desc(abi.MODEL_GAUSS_MEAN, n=4096, sd=1.0, stream=abi.STREAM_REF, mean_a=ma, mean_b=mb)
    N = [8192 // 2 ** l for l in range(6)]  # the BASELINE fixed counts (one estimator)
    plan = po.make_plan(2, 8, N)
    ck = C.c_double()
    dt = po.ref_lib().ref_throughput(C.byref(rdesc), 0, 1e-12, C.byref(plan), MASTER, threads, C.byref(ck))
    if dt < 0:
        raise RuntimeError(po.ref_lib().ref_last_error().decode())
    return {"value": sum(N) / dt, "unit": "level-samples/s", "cores": threads, "kind": "reference",
            "sample": f"config 1 BASELINE counts N_l={N} (one estimator), full reference per-replication body "
                      f"(mt19937_64 + Box-Muller draw of x, y, draw_realization, sketch_inner fine + coarse), "
                      f"{dt:.2f} s wall on {threads} threads"}


def cpu_baseline(cid, c, levels_c):
    try:
        if cid == 1:
            return _cpu_config1_baseline(c)
        return _cpu_component_baseline(cid, c, levels_c)
    except Exception as e:  # reported, not fatal
        return {"value": None, "unit": "level-samples/s", "cores": None, "kind": "unavailable", "sample": str(e)}


# --------------------------------------------------------------- GPU timing


def measure(ids, steps=3, with_cpu=True, device=0):
    """One block per configuration id; runs on `device` (rank 0 at N = 1)."""
    import torch

    import bench
    from paper_1904_00429_b200 import mlsketch as g
    from paper_1904_00429_b200._lib import lib
    L = lib()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    tf32 = L.mlsk_measure_tf32_peak(device, 256)
    # B200_PROFILING.md: the burst peak is the denominator for a kernel timed
    # alone, the sustained one (power-capped clocks) for a kernel timed inside a
    # long step; a block whose timed region runs >= 1 s (config 5) uses it.
    # The TF32 probe alone never reaches the 1000 W cap (it stays at 1965 MHz
    # for seconds: measured), so the sustained TF32 figure is the burst one
    # scaled by MEASURED_PEAKS.json's cuBLAS bf16 sustained / burst ratio.
    tf32_sus, sus_note = None, None
    try:
        import json as _json
        pk = _json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")))
        ratio = pk["bf16_tflops_sustained"] / pk["bf16_tflops"]
        tf32_sus = tf32 * ratio
        sus_note = f"burst x {ratio:.3f} (MEASURED_PEAKS.json bf16 sustained / burst)"
    except Exception:
        pass
    idx_rate = L.mlsk_measure_index_rate(device) if 1 in ids else None
    cfgs = configs(g)
    out = {}
    for cid in ids:
        c = cfgs[cid]
        L_ = len(c["N"]) - 1
        levels_c = [c["c0"] * 2 ** l for l in range(L_ + 1)]
        opts = g.EstimatorOptions(device=device, stream=stream.cuda_stream, engine="fused")
        sess = g.MlmcSession(c["model"], g.target_identity(), 2, L_, MASTER, c0=c["c0"], options=opts)
        sess.run_round(c["N"])  # warm-up
        torch.cuda.synchronize()
        L.mlsk_profile_reset()
        L.mlsk_profile_enable(1)
        launches0 = L.mlsk_kernel_launch_count()
        cols = (C.c_int64 * 2)()
        L.mlsk_contraction_columns(cols, 1)
        nsteps = max(steps, 20) if c.get("inner") else steps  # config 1: 0.4 ms steps
        with bench.ClockSampler(device) as clk:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(nsteps):
                sess.run_round(c["N"])
            e1.record(stream)
            e1.synchronize()
        L.mlsk_profile_enable(0)
        launches = L.mlsk_kernel_launch_count() - launches0
        L.mlsk_contraction_columns(cols, 0)
        ms = e0.elapsed_time(e1) / nsteps
        kern = profile_read(L)
        samples = sum(c["N"])
        blk = {"workload": c["workload"], "ms_per_step": ms, "value": samples / (ms * 1e-3),
               "unit": "level-samples/s", "steps": nsteps, "gpu_launches": launches, "kernels": kern,
               "clocks": clk.summary()}
        if c.get("inner"):
            idx = sum(cl * n for cl, n in zip(levels_c, c["N"]))
            # a single estimator (the BASELINE counts) is latency-bound: time it too
            one = [n // 64 for n in c["N"]]
            sess.run_round(one)
            torch.cuda.synchronize()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record(stream)
            for _ in range(10):
                sess.run_round(one)
            f1.record(stream)
            f1.synchronize()
            blk["single_estimator_ms"] = f0.elapsed_time(f1) / 10
            achieved = idx / (ms * 1e-3)
            blk["index_samples_per_s"] = achieved
            blk["normals_per_s"] = 2 * achieved
            blk["roofline"] = {"bound": "rng", "achieved": achieved / 1e9, "peak": idx_rate / 1e9 if idx_rate else None,
                               "unit": "G index-samples/s", "frac": achieved / idx_rate if idx_rate else None,
                               "traffic": None, "kernel": "k_fused_inner_multi (whole step)",
                               "peak_source": "mlsk_measure_index_rate in this run: the per-index work "
                                              "(Philox index + Philox/Box-Muller pair + mean gathers) alone",
                               "algorithmic": "2 c_l fp64 flops, 16 c_l bytes (means) and 2 c_l normals per "
                                              "level-sample: far below HBM / fp64 bounds, the RNG is the bound"}
        else:
            flops = alg_flops(cid, c, levels_c)
            gem = kern.get("gemm_tf32x3", {"ms": 0.0, "launches": 0})
            ach = flops * nsteps / (gem["ms"] * 1e-3) / 1e12 if gem["ms"] > 0 else None
            # a long timed region, or one that ran under the power cap (config 5: ~1450 MHz),
            # is measured against the sustained peak
            cs = blk["clocks"] or {}
            capped = bool(cs.get("sm_mhz") and cs.get("sm_max_mhz") and cs["sm_mhz"] < 0.9 * cs["sm_max_mhz"])
            long_region = (ms * nsteps >= 500.0 or capped) and tf32_sus
            peak_t = tf32_sus if long_region else tf32
            which = f"sustained: {sus_note}" if long_region else "burst"
            blk["sampled_gemm_tflops"] = sum(2.0 * c["m"] * c["p"] * cl * n for cl, n in zip(levels_c, c["N"])) \
                / (ms * 1e-3) / 1e12
            blk["reference_convention_tflops"] = sum(
                2.0 * c["m"] * c["p"] * (cl + (levels_c[l - 1] if l > 0 else 0)) * n
                for l, (cl, n) in enumerate(zip(levels_c, c["N"]))) / (ms * 1e-3) / 1e12
            blk["algorithmic_tflops"] = flops / (ms * 1e-3) / 1e12
            blk["step_frac_of_peak"] = blk["algorithmic_tflops"] / (peak_t / 3)
            blk["peaks_tf32"] = {"burst": tf32, "sustained": tf32_sus, "used": which}
            bfx = os.environ.get("MLSK_TC_BF16X", "1") != "0"
            # FP16 pairs (bounded models: configs 3, 4) and FP16 hi + BF16 cross terms (config 5) both run
            # 3 K = 16 MMAs per K-chunk; MLSK_TC_H16=0: TF32 hi x hi + BF16 cross terms, 4 MMA slots instead of 6
            h16 = bfx and os.environ.get("MLSK_TC_H16", "1") != "0"
            # own ceiling: three 16-bit K = 16 MMAs per K-chunk = the dense bf16 / fp16 rate
            # (MEASURED_PEAKS.json, cuBLAS bf16: burst, or sustained for a long / power-capped region) / 3;
            # TF32 + BF16 cross terms: 4 MMA slots instead of 6 -> TF32 / 2
            own = peak_t / 2 if bfx else peak_t / 3
            if h16:
                try:
                    own = (pk["bf16_tflops_sustained"] if long_region else pk["bf16_tflops"]) / 3
                except Exception:
                    own = peak_t * 2 / 3
            if h16 and cid == 5:
                kernel_desc = ("k_gemm_tf32x3 (tcgen05.mma cta_group::2 kind::f16: per 16-column K-chunk 3 MMAs, one FP16 "
                               "hi x hi + two BF16 cross terms over fp16(x) | bf16(x) and bf16(x - hi))")
            elif h16:
                kernel_desc = ("k_gemm_tf32x3 (tcgen05.mma cta_group::2 kind::f16: per 16-column K-chunk 3 FP16 MMAs over "
                               "fp16(x) | fp16(x - fp16(x)) pairs: hi x hi, hi x lo, lo x hi)")
            elif bfx:
                kernel_desc = ("k_gemm_tf32x3 (tcgen05.mma cta_group::2: per 16-column K-chunk 2 kind::tf32 MMAs for "
                               "hi x hi + 2 kind::f16 BF16 MMAs for the cross terms)")
            else:
                kernel_desc = "k_gemm_tf32x3 (tcgen05.mma kind::tf32, 3 MMAs per K-step)"
            blk["roofline"] = {"bound": "tensor", "achieved": ach, "peak": peak_t / 3, "unit": "TFLOP/s",
                               "frac": ach / (peak_t / 3) if ach else None, "traffic": None,
                               "kernel": kernel_desc,
                               "peak_source": f"dense TF32 tcgen05 measured in this run, {which} "
                                              f"({peak_t:.0f} TFLOP/s) / 3",
                               # SURVEY 8(d)'s fp32 peak is TF32 / 3 (3xTF32).  With split 16-bit operands a
                               # K-chunk costs three 16-bit MMAs instead of six TF32 ones, so `frac` can exceed 1;
                               # the kernel's own ceiling is the measured dense bf16 rate / 3: both are given.
                               "own_ceiling": own,
                               "frac_of_own_ceiling": (ach / own) if ach else None,
                               "algorithmic": ("P(P+1) c + 2 P D c flops per level-sample (SYRK + features)"
                                               if cid == 4 else "2 m p c flops per level-sample")}
        if not c.get("inner"):
            blk["contraction"] = bench.contraction_note(cols[0], cols[1])
        attach_traffic(cid, blk)
        if with_cpu:
            blk["cpu_baseline"] = cpu_baseline(cid, c, levels_c)
        out[str(cid)] = blk
        sess.close()
    return out
