#!/usr/bin/env python
"""bench.py -- MLMC sampled-product level estimator on B200 (BASELINE.json config 2).

Workload (config 2, the metric's single-GPU configuration): A 256x4096 and
B 4096x256 fp64, A = M + 0.5 N(0,1), B = P + 0.5 N(0,1), M, P ~ U(-1,1) fixed
from the seed, c_l = 32 * 2^l for l = 0..6 (c_6 = 2048), coarse = first half.
One STEP is one round of the MLMC driver at the standard allocation's level
mix (N_l proportional to sqrt(V_l / C_l) ~ 1/c_l, so every level costs the
same): N_l = 256 * 2^(6-l) = 16384 ... 256 level-samples per GPU.  Data are
synthetic (no dataset is involved); inputs are generated on the device (the
means are resident in HBM; the per-sample noise is generated in-kernel).

  value  = level-samples / s over all ranks (weak scaling: every rank runs its
           own N_l, sharded by 64-replication chunks, then one NCCL all-reduce of
           the per-level (sum Y, sum ||Y||^2, count) buffers per round)
  e2e    = the same metric through the public API (mlsketch.mlmc_matmul) with the
           means passed from pinned HOST buffers and the report read back,
           host<->device copies inside the timed region
  roofline = the dominant kernel (k_gemm_f64, DMMA) against the fp64 tensor-pipe
           peak measured in this run; algorithmic flops = 2 m p c per level-sample

--impl reference times the reference's own CPU implementation (compiled from
/root/reference into oracle/_ref, else the oracle port) on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MASTER = 20260823
M_, N_, P_ = 256, 4096, 256
C0, LEVELS = 32, 6
STEP_N = [256 * 2 ** (LEVELS - l) for l in range(LEVELS + 1)]          # 16384 ... 256
CPU_SAMPLE_N = [512, 256, 128, 64, 32, 16, 8]                          # bounded CPU sample
REF_STEP_N = [128, 64, 32, 16, 8, 4, 2]                                # --impl reference step
METRIC = "MLMC level-samples/s (config 2: 256x4096x256 fp64, c_l=32*2^l, L=6, standard-allocation level mix)"
UNIT = "level-samples/s"


# seconds of device warm-up (memory writes + DMMA) before the warm-up steps;
# MLSK_BENCH_WARM_S=0 for profiler passes (keeps the launch list to the steps)
GPU_WARM_S = float(os.environ.get("MLSK_BENCH_WARM_S", "2.5"))


def flops_of(N):
    return sum(2.0 * M_ * P_ * C0 * 2 ** l * n for l, n in enumerate(N))


def ref_convention_flops_of(N):
    """The reference's own cost convention (two passes, estimators.cpp:137-147): 2 m p (c_l + c_{l-1})."""
    return sum(2.0 * M_ * P_ * (C0 * 2 ** l + (C0 * 2 ** (l - 1) if l > 0 else 0)) * n for l, n in enumerate(N))


def panel_bytes_of(N):
    """Algorithmic bytes the GEMM reads: the sampled columns of A and rows of B (fp64)."""
    return sum(8.0 * (M_ + P_) * C0 * 2 ** l * n for l, n in enumerate(N))


_U64 = 0xFFFFFFFFFFFFFFFF


def _mix(z):  # RngStream::mix, rng.hpp:22-27 (pure host arithmetic: the reference arm loads no product code)
    z = (z + 0x9E3779B97F4A7C15) & _U64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _U64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _U64
    return z ^ (z >> 31)


def derive_seed(master, a, b):  # RngStream::derive_seed, rng.hpp:31-37
    return _mix(_mix(_mix(master) ^ ((a + 0x9E3779B97F4A7C15) & _U64)) ^ ((b + 0xBF58476D1CE4E5B9) & _U64))


def data_seed(config=2):
    """Seed of the config's fixed-from-seed data: derive_seed(master, 0xD47A0000 + config, 0)."""
    return derive_seed(MASTER, 0xD47A0000 + config, 0)


def config_dict(world, flush, warm=None):
    d = {"workload": "config2: A 256x4096, B 4096x256 fp64 gaussian(U(-1,1) means, sd 0.5); "
                        "c0=32, M=2, L=6; step = N_l = 256*2^(6-l) per GPU",
            "m": M_, "n": N_, "p": P_, "c0": C0, "M": 2, "L": LEVELS, "N_per_gpu": STEP_N,
            "stream": "philox4x32-10", "engine": "fused (gen_panels_f64 + gemm_f64 DMMA)",
            "l2": flush, "parallelism": f"dp{world} (64-replication chunk sharding)"}
    if warm:
        d["device_warmup"] = warm
    return d


# ---------------------------------------------------------------- clocks


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        # NVML (microseconds per query) at ~20 ms intervals; nvidia-smi (100+ ms
        # per call) only when pynvml is unavailable
        nv = None
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.device)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            bits = [getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
                    getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
                    getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
                    getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4)]
        except Exception:
            nv = None

        def run_nvml():
            while not self._stop.is_set():
                try:
                    sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                    try:
                        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    except Exception:
                        r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                    self.rows.append([str(sm), str(mx), "", ""] + ["Active" if r & b else "Not Active" for b in bits])
                except Exception:
                    pass
                self._stop.wait(0.1)  # sparse: NVML queries contend with the launching thread

        def run_smi():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.rows.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=run_nvml if nv is not None else run_smi, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 4 + i and r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------- CPU baselines


def cpu_reference_run(N, threads=None):
    """Reference (or oracle-port) CPU time for level counts N; returns (seconds, kind)."""
    import ctypes as C
    from oracle import pyoracle as po
    from paper_1904_00429_b200 import _abi as abi
    threads = threads or os.cpu_count()
    desc = po.model_desc(abi.MODEL_GAUSS_MEAN, n=N_, m=M_, p=P_, sd=0.5, mean_lo=-1.0, mean_hi=1.0,
                         stream=abi.STREAM_REF, data_seed=data_seed())
    om = po.OracleModel(desc)
    if os.path.exists(po.REF_SO):
        ma, mb = om.means()
        rdesc = po.model_desc(abi.MODEL_GAUSS_MEAN, n=N_, m=M_, p=P_, sd=0.5, stream=abi.STREAM_REF,
                              mean_a=ma, mean_b=mb)
        plan = po.make_plan(2, C0, N)
        ck = C.c_double()
        dt = po.ref_lib().ref_throughput(C.byref(rdesc), 0, 1e-12, C.byref(plan), MASTER, threads, C.byref(ck))
        if dt < 0:
            raise RuntimeError(po.ref_lib().ref_last_error().decode())
        return dt, "reference", threads
    # oracle port: single-threaded C restatement of the same per-replication work
    t0 = time.perf_counter()
    om.mlmc(2, C0, N, MASTER)
    return time.perf_counter() - t0, "port", 1


def cpu_baseline_obj(N):
    dt, kind, cores = cpu_reference_run(N)
    return {"value": sum(N) / dt, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"config 2, N_l={N} (full reference per-replication work: fresh 256x4096 + 4096x256 "
                      f"mt19937_64/Box-Muller draw, draw_realization, sketch_matmul fine + coarse), "
                      f"{dt:.2f} s wall"}


def run_reference_arm(args, rank):
    if rank != 0:
        return 0
    for _ in range(args.warmup):
        cpu_reference_run([1] * (LEVELS + 1))
    times = []
    kind, cores = None, None
    for _ in range(args.steps):
        dt, kind, cores = cpu_reference_run(REF_STEP_N)
        times.append(dt)
    total = sum(times)
    value = args.steps * sum(REF_STEP_N) / total
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": "config2 (reference CPU, bounded sample per step)", "m": M_, "n": N_, "p": P_,
                       "c0": C0, "M": 2, "L": LEVELS, "N_per_step": REF_STEP_N, "threads": cores},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": f"N_l={REF_STEP_N} per step"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------- GPU arm


def relaunch(n):
    """`bench.py --gpus N` outside torchrun: run itself as N ranks (one process
    per GPU) under torch.distributed.run on 127.0.0.1 and return its exit code."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")          # NCCL's init lines show every rank joining
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)



def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mlsk", choices=["mlsk", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--configs", default="1,3,4,5",
                    help="BASELINE configs measured as extra blocks of the JSON line (N=1 only; '' = none)")
    args = ap.parse_args()

    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl != "reference":
        return relaunch(args.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference_arm(args, rank)
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")

    import torch
    device = local_rank % max(1, torch.cuda.device_count())
    torch.cuda.set_device(device)
    dist = None
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("MLSK_DIST_BACKEND", "nccl")  # gloo: multi-rank tests on one GPU
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", device))
        else:
            dist.init_process_group(backend)

    from paper_1904_00429_b200 import mlsketch as g
    from paper_1904_00429_b200._lib import lib
    L = lib()

    stream = torch.cuda.Stream()            # explicit stream: the library orders its work on it
    torch.cuda.set_stream(stream)
    opts = g.EstimatorOptions(device=device, stream=stream.cuda_stream, rank=rank, world=world, engine="fused")
    model = g.gaussian_mean_matrix_model(M_, N_, P_, sd=0.5, mean_lo=-1.0, mean_hi=1.0, data_seed=data_seed())
    sess = g.MlmcSession(model, g.target_identity(), 2, LEVELS, MASTER, c0=C0, options=opts)
    dN = [n * world for n in STEP_N]          # global counts; this rank runs its chunks (~N_l)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")   # 512 MB > L2 (126 MB)

    class _Dev:  # zero-copy torch view of the session's packed device buffer
        def __init__(self, ptr, n):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                             "version": 3, "stream": None}

    def step():
        sess.run_round(dN)
        if dist is not None:
            p, n = sess.level_buffer()          # packed on the same stream (device-side)
            dist.all_reduce(torch.as_tensor(_Dev(p, n), device="cuda"))

    # Bring the device out of its idle state before the warm-up steps: a freshly
    # started box runs the first ~1 s of work at a lower effective speed (the SM
    # clock reads max, the memory side ramps), which W = 3 short steps do not cover.
    t_warm = time.perf_counter()
    while time.perf_counter() - t_warm < GPU_WARM_S:
        flush.add_(1.0)                      # HBM traffic
        L.mlsk_measure_fp64_peak(device)     # DMMA work (~tens of ms)
        torch.cuda.synchronize()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    peak = L.mlsk_measure_fp64_peak(device)
    L.mlsk_profile_reset()
    L.mlsk_profile_enable(1)
    launches0 = L.mlsk_kernel_launch_count()
    import ctypes as C
    cols = (C.c_int64 * 2)()
    L.mlsk_contraction_columns(cols, 1)   # reset the executed / sampled column counters
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    flush.zero_()                               # evict L2 once; per-step inputs (15 GB of panels) exceed L2
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    with ClockSampler(device) as clk:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        e1.synchronize()
    step_ms = [e0.elapsed_time(e1) / args.steps] * args.steps
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    L.mlsk_profile_enable(0)
    launches = L.mlsk_kernel_launch_count() - launches0
    L.mlsk_contraction_columns(cols, 0)
    contraction = contraction_note(cols[0], cols[1])
    total_ms = sum(step_ms)
    if dist is not None:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())

    # per-kernel event timings (this rank)
    kern = {}
    name = C.create_string_buffer(64)
    nl, ms = C.c_int64(), C.c_double()
    n_entries = L.mlsk_profile_read(0, name, 64, C.byref(nl), C.byref(ms))
    for i in range(n_entries):
        L.mlsk_profile_read(i, name, 64, C.byref(nl), C.byref(ms))
        kern[name.value.decode()] = {"launches": nl.value, "ms": ms.value}

    samples_total = args.steps * sum(dN)
    value = samples_total / (total_ms * 1e-3)
    flops_total = args.steps * flops_of(dN)
    gemm = kern.get("gemm_f64", {"launches": 0, "ms": 0.0})
    rank_flops = args.steps * flops_of(STEP_N)
    achieved = rank_flops / (gemm["ms"] * 1e-3) / 1e12 if gemm["ms"] > 0 else None
    # dram traffic per average launch: the ratio (dram bytes / algorithmic panel
    # bytes) of a full batch captured with ncu --set full, times this run's
    # algorithmic bytes per launch
    traffic = None
    step_traffic = None
    prof_json = os.path.join(ROOT, "profiles", "gemm_f64_traffic.json")
    if os.path.exists(prof_json) and gemm["launches"] > 0:
        try:
            pj = json.load(open(prof_json))
            ratio = pj.get("dram_over_algorithmic")
            traffic = (ratio * (contraction["executed_over_sampled"] or 1.0) * args.steps * panel_bytes_of(STEP_N)
                       / gemm["launches"]) if ratio else None
            sr = pj.get("step_dram_over_algorithmic")
            if sr:  # generator + GEMM DRAM bytes of a whole step (not the GEMM's reads alone)
                # the captured ratio is per batch of panels; with merged sampled columns the step
                # generates and reads panels for the executed columns only
                ex = contraction["executed_over_sampled"] or 1.0
                step_traffic = {"dram_bytes_per_step": sr * ex * panel_bytes_of(STEP_N),
                                "algorithmic_bytes_per_step": panel_bytes_of(STEP_N), "ratio": sr * ex,
                                "per_batch_ratio": sr, "executed_over_sampled_columns": ex,
                                "source": pj.get("source")}
        except Exception:
            traffic = None

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(g, torch, device, args, rank, world, dist)

    cpu = None
    if not args.no_cpu_baseline and rank == 0 and world == 1:
        try:
            cpu = cpu_baseline_obj(CPU_SAMPLE_N)
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "unavailable", "sample": str(e)}

    blocks = None
    if args.configs and world == 1:
        # the other BASELINE configurations, same timing rules (bench_configs_lib.py)
        import bench_configs_lib
        torch.cuda.synchronize()
        blocks = bench_configs_lib.measure([int(x) for x in args.configs.split(",") if x], steps=3,
                                           with_cpu=not args.no_cpu_baseline, device=device)
        torch.cuda.set_stream(stream)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": config_dict(world, "inputs larger than L2: each step generates ~15 GB of sampled panels; "
                                             "L2 flushed (512 MB write) before the timed region",
                                      warm=f"{GPU_WARM_S} s of device memory writes and DMMA work before the "
                                           f"{args.warmup} warm-up steps"),
                "sampled_gemm_tflops": flops_total / (total_ms * 1e-3) / 1e12,
                # roofline_time / measured_time of the whole step (flops-bound), and the
                # reference-convention rate (fine and coarse as two passes: 2 m p (c_l + c_{l-1}))
                "step_frac_of_peak": (flops_total / world / (total_ms * 1e-3) / 1e12 / peak) if peak > 0 else None,
                "reference_convention_tflops": args.steps * ref_convention_flops_of(dN) / (total_ms * 1e-3) / 1e12,
                "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                             "frac": (achieved / peak) if achieved and peak > 0 else None,
                             "traffic": traffic, "kernel": "k_gemm_f64 (DMMA m8n8k4, fp64)",
                             "peak_source": "fp64 DMMA throughput measured in this run "
                                            "(MEASURED_PEAKS.json has no fp64 entry)",
                             "algorithmic": "2*m*p*c_l flops per level-sample"},
                "step_traffic": step_traffic,
                "contraction": contraction,
                "kernels": kern,
                "step_fraction_gemm": (gemm["ms"] / sum(v["ms"] for v in kern.values())) if kern else None,
                "gpu_launches": launches,
                "clocks": clk.summary(),
                "e2e": e2e,
                "cpu_baseline": cpu}
        if blocks is not None:
            line["configs"] = blocks
        print(json.dumps(line), flush=True)
    sess.close()
    if dist is not None:
        dist.destroy_process_group()
    return 0


def contraction_note(executed, sampled):
    """Merged sampled columns (include/mlsk.h mlsk_contraction_columns): the GEMMs run over the
    distinct sampled columns of a level-sample (summed weights; fine / coarse pairs cancel), so
    the executed K is below the sampled c_l at the deep levels.  `value`, `sampled_gemm_tflops`
    and `roofline.achieved` count the ALGORITHMIC work (2 m p c_l per level-sample)."""
    return {"executed_columns": int(executed), "sampled_columns": int(sampled),
            "executed_over_sampled": (executed / sampled) if sampled else None,
            "note": "merged sampled columns: K runs over the distinct columns of each level-sample (padded to "
                    "K-chunks); algorithmic flops = 2 m p c_l per level-sample, executed flops = that x "
                    "executed_over_sampled; MLSK_MERGE=0 runs every sampled index"}


def run_e2e(g, torch, device, args, rank=0, world=1, dist=None):
    """Public-API call per step on every rank: means from pinned host buffers ->
    device, this rank's replication chunks of all levels (global counts
    N_l * world, rank-sharded as the library's multi-GPU path does), the
    per-level sums all-reduced across ranks, the report on the host.  Timed by
    wall clock between barriers, max over ranks; value = all ranks' samples /
    that time."""
    import numpy as np
    # the config's means as host arrays (read back once from the seeded model)
    seeded = g.gaussian_mean_matrix_model(M_, N_, P_, sd=0.5, data_seed=data_seed())
    ma, mb = g.model_data(seeded, 0), g.model_data(seeded, 1)
    pa = torch.from_numpy(ma).pin_memory().numpy()
    pb = torch.from_numpy(mb).pin_memory().numpy()
    model = g.gaussian_mean_matrix_model(M_, N_, P_, sd=0.5, mean_a=pa, mean_b=pb)
    plan = g.LevelPlan(2, LEVELS, [n * world for n in STEP_N], c0=C0)
    opts = g.EstimatorOptions(device=device, engine="fused", rank=rank, world=world)
    cells = M_ * P_
    levels = LEVELS + 1
    on_dev = world > 1 and dist.get_backend() == "nccl"  # gloo (multi-rank tests on one GPU): host buffer
    red = torch.empty(levels * (cells + 1), dtype=torch.float64, device="cuda" if on_dev else "cpu") \
        if world > 1 else None

    def call(seed):
        r = g.mlmc_matmul(model, g.target_identity(), plan, seed, opts)
        if world > 1:  # the global level sums: one all-reduce of [sum Y | sum ||Y||^2] per level
            host = np.concatenate([np.append(np.asarray(st.sum, dtype=np.float64).ravel(), st.sum_of_squares)
                                   for st in r.per_level])
            red.copy_(torch.from_numpy(host))
            dist.all_reduce(red)
            if on_dev:
                red.cpu()
        return r

    for _ in range(max(1, args.warmup)):
        call(MASTER)
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    calls = []
    for i in range(args.steps):
        tc = time.perf_counter()
        call(MASTER + 1 + i)
        calls.append(1e3 * (time.perf_counter() - tc))
    dt = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([dt], dtype=torch.float64, device="cuda" if on_dev else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    # what one rank's call moves: the two mean matrices and the replication runs
    # (24 B each: one per level at world 1, one per owned 64-chunk when sharded;
    # the index lists are expanded on the device) in, each level's
    # [sum Y | sum ||Y||^2] out (mlsk_api.cu read_levels); with world > 1 also
    # the all-reduce buffer in and out
    runs = levels if world == 1 else sum(len(range(rank, (n * world + 63) // 64, world)) for n in STEP_N)
    h2d = pa.nbytes + pb.nbytes + 24 * runs + (8 * levels * (cells + 1) if world > 1 else 0)
    d2h = 8 * levels * (cells + 1) * (2 if world > 1 else 1)
    return {"value": world * args.steps * sum(STEP_N) / dt, "unit": UNIT,
            "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h),
            "call_ms": {"median": statistics.median(calls), "max": max(calls)},
            "note": "mlsketch.mlmc_matmul with host mean buffers on every rank (rank-sharded global plan, "
                    "level sums all-reduced); wall clock between barriers, max over ranks"}


if __name__ == "__main__":
    sys.exit(main())
