"""Regenerate the golden fixtures in tests/golden/ (run in the build container).

* philox_kat.json  -- libcudacxx cuda::std::philox4x32 outputs (the C++26
  std::philox4x32, whose 10000th default output the standard fixes at
  1955073260), compiled from the headers vendored with flashinfer.
* ref_streams.json / ref_draws.json / ref_estimates.json -- outputs of the
  UNMODIFIED reference library (/root/reference/proj/src compiled into
  oracle/_ref by oracle/Makefile) driven through its public API by
  oracle/ref_harness.cpp: mt19937_64 substreams, Box-Muller normals, index
  sets, model draws and per-level estimator sums, as exact IEEE bit patterns.

The tests compare the CPU oracle against these files wherever the reference
tree is absent (e.g. on the GPU box).  Usage:  python tests/golden/make_golden.py
"""
import glob
import hashlib
import json
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import pyoracle as po  # noqa: E402
from paper_1904_00429_b200 import _abi as abi  # noqa: E402

MASTER = 20260823  # proj/tests/acceptance.cpp:41


def hexs(a):
    return [float(x).hex() for x in np.asarray(a, dtype=np.float64).ravel()]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def philox_kat():
    inc = glob.glob("/opt/prime-rl/.venv/lib/python3.12/site-packages/flashinfer/data/cccl/"
                    "libcudacxx/include")
    if not inc:
        print("libcudacxx headers not found; philox_kat.json left as is")
        return
    exe = "/tmp/mlsk_philox_kat"
    subprocess.run(["g++", "-std=c++17", "-O1", f"-I{inc[0]}", os.path.join(HERE, "philox_kat.cpp"),
                    "-o", exe], check=True)
    out = json.loads(subprocess.run([exe], check=True, capture_output=True, text=True).stdout)
    out["generator"] = "libcudacxx cuda::std::philox4x32 (flashinfer-vendored CCCL headers)"
    out["cxx26_default_10000th"] = 1955073260
    with open(os.path.join(HERE, "philox_kat.json"), "w") as f:
        json.dump(out, f, indent=1)


def gauss_vec_desc(stream=abi.STREAM_REF, n=4096):
    return po.model_desc(abi.MODEL_GAUSS_MEAN, n=n, sd=1.0, mean_lo=0.0, mean_hi=1.0,
                         stream=stream, data_seed=po.oracle_lib().orc_derive_seed(MASTER, 0xD47A0001, 0))


def gauss_mat_desc(m, n, p, stream=abi.STREAM_REF):
    return po.model_desc(abi.MODEL_GAUSS_MEAN, n=n, m=m, p=p, sd=0.5, mean_lo=-1.0, mean_hi=1.0,
                         stream=stream, data_seed=po.oracle_lib().orc_derive_seed(MASTER, 0xD47A0002, 0))


def model_params(desc):
    return {"kind": desc.kind, "m": desc.m, "n": desc.n, "p": desc.p, "sd": desc.sd,
            "mean_lo": desc.mean_lo, "mean_hi": desc.mean_hi, "data_seed": int(desc.data_seed),
            "stream": desc.stream_mode}


def with_means(desc):
    """Reference-side descriptor carrying the oracle-generated means."""
    om = po.OracleModel(desc)
    ma, mb = om.means()
    d = po.model_desc(desc.kind, n=desc.n, m=desc.m, p=desc.p, sd=desc.sd, stream=desc.stream_mode,
                      mean_a=ma, mean_b=mb, data_seed=desc.data_seed, mean_lo=desc.mean_lo,
                      mean_hi=desc.mean_hi)
    return d, ma, mb


def ref_streams():
    R = po.ref_lib()
    out = {"derive_seed": [], "u64": [], "normals": [], "indices": []}
    for (m, a, b) in [(1, 0, 0), (MASTER, 3, 7), (MASTER, 0xFFFFFFFF, 12), (42, 7, 299)]:
        out["derive_seed"].append([m, a, b, int(R.ref_derive_seed(m, a, b))])
    for seed in [123, 2026, R.ref_derive_seed(MASTER, 1, 0)]:
        u = np.zeros(700, dtype=np.uint64)
        R.ref_u64_stream(seed, 700, u.ctypes.data_as(po._u64p))
        out["u64"].append({"seed": int(seed), "values": [int(x) for x in u]})
        z = np.zeros(101)
        R.ref_normals(seed, 101, z.ctypes.data_as(po._f64p))
        out["normals"].append({"seed": int(seed), "values": hexs(z)})
        for n in (4096, 1000, 3, 1):
            ix = np.zeros(65, dtype=np.uint32)
            R.ref_indices(seed, n, 65, ix.ctypes.data_as(po._u32p))
            out["indices"].append({"seed": int(seed), "n": n, "values": [int(x) for x in ix]})
    with open(os.path.join(HERE, "ref_streams.json"), "w") as f:
        json.dump(out, f)


def ref_draws():
    out = []
    cases = [("config1", gauss_vec_desc(), [(1, 0, 8), (3, 17, 64), (5, 2, 256)]),
             ("config2", gauss_mat_desc(256, 4096, 256), [(0, 0, 32), (2, 5, 128)]),
             ("paper_inner", po.model_desc(abi.MODEL_PAPER_INNER, n=1000, stream=abi.STREAM_REF),
              [(1, 0, 7), (2, 9, 49)]),
             ("paper_matrix", po.model_desc(abi.MODEL_PAPER_MATRIX, n=1000, m=10, p=10,
                                            stream=abi.STREAM_REF), [(1, 3, 4), (2, 1, 16)])]
    for name, desc, samples in cases:
        if desc.kind == abi.MODEL_GAUSS_MEAN:
            rdesc, ma, mb = with_means(desc)
        else:
            rdesc = desc
        for (tag, k, c) in samples:
            idx, a, b = po.ref_draw(rdesc, MASTER, tag, k, c)
            rec = {"case": name, "model": model_params(desc), "tag": tag, "k": k, "c": c, "indices": [int(x) for x in idx],
                   "a_sha256": sha(a), "b_sha256": sha(b),
                   "a_head": hexs(a.ravel()[:16]), "b_head": hexs(b.ravel()[:16])}
            out.append(rec)
    with open(os.path.join(HERE, "ref_draws.json"), "w") as f:
        json.dump(out, f, indent=0)


def ref_estimates():
    out = []

    def rec(name, desc, M, c0, N, seed, target=abi.TARGET_IDENTITY, tp=1e-12, native=False,
            threads=4):
        r = po.ref_mlmc(desc, M, c0, N, seed, target=target, tp=tp, threads=threads, native=native)
        out.append({"case": name, "model": model_params(desc), "M": M, "c0": c0, "N": list(N), "seed": seed, "target": target,
                    "native": native, "value": hexs(r.value),
                    "level_estimate_sha256": sha(r.level_estimate),
                    "level_estimate_head": hexs(r.level_estimate.ravel()[:8]),
                    "level_mean_sq": hexs(r.level_mean_sq),
                    "cost_units": [int(x) for x in r.cost_units],
                    "total_cost_units": r.total_cost_units})

    d1, _, _ = with_means(gauss_vec_desc())
    rec("config1", d1, 2, 8, [256, 128, 64, 32, 16, 8], MASTER)
    d2, _, _ = with_means(gauss_mat_desc(32, 512, 16))
    rec("config2_small", d2, 2, 32, [8, 6, 4, 2], MASTER)
    for tgt in (abi.TARGET_IDENTITY, abi.TARGET_F1, abi.TARGET_F2):
        rec("paper_inner", po.model_desc(abi.MODEL_PAPER_INNER, n=1000, stream=abi.STREAM_REF),
            3, 1, [300, 100, 33], 314, target=tgt, native=True)
    rec("paper_matrix_f2", po.model_desc(abi.MODEL_PAPER_MATRIX, n=1000, m=10, p=10,
                                         stream=abi.STREAM_REF), 4, 1, [40, 10], 11,
        target=abi.TARGET_F2, native=True)
    rec("constant_inner", po.model_desc(abi.MODEL_CONSTANT_ONES, n=37, stream=abi.STREAM_REF),
        3, 1, [9, 3, 1], 77, native=True)
    rec("constant_matrix", po.model_desc(abi.MODEL_CONSTANT_ONES, n=4, m=3, p=2,
                                         stream=abi.STREAM_REF), 3, 1, [9, 3, 1], 77, native=True)
    rec("deterministic_inner", po.model_desc(abi.MODEL_DETERMINISTIC, n=2, stream=abi.STREAM_REF),
        10, 1, [800, 80, 8, 1], 5, native=True)
    rec("deterministic_matrix", po.model_desc(abi.MODEL_DETERMINISTIC, n=2, m=2, p=2,
                                              stream=abi.STREAM_REF), 2, 1, [4, 2, 1], 5, native=True)
    mc = []
    for (name, desc, L, N, M, seed) in [
            ("paper_matrix", po.model_desc(abi.MODEL_PAPER_MATRIX, n=1000, m=10, p=10,
                                           stream=abi.STREAM_REF), 1, 70, 4, 23),
            ("deterministic_inner", po.model_desc(abi.MODEL_DETERMINISTIC, n=2,
                                                  stream=abi.STREAM_REF), 3, 2000, 2, 41)]:
        r = po.ref_mc(desc, L, N, M, seed)
        mc.append({"case": name, "model": model_params(desc), "L": L, "N": N, "M": M, "seed": seed, "value": hexs(r.value),
                   "total_cost_units": r.total_cost_units})
    with open(os.path.join(HERE, "ref_estimates.json"), "w") as f:
        json.dump({"mlmc": out, "mc": mc}, f, indent=0)


if __name__ == "__main__":
    po.build(ref=True)
    philox_kat()
    ref_streams()
    ref_draws()
    ref_estimates()
    print("golden fixtures written to", HERE)
