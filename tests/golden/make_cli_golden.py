"""Regenerate the CLI / planner / reference-value golden fixtures (run in the
build container, where /root/reference exists).

The reference CLI (proj/tools/mlsketch_main.cpp) cannot be compiled here
(CLI11.hpp is missing), so oracle/ref_harness.cpp restates its `sweep
--no-timing` and `estimate` commands on top of the UNMODIFIED reference
library (compiled from /root/reference/proj/src by oracle/Makefile) and this
script stores the text they print, byte for byte:

  cli_golden.json  -- {"sweep": [{args, csv}], "estimate": [{args, text}],
                       "plans": [{eps, M, c1, c2, n, L, N, n_cap_applied, N_mc}],
                       "reference_values": [{model, target, count, seed, mean (hex), se (hex)}]}

Usage:  python tests/golden/make_cli_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import pyoracle as po  # noqa: E402
from paper_1904_00429_b200 import _abi as abi  # noqa: E402

SWEEPS = [
    dict(mode="inner", model="paper-inner", target="f1", m_list=[2, 3, 5], eps=0.2, reps=2, n_ref=20000, seed=1),
    dict(mode="inner", model="constant-ones", target="identity", m_list=[2, 4], eps=0.25, reps=1, n_ref=500,
         seed=11),
    dict(mode="matmul", model="paper-matrix", target="f2", m_list=[3, 4], eps=0.2, reps=1, n_ref=4000, seed=1),
    dict(mode="matmul", model="deterministic", target="identity", m_list=[2], eps=0.3, reps=2, n_ref=64, seed=5),
]
ESTIMATES = [
    dict(mode="inner", model="paper-inner", target="f1", M=7, eps=0.1, seed=1),
    dict(mode="inner", model="paper-inner", target="identity", M=3, eps=0.15, seed=99),
    dict(mode="matmul", model="paper-matrix", target="f2", M=4, eps=0.1, seed=7),
    dict(mode="matmul", model="paper-matrix", target="identity", M=10, eps=0.2, seed=3),
]
PLANS = [(eps, M, c1, c2, n) for eps in (0.05, 0.1, 0.2, 0.3) for M in (2, 3, 4, 7, 10, 32)
         for c1, c2 in ((1.0, 1.0), (0.5, 2.0), (3.0, 0.25)) for n in (1, 100, 1000, 4096)]
REFVALS = [
    (abi.MODEL_PAPER_INNER, 1000, 0, 0, abi.TARGET_F1, 300, 17),
    (abi.MODEL_PAPER_INNER, 1000, 0, 0, abi.TARGET_IDENTITY, 129, 5),
    (abi.MODEL_PAPER_MATRIX, 1000, 10, 10, abi.TARGET_F2, 150, 23),
    (abi.MODEL_PAPER_MATRIX, 1000, 10, 10, abi.TARGET_IDENTITY, 65, 3),
    (abi.MODEL_DETERMINISTIC, 2, 2, 2, abi.TARGET_IDENTITY, 1, 1),
]


def main():
    out = {"sweep": [], "estimate": [], "plans": [], "reference_values": []}
    for a in SWEEPS:
        csv = po.ref_sweep_csv(a["mode"], a["model"], a["target"], a["m_list"], eps=a["eps"], reps=a["reps"],
                               n_ref=a["n_ref"], seed=a["seed"], threads=8)
        out["sweep"].append(dict(args=a, csv=csv))
    for a in ESTIMATES:
        txt = po.ref_estimate_text(a["mode"], a["model"], a["target"], M=a["M"], eps=a["eps"], seed=a["seed"],
                                   threads=8)
        out["estimate"].append(dict(args=a, text=txt))
    for eps, M, c1, c2, n in PLANS:
        L, N, cap, nmc = po.ref_make_plan(eps, M, c1, c2, n)
        out["plans"].append(dict(eps=eps, M=M, c1=c1, c2=c2, n=n, L=L, N=N, n_cap_applied=cap, N_mc=nmc))
    for kind, n, m, p, tgt, count, seed in REFVALS:
        d = po.model_desc(kind, n, m, p, stream=abi.STREAM_REF)
        mean, se = po.ref_reference_value(d, count, seed, target=tgt, threads=8)
        out["reference_values"].append(dict(kind=kind, n=n, m=m, p=p, target=tgt, count=count, seed=seed,
                                            mean=[float(x).hex() for x in mean], se=float(se).hex()))
    with open(os.path.join(HERE, "cli_golden.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", os.path.join(HERE, "cli_golden.json"))


if __name__ == "__main__":
    main()
