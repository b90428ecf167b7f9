"""Drop-in command line: the reference CLI's `estimate` and `sweep` commands
(proj/tools/mlsketch_main.cpp) on the B200 engine, same options and output.

    python -m paper_1904_00429_b200.cli estimate --mode matmul --m 4 --seed 7
    python -m paper_1904_00429_b200.cli sweep --mode inner --m-list 2,3 --no-timing --out sweep.csv

Output formats follow mlsketch_main.cpp:
  * `estimate` (:250-316): a header line, the plan line, the per-level table
    ("level  N  estimate|frob_estimate  mean_sq_diff  cost_units"), then the
    estimate (matrix mode: the value matrix) and cost / time / seed lines;
  * `sweep` (:110-198): CSV "M,L,M_pow_L,RE_mlmc,time_mlmc_s,cost_units_mlmc,
    RE_mc,time_mc_s,cost_units_mc,seed", one row per (M, rep), RE against the
    MC reference value keyed derive_seed(seed, 999983, 0); with --no-timing the
    time columns are 0.000 and the file is byte-identical to the reference's
    (the paper models run on the reference mt19937_64 stream in the exact
    engine, bit-identical per level).
Exit codes (:402-421): 0 ok, 1 usage / invalid argument, 3 I/O or runtime.
`fm-curve` and `oracle` (analysis / enumeration suite) are not on the hot
path and are not provided.
"""
from __future__ import annotations

import argparse
import math
import sys
from typing import List, Optional

import numpy as np

from . import mlsketch as g
from . import planner
from ._lib import MlskRuntimeError

EXIT_OK, EXIT_USAGE, EXIT_IO = 0, 1, 3
REF_TAG = 999983  # mlsketch_main.cpp:26


class UsageError(Exception):
    pass


class IoError(Exception):
    pass


# ------------------------------------------------------------- helpers


def frobenius_norm_sq(x) -> float:
    """tensor.cpp:141-147: sequential sum of squares (no pairwise summation)."""
    s = 0.0
    for v in np.asarray(x, dtype=np.float64).ravel().tolist():
        s += v * v
    return s


def relative_error(estimate, reference) -> float:
    """tensor.cpp:152-174: |e - r| / |r| for scalars, Frobenius ratio for matrices."""
    if np.ndim(reference) == 0:
        e, r = float(estimate), float(reference)
        if r == 0.0:
            return 0.0 if e == 0.0 else math.inf
        return abs(e - r) / abs(r)
    e = np.asarray(estimate, dtype=np.float64).ravel().tolist()
    r = np.asarray(reference, dtype=np.float64).ravel().tolist()
    if len(e) != len(r):
        raise ValueError("relative_error: shape mismatch")
    num = 0.0
    for a, b in zip(e, r):
        d = a - b
        num += d * d
    den = frobenius_norm_sq(r)
    if den == 0.0:
        return 0.0 if num == 0.0 else math.inf
    return math.sqrt(num / den)


class _Out:
    """--out sink; '-' is stdout (mlsketch_main.cpp:37-56)."""

    def __init__(self, path: str):
        self.path = path
        if path == "-":
            self.f = sys.stdout
            self.own = False
        else:
            try:
                self.f = open(path, "w", newline="\n")
            except OSError:
                raise IoError("cannot open output file: " + path)
            self.own = True

    def write(self, s: str) -> None:
        try:
            self.f.write(s)
        except OSError:
            raise IoError("write failure on output stream")

    def close(self) -> None:
        if self.own:
            self.f.close()
        else:
            self.f.flush()


def _model_for(mode: str, key: str):
    if mode == "inner":
        m = g.vector_model_by_key(key)
        if m is None:
            raise UsageError("unknown vector model: " + key)
    else:
        m = g.matrix_model_by_key(key)
        if m is None:
            raise UsageError("unknown matrix model: " + key)
    return m


def _target(key: str):
    t = g.target_by_key(key)
    if t is None:
        raise UsageError("unknown target: " + key)
    return t


def _shape(model):
    return g._shape(model)


# ------------------------------------------------------------- commands


def cmd_estimate(a) -> int:
    """mlsketch_main.cpp:250-316"""
    if a.mode not in ("inner", "matmul"):
        raise UsageError("unknown mode: " + a.mode)
    model_key = a.model or ("paper-inner" if a.mode == "inner" else "paper-matrix")
    target_key = a.target or ("f1" if a.mode == "inner" else "f2")
    f = _target(target_key)
    opts = g.EstimatorOptions(threads=a.threads, device=a.device)
    out = sys.stdout
    out.write("mode=%s model=%s target=%s\n" % (a.mode, model_key, target_key))
    model = _model_for(a.mode, model_key)
    plan = planner.make_plan(a.epsilon, a.m, a.c1, a.c2, model.n)
    cap = " (depth set by dimension cap)" if plan.n_cap_applied else ""
    if a.mode == "inner":
        rep = g.mlmc_inner(model, f, plan, a.seed, opts)
        out.write("M=%d L=%d epsilon=%g n=%d%s\n" % (plan.M, plan.L, plan.epsilon, model.n, cap))
        out.write("level  N          estimate        mean_sq_diff    cost_units\n")
        for st in rep.per_level:
            out.write("%-5d  %-9d  %-14.8g  %-14.8g  %d\n" % (st.level, st.replication_count, st.estimate,
                                                               st.sample_mean_of_squares, st.cost_units))
        out.write("estimate=%.10g\ntotal_cost_units=%d\nwall_time_s=%.3f\nseed=%d\n"
                  % (rep.value, rep.total_cost_units, rep.wall_time_seconds, rep.seed))
    else:
        rep = g.mlmc_matmul(model, f, plan, a.seed, opts)
        rows, cols = _shape(model)
        out.write("M=%d L=%d epsilon=%g n=%d m=%d d=%d%s\n" % (plan.M, plan.L, plan.epsilon, model.n, rows, cols,
                                                               cap))
        out.write("level  N          frob_estimate   mean_sq_diff    cost_units\n")
        for st in rep.per_level:
            out.write("%-5d  %-9d  %-14.8g  %-14.8g  %d\n"
                      % (st.level, st.replication_count, math.sqrt(frobenius_norm_sq(st.estimate)),
                         st.sample_mean_of_squares, st.cost_units))
        v = np.asarray(rep.value).reshape(rows, cols)
        out.write("estimate (%dx%d):\n" % (rows, cols))
        for i in range(rows):
            out.write("".join(("  " if j == 0 else " ") + "%.8g" % v[i, j] for j in range(cols)) + "\n")
        out.write("total_cost_units=%d\nwall_time_s=%.3f\nseed=%d\n"
                  % (rep.total_cost_units, rep.wall_time_seconds, rep.seed))
    out.flush()
    return EXIT_OK


def _sweep_defaults(a) -> None:
    """apply_mode_defaults, mlsketch_main.cpp:80-110"""
    if a.mode not in ("inner", "matmul"):
        raise UsageError("unknown mode: " + a.mode)
    if not a.model:
        a.model = "paper-inner" if a.mode == "inner" else "paper-matrix"
    if not a.target:
        a.target = "f1" if a.mode == "inner" else "f2"
    if not a.m_list:
        a.m_list = list(range(2, 13)) if a.mode == "inner" else [3, 4, 6, 9, 10, 12, 32]
    if any(M < 2 for M in a.m_list):
        raise UsageError("every M must be at least 2")
    if a.reps < 1:
        raise UsageError("--reps must be at least 1")
    if a.threads < 1:
        raise UsageError("--threads must be at least 1")
    if a.n_ref < 1:
        raise UsageError("--n-ref must be at least 1")


def cmd_sweep(a) -> int:
    """mlsketch_main.cpp:112-198"""
    _sweep_defaults(a)
    f = _target(a.target)
    model = _model_for(a.mode, a.model)
    out = _Out(a.out)
    try:
        out.write("M,L,M_pow_L,RE_mlmc,time_mlmc_s,cost_units_mlmc,RE_mc,time_mc_s,cost_units_mc,seed\n")
        ref_seed = g.RngStream.derive_seed(a.seed, REF_TAG, 0)
        opts = g.EstimatorOptions(threads=a.threads, device=a.device)
        inner = a.mode == "inner"
        ref = (g.reference_inner if inner else g.reference_matmul)(model, f, a.n_ref, ref_seed, opts)
        for M in a.m_list:
            plan = planner.make_plan(a.epsilon, M, a.c1, a.c2, model.n)
            N_mc = planner.plan_N_mc(a.epsilon, a.c2)
            for rep in range(a.reps):
                row_seed = g.RngStream.derive_seed(a.seed, M, rep)
                ml = (g.mlmc_inner if inner else g.mlmc_matmul)(
                    model, f, plan, g.RngStream.derive_seed(row_seed, 1, 0), opts)
                mc = (g.mc_inner if inner else g.mc_matmul)(
                    model, f, plan.L, N_mc, M, g.RngStream.derive_seed(row_seed, 2, 0), opts)
                out.write("%d,%d,%d,%s,%s,%d,%s,%s,%d,%d\n" % (
                    M, plan.L, planner.int_pow(M, plan.L),
                    "%.6e" % relative_error(ml.value, ref.value),
                    "%.3f" % (ml.wall_time_seconds if a.timing else 0.0), ml.total_cost_units,
                    "%.6e" % relative_error(mc.value, ref.value),
                    "%.3f" % (mc.wall_time_seconds if a.timing else 0.0), mc.total_cost_units, row_seed))
    finally:
        out.close()
    return EXIT_OK


# ---------------------------------------------------------------- parser


def _m_list(s: str) -> List[int]:
    try:
        return [int(x) for x in s.split(",") if x.strip() != ""]
    except ValueError:
        raise argparse.ArgumentTypeError("comma-separated list of integers expected")


def _config_args(path: str) -> List[str]:
    """--config: flat key=value file (CLI11 config), turned into flags that the
    command line then overrides."""
    out = []
    try:
        lines = open(path).read().splitlines()
    except OSError:
        raise UsageError("cannot read config file: " + path)
    for line in lines:
        line = line.strip()
        if not line or line[0] in "#;[":
            continue
        if "=" not in line:
            raise UsageError("config: expected key=value: " + line)
        k, v = (x.strip() for x in line.split("=", 1))
        v = v.strip("\"'")
        flag = "--" + k.replace("_", "-")
        if v.lower() in ("true", "false") and k in ("timing",):
            out.append(flag if v.lower() == "true" else "--no-" + k)
        else:
            out.extend([flag, v])
    return out


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="mlsketch",
                                 description="Multilevel sketch estimators for inner and matrix products (B200)")
    ap.add_argument("--config", default="", help="flat key=value option file (flags override it)")
    sub = ap.add_subparsers(dest="command", required=True)

    s = sub.add_parser("sweep", help="M-sweep comparing the multilevel estimator to the single-level baseline; "
                                     "writes a CSV")
    s.add_argument("--mode", default="inner")
    s.add_argument("--model", default="")
    s.add_argument("--target", default="")
    s.add_argument("--m-list", type=_m_list, default=None)
    s.add_argument("--epsilon", type=float, default=0.1)
    s.add_argument("--c1", type=float, default=1.0)
    s.add_argument("--c2", type=float, default=1.0)
    s.add_argument("--seed", type=int, default=1)
    s.add_argument("--reps", type=int, default=1)
    s.add_argument("--n-ref", type=int, default=100000)
    s.add_argument("--out", default="-")
    s.add_argument("--threads", type=int, default=1)
    s.add_argument("--device", type=int, default=-1)
    s.add_argument("--timing", dest="timing", action="store_true", default=True)
    s.add_argument("--no-timing", dest="timing", action="store_false")

    e = sub.add_parser("estimate", help="one multilevel estimate with a per-level breakdown")
    e.add_argument("--mode", default="inner")
    e.add_argument("--model", default="")
    e.add_argument("--target", default="")
    e.add_argument("--m", type=int, default=7)
    e.add_argument("--epsilon", type=float, default=0.1)
    e.add_argument("--c1", type=float, default=1.0)
    e.add_argument("--c2", type=float, default=1.0)
    e.add_argument("--seed", type=int, default=1)
    e.add_argument("--threads", type=int, default=1)
    e.add_argument("--device", type=int, default=-1)
    return ap


def main(argv: Optional[List[str]] = None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    ap = build_parser()
    try:
        if "--config" in argv:
            i = argv.index("--config")
            if i + 1 >= len(argv):
                raise UsageError("--config needs a path")
            path = argv[i + 1]
            rest = argv[:i] + argv[i + 2:]
            cmd = next((j for j, x in enumerate(rest) if x in ("sweep", "estimate")), None)
            if cmd is None:
                raise UsageError("a subcommand is required")
            argv = rest[:cmd + 1] + _config_args(path) + rest[cmd + 1:]
    except UsageError as ex:
        sys.stderr.write("error: %s\n" % ex)
        return EXIT_USAGE
    try:
        a = ap.parse_args(argv)
    except SystemExit as ex:
        return EXIT_OK if ex.code == 0 else EXIT_USAGE
    try:
        if a.command == "sweep":
            return cmd_sweep(a)
        return cmd_estimate(a)
    except (UsageError, ValueError) as ex:
        sys.stderr.write("error: %s\n" % ex)
        return EXIT_USAGE
    except (IoError, MlskRuntimeError, OSError) as ex:
        sys.stderr.write("error: %s\n" % ex)
        return EXIT_IO


if __name__ == "__main__":
    sys.exit(main())
