"""Drop-in CLI (paper_1904_00429_b200/cli.py), planner and reference values
against the reference's own outputs (tests/golden/cli_golden.json, made by
tests/golden/make_cli_golden.py from the compiled reference library).

CPU tests: the planner restatement (planner.cpp) on a 288-point grid, the
relative-error semantics, and the CLI's argument errors / exit codes.
GPU tests: `sweep --no-timing` CSVs and `estimate` outputs.  Models whose draw
uses no transcendental (constant-ones, deterministic) are byte-identical; the
paper models draw through the device's log / exp, which may differ from glibc
in the last ulp, so their floating fields are compared at 1e-9 relative and
every integer field (M, L, M^L, N_l, cost units, seeds) exactly.
"""
import io
import json
import math
import os
import re
import sys
from contextlib import redirect_stdout

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "cli_golden.json")))
EXACT_MODELS = ("constant-ones", "deterministic")


def test_planner_matches_reference_grid():
    from paper_1904_00429_b200 import planner
    for g in GOLD["plans"]:
        p = planner.make_plan(g["eps"], g["M"], g["c1"], g["c2"], g["n"])
        assert (p.L, list(p.N), p.n_cap_applied) == (g["L"], g["N"], g["n_cap_applied"]), g
        assert planner.plan_N_mc(g["eps"], g["c2"]) == g["N_mc"], g


def test_planner_rejects_reference_invalid_inputs():
    from paper_1904_00429_b200 import planner
    for bad in [(0.0, 2), (0.5, 2), (0.1, 1)]:  # planner.cpp:20-27
        with pytest.raises(ValueError):
            planner.make_plan(bad[0], bad[1], 1.0, 1.0, 10)
    with pytest.raises(ValueError):
        planner.plan_N_mc(0.1, 0.0)
    with pytest.raises(ValueError):
        planner.plan_L_capped(0.1, 2, 1.0, 0)


def test_relative_error_semantics():
    from paper_1904_00429_b200.cli import relative_error
    assert relative_error(3.0, 2.0) == 0.5
    assert relative_error(0.0, 0.0) == 0.0
    assert relative_error(1.0, 0.0) == math.inf
    assert relative_error(np.zeros((2, 2)), np.zeros((2, 2))) == 0.0
    assert relative_error(np.ones((2, 2)), np.zeros((2, 2))) == math.inf
    assert relative_error(np.array([[3.0, 4.0]]), np.array([[0.0, 0.0]]) + 1.0) == math.sqrt(13.0 / 2.0)


@pytest.mark.parametrize("argv", [
    ["sweep", "--mode", "tensor"],
    ["sweep", "--m-list", "1,2"],
    ["sweep", "--reps", "0"],
    ["sweep", "--n-ref", "0"],
    ["sweep", "--target", "nope"],
    ["sweep", "--mode", "matmul", "--model", "paper-inner"],
    ["estimate", "--mode", "inner", "--model", "paper-matrix"],
    ["estimate", "--target", "nope"],
    ["estimate", "--epsilon", "0.5"],
    ["estimate", "--m", "1"],
    ["bogus"],
])
def test_cli_usage_errors_exit_1(argv, capsys):
    from paper_1904_00429_b200 import cli
    assert cli.main(argv) == cli.EXIT_USAGE


def test_cli_unwritable_output_exits_3(tmp_path):
    from paper_1904_00429_b200 import cli
    assert cli.main(["sweep", "--out", str(tmp_path / "no" / "such" / "dir.csv")]) == cli.EXIT_IO


# ------------------------------------------------------------------ GPU


def _run(argv):
    from paper_1904_00429_b200 import cli
    buf = io.StringIO()
    with redirect_stdout(buf):
        rc = cli.main(argv)
    assert rc == 0
    return buf.getvalue()


def _fields_close(a: str, b: str, rtol: float):
    """Same tokens; numeric tokens equal (integers) or within rtol (floats)."""
    ta, tb = re.split(r"([,\s=()x:]+)", a), re.split(r"([,\s=()x:]+)", b)
    assert len(ta) == len(tb), (a, b)
    for x, y in zip(ta, tb):
        if x == y:
            continue
        fx, fy = float(x), float(y)  # differing tokens must be floats
        assert re.search(r"[.eE]", x) and re.search(r"[.eE]", y), (x, y)
        assert abs(fx - fy) <= rtol * max(abs(fx), abs(fy)), (x, y)


@pytest.mark.gpu
@pytest.mark.parametrize("case", range(len(GOLD["sweep"])))
def test_sweep_csv_matches_reference(gpu, tmp_path, case):
    g = GOLD["sweep"][case]
    a = g["args"]
    out = tmp_path / "sweep.csv"
    _run(["sweep", "--mode", a["mode"], "--model", a["model"], "--target", a["target"], "--m-list",
          ",".join(str(m) for m in a["m_list"]), "--epsilon", str(a["eps"]), "--reps", str(a["reps"]),
          "--n-ref", str(a["n_ref"]), "--seed", str(a["seed"]), "--no-timing", "--out", str(out)])
    got = out.read_bytes().decode()
    if a["model"] in EXACT_MODELS:
        assert got == g["csv"]
    else:
        _fields_close(got, g["csv"], 1e-9)


@pytest.mark.gpu
@pytest.mark.parametrize("case", range(len(GOLD["estimate"])))
def test_estimate_output_matches_reference(gpu, case):
    g = GOLD["estimate"][case]
    a = g["args"]
    got = _run(["estimate", "--mode", a["mode"], "--model", a["model"], "--target", a["target"], "--m", str(a["M"]),
                "--epsilon", str(a["eps"]), "--seed", str(a["seed"])])
    got = re.sub(r"wall_time_s=[0-9.]+", "wall_time_s=0.000", got)
    _fields_close(got, g["text"], 1e-9)


@pytest.mark.gpu
def test_reference_values_match_reference(gpu):
    from paper_1904_00429_b200 import _abi as abi
    for g in GOLD["reference_values"]:
        if g["kind"] == abi.MODEL_PAPER_INNER:
            model = gpu.paper_inner_model()
        elif g["kind"] == abi.MODEL_PAPER_MATRIX:
            model = gpu.paper_matrix_model()
        else:
            model = gpu.deterministic_matrix_model()
        f = {abi.TARGET_F1: gpu.target_f1(), abi.TARGET_F2: gpu.target_f2(),
             abi.TARGET_IDENTITY: gpu.target_identity()}[g["target"]]
        want = np.array([float.fromhex(x) for x in g["mean"]])
        se_want = float.fromhex(g["se"])
        if isinstance(model, gpu.VectorPairModel):
            r = gpu.reference_inner(model, f, g["count"], g["seed"])
            got = np.array([r.value])
        else:
            r = gpu.reference_matmul(model, f, g["count"], g["seed"])
            got = np.asarray(r.value).ravel()
        if g["kind"] == abi.MODEL_DETERMINISTIC:
            assert np.array_equal(got, want) and r.std_error == se_want
        else:
            np.testing.assert_allclose(got, want, rtol=1e-9, atol=1e-9 * np.abs(want).max())
            assert abs(r.std_error - se_want) <= 1e-7 * max(se_want, 1e-300)
        assert r.count == g["count"]


@pytest.mark.gpu
def test_reference_value_rejects_zero_count(gpu):
    with pytest.raises(ValueError):
        gpu.reference_inner(gpu.paper_inner_model(), gpu.target_f1(), 0, 1)
