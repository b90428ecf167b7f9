"""A-priori level planner: the reference's planner.cpp restated in Python.

Host-side arithmetic only (a few logs and ceilings per plan); it feeds the
drop-in CLI (cli.py) so that `estimate` / `sweep` pick exactly the levels and
replication counts the reference CLI picks.  Python floats are IEEE doubles
and math.log is the C library's log, so every intermediate matches the
reference's (proj/src/planner.cpp).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List

from .mlsketch import LevelPlan

INV_E = 0.36787944117144233  # planner.cpp:11


def _ceil_snapped(x: float) -> int:
    """planner.cpp:15-18: ceiling with a small absolute snap."""
    eps = 1e-9 + 1e-12 * abs(x)
    return int(math.ceil(x - eps))


def _check_plan_inputs(epsilon: float, M: int) -> None:  # planner.cpp:20-27
    if not (epsilon > 0.0) or not (epsilon < INV_E):
        raise ValueError("planner: epsilon must lie in (0, 1/e)")
    if M < 2:
        raise ValueError("planner: M must be at least 2")


def int_pow(M: int, l: int) -> int:  # planner.cpp:31-37
    return int(M) ** int(l)


def plan_L(epsilon: float, M: int, c1: float) -> int:  # planner.cpp:39-48
    _check_plan_inputs(epsilon, M)
    if not (c1 > 0.0):
        raise ValueError("plan_L: c1 must be positive")
    arg = 2.0 * c1 * c1 / (epsilon * epsilon)
    x = math.log(arg) / math.log(float(M))
    L = _ceil_snapped(x)
    return L if L > 0 else 0


def plan_L_capped(epsilon: float, M: int, c1: float, n: int) -> int:  # planner.cpp:50-63
    if n == 0:
        raise ValueError("plan_L_capped: n must be positive")
    base = plan_L(epsilon, M, c1)
    cap, p = 0, 1
    while p < n:  # smallest L with M^L >= n, in integers
        p *= M
        cap += 1
    return base if base > cap else cap


def plan_Nl(epsilon: float, M: int, L: int, c2: float) -> List[int]:  # planner.cpp:65-81
    _check_plan_inputs(epsilon, M)
    if not (c2 > 0.0):
        raise ValueError("plan_Nl: c2 must be positive")
    common = 2.0 * float(L + 1) * c2 / (epsilon * epsilon)
    N = []
    Ml = 1.0
    for _ in range(L + 1):
        v = _ceil_snapped(common / Ml)
        N.append(v if v > 1 else 1)
        Ml *= float(M)
    return N


def plan_N_mc(epsilon: float, c2: float) -> int:  # planner.cpp:83-92
    if not (epsilon > 0.0) or not (epsilon < INV_E):
        raise ValueError("planner: epsilon must lie in (0, 1/e)")
    if not (c2 > 0.0):
        raise ValueError("plan_N_mc: c2 must be positive")
    v = _ceil_snapped(2.0 * c2 / (epsilon * epsilon))
    return v if v > 1 else 1


def make_plan(epsilon: float, M: int, c1: float, c2: float, n: int) -> LevelPlan:  # planner.cpp:94-100
    base = plan_L(epsilon, M, c1)
    L = plan_L_capped(epsilon, M, c1, n)
    return LevelPlan(M, L, plan_Nl(epsilon, M, L, c2), epsilon, c1, c2, L > base)


@dataclass
class CostReport:  # planner.hpp CostReport
    mlmc_cost_units: int
    mc_cost_units: int
    bound: float


def c4_constant(c1: float, c2: float, M: int, md: int) -> float:  # planner.cpp:127-136
    if M < 2 or md == 0 or not (c1 > 0.0) or not (c2 > 0.0):
        raise ValueError("c4_constant: invalid inputs")
    Md = float(M)
    c3 = float(md) * (1.0 + 1.0 / Md)
    c5 = (1.0 + max(0.0, math.log(2.0 * c1 * c1))) / math.log(Md) + 2.0
    return 2.0 * c2 * c3 * c5 * c5 + 2.0 * c3 * c1 * c1 * Md * Md / (Md - 1.0)


def predicted_cost(plan: LevelPlan, N_mc: int, md: int) -> CostReport:  # planner.cpp:102-125
    if md == 0:
        raise ValueError("predicted_cost: md must be positive")
    if len(plan.N) != plan.L + 1:
        raise ValueError("predicted_cost: malformed plan")
    mlmc = 0
    for l in range(plan.L + 1):
        per_rep = int_pow(plan.M, l) + (int_pow(plan.M, l - 1) if l > 0 else 0)
        mlmc += plan.N[l] * per_rep * md
    mc = N_mc * int_pow(plan.M, plan.L) * md
    lg = math.log(plan.epsilon)
    bound = c4_constant(plan.c1, plan.c2, plan.M, md) / (plan.epsilon * plan.epsilon) * lg * lg
    return CostReport(mlmc, mc, bound)
