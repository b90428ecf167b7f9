"""BASELINE configs 1-4 as full adaptive MLMC runs on one GPU: the
standard allocation for the target RMSE, then the achieved error against the
exact product of the means (statistics check of BASELINE.json's north star).

    python tools/run_adaptive.py [--config 2] [--eps-rel 1e-2] [--repeats 1]

Prints one JSON line per run: rounds, N_l, cost, wall time, the estimator's
own RMSE estimate sqrt(sum V_l / N_l) and the achieved relative Frobenius
error vs the exact E[A] E[B].
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_00429_b200 import driver  # noqa: E402
from paper_1904_00429_b200 import mlsketch as g  # noqa: E402

MASTER = 20260823


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4])
    ap.add_argument("--eps-rel", type=float, default=1e-2)
    ap.add_argument("--repeats", type=int, default=1)
    args = ap.parse_args()
    ds = g.RngStream.derive_seed(MASTER, 0xD47A0000 + args.config, 0)
    if args.config == 1:
        model = g.gaussian_mean_model(4096, sd=1.0, mean_lo=0.0, mean_hi=1.0, data_seed=ds)
        M, c0, L = 2, 8, 5
    elif args.config == 2:
        model = g.gaussian_mean_matrix_model(256, 4096, 256, sd=0.5, data_seed=ds)
        M, c0, L = 2, 32, 6
    elif args.config == 3:  # fp32, tcgen05 3xTF32 engine
        model = g.gaussian_mean_matrix_model(1024, 16384, 1024, sd=1.0, data_seed=ds, dtype=1)
        M, c0, L = 2, 64, 8
    else:  # config 4: RFF Gram, error against K_n (the n-feature Gram the sketch estimates)
        model = g.rff_gram_model(4096, 2 ** 16, dim=64, sigma=4.0, data_seed=ds)
        M, c0, L = 2, 128, 9
    gt = g.ground_truth(model)
    if isinstance(gt, tuple):  # RFF: (K_n, exact Gaussian kernel)
        gt = gt[0]
    exact = np.atleast_1d(np.asarray(gt, dtype=np.float64)).ravel()
    norm = float(np.linalg.norm(exact))
    eps = args.eps_rel * norm
    for rep in range(args.repeats):
        seed = g.RngStream.derive_seed(MASTER, 0xAD0, rep)
        sess = g.MlmcSession(model, g.target_identity(), M, L, seed, c0=c0)
        t0 = time.perf_counter()
        r = driver.adaptive_mlmc(sess, M, c0, L, eps=eps, n_pilot=256, max_rounds=12)
        dt = time.perf_counter() - t0
        err = float(np.linalg.norm(np.asarray(r.value).ravel() - exact))
        flops = sum(2.0 * (sess.cells) * c0 * M ** l * n for l, n in enumerate(r.N))
        print(json.dumps({
            "config": args.config, "eps_rel": args.eps_rel, "seed": seed, "rounds": r.rounds, "N": r.N,
            "level_samples": int(sum(r.N)), "cost_units": r.cost_units, "wall_s": dt,
            "sampled_gemm_tflops": flops / dt / 1e12,
            "rmse_estimate_rel": r.rmse_estimate / norm, "achieved_error_rel": err / norm,
            "error_over_rmse": err / r.rmse_estimate if r.rmse_estimate > 0 else None,
            "variances": [float(v) for v in r.stats.variances]}), flush=True)
        sess.close()


if __name__ == "__main__":
    main()
