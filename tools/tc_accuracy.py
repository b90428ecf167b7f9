"""Per-level accuracy of the fused fp32 (3xTF32 tcgen05) engine at the
BASELINE configs' full shapes: one or two level-samples per level, rows /
columns subsets of the level sum against the CPU oracle (fp64 arithmetic on
the same fp32 draws).  Prints one JSON line per (config, level)."""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import pyoracle  # noqa: E402  (test infrastructure: the checker)
from paper_1904_00429_b200 import mlsketch as g  # noqa: E402
import test_gpu_hierarchy as H  # noqa: E402


def models():
    return {
        3: (lambda: g.gaussian_mean_matrix_model(1024, 16384, 1024, sd=1.0, data_seed=H.data_seed(g, 3), dtype=1), 64, 8),
        4: (lambda: g.rff_gram_model(4096, 2 ** 16, dim=64, sigma=4.0, data_seed=H.data_seed(g, 4)), 128, 9),
        5: (lambda: g.student_t_matrix_model(8192, 2 ** 20, 8192, data_seed=H.data_seed(g, 5)), 256, 10),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="3,4,5")
    ap.add_argument("--samples", type=int, default=1)
    ap.add_argument("--rows", type=int, default=32)
    a = ap.parse_args()
    for cfg in [int(x) for x in a.configs.split(",")]:
        mk, c0, L = models()[cfg]
        model = mk()
        dN = [a.samples] * (L + 1)
        t0 = time.time()
        r = H.level_rounds(g, model, c0, L, dN)
        om = pyoracle.OracleModel(model.desc())
        for l, st in enumerate(r.per_level):
            c = c0 * 2 ** l
            rows = H.subset(om.rows, a.rows, 2 * l)
            cols = H.subset(om.cols, a.rows, 2 * l + 1)
            want = sum(om.y_subset(H.MASTER, l, k, c, c // 2 if l > 0 else 0, rows, cols) for k in range(dN[l]))
            got = np.asarray(st.sum, dtype=np.float64)[np.ix_(rows, cols)]
            print(json.dumps({"config": cfg, "level": l, "c": c, "frob_rel": H.frob_rel(got, want),
                              "max_abs_rel": float(np.max(np.abs(got - want)) / np.max(np.abs(want)))}), flush=True)
        print(json.dumps({"config": cfg, "seconds": time.time() - t0}), flush=True)


if __name__ == "__main__":
    main()
