"""The philox-mode transform definition (include/mlsk_stream_spec.h) on the
CPU oracle: accuracy of the table-driven log / sincos and the moments of the
resulting normals and Student-t variates."""
import ctypes as C
import math

import numpy as np


def test_log_and_sincos_accuracy(oracle):
    L = oracle.oracle_lib()
    rng = np.random.default_rng(7)
    xs = np.concatenate([rng.random(20000), 1 - rng.random(500) * 1e-12, [1.0, 2 ** -52, 0.6875, 0.999999]])
    worst = 0.0
    for x in xs[xs > 0]:
        t = math.log(x)
        if t != 0:
            worst = max(worst, abs(L.orc_log_unit(float(x)) - t) / abs(t))
    assert worst < 4e-16
    c, s = C.c_double(), C.c_double()
    err = 0.0
    for u in np.floor(rng.random(20000) * 2 ** 52) / 2 ** 52:
        L.orc_sincos_turn(float(u), C.byref(c), C.byref(s))
        err = max(err, abs(c.value - math.cos(2 * math.pi * u)), abs(s.value - math.sin(2 * math.pi * u)))
    assert err < 2e-15


def test_normal_moments(oracle):
    L = oracle.oracle_lib()
    rng = np.random.default_rng(11)
    z0, z1 = C.c_double(), C.c_double()
    zs = []
    for a, b in rng.integers(0, 2 ** 63, (100000, 2), dtype=np.uint64):
        L.orc_box_muller(int(a) * 2 + 1, int(b) * 2, C.byref(z0), C.byref(z1))
        zs += [z0.value, z1.value]
    z = np.array(zs)
    n = z.size
    assert abs(z.mean()) < 4 / math.sqrt(n)
    assert abs(z.var() - 1) < 4 * math.sqrt(2 / n)
    assert abs((z ** 4).mean() - 3) < 4 * math.sqrt(96 / n)


def test_philox_gauss_model_draw_is_keyed_by_column(oracle):
    """Duplicated indices reuse the same generated column."""
    from paper_1904_00429_b200 import _abi as abi
    om = oracle.OracleModel(oracle.model_desc(abi.MODEL_GAUSS_MEAN, n=8, m=5, p=3, sd=0.5, data_seed=4))
    idx, a, b = om.draw(9, 2, 17, 64)
    for t in range(64):
        for u in range(64):
            if idx[t] == idx[u]:
                np.testing.assert_array_equal(a[:, t], a[:, u])
                np.testing.assert_array_equal(b[t], b[u])
