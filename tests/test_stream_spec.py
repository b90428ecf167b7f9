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


# ---- the Student-t(3) model (BASELINE config 5) restated from the spec text
# (include/mlsk_stream_spec.h, "student-t means") in plain Python: pins the
# oracle's draw -- and through tests/test_gpu_hierarchy.py the device's -- to
# the written definition, one Philox block per (column, row quad) for the means

_M32 = 0xFFFFFFFF


def _philox(c, key):
    c = [x & _M32 for x in c]
    k0, k1 = key & _M32, key >> 32
    for _ in range(10):
        p0 = 0xD2511F53 * c[0]
        p1 = 0xCD9E8D57 * c[2]
        c = [((p1 >> 32) ^ c[1] ^ k0) & _M32, p1 & _M32, ((p0 >> 32) ^ c[3] ^ k1) & _M32, p0 & _M32]
        k0 = (k0 + 0x9E3779B9) & _M32
        k1 = (k1 + 0xBB67AE85) & _M32
    return c


def _mix(z):
    m = 0xFFFFFFFFFFFFFFFF
    z = (z + 0x9E3779B97F4A7C15) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def _derive(master, a, b):
    m = 0xFFFFFFFFFFFFFFFF
    return _mix(_mix(_mix(master) ^ ((a + 0x9E3779B97F4A7C15) & m)) ^ ((b + 0xBF58476D1CE4E5B9) & m))


def test_student_t_draw_matches_spec_text(oracle):
    from paper_1904_00429_b200 import _abi as abi
    L = oracle.oracle_lib()
    f32 = np.float32
    m, n, p, data_seed = 12, 256, 9, 77
    lo, hi = -0.5, 0.5
    om = oracle.OracleModel(oracle.model_desc(abi.MODEL_STUDENT_T, n=n, m=m, p=p, nu=3.0, mean_lo=lo, mean_hi=hi,
                                              data_seed=data_seed, dtype=abi.F32))
    seed, tag, k, c = 20260823, 3, 41, 16
    idx, a, b = om.draw(seed, tag, k, c)
    key = _derive(seed, tag, k)
    z = [C.c_float() for _ in range(4)]

    def entry(col, row, which):
        r = _philox([col, row, which, 5], key)  # MLSK_CTR_T
        L.orc_box_muller_f(r[0], r[1], C.byref(z[0]), C.byref(z[1]))
        L.orc_box_muller_f(r[2], r[3], C.byref(z[2]), C.byref(z[3]))
        zz = [f32(v.value) for v in z]
        v = (zz[1] * zz[1] + zz[2] * zz[2]) + zz[3] * zz[3]
        t = zz[0] / np.sqrt(v / f32(3.0))
        dkey = _derive(data_seed, 0xD47A, which)
        rd = _philox([col, row >> 2, 0, 6], dkey)  # MLSK_CTR_SMEAN: one block per row quad
        mean = f32(lo) + f32(hi - lo) * (f32(rd[row & 3] >> 8) * f32(2.0 ** -24))
        return float(f32(mean + t))

    for t_ in range(c):
        col = int(idx[t_]) - 1
        for r_ in range(m):
            assert a[r_, t_] == entry(col, r_, 0), (r_, t_)
        for q in range(p):
            assert b[t_, q] == entry(col, q, 1), (t_, q)


def test_gauss_draws_match_spec_text(oracle):
    """fp64 gauss (configs 1-2): one Philox block per (column, row pair),
    z0 / z1 for the even / odd row (B: counter purpose CTR_B); fp32 gauss
    (config 3): one block per (column, row quad), four fp32 normals."""
    from paper_1904_00429_b200 import _abi as abi
    L = oracle.oracle_lib()
    f32 = np.float32
    z0, z1 = C.c_double(), C.c_double()
    zf = [C.c_float() for _ in range(4)]
    seed, tag, k, c = 11, 2, 5, 12
    key = _derive(seed, tag, k)
    for dtype in (abi.F64, abi.F32):
        om = oracle.OracleModel(oracle.model_desc(abi.MODEL_GAUSS_MEAN, n=128, m=10, p=7, sd=0.5, data_seed=3,
                                                  dtype=dtype))
        ma, mb = om.means()
        ma = ma.reshape(10, 128)
        mb = mb.reshape(128, 7)
        idx, a, b = om.draw(seed, tag, k, c)
        for t_ in range(c):
            j = int(idx[t_]) - 1
            for which, rows, out, mean in ((0, 10, a[:, t_], ma[:, j]), (1, 7, b[t_, :], mb[j, :])):
                ctr = 2 + which  # MLSK_CTR_A / MLSK_CTR_B
                for r_ in range(rows):
                    if dtype == abi.F64:
                        blk = _philox([j, r_ >> 1, 0, ctr], key)
                        L.orc_box_muller(blk[0] | (blk[1] << 32), blk[2] | (blk[3] << 32), C.byref(z0), C.byref(z1))
                        zz = z1.value if r_ & 1 else z0.value
                        want = mean[r_] + 0.5 * zz
                    else:
                        blk = _philox([j, r_ >> 2, 0, ctr], key)
                        L.orc_box_muller_f(blk[0], blk[1], C.byref(zf[0]), C.byref(zf[1]))
                        L.orc_box_muller_f(blk[2], blk[3], C.byref(zf[2]), C.byref(zf[3]))
                        want = float(f32(mean[r_]) + f32(0.5) * f32(zf[r_ & 3].value))
                    assert out[r_] == want, (dtype, which, r_, t_)
