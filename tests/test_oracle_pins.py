"""Pin the CPU oracle before trusting it (CPU-only).

* Philox4x32-10 against libcudacxx's cuda::std::philox4x32 outputs and the
  C++26 known answer for the 10000th value (tests/golden/philox_kat.json).
* The reference-stream restatement (SplitMix64 derive, mt19937_64, Box-Muller,
  index draws, model draws, per-level estimator sums) bit-for-bit against the
  outputs of the reference library compiled from /root/reference
  (tests/golden/ref_*.json, made by tests/golden/make_golden.py).
* When the compiled reference (oracle/_ref) is available, the same against it
  live on fresh seeds.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from paper_1904_00429_b200 import _abi as abi

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def hexd(values):
    return np.array([float.fromhex(v) for v in values])


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_philox_cxx26_known_answer(oracle):
    kat = load("philox_kat.json")
    assert kat["default_10000th"] == kat["cxx26_default_10000th"] == 1955073260
    # std::philox4x32 output i = block(counter = i // 4, key = (seed, 0))[i % 4]
    def stream(seed, count):
        out = []
        for blk in range((count + 3) // 4):
            out.extend(int(x) for x in oracle.philox([blk, 0, 0, 0], [seed & 0xFFFFFFFF, 0]))
        return out[:count]
    assert stream(20111115, 10000)[-1] == 1955073260
    for s in kat["streams"]:
        assert stream(s["seed"], len(s["out"])) == s["out"], s["seed"]


def test_derive_seed_and_mt19937_64(oracle):
    g = load("ref_streams.json")
    L = oracle.oracle_lib()
    for m, a, b, want in g["derive_seed"]:
        assert L.orc_derive_seed(m, a, b) == want
    for rec in g["u64"]:
        got = oracle.mt64_stream(rec["seed"], len(rec["values"]))
        assert [int(x) for x in got] == rec["values"]


def test_reference_normals_and_indices(oracle):
    import ctypes as C
    g = load("ref_streams.json")
    L = oracle.oracle_lib()
    L.orc_ref_init.argtypes = [C.c_void_p, C.c_uint64]
    L.orc_ref_normal.restype = C.c_double
    L.orc_ref_normal.argtypes = [C.c_void_p]
    L.orc_ref_next_u64.restype = C.c_uint64
    L.orc_ref_next_u64.argtypes = [C.c_void_p]
    state = C.create_string_buffer(312 * 8 + 64)
    for rec in g["normals"]:
        L.orc_ref_init(state, rec["seed"])
        got = np.array([L.orc_ref_normal(state) for _ in rec["values"]])
        np.testing.assert_array_equal(got, hexd(rec["values"]))
    for rec in g["indices"]:
        n = rec["n"]
        cum = np.zeros(n)
        L.orc_uniform_cumulative(n, cum.ctypes.data_as(oracle._f64p))
        L.orc_ref_init(state, rec["seed"])
        got = [int(L.orc_index_from_u64(L.orc_ref_next_u64(state), n, cum.ctypes.data_as(oracle._f64p)))
               for _ in rec["values"]]
        assert got == rec["values"], (rec["seed"], n)


def _desc_from(params, oracle):
    return oracle.model_desc(params["kind"], n=params["n"], m=params["m"], p=params["p"], sd=params["sd"],
                             mean_lo=params["mean_lo"], mean_hi=params["mean_hi"],
                             data_seed=params["data_seed"], stream=params["stream"])


def test_reference_model_draws(oracle):
    for rec in load("ref_draws.json"):
        om = oracle.OracleModel(_desc_from(rec["model"], oracle))
        idx, a, b = om.draw(20260823, rec["tag"], rec["k"], rec["c"])
        assert [int(x) for x in idx] == rec["indices"], rec["case"]
        assert sha(a) == rec["a_sha256"], rec["case"]
        assert sha(b) == rec["b_sha256"], rec["case"]
        np.testing.assert_array_equal(a.ravel()[:16], hexd(rec["a_head"]))


def test_reference_estimates_bit_exact(oracle):
    g = load("ref_estimates.json")
    for rec in g["mlmc"]:
        om = oracle.OracleModel(_desc_from(rec["model"], oracle))
        r = om.mlmc(rec["M"], rec["c0"], rec["N"], rec["seed"], target=rec["target"])
        np.testing.assert_array_equal(r.value, hexd(rec["value"]), err_msg=rec["case"])
        assert sha(r.level_estimate) == rec["level_estimate_sha256"], rec["case"]
        np.testing.assert_array_equal(r.level_mean_sq, hexd(rec["level_mean_sq"]), err_msg=rec["case"])
        assert [int(x) for x in r.cost_units] == rec["cost_units"]
        assert r.total_cost_units == rec["total_cost_units"]
    for rec in g["mc"]:
        om = oracle.OracleModel(_desc_from(rec["model"], oracle))
        r = om.mc(rec["L"], rec["N"], rec["M"], 1, rec["seed"])
        np.testing.assert_array_equal(r.value, hexd(rec["value"]), err_msg=rec["case"])
        assert r.total_cost_units == rec["total_cost_units"]


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj"), reason="reference tree not present")
def test_live_reference_fresh_seeds(oracle):
    """Oracle == compiled reference on seeds the fixtures do not contain."""
    for seed in (1, 777, 2 ** 40 + 3):
        d = oracle.model_desc(abi.MODEL_GAUSS_MEAN, n=256, m=8, p=6, sd=0.5, mean_lo=-1, mean_hi=1,
                              stream=abi.STREAM_REF, data_seed=seed)
        om = oracle.OracleModel(d)
        ma, mb = om.means()
        rd = oracle.model_desc(abi.MODEL_GAUSS_MEAN, n=256, m=8, p=6, sd=0.5, stream=abi.STREAM_REF,
                               mean_a=ma, mean_b=mb)
        r1 = om.mlmc(2, 4, [70, 33, 10], seed)
        r2 = oracle.ref_mlmc(rd, 2, 4, [70, 33, 10], seed, threads=3)
        np.testing.assert_array_equal(r1.level_sum, r2.level_sum)
        np.testing.assert_array_equal(r1.level_sumsq, r2.level_sumsq)
        # the composed c0 loop equals the reference's own mlmc_matmul at c0 = 1
        r3 = oracle.ref_mlmc(rd, 3, 1, [20, 9, 4], seed, native=True, threads=2)
        r4 = om.mlmc(3, 1, [20, 9, 4], seed)
        np.testing.assert_array_equal(r3.level_estimate, r4.level_estimate)
        np.testing.assert_array_equal(r3.level_mean_sq, r4.level_mean_sq)
