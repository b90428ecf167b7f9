"""The device's restatement of glibc's log / sin / cos (paper_1904_00429_b200/
csrc/mlsk_libm.cuh) against the system libm, bit for bit.

The reference's Box-Muller normals, exponentials, paper-model draws and
target f2 call glibc (rng.hpp:55-70, models.cpp:12-52,111-116); on FMA/AVX2
CPUs glibc's ifunc resolvers pick __log_fma / __sin_fma / __cos_fma.  The
header compiles for the host too, so here it is compiled with g++ and
compared with the libm this process would call, over millions of arguments
in every branch (Taylor, table, pi/2-reduced ranges; log near 1, generic,
subnormal).  The GPU tests then compare the device's draws with the oracle's
(glibc) ones."""
import hashlib
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBM = "/lib/x86_64-linux-gnu/libm.so.6"
GLIBC_239_SHA = "3c24a53ee35c2ce0c67240e62bff699c4bddcd7cf8993d5d7ad29157ba072c99"


def _cpu_has_fma():
    try:
        flags = open("/proc/cpuinfo").read()
    except OSError:
        return False
    return " fma " in flags and " avx2 " in flags


def _libm_sha():
    try:
        return hashlib.sha256(open(LIBM, "rb").read()).hexdigest()
    except OSError:
        return None


needs_glibc = pytest.mark.skipif(_libm_sha() != GLIBC_239_SHA or not _cpu_has_fma(),
                                 reason="restatement is of the FMA build of Ubuntu glibc 2.39-0ubuntu8.5")


@pytest.fixture(scope="module")
def checker(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("libm") / "libm_check")
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-o", exe,
                    os.path.join(ROOT, "tests", "native", "libm_check.cpp"), "-lm"], check=True)
    return exe


@needs_glibc
@pytest.mark.parametrize("seed", [1, 20260823])
def test_restatement_bitexact_vs_glibc(checker, seed):
    out = subprocess.run([checker, "1000000", str(seed)], capture_output=True, text=True)
    rows = [line.split() for line in out.stdout.strip().splitlines()]
    assert len(rows) == 16, out.stdout + out.stderr
    bad = [r for r in rows if int(r[2]) != 0]
    assert not bad, bad
    assert out.returncode == 0


@needs_glibc
def test_generated_tables_match_libm(tmp_path):
    """tools/gen_libm_tables.py reproduces the committed header from the libm."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("gen", os.path.join(ROOT, "tools", "gen_libm_tables.py"))
    gen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gen)
    committed = open(gen.OUT).read()
    gen.OUT = str(tmp_path / "t.h")
    gen.main()
    assert open(gen.OUT).read() == committed
