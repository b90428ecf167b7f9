"""Negative control of the parity harness (the reference's
`mlsketch oracle --inject-rescale-bug`, proj/tools/mlsketch_main.cpp:219-221,
which perturbs the 1/xi rescale by 1 + 1e-6 and must make its oracle fail).

A variant of the CUDA library is built with -DMLSK_INJECT_RESCALE_BUG=1 (every
level-sample rescale n / c scaled by 1 + 1e-6, exact and fused engines) and a
subset of the parity tests is run against it in a subprocess through
MLSK_LIB_PATH: each of them must FAIL.  The same tests pass on the product
build (they are part of this suite), so the tolerances are tight enough to
see a 1e-6 rescale error.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VARIANT = os.path.join(ROOT, "_exp", "libmlsk_rescale_bug.so")

PARITY_TESTS = [
    "tests/test_gpu_exact.py::test_config1_philox_exact_bitexact",
    "tests/test_gpu_exact.py::test_config2_small_philox_bitexact",
    "tests/test_gpu_hierarchy.py::test_config2_all_levels_fused_vs_exact_and_oracle",
]


@pytest.fixture(scope="module")
def bug_lib():
    src_dir = os.path.join(ROOT, "paper_1904_00429_b200", "csrc")
    newest = max(os.path.getmtime(os.path.join(src_dir, f)) for f in os.listdir(src_dir))
    if not os.path.exists(VARIANT) or os.path.getmtime(VARIANT) < newest:
        subprocess.run([sys.executable, os.path.join(ROOT, "tools", "build_variant.py"), "rescale_bug",
                        "-DMLSK_INJECT_RESCALE_BUG=1"], check=True, cwd=ROOT, capture_output=True, timeout=900)
    return VARIANT


@pytest.mark.gpu
@pytest.mark.parametrize("test_id", PARITY_TESTS)
def test_parity_tests_fail_on_injected_rescale_bug(bug_lib, test_id):
    env = dict(os.environ, MLSK_LIB_PATH=bug_lib)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "gpu", test_id],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 1, f"expected the parity test to fail on the perturbed build (rc={r.returncode}):\n{out[-3000:]}"
    assert "1 failed" in out, out[-3000:]
