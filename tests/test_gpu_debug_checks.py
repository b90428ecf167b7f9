"""Device-side invariant checks in place of compute-sanitizer, which is closed
on this GPU pool (profiles/r02_compute_sanitizer_unavailable.txt).

A variant of the CUDA library built with -DMLSK_DEBUG_CHECKS=1 traps on any
violated index / offset invariant (MLSK_DCHECK in mlsk_device.cuh: sampled
index outside [1, n], a panel read outside the batch's samples / K-chunks /
tile grid, a replication run or level part out of range).  Small cases of
every engine (tools/sanitize_cases.py) and a set of parity tests run against
it in subprocesses through MLSK_LIB_PATH and must pass -- the same results
with every check on.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VARIANT = os.path.join(ROOT, "_exp", "libmlsk_debug_checks.so")


@pytest.fixture(scope="module")
def debug_lib():
    src_dir = os.path.join(ROOT, "paper_1904_00429_b200", "csrc")
    newest = max(os.path.getmtime(os.path.join(src_dir, f)) for f in os.listdir(src_dir))
    if not os.path.exists(VARIANT) or os.path.getmtime(VARIANT) < newest:
        subprocess.run([sys.executable, os.path.join(ROOT, "tools", "build_variant.py"), "debug_checks",
                        "-DMLSK_DEBUG_CHECKS=1"], check=True, cwd=ROOT, capture_output=True, timeout=900)
    return VARIANT


@pytest.mark.gpu
def test_every_engine_under_device_checks(debug_lib):
    env = dict(os.environ, MLSK_LIB_PATH=debug_lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py")], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "sanitize cases done" in r.stdout, (r.stdout + r.stderr)[-3000:]
    assert "MLSK_DCHECK failed" not in r.stdout + r.stderr


@pytest.mark.gpu
def test_parity_tests_under_device_checks(debug_lib):
    env = dict(os.environ, MLSK_LIB_PATH=debug_lib)
    tests = ["tests/test_gpu_hierarchy.py", "tests/test_gpu_tc.py", "tests/test_gpu_fused.py", "tests/test_gpu_edge.py",
             "tests/test_gpu_merge.py"]
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "gpu", *tests],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
