"""C-ABI boundary checks that need no GPU: the library loads, exports every
entry point include/mlsk.h declares, and fails loudly (no CPU fallback)
when no device is present."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "mlsk.h")).read()
    return sorted(set(re.findall(r"\b(mlsk_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_symbols()
    for must in ("mlsk_mlmc_inner", "mlsk_mlmc_matmul", "mlsk_mc_inner", "mlsk_mc_matmul",
                 "mlsk_session_create", "mlsk_session_run_round", "mlsk_sketch_matmul", "mlsk_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1904_00429_b200 import _lib
    L = _lib.lib()
    missing = [n for n in declared_symbols() if not hasattr(L, n)]
    assert not missing, missing
    assert L.mlsk_version().decode() == "mlsk-b200 0.1.0"


def test_derive_seed_matches_reference_definition():
    from paper_1904_00429_b200 import _lib
    from paper_1904_00429_b200.mlsketch import RngStream

    def mix(z):
        z = (z + 0x9E3779B97F4A7C15) & (2 ** 64 - 1)
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2 ** 64 - 1)
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2 ** 64 - 1)
        return z ^ (z >> 31)

    for m, a, b in [(1, 0, 0), (20260823, 3, 7), (42, 0xFFFFFFFF, 12)]:
        h = mix(m)
        h = mix(h ^ ((a + 0x9E3779B97F4A7C15) & (2 ** 64 - 1)))
        h = mix(h ^ ((b + 0xBF58476D1CE4E5B9) & (2 ** 64 - 1)))
        assert RngStream.derive_seed(m, a, b) == h
        assert _lib.lib().mlsk_derive_seed(m, a, b) == h  # the C-ABI's host function


def test_no_cpu_fallback_without_device():
    from paper_1904_00429_b200 import _lib, mlsketch as g
    if _lib.lib().mlsk_device_count() > 0:
        pytest.skip("a CUDA device is visible")
    with pytest.raises(_lib.MlskRuntimeError, match="no CUDA device"):
        g.mlmc_inner(g.deterministic_model(2), g.target_identity(), g.LevelPlan(2, 1, [4, 4]), 1)
    with pytest.raises(_lib.MlskRuntimeError):
        g.sketch_inner([1, 2], [3, 4], [1])


def test_invalid_arguments_map_to_value_error_before_device_use():
    from paper_1904_00429_b200 import mlsketch as g
    with pytest.raises(ValueError):
        g.mlmc_inner(g.deterministic_model(2), g.target_identity(), g.LevelPlan(2, 2, [10, 10]), 1)
    with pytest.raises(ValueError):
        g.target_f2(-1.0)
    with pytest.raises(ValueError):
        g.constant_ones_model(0)


def _build_cpp_example(tmp_path):
    import subprocess
    lib = os.path.join(ROOT, "paper_1904_00429_b200", "_lib")
    exe = str(tmp_path / "cppex")
    subprocess.run(["g++", "-std=c++17", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "cpp_reference_api.cpp"), "-L" + lib, "-lmlsk",
                    "-Wl,-rpath," + lib, "-o", exe], check=True)
    return exe


def test_cpp_wrapper_restores_reference_signatures(tmp_path):
    """include/mlsk.hpp compiles against the ABI; without a device the call
    fails loudly (std::runtime_error -> exit 3, the CLI's runtime code)."""
    import subprocess
    from paper_1904_00429_b200 import _lib
    exe = _build_cpp_example(tmp_path)
    if _lib.lib().mlsk_device_count() > 0:
        pytest.skip("a CUDA device is visible (tests/test_gpu_* run the example)")
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 3 and "no CUDA device" in r.stdout


@pytest.mark.gpu
def test_cpp_wrapper_on_device(tmp_path):
    import subprocess
    exe = _build_cpp_example(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout
    assert r.stdout.startswith("value 37.0 level1 0.0")
    assert "reference 19.0 22.0 43.0 50.0 se 0.0" in r.stdout
    assert "deterministic 1 vs 2 devices identical 1" in r.stdout
    assert "resume identical 1" in r.stdout
