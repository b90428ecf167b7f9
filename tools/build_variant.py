"""Build an experimental variant of the CUDA library with extra -D flags into
_exp/libmlsk_<name>.so (load it with MLSK_LIB_PATH=...; A/B runs on one box).
  python tools/build_variant.py old -DMLSK_TC_STAGES=4 -DMLSK_GEN_TF32_MINB=1"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1904_00429_b200 import build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
os.makedirs(os.path.join(ROOT, "_exp"), exist_ok=True)
out = os.path.join(ROOT, "_exp", f"libmlsk_{name}.so")
cmd = [os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc"), *b.NVCC_FLAGS, *defs, "-o", out, *b.sources()]
print(" ".join(cmd))
subprocess.check_call(cmd)
