"""Static SASS instruction counts per kernel of the built library -> profiles/r02_sass_summary.json
(the mnemonics that show which hardware paths a kernel uses: UTCHMMA / LDTM / UTCBAR = tcgen05 + TMEM,
UBLKCP = bulk (TMA) copies, DMMA / HMMA = mma.sync tensor paths, REDG = L2 reductions).

  python tools/sass_summary.py [lib.so] > profiles/r02_sass_summary.json
"""
import collections
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_1904_00429_b200", "_lib", "libmlsk.so")
WATCH = ["UTCHMMA", "UTCQMMA", "LDTM", "STTM", "UTCBAR", "UTCCP", "UBLKCP", "SYNCS", "DMMA", "HMMA", "REDG", "RED",
         "ATOMG", "MUFU", "DFMA", "DMUL", "DADD", "FFMA", "IMAD.WIDE", "LDGSTS"]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
kern = collections.OrderedDict()
cur = None
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        name = m.group(1)
        f = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip() or name
        mm = re.search(r"\b(k_\w+)", f)
        short = mm.group(1) if mm else f
        cur = kern.setdefault(short, collections.Counter())
        continue
    if cur is None:
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_.]+)", line)
    if not m:
        continue
    op = m.group(1)
    for w in WATCH:
        if op == w or op.startswith(w + "."):
            cur[w] += 1
            break
print(json.dumps({"source": "cuobjdump -sass paper_1904_00429_b200/_lib/libmlsk.so (static instruction counts per "
                            "kernel, all template instantiations of a kernel summed; tools/sass_summary.py)",
                  "kernels": {k: dict(v) for k, v in kern.items() if v}}, indent=1))
