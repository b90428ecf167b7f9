"""Report which golden CLI outputs the B200 CLI reproduces byte for byte
(tests/test_cli.py asserts tolerance-level agreement for the paper models)."""
import io
import json
import os
import re
import sys
import tempfile
from contextlib import redirect_stdout

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_00429_b200 import cli  # noqa: E402

G = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "cli_golden.json")))
for g in G["sweep"]:
    a = g["args"]
    with tempfile.NamedTemporaryFile(suffix=".csv") as f:
        cli.main(["sweep", "--mode", a["mode"], "--model", a["model"], "--target", a["target"], "--m-list",
                  ",".join(map(str, a["m_list"])), "--epsilon", str(a["eps"]), "--reps", str(a["reps"]),
                  "--n-ref", str(a["n_ref"]), "--seed", str(a["seed"]), "--no-timing", "--out", f.name])
        got = open(f.name).read()
    print("sweep", a["mode"], a["model"], a["target"], "byte-identical" if got == g["csv"] else "DIFFERS")
for g in G["estimate"]:
    a = g["args"]
    buf = io.StringIO()
    with redirect_stdout(buf):
        cli.main(["estimate", "--mode", a["mode"], "--model", a["model"], "--target", a["target"], "--m", str(a["M"]),
                  "--epsilon", str(a["eps"]), "--seed", str(a["seed"])])
    got = re.sub(r"wall_time_s=[0-9.]+", "wall_time_s=0.000", buf.getvalue())
    print("estimate", a["mode"], a["model"], a["target"], "identical (bar wall time)" if got == g["text"] else "DIFFERS")
