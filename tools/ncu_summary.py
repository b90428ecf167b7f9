"""Summarise ncu reports (--set full) and launch lists into profiles/.

  python tools/ncu_summary.py report.ncu-rep [...]   -> JSON summary per kernel
  python tools/ncu_summary.py --launches launches.csv -> per-kernel share of the step
"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
]


def summarize(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    out = []
    for v in rows[2:]:
        d = {"kernel": v[head.index("Kernel Name")][:120]}
        for m in METRICS:
            if m in head:
                i = head.index(m)
                d[m] = {"value": v[i], "unit": units[i]}
        stalls = {}
        for i, k in enumerate(head):
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
                try:
                    if float(v[i]) > 0:
                        stalls[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v[i])
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1.0
        d["stall_share"] = {k: round(x / tot, 3) for k, x in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]}
        out.append(d)
    return out


def launches(path):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    per = {}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].split("::")[-1].split("<")[0]
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(
            r.get("Metric Unit", "us"), 1.0)
        e = per.setdefault(name, [0, 0.0])
        e[0] += 1
        e[1] += v * scale
    tot = sum(x[1] for x in per.values()) or 1.0
    return {k: {"launches": n, "us": round(t, 1), "share": round(t / tot, 4)}
            for k, (n, t) in sorted(per.items(), key=lambda kv: -kv[1][1])}


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        print(json.dumps(launches(sys.argv[2]), indent=1))
    else:
        print(json.dumps([k for r in sys.argv[1:] for k in summarize(r)], indent=1))
