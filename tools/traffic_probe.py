"""DRAM traffic of a whole bench step, per kernel, for every configuration
(the `traffic` / `step_traffic` fields of bench.py's per-config blocks).

Runs two rounds of the configuration's bench step (the session bench.py's
per-config block builds: same model, seed, stream and level mix) under

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
      --clock-control none -k regex:<the step's kernels>

and writes, per configuration, the DRAM bytes per launch of each kernel and
per step, next to the step's algorithmic bytes (config 1
16 c_l, config 3 (m + p) 4 c_l, config 4 (D + 1) 4 c_l, config 5 0 per
level-sample).  ncu serialises the launches and flushes the caches before
each one, so the bytes are an upper bound of what the pipelined step moves.

  python tools/traffic_probe.py [--configs 1,3,4,5] [--out profiles/tc_traffic.json]
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

KERNELS = "k_gemm_tf32x3|k_gen_panels|k_reduce_tiles_tc|k_mirror_lower|k_kpar_combine|k_sum_sq|" \
          "k_fused_inner|k_reduce_inner|k_expand_ks|k_mk_"
METRICS = "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "us": 1.0,
         "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def short(name):
    return name.split("(")[0].split("::")[-1].split("<")[0].strip().replace("void ", "")


def parse(path):
    text = open(path).read()
    start = text.find('"ID"')
    per = {}
    launches = {}
    for r in csv.DictReader(io.StringIO(text[start:])):
        k = short(r["Kernel Name"])
        v = float(r["Metric Value"].replace(",", "")) * SCALE.get(r.get("Metric Unit", ""), 1.0)
        per.setdefault(k, {}).setdefault(r["Metric Name"], 0.0)
        per[k][r["Metric Name"]] += v
        launches.setdefault(k, set()).add(r["ID"])
    return {k: {"launches": len(launches[k]), **m} for k, m in per.items()}


def alg_bytes_per_step(cid, c, levels_c):
    per = {1: 16.0, 3: (c["m"] + c["p"]) * 4.0, 4: (64 + 1) * 4.0, 5: 0.0}[cid]
    return per * sum(cl * n for cl, n in zip(levels_c, c["N"]))


def child(cid):
    import torch

    import bench_configs_lib
    from paper_1904_00429_b200 import mlsketch as g
    c = bench_configs_lib.configs(g)[cid]
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    opts = g.EstimatorOptions(device=0, stream=stream.cuda_stream, engine="fused")
    sess = g.MlmcSession(c["model"], g.target_identity(), 2, len(c["N"]) - 1, bench_configs_lib.MASTER, c0=c["c0"],
                         options=opts)
    for _ in range(2):
        sess.run_round(c["N"])
    torch.cuda.synchronize()
    sess.close()


def main():
    if len(sys.argv) == 3 and sys.argv[1] == "--child":
        return child(int(sys.argv[2]))
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,3,4,5")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "tc_traffic.json"))
    ap.add_argument("--logdir", default=os.path.join(ROOT, "gpurun_out", "traffic"))
    a = ap.parse_args()
    os.makedirs(a.logdir, exist_ok=True)
    import bench_configs_lib
    from paper_1904_00429_b200 import mlsketch as g
    cfgs = bench_configs_lib.configs(g)
    out = json.load(open(a.out)) if os.path.exists(a.out) else {}
    for cid in [int(x) for x in a.configs.split(",") if x]:
        c = cfgs[cid]
        log = os.path.join(a.logdir, f"config{cid}.csv")
        cmd = ["ncu", "--metrics", METRICS, "--clock-control", "none", "--csv", "--log-file", log,
               "-k", f"regex:{KERNELS}", sys.executable, os.path.abspath(__file__), "--child", str(cid)]
        r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=3000)
        if r.returncode != 0:
            print(r.stdout[-2000:], r.stderr[-2000:])
            raise SystemExit(f"ncu run of config {cid} failed ({r.returncode})")
        per = parse(log)
        steps = 2
        levels_c = [c["c0"] * 2 ** l for l in range(len(c["N"]))]
        kern = {}
        dram_step = 0.0
        for k, m in sorted(per.items()):
            b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
            kern[k] = {"launches_per_step": m["launches"] / steps,
                       "dram_bytes_per_launch": b / m["launches"],
                       "dram_read_bytes_per_launch": m.get("dram__bytes_read.sum", 0.0) / m["launches"],
                       "dram_write_bytes_per_launch": m.get("dram__bytes_write.sum", 0.0) / m["launches"],
                       "us_per_launch_cold": m.get("gpu__time_duration.sum", 0.0) / m["launches"]}
            dram_step += b / steps
        alg = alg_bytes_per_step(cid, c, levels_c)
        out[str(cid)] = {
            "kernels": kern, "dram_bytes_per_step": dram_step, "algorithmic_bytes_per_step": alg,
            "ratio": dram_step / alg if alg else None,
            "source": f"ncu --metrics {METRICS} --clock-control none over two rounds of the config-{cid} bench "
                      "step (tools/traffic_probe.py; launches serialised, caches flushed before each)"}
        print(cid, json.dumps(out[str(cid)])[:400], flush=True)
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
