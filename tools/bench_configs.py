"""Per-configuration throughput of the B200 engines (BASELINE.json configs 1, 3,
4, 5): the same blocks bench.py adds to its JSON line (bench_configs_lib.py),
one JSON line per configuration.

  python tools/bench_configs.py [--configs 1,3,4,5] [--steps 3] [--no-cpu-baseline]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench_configs_lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,3,4,5")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    a = ap.parse_args()
    ids = [int(x) for x in a.configs.split(",") if x]
    out = bench_configs_lib.measure(ids, steps=a.steps, with_cpu=not a.no_cpu_baseline)
    for cid, blk in out.items():
        print(json.dumps({"config": int(cid), **blk}), flush=True)


if __name__ == "__main__":
    main()
