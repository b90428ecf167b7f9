"""Print the key numbers of a bench.py JSON line (last line of a log)."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r = d.get("roofline") or {}
k = d.get("kernels") or {}
print(f"value {d['value']:.4g} {d['unit']}  ms/step {d['ms_per_step']:.2f}  "
      f"sampled-GEMM {d.get('sampled_gemm_tflops', 0):.2f} TF/s")
if r:
    print(f"roofline gemm achieved {r.get('achieved')} of {r.get('peak')} -> frac {r.get('frac')}")
for name, v in k.items():
    print(f"  {name:16s} {v['launches']:6d} launches  {v['ms']:9.2f} ms")
if d.get("e2e"):
    print("e2e", d["e2e"].get("value"), "clocks", d.get("clocks"))
if d.get("cpu_baseline"):
    print("cpu", d["cpu_baseline"])
