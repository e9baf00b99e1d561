"""One-line summary of a bench.py JSON line on stdin (for gpurun logs)."""
import json
import sys

try:
    d = json.loads(sys.stdin.read())
except Exception as e:  # noqa: BLE001
    print("no JSON line:", e)
    sys.exit(0)
print(f"{d['config']['workload']} n_gpus={d['n_gpus']} value={d['value']:.4g} ms={d['ms_per_step']:.3f} "
      f"e2e={d['e2e']['value'] if d.get('e2e') else None} clocks={d.get('clocks')}")
for k, v in d["kernels"].items():
    if v["launches"]:
        print(f"  {k:18s} n={v['launches']:3d} avg={v['ms_avg']:.4f} ms")
r = d["roofline"]
print(f"  roofline {r['kernel']} {r['bound']} frac={r['frac']:.3f} step lbl={d['step_roofline']['frac_level_by_level']:.3f}")
