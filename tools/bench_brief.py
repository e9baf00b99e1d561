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
for k, v in d.get("kernels", {}).items():
    if v.get("launches"):
        print(f"  {k:18s} n={v['launches']:3d} avg={v['ms_avg']:.4f} ms")
r = d.get("roofline") or {}
lbl = (d.get("step_roofline") or {}).get("frac_level_by_level")
print(f"  roofline {r.get('kernel')} {r.get('bound')} frac={r.get('frac')} step lbl={lbl}")
