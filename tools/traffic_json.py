"""Turn the ncu single-pass DRAM-traffic CSV of tools/gpu_full.sh (one apply: S0, 4 bands, SL at cfg4) into
profiles/<round>_traffic_cfg4.json, the per-launch `traffic` bench.py reports in its roofline object.

    python tools/traffic_json.py gpurun_out/traffic.csv profiles/r1_traffic_cfg4.json
"""
import csv
import io
import json
import sys
from collections import OrderedDict

src, dst = sys.argv[1], sys.argv[2]
lines = [ln for ln in open(src) if ln.startswith('"')]
rows = list(csv.DictReader(io.StringIO("".join(lines))))
launches = OrderedDict()
for r in rows:
    launches.setdefault(r["ID"], {"kernel": r["Kernel Name"]})[r["Metric Name"]] = float(r["Metric Value"])
seq = list(launches.values())
assert len(seq) == 6, [s["kernel"][:40] for s in seq]
classes = ["s0", "xfer_first_half", "xfer_first_half", "xfer_switch", "xfer_second_half", "xfer_second_half"]
# schedule order at cfg4 (l0 = 6, h = 10, D = 14): S0, bands (7,8), (9,10 + switch), (11,12), (13,14), SL
classes = ["s0", "xfer_first_half", "xfer_switch", "xfer_second_half", "xfer_second_half", "sl"]
out = {"what": "dram__bytes_read.sum + dram__bytes_write.sum per launch, ncu --metrics (single pass, --clock-control "
               "none), tools/gpu_full.sh: `python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e` (cfg4, "
               "N=2^20, 256 RHS)",
       "workload": "cfg4", "bytes_per_launch": {}, "ncu_duration_ns": {}, "kernels": {}}
for c, s in zip(classes, seq):
    b = int(s["dram__bytes_read.sum"] + s["dram__bytes_write.sum"])
    out["bytes_per_launch"].setdefault(c, b)
    out["ncu_duration_ns"].setdefault(c, []).append(int(s["gpu__time_duration.sum"]))
    out["kernels"][c] = s["kernel"].split("(")[0]
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps(out, indent=1))
