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
# classes by name: the leaf kernels by their names; the bands of an apply follow its S0 in schedule order
# (cfg4: levels (7,8), (9,10 + switch), (11,12), (13,14)); bands before the S0 end the previous apply
names = [s["kernel"] for s in seq]
i0 = next(i for i, n in enumerate(names) if " s0_" in n or n.startswith("void s0_"))
band_order = ["xfer_first_half", "xfer_switch", "xfer_second_half", "xfer_second_half"]
classes, nb = [], 0
for i, n in enumerate(names):
    if "s0_" in n:
        classes.append("s0")
    elif "sl_" in n:
        classes.append("sl")
    elif i > i0:
        classes.append(band_order[nb]); nb += 1
    else:
        classes.append("xfer_second_half")
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
