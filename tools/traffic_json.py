"""Turn an ncu single-pass DRAM-traffic CSV (tools/gpu_run.sh "traffic:..." step: S0, the bands, SL of one apply)
into profiles/<round>_traffic_<workload>.json, the per-launch `traffic` bench.py reports in its roofline object.

    python tools/traffic_json.py gpurun_out/X_traffic.csv profiles/r2_traffic_cfg4.json cfg4 \
        xfer_first_half,xfer_switch,xfer_second_half,xfer_second_half
"""
import csv
import io
import json
import sys
from collections import OrderedDict

src, dst = sys.argv[1], sys.argv[2]
workload = sys.argv[3] if len(sys.argv) > 3 else "cfg4"
band_order = (sys.argv[4] if len(sys.argv) > 4 else
              "xfer_first_half,xfer_switch,xfer_second_half,xfer_second_half").split(",")
lines = [ln for ln in open(src) if ln.startswith('"')]
rows = list(csv.DictReader(io.StringIO("".join(lines))))
launches = OrderedDict()
for r in rows:
    launches.setdefault(r["ID"], {"kernel": r["Kernel Name"]})[r["Metric Name"]] = float(r["Metric Value"])
seq = [s for s in launches.values() if not s["kernel"].startswith(("expand_", "compose"))]   # plan finalization
names = [s["kernel"] for s in seq]
# one apply: the first S0 launch through the next SL launch; the bands in between follow the schedule order
i0 = next(i for i, n in enumerate(names) if "s0_" in n)
i1 = next(i for i in range(i0, len(names)) if "sl_" in names[i])
seq, names = seq[i0:i1 + 1], names[i0:i1 + 1]
assert len(names) == len(band_order) + 2, names
classes = ["s0"] + band_order + ["sl"]
out = {"what": "dram__bytes_read.sum + dram__bytes_write.sum per launch, ncu --metrics (single pass, --clock-control "
               "none) of `python bench.py --config " + workload + " --steps 1 --warmup 1 --no-cpu-baseline --no-e2e`",
       "workload": workload, "bytes_per_launch": {}, "ncu_duration_ns": {}, "kernels": {}}
for c, s in zip(classes, seq):
    b = int(s["dram__bytes_read.sum"] + s["dram__bytes_write.sum"])
    out["bytes_per_launch"].setdefault(c, b)
    out["ncu_duration_ns"].setdefault(c, []).append(int(s["gpu__time_duration.sum"]))
    out["kernels"][c] = s["kernel"].split("(")[0]
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps(out, indent=1))
