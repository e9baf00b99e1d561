"""Per-kernel averages (time, DRAM read / write) from an ncu --metrics CSV (gpu__time_duration, dram bytes)."""
import collections
import csv
import io
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.DictReader(io.StringIO("".join(lines))))
L = collections.OrderedDict()
for r in rows:
    L.setdefault(r["ID"], {"k": r["Kernel Name"][:80]})[r["Metric Name"]] = float(r["Metric Value"])
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for v in L.values():
    a = agg[v["k"]]
    a[0] += 1
    a[1] += v.get("gpu__time_duration.sum", 0)
    a[2] += v.get("dram__bytes_read.sum", 0)
    a[3] += v.get("dram__bytes_write.sum", 0)
print(f"{'n':>4} {'ms/launch':>10} {'rd GB':>8} {'wr GB':>8} {'GB/s':>8}  kernel")
for k, a in agg.items():
    t = a[1] / a[0] / 1e9
    print(f"{a[0]:4d} {t * 1e3:10.3f} {a[2] / a[0] / 1e9:8.2f} {a[3] / a[0] / 1e9:8.2f} "
          f"{(a[2] + a[3]) / a[0] / t / 1e9:8.0f}  {k}")
