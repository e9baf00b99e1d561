"""Top stall instructions of one kernel from an ncu report's source page (SASS view).
    python tools/ncu_source_top.py report.ncu-rep kernel_regex [N]"""
import csv
import io
import subprocess
import sys

rep, rx = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{rx}", "--launch-count", "1"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]
ia, isrc, ist, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), \
    hdr.index("Instructions Executed")
data = [(int(r[ist] or 0), int(r[iex] or 0), r[ia], r[isrc].strip()) for r in rows[1:]
        if len(r) > iex and (r[ist] or "0").isdigit() and (r[iex] or "0").isdigit()]
tot = sum(d[0] for d in data)
totx = sum(d[1] for d in data)
print(f"total stall samples {tot}, instructions executed {totx}")
kinds = {}
for s, x, a, src in data:
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    k = kinds.setdefault(op, [0, 0])
    k[0] += s
    k[1] += x
print("by opcode (samples, executed):")
for op, (s, x) in sorted(kinds.items(), key=lambda kv: -kv[1][0])[:15]:
    print(f"  {op:12s} {s:8d} {100 * s / max(tot, 1):5.1f}%  exec {x:10d} {100 * x / max(totx, 1):5.1f}%")
print("top instructions:")
for s, x, a, src in sorted(data, reverse=True)[:n]:
    print(f"  {s:7d} {x:9d} {a[-5:]} {src[:90]}")
