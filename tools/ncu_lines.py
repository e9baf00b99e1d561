"""Warp-stall samples and executed instructions per CUDA source line of one kernel (ncu --set full report of a
-lineinfo build, --import-source on):  python tools/ncu_lines.py report.ncu-rep kernel_regex [N]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep, rx = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name",
                      f"regex:{rx}", "--launch-count", "1"], capture_output=True, text=True).stdout
fname, cur, hdr = "?", None, None
samp, execd, src = defaultdict(int), defaultdict(int), {}
for r in csv.reader(out.splitlines()):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 8:
        continue
    if r[0]:   # a source line
        cur = (fname, int(r[0]))
        src[cur] = r[1].strip()
        continue
    if cur is None:
        continue
    try:
        samp[cur] += int(r[4] or 0)
        execd[cur] += int(r[7] or 0)
    except ValueError:
        pass
tot = sum(samp.values()) or 1
print(f"total stall samples {tot}")
for k in sorted(samp, key=lambda k: -samp[k])[:n]:
    print(f"{samp[k]:7d} {100 * samp[k] / tot:5.1f}% exec {execd[k]:11d}  {k[0]}:{k[1]:<5d} {src[k][:90]}")
