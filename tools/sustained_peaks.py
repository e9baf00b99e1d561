"""Run tools/sustained_peaks (>= 4 s FFMA and kind::tf32 MMA loads on every SM) while sampling nvidia-smi clocks and
power, and write profiles/<round>_sustained_peaks.json (bench.py reports its alu / tensor fractions against these
measured sustained rates beside the nominal / derived peaks).   python tools/sustained_peaks.py r2"""
import json
import os
import statistics
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
rnd = sys.argv[1] if len(sys.argv) > 1 else "r2"
binary = os.path.join(HERE, "sustained_peaks")
if not os.path.exists(binary):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", binary,
                           os.path.join(HERE, "sustained_peaks.cu")])
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                        "-lms", "200"], stdout=subprocess.PIPE, text=True)
try:
    out = subprocess.run([binary], capture_output=True, text=True, timeout=300)
finally:
    smi.terminate()
rows = [ln.split(",") for ln in smi.communicate()[0].splitlines() if "," in ln]
clk = [float(r[0]) for r in rows if r[0].strip().replace(".", "").isdigit()]
pw = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
res = json.loads(out.stdout.strip().splitlines()[-1])
res["clocks_during_run"] = {"sm_mhz_median": statistics.median(clk) if clk else None,
                            "sm_mhz_min": min(clk) if clk else None, "power_w_max": max(pw) if pw else None,
                            "samples": len(clk)}
res["how"] = ("tools/sustained_peaks.cu: FFMA 8 independent chains x 148*8 CTAs of 256 threads; tf32 tcgen05.mma "
              "M=128 N=256 K=8 from SMEM, one issuer per SM, 2 accumulators; each run calibrated to > 4 s")
dst = os.path.join(ROOT, "profiles", f"{rnd}_sustained_peaks.json")
json.dump(res, open(dst, "w"), indent=1)
print(json.dumps(res))
