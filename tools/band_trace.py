"""Timeline of the tensor-core band kernel (CTA 0): per job, SM-clock events relative to job 0's start."""
import os
import sys
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_04128_b200 import bf  # noqa: E402
from paper_1803_04128_b200 import workloads as W  # noqa: E402

w = W.CONFIGS["cfg4"].with_(log2n=int(sys.argv[1]) if len(sys.argv) > 1 else 18)
plan = bf.Plan.build_fio(bf.fio_of(w), max_nrhs_chunk=w.nrhs)
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 0     # 0 = composed band (default), 1/2 = level-by-level
if mode:
    plan.set_option(bf.BF_OPT_BAND_COMPOSE, 0)
    plan.set_option(bf.BF_OPT_BAND_PIPELINES, mode)
plan.set_option(bf.BF_OPT_BAND_TRACE_J0, int(sys.argv[3]) if len(sys.argv) > 3 else 0)
F = torch.randn(w.nrhs, w.n, dtype=torch.complex64, device="cuda")
G = torch.empty_like(F)
for _ in range(2):
    plan.apply(F, G, w.nrhs)
torch.cuda.synchronize()
plan.set_timing(True)
plan.apply(F, G, w.nrhs)
torch.cuda.synchronize()
print("kernel ms:", {k: round(v[0], 3) for k, v in plan.timing().items() if v[1]})
plan.set_timing(False)
for _ in range(int(os.environ.get("BT_WARM", "1"))):   # BT_WARM > 1: trace inside a sustained (power-capped) run
    plan.apply(F, G, w.nrhs)
torch.cuda.synchronize()
T = bf.debug_band_trace()   # the last band launch of the apply (second half)
if mode:
    names = ["split0", "split1", "L1iss", "E1beg", "E1end", "L2iss", "E2beg", "E2end", "load", "L1wait", "L2wait", "mmaEnd"]
    t0, ref = T[0, 8], 2
else:
    names = ["rawful", "splbeg", "splend", "mmabeg", "mmaend", "epibeg", "epiend", "ldbeg", "ldend", "wcbeg", "wcend",
             "wfull"]
    t0, ref = T[0, 7], 3
print("job " + " ".join(f"{n:>7s}" for n in names))
for j in range(0, 40):
    print(f"{j:3d} " + " ".join(f"{(T[j, k] - t0) if T[j, k] else -1:7d}" for k in range(12)))
d = np.diff(T[8:40, ref])
print("steady-state clocks per job (MMA issue to MMA issue):", np.median(d), "mean over jobs 1..63:",
      (T[63, ref] - T[1, ref]) / 62.0, "max gap:", np.max(np.diff(T[1:64, ref])))
