"""Timeline of the tensor-core SL kernel (one CTA, 64 consecutive K chunks): SM-clock events per chunk."""
import os
import sys
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_04128_b200 import bf  # noqa: E402
from paper_1803_04128_b200 import workloads as W  # noqa: E402

w = W.CONFIGS["cfg4"].with_(log2n=int(sys.argv[1]) if len(sys.argv) > 1 else 18)
plan = bf.Plan.build_fio(bf.fio_of(w), max_nrhs_chunk=w.nrhs)
plan.set_option(bf.BF_OPT_BAND_TRACE_J0, int(sys.argv[2]) if len(sys.argv) > 2 else 64)
F = torch.randn(w.nrhs, w.n, dtype=torch.complex64, device="cuda")
G = torch.empty_like(F)
for _ in range(2):
    plan.apply(F, G, w.nrhs)
torch.cuda.synchronize()
T = bf.debug_band_trace()   # SL is the last kernel of the apply: its events overwrite the band's
names = ["load", "splitIn", "splitEnd", "mmaGo", "mmaIss", "drain0", "drain1", "-", "-", "waitA", "waitB", "splitGo"]
t0 = T[0, 0]
print("chk " + " ".join(f"{n:>8s}" for n in names))
for j in range(0, 40):
    print(f"{j:3d} " + " ".join(f"{(T[j, k] - t0) if T[j, k] else -1:8d}" for k in range(12)))
print("mean clocks per chunk (mmaIss):", (T[63, 4] - T[1, 4]) / 62.0)
