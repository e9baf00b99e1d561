"""Quick device timing of the NUFFT path at a config's size (diagnostic; bench.py --path nufft is the bench line)."""
import sys
import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1803_04128_b200 import bf
from paper_1803_04128_b200 import workloads as W

LN = int(sys.argv[1]) if len(sys.argv) > 1 else 20
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 256
chunk = int(sys.argv[3]) if len(sys.argv) > 3 else nrhs
N = 1 << LN
plan = bf.NufftPlan.build_fio(bf.fio(W.K_FIO, W.A_CFG1, LN, 1, 2), max_nrhs_chunk=chunk)
print(plan.info())
F = torch.from_numpy(np.ascontiguousarray(W.rhs(N, nrhs, 3).T)).cuda()
G = torch.empty_like(F)
for _ in range(3):
    plan.apply(F, G, nrhs)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    plan.apply(F, G, nrhs)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"N=2^{LN} nrhs={nrhs} chunk={chunk}: {ms:.3f} ms per apply, {N * nrhs / ms * 1e3:.3e} N*RHS/s")
