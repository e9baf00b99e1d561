"""A few small applies covering every kernel family, for compute-sanitizer (memcheck / racecheck / synccheck):
    compute-sanitizer --tool memcheck python tools/sanitize_cases.py
FP32 SIMT (cfg1 shape, nv = 2), small-batch persistent kernels (nv = 16, 32), tensor-core S0 / composed band /
SL (nv = 128; and nv = 64 with the precomposed band), index-sharded emulated plan with the fused exchange."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1803_04128_b200 import bf  # noqa: E402
from paper_1803_04128_b200 import workloads as W  # noqa: E402


def run(plan, N, nrhs, seed):
    F = W.rhs(N, nrhs, seed)
    Ft = torch.from_numpy(np.ascontiguousarray(F.T)).cuda()
    Gt = torch.empty_like(Ft)
    plan.apply(Ft, Gt, nrhs)
    torch.cuda.synchronize()
    assert torch.isfinite(torch.view_as_real(Gt)).all()
    plan.destroy()


cases = [
    ("cfg1 SIMT nv=2", W.K_FIO, W.A_CFG1, 10, 4, 12, 1, {}),
    ("small batch nv=16", W.K_FIO, W.A_CFG1, 14, 6, 10, 8, {}),
    ("small batch nv=32 leaf 32", W.K_FIO, W.A_CFG2, 14, 5, 10, 16, {}),
    ("tensor cores nv=128", W.K_FIO, W.A_CFG1, 12, 6, 10, 64, {}),
    ("tensor cores nv=64 precomposed", W.K_FIO, W.A_CFG1, 14, 6, 10, 32, {}),
]
for name, k, a, LN, l0, r, nrhs, _ in cases:
    run(bf.Plan.build_fio(bf.fio(k, a, LN, l0, r), max_nrhs_chunk=nrhs), 1 << LN, nrhs, 1)
    print("ok", name, flush=True)
p = bf.Plan.build_fio_emulated(bf.fio(W.K_FIO, W.A_CFG1, 14, 5, 10), 2, max_nrhs_chunk=8)
p.set_option(bf.BF_OPT_EXCHANGE, 1)
run(p, 1 << 14, 8, 2)
print("ok emulated shards, fused exchange", flush=True)
