"""Diagnostic (GPU): per-vector-tile errors of the three-level band against the oracle and the two-level bands."""
import sys
import numpy as np
import torch

sys.path.insert(0, ".")
import oracle
from paper_1803_04128_b200 import bf
from paper_1803_04128_b200 import workloads as W


def apply(plan, F):
    Ft = torch.from_numpy(np.ascontiguousarray(F.T)).cuda()
    Gt = torch.empty_like(Ft)
    plan.apply(Ft, Gt, F.shape[1])
    torch.cuda.synchronize()
    return np.asfortranarray(Gt.cpu().numpy().T).astype(np.complex128)


import os
for (r, l0, LN, nrhs, chunk) in [(8, 5, 16, 128, 128), (8, 6, 18, 64, 64), (6, 5, 16, 100, 100)][:int(os.environ.get("NCASE", "3"))]:
    N = 1 << LN
    F = W.rhs(N, nrhs, 90 + r + LN)
    k = bf.fio(W.K_FIO, W.A_CFG1, LN, l0, r)
    cols = sorted({0, 1, 31, 32, nrhs // 2, nrhs - 1})
    R = oracle.bf_apply(W.K_FIO, W.A_CFG1, LN, l0, r, F[:, cols])
    out = {}
    for name, opts in [("band3", {}), ("band2_onchip", {bf.BF_OPT_BAND3: 0}),
                       ("simt", {bf.BF_OPT_TENSOR_CORES: 0})][:int(os.environ.get("NVAR", "4"))]:
        plan = bf.Plan.build_fio(k, max_nrhs_chunk=chunk)
        for o, v in opts.items():
            plan.set_option(o, v)
        G = apply(plan, F)
        G2 = apply(plan, F)
        plan.destroy()
        e = oracle.rel_l2(G[:, cols], R, axis=0)
        print(f"r={r} LN={LN} nrhs={nrhs} {name:18s} repeat_equal={np.array_equal(G, G2)} err per col {cols}:",
              " ".join(f"{x:.1e}" for x in e), flush=True)
        out[name] = G
    if "band2_onchip" not in out:
        continue
    d = np.abs(out["band3"] - out["band2_onchip"]).max(axis=0) / np.abs(out["band2_onchip"]).max(axis=0)
    bad = np.nonzero(d > 1e-5)[0]
    print("  band3 vs band2: columns with rel max diff > 1e-5:", bad[:40], len(bad))
