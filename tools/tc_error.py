"""Error of the tensor-core path vs the FP32 SIMT path and the oracle (diagnostic, prints a table)."""
import sys
import os
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_1803_04128_b200 import bf  # noqa: E402
from paper_1803_04128_b200 import workloads as W  # noqa: E402


def run(plan, F):
    Ft = torch.from_numpy(np.ascontiguousarray(F.T)).cuda()
    Gt = torch.empty_like(Ft)
    plan.apply(Ft, Gt, F.shape[1])
    torch.cuda.synchronize()
    return np.asfortranarray(Gt.cpu().numpy().T).astype(np.complex128)


for name, w, cols in [("cfg3", W.CONFIGS["cfg3"], [0, 63]),
                      ("cfg4@2^16", W.CONFIGS["cfg4"].with_(log2n=16), [0, 255]),
                      ("cfg4@2^14", W.CONFIGS["cfg4"].with_(log2n=14), [0, 255])]:
    F = W.rhs(w.n, w.nrhs, w.seed)
    plan = bf.Plan.build_fio(bf.fio_of(w), max_nrhs_chunk=w.nrhs)
    tc = plan.info()["tc_classes"]
    Gt = run(plan, F)
    plan.set_tensor_cores(False)
    Gs = run(plan, F)
    plan.destroy()
    R = oracle.bf_apply(w.kernel, w.amp, w.log2n, w.log2leaf, w.rank, F[:, cols])
    et = oracle.rel_l2(Gt[:, cols], R, axis=0)
    es = oracle.rel_l2(Gs[:, cols], R, axis=0)
    d = oracle.rel_l2(Gt, Gs, axis=0)
    print(f"{name:10s} tc={tc} err_tc={et.max():.2e} err_simt={es.max():.2e} max|tc-simt|={d.max():.2e}", flush=True)
