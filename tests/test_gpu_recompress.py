"""GPU parity of the recompressed butterfly (bf_plan_recompress, DESIGN R21) against
the oracle's recompression (oracle/recompress.py: the same balanced-truncation sweep written with numpy eigh / svd
in FP64 on the oracle's own blocks).  The truncated operator is independent of the Gram square roots each side
picks, so the bar is the north_star's 1e-5 per column; every kernel family runs the rank-8 factors.
"""
import numpy as np
import pytest

import oracle
from oracle import recompress as RC
from paper_1803_04128_b200 import bf
from paper_1803_04128_b200 import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

PARITY = 1e-5


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.init()
    yield


def gpu_apply(plan, F):
    Ft = torch.from_numpy(np.ascontiguousarray(F.T)).cuda()
    Gt = torch.empty_like(Ft)
    plan.apply(Ft, Gt, F.shape[1])
    torch.cuda.synchronize()
    return np.asfortranarray(Gt.cpu().numpy().T)


@pytest.mark.parametrize("kernel,amp,LN,l0,r,rp,nrhs", [
    (W.K_FIO, W.A_CFG1, 12, 5, 12, 8, 4),        # nv = 8: small-batch kernels
    (W.K_FIO, W.A_CFG1, 12, 5, 12, 8, 1),        # nv = 2: tiny kernels
    (W.K_FIO, W.A_CFG1, 14, 5, 12, 8, 64),       # nv = 128: tensor cores at rank 8
    (W.K_FIO_JUMP, W.A_CFG3, 12, 4, 10, 6, 3),   # n_amp 4, odd nrhs, leaf 16, 10 -> 6
    (W.K_FIO, W.A_CFG2, 10, 5, 12, 8, 2),        # h == l0: the switch inside V0
])
def test_recompressed_parity(kernel, amp, LN, l0, r, rp, nrhs):
    F = W.rhs(1 << LN, nrhs, 500 + LN)
    src = bf.Plan.build_fio(bf.fio(kernel, amp, LN, l0, r), max_nrhs_chunk=1)
    plan = src.recompress(rp, max_nrhs_chunk=nrhs)
    src.destroy()
    info = plan.info()
    G = gpu_apply(plan, F)
    plan.destroy()
    assert info["rank"] == rp
    cols = list(range(nrhs)) if nrhs <= 8 else [0, nrhs - 1]
    R = RC.bf_apply_recompressed(kernel, amp, LN, l0, r, rp, F[:, cols].astype(np.complex128))
    err = oracle.rel_l2(G[:, cols].astype(np.complex128), R, axis=0)
    assert np.all(err <= PARITY), (err, info["tc_classes"])


def test_recompressed_cfg4_shape_vs_direct():
    # cfg4's kernel at N = 2^16 with 256 RHS (tensor cores): rank 12 -> 8 within eps/2 of the direct sum plus the
    # 3xTF32 path's own error (~1.5e-6, the same bound as the dense plan's test_parity_config)
    w = W.CONFIGS["cfg4"].with_(log2n=16)
    F = W.rhs(w.n, w.nrhs, 9, cols=[0, 255])
    Fb = np.asfortranarray(np.repeat(F, 128, axis=1))
    src = bf.Plan.build_fio(bf.fio(w.kernel, w.amp, w.log2n, w.log2leaf, 12), max_nrhs_chunk=1)
    plan = src.recompress(8, max_nrhs_chunk=256)
    src.destroy()
    assert "s0" in plan.info()["tc_classes"]
    G = gpu_apply(plan, Fb)
    plan.destroy()
    rows = W.sample_rows(w.n, w.seed)
    gd = oracle.direct_rows(w.kernel, w.amp, w.log2n, F, rows)
    err = oracle.rel_l2(G[rows][:, [0, 255]].astype(np.complex128), gd, axis=0)
    assert np.all(err <= w.eps / 2 + 2e-6), err


def test_recompress_errors():
    k = bf.fio(W.K_FIO, W.A_CFG1, 10, 4, 10)
    src = bf.Plan.build_fio(k, max_nrhs_chunk=1)
    with pytest.raises(bf.BFError):
        src.recompress(12)            # rank above the source's
    st = bf.Plan.build_fio_structured(k, max_nrhs_chunk=1)
    with pytest.raises(bf.BFError):
        st.recompress(8)              # structured plans: not supported
    st.destroy()
    src.destroy()


def test_recompressed_cfg4_full():
    """cfg4 at full size (N = 2^20, 256 RHS) in the bench's launch configuration (rank 12 recompressed to 8, one
    chunk of 256 columns): sampled columns against the direct sum (a property at any size: within eps/2 plus the
    3xTF32 error) and -- with BF_FULL_RECOMPRESS_PARITY=1, ~12 min and ~90 GB of host memory -- against the
    oracle's own recompression of its FP64 blocks (profiles/r2_v3_pytest_recompress_full.txt)."""
    import os
    w = W.CONFIGS["cfg4"]
    F = W.rhs(w.n, w.nrhs, w.seed)
    src = bf.Plan.build_fio(bf.fio(w.kernel, w.amp, w.log2n, w.log2leaf, 12), max_nrhs_chunk=1)
    plan = src.recompress(8, max_nrhs_chunk=w.nrhs)
    src.destroy()
    G = gpu_apply(plan, F)
    plan.destroy()
    cols = [0, 200]
    rows = W.sample_rows(w.n, w.seed)
    gd = oracle.direct_rows(w.kernel, w.amp, w.log2n, F[:, cols], rows)
    assert np.all(oracle.rel_l2(G[rows][:, cols].astype(np.complex128), gd, axis=0) <= w.eps / 2 + 2e-6)
    if os.environ.get("BF_FULL_RECOMPRESS_PARITY") == "1":
        R = RC.bf_apply_recompressed(w.kernel, w.amp, w.log2n, w.log2leaf, 12, 8, F[:, cols].astype(np.complex128))
        err = oracle.rel_l2(G[:, cols].astype(np.complex128), R, axis=0)
        assert np.all(err <= PARITY), err
