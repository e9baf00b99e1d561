"""GPU parity of the small-batch transfer bands (bf_small.cu: 8 <= nv < 128 vectors, nv % 8 == 0) -- the
path of cfg2 (nv = 32), cfg5 (nv = 16) and cfg4 sharded over 8 GPUs (nv = 64).

Each case is checked (1) against the CPU oracle per RHS column at the north_star bar (relative l2 <= 1e-5),
(2) bitwise against the same plan with the bands off (BF_OPT_SMALL_BATCH = 0: one transfer level per launch,
xfer_kernel), which performs every complex MAC in the same FP32 order, and (3) for the launch count the
plan reports (two levels per launch).
"""
import numpy as np
import pytest

import oracle
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


def _apply(plan, F):
    Ft = torch.from_numpy(np.ascontiguousarray(F.T)).cuda()
    Gt = torch.empty_like(Ft)
    plan.apply(Ft, Gt, F.shape[1])
    torch.cuda.synchronize()
    return np.asfortranarray(Gt.cpu().numpy().T)


SMALL = [
    # kernel, amp, LN, l0, r, nrhs, oracle columns          what it exercises
    (W.K_FIO, W.A_CFG1, 16, 6, 10, 8, [0, 7]),              # cfg5 shape (nv 16, 1 pass of 2 vectors per lane)
    (W.K_FIO, W.A_CFG2, 16, 5, 10, 16, [0, 15]),            # cfg2 itself (nv 32, levels 6-8 | 9-11: K = 2 + 1)
    (W.K_FIO, W.A_ONE, 14, 5, 8, 8, None),                  # nv 8 (1 vector per lane), r = 8
    (W.K_FIO, W.A_CFG1, 14, 5, 10, 12, [3]),                # nv 24: 3 passes of 8
    (W.K_FIO_JUMP, W.A_CFG3, 14, 5, 12, 12, [0, 11]),       # n_amp 4, nv 48: 3 passes of 16, r = 12
    (W.K_FIO, W.A_CFG1, 14, 6, 10, 32, [0, 31]),            # nv 64 (cfg4 / 8 GPUs): 2 passes of 32
    (W.K_FIO, W.A_CFG1, 14, 6, 16, 48, [47]),               # nv 96, r = 16
    (W.K_DFT, W.A_CFG1, 14, 5, 6, 4, None),                 # r = 6, DFT kernel
    (W.K_FIO, W.A_CFG2, 14, 4, 14, 20, [19]),               # r = 14, leaf 16: 6 levels (K = 2 + 1 per half)
    (W.K_FIO, W.A_CFG1, 12, 4, 10, 4, None),                # h = l0 + 2: one band per half
]


@pytest.mark.parametrize("kernel,amp,LN,l0,r,nrhs,cols", SMALL)
def test_small_batch_parity(kernel, amp, LN, l0, r, nrhs, cols):
    N = 1 << LN
    F = W.rhs(N, nrhs, 600 + LN + r)
    plan = bf.Plan.build_fio(bf.fio(kernel, amp, LN, l0, r), max_nrhs_chunk=nrhs)
    plan.set_tensor_cores(False)          # nv = 64 would otherwise put S0 / SL on the tensor cores
    info = plan.info()
    nx = LN - 2 * l0
    launches = sum(info["class_launches"][k] for k in ("xfer_first_half", "xfer_switch", "xfer_second_half"))
    assert launches == (nx + 1) // 2, info["class_launches"]   # bands of 2 (unsharded: across h too)
    G = _apply(plan, F)
    plan.set_option(bf.BF_OPT_SMALL_BATCH, 0)
    G1 = _apply(plan, F)
    plan.destroy()
    assert np.array_equal(G, G1), "small-batch band == one level per launch, bitwise"
    cols = list(range(nrhs)) if cols is None else cols
    R = oracle.bf_apply(kernel, amp, LN, l0, r, F[:, cols])
    err = oracle.rel_l2(G[:, cols].astype(np.complex128), R, axis=0)
    assert np.all(err <= PARITY), err


def test_small_batch_ragged_chunks_and_fallback():
    """chunks of 40 + 40 + 20 vectors (nrhs 50, chunk 20, n_amp 2): two band chunks and one chunk whose nv is not a
    multiple of 8 (per-level kernels); every column within the bar, batch-consistent with a 1-column apply."""
    k = bf.fio(W.K_FIO, W.A_CFG1, 14, 5, 10)
    F = W.rhs(1 << 14, 50, 77)
    plan = bf.Plan.build_fio(k, max_nrhs_chunk=20)
    plan.set_tensor_cores(False)
    G = _apply(plan, F)
    R = oracle.bf_apply(W.K_FIO, W.A_CFG1, 14, 5, 10, F[:, [0, 25, 49]])
    err = oracle.rel_l2(G[:, [0, 25, 49]].astype(np.complex128), R, axis=0)
    assert np.all(err <= PARITY), err
    p1 = bf.Plan.build_fio(k, max_nrhs_chunk=4)          # nv 8: band kernel with 1 vector per lane
    assert np.array_equal(_apply(p1, np.asfortranarray(F[:, 20:24])), G[:, 20:24])


def test_small_batch_mutation():
    """A wrong block in any transfer level makes parity fail with the small-batch bands (the test can fail)."""
    LN, l0, r = 12, 4, 10
    N = 1 << LN
    k = bf.fio(W.K_FIO, W.A_CFG1, LN, l0, r)
    a, b = bf.build_amp(k)
    v0 = bf.build_blocks(k, bf.BF_STAGE_V0, 0, N)
    xf = [bf.build_blocks(k, bf.BF_STAGE_XFER0 + i, 0, N) for i in range(LN - 2 * l0)]
    sw = bf.build_blocks(k, bf.BF_STAGE_SW, 0, N)
    u = bf.build_blocks(k, bf.BF_STAGE_U, 0, N)
    F = W.rhs(N, 8, 5)
    R = oracle.bf_apply(W.K_FIO, W.A_CFG1, LN, l0, r, F)
    for lvl in range(len(xf)):
        xm = [x.copy() for x in xf]
        xm[lvl][N // 5] *= 1j
        pm = bf.Plan.from_arrays(LN, l0, r, a, b, v0, xm, sw, u, max_nrhs_chunk=8)
        err = oracle.rel_l2(_apply(pm, F).astype(np.complex128), R, axis=0)
        pm.destroy()
        assert np.all(err > 1e-4), (lvl, err)
