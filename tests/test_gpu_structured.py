"""GPU parity of the structured interpolative factors (include/bf.h "structured plans";
bf_struct.cu) against the oracle, which regenerates every block of Algorithm 4.1 from its own equation.

A structured plan stores phases and one shared Lagrange matrix per level instead of dense blocks (the grids of
a level are translates); the coefficients between stages differ from the dense plan's by known phase
diagonals, but the operator is the same, so the bar is the same: 1e-5 relative l2 per column (north_star).
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


def gpu_apply(plan, F):
    Ft = torch.from_numpy(np.ascontiguousarray(F.T)).cuda()
    Gt = torch.empty_like(Ft)
    plan.apply(Ft, Gt, F.shape[1])
    torch.cuda.synchronize()
    return np.asfortranarray(Gt.cpu().numpy().T)


CASES = [  # kernel, amp, LN, l0, r, nrhs, chunk          what it exercises
    (W.K_FIO, W.A_CFG1, 16, 6, 10, 8, 8),            # cfg5's shape at reduced N: nv = 16
    (W.K_FIO, W.A_CFG2, 14, 5, 10, 16, 16),          # cfg2's shape: nv = 32
    (W.K_FIO, W.A_CFG1, 10, 4, 12, 1, 1),            # cfg1: nv = 2
    (W.K_FIO_PAPER, W.A_ONE, 12, 4, 8, 3, 3),        # odd nv
    (W.K_FIO, W.A_CFG1, 8, 4, 10, 2, 2),             # h == l0: dense V0 carrying the switch
    (W.K_FIO, W.A_CFG1, 10, 4, 10, 3, 3),            # h == l0 + 1: the only first-half level is the dense one
    (W.K_FIO_JUMP, W.A_CFG3, 14, 5, 12, 5, 4),       # n_amp 4, r 12, ragged chunks (4 + 1)
    (W.K_FIO, W.A_CFG2, 16, 6, 16, 2, 2),            # r = 16
    (W.K_DFT, W.A_CFG1, 14, 6, 6, 7, 7),             # r = 6
    (W.K_FIO, W.A_CFG1, 14, 5, 10, 40, 40),          # nv = 80: small-batch range
    (W.K_FIO, W.A_CFG1, 14, 6, 10, 128, 128),        # nv = 256: tensor cores on dense blocks expanded at finalize
    (W.K_FIO_JUMP, W.A_CFG3, 14, 5, 10, 16, 16),     # nv = 64, n_amp 4: tensor cores, expanded
]


@pytest.mark.parametrize("kernel,amp,LN,l0,r,nrhs,chunk", CASES)
def test_structured_parity(kernel, amp, LN, l0, r, nrhs, chunk):
    N = 1 << LN
    F = W.rhs(N, nrhs, 300 + LN)
    plan = bf.Plan.build_fio_structured(bf.fio(kernel, amp, LN, l0, r), max_nrhs_chunk=chunk)
    info = plan.info()
    G = gpu_apply(plan, F)
    plan.destroy()
    assert info["structured"] == 1
    cols = list(range(nrhs)) if nrhs <= 16 else [0, nrhs // 2, nrhs - 1]
    R = oracle.bf_apply(kernel, amp, LN, l0, r, F[:, cols])
    err = oracle.rel_l2(G[:, cols].astype(np.complex128), R, axis=0)
    assert np.all(err <= PARITY), (err, info["tc_classes"])
    assert np.all(np.isfinite(G))


def test_structured_vs_dense_and_factor_bytes():
    # the same operator as the dense plan (different FP32 rounding order), with ~6x fewer factor bytes
    w = W.CONFIGS["cfg5"].with_(log2n=18)
    k = bf.fio_of(w)
    F = W.rhs(w.n, w.nrhs, 77)
    ps = bf.Plan.build_fio_structured(k, max_nrhs_chunk=w.nrhs)
    pd = bf.Plan.build_fio(k, max_nrhs_chunk=w.nrhs)
    Gs, Gd = gpu_apply(ps, F), gpu_apply(pd, F)
    fs, fd = ps.info()["factor_bytes"], pd.info()["factor_bytes"]
    ps.destroy()
    pd.destroy()
    err = oracle.rel_l2(Gs.astype(np.complex128), Gd.astype(np.complex128), axis=0)
    assert np.all(err <= 2e-6), err
    assert fd / fs > 5.0, (fd, fs)


def test_structured_cfg5_full():
    """cfg5 at full size (N = 2^22, 8 RHS) on structured factors (14.4 GB instead of 110 GB); sampled column."""
    w = W.CONFIGS["cfg5"]
    F = W.rhs(w.n, w.nrhs, w.seed)
    plan = bf.Plan.build_fio_structured(bf.fio_of(w), max_nrhs_chunk=w.nrhs)
    fb = plan.info()["factor_bytes"]
    G = gpu_apply(plan, F)
    plan.destroy()
    assert fb < 15e9, fb
    cols = [5]
    R = oracle.bf_apply(w.kernel, w.amp, w.log2n, w.log2leaf, w.rank, F[:, cols])
    err = oracle.rel_l2(G[:, cols].astype(np.complex128), R, axis=0)
    assert np.all(err <= PARITY), err


def test_structured_bad_descriptor():
    import ctypes

    class D(ctypes.Structure):
        _fields_ = [("abi_version", ctypes.c_int32), ("log2n", ctypes.c_int32), ("log2leaf", ctypes.c_int32),
                    ("rank", ctypes.c_int32), ("n_amp", ctypes.c_int32), ("memory", ctypes.c_int32),
                    ("amp_a", ctypes.c_void_p), ("amp_b", ctypes.c_void_p), ("s0_kind", ctypes.c_int32),
                    ("s0_lag", ctypes.c_void_p), ("s0_data", ctypes.c_void_p), ("xfer", ctypes.c_void_p),
                    ("sl_lag", ctypes.c_void_p), ("sl_phase", ctypes.c_void_p)]
    d = D(bf.BF_ABI_VERSION, 10, 4, 10, 2, bf.BF_MEM_HOST, None, None, 1, None, None, None, None, None)
    h = ctypes.c_void_p()
    st = bf.lib().bf_plan_create_structured(ctypes.byref(d), 0, 1, ctypes.byref(h))
    assert st == 1 and not h.value   # BF_ERR_INVALID_ARG: NULL arrays
    d.s0_kind = 7
    assert bf.lib().bf_plan_create_structured(ctypes.byref(d), 0, 1, ctypes.byref(h)) == 1


@pytest.mark.parametrize("LN,l0,nrhs", [(16, 6, 8), (14, 5, 16), (12, 4, 1)])
def test_structured_band_vs_single_levels(LN, l0, nrhs):
    # the fused two-level structured band (BF_OPT_SMALL_BATCH = 1) against one level per launch: the first- and
    # second-half levels compute in the same FP32 order (bitwise); the dense level h differs in order only
    k = bf.fio(W.K_FIO, W.A_CFG1, LN, l0, 10)
    F = W.rhs(1 << LN, nrhs, 91)
    plan = bf.Plan.build_fio_structured(k, max_nrhs_chunk=nrhs)
    G1 = gpu_apply(plan, F)
    plan.set_option(bf.BF_OPT_SMALL_BATCH, 0)
    G0 = gpu_apply(plan, F)
    plan.destroy()
    err = oracle.rel_l2(G1.astype(np.complex128), G0.astype(np.complex128), axis=0)
    assert np.all(err <= 1e-6), err
