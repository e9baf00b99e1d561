"""GPU parity of the NUFFT path (include/bf_nufft.h, NEXT-4: eqn:tg3 with one-dimensional type-2 NUFFTs on the
xi < 0 / xi >= 0 submatrices) against the oracle.

The NUFFT computes the operator K itself (not a butterfly of it), so the reference is the oracle's direct sum O0
(full phase, unsplit amplitude) and, at small N, the oracle's own NUFFT path (Alg. 6 decision + rlr + eqn:tg3 by
definition).  Tolerance: the spreading kernel is chosen for eps = 1e-6 (w = 8 points, ES kernel error ~1e-7) and
the device arithmetic is FP32 (cuFFT C2C single, error ~1e-7 sqrt(log N)); the bar is the north_star's 1e-5
relative l2 per RHS column."""
import numpy as np
import pytest

import oracle
import oracle.nufft as NU
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


def _apply(plan, F, nrhs=None):
    nrhs = F.shape[1] if nrhs is None else nrhs
    Ft = torch.from_numpy(np.ascontiguousarray(F.T)).cuda()
    Gt = torch.full_like(Ft, float("nan"))
    plan.apply(Ft, Gt, nrhs)
    torch.cuda.synchronize()
    return np.asfortranarray(Gt.cpu().numpy().T).astype(np.complex128)


CASES = [
    # kernel, amp, LN, nrhs, chunk, rows (None = all)
    (W.K_FIO, W.A_CFG1, 10, 1, 1, None),          # cfg1
    (W.K_DFT, W.A_CFG1, 10, 1, 1, None),          # cfg1 DFT sanity case
    (W.K_FIO, W.A_CFG2, 16, 16, 16, "sample"),    # cfg2 shape
    (W.K_FIO_JUMP, W.A_CFG3, 12, 8, 8, None),     # cfg3 kernel (jump in the amplitude split, R8)
    (W.K_FIO, W.A_CFG1, 12, 5, 2, None),          # ragged chunks 2 + 2 + 1
    (W.K_FIO, W.A_CFG1, 20, 8, 8, "sample"),      # cfg4 size
]


@pytest.mark.parametrize("kernel,amp,LN,nrhs,chunk,rows", CASES)
def test_nufft_parity_direct_sum(kernel, amp, LN, nrhs, chunk, rows):
    N = 1 << LN
    F = W.rhs(N, nrhs, 40 + LN)
    plan = bf.NufftPlan.build_fio(bf.fio(kernel, amp, LN, 1, 2), max_nrhs_chunk=chunk, eps=1e-6)
    info = plan.info()
    assert info["width"] == 8 and info["grid"] == N and info["n"] == N
    G = _apply(plan, F)
    plan.destroy()
    assert np.all(np.isfinite(G))
    r = np.arange(N) if rows is None else W.sample_rows(N, LN)
    R = oracle.direct_rows(kernel, amp, LN, F.astype(np.complex128), r)
    err = oracle.rel_l2(G[r], R, axis=0)
    assert np.all(err <= PARITY), err


def test_nufft_matches_oracle_nufft_path():
    """Against the oracle's Alg. 6 + rlr + eqn:tg3 (the paper's NUFFT path step by step) at N = 2^10."""
    LN = 10
    F = W.rhs(1 << LN, 3, 9)
    plan = bf.NufftPlan.build_fio(bf.fio(W.K_FIO, W.A_CFG1, LN, 1, 2), max_nrhs_chunk=3)
    G = _apply(plan, F)
    plan.destroy()
    R, dec = NU.nufft_path_rows(W.K_FIO, W.A_CFG1, LN, F, np.arange(1 << LN))
    assert [y for y, _ in dec] == [1, 1]
    assert np.all(oracle.rel_l2(G, R, axis=0) <= PARITY)


def test_nufft_generic_plan_one_submatrix():
    """bf_nufft_create with n_sub = 1 and t = x: the DFT kernel over the whole frequency range, one NUFFT."""
    LN = 12
    N = 1 << LN
    a, b = oracle.amp_terms(W.A_CFG1, LN)
    plan = bf.NufftPlan.create(np.arange(N)[None, :] / N, a, b, eps=1e-6, max_nrhs_chunk=4)
    assert plan.info()["grid"] == 2 * N
    F = W.rhs(N, 4, 77)
    G = _apply(plan, F)
    plan.destroy()
    R = oracle.direct_rows(W.K_DFT, W.A_CFG1, LN, F.astype(np.complex128), np.arange(N))
    assert np.all(oracle.rel_l2(G, R, axis=0) <= PARITY)


@pytest.mark.parametrize("eps,bar", [(1e-3, 1e-2), (1e-4, 1e-3), (1e-9, 2e-6)])
def test_nufft_accuracy_follows_eps(eps, bar):
    """The kernel width follows eps (w = ceil(-log10 eps) + 2); the error follows it down to the FP32 floor."""
    LN = 14
    F = W.rhs(1 << LN, 2, 8)
    plan = bf.NufftPlan.build_fio(bf.fio(W.K_FIO, W.A_CFG1, LN, 1, 2), max_nrhs_chunk=2, eps=eps)
    G = _apply(plan, F)
    plan.destroy()
    r = W.sample_rows(1 << LN, 1)
    R = oracle.direct_rows(W.K_FIO, W.A_CFG1, LN, F.astype(np.complex128), r)
    assert np.all(oracle.rel_l2(G[r], R, axis=0) <= bar)


def test_nufft_agrees_with_butterfly_and_invariants():
    """The two paths of the unified framework compute the same K: NUFFT vs the tensor-core butterfly within
    both errors; linearity; column independence; nrhs = 0; determinism; argument errors."""
    LN, nrhs = 14, 64
    N = 1 << LN
    k = bf.fio(W.K_FIO, W.A_CFG1, LN, 6, 10)
    F = W.rhs(N, nrhs, 3)
    nu = bf.NufftPlan.build_fio(k, max_nrhs_chunk=nrhs)
    bp = bf.Plan.build_fio(k, max_nrhs_chunk=nrhs)
    Gn = _apply(nu, F)
    Fb = torch.from_numpy(np.ascontiguousarray(F.T)).cuda()
    Gb = torch.empty_like(Fb)
    bp.apply(Fb, Gb, nrhs)
    torch.cuda.synchronize()
    Gb = np.asfortranarray(Gb.cpu().numpy().T).astype(np.complex128)
    bp.destroy()
    assert np.all(oracle.rel_l2(Gn, Gb, axis=0) <= 1e-5)
    assert np.array_equal(_apply(nu, F), Gn)
    G2 = _apply(nu, (2 * F[:, :4] + 1j * F[:, 4:8]).astype(np.complex64))
    assert oracle.rel_l2(G2, 2 * Gn[:, :4] + 1j * Gn[:, 4:8]) <= 1e-6
    g1 = _apply(nu, np.asfortranarray(F[:, 5:6]))
    assert oracle.rel_l2(g1[:, 0], Gn[:, 5]) <= 1e-6
    Ft = torch.from_numpy(np.ascontiguousarray(F.T)).cuda()
    Gt = torch.full_like(Ft, 7.0)
    nu.apply(Ft, Gt, 0)
    torch.cuda.synchronize()
    assert bool((Gt == 7.0).all())
    with pytest.raises(bf.BFError):
        nu.apply(Ft, Gt, nrhs, ldf=N - 1)
    with pytest.raises(bf.BFError):
        nu.apply(Ft, Ft, nrhs)
    nu.destroy()


def test_nufft_minimum_size_and_alignment():
    """N = 16 (the smallest plan: two submatrices of 8 frequencies) against the direct sum; an odd ldf or a
    misaligned F is refused (the placement reads F in 16-byte pieces)."""
    LN = 4
    N = 1 << LN
    F = W.rhs(N, 3, 6)
    plan = bf.NufftPlan.build_fio(bf.fio(W.K_FIO, W.A_CFG1, LN, 1, 2), max_nrhs_chunk=3)
    G = _apply(plan, F)
    R = oracle.direct_rows(W.K_FIO, W.A_CFG1, LN, F.astype(np.complex128), np.arange(N))
    assert np.all(oracle.rel_l2(G, R, axis=0) <= PARITY)
    Fb = torch.zeros(3 * (N + 1) + 1, dtype=torch.complex64, device="cuda")
    Gb = torch.zeros(3 * N, dtype=torch.complex64, device="cuda")
    with pytest.raises(bf.BFError):
        plan.apply(Fb, Gb, 3, ldf=N + 1)                 # odd ldf
    with pytest.raises(bf.BFError):
        plan.apply(Fb[1:], Gb, 3)                        # F at 8 mod 16 bytes
    plan.destroy()
