"""Pins for the oracle's adjoint apply (O0*, O8 in oracle/bf_oracle.c; SURVEY 8(f) NEXT-4:
the adjoint K* that Scenario 2 and FIO composition need).

K*(xi_j, x_i) = conj(K(x_i, xi_j)).  The pins tie the adjoint to things fixed independently of its
own code: the dense kernel matrix (brute force), the FFT (the DFT kernel's adjoint is a forward FFT
of the sign-alternated input), the oracle's FORWARD butterfly (assembled densely, its conjugate
transpose must equal the adjoint butterfly assembled densely: a wrong index, a missing conjugate or
a transposed block in the reverse sweep fails it), and the truncation error bound of eqn:BFM
(BF* vs the direct adjoint sum <= eps/2 as for the forward, DESIGN R10).
"""
import numpy as np
import pytest

import oracle
from paper_1803_04128_b200 import workloads as W


def test_direct_adjoint_is_conj_transpose_of_dense_kernel():
    LN = 8
    N = 1 << LN
    F = W.rhs(N, 3, 21).astype(np.complex128)
    for kernel, amp in ((W.K_FIO, W.A_CFG1), (W.K_FIO_JUMP, W.A_CFG3)):
        K = oracle.dense_kernel(kernel, amp, LN)
        rows = np.arange(N)
        g = oracle.direct_adjoint_rows(kernel, amp, LN, F, rows)
        assert np.max(np.abs(g - K.conj().T @ F)) <= 1e-10 * np.max(np.abs(g))


def test_direct_adjoint_dft_closed_form():
    # Phi = x xi, alpha = 1: K*(xi_j, x_i) = e^{-2 pi i i (j - N/2)/N} = (-1)^i e^{-2 pi i ij/N}
    LN = 10
    N = 1 << LN
    F = W.rhs(N, 2, 13).astype(np.complex128)
    want = np.fft.fft(F * ((-1.0) ** np.arange(N))[:, None], axis=0)
    rows = W.sample_rows(N, 13, 64)
    g = oracle.direct_adjoint_rows(W.K_DFT, W.A_ONE, LN, F, rows)
    assert oracle.rel_l2(g, want[rows]) <= 1e-12


@pytest.mark.parametrize("r,tol", [(10, 1e-7), (12, 1e-9)])
def test_bf_adjoint_dft_against_fft(r, tol):
    LN = 12
    N = 1 << LN
    F = W.rhs(N, 1, 17).astype(np.complex128)
    want = np.fft.fft(F[:, 0] * (-1.0) ** np.arange(N))
    g = oracle.bf_apply_adjoint(W.K_DFT, W.A_ONE, LN, 4, r, F)[:, 0]
    assert oracle.rel_l2(g, want) <= tol


@pytest.mark.parametrize("kernel,amp,LN,l0,r", [(W.K_FIO, W.A_CFG1, 8, 4, 8),
                                                 (W.K_FIO_JUMP, W.A_CFG3, 8, 3, 6),
                                                 (W.K_FIO, W.A_CFG2, 10, 5, 10)])
def test_bf_adjoint_is_conj_transpose_of_forward_bf(kernel, amp, LN, l0, r):
    # brute force: both operators assembled densely from their action on every unit vector
    N = 1 << LN
    I = np.eye(N, dtype=np.complex128)
    B = oracle.bf_apply(kernel, amp, LN, l0, r, I, vchunk=N)
    Bs = oracle.bf_apply_adjoint(kernel, amp, LN, l0, r, I, vchunk=N)
    assert np.max(np.abs(Bs - B.conj().T)) <= 1e-12 * np.max(np.abs(B))


def test_adjoint_inner_product_identity():
    # <K f, g> = <f, K* g> for the butterfly operators at a size where dense assembly is too big
    w = W.CONFIGS["cfg3"].with_(log2n=12, nrhs=2)
    f = W.rhs(w.n, 2, 31).astype(np.complex128)
    g = W.rhs(w.n, 2, 32).astype(np.complex128)
    Kf = oracle.bf_apply(w.kernel, w.amp, w.log2n, w.log2leaf, w.rank, f)
    Ksg = oracle.bf_apply_adjoint(w.kernel, w.amp, w.log2n, w.log2leaf, w.rank, g)
    lhs = np.sum(np.conj(g) * Kf, axis=0)
    rhs = np.sum(np.conj(Ksg) * f, axis=0)
    assert np.all(np.abs(lhs - rhs) <= 1e-12 * np.abs(lhs).max())


@pytest.mark.parametrize("name,LN", [("cfg1", 10), ("cfg2", 14), ("cfg3", 14), ("cfg4", 14)])
def test_bf_adjoint_vs_direct_within_eps(name, LN):
    # the adjoint of the factorization is as accurate as the factorization: eps^b <= eps/2 (DESIGN R10)
    w = W.CONFIGS[name]
    w = w.with_(log2n=LN, log2leaf=min(w.log2leaf, LN // 2))
    F = W.rhs(w.n, 1, w.seed + 40).astype(np.complex128)
    rows = W.sample_rows(w.n, w.seed)
    gd = oracle.direct_adjoint_rows(w.kernel, w.amp, w.log2n, F, rows)
    gb = oracle.bf_apply_adjoint(w.kernel, w.amp, w.log2n, w.log2leaf, w.rank, F)
    assert oracle.rel_l2(gb[rows], gd) <= w.eps / 2
