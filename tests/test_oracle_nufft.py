"""Pins of the oracle's NUFFT path (oracle/nufft.py: Alg. 6 + Alg. rlr + eqn:tg3 by definition), all CPU.

What fixes them from outside the module: the C oracle's direct sum O0 (full phase, unsplit amplitude; independent
code), plain numpy SVD truncation, and the paper's statements about which matrices admit the NUFFT (P:551-571:
a rank-1 phase does, the piecewise-smooth FIO kernel only on its submatrices split at xi = 0, eqn:phlr P:1125)."""
import numpy as np
import pytest

import oracle
import oracle.nufft as NU
from paper_1803_04128_b200 import workloads as W


def test_rlr_recovers_low_rank():
    rng = np.random.default_rng(1)
    m, n, r = 300, 240, 5
    A = (rng.standard_normal((m, r)) + 1j * rng.standard_normal((m, r))) @ \
        (rng.standard_normal((r, n)) + 1j * rng.standard_normal((r, n)))
    U0, S0, V0 = NU.rlr(lambda I, J: A[np.ix_(I, J)], m, n, r, 4, rng)
    assert np.linalg.norm(U0 @ np.diag(S0) @ V0.conj().T - A) <= 1e-10 * np.linalg.norm(A)
    assert np.allclose(S0, np.linalg.svd(A, compute_uv=False)[:r], rtol=1e-10)


def test_rlr_truncation_near_svd():
    """Rank-r approximation of a matrix with decaying spectrum: within a small factor of the SVD truncation."""
    rng = np.random.default_rng(2)
    m, n = 256, 200
    X, _ = np.linalg.qr(rng.standard_normal((m, 40)))
    Y, _ = np.linalg.qr(rng.standard_normal((n, 40)))
    A = X @ np.diag(10.0 ** -np.arange(40.0) * 0.5) @ Y.T
    r = 8
    U0, S0, V0 = NU.rlr(lambda I, J: A[np.ix_(I, J)], m, n, r, 4, rng)
    err = np.linalg.norm(U0 @ np.diag(S0) @ V0.conj().T - A, 2)
    best = np.linalg.svd(A, compute_uv=False)[r]
    assert err <= 50 * best, (err, best)


@pytest.mark.parametrize("kernel", [W.K_FIO, W.K_FIO_JUMP])
def test_decision_full_matrix_rejects_fio(kernel):
    """The FIO phase x xi + c(x)|xi| is rank 2 with a non-smooth residual after its rank-1 part: e^{2 pi i residual}
    is not low rank, so Alg. 6 answers y = 0 (use the butterfly) on the whole matrix."""
    LN = 10
    U1, V1 = NU.phase_factors(kernel, LN)
    U2, V2 = NU.amp_factors(W.A_CFG1, LN)
    y, n, *_ = NU.decide(U1, V1, U2, V2, r=1, r_eps=4, q=8, eps=1e-9, rng=np.random.default_rng(0))
    assert y == 0 and n > 4, n


@pytest.mark.parametrize("kernel,amp", [(W.K_FIO, W.A_CFG1), (W.K_FIO_JUMP, W.A_CFG3), (W.K_FIO, W.A_CFG2)])
def test_decision_halves_accept(kernel, amp):
    """On each half (xi < 0, xi >= 0) the phase is exactly rank 1, the residual vanishes and the sample's rank is the
    amplitude's: y = 1 with n = the number of amplitude terms (rank of the amplitude on the half)."""
    LN = 10
    for cols in NU.halves(LN):
        U1, V1 = NU.phase_factors(kernel, LN, cols)
        U2, V2 = NU.amp_factors(amp, LN, cols)
        y, n, P, Q, U, V = NU.decide(U1, V1, U2, V2, r=1, r_eps=U2.shape[1] + 2, q=8, eps=1e-9,
                                     rng=np.random.default_rng(3))
        assert y == 1 and n <= U2.shape[1], n
        ph = U1 @ V1.T
        assert np.abs(P @ Q.T - ph).max() <= 1e-9 * np.abs(ph).max()


def test_decision_dft_accepts_whole_matrix():
    LN = 10
    U1, V1 = NU.phase_factors(W.K_DFT, LN)
    U2, V2 = NU.amp_factors(W.A_CFG1, LN)
    y, n, *_ = NU.decide(U1, V1, U2, V2, r=1, r_eps=4, q=8, eps=1e-9, rng=np.random.default_rng(4))
    assert y == 1 and n <= 2


@pytest.mark.parametrize("kernel,amp,LN", [(W.K_FIO, W.A_CFG1, 10), (W.K_FIO_JUMP, W.A_CFG3, 10),
                                           (W.K_FIO, W.A_CFG2, 12), (W.K_DFT, W.A_CFG1, 10)])
def test_nufft_path_equals_direct_sum(kernel, amp, LN):
    """The whole oracle NUFFT path (decision + rlr factors + eqn:tg3 on both halves) against the C oracle's direct
    sum O0 with the full phase and the unsplit amplitude: the same operator, to rounding."""
    N = 1 << LN
    F = W.rhs(N, 3, 5).astype(np.complex128)
    rows = np.arange(N) if LN <= 10 else W.sample_rows(N, 5)
    g, dec = NU.nufft_path_rows(kernel, amp, LN, F, rows)
    assert all(y == 1 for y, _ in dec)
    gd = oracle.direct_rows(kernel, amp, LN, F, rows)
    assert oracle.rel_l2(g, gd) <= 1e-10
