"""The library's Algorithm 6 (bf_nufft_decide, host C++, no GPU) against the oracle's (oracle/nufft.py) and the
closed forms: the same decisions (y = 0 on the whole FIO matrix, y = 1 on its xi halves and on the DFT), the same
numerical ranks, and targets t(x) = x -+ c(x) on the halves (the phase factors are exact, so the rank-1 part is)."""
import numpy as np
import pytest

import oracle.nufft as NU
from paper_1803_04128_b200 import bf
from paper_1803_04128_b200 import workloads as W


def _both(kernel, amp, LN, cols, budget, eps=1e-9):
    U1, V1 = NU.phase_factors(kernel, LN, cols)
    U2, V2 = NU.amp_factors(amp, LN, cols)
    yo, no, P, Q, *_ = NU.decide(U1, V1, U2, V2, r=1, r_eps=budget, q=8, eps=eps, rng=np.random.default_rng(0))
    N = 1 << LN
    xi = (np.arange(N) if cols is None else np.asarray(cols)) - N // 2
    yl, nl, t = bf.nufft_decide(U1.T, V1.T, U2.T, V2.T, xi=xi.astype(np.float64), rank_budget=budget, q=8, eps=eps,
                                seed=1)
    return (yo, no), (yl, nl, t)


@pytest.mark.parametrize("kernel", [W.K_FIO, W.K_FIO_JUMP, W.K_FIO_PAPER])
def test_whole_matrix_rejected(kernel):
    (yo, no), (yl, nl, t) = _both(kernel, W.A_CFG1, 10, None, 4)
    assert yo == yl == 0 and nl > 4 and no > 4 and t is None


@pytest.mark.parametrize("kernel,amp", [(W.K_FIO, W.A_CFG1), (W.K_FIO_JUMP, W.A_CFG3), (W.K_FIO, W.A_CFG2),
                                        (W.K_FIO_PAPER, W.A_ONE)])
def test_halves_accepted_with_targets(kernel, amp):
    LN = 12
    N = 1 << LN
    x = np.arange(N) / N
    c = NU._c_of(kernel, x)
    for s, cols in enumerate(NU.halves(LN)):
        (yo, no), (yl, nl, t) = _both(kernel, amp, LN, cols, oracle_n_amp(amp) + 2)
        assert yo == yl == 1 and nl == no <= oracle_n_amp(amp)
        # P q^T = t(x) xi exactly: t = x - c(x) on xi < 0 (|xi| = -xi), x + c(x) on xi >= 0
        ref = x - c if s == 0 else x + c
        assert np.abs(t - ref).max() <= 1e-12


def test_dft_whole_matrix_accepted():
    (yo, no), (yl, nl, t) = _both(W.K_DFT, W.A_CFG1, 10, None, 4)
    assert yo == yl == 1 and nl == no
    assert np.abs(t - np.arange(1024) / 1024).max() <= 1e-12


def test_non_frequency_column_factor_is_type3():
    """A rank-1 phase p(x) q(xi) with q not a multiple of xi needs a type-3 NUFFT: the decision says y = 1 but asking
    for type-2 targets fails with BF_ERR_NOT_SUPPORTED."""
    N = 256
    x = np.arange(N) / N
    xi = np.arange(N) - N / 2.0
    u1, v1 = x[None, :], (xi ** 2 / N)[None, :]
    u2, v2 = np.ones((1, N)), np.ones((1, N))
    y, n, _ = bf.nufft_decide(u1, v1, u2, v2, xi=None, want_targets=False)
    assert y == 1 and n == 1
    with pytest.raises(bf.BFError):
        bf.nufft_decide(u1, v1, u2, v2, xi=xi)


def oracle_n_amp(amp):
    return W.N_AMP[amp]
