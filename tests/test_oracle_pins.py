"""Pins for the CPU oracle (oracle/bf_oracle.c), each against something other than
the oracle itself: values the paper prints, closed forms, textbook/library
special cases, hand-derived values and brute force on tiny inputs.

A plausible mistake anywhere in the oracle (a dropped term, a wrong sign or
index, a transposed operand, the literal garbled grid of eqn:gdA) fails at
least one of these.
"""
import os

import numpy as np
import pytest

import oracle
from paper_1803_04128_b200 import workloads as W

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ----------------------------------------------------------------------------
# Algorithm 2 machinery: grids (eqn:gdA P:214-226), Lagrange basis
# ----------------------------------------------------------------------------
def test_grid_hand_values():
    # DESIGN R2 (ascending z_t) + R3 (round half away): hand evaluation, 1-based.
    assert list(oracle.grid(0, 10, 3) + 1) == [1, 6, 10]
    assert list(oracle.grid(0, 16, 5) + 1) == [1, 4, 9, 13, 16]
    # n = r: the scaling term vanishes -> every index
    assert list(oracle.grid(0, 12, 12)) == list(range(12))
    # shifting ("simply shift the grid points accordingly")
    assert list(oracle.grid(640, 64, 10)) == list(oracle.grid(0, 64, 10) + 640)


@pytest.mark.parametrize("n,r", [(16, 6), (16, 12), (32, 10), (64, 10), (1024, 10), (1 << 20, 12)])
def test_grid_properties(n, r):
    g = oracle.grid(0, n, r)
    assert g[0] == 0 and g[-1] == n - 1                 # end points of the block
    assert np.all(np.diff(g) >= 1)                      # strictly increasing: no repeated points
    # symmetric up to ties: t + (n-r)(z_t+1/2) can be an exact .5 tie in real arithmetic whose side is
    # then decided by the IEEE value of cos (DESIGN R3); both sides of the build evaluate the same expression
    assert np.all(np.abs(g + g[::-1] - (n - 1)) <= 1)
    # Chebyshev clustering towards the ends: the end gaps are the smallest gaps
    d = np.diff(g)
    assert d[0] <= d[len(d) // 2] and d[-1] <= d[len(d) // 2]


def test_lagrange_hand_values():
    w = [oracle.lagrange([1, 5, 9], t, 3.0) for t in range(3)]
    assert np.allclose(w, [0.375, 0.75, -0.125], atol=1e-15)   # S:235, checked by hand


def test_lagrange_textbook_properties():
    g = oracle.grid(0, 64, 10)
    for t in range(10):                                  # node exactness M_t(g_s) = delta_ts
        for s in range(10):
            assert oracle.lagrange(g, t, float(g[s])) == pytest.approx(1.0 if s == t else 0.0, abs=1e-12)
    for q in range(64):                                  # reproduces polynomials of degree < r
        for k in range(4):
            val = sum(oracle.lagrange(g, t, float(q)) * (g[t] / 64.0) ** k for t in range(10))
            assert val == pytest.approx((q / 64.0) ** k, abs=1e-11)


def test_center():
    # "closest to the mean of all indices", ties to the smaller index (DESIGN R4)
    assert oracle.center(0, 4) == 1 and oracle.center(0, 5) == 2 and oracle.center(10, 1) == 10


# ----------------------------------------------------------------------------
# Phase, amplitude and the direct sum O0
# ----------------------------------------------------------------------------
def test_phase_hand_values():
    LN = 10
    N = 1 << LN
    for k in (W.K_FIO, W.K_FIO_PAPER):
        assert oracle.phi(k, LN, 0, N // 2 + 4) == pytest.approx(0.5)     # x=0, xi=4: c(0)|xi| = 4/8 -> K=-1
        assert oracle.phi(k, LN, 123, N // 2) == 0.0                      # column xi = 0 has Phi = 0
    # x = 1/4, xi = 16: x xi = 4; c(1/4) = 3/16 (config) or 2.2/16 (paper)
    assert oracle.phi(W.K_FIO, LN, N // 4, N // 2 + 16) == pytest.approx(7.0)
    assert oracle.phi(W.K_FIO_PAPER, LN, N // 4, N // 2 + 16) == pytest.approx(6.2)
    assert oracle.phi(W.K_DFT, LN, N // 4, N // 2 + 16) == pytest.approx(4.0)
    # cfg3 jump: +0.25 xi for x > 1/3, -0.25 xi for x < 1/3
    assert oracle.phi(W.K_FIO_JUMP, LN, N // 2, N // 2 + 8, True) == pytest.approx(0.5 * 8 + 2.0 / 16 * 8 + 2.0)  # c(1/2) = 2/16
    assert oracle.phi(W.K_FIO_JUMP, LN, 0, N // 2 + 8, True) == pytest.approx(1.0 - 2.0)


def test_direct_sum_dft_closed_form():
    # Phi = x xi: g = sum_k a_k o ((-1)^i N ifft(b_k o f))  (numpy's FFT, not the oracle)
    w = W.CONFIGS["cfg1_dft"]
    N = w.n
    F = W.rhs(N, 2, 7).astype(np.complex128)
    a, b = oracle.amp_terms(w.amp, w.log2n)
    sign = (-1.0) ** np.arange(N)
    ref = np.stack([sum(a[k] * sign * N * np.fft.ifft(b[k] * F[:, c]) for k in range(2)) for c in range(2)], 1)
    g = oracle.direct_rows(w.kernel, w.amp, w.log2n, F, np.arange(N))
    assert oracle.rel_l2(g, ref) < 1e-12


def test_direct_sum_x0_row_closed_form():
    # row x = 0 of the config FIO kernel: Phi = |xi|/8, alpha(0, xi) = 1 + 0.5 cos(pi xi/N)
    LN = 10
    N = 1 << LN
    F = W.rhs(N, 1, 3).astype(np.complex128)[:, 0]
    xi = np.arange(N) - N // 2
    ref = np.sum((1 + 0.5 * np.cos(np.pi * xi / N)) * np.exp(2j * np.pi * np.abs(xi) / 8) * F)
    g = oracle.direct_rows(W.K_FIO, W.A_CFG1, LN, F[:, None], [0])[0, 0]
    assert abs(g - ref) / abs(ref) < 1e-12


def test_amplitude_split_exact():
    # sum_k a_k(x) b_k(xi) = alpha(x, xi) * e^{2 pi i (Phi_full - Phi_bf)}  (DESIGN R8, R11) to 1e-15
    LN = 8
    N = 1 << LN
    rng = np.random.default_rng(0)
    for amp, kernel in ((W.A_CFG1, W.K_FIO), (W.A_CFG2, W.K_FIO), (W.A_CFG3, W.K_FIO_JUMP), (W.A_ONE, W.K_FIO)):
        a, b = oracle.amp_terms(amp, LN)
        K = oracle.dense_kernel(kernel, amp, LN)
        for _ in range(200):
            i, j = rng.integers(0, N, 2)
            # jump factor by hand: 0.25 sign(x - 1/3) xi for cfg3, none otherwise
            phase = 0.25 * (1 if 3 * i > N else -1) * (j - N // 2) if kernel == W.K_FIO_JUMP else 0.0
            lhs = np.sum(a[:, i] * b[:, j]) * np.exp(2j * np.pi * oracle.phi(kernel, LN, i, j, False))
            assert abs(lhs - K[i, j]) < 1e-12
            alpha_hand = {W.A_CFG1: 1 + 0.5 * np.cos(2 * np.pi * i / N) * np.cos(np.pi * (j - N / 2) / N),
                          W.A_CFG2: (1 + 0.3 * np.sin(2 * np.pi * i / N)) * (1 + 0.3 * np.cos(2 * np.pi * (j - N / 2) / N)),
                          W.A_CFG3: np.exp(-(i / N - 0.5) ** 2) * (1 + 0.2 * np.sin(4 * np.pi * (j - N / 2) / N)),
                          W.A_ONE: 1.0}[amp]
            assert abs(np.sum(a[:, i] * b[:, j]) - alpha_hand * np.exp(2j * np.pi * (phase - np.floor(phase)))) < 1e-15 * 4


def test_dense_kernel_hand_values():
    LN = 6
    N = 1 << LN
    K = oracle.dense_kernel(W.K_FIO, W.A_ONE, LN)
    assert np.allclose(np.abs(K), 1.0, atol=1e-14)        # unimodular
    assert np.allclose(K[:, N // 2], 1.0, atol=1e-14)     # column xi = 0
    assert abs(K[0, N // 2 + 4] + 1.0) < 1e-14            # x=0, xi=4 -> -1


# ----------------------------------------------------------------------------
# O1-O7: the butterfly (Algorithm 4.1)
# ----------------------------------------------------------------------------
def _golden_tab():
    rows = []
    with open(os.path.join(GOLDEN, "tab_1d_fio_eps_b.txt")) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                n, r, e = line.split()
                rows.append((int(n), int(r), float(e)))
    return rows


@pytest.mark.parametrize("N,r,eps_paper", _golden_tab())
def test_bf_reproduces_paper_tab_1d_fio(N, r, eps_paper):
    """The paper-printed eps^b of tab:1D-FIO within 2x: kernel eqn:1D-FIO-kernal,
    alpha=1, leaf 16 (DESIGN R1), one random vector, 256 random rows."""
    LN = N.bit_length() - 1
    F = W.rhs(N, 1, 0)
    rows = W.sample_rows(N, 0)
    gd = oracle.direct_rows(W.K_FIO_PAPER, W.A_ONE, LN, F, rows)
    gb = oracle.bf_apply(W.K_FIO_PAPER, W.A_ONE, LN, 4, r, F)
    eps = oracle.rel_l2(gb[rows], gd)
    if N >= 16384 and r == 12:
        # the paper's value is floored by its recovery error eps^K = 2.12e-10; ours may only be lower
        assert eps < 2.0 * eps_paper
    else:
        assert 0.5 * eps_paper < eps < 2.0 * eps_paper


@pytest.mark.parametrize("r,tol", [(10, 3e-8), (12, 2e-10)])
def test_bf_dft_against_fft(r, tol):
    # Phi = x xi reduces the transform to a DFT: compare with numpy's FFT on all rows
    N, LN = 1024, 10
    F = W.rhs(N, 1, 11).astype(np.complex128)
    ref = ((-1.0) ** np.arange(N)) * N * np.fft.ifft(F[:, 0])
    g = oracle.bf_apply(W.K_DFT, W.A_ONE, LN, 4, r, F)[:, 0]
    assert oracle.rel_l2(g, ref) < tol


@pytest.mark.parametrize("LN,l0,r,tol", [(8, 4, 10, 1e-6), (8, 3, 8, 1e-4), (10, 4, 10, 1e-6)])
def test_bf_dense_assembly_brute_force(LN, l0, r, tol):
    """Assemble the butterfly densely (apply to every e_j) and compare with the dense kernel.
    LN=8,l0=4: no transfer level (h = l0); LN=8,l0=3 and LN=10,l0=4: one level per half."""
    N = 1 << LN
    I = np.eye(N, dtype=np.complex128)
    B = oracle.bf_apply(W.K_FIO, W.A_CFG1, LN, l0, r, I, vchunk=N)
    K = oracle.dense_kernel(W.K_FIO, W.A_CFG1, LN)
    assert np.linalg.norm(B - K) / np.linalg.norm(K) < tol


def test_bf_error_monotone_in_r():
    N, LN = 4096, 12
    F = W.rhs(N, 1, 5)
    rows = W.sample_rows(N, 5)
    gd = oracle.direct_rows(W.K_FIO, W.A_CFG1, LN, F, rows)
    errs = [oracle.rel_l2(oracle.bf_apply(W.K_FIO, W.A_CFG1, LN, 5, r, F)[rows], gd) for r in (6, 8, 10, 12, 14)]
    assert all(e2 < e1 for e1, e2 in zip(errs, errs[1:]))


def test_bf_linear_and_zero():
    N, LN = 1024, 10
    F = W.rhs(N, 3, 9).astype(np.complex128)
    G = oracle.bf_apply(W.K_FIO, W.A_CFG2, LN, 4, 10, F)
    assert np.all(oracle.bf_apply(W.K_FIO, W.A_CFG2, LN, 4, 10, np.zeros((N, 1))) == 0)
    Gs = oracle.bf_apply(W.K_FIO, W.A_CFG2, LN, 4, 10, (2 - 1j) * F[:, :1] + 0.5 * F[:, 1:2])
    assert oracle.rel_l2(Gs[:, 0], (2 - 1j) * G[:, 0] + 0.5 * G[:, 1]) < 1e-13
    # columns are independent of the chunking of the vectors
    G2 = oracle.bf_apply(W.K_FIO, W.A_CFG2, LN, 4, 10, F, vchunk=1)
    assert np.array_equal(G, G2)


def test_bf_blocks_interpolate_the_kernel():
    """Complementary low-rank property (eqn:glr P:640-645) in block form: the expansion of
    eqn:1 reproduces u^B(x) = sum_{xi in B} K(x,xi) g(xi) on A, and the switch block of
    P:764-766 is the kernel sampled at the nodes."""
    LN, l0, r = 10, 4, 12
    N, n0 = 1 << LN, 1 << l0
    K = oracle.dense_kernel(W.K_FIO, W.A_ONE, LN)
    g = W.rhs(N, 1, 1).astype(np.complex128)[:, 0]
    a, b = 3, 17
    A = np.arange(a * (N // n0), (a + 1) * (N // n0))
    B = np.arange(b * n0, (b + 1) * n0)
    V = oracle.bf_block(W.K_FIO, LN, l0, r, 0, l0, a, b)
    delta = V @ g[B]
    gB = oracle.grid(B[0], n0, r)
    approx = np.exp(2j * np.pi * np.array([[oracle.phi(W.K_FIO, LN, x, s) for s in gB] for x in A])) @ delta
    exact = K[np.ix_(A, B)] @ g[B]
    assert np.linalg.norm(approx - exact) / np.linalg.norm(exact) < 1e-8
    h = LN // 2
    S = oracle.bf_block(W.K_FIO, LN, l0, r, 2, h, 5, 9)
    gA = oracle.grid(5 * (N >> h), N >> h, r)
    gBh = oracle.grid(9 << h, 1 << h, r)
    assert np.allclose(S, K[np.ix_(gA, gBh)], atol=1e-13)


@pytest.mark.parametrize("name", ["cfg1", "cfg1_dft", "cfg2", "cfg3", "cfg4"])
def test_bf_vs_direct_per_config(name):
    """BF vs the direct sum within eps/2 on the eps^b row sample (DESIGN R10), one RHS."""
    w = W.CONFIGS[name]
    F = W.rhs(w.n, w.nrhs, w.seed, cols=[0])
    rows = W.sample_rows(w.n, w.seed)
    gd = oracle.direct_rows(w.kernel, w.amp, w.log2n, F, rows)
    gb = oracle.bf_apply(w.kernel, w.amp, w.log2n, w.log2leaf, w.rank, F)
    assert oracle.rel_l2(gb[rows], gd) <= w.eps / 2


def test_rhs_generator_column_subset():
    full = W.rhs(256, 5, 3)
    sub = W.rhs(256, 5, 3, cols=[1, 4])
    assert np.array_equal(full[:, [1, 4]], sub)
    assert full.dtype == np.complex64 and full.flags.f_contiguous


@pytest.mark.slow
def test_bf_vs_direct_cfg5():
    """cfg5 (N = 2^22): r = 10 keeps the BF within eps/2 of the direct sum on the eps^b rows (reading R10 at the
    largest N; the survey's probe value was 4.3e-7).  ~100 s on 8 cores."""
    w = W.CONFIGS["cfg5"]
    F = W.rhs(w.n, w.nrhs, w.seed, cols=[0])
    rows = W.sample_rows(w.n, w.seed)
    gd = oracle.direct_rows(w.kernel, w.amp, w.log2n, F, rows)
    gb = oracle.bf_apply(w.kernel, w.amp, w.log2n, w.log2leaf, w.rank, F)
    assert oracle.rel_l2(gb[rows], gd) <= w.eps / 2


def _stored_inputs(kernel, amp, LN, l0, r, dtype=np.complex128):
    a, b = oracle.amp_terms(amp, LN)
    v0 = oracle.bf_blocks(kernel, LN, l0, r, 0).astype(dtype)
    xf = [oracle.bf_blocks(kernel, LN, l0, r, 1, l).astype(dtype) for l in range(l0 + 1, LN - l0 + 1)]
    sw = oracle.bf_blocks(kernel, LN, l0, r, 2).astype(dtype)
    u = oracle.bf_blocks(kernel, LN, l0, r, 3).astype(dtype)
    return a, b, v0, xf, sw, u


@pytest.mark.parametrize("kernel,amp,LN,l0,r", [(W.K_FIO, W.A_CFG1, 10, 4, 12), (W.K_FIO_JUMP, W.A_CFG3, 12, 4, 10)])
def test_bf_stored_mode(kernel, amp, LN, l0, r):
    """bf-stored (SURVEY 8(c) oracle modes): O1-O7 applied to supplied blocks.  (1) With the oracle's own FP64
    blocks it equals the on-the-fly mode; (2) with the blocks rounded to complex64 -- the precision the GPU path
    stores its factors in -- it stays within a few 1e-7 of it: the factor storage alone accounts for that much
    of the GPU-vs-oracle error, the rest is FP32 arithmetic; (3) a wrong block is detected."""
    F = W.rhs(1 << LN, 3, 7)
    otf = oracle.bf_apply(kernel, amp, LN, l0, r, F)
    a, b, v0, xf, sw, u = _stored_inputs(kernel, amp, LN, l0, r)
    st = oracle.bf_apply_stored(LN, l0, r, a, b, v0, xf, sw, u, F)
    assert np.all(oracle.rel_l2(st, otf, axis=0) <= 1e-14)
    c64 = [x.astype(np.complex64) for x in (v0, sw, u)]
    st32 = oracle.bf_apply_stored(LN, l0, r, a.astype(np.complex64), b.astype(np.complex64), c64[0],
                                  [x.astype(np.complex64) for x in xf], c64[1], c64[2], F)
    e = oracle.rel_l2(st32, otf, axis=0)
    assert np.all(e <= 5e-7) and np.all(e >= 1e-9), e
    xm = [x.copy() for x in xf]
    xm[0][5] *= -1
    bad = oracle.bf_apply_stored(LN, l0, r, a, b, v0, xm, sw, u, F)
    assert np.all(oracle.rel_l2(bad, otf, axis=0) > 1e-3)
