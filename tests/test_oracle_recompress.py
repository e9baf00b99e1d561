"""Pins for the oracle's recompression of the butterfly (oracle/recompress.py, DESIGN
R21), each against something other than the recompression itself: the un-recompressed butterfly (rp = r must
reproduce it to rounding: every projector is then the identity on the kept space), the direct sum (the paper's
error measure eps^b: the rank-8 recompression of the rank-12 interpolative factorization stays within
eps/2 = 5e-7), the dense kernel (brute force at N = 256), the SVD of one block (a single-level operator whose
truncation must equal numpy's rank-rp SVD truncation), and monotonicity in rp.
"""
import numpy as np
import pytest

import oracle
from oracle import recompress as RC
from paper_1803_04128_b200 import workloads as W


def _stored(V0, X, U, LN, l0, r, F):
    N = 1 << LN
    a = np.ones((1, N), np.complex128)
    I = np.broadcast_to(np.eye(r, dtype=np.complex128), (N, r, r))
    return oracle.bf_apply_stored(LN, l0, r, a, a, V0, [X[l] for l in sorted(X)], I, U, F)


def test_full_rank_is_exact_on_random_factors():
    # random (well-conditioned) factors: with rp = r every projector Q P is the identity, so the sweep must
    # reproduce the operator to rounding -- pins the Gram propagation and the index maps of every level
    LN, l0, r = 10, 3, 6
    N, n0 = 1 << LN, 1 << l0
    rng = np.random.default_rng(5)
    cg = lambda *s: rng.standard_normal(s) + 1j * rng.standard_normal(s)
    V0 = cg(N, r, n0)
    X = {l: cg(N, r, 2 * r) for l in range(l0 + 1, LN - l0 + 1)}
    U = cg(N, n0, r)
    F = W.rhs(N, 2, 3).astype(np.complex128)
    V0n, Xn, Un, _ = RC.recompress(V0, X, U, LN, l0, r)
    assert oracle.rel_l2(_stored(V0n, Xn, Un, LN, l0, r, F), _stored(V0, X, U, LN, l0, r, F)) <= 1e-11


def test_full_rank_paper_factors():
    # the paper's factors have nearly rank-deficient blocks (true rank ~8 of r = 10): rp = r keeps them to the
    # rounding that the tiny singular values amplify
    LN, l0, r = 10, 4, 10
    F = W.rhs(1 << LN, 2, 3).astype(np.complex128)
    g0 = oracle.bf_apply(W.K_FIO, W.A_CFG1, LN, l0, r, F)
    g1 = RC.bf_apply_recompressed(W.K_FIO, W.A_CFG1, LN, l0, r, r, F)
    assert oracle.rel_l2(g1, g0) <= 1e-6


@pytest.mark.parametrize("LN,l0,r,rp", [(12, 5, 12, 8), (14, 5, 12, 8), (12, 5, 10, 8)])
def test_recompressed_within_eps(LN, l0, r, rp):
    F = W.rhs(1 << LN, 1, 11).astype(np.complex128)
    rows = W.sample_rows(1 << LN, 3)
    gd = oracle.direct_rows(W.K_FIO, W.A_CFG1, LN, F, rows)
    g = RC.bf_apply_recompressed(W.K_FIO, W.A_CFG1, LN, l0, r, rp, F)
    assert oracle.rel_l2(g[rows], gd) <= 5e-7


def test_error_monotone_in_rank():
    LN, l0, r = 12, 5, 12
    F = W.rhs(1 << LN, 1, 12).astype(np.complex128)
    rows = W.sample_rows(1 << LN, 4)
    gd = oracle.direct_rows(W.K_FIO, W.A_CFG1, LN, F, rows)
    errs = [oracle.rel_l2(RC.bf_apply_recompressed(W.K_FIO, W.A_CFG1, LN, l0, r, rp, F)[rows], gd) for rp in (4, 6, 8)]
    assert errs[0] > errs[1] > errs[2], errs


def test_dense_brute_force():
    LN, l0 = 8, 4
    N = 1 << LN
    I = np.eye(N, dtype=np.complex128)
    B = RC.bf_apply_recompressed(W.K_FIO, W.A_CFG1, LN, l0, 12, 8, I, vchunk=N)
    K = oracle.dense_kernel(W.K_FIO, W.A_CFG1, LN)
    assert np.linalg.norm(B - K) / np.linalg.norm(K) <= 5e-7


def test_single_level_is_svd_truncation():
    # LN = 2 l0: no transfer level, the butterfly is U (Sw V0) per pair -- blocks K(A,B) = U[a,b] (Sw V0)[a',b']
    # summed over the leaf pairs.  With one coefficient space per pair the balanced truncation of each pair must
    # equal the SVD truncation of its own block S_p R_p = U[p] W0[p] (numpy's svd, rank rp).
    LN, l0, r, rp = 8, 4, 10, 5
    V0, X, U = RC.folded_factors(W.K_FIO, LN, l0, r)
    assert not X
    V0n, _, Un, _ = RC.recompress(V0, X, U, LN, l0, rp)
    N = 1 << LN
    for p in (0, 7, 100, N - 1):
        # LN = 2 l0: S0 and SL act on the same level (l0 = D) and index its pair (A, B) the same way
        K = U[p] @ V0[p]
        Kn = Un[p] @ V0n[p]
        u, s, vh = np.linalg.svd(K)
        Kt = (u[:, :rp] * s[:rp]) @ vh[:rp]
        assert np.linalg.norm(Kn - Kt) <= 1e-9 * np.linalg.norm(K), p


def _downstream(X, U, LN, l0, l, D):
    """Brute force: the output of the factors above level l applied to coefficients d (N x r at level l)."""
    def run(d):
        N = d.shape[0]
        for m in range(l + 1, D + 1):
            nb = 1 << (LN - m)
            nd = np.zeros_like(d)
            for pp in range(N):
                a, b = pp // nb, pp % nb
                q0 = (a >> 1) * (2 * nb) + 2 * b
                nd[pp] = X[m][pp] @ np.concatenate([d[q0], d[q0 + 1]])
            d = nd
        n0 = 1 << l0
        g = np.zeros(N, np.complex128)
        for pp in range(N):
            g[(pp // n0) * n0:(pp // n0 + 1) * n0] += U[pp] @ d[pp]
        return g
    return run


def _upstream(V0, X, LN, l0, l):
    """Brute force: the level-l coefficients (N x r) of an input f."""
    def run(f):
        N, n0 = f.shape[0], 1 << l0
        nleaf = N // n0
        d = np.stack([V0[pp] @ f[(pp % nleaf) * n0:(pp % nleaf + 1) * n0] for pp in range(N)])
        for m in range(l0 + 1, l + 1):
            nb = 1 << (LN - m)
            nd = np.zeros_like(d)
            for pp in range(N):
                a, b = pp // nb, pp % nb
                q0 = (a >> 1) * (2 * nb) + 2 * b
                nd[pp] = X[m][pp] @ np.concatenate([d[q0], d[q0 + 1]])
            d = nd
        return d
    return run


def test_grams_against_brute_force():
    # Gamma_out[l][p] = S_p^H S_p and Gamma_in[l][p] = R_p R_p^H with S_p, R_p assembled by applying the factors
    # to unit coefficient vectors / unit inputs (the definition), on the paper's factors at N = 256
    LN, l0, r = 8, 3, 6
    N = 1 << LN
    V0, X, U = RC.folded_factors(W.K_FIO, LN, l0, r)
    Go, Gi = RC.gram_out(X, U, LN, l0), RC.gram_in(V0, X, LN, l0)
    for l in (l0, l0 + 2, LN - l0):
        down, up = _downstream(X, U, LN, l0, l, LN - l0), _upstream(V0, X, LN, l0, l)
        R = np.stack([up(np.eye(N, dtype=np.complex128)[:, j]) for j in range(N)], axis=-1)   # [pair][t][input j]
        for p in (1, 77, N - 2):
            S = np.zeros((N, r), np.complex128)
            for s in range(r):
                d = np.zeros((N, r), np.complex128)
                d[p, s] = 1
                S[:, s] = down(d)
            assert np.allclose(Go[l][p], S.conj().T @ S, rtol=1e-10, atol=1e-10 * np.abs(Go[l][p]).max())
            assert np.allclose(Gi[l][p], R[p] @ R[p].conj().T, rtol=1e-10, atol=1e-10 * np.abs(Gi[l][p]).max())


def test_rank_rule():
    """Reading R21: r' = 8 is the smallest even rank whose recompression stays within eps/2 = 5e-7 of the direct
    sum at eps = 1e-6 (cfg4's kernel and leaf 64, at N = 2^14); r' = 6 does not."""
    LN, l0 = 14, 6
    F = W.rhs(1 << LN, 1, 11).astype(np.complex128)
    rows = W.sample_rows(1 << LN, 3)
    gd = oracle.direct_rows(W.K_FIO, W.A_CFG1, LN, F, rows)
    e = {rp: oracle.rel_l2(RC.bf_apply_recompressed(W.K_FIO, W.A_CFG1, LN, l0, 12, rp, F)[rows], gd) for rp in (6, 8)}
    assert e[8] <= 5e-7 < e[6], e
