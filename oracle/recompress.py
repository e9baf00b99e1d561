"""oracle.recompress -- TEST INFRASTRUCTURE ONLY (same rules as oracle/__init__.py).

A plain FP64 numpy transcription of the recompression of the interpolative butterfly factorization (SURVEY 8(f)
NEXT-3: "structure-preserving sweeping matrix compression", deferred there to [IBF]; DESIGN.md
reading R21).  Every coefficient space of the factor product eqn:BFM -- delta_l[p] in C^r for pair p
at level l -- carries the block K(A,B) = S_p R_p of the operator (R_p: input -> delta_l[p], S_p: delta_l[p] ->
output).  Balanced truncation keeps the r' dominant directions of each block:

    Gamma_out[p] = S_p^H S_p   (top-down:  U^H U at level D;  sum_e W_c^H Gamma_out[parent_e] W_c below)
    Gamma_in[p]  = R_p R_p^H   (bottom-up, from the ALREADY TRUNCATED lower levels)
    C = Gamma_out^{1/2} Gamma_in^{1/2} = X Sigma Y^H,   P = Sigma_r'^{-1/2} X_r'^H Gamma_out^{1/2},
                                                        Q = Gamma_in^{1/2} Y_r' Sigma_r'^{-1/2}
so that S_p Q P R_p is the best rank-r' approximation of K(A,B) (the product of the two Gram square roots has
the block's singular values).  The new factors are  V0' = P V0,  W'_l = P_l W_l blockdiag(Q_{l-1}(q_0),
Q_{l-1}(q_1)),  U' = U Q_D  (rank r', the switch already folded into level h).  Square roots and SVD are
numpy's eigh / svd (library primitives); no blocking, no fusion.
"""
from __future__ import annotations

import numpy as np

from . import bf_blocks


def folded_factors(kernel: int, LN: int, l0: int, r: int):
    """The oracle's FP64 blocks (bf-stored layout, row-major) with the switch folded into the level-h factor
    (V0 when h == l0): V0 [N][r][n0], X {l: [N][r][2r]} for l = l0+1..D, U [N][n0][r]."""
    D, h = LN - l0, LN // 2
    V0 = bf_blocks(kernel, LN, l0, r, 0)
    X = {l: bf_blocks(kernel, LN, l0, r, 1, l) for l in range(l0 + 1, D + 1)}
    S = bf_blocks(kernel, LN, l0, r, 2)
    U = bf_blocks(kernel, LN, l0, r, 3)
    if h > l0:
        X[h] = np.einsum("pts,psk->ptk", S, X[h])
    else:
        V0 = np.einsum("pts,psk->ptk", S, V0)
    return V0, X, U


def _hsqrt(G):
    """Hermitian PSD square roots of a stack of matrices (eigendecomposition; negative rounding clipped)."""
    G = (G + np.conj(np.swapaxes(G, -1, -2))) / 2
    w, V = np.linalg.eigh(G)
    w = np.sqrt(np.clip(w, 0.0, None))
    return (V * w[..., None, :]) @ np.conj(np.swapaxes(V, -1, -2))


def _truncate(Gin, Gout, rp):
    Ti, To = _hsqrt(Gin), _hsqrt(Gout)
    Xs, sv, Yh = np.linalg.svd(To @ Ti)
    sq = 1.0 / np.sqrt(sv[:, :rp])
    P = sq[:, :, None] * (np.conj(np.swapaxes(Xs[:, :, :rp], 1, 2)) @ To)
    Q = (Ti @ np.conj(np.swapaxes(Yh[:, :rp, :], 1, 2))) * sq[:, None, :]
    return P, Q, sv


def gram_out(X, U, LN: int, l0: int):
    """Gamma_out[l][p] = S_p^H S_p for every level l0..D: U^H U at D, then top-down through the parents
    (2a + e, b >> 1) at l + 1, whose column block c = b & 1 multiplies delta_l[p]."""
    N, r = U.shape[0], U.shape[2]
    D = LN - l0
    p = np.arange(N)
    G = {D: np.einsum("pjt,pjs->pts", np.conj(U), U)}
    for l in range(D - 1, l0 - 1, -1):
        nb = 1 << (LN - l)
        a, b = p // nb, p % nb
        c = b & 1
        acc = np.zeros((N, r, r), np.complex128)
        X4 = X[l + 1].reshape(N, r, 2, r)
        for e in (0, 1):
            pp = (2 * a + e) * (nb // 2) + (b >> 1)
            Wc = X4[pp, :, c, :]                                      # [N][t][s]
            acc += np.conj(np.swapaxes(Wc, 1, 2)) @ G[l + 1][pp] @ Wc
        G[l] = acc
    return G


def _gram_in_next(Wt, Ginp, q0, k):
    """Gamma_in of level l from its blocks Wt (acting on the level-(l-1) coefficients, k per pair) and the
    level-(l-1) Grams: the two children q0, q0 + 1 have disjoint inputs, so their Grams add."""
    return sum(Wt[:, :, c * k:(c + 1) * k] @ Ginp[q0 + c] @ np.conj(np.swapaxes(Wt[:, :, c * k:(c + 1) * k], 1, 2))
               for c in (0, 1))


def gram_in(V0, X, LN: int, l0: int):
    """Gamma_in[l][p] = R_p R_p^H of the untruncated factors (tests; the sweep uses the same recursion on the
    truncated ones)."""
    N = V0.shape[0]
    p = np.arange(N)
    G = {l0: V0 @ np.conj(np.swapaxes(V0, 1, 2))}
    for l in range(l0 + 1, LN - l0 + 1):
        nb = 1 << (LN - l)
        q0 = (p // nb >> 1) * (2 * nb) + 2 * (p % nb)
        G[l] = _gram_in_next(X[l], G[l - 1], q0, V0.shape[1])
    return G


def recompress(V0, X, U, LN: int, l0: int, rp: int):
    """Balanced-truncation sweep to rank rp.  Returns (V0', X', U', tail) with tail[l] = max over pairs of
    sigma_{rp+1} / sigma_1 at level l (the relative singular value each block drops)."""
    N, r = V0.shape[0], V0.shape[1]
    D = LN - l0
    p = np.arange(N)
    Gout = gram_out(X, U, LN, l0)
    tail = {}
    Gin = V0 @ np.conj(np.swapaxes(V0, 1, 2))
    P, Q, sv = _truncate(Gin, Gout[l0], rp)
    tail[l0] = float(np.max(sv[:, rp] / sv[:, 0])) if rp < r else 0.0
    V0n = P @ V0
    Ginp = P @ Gin @ np.conj(np.swapaxes(P, 1, 2))   # Gram of the truncated coefficients (rp x rp)
    Xn = {}
    for l in range(l0 + 1, D + 1):
        nb = 1 << (LN - l)
        q0 = (p // nb >> 1) * (2 * nb) + 2 * (p % nb)
        Wt = np.concatenate([X[l][:, :, c * r:(c + 1) * r] @ Q[q0 + c] for c in (0, 1)], axis=2)   # [N][r][2rp]
        Gin = _gram_in_next(Wt, Ginp, q0, rp)
        P, Q, sv = _truncate(Gin, Gout[l], rp)
        tail[l] = float(np.max(sv[:, rp] / sv[:, 0])) if rp < r else 0.0
        Xn[l] = P @ Wt
        Ginp = P @ Gin @ np.conj(np.swapaxes(P, 1, 2))
    Un = U @ Q
    return V0n, Xn, Un, tail


def bf_apply_recompressed(kernel: int, amp: int, LN: int, l0: int, r: int, rp: int, F: np.ndarray,
                          vchunk: int = 64):
    """g = sum_k a_k o BF'(b_k o f) with BF' the rank-rp recompression of the rank-r interpolative factorization
    (bf-stored mode of the C oracle, identity switch: the switch is inside level h)."""
    from . import amp_terms, bf_apply_stored
    V0n, Xn, Un, _ = recompress(*folded_factors(kernel, LN, l0, r), LN, l0, rp)
    a, b = amp_terms(amp, LN)
    N = 1 << LN
    I = np.broadcast_to(np.eye(rp, dtype=np.complex128), (N, rp, rp))
    return bf_apply_stored(LN, l0, rp, a, b, V0n, [Xn[l] for l in sorted(Xn)], I, Un, F, vchunk=vchunk)
