"""oracle.nufft -- TEST INFRASTRUCTURE ONLY (same rules as oracle/__init__.py: only tests/, smoke() and bench.py's
cpu_baseline / reference legs import it; it shares no code with paper_1803_04128_b200/).

The NUFFT path of the paper (second half), plain FP64 numpy/scipy, step by step:

* Algorithm rlr: randomized low-rank factorization K ~ U0 S0 V0^* from sampled rows and
  columns with pivoted QR / LQ, the pseudo-inverse core and its SVD;
* Algorithm dc (Alg. 6): the O(N) decision whether the NUFFT applies -- r-leading randomized SVD of
  the phase factorization U1 V1^*, rank of rq sampled columns of (U2 V2^*) o e^{2 pi i (U1 V1^* - P Q^*)} by
  pivoted QR, and (if y = 1) Algorithm rlr of that matrix with rank r_eps;
* eqn:tg3 evaluated by its definition: g(x) = sum_k a_k(x) sum_xi e^{2 pi i sum_j p_j(x) q_j(xi)}
  b_k(xi) f(xi), a direct O(N^2) sum (all rows for small N, a row sample otherwise) -- what the GPU's type-2
  NUFFT approximates.

Readings (R24-R26): Alg. 6's "If n < r, let y = 1" is read with r the rank budget r_eps of step 4 (the
phase rank parameter r <= 3 cannot bound a sample's amplitude rank); the matrices of the configs' kernels are
split by the sign of xi ("the NUFFT approach ... can be applied to submatrices of K"; eqn:phlr P:1125-1131
for the wave-equation FIO), on which Phi(x, xi) = (x +- c(x)) xi is exactly rank 1 (cfg3's jump rides in the
amplitude split, R8).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

from . import A_CFG1, A_CFG2, A_CFG3, A_ONE, K_DFT, K_FIO, K_FIO_JUMP, K_FIO_PAPER, amp_terms  # noqa: F401


# ---------------------------------------------------------------------------------------------------------------
# The kernels' phase and amplitude as low-rank factorizations (the inputs of Alg. 6), on the grid of
# eqn:1D-xandxi (P:905-907, 0-based): x_i = i/N, xi_j = j - N/2.
# ---------------------------------------------------------------------------------------------------------------
def _c_of(kernel: int, x):
    if kernel in (K_FIO, K_FIO_JUMP):
        return (2.0 + np.sin(2.0 * np.pi * x)) / 16.0
    if kernel == K_FIO_PAPER:
        return (2.0 + 0.2 * np.sin(2.0 * np.pi * x)) / 16.0
    return np.zeros_like(x)


def phase_factors(kernel: int, LN: int, cols=None):
    """Phi = U1 V1^T exactly (real): U1 = [x, c(x)], V1 = [xi, |xi|] restricted to the columns `cols` (default all);
    the DFT kernel has only x xi.  cfg3's jump 0.25 sign(x - 1/3) xi is carried by its amplitude split (A_CFG3,
    DESIGN R8), as for the butterfly."""
    N = 1 << LN
    i = np.arange(N)
    x = i / N
    j = np.arange(N) if cols is None else np.asarray(cols)
    xi = (j - N // 2).astype(np.float64)
    U, V = [x], [xi]
    if kernel != K_DFT:
        U.append(_c_of(kernel, x))
        V.append(np.abs(xi))
    return np.stack(U, 1), np.stack(V, 1)


def amp_factors(amp: int, LN: int, cols=None):
    """alpha = U2 V2^T exactly: U2 = [a_k], V2 = [b_k] (the oracle's amplitude split, DESIGN R11)."""
    a, b = amp_terms(amp, LN)
    if cols is not None:
        b = b[:, np.asarray(cols)]
    return a.T.copy(), b.T.copy()


# ---------------------------------------------------------------------------------------------------------------
# Algorithm rlr
# ---------------------------------------------------------------------------------------------------------------
def rlr(entries, m: int, n: int, r: int, q: int, rng, sweeps: int = 3):
    """K ~ U0 diag(S0) V0^* for K given by entries(rows, cols) -> the submatrix.  Returns U0 (m x r), S0 (r,),
    V0 (n x r)."""
    pi_col = np.zeros(0, np.int64)
    pi_row = np.zeros(0, np.int64)
    for _ in range(sweeps):   # lines 4-5, repeated
        I = np.union1d(rng.choice(m, min(m, r * q), replace=False), pi_row)
        _, perm = sla.qr(entries(I, np.arange(n)), mode="r", pivoting=True)   # K_{I,:} P = Q R
        pi_col = np.sort(perm[:r])
        J = np.union1d(rng.choice(n, min(n, r * q), replace=False), pi_col)
        _, perm = sla.qr(entries(np.arange(m), J).conj().T, mode="r", pivoting=True)   # P K_{:,J} = L Q
        pi_row = np.sort(perm[:r])
    Qc, _, _ = sla.qr(entries(np.arange(m), pi_col), mode="economic", pivoting=True)
    Qr, _, _ = sla.qr(entries(pi_row, np.arange(n)).conj().T, mode="economic", pivoting=True)
    Qc, Qr = Qc[:, :r], Qr[:, :r]
    J = np.union1d(pi_col, rng.choice(n, min(n, r * q), replace=False))
    I = np.union1d(pi_row, rng.choice(m, min(m, r * q), replace=False))
    M = np.linalg.pinv(Qc[I, :]) @ entries(I, J) @ np.linalg.pinv(Qr.conj().T[:, J])
    UM, SM, VMh = np.linalg.svd(M)
    return Qc @ UM, SM, (VMh @ Qr.conj().T).conj().T


# ---------------------------------------------------------------------------------------------------------------
# Algorithm dc (Alg. 6)
# ---------------------------------------------------------------------------------------------------------------
def decide(U1, V1, U2, V2, r: int, r_eps: int, q: int, eps: float, rng):
    """Returns (y, n, P, Q, U, V): y = 1 if the NUFFT applies; n the numerical rank of the rq sampled columns;
    P, Q (real, N x r) with P Q^T the r-leading part of U1 V1^T (P scaled by the singular values); if y = 1,
    U (N x r_eps), V (N x r_eps) with (U2 V2^T) o e^{2 pi i (U1 V1^T - P Q^T)} ~ U V^T."""
    m, n_cols = U1.shape[0], V1.shape[0]
    r1 = U1.shape[1]
    # step 1: approximate r-leading SVD of the rank-r1 matrix U1 V1^T, randomized with a test matrix of more than
    # r1 columns ([Gu, randomSVD]): Y = U1 (V1^T Omega), orthonormal basis, B = Qy^T U1 V1^T, SVD of B
    Om = rng.standard_normal((n_cols, r1 + 4))
    Qy, _ = np.linalg.qr(U1 @ (V1.T @ Om))
    B = (Qy.T @ U1) @ V1.T
    Ub, S, Wt = np.linalg.svd(B, full_matrices=False)
    P = (Qy @ Ub[:, :r]) * S[:r]          # P Sigma -> P
    Q = Wt[:r].T

    def entries(I, J):   # (U2 V2^T) o e^{2 pi i (U1 V1^T - P Q^T)} on rows I, columns J
        ph = U1[I] @ V1[J].T - P[I] @ Q[J].T
        return (U2[I] @ V2[J].T) * np.exp(2j * np.pi * (ph - np.floor(ph)))

    # step 2: rq sampled columns, pivoted QR, rank at eps relative to R(1,1)
    J = np.sort(rng.choice(n_cols, min(n_cols, r * q), replace=False))
    R, _ = sla.qr(entries(np.arange(m), J), mode="r", pivoting=True)
    d = np.abs(np.diag(R))
    n = int(np.sum(d > d[0] * eps))
    # step 3 (reading R24: the rank budget is r_eps)
    y = int(n <= r_eps)
    if not y:
        return y, n, P, Q, None, None
    # step 4: Algorithm rlr with rank r_eps
    U0, S0, V0 = rlr(entries, m, n_cols, r_eps, q, rng)
    return y, n, P, Q, U0 * S0, V0.conj()


# ---------------------------------------------------------------------------------------------------------------
# eqn:tg3 by its definition
# ---------------------------------------------------------------------------------------------------------------
def tg3_rows(P, Q, U, V, F, rows, chunk: int = 1 << 14):
    """g(x_i) = sum_k U[i, k] sum_j e^{2 pi i P[i] . Q[j]} V[j, k] F[j, c] for the rows `rows` (direct sum, columns
    in chunks)."""
    rows = np.asarray(rows)
    out = np.zeros((len(rows), F.shape[1]), np.complex128)
    for j0 in range(0, Q.shape[0], chunk):
        ph = P[rows] @ Q[j0:j0 + chunk].T
        E = np.exp(2j * np.pi * (ph - np.floor(ph)))          # len(rows) x chunk
        for k in range(U.shape[1]):
            out += U[rows, k][:, None] * (E @ (V[j0:j0 + chunk, k][:, None] * F[j0:j0 + chunk]))
    return out


def halves(LN: int):
    """Column index sets of the two submatrices (xi < 0, xi >= 0)."""
    N = 1 << LN
    return np.arange(N // 2), np.arange(N // 2, N)


def nufft_path_rows(kernel: int, amp: int, LN: int, F, rows, eps: float = 1e-6, seed: int = 0):
    """The NUFFT path end to end on the oracle side: Alg. 6 on each half (r = 1), then eqn:tg3 by its definition on
    that half, summed.  Returns (g_rows, decisions) -- decisions [(y, n)] per half; raises if a half is rejected."""
    rng = np.random.default_rng(seed)
    F = np.asarray(F, np.complex128)
    g = np.zeros((len(rows), F.shape[1]), np.complex128)
    dec = []
    for cols in halves(LN):
        U1, V1 = phase_factors(kernel, LN, cols)
        U2, V2 = amp_factors(amp, LN, cols)
        y, n, P, Q, U, V = decide(U1, V1, U2, V2, r=1, r_eps=U2.shape[1] + 2, q=8, eps=eps * 1e-3, rng=rng)
        dec.append((y, n))
        if not y:
            raise ValueError(f"NUFFT not applicable on a half (numerical rank {n})")
        g += tg3_rows(P, Q, U, V, F[cols], rows)
    return g, dec
