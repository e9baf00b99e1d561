"""Host logic of the structured interpolative factors (include/bf.h "structured plans"):
the product builder's phases and shared Lagrange matrices (bf_build_structured / bf_build_structured_lag),
applied here densely in numpy exactly as bf.h defines the structured stages, must give the same operator as the
oracle's butterfly (Algorithm 4.1 with every block from its own equation), assembled on every unit vector.
The only differences allowed are the complex64 / FP32 storage of phases and Lagrange weights (~1e-7).
"""
import numpy as np
import pytest

import oracle
from paper_1803_04128_b200 import bf
from paper_1803_04128_b200 import workloads as W

BF_STAGE_V0, BF_STAGE_U, BF_STAGE_XFER0 = 0, 2, 16


def structured_apply(w, Y):
    """BF(Y) (Y: N x nv) from the builder's structured factors, per the stage formulas of include/bf.h."""
    k = bf.fio_of(w)
    LN, l0, r = w.log2n, w.log2leaf, w.rank
    N, n0 = 1 << LN, 1 << l0
    h, D = LN // 2, LN - l0
    nleaf = N >> l0
    nv = Y.shape[1]
    Yl = Y.reshape(nleaf, n0, nv)
    if h == l0:   # dense V0 carrying the switch
        V = bf.build_structured(k, BF_STAGE_V0, 0, N, n0 * r).astype(np.complex128).reshape(n0, nleaf, n0, r)
        eta = np.einsum("abjt,bjv->abtv", V, Yl)
    else:
        om = bf.build_structured(k, BF_STAGE_V0, 0, N, n0).astype(np.complex128).reshape(n0, nleaf, n0)
        L0 = bf.build_structured_lag(k, BF_STAGE_V0, r * n0).astype(np.float64).reshape(n0, r)   # [j][t]
        eta = np.einsum("jt,abj,bjv->abtv", L0, om, Yl)
    cur = eta.reshape(N, r, nv)
    for i in range(D - l0):
        l = l0 + 1 + i
        sh = LN - l
        X = np.repeat(cur.reshape(1 << (l - 1), 1 << sh, 2, r, nv), 2, axis=0)   # [a][b][c][s][v]
        stage = BF_STAGE_XFER0 + i
        if l == h:   # first-half level followed by the switch with its phases: Sw' L1 (psi o x)
            d = bf.build_structured(k, stage, 0, N, 2 * r + r * r).astype(np.complex128).reshape(1 << l, 1 << sh, -1)
            psi = d[..., :2 * r].reshape(1 << l, 1 << sh, 2, r)
            Sw = d[..., 2 * r:].reshape(1 << l, 1 << sh, r, r)   # column-major: [s][t]
            L1 = bf.build_structured_lag(k, stage, 2 * r * r).astype(np.float64).reshape(2, r, r)
            y = np.einsum("cst,abcs,abcsv->abtv", L1, psi, X)
            out = np.einsum("abst,absv->abtv", Sw, y)
        elif l < h:
            psi = bf.build_structured(k, stage, 0, N, 2 * r).astype(np.complex128).reshape(1 << l, 1 << sh, 2, r)
            L1 = bf.build_structured_lag(k, stage, 2 * r * r).astype(np.float64).reshape(2, r, r)   # [c][s][t]
            out = np.einsum("cst,abcs,abcsv->abtv", L1, psi, X)
        else:
            chi = bf.build_structured(k, stage, 0, N, 2 * r).astype(np.complex128).reshape(1 << l, 1 << sh, 2, r)
            L2 = bf.build_structured_lag(k, stage, 2 * r * r).astype(np.float64).reshape(2, r, r)   # [e][s][t]
            out = np.empty((1 << l, 1 << sh, r, nv), np.complex128)
            for e in (0, 1):
                z = np.einsum("st,abcsv->abctv", L2[e], X[e::2])
                out[e::2] = np.einsum("abct,abctv->abtv", chi[e::2], z)
        cur = out.reshape(N, r, nv)
    Om = bf.build_structured(k, BF_STAGE_U, 0, N, n0).astype(np.complex128).reshape(N // n0, n0, n0)   # [a][b][j]
    Lsl = bf.build_structured_lag(k, BF_STAGE_U, n0 * r).astype(np.float64).reshape(r, n0)            # [t][j]
    z = cur.reshape(N // n0, n0, r, nv)
    U = np.einsum("abj,tj,abtv->ajv", Om, Lsl, z)
    return U.reshape(N, nv)


@pytest.mark.parametrize("kernel,amp,LN,l0,r", [(W.K_FIO, W.A_CFG1, 8, 3, 6),     # h = 4: 1 first, h, 3 second
                                                 (W.K_FIO, W.A_CFG2, 10, 4, 8),    # 1 first level, h, 2 second
                                                 (W.K_DFT, W.A_ONE, 10, 3, 8),     # 2 first levels
                                                 (W.K_FIO_JUMP, W.A_CFG3, 8, 4, 8),  # h == l0: dense V0 with switch
                                                 (W.K_FIO, W.A_CFG1, 12, 5, 10)])  # h - 1 = l0
def test_structured_operator_equals_oracle_bf(kernel, amp, LN, l0, r):
    w = W.CONFIGS["cfg1"].with_(kernel=kernel, amp=amp, log2n=LN, log2leaf=l0, rank=r)
    N = 1 << LN
    if LN <= 10:
        F = np.eye(N, dtype=np.complex128)
    else:
        F = W.rhs(N, 8, 5).astype(np.complex128)
    a, b = oracle.amp_terms(amp, LN)
    G = np.zeros_like(F)
    for kk in range(a.shape[0]):
        G += a[kk][:, None] * structured_apply(w, b[kk][:, None] * F)
    R = oracle.bf_apply(kernel, amp, LN, l0, r, F, vchunk=min(N, 256))
    err = np.linalg.norm(G - R) / np.linalg.norm(R)
    assert err <= 2e-6, err


def test_structured_factor_bytes_model():
    # per pair: n0 + 2r per structured level + r^2 (switch at level h) + n0, against r n0 + 2 r^2 per level + n0 r
    w = W.CONFIGS["cfg5"]
    n0, r, nx = w.leaf, w.rank, w.log2n - 2 * w.log2leaf
    dense = r * n0 + nx * 2 * r * r + n0 * r
    struct = n0 + nx * 2 * r + r * r + n0
    assert 8 * w.n * dense / 1e9 == pytest.approx(110.1, rel=0.01)   # the switch folded into level h
    assert 8 * w.n * struct / 1e9 == pytest.approx(14.36, rel=0.01)
