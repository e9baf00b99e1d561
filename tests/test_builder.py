"""The host factor builder (product, csrc/bf_build.cpp) against the oracle's
blocks (oracle/bf_oracle.c), element by element.  The two are independent
implementations; the expected values come from the oracle only.

Tolerance: the builder stores complex64, so each entry carries a relative
rounding error <= 2^-24 of its magnitude (|entries| are O(1): unimodular
phases times Lagrange weights); 4e-7 absolute leaves margin for |entry| <= ~4.
"""
import numpy as np
import pytest

import oracle
from paper_1803_04128_b200 import bf
from paper_1803_04128_b200 import workloads as W

TOL = 4e-7


def _blocks_match(kernel, LN, l0, r, pairs):
    N, n0, h, D = 1 << LN, 1 << l0, LN // 2, LN - l0
    k = bf.fio(kernel, W.A_CFG1, LN, l0, r)
    worst = 0.0
    for p in pairs:
        p = int(p)
        a, b = divmod(p, N // n0)
        got = bf.build_blocks(k, bf.BF_STAGE_V0, p, 1)[0].reshape(n0, r).T          # column-major r x n0
        worst = max(worst, np.abs(got - oracle.bf_block(kernel, LN, l0, r, 0, l0, a, b)).max())
        for l in range(l0 + 1, D + 1):
            a, b = divmod(p, 1 << (LN - l))
            got = bf.build_blocks(k, bf.BF_STAGE_XFER0 + l - l0 - 1, p, 1)[0].reshape(2 * r, r).T
            worst = max(worst, np.abs(got - oracle.bf_block(kernel, LN, l0, r, 1, l, a, b)).max())
        a, b = divmod(p, 1 << (LN - h))
        got = bf.build_blocks(k, bf.BF_STAGE_SW, p, 1)[0].reshape(r, r).T
        worst = max(worst, np.abs(got - oracle.bf_block(kernel, LN, l0, r, 2, h, a, b)).max())
        a, b = divmod(p, n0)
        got = bf.build_blocks(k, bf.BF_STAGE_U, p, 1)[0].reshape(r, n0).T             # column-major n0 x r
        worst = max(worst, np.abs(got - oracle.bf_block(kernel, LN, l0, r, 3, D, a, b)).max())
    return worst


@pytest.mark.parametrize("kernel,LN,l0,r", [
    (W.K_FIO, 10, 4, 12),          # cfg1
    (W.K_DFT, 10, 4, 12),          # cfg1 DFT
    (W.K_FIO_PAPER, 12, 4, 8),     # tab:1D-FIO kernel
    (W.K_FIO, 16, 5, 10),          # cfg2
    (W.K_FIO_JUMP, 18, 5, 10),     # cfg3 (BF on the smooth phase)
    (W.K_FIO, 20, 6, 10),          # cfg4
    (W.K_FIO, 8, 4, 10),           # h == l0: no transfer level
    (W.K_FIO, 12, 3, 6),           # leaf 8
])
def test_builder_blocks_match_oracle(kernel, LN, l0, r):
    N = 1 << LN
    rng = np.random.default_rng(LN * 100 + l0)
    pairs = list(rng.integers(0, N, 12)) + [0, N - 1, N // 2, N // 3]
    assert _blocks_match(kernel, LN, l0, r, pairs) < TOL


@pytest.mark.parametrize("amp,kernel", [(W.A_ONE, W.K_FIO), (W.A_CFG1, W.K_FIO), (W.A_CFG2, W.K_FIO),
                                        (W.A_CFG3, W.K_FIO_JUMP)])
def test_builder_amplitude_matches_oracle(amp, kernel):
    LN = 12
    a, b = bf.build_amp(bf.fio(kernel, amp, LN, 4, 10))
    ao, bo = oracle.amp_terms(amp, LN)
    assert a.shape == ao.shape and b.shape == bo.shape
    assert np.abs(a - ao).max() < 1.2e-7 and np.abs(b - bo).max() < 1.2e-7


def test_builder_block_ranges_consistent():
    # a range build equals the concatenation of single-block builds (slicing for the streaming upload)
    k = bf.fio(W.K_FIO, W.A_CFG1, 12, 4, 10)
    for stage in (bf.BF_STAGE_V0, bf.BF_STAGE_SW, bf.BF_STAGE_U, bf.BF_STAGE_XFER0, bf.BF_STAGE_XFER0 + 3):
        whole = bf.build_blocks(k, stage, 100, 7)
        parts = np.concatenate([bf.build_blocks(k, stage, 100 + i, 1) for i in range(7)])
        assert np.array_equal(whole, parts)


def test_builder_rejects_bad_arguments():
    k = bf.fio(W.K_FIO, W.A_CFG1, 12, 4, 10)
    with pytest.raises(bf.BFError):
        bf.build_blocks(k, bf.BF_STAGE_V0, 4090, 10)          # past the last pair
    with pytest.raises(ValueError):
        bf.build_blocks(k, bf.BF_STAGE_XFER0 + 4, 0, 1)       # only 4 transfer levels at LN=12, l0=4
    with pytest.raises(bf.BFError):
        bf.build_amp(bf.fio(W.K_FIO, 9, 12, 4, 10))           # unknown amplitude
