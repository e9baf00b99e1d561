"""Seeded synthetic workloads (BASELINE.json ``configs``), shared by the CUDA path,
the tests and bench.py.

This module holds NO arithmetic of the method: only the configuration table
(sizes, ids, seeds), the seeded RHS generator and the seeded row sample.  The
oracle (``oracle/``) and the CUDA path (``paper_1803_04128_b200``) both consume
what it produces; neither imports the other.

Readings: r from eps per R10, r_amp and the amplitude
split per R11, RHS recipe per R13, row sample per R12.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# kernel ids (same numbering in the oracle and in include/bf_build.h)
K_FIO, K_FIO_PAPER, K_DFT, K_FIO_JUMP = 0, 1, 2, 3
# amplitude ids
A_ONE, A_CFG1, A_CFG2, A_CFG3 = 0, 1, 2, 3
N_AMP = {A_ONE: 1, A_CFG1: 2, A_CFG2: 2, A_CFG3: 4}


@dataclass(frozen=True)
class Workload:
    name: str
    kernel: int
    amp: int
    log2n: int
    log2leaf: int
    rank: int
    nrhs: int
    seed: int
    eps: float

    @property
    def n(self) -> int:
        return 1 << self.log2n

    @property
    def leaf(self) -> int:
        return 1 << self.log2leaf

    @property
    def n_amp(self) -> int:
        return N_AMP[self.amp]

    @property
    def nvec(self) -> int:
        return self.nrhs * self.n_amp

    def with_(self, **kw) -> "Workload":
        d = dict(self.__dict__)
        d.update(kw)
        return Workload(**d)


# BASELINE.json configs 1-5 (+ the DFT sanity case of config 1).  r per DESIGN R10.
CONFIGS = {
    "cfg1": Workload("cfg1", K_FIO, A_CFG1, 10, 4, 12, 1, 0, 1e-8),
    "cfg1_dft": Workload("cfg1_dft", K_DFT, A_CFG1, 10, 4, 12, 1, 0, 1e-8),
    "cfg2": Workload("cfg2", K_FIO, A_CFG2, 16, 5, 10, 16, 1, 1e-6),
    "cfg3": Workload("cfg3", K_FIO_JUMP, A_CFG3, 18, 5, 10, 64, 2, 1e-6),
    "cfg4": Workload("cfg4", K_FIO, A_CFG1, 20, 6, 10, 256, 3, 1e-6),
    "cfg5": Workload("cfg5", K_FIO, A_CFG1, 22, 6, 10, 8, 4, 1e-6),
}


def rhs(n: int, nrhs: int, seed: int, cols=None) -> np.ndarray:
    """complex64 N x nrhs, column-major (Fortran order), i.i.d. N(0,1) real and
    imaginary parts from numpy's default_rng(seed) (DESIGN R13):
    Z = rng.standard_normal((nrhs, N, 2)); F[j, c] = Z[c, j, 0] + i Z[c, j, 1].
    ``cols`` selects a subset of columns (same values as the full draw)."""
    rng = np.random.default_rng(seed)
    if cols is None:
        z = rng.standard_normal((nrhs, n, 2), dtype=np.float64)
        f = (z[..., 0] + 1j * z[..., 1]).astype(np.complex64)
        return np.asfortranarray(f.T)
    cols = list(cols)
    out = np.empty((n, len(cols)), np.complex64, order="F")
    want = {c: k for k, c in enumerate(cols)}
    for c in range(max(cols) + 1):   # stream column by column: identical values, bounded memory
        z = rng.standard_normal((1, n, 2), dtype=np.float64)
        if c in want:
            out[:, want[c]] = (z[0, :, 0] + 1j * z[0, :, 1]).astype(np.complex64)
    return out


def sample_rows(n: int, seed: int, count: int = 256) -> np.ndarray:
    """The eps^b row sample S: sorted first `count` of a seeded permutation,
    seed 1000 + config seed (DESIGN R12)."""
    if count >= n:
        return np.arange(n, dtype=np.int64)
    rng = np.random.default_rng(1000 + seed)
    return np.sort(rng.permutation(n)[:count]).astype(np.int64)
