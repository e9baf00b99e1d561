"""oracle -- TEST INFRASTRUCTURE ONLY.

ctypes wrapper around ``oracle/bf_oracle.c``: a plain double-precision CPU
transcription of the IBF-MAT apply of arXiv:1803.04128 (direct sum O0 and the
on-the-fly butterfly O1-O7 of Algorithm 4.1).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  It shares no code with
``paper_1803_04128_b200`` (the CUDA path) and never imports it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bf_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# kernel ids (phase functions), see bf_oracle.c
K_FIO, K_FIO_PAPER, K_DFT, K_FIO_JUMP = 0, 1, 2, 3
# amplitude ids
A_ONE, A_CFG1, A_CFG2, A_CFG3 = 0, 1, 2, 3

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (C11, -O2, OpenMP). Building the checker is not using it."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-std=gnu11", "-O2", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        i64, i32, dbl, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_void_p
        lib.orc_version.restype = i32
        lib.orc_grid.argtypes = [i64, i64, i32, vp]
        lib.orc_center.argtypes = [i64, i64]
        lib.orc_center.restype = i64
        lib.orc_lagrange.argtypes = [vp, i32, i32, dbl]
        lib.orc_lagrange.restype = dbl
        lib.orc_phi.argtypes = [i32, i32, i64, i64, i32]
        lib.orc_phi.restype = dbl
        lib.orc_n_amp.argtypes = [i32]
        lib.orc_n_amp.restype = i32
        lib.orc_amp_term.argtypes = [i32, i32, i32, i32, vp]
        lib.orc_amp_term.restype = i32
        lib.orc_direct_rows.argtypes = [i32, i32, i32, i64, vp, i64, vp, i64, vp]
        lib.orc_dense_kernel.argtypes = [i32, i32, i32, vp]
        lib.orc_bf_block.argtypes = [i32, i32, i32, i32, i32, i32, i64, i64, vp]
        lib.orc_bf_block.restype = i32
        lib.orc_bf_apply.argtypes = [i32, i32, i32, i32, i32, i64, vp, i64, vp, i64, i64]
        lib.orc_bf_apply.restype = i32
        lib.orc_num_threads.restype = i32
        lib.orc_bf_blocks.argtypes = [i32, i32, i32, i32, i32, i32, vp]
        lib.orc_bf_blocks.restype = i32
        lib.orc_bf_apply_stored.argtypes = [i32, i32, i32, i32, vp, vp, vp, vp, vp, vp, i64, vp, i64, vp, i64, i64]
        lib.orc_bf_apply_stored.restype = i32
        lib.orc_bf_apply_adjoint.argtypes = [i32, i32, i32, i32, i32, i64, vp, i64, vp, i64, i64]
        lib.orc_bf_apply_adjoint.restype = i32
        lib.orc_direct_adjoint_rows.argtypes = [i32, i32, i32, i64, vp, i64, vp, i64, vp]
        _lib = lib
    return _lib


def _c128(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex128)


def num_threads() -> int:
    return int(_load().orc_num_threads())


def grid(lo: int, n: int, r: int) -> np.ndarray:
    """Mock-Chebyshev nodes of block [lo, lo+n) (eqn:gdA P:214-226, DESIGN R2/R3), 0-based."""
    g = np.zeros(r, dtype=np.int64)
    _load().orc_grid(lo, n, r, g.ctypes.data)
    return g


def center(lo: int, n: int) -> int:
    return int(_load().orc_center(lo, n))


def lagrange(g, t: int, q: float) -> float:
    g = np.ascontiguousarray(g, dtype=np.int64)
    return float(_load().orc_lagrange(g.ctypes.data, len(g), t, q))


def phi(kernel: int, LN: int, i: int, j: int, full: bool = True) -> float:
    return float(_load().orc_phi(kernel, LN, i, j, int(full)))


def n_amp(amp: int) -> int:
    return int(_load().orc_n_amp(amp))


def amp_terms(amp: int, LN: int):
    """(a, b): complex128 arrays [n_amp][N] of the amplitude split (DESIGN R11)."""
    N = 1 << LN
    k = n_amp(amp)
    a = np.zeros((k, N), np.complex128)
    b = np.zeros((k, N), np.complex128)
    for t in range(k):
        _load().orc_amp_term(amp, LN, t, 0, a[t].ctypes.data)
        _load().orc_amp_term(amp, LN, t, 1, b[t].ctypes.data)
    return a, b


def direct_rows(kernel: int, amp: int, LN: int, F: np.ndarray, rows) -> np.ndarray:
    """O0: rows of g = K F (F: N x nrhs). Returns len(rows) x nrhs complex128."""
    F = np.asfortranarray(F, dtype=np.complex128)
    N, nrhs = F.shape
    assert N == 1 << LN
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.zeros((len(rows), nrhs), np.complex128, order="F")
    _load().orc_direct_rows(kernel, amp, LN, nrhs, F.ctypes.data, N, rows.ctypes.data, len(rows), out.ctypes.data)
    return out


def dense_kernel(kernel: int, amp: int, LN: int) -> np.ndarray:
    N = 1 << LN
    K = np.zeros((N, N), np.complex128)
    _load().orc_dense_kernel(kernel, amp, LN, K.ctypes.data)
    return K


def bf_block(kernel: int, LN: int, l0: int, r: int, stage: int, level: int, a: int, b: int) -> np.ndarray:
    """One block of Algorithm 4.1 in FP64. stage 0: init r x n0; 1: transfer r x 2r at `level`;
    2: switch r x r; 3: termination n0 x r."""
    n0 = 1 << l0
    shape = {0: (r, n0), 1: (r, 2 * r), 2: (r, r), 3: (n0, r)}[stage]
    out = np.zeros(shape, np.complex128)
    rc = _load().orc_bf_block(kernel, LN, l0, r, stage, level, a, b, out.ctypes.data)
    if rc:
        raise ValueError("orc_bf_block: bad arguments")
    return out


def bf_apply(kernel: int, amp: int, LN: int, l0: int, r: int, F: np.ndarray, vchunk: int = 64) -> np.ndarray:
    """O1-O7: g = sum_k a_k o BF(b_k o f) for every column of F (N x nrhs)."""
    F = np.asfortranarray(F, dtype=np.complex128)
    N, nrhs = F.shape
    assert N == 1 << LN
    G = np.zeros((N, nrhs), np.complex128, order="F")
    rc = _load().orc_bf_apply(kernel, amp, LN, l0, r, nrhs, F.ctypes.data, N, G.ctypes.data, N, vchunk)
    if rc:
        raise ValueError(f"orc_bf_apply failed ({rc})")
    return G


def bf_apply_adjoint(kernel: int, amp: int, LN: int, l0: int, r: int, F: np.ndarray, vchunk: int = 64) -> np.ndarray:
    """O8: the adjoint apply g = sum_k conj(b_k) o BF*(conj(a_k) o f), F indexed by x (N x nrhs), result by xi."""
    F = np.asfortranarray(F, dtype=np.complex128)
    N, nrhs = F.shape
    assert N == 1 << LN
    G = np.zeros((N, nrhs), np.complex128, order="F")
    rc = _load().orc_bf_apply_adjoint(kernel, amp, LN, l0, r, nrhs, F.ctypes.data, N, G.ctypes.data, N, vchunk)
    if rc:
        raise ValueError(f"orc_bf_apply_adjoint failed ({rc})")
    return G


def direct_adjoint_rows(kernel: int, amp: int, LN: int, F: np.ndarray, rows) -> np.ndarray:
    """O0*: xi-rows of g = K* F (F: N x nrhs over x). Returns len(rows) x nrhs complex128."""
    F = np.asfortranarray(F, dtype=np.complex128)
    N, nrhs = F.shape
    assert N == 1 << LN
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.zeros((len(rows), nrhs), np.complex128, order="F")
    _load().orc_direct_adjoint_rows(kernel, amp, LN, nrhs, F.ctypes.data, N, rows.ctypes.data, len(rows),
                                    out.ctypes.data)
    return out


def bf_blocks(kernel: int, LN: int, l0: int, r: int, stage: int, level: int = 0) -> np.ndarray:
    """Every block of one stage in pair order, FP64 (the bf-stored input layout): [N, rows, cols]."""
    n0 = 1 << l0
    shape = {0: (r, n0), 1: (r, 2 * r), 2: (r, r), 3: (n0, r)}[stage]
    out = np.zeros((1 << LN,) + shape, np.complex128)
    if _load().orc_bf_blocks(kernel, LN, l0, r, stage, level, out.ctypes.data):
        raise ValueError("orc_bf_blocks: bad arguments")
    return out


def bf_apply_stored(LN: int, l0: int, r: int, a: np.ndarray, b: np.ndarray, v0, xfer, sw, u,
                    F: np.ndarray, vchunk: int = 64) -> np.ndarray:
    """bf-stored: O1-O7 with caller-supplied blocks (any precision, upcast to FP64) and amplitude terms
    a, b ([n_amp][N]); layouts as bf_blocks returns them."""
    F = np.asfortranarray(F, dtype=np.complex128)
    N, nrhs = F.shape
    arrs = [np.ascontiguousarray(x, dtype=np.complex128) for x in (a, b, v0, sw, u)]
    xs = [np.ascontiguousarray(x, dtype=np.complex128) for x in xfer]
    xp = (ctypes.c_void_p * max(1, len(xs)))(*[x.ctypes.data for x in xs])
    G = np.zeros((N, nrhs), np.complex128, order="F")
    rc = _load().orc_bf_apply_stored(LN, l0, r, arrs[0].shape[0], arrs[0].ctypes.data, arrs[1].ctypes.data,
                                     arrs[2].ctypes.data, ctypes.cast(xp, ctypes.c_void_p), arrs[3].ctypes.data,
                                     arrs[4].ctypes.data, nrhs, F.ctypes.data, N, G.ctypes.data, N, vchunk)
    if rc:
        raise ValueError(f"orc_bf_apply_stored failed ({rc})")
    return G


def rel_l2(x: np.ndarray, ref: np.ndarray, axis=None):
    """Relative l2 error ||x-ref|| / ||ref|| (eps^b definition)."""
    num = np.sqrt(np.sum(np.abs(x - ref) ** 2, axis=axis))
    den = np.sqrt(np.sum(np.abs(ref) ** 2, axis=axis))
    return num / den
