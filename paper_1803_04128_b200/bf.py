"""Thin ctypes binding of the C ABI in include/bf.h and include/bf_build.h.

Argument marshalling only: every step of the apply runs in the CUDA kernels of
``libbfapply.so``; the factors are built by the library's host builder.  There
is no Python or CPU fallback: if the library is missing or a call fails, an
exception is raised.  Torch is used by callers only for device memory and
streams (pass ``tensor.data_ptr()`` and ``torch.cuda.current_stream().cuda_stream``
or hand tensors directly to the helpers below).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BF_LIB") or os.path.join(HERE, "libbfapply.so")   # BF_LIB: tuning variants only

BF_ABI_VERSION = 1
BF_MEM_HOST, BF_MEM_DEVICE = 0, 1
BF_STAGE_V0, BF_STAGE_SW, BF_STAGE_U, BF_STAGE_AMP_A, BF_STAGE_AMP_B, BF_STAGE_XFER0 = 0, 1, 2, 3, 4, 16
BF_NUM_KCLASS = 6
KCLASS_NAMES = ("s0", "xfer_first_half", "xfer_switch", "xfer_second_half", "sl", "exchange")
BF_SHARD_NONE, BF_SHARD_NCCL, BF_SHARD_EMULATED = 0, 1, 2
BF_OPT_TENSOR_CORES = 1
BF_OPT_EXCHANGE = 4
BF_OPT_BAND_COMPOSE = 5
BF_OPT_HOST_PIECES = 8
BF_OPT_LEAF_MULTICAST = 9
BF_OPT_SMALL_BATCH = 10
BF_OPT_BAND_PRECOMPOSE = 11
BF_OPT_BAND3 = 12
STATUS = {0: "BF_OK", 1: "BF_ERR_INVALID_ARG", 2: "BF_ERR_SHAPE", 3: "BF_ERR_ALIGNMENT", 4: "BF_ERR_OOM",
          5: "BF_ERR_CUDA", 6: "BF_ERR_NCCL", 7: "BF_ERR_NOT_SUPPORTED", 8: "BF_ERR_STATE"}

# every symbol include/*.h declares (checked by tests/test_abi.py)
EXPORTS = ("bf_plan_create", "bf_plan_alloc", "bf_plan_upload", "bf_plan_finalize", "bf_apply", "bf_apply_ex", "bf_apply_graph",
           "bf_apply_host", "bf_apply_host_async", "bf_apply_host_wait", "bf_workspace_bytes", "bf_plan_get_info", "bf_plan_set_timing", "bf_plan_timing", "bf_plan_set_option",
           "bf_plan_destroy", "bf_last_error", "bf_abi_version", "bf_build_n_amp", "bf_build_amp", "bf_build_blocks",
           "bf_build_block_elems", "bf_plan_build_fio", "bf_nccl_get_unique_id", "bf_plan_alloc_sharded",
           "bf_plan_create_sharded", "bf_shard_pairs", "bf_plan_build_fio_sharded", "bf_plan_build_fio_emulated", "bf_plan_create_adjoint",
           "bf_plan_create_structured", "bf_plan_build_fio_structured", "bf_build_structured",
           "bf_build_structured_lag", "bf_plan_recompress", "bf_nufft_create", "bf_nufft_apply",
           "bf_nufft_get_info", "bf_nufft_destroy", "bf_nufft_build_fio", "bf_nufft_decide")


class BFError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class bf_desc_t(ctypes.Structure):
    _fields_ = [("abi_version", ctypes.c_int32), ("log2n", ctypes.c_int32), ("log2leaf", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("n_amp", ctypes.c_int32), ("memory", ctypes.c_int32),
                ("amp_a", ctypes.c_void_p), ("amp_b", ctypes.c_void_p), ("v0", ctypes.c_void_p),
                ("xfer", ctypes.POINTER(ctypes.c_void_p)), ("sw", ctypes.c_void_p), ("u", ctypes.c_void_p)]


class bf_plan_info_t(ctypes.Structure):
    _fields_ = [("log2n", ctypes.c_int32), ("log2leaf", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("n_amp", ctypes.c_int32), ("switch_level", ctypes.c_int32), ("n_xfer", ctypes.c_int32),
                ("n", ctypes.c_int64), ("max_nrhs_chunk", ctypes.c_int64), ("factor_bytes", ctypes.c_int64),
                ("workspace_bytes", ctypes.c_int64), ("launches_per_chunk", ctypes.c_int32),
                ("device", ctypes.c_int32), ("class_launches", ctypes.c_int32 * 6),
                ("class_levels", ctypes.c_int32 * 6), ("world", ctypes.c_int32), ("shard_rank", ctypes.c_int32),
                ("sharding", ctypes.c_int32), ("rows_local", ctypes.c_int64), ("tc_weight_bytes", ctypes.c_int64),
                ("tc_class_mask", ctypes.c_int32), ("structured", ctypes.c_int32)]


class bf_fio_t(ctypes.Structure):
    _fields_ = [("abi_version", ctypes.c_int32), ("kernel", ctypes.c_int32), ("amp", ctypes.c_int32),
                ("log2n", ctypes.c_int32), ("log2leaf", ctypes.c_int32), ("rank", ctypes.c_int32)]


_lib = None


class bf_nufft_desc_t(ctypes.Structure):
    _fields_ = [("abi_version", ctypes.c_int32), ("log2n", ctypes.c_int32), ("n_amp", ctypes.c_int32),
                ("n_sub", ctypes.c_int32), ("targets", ctypes.c_void_p), ("amp_a", ctypes.c_void_p),
                ("amp_b", ctypes.c_void_p), ("eps", ctypes.c_double)]


class bf_nufft_decide_t(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int64), ("n", ctypes.c_int64), ("r1", ctypes.c_int32), ("r2", ctypes.c_int32),
                ("u1", ctypes.c_void_p), ("v1", ctypes.c_void_p), ("u2", ctypes.c_void_p), ("v2", ctypes.c_void_p),
                ("xi", ctypes.c_void_p), ("rank_budget", ctypes.c_int32), ("q", ctypes.c_int32),
                ("eps", ctypes.c_double), ("seed", ctypes.c_uint64)]


def nufft_decide(u1, v1, u2, v2, xi=None, rank_budget: int = 4, q: int = 8, eps: float = 1e-9, seed: int = 0,
                 want_targets: bool = True):
    """Algorithm 6 (bf_nufft_decide) on host factors: u1 [r1][m], v1 [r1][n] real; u2 [r2][m], v2 [r2][n] complex.
    Returns (y, n_rank, targets or None)."""
    u1 = np.ascontiguousarray(u1, np.float64)
    v1 = np.ascontiguousarray(v1, np.float64)
    u2 = np.ascontiguousarray(u2, np.complex128)
    v2 = np.ascontiguousarray(v2, np.complex128)
    m, n = u1.shape[1], v1.shape[1]
    xa = None if xi is None else np.ascontiguousarray(xi, np.float64)
    d = bf_nufft_decide_t(m, n, u1.shape[0], u2.shape[0], u1.ctypes.data, v1.ctypes.data, u2.ctypes.data,
                          v2.ctypes.data, None if xa is None else xa.ctypes.data, rank_budget, q, eps, seed)
    y, nr = ctypes.c_int32(), ctypes.c_int32()
    t = np.zeros(m, np.float64) if (want_targets and xa is not None) else None
    _check(lib().bf_nufft_decide(ctypes.byref(d), ctypes.byref(y), ctypes.byref(nr),
                                 None if t is None else t.ctypes.data))
    return int(y.value), int(nr.value), (t if y.value else None)


class bf_nufft_info_t(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("width", ctypes.c_int32), ("beta", ctypes.c_double), ("grid", ctypes.c_int64),
                ("workspace_bytes", ctypes.c_int64), ("launches_per_chunk", ctypes.c_int32)]


def lib():
    """Load libbfapply.so (fails loudly when the CUDA extension is missing)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        if "BF_NCCL_LIB" not in os.environ:
            # index-sharded plans dlopen NCCL on first use: point them at the NCCL torch.distributed uses
            # (the nvidia-nccl wheel), not whichever libnccl.so.2 the loader finds first
            import importlib.util
            try:
                spec = importlib.util.find_spec("nvidia.nccl")
            except (ImportError, ValueError):
                spec = None
            for d in (spec.submodule_search_locations or []) if spec else []:
                cand = os.path.join(d, "lib", "libnccl.so.2")
                if os.path.exists(cand):
                    os.environ["BF_NCCL_LIB"] = cand
                    break
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
        P = ctypes.POINTER
        sigs = {
            "bf_plan_create": ([P(bf_desc_t), ctypes.c_int, i64, P(vp)], i32),
            "bf_plan_alloc": ([P(bf_desc_t), ctypes.c_int, i64, P(vp)], i32),
            "bf_plan_upload": ([vp, i32, i64, i64, vp, i32], i32),
            "bf_plan_finalize": ([vp], i32),
            "bf_plan_create_adjoint": ([vp, i64, P(vp)], i32),
            "bf_plan_recompress": ([vp, i32, i64, P(vp)], i32),
            "bf_plan_create_structured": ([vp, ctypes.c_int, i64, P(vp)], i32),
            "bf_build_structured": ([P(bf_fio_t), i32, i64, i64, vp], i32),
            "bf_build_structured_lag": ([P(bf_fio_t), i32, vp], i32),
            "bf_plan_build_fio_structured": ([P(bf_fio_t), ctypes.c_int, i64, i64, P(vp)], i32),
            "bf_apply": ([vp, vp, vp, i64, vp], i32),
            "bf_apply_ex": ([vp, vp, i64, vp, i64, i64, vp, sz, vp], i32),
            "bf_apply_graph": ([vp, vp, vp, i64, vp], i32),
            "bf_apply_host": ([vp, vp, vp, i64, vp], i32),
            "bf_apply_host_async": ([vp, vp, vp, i64, vp], i32),
            "bf_apply_host_wait": ([vp], i32),
            "bf_workspace_bytes": ([vp, i64], sz),
            "bf_plan_get_info": ([vp, P(bf_plan_info_t)], i32),
            "bf_plan_set_timing": ([vp, i32], i32),
            "bf_plan_set_option": ([vp, i32, ctypes.c_int64], i32),
            "bf_plan_timing": ([vp, P(ctypes.c_double), P(i64)], i32),
            "bf_plan_destroy": ([vp], i32),
            "bf_last_error": ([], ctypes.c_char_p),
            "bf_abi_version": ([], i32),
            "bf_build_n_amp": ([i32], i32),
            "bf_build_amp": ([P(bf_fio_t), vp, vp], i32),
            "bf_build_blocks": ([P(bf_fio_t), i32, i64, i64, vp], i32),
            "bf_build_block_elems": ([P(bf_fio_t), i32], i64),
            "bf_plan_build_fio": ([P(bf_fio_t), ctypes.c_int, i64, i64, P(vp)], i32),
            "bf_nccl_get_unique_id": ([vp], i32),
            "bf_plan_alloc_sharded": ([P(bf_desc_t), ctypes.c_int, i64, i32, i32, vp, P(vp)], i32),
            "bf_plan_create_sharded": ([P(bf_desc_t), ctypes.c_int, i64, i32, i32, vp, P(vp)], i32),
            "bf_shard_pairs": ([i32, i32, i32, i32, i32, vp], i32),
            "bf_plan_build_fio_sharded": ([P(bf_fio_t), ctypes.c_int, i32, i32, vp, i64, i64, P(vp)], i32),
            "bf_plan_build_fio_emulated": ([P(bf_fio_t), ctypes.c_int, i32, i64, i64, P(vp)], i32),
            "bf_nufft_create": ([P(bf_nufft_desc_t), ctypes.c_int, i64, P(vp)], i32),
            "bf_nufft_apply": ([vp, vp, i64, vp, i64, i64, vp], i32),
            "bf_nufft_get_info": ([vp, P(bf_nufft_info_t)], i32),
            "bf_nufft_destroy": ([vp], i32),
            "bf_nufft_build_fio": ([P(bf_fio_t), ctypes.c_int, i64, ctypes.c_double, P(vp)], i32),
            "bf_nufft_decide": ([P(bf_nufft_decide_t), P(i32), P(i32), vp], i32),
        }
        for name, (args, res) in sigs.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        if L.bf_abi_version() != BF_ABI_VERSION:
            raise ImportError("libbfapply.so ABI version mismatch")
        _lib = L
    return _lib


def _check(status: int):
    if status != 0:
        raise BFError(status, lib().bf_last_error().decode())


def fio(kernel: int, amp: int, log2n: int, log2leaf: int, rank: int) -> bf_fio_t:
    return bf_fio_t(BF_ABI_VERSION, kernel, amp, log2n, log2leaf, rank)


def fio_of(w) -> bf_fio_t:
    """bf_fio_t of a workloads.Workload."""
    return fio(w.kernel, w.amp, w.log2n, w.log2leaf, w.rank)


def build_amp(k: bf_fio_t):
    """(a, b) complex64 [n_amp][N] from the host builder."""
    na = lib().bf_build_n_amp(k.amp)
    if na < 1:
        raise BFError(1, f"unknown amplitude id {k.amp}")
    n = 1 << k.log2n
    a = np.zeros((na, n), np.complex64)
    b = np.zeros((na, n), np.complex64)
    _check(lib().bf_build_amp(ctypes.byref(k), a.ctypes.data, b.ctypes.data))
    return a, b


def build_blocks(k: bf_fio_t, stage: int, begin: int, count: int) -> np.ndarray:
    """count blocks of `stage` from the host builder, complex64, each flattened (bf.h layouts)."""
    e = lib().bf_build_block_elems(ctypes.byref(k), stage)
    if e <= 0:
        raise ValueError("bad stage")
    out = np.zeros((count, e), np.complex64)
    _check(lib().bf_build_blocks(ctypes.byref(k), stage, begin, count, out.ctypes.data))
    return out


def build_structured(k: bf_fio_t, stage: int, begin: int, count: int, per: int) -> np.ndarray:
    """Host builder: structured per-pair data of one stage (`per` complex64 per pair; bf_build.h)."""
    out = np.zeros((count, per), np.complex64)
    _check(lib().bf_build_structured(ctypes.byref(k), stage, begin, count, out.ctypes.data))
    return out


def build_structured_lag(k: bf_fio_t, stage: int, size: int) -> np.ndarray:
    out = np.zeros(size, np.float32)
    _check(lib().bf_build_structured_lag(ctypes.byref(k), stage, out.ctypes.data))
    return out


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId (to broadcast to every rank of an index-sharded plan)."""
    buf = ctypes.create_string_buffer(128)
    _check(lib().bf_nccl_get_unique_id(buf))
    return buf.raw


def shard_pairs(log2n: int, log2leaf: int, world: int, rank: int, which: int) -> np.ndarray:
    """Global level-h pair indices of a rank's send buffer (0), receive buffer (1) or second-half order (2)."""
    out = np.zeros((1 << log2n) // world, np.int64)
    _check(lib().bf_shard_pairs(log2n, log2leaf, world, rank, which, out.ctypes.data))
    return out


def _ptr(x) -> int:
    """Device/host pointer of a torch tensor, numpy array or raw int."""
    if isinstance(x, int):
        return x
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()


def _stream(stream) -> int:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


class Plan:
    """Owns a bf_plan_t."""

    def __init__(self, handle: int):
        self._h = ctypes.c_void_p(handle)

    # -- construction ------------------------------------------------------------
    @classmethod
    def build_fio(cls, k: bf_fio_t, device: int = 0, max_nrhs_chunk: int = 1, staging_bytes: int = 256 << 20):
        """Host builder -> streaming upload -> finalized plan (bf_plan_build_fio)."""
        h = ctypes.c_void_p()
        _check(lib().bf_plan_build_fio(ctypes.byref(k), device, max_nrhs_chunk, staging_bytes, ctypes.byref(h)))
        return cls(h.value)

    @classmethod
    def build_fio_structured(cls, k: bf_fio_t, device: int = 0, max_nrhs_chunk: int = 1,
                             staging_bytes: int = 256 << 20):
        """Structured interpolative factors (phases + shared Lagrange matrices, NEXT-1) -> finalized plan."""
        h = ctypes.c_void_p()
        _check(lib().bf_plan_build_fio_structured(ctypes.byref(k), device, max_nrhs_chunk, staging_bytes,
                                                  ctypes.byref(h)))
        return cls(h.value)

    @classmethod
    def build_fio_sharded(cls, k: bf_fio_t, rank: int, world: int, nccl_id: bytes, device: int = 0,
                          max_nrhs_chunk: int = 1, staging_bytes: int = 256 << 20):
        """This rank's shard of the index-sharded plan; bf_apply then takes the local N/world rows."""
        h = ctypes.c_void_p()
        idb = ctypes.create_string_buffer(nccl_id, 128)
        _check(lib().bf_plan_build_fio_sharded(ctypes.byref(k), device, rank, world, idb, max_nrhs_chunk,
                                               staging_bytes, ctypes.byref(h)))
        return cls(h.value)

    @classmethod
    def build_fio_emulated(cls, k: bf_fio_t, world: int, device: int = 0, max_nrhs_chunk: int = 1,
                           staging_bytes: int = 256 << 20):
        """All `world` index shards on one device (exchange by device copies); full N-row F/G."""
        h = ctypes.c_void_p()
        _check(lib().bf_plan_build_fio_emulated(ctypes.byref(k), device, world, max_nrhs_chunk, staging_bytes,
                                                ctypes.byref(h)))
        return cls(h.value)

    @classmethod
    def from_arrays(cls, log2n, log2leaf, rank, amp_a, amp_b, v0, xfer, sw, u, device=0, max_nrhs_chunk=1,
                    memory=BF_MEM_HOST):
        """bf_plan_create from complete factor arrays (numpy complex64 host arrays or device tensors)."""
        xs = (ctypes.c_void_p * max(1, len(xfer)))(*[_ptr(x) for x in xfer])
        d = bf_desc_t(BF_ABI_VERSION, log2n, log2leaf, rank, amp_a.shape[0], memory, _ptr(amp_a), _ptr(amp_b),
                      _ptr(v0), ctypes.cast(xs, ctypes.POINTER(ctypes.c_void_p)), _ptr(sw), _ptr(u))
        h = ctypes.c_void_p()
        _check(lib().bf_plan_create(ctypes.byref(d), device, max_nrhs_chunk, ctypes.byref(h)))
        return cls(h.value)

    def adjoint(self, max_nrhs_chunk: int | None = None) -> "Plan":
        """bf_plan_create_adjoint: a new plan applying K* = sum_k conj(b_k) o BF*(conj(a_k) o .), built on the
        device from this (finalized, unsharded) plan's factors."""
        if max_nrhs_chunk is None:
            max_nrhs_chunk = self.info()["max_nrhs_chunk"]
        h = ctypes.c_void_p()
        _check(lib().bf_plan_create_adjoint(self._h, max_nrhs_chunk, ctypes.byref(h)))
        return Plan(h.value)

    def recompress(self, rank: int, max_nrhs_chunk: int | None = None) -> "Plan":
        """bf_plan_recompress: a new plan of rank `rank` (balanced truncation of this plan's factors, NEXT-3)."""
        if max_nrhs_chunk is None:
            max_nrhs_chunk = self.info()["max_nrhs_chunk"]
        h = ctypes.c_void_p()
        _check(lib().bf_plan_recompress(self._h, rank, max_nrhs_chunk, ctypes.byref(h)))
        return Plan(h.value)

    # -- apply ---------------------------------------------------------------------
    def apply(self, F, G, nrhs: int, stream=None):
        """G = sum_k a_k o BF(b_k o F) on device buffers (N x nrhs column-major, ld = N)."""
        _check(lib().bf_apply(self._h, _ptr(F), _ptr(G), nrhs, _stream(stream)))

    def apply_graph(self, F, G, nrhs: int, stream=None):
        """As apply, as one launch of the plan's cached CUDA graph of it (captured at the first call with these
        F, G, nrhs; include/bf.h bf_apply_graph)."""
        _check(lib().bf_apply_graph(self._h, _ptr(F), _ptr(G), nrhs, _stream(stream)))

    def apply_ex(self, F, ldf, G, ldg, nrhs, workspace=None, workspace_bytes=0, stream=None):
        _check(lib().bf_apply_ex(self._h, _ptr(F), ldf, _ptr(G), ldg, nrhs,
                                 None if workspace is None else _ptr(workspace), workspace_bytes, _stream(stream)))

    def apply_host(self, F_host, G_host, nrhs: int, stream=None):
        """End to end with host buffers (copies inside the call)."""
        _check(lib().bf_apply_host(self._h, _ptr(F_host), _ptr(G_host), nrhs, _stream(stream)))

    def apply_host_async(self, F_host, G_host, nrhs: int, stream=None):
        """End to end with (pinned) host buffers, asynchronous: returns at once; see apply_host_wait."""
        _check(lib().bf_apply_host_async(self._h, _ptr(F_host), _ptr(G_host), nrhs, _stream(stream)))

    def apply_host_wait(self):
        _check(lib().bf_apply_host_wait(self._h))

    # -- introspection -------------------------------------------------------------
    def info(self) -> dict:
        i = bf_plan_info_t()
        _check(lib().bf_plan_get_info(self._h, ctypes.byref(i)))
        out = {f: getattr(i, f) for f, _ in bf_plan_info_t._fields_}
        out["class_launches"] = dict(zip(KCLASS_NAMES, list(i.class_launches)))
        out["class_levels"] = dict(zip(KCLASS_NAMES, list(i.class_levels)))
        out["tc_classes"] = [n for c, n in enumerate(KCLASS_NAMES) if i.tc_class_mask >> c & 1]
        return out

    def workspace_bytes(self, nrhs_chunk: int) -> int:
        return int(lib().bf_workspace_bytes(self._h, nrhs_chunk))

    def set_option(self, option: int, value: int):
        _check(lib().bf_plan_set_option(self._h, int(option), int(value)))

    def set_tensor_cores(self, enable: bool):
        self.set_option(BF_OPT_TENSOR_CORES, int(enable))

    def set_timing(self, enable: bool):
        _check(lib().bf_plan_set_timing(self._h, int(enable)))

    def timing(self):
        ms = (ctypes.c_double * BF_NUM_KCLASS)()
        n = (ctypes.c_int64 * BF_NUM_KCLASS)()
        _check(lib().bf_plan_timing(self._h, ms, n))
        return {KCLASS_NAMES[i]: (ms[i], n[i]) for i in range(BF_NUM_KCLASS)}

    def destroy(self):
        if self._h is not None and self._h.value:
            _check(lib().bf_plan_destroy(self._h))
        self._h = None

    def __del__(self):
        try:
            if getattr(self, "_h", None) is not None and self._h.value:
                lib().bf_plan_destroy(self._h)
        except Exception:
            pass


class NufftPlan:
    """Owns a bf_nufft_t: the NUFFT path of include/bf_nufft.h (eqn:tg3 with one-dimensional type-2 NUFFTs on the
    frequency submatrices)."""

    def __init__(self, handle: int):
        self._h = ctypes.c_void_p(handle)

    @classmethod
    def build_fio(cls, k: bf_fio_t, device: int = 0, max_nrhs_chunk: int = 1, eps: float = 1e-6):
        """Closed-form targets t_-(x) = x - c(x), t_+(x) = x + c(x) and the amplitude split (bf_nufft_build_fio)."""
        h = ctypes.c_void_p()
        _check(lib().bf_nufft_build_fio(ctypes.byref(k), device, max_nrhs_chunk, eps, ctypes.byref(h)))
        return cls(h.value)

    @classmethod
    def create(cls, targets: np.ndarray, amp_a: np.ndarray, amp_b: np.ndarray, eps: float = 1e-6, device: int = 0,
               max_nrhs_chunk: int = 1):
        """targets: float64 [n_sub][N]; amp_a, amp_b: complex64 [n_amp][N] (host arrays, copied)."""
        t = np.ascontiguousarray(targets, np.float64)
        a = np.ascontiguousarray(amp_a, np.complex64)
        b = np.ascontiguousarray(amp_b, np.complex64)
        n_sub, N = t.shape
        d = bf_nufft_desc_t(BF_ABI_VERSION, int(N).bit_length() - 1, a.shape[0], n_sub, t.ctypes.data, a.ctypes.data,
                            b.ctypes.data, eps)
        h = ctypes.c_void_p()
        _check(lib().bf_nufft_create(ctypes.byref(d), device, max_nrhs_chunk, ctypes.byref(h)))
        return cls(h.value)

    def apply(self, F, G, nrhs: int, ldf: int = 0, ldg: int = 0, stream=None):
        """G = the NUFFT path applied to F (device buffers, N x nrhs column-major; ld 0 = N)."""
        n = self.n
        _check(lib().bf_nufft_apply(self._h, _ptr(F), ldf or n, _ptr(G), ldg or n, nrhs, _stream(stream)))

    def info(self) -> dict:
        i = bf_nufft_info_t()
        _check(lib().bf_nufft_get_info(self._h, ctypes.byref(i)))
        return {f: getattr(i, f) for f, _ in bf_nufft_info_t._fields_}

    @property
    def n(self) -> int:
        return int(self.info()["n"])

    def destroy(self):
        if self._h is not None and self._h.value:
            _check(lib().bf_nufft_destroy(self._h))
        self._h = None
