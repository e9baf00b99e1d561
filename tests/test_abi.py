"""The C-ABI library loads and exports every symbol include/*.h declares; host-side
argument validation works without a GPU (no compute calls here)."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_1803_04128_b200 import bf

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    names = set()
    for h in ("bf.h", "bf_build.h", "bf_nufft.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*(bf_[a-z0-9_]+)\s*\(", src, re.M):
            names.add(m.group(1))
    return names


def test_header_declarations_are_exported():
    declared = _declared_functions()
    assert len(declared) >= 19
    assert declared == set(bf.EXPORTS)
    L = bf.lib()
    for name in declared:
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", bf.LIB_PATH], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert declared <= exported


def test_no_torch_in_the_abi():
    for h in ("bf.h", "bf_build.h", "bf_nufft.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        assert "torch" not in src.lower().replace("no torch", "") and "at::" not in src
    out = subprocess.run(["ldd", bf.LIB_PATH], capture_output=True, text=True).stdout
    libs = [ln.split()[0] for ln in out.splitlines() if ln.strip()]   # library names (not load addresses)
    assert libs and not any("torch" in x or x.startswith("libc10") for x in libs), libs


def test_abi_version():
    assert bf.lib().bf_abi_version() == bf.BF_ABI_VERSION


def test_validation_errors_without_gpu():
    L = bf.lib()
    h = ctypes.c_void_p()
    d = bf.bf_desc_t(bf.BF_ABI_VERSION, 11, 4, 10, 2, 0)   # odd log2n
    assert L.bf_plan_alloc(ctypes.byref(d), 0, 1, ctypes.byref(h)) == 2          # BF_ERR_SHAPE
    assert "log2n" in L.bf_last_error().decode()
    d = bf.bf_desc_t(bf.BF_ABI_VERSION, 12, 4, 11, 2, 0)   # odd rank
    assert L.bf_plan_alloc(ctypes.byref(d), 0, 1, ctypes.byref(h)) == 7          # BF_ERR_NOT_SUPPORTED
    d = bf.bf_desc_t(bf.BF_ABI_VERSION, 12, 4, 10, 3, 0)   # n_amp 3
    assert L.bf_plan_alloc(ctypes.byref(d), 0, 1, ctypes.byref(h)) == 7
    d = bf.bf_desc_t(bf.BF_ABI_VERSION, 12, 3, 10, 2, 0)   # rank > leaf
    assert L.bf_plan_alloc(ctypes.byref(d), 0, 1, ctypes.byref(h)) == 2
    d = bf.bf_desc_t(99, 12, 4, 10, 2, 0)                   # wrong abi version
    assert L.bf_plan_alloc(ctypes.byref(d), 0, 1, ctypes.byref(h)) == 1
    assert L.bf_apply(None, None, None, 1, None) == 1
    assert L.bf_plan_set_option(None, bf.BF_OPT_TENSOR_CORES, 1) == 1            # NULL plan
    assert L.bf_plan_destroy(None) == 0
    assert L.bf_workspace_bytes(None, 4) == 0


def test_no_device_fails_loudly():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    L = bf.lib()
    h = ctypes.c_void_p()
    d = bf.bf_desc_t(bf.BF_ABI_VERSION, 12, 4, 10, 2, 0)
    st = L.bf_plan_alloc(ctypes.byref(d), 0, 1, ctypes.byref(h))
    assert st in (1, 5) and not h.value      # BF_ERR_INVALID_ARG (no device) or BF_ERR_CUDA
    with pytest.raises(bf.BFError):
        bf.Plan.build_fio(bf.fio(0, 1, 12, 4, 10))


def test_nufft_validation_without_gpu():
    L = bf.lib()
    h = ctypes.c_void_p()
    t = (ctypes.c_double * 32)()
    a = (ctypes.c_float * 64)()
    d = bf.bf_nufft_desc_t(bf.BF_ABI_VERSION, 4, 1, 3, ctypes.addressof(t), ctypes.addressof(a), ctypes.addressof(a), 1e-6)
    assert L.bf_nufft_create(ctypes.byref(d), 0, 1, ctypes.byref(h)) == 2          # n_sub 3: BF_ERR_SHAPE
    d.n_sub, d.eps = 2, 0.5
    assert L.bf_nufft_create(ctypes.byref(d), 0, 1, ctypes.byref(h)) == 2          # eps out of range
    assert "eps" in L.bf_last_error().decode()
    d.targets = None
    assert L.bf_nufft_create(ctypes.byref(d), 0, 1, ctypes.byref(h)) == 1          # null array
    assert L.bf_nufft_apply(None, None, 16, None, 16, 1, None) == 1
    assert L.bf_nufft_destroy(None) == 0
