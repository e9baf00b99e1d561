"""Build the in-tree C-ABI library ``libbfapply.so`` (sm_100a CUDA kernels + plan +
host factor builder) with nvcc / g++.  No torch involvement: the library links
only the CUDA runtime (static) and libgomp."""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
LIB = os.path.join(HERE, "libbfapply.so")
BUILD_DIR = os.path.join(HERE, "_build")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr"]
NVCC_FLAGS += [f"-D{m}" for m in os.environ.get("BF_NVCC_DEFINES", "").split()]   # tuning experiments only
CXX_FLAGS = ["-O3", "-std=c++17", "-fPIC", "-fopenmp", "-march=x86-64-v3", "-ffp-contract=off", "-Wall"]

CU_SOURCES = ["bf_kernels.cu", "bf_small.cu", "bf_struct.cu", "bf_recompress.cu", "bf_tc.cu", "bf_band3.cu", "bf_nufft.cu", "bf_plan.cu"]
CXX_SOURCES = ["bf_build.cpp", "bf_decide.cpp"]
HEADERS = ["bf_internal.h", "bf_plan_internal.h", "bf_shard.h", "tc_sm100.cuh"]


def _digest() -> str:
    h = hashlib.sha256()
    for f in CU_SOURCES + CXX_SOURCES + HEADERS:
        with open(os.path.join(CSRC, f), "rb") as fh:
            h.update(fh.read())
    for f in sorted(os.listdir(INCLUDE)):
        with open(os.path.join(INCLUDE, f), "rb") as fh:
            h.update(fh.read())
    h.update(" ".join(ARCH + NVCC_FLAGS + CXX_FLAGS).encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False, out: str | None = None) -> str:
    """Build libbfapply.so (or, with `out`, a tuning variant at that path from a separate build directory)."""
    global LIB, BUILD_DIR
    if out:
        LIB, BUILD_DIR = out, out + ".build"
    stamp = os.path.join(BUILD_DIR, "digest")
    dig = _digest()
    if not force and os.path.exists(LIB) and os.path.exists(stamp) and open(stamp).read() == dig:
        return LIB
    os.makedirs(BUILD_DIR, exist_ok=True)
    jobs = []
    for src in CU_SOURCES:
        obj = os.path.join(BUILD_DIR, src + ".o")
        cmd = [NVCC, *ARCH, *NVCC_FLAGS, "-I", INCLUDE, "-c", os.path.join(CSRC, src), "-o", obj]
        jobs.append((cmd, os.path.join(BUILD_DIR, src + ".ptxas.log"), obj))
    for src in CXX_SOURCES:
        obj = os.path.join(BUILD_DIR, src + ".o")
        cmd = ["g++", *CXX_FLAGS, "-I", INCLUDE, "-I", "/usr/local/cuda/include", "-c", os.path.join(CSRC, src),
               "-o", obj]
        jobs.append((cmd, None, obj))
    from concurrent.futures import ThreadPoolExecutor   # the translation units compile independently
    with ThreadPoolExecutor(max_workers=len(jobs)) as ex:
        for f in [ex.submit(_run, c, log, verbose) for c, log, _ in jobs]:
            f.result()
    objs = [o for _, _, o in jobs]
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-Xcompiler", "-fopenmp", "-lgomp",
           "-L/usr/local/cuda/lib64", "-lcufft", "-Xlinker", "-rpath=/usr/local/cuda/lib64"]
    _run(cmd, None, verbose)
    os.replace(tmp, LIB)
    with open(stamp, "w") as f:
        f.write(dig)
    return LIB


def _run(cmd, log, verbose):
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    p = subprocess.run(cmd, capture_output=True, text=True)
    if log:
        with open(log, "w") as f:
            f.write(p.stdout + p.stderr)
    if p.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{p.stdout}\n{p.stderr}")


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
