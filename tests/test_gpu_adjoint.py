"""GPU parity of the adjoint apply (bf_plan_create_adjoint) against
the oracle's O8 (the forward factors conjugate-transposed in reverse order, generated on the fly in FP64).

The adjoint plan re-assembles the forward plan's blocks into a butterfly of the same shape and runs the
forward kernels, so every kernel family is exercised: tiny (nv <= 4), small-batch (8 <= nv < 128), the
tcgen05 tensor-core path (nv >= 64) and the FP32 kernels (odd nv).  Bar: 1e-5 relative l2 per column
(north_star), as for the forward.
"""
import numpy as np
import pytest

import oracle
from paper_1803_04128_b200 import bf
from paper_1803_04128_b200 import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

PARITY = 1e-5


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.init()
    yield


def to_dev(F):
    return torch.from_numpy(np.ascontiguousarray(F.T)).cuda()


def gpu_apply(plan, F):
    Ft = to_dev(F)
    Gt = torch.empty_like(Ft)
    plan.apply(Ft, Gt, F.shape[1])
    torch.cuda.synchronize()
    return np.asfortranarray(Gt.cpu().numpy().T)


CASES = [  # (config, overrides, columns compared)
    ("cfg1", dict(), None),                                   # nv = 2: tiny kernels
    ("cfg1_dft", dict(), None),
    ("cfg2", dict(log2n=14), None),                           # nv = 32: small-batch kernels
    ("cfg5", dict(log2n=16), None),                           # nv = 16
    ("cfg3", dict(log2n=14, nrhs=16), [0, 15]),               # nv = 64, 4 amplitude terms: tensor cores
    ("cfg4", dict(log2n=14, nrhs=128), [0, 77, 127]),         # nv = 256: tensor cores, composed bands
    ("cfg4", dict(log2n=12, nrhs=3), None),                   # odd nv: FP32 kernels
    ("cfg2", dict(log2n=10, log2leaf=5, nrhs=4), None),       # h == l0: no transfer level before the switch
    ("cfg4", dict(log2n=16, log2leaf=5, rank=8, nrhs=64), [0, 63]),   # r = 8, 128 vectors: three-level bands 3 + 3
]


@pytest.mark.parametrize("name,over,cols", CASES)
def test_adjoint_parity(name, over, cols):
    w = W.CONFIGS[name].with_(**over)
    fwd = bf.Plan.build_fio(bf.fio_of(w), max_nrhs_chunk=w.nrhs)
    adj = fwd.adjoint()
    fwd.destroy()
    F = W.rhs(w.n, w.nrhs, w.seed + 500)
    G = gpu_apply(adj, F)
    info = adj.info()
    adj.destroy()
    cols = list(range(w.nrhs)) if cols is None else cols
    R = oracle.bf_apply_adjoint(w.kernel, w.amp, w.log2n, w.log2leaf, w.rank, F[:, cols])
    err = oracle.rel_l2(G[:, cols].astype(np.complex128), R, axis=0)
    assert np.all(err <= PARITY), (name, over, info["tc_classes"], err)


@pytest.mark.parametrize("name,over", [("cfg2", dict(log2n=14)), ("cfg4", dict(log2n=14, nrhs=128)),
                                       ("cfg1", dict())])
def test_adjoint_of_adjoint_is_forward_bitwise(name, over):
    # the re-assembly is exact and an involution on the blocks: (K*)* runs the forward's blocks in the same
    # kernels, so the results are bitwise equal
    w = W.CONFIGS[name].with_(**over)
    fwd = bf.Plan.build_fio(bf.fio_of(w), max_nrhs_chunk=w.nrhs)
    adj = fwd.adjoint()
    adj2 = adj.adjoint()
    F = W.rhs(w.n, w.nrhs, w.seed + 600)
    G1 = gpu_apply(fwd, F)
    G2 = gpu_apply(adj2, F)
    for p in (fwd, adj, adj2):
        p.destroy()
    assert np.array_equal(G1, G2)


def test_adjoint_inner_product_identity_tensor_cores():
    # <K f, g> = <f, K* g> with both applies on the GPU at a size beyond the oracle's dense assembly
    w = W.CONFIGS["cfg4"].with_(log2n=16, nrhs=128)
    fwd = bf.Plan.build_fio(bf.fio_of(w), max_nrhs_chunk=w.nrhs)
    adj = fwd.adjoint()
    f = W.rhs(w.n, w.nrhs, 71)
    g = W.rhs(w.n, w.nrhs, 72)
    Kf = gpu_apply(fwd, f).astype(np.complex128)
    Ksg = gpu_apply(adj, g).astype(np.complex128)
    assert "s0" in adj.info()["tc_classes"]
    fwd.destroy()
    adj.destroy()
    lhs = np.sum(np.conj(g.astype(np.complex128)) * Kf, axis=0)
    rhs = np.sum(np.conj(Ksg) * f.astype(np.complex128), axis=0)
    scale = np.linalg.norm(g, axis=0) * np.linalg.norm(Kf, axis=0)
    assert np.all(np.abs(lhs - rhs) <= 1e-5 * scale)


def test_adjoint_errors():
    w = W.CONFIGS["cfg1"]
    k = bf.fio_of(w)
    with pytest.raises(bf.BFError):   # not finalized
        import ctypes
        meta = bf.bf_desc_t(bf.BF_ABI_VERSION, w.log2n, w.log2leaf, w.rank, w.n_amp, bf.BF_MEM_HOST,
                            None, None, None, None, None, None)
        h = ctypes.c_void_p()
        bf._check(bf.lib().bf_plan_alloc(ctypes.byref(meta), 0, 1, ctypes.byref(h)))
        p = bf.Plan(h.value)
        p.adjoint()
    emu = bf.Plan.build_fio_emulated(k, world=2, max_nrhs_chunk=1) if w.log2n >= 2 * w.log2leaf + 2 else None
    if emu is not None:
        with pytest.raises(bf.BFError):
            emu.adjoint()
        emu.destroy()
