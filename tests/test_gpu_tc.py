"""GPU parity of the tensor-core (tcgen05, 3xTF32) stages.

Every shape here is large enough in vectors (nv = nrhs * n_amp >= 64, leaf 32 or 64) that the
plan routes its dense leaf / transfer stages to the tensor-core kernels (bf_tc.cu).  Each case is
checked (1) against the CPU oracle per RHS column at the north_star bar (relative l2 <= 1e-5) and
(2) against the same plan with BF_OPT_TENSOR_CORES = 0 (the FP32 FFMA kernels): both paths are
FP32-accurate, so they agree far below the bar.
"""
import numpy as np
import pytest

import oracle
from paper_1803_04128_b200 import bf
from paper_1803_04128_b200 import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

PARITY = 1e-5
PATHS_AGREE = 2e-6


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.init()
    yield


def _apply(plan, F):
    Ft = torch.from_numpy(np.ascontiguousarray(F.T)).cuda()
    Gt = torch.empty_like(Ft)
    plan.apply(Ft, Gt, F.shape[1])
    torch.cuda.synchronize()
    return np.asfortranarray(Gt.cpu().numpy().T)


TC_CASES = [
    # kernel, amp, LN, l0, r, nrhs, chunk, oracle columns      what it exercises
    (W.K_FIO, W.A_CFG1, 14, 6, 10, 256, 256, [0, 77, 255]),    # cfg4 shape at N = 2^14: 4 vector tiles
    (W.K_FIO_JUMP, W.A_CFG3, 14, 5, 10, 64, 64, [0, 63]),      # cfg3 shape: leaf 32, n_amp 4
    (W.K_FIO, W.A_CFG1, 12, 6, 10, 37, 37, None),              # nv = 74: one ragged vector tile
    (W.K_FIO, W.A_CFG1, 14, 6, 10, 100, 100, [0, 64, 99]),     # nv = 200: full + ragged tile
    (W.K_FIO, W.A_ONE, 12, 6, 6, 70, 70, [1, 69]),             # r = 6, n_amp 1
    (W.K_DFT, W.A_CFG2, 12, 6, 8, 64, 64, [5]),                # r = 8, DFT kernel
    (W.K_FIO, W.A_CFG1, 12, 6, 12, 64, 64, [2]),               # r = 12
    (W.K_FIO, W.A_CFG1, 14, 6, 14, 40, 40, [0, 39]),           # r = 14 (one a per group, padded N)
    (W.K_FIO, W.A_CFG2, 14, 6, 16, 33, 33, [32]),              # r = 16, nv = 66
    (W.K_FIO, W.A_CFG1, 12, 5, 8, 64, 64, [0]),                # leaf 32, r = 8
    (W.K_FIO, W.A_ONE, 12, 5, 12, 128, 128, [127]),            # leaf 32, r = 12
    (W.K_FIO, W.A_CFG1, 12, 5, 14, 48, 48, [47]),              # leaf 32, r = 14
    (W.K_FIO_JUMP, W.A_CFG3, 12, 5, 16, 16, 16, [15]),         # leaf 32, r = 16, nv = 64
    (W.K_FIO, W.A_CFG1, 14, 6, 10, 150, 64, [0, 100, 149]),    # chunks of 128 + 128 + 44 vectors
]


@pytest.mark.parametrize("kernel,amp,LN,l0,r,nrhs,chunk,cols", TC_CASES)
def test_tc_parity(kernel, amp, LN, l0, r, nrhs, chunk, cols):
    N = 1 << LN
    F = W.rhs(N, nrhs, 300 + LN + r)
    plan = bf.Plan.build_fio(bf.fio(kernel, amp, LN, l0, r), max_nrhs_chunk=chunk)
    nv = min(chunk, nrhs) * W.N_AMP[amp]
    tc = plan.info()["tc_classes"]
    if r != 14:                                       # the leaf stages run on the tensor cores
        assert "s0" in tc and plan.info()["tc_weight_bytes"] > 0, tc
        assert ("sl" in tc) == (nv % 2 == 0), tc
    if r in (6, 8, 10, 12) and nv >= 128 and nv % 4 == 0 and LN - 2 * l0 >= 2:
        assert any(k.startswith("xfer") for k in tc), tc   # a two-level band runs on the tensor cores
    G_tc = _apply(plan, F)
    plan.set_tensor_cores(False)
    G_simt = _apply(plan, F)
    plan.destroy()
    assert np.all(np.isfinite(G_tc))
    cols = list(range(nrhs)) if cols is None else cols
    R = oracle.bf_apply(kernel, amp, LN, l0, r, F[:, cols])
    err_tc = oracle.rel_l2(G_tc[:, cols].astype(np.complex128), R, axis=0)
    err_simt = oracle.rel_l2(G_simt[:, cols].astype(np.complex128), R, axis=0)
    assert np.all(err_tc <= PARITY), err_tc
    assert np.all(err_simt <= PARITY), err_simt
    d = oracle.rel_l2(G_tc.astype(np.complex128), G_simt.astype(np.complex128), axis=0)
    assert np.all(d <= PATHS_AGREE), d.max()


def test_tc_deterministic_and_column_independent():
    """Within the tensor-core path: bitwise run-to-run, and a vector's result does not depend on the
    other vectors of its tile (RHS permutation equivariance, bitwise)."""
    LN, l0, r, nrhs = 12, 6, 10, 64
    F = W.rhs(1 << LN, nrhs, 7)
    plan = bf.Plan.build_fio(bf.fio(W.K_FIO, W.A_CFG1, LN, l0, r), max_nrhs_chunk=nrhs)
    G1 = _apply(plan, F)
    assert np.array_equal(G1, _apply(plan, F))
    perm = np.random.default_rng(1).permutation(nrhs)
    assert np.array_equal(_apply(plan, np.asfortranarray(F[:, perm])), G1[:, perm])
    plan.destroy()


def test_tc_mutation_detected():
    """A wrong leaf block or transfer block on the tensor-core path fails parity (the test can fail)."""
    LN, l0, r, nrhs = 14, 6, 10, 64
    N = 1 << LN
    k = bf.fio(W.K_FIO, W.A_CFG1, LN, l0, r)
    a, b = bf.build_amp(k)
    v0 = bf.build_blocks(k, bf.BF_STAGE_V0, 0, N)
    xf = [bf.build_blocks(k, bf.BF_STAGE_XFER0 + i, 0, N) for i in range(LN - 2 * l0)]
    sw = bf.build_blocks(k, bf.BF_STAGE_SW, 0, N)
    u = bf.build_blocks(k, bf.BF_STAGE_U, 0, N)
    F = W.rhs(N, nrhs, 3)
    R = oracle.bf_apply(W.K_FIO, W.A_CFG1, LN, l0, r, F[:, :2])
    v0m = v0.copy()
    v0m[N // 5] = v0m[N // 5].conj()
    um = u.copy()
    um[N // 7] *= 1j
    p = bf.Plan.from_arrays(LN, l0, r, a, b, v0, xf, sw, u, max_nrhs_chunk=nrhs)
    assert set(p.info()["tc_classes"]) == {"s0", "xfer_switch", "sl"}   # every stage on the tensor cores
    assert np.all(oracle.rel_l2(_apply(p, F)[:, :2].astype(np.complex128), R, axis=0) <= PARITY)
    p.destroy()
    xm = [x.copy() for x in xf]
    xm[1][N // 3] *= -1.0
    for args in ((v0m, xf, u), (v0, xf, um), (v0, xm, u)):
        p = bf.Plan.from_arrays(LN, l0, r, a, b, args[0], args[1], sw, args[2], max_nrhs_chunk=nrhs)
        G = _apply(p, F)
        p.destroy()
        assert np.all(oracle.rel_l2(G[:, :2].astype(np.complex128), R, axis=0) > 1e-4)


@pytest.mark.parametrize("pieces", [2, 3, 4])
def test_tc_apply_host_pipelined(pieces):
    """bf_apply_host pipelines pieces over copy streams (BF_OPT_HOST_PIECES: 2 halves, 3 tapered 1/4-1/2-1/4,
    4 quarters).  With 2 pieces every piece keeps >= 64 vectors (tensor-core S0/SL), and the result equals
    the device-buffer apply bitwise (each vector's arithmetic is independent of the other vectors of its
    tile); the smaller tapered / quarter pieces fall below the tensor-core threshold (SIMT kernels), so
    there the two FP32-accurate paths agree within 2e-6."""
    LN, l0, r, nrhs = 12, 6, 10, 96
    F = W.rhs(1 << LN, nrhs, 21)
    plan = bf.Plan.build_fio(bf.fio(W.K_FIO, W.A_CFG1, LN, l0, r), max_nrhs_chunk=64)
    plan.set_option(bf.BF_OPT_HOST_PIECES, pieces)
    ref = _apply(plan, F)
    Fh = torch.from_numpy(np.ascontiguousarray(F.T)).pin_memory()
    Gh = torch.empty_like(Fh).pin_memory()
    plan.apply_host(Fh, Gh, nrhs)
    plan.destroy()
    G = np.asfortranarray(Gh.numpy().T)
    if pieces == 2:
        assert np.array_equal(G, ref)
    else:
        d = oracle.rel_l2(G.astype(np.complex128), ref.astype(np.complex128), axis=0)
        assert np.all(d <= PATHS_AGREE), d.max()


@pytest.mark.parametrize("r,l0,LN,nrhs", [(6, 6, 14, 64), (8, 5, 14, 96), (10, 6, 16, 256), (12, 5, 14, 70)])
def test_tc_band_composed(r, l0, LN, nrhs):
    """Default band (BF_OPT_BAND_COMPOSE = 1): both levels of a band as one composed 4 x 4 block operator
    per group, formed in FP32 on chip.  Checked against the oracle (which applies the levels one after
    the other in FP64) and against the level-by-level tensor-core band (same algebra, other rounding)."""
    F = W.rhs(1 << LN, nrhs, 40 + r)
    plan = bf.Plan.build_fio(bf.fio(W.K_FIO, W.A_CFG1, LN, l0, r), max_nrhs_chunk=nrhs)
    assert any(k.startswith("xfer") for k in plan.info()["tc_classes"])
    Gc = _apply(plan, F)
    plan.set_option(bf.BF_OPT_BAND_COMPOSE, 0)
    Gl = _apply(plan, F)
    with pytest.raises(bf.BFError):
        plan.set_option(bf.BF_OPT_BAND_COMPOSE, 2)
    plan.destroy()
    cols = [0, nrhs // 2, nrhs - 1]
    R = oracle.bf_apply(W.K_FIO, W.A_CFG1, LN, l0, r, F[:, cols])
    assert np.all(oracle.rel_l2(Gc[:, cols].astype(np.complex128), R, axis=0) <= PARITY)
    d = oracle.rel_l2(Gc.astype(np.complex128), Gl.astype(np.complex128), axis=0)
    assert np.all(d <= PATHS_AGREE), d.max()
    assert not np.array_equal(Gc, Gl)                 # the composed kernel really ran


def test_tc_scale_equivariance():
    """The 3xTF32 path is exactly homogeneous under power-of-two scaling of F (every rounding, including the
    tf32 hi/lo split, commutes with 2^k while nothing over- or underflows): G(2^k F) == 2^k G(F) bitwise."""
    LN, l0, r, nrhs = 12, 6, 10, 64
    F = W.rhs(1 << LN, nrhs, 9)
    plan = bf.Plan.build_fio(bf.fio(W.K_FIO, W.A_CFG1, LN, l0, r), max_nrhs_chunk=nrhs)
    G = _apply(plan, F)
    for k in (60, -60):
        Gk = _apply(plan, np.asfortranarray(F * np.float32(2.0 ** k)).astype(np.complex64))
        assert np.all(np.isfinite(Gk))
        assert np.array_equal(Gk, (G * np.float32(2.0 ** k)).astype(np.complex64)), k
    plan.destroy()


@pytest.mark.parametrize("LN,nrhs", [(14, 128), (14, 100), (12, 192), (16, 256)])
def test_tc_leaf_multicast(LN, nrhs):
    """BF_OPT_LEAF_MULTICAST (default 1): the 3xTF32 S0 and SL as 2-CTA clusters that each bulk-copy half of
    every weight-image tile and multicast it to both.  Same arithmetic per vector as the one-CTA kernel, so the result is
    bitwise equal (even vector-tile counts use the clusters: nv = 256, 200 (ragged), 512; nv = 384 falls
    back to one CTA per tile)."""
    l0, r = 6, 10
    F = W.rhs(1 << LN, nrhs, 80 + LN)
    plan = bf.Plan.build_fio(bf.fio(W.K_FIO, W.A_CFG1, LN, l0, r), max_nrhs_chunk=nrhs)
    assert {"s0", "sl"} <= set(plan.info()["tc_classes"])
    Gm = _apply(plan, F)
    plan.set_option(bf.BF_OPT_LEAF_MULTICAST, 0)
    G1 = _apply(plan, F)
    plan.destroy()
    assert np.array_equal(Gm, G1)
    R = oracle.bf_apply(W.K_FIO, W.A_CFG1, LN, l0, r, F[:, [0, nrhs - 1]])
    assert np.all(oracle.rel_l2(Gm[:, [0, nrhs - 1]].astype(np.complex128), R, axis=0) <= PARITY)


@pytest.mark.parametrize("nrhs", [128, 8])
def test_cuda_graph_capture(nrhs):
    """bf_apply only enqueues (no allocation, no host synchronization), so it can be captured
    into a CUDA graph; replays equal the eager apply bitwise, also after the input buffer is refilled.
    nrhs = 128 runs the tensor-core kernels (incl. the cluster-launched SL), nrhs = 8 the SIMT ones."""
    LN, l0, r = 14, 6, 10
    plan = bf.Plan.build_fio(bf.fio(W.K_FIO, W.A_CFG1, LN, l0, r), max_nrhs_chunk=nrhs)
    F1 = torch.from_numpy(np.ascontiguousarray(W.rhs(1 << LN, nrhs, 5).T)).cuda()
    F2 = torch.from_numpy(np.ascontiguousarray(W.rhs(1 << LN, nrhs, 6).T)).cuda()
    ref1, ref2 = torch.empty_like(F1), torch.empty_like(F1)
    plan.apply(F1, ref1, nrhs)
    plan.apply(F2, ref2, nrhs)
    torch.cuda.synchronize()
    Fin, Gout = F1.clone(), torch.empty_like(F1)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        plan.apply(Fin, Gout, nrhs)      # warm-up on the capture stream
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        plan.apply(Fin, Gout, nrhs)
    Gout.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(Gout, ref1)
    Fin.copy_(F2)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(Gout, ref2)
    del g
    plan.destroy()


@pytest.mark.parametrize("nrhs", [128, 8, 1])
def test_apply_graph(nrhs):
    """bf_apply_graph (include/bf.h): one launch of the plan's cached graph of bf_apply equals the eager apply
    bitwise (tensor-core, small-batch and tiny kernels: nrhs 128 / 8 / 1); new inputs in the same buffer are
    read at every launch; other buffers or nrhs re-capture; an option change drops the graph and the next
    call captures the new kernel sequence."""
    LN, l0, r = 14, 6, 10
    plan = bf.Plan.build_fio(bf.fio(W.K_FIO, W.A_CFG1, LN, l0, r), max_nrhs_chunk=nrhs)
    F1 = torch.from_numpy(np.ascontiguousarray(W.rhs(1 << LN, nrhs, 5).T)).cuda()
    F2 = torch.from_numpy(np.ascontiguousarray(W.rhs(1 << LN, nrhs, 6).T)).cuda()
    ref1, ref2 = torch.empty_like(F1), torch.empty_like(F1)
    plan.apply(F1, ref1, nrhs)
    plan.apply(F2, ref2, nrhs)
    torch.cuda.synchronize()
    Fin, G = F1.clone(), torch.zeros_like(F1)
    s = torch.cuda.Stream()
    plan.apply_graph(Fin, G, nrhs, stream=s)
    s.synchronize()
    assert torch.equal(G, ref1)
    Fin.copy_(F2)
    torch.cuda.synchronize()
    G.zero_()
    torch.cuda.synchronize()
    plan.apply_graph(Fin, G, nrhs, stream=s)
    s.synchronize()
    assert torch.equal(G, ref2)
    G2 = torch.zeros_like(F1)
    plan.apply_graph(F1, G2, nrhs)          # other buffers: re-captured, default stream
    torch.cuda.synchronize()
    assert torch.equal(G2, ref1)
    if nrhs > 1:                            # fewer columns of the same buffers
        G3 = torch.zeros_like(F1)
        plan.apply_graph(F1, G3, nrhs // 2)
        torch.cuda.synchronize()
        assert torch.equal(G3[: nrhs // 2], ref1[: nrhs // 2]) and not G3[nrhs // 2:].any()
    plan.set_tensor_cores(False)            # drops the graph; the FP32 kernels agree within parity
    G4 = torch.zeros_like(F1)
    plan.apply_graph(F1, G4, nrhs)
    ref4 = torch.empty_like(F1)
    plan.apply(F1, ref4, nrhs)
    torch.cuda.synchronize()
    assert torch.equal(G4, ref4)
    plan.destroy()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_rhs_shards_concatenate_to_one_gpu(world):
    """bench.py's RHS sharding: each rank applies columns [q nrhs/G, (q+1) nrhs/G) with its own
    replicated plan; the blocks concatenate to the one-GPU result.  Bitwise while every shard takes the same
    kernels as the full batch (each vector's reduction order does not depend on the batch); a shard whose
    vector count falls to another kernel class agrees within the paths' FP32 agreement."""
    import bench
    k = bf.fio(W.K_FIO, W.A_CFG1, 14, 6, 10)   # cfg4's shape at N = 2^14
    nrhs = 256
    F = W.rhs(1 << 14, nrhs, 3)
    for pre in (0, 1):   # 0: every plan composes its bands on chip (kernel choice independent of the chunk)
        full = bf.Plan.build_fio(k, max_nrhs_chunk=nrhs)
        full.set_option(bf.BF_OPT_BAND_PRECOMPOSE, pre)
        ref, tc_full = _apply(full, F), set(full.info()["tc_classes"])
        full.destroy()
        blocks, same = [], True
        for q in range(world):
            c0, c1 = bench.rhs_columns(nrhs, world, q)
            p = bf.Plan.build_fio(k, max_nrhs_chunk=c1 - c0)
            p.set_option(bf.BF_OPT_BAND_PRECOMPOSE, pre)
            same &= set(p.info()["tc_classes"]) == tc_full
            blocks.append(_apply(p, np.asfortranarray(F[:, c0:c1])))
            p.destroy()
        G = np.concatenate(blocks, axis=1)
        if same and not pre:
            assert np.array_equal(G, ref)
        else:
            err = oracle.rel_l2(G.astype(np.complex128), ref.astype(np.complex128), axis=0)
            assert np.all(err <= PATHS_AGREE), err.max()


@pytest.mark.parametrize("r,l0,LN,nrhs", [(10, 6, 16, 32), (8, 5, 14, 64), (12, 5, 14, 48), (6, 6, 14, 100)])
def test_tc_band_precomposed(r, l0, LN, nrhs):
    """Plans of <= 256 vectors per chunk compose each band's two-level operator at finalization (FP64) and the
    band kernel only embeds and splits it (BF_OPT_BAND_PRECOMPOSE = 1, default); 0 composes on chip in FP32.
    Both meet the oracle bar and agree like two FP32-accurate paths; the precomposed operators are counted in
    factor_bytes (16 r^2 complex per group of 4 pairs: the bytes of the two levels' blocks)."""
    F = W.rhs(1 << LN, nrhs, 80 + r)
    k = bf.fio(W.K_FIO, W.A_CFG1, LN, l0, r)
    plan = bf.Plan.build_fio(k, max_nrhs_chunk=nrhs)
    info = plan.info()
    assert any(c.startswith("xfer") for c in info["tc_classes"])
    bands = (LN - 2 * l0) // 2
    base = bf.Plan.build_fio(k, max_nrhs_chunk=300)       # > 256 vectors: no precomposed operators
    assert info["factor_bytes"] - base.info()["factor_bytes"] == bands * 8 * (1 << LN) * 4 * r * r
    base.destroy()
    Gp = _apply(plan, F)
    plan.set_option(bf.BF_OPT_BAND_PRECOMPOSE, 0)
    Gc = _apply(plan, F)
    with pytest.raises(bf.BFError):
        plan.set_option(bf.BF_OPT_BAND_PRECOMPOSE, 2)
    plan.destroy()
    cols = [0, nrhs - 1]
    R = oracle.bf_apply(W.K_FIO, W.A_CFG1, LN, l0, r, F[:, cols])
    for G in (Gp, Gc):
        assert np.all(oracle.rel_l2(G[:, cols].astype(np.complex128), R, axis=0) <= PARITY)
    d = oracle.rel_l2(Gp.astype(np.complex128), Gc.astype(np.complex128), axis=0)
    assert np.all(d <= PATHS_AGREE), d.max()
    assert not np.array_equal(Gp, Gc)


@pytest.mark.parametrize("r,l0,LN,nrhs,chunk", [(8, 5, 16, 128, 128),   # 6 levels: 3 + 3, 2 vector tiles
                                                (6, 5, 16, 100, 100),   # r = 6, nv = 200: full + ragged tile
                                                (8, 6, 18, 64, 64),     # one vector tile per group
                                                (8, 5, 18, 128, 128),   # 8 levels: 3 + 3 + 2 (cfg4's schedule)
                                                (8, 5, 16, 150, 64)])   # chunks of 128 + 128 + 44 vectors
def test_tc_band3(r, l0, LN, nrhs, chunk):
    """Three-level tensor-core bands (bf_band3.cu, BF_OPT_BAND3 = 1, default for r in {6, 8} and >= 128 vectors):
    three adjacent factors of eqn:BFM applied as one 8 x 8 block operator per group of 8 pairs, composed at
    finalization in FP64.  Against the oracle at the bar, against the two-level bands (BF_OPT_BAND3 = 0) like two
    FP32-accurate paths; the schedule (launches per class) and the operator bytes in factor_bytes."""
    N = 1 << LN
    F = W.rhs(N, nrhs, 90 + r + LN)
    k = bf.fio(W.K_FIO, W.A_CFG1, LN, l0, r)
    plan = bf.Plan.build_fio(k, max_nrhs_chunk=chunk)
    info = plan.info()
    nlev = LN - 2 * l0
    n3 = {6: 2, 8: 2}[nlev]
    nb = n3 + (nlev - 3 * n3) // 2
    assert sum(info["class_launches"][c] for c in ("xfer_first_half", "xfer_switch", "xfer_second_half")) == nb, info
    assert any(c.startswith("xfer") for c in info["tc_classes"])
    G3 = _apply(plan, F)
    for _ in range(3):   # run-to-run bitwise (a B-tile hazard once showed up as non-determinism in one vector tile)
        assert np.array_equal(_apply(plan, F), G3)
    plan.set_option(bf.BF_OPT_BAND3, 0)
    G2 = _apply(plan, F)
    with pytest.raises(bf.BFError):
        plan.set_option(bf.BF_OPT_BAND3, 2)
    plan.destroy()
    base = bf.Plan.build_fio(k, max_nrhs_chunk=16)          # 32 vectors: no three-level operators
    # three-level operators (64 r^2 complex per 8 pairs) + the remaining two-level bands' precomposed operators
    cmp2 = ((nlev - 3 * n3) // 2) * 8 * N * 4 * r * r if 2 * chunk <= 256 else 0
    assert info["factor_bytes"] - base.info()["factor_bytes"] == n3 * 8 * N * 8 * r * r + cmp2, info
    base.destroy()
    assert np.all(np.isfinite(G3))
    cols = [0, nrhs // 2, nrhs - 1]
    R = oracle.bf_apply(W.K_FIO, W.A_CFG1, LN, l0, r, F[:, cols])
    for G in (G3, G2):
        assert np.all(oracle.rel_l2(G[:, cols].astype(np.complex128), R, axis=0) <= PARITY)
    d = oracle.rel_l2(G3.astype(np.complex128), G2.astype(np.complex128), axis=0)
    assert np.all(d <= PATHS_AGREE), d.max()
