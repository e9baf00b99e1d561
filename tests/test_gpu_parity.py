"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by
element on the same seeded inputs.

Bar (north_star): relative l2 error <= 1e-5 per RHS column against the oracle's
FP64 application of the same butterfly (the oracle regenerates every block from
its formula; the GPU uses the product builder's complex64 blocks and FP32
accumulation -- expected ~2-5e-7).
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


def to_dev(F: np.ndarray):
    """N x nrhs column-major complex64 host array -> device tensor with the same memory layout."""
    return torch.from_numpy(np.ascontiguousarray(F.T)).cuda()


def from_dev(T) -> np.ndarray:
    return np.asfortranarray(T.cpu().numpy().T)


def gpu_apply(plan: bf.Plan, F: np.ndarray) -> np.ndarray:
    Ft = to_dev(F)
    Gt = torch.empty_like(Ft)
    plan.apply(Ft, Gt, F.shape[1])
    torch.cuda.synchronize()
    return from_dev(Gt)


def per_col_err(G, R):
    return oracle.rel_l2(G.astype(np.complex128), R, axis=0)


# ---------------------------------------------------------------------------
# every BASELINE config (cfg5 at full size is in test_cfg5_full)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name,sample_cols", [("cfg1", None), ("cfg1_dft", None), ("cfg2", None),
                                              ("cfg3", [0, 17, 42, 63]), ("cfg4", [0, 255])])
def test_parity_config(name, sample_cols):
    w = W.CONFIGS[name]
    F = W.rhs(w.n, w.nrhs, w.seed)
    plan = bf.Plan.build_fio(bf.fio_of(w), max_nrhs_chunk=w.nrhs)   # the launch configuration bench.py times
    G = gpu_apply(plan, F)
    plan.destroy()
    cols = list(range(w.nrhs)) if sample_cols is None else sample_cols
    R = oracle.bf_apply(w.kernel, w.amp, w.log2n, w.log2leaf, w.rank, F[:, cols])
    err = per_col_err(G[:, cols], R)
    assert np.all(err <= PARITY), err
    # and against the truth (direct sum) on the eps^b row sample: within the construction tolerance
    rows = W.sample_rows(w.n, w.seed)
    gd = oracle.direct_rows(w.kernel, w.amp, w.log2n, F[:, cols[:1]], rows)
    assert oracle.rel_l2(G[rows][:, cols[:1]].astype(np.complex128), gd) <= w.eps / 2 + 2e-6
    assert np.all(np.isfinite(G))


def test_cfg5_full():
    """cfg5 (N = 2^22, 8 RHS) on one GPU: 113 GB of factors; sampled columns vs the oracle."""
    w = W.CONFIGS["cfg5"]
    free, _ = torch.cuda.mem_get_info()
    if free < 135e9:
        pytest.skip(f"needs ~130 GB of device memory, {free / 1e9:.0f} GB free")
    F = W.rhs(w.n, w.nrhs, w.seed)
    plan = bf.Plan.build_fio(bf.fio_of(w), max_nrhs_chunk=w.nrhs)
    G = gpu_apply(plan, F)
    plan.destroy()
    cols = [3]
    R = oracle.bf_apply(w.kernel, w.amp, w.log2n, w.log2leaf, w.rank, F[:, cols])
    assert np.all(per_col_err(G[:, cols], R) <= PARITY)


# ---------------------------------------------------------------------------
# shapes and edge cases at sizes the oracle finishes in seconds (several tiles + ragged tails)
# ---------------------------------------------------------------------------
EDGE = [
    # kernel, amp, LN, l0, r, nrhs, chunk          what it exercises
    (W.K_FIO, W.A_CFG1, 8, 4, 10, 1, 1),           # h == l0: no transfer level, standalone switch
    (W.K_FIO, W.A_CFG1, 12, 3, 6, 3, 2),           # leaf 8, r=6, ragged RHS chunking (2 + 1)
    (W.K_FIO_PAPER, W.A_ONE, 12, 4, 8, 3, 3),      # n_amp = 1, nv = 3 (odd: 1-vector thread tiles)
    (W.K_FIO_JUMP, W.A_CFG3, 14, 5, 12, 5, 4),     # n_amp = 4, jump folded, ragged chunk
    (W.K_FIO, W.A_CFG2, 16, 6, 16, 2, 2),          # r = 16, leaf 64
    (W.K_DFT, W.A_CFG1, 14, 6, 14, 7, 7),          # r = 14, nv = 14
    (W.K_FIO, W.A_CFG1, 16, 6, 10, 8, 8),          # cfg5's shape at reduced N (nv = 16)
    (W.K_FIO, W.A_CFG1, 14, 5, 10, 33, 33),        # nv = 66: multi-tile vector columns + tail
    (W.K_FIO, W.A_CFG1, 14, 5, 10, 70, 70),        # nv = 140: tiled S0/SL + bands, ragged second vector tile
    (W.K_FIO_JUMP, W.A_CFG3, 12, 4, 8, 25, 25),    # nv = 100: tiled leaf kernels with leaf 16, n_amp 4
    (W.K_FIO, W.A_ONE, 14, 6, 12, 132, 132),       # nv = 132, n_amp 1, r = 12 bands
    (W.K_FIO, W.A_CFG2, 16, 6, 10, 96, 40),        # chunks of 80 + 80 + 32 vectors (tiled, tiled, fallback)
]


@pytest.mark.parametrize("kernel,amp,LN,l0,r,nrhs,chunk", EDGE)
def test_parity_edge(kernel, amp, LN, l0, r, nrhs, chunk):
    N = 1 << LN
    F = W.rhs(N, nrhs, 100 + LN)
    plan = bf.Plan.build_fio(bf.fio(kernel, amp, LN, l0, r), max_nrhs_chunk=chunk)
    G = gpu_apply(plan, F)
    plan.destroy()
    R = oracle.bf_apply(kernel, amp, LN, l0, r, F)
    err = per_col_err(G, R)
    assert np.all(err <= PARITY), err


def _small_plan(nrhs_chunk=4):
    return bf.Plan.build_fio(bf.fio(W.K_FIO, W.A_CFG1, 12, 4, 10), max_nrhs_chunk=nrhs_chunk)


def test_zero_rhs_and_zero_input():
    plan = _small_plan()
    N = 1 << 12
    Ft = torch.zeros((3, N), dtype=torch.complex64, device="cuda")
    Gt = torch.full_like(Ft, 7.0)
    plan.apply(Ft, Gt, 0)                      # nrhs = 0: no-op
    torch.cuda.synchronize()
    assert torch.all(Gt == 7.0)
    plan.apply(Ft, Gt, 3)                      # f = 0 -> g = 0 exactly
    torch.cuda.synchronize()
    assert torch.all(Gt == 0)


def test_deterministic_and_batch_consistent():
    plan = _small_plan(nrhs_chunk=16)
    N = 1 << 12
    F = W.rhs(N, 16, 5)
    G1 = gpu_apply(plan, F)
    G2 = gpu_apply(plan, F)
    assert np.array_equal(G1, G2)                         # run to run, bitwise
    Gs = gpu_apply(plan, np.asfortranarray(F[:, 5:6]))    # a column alone == the same column in the batch
    assert np.array_equal(Gs[:, 0], G1[:, 5])
    perm = np.random.default_rng(0).permutation(16)       # RHS permutation equivariance
    Gp = gpu_apply(plan, np.asfortranarray(F[:, perm]))
    assert np.array_equal(Gp, G1[:, perm])


def test_linearity():
    plan = _small_plan()
    N = 1 << 12
    F = W.rhs(N, 2, 8)
    G = gpu_apply(plan, F)
    Fc = np.asfortranarray(((2 - 1j) * F[:, 0] + 0.5 * F[:, 1])[:, None].astype(np.complex64))
    Gc = gpu_apply(plan, Fc)
    ref = (2 - 1j) * G[:, 0].astype(np.complex128) + 0.5 * G[:, 1]
    assert oracle.rel_l2(Gc[:, 0].astype(np.complex128), ref) < 1e-6


def test_apply_ex_leading_dims_and_workspace():
    plan = _small_plan(nrhs_chunk=3)
    N, ld, nrhs = 1 << 12, (1 << 12) + 10, 5
    F = W.rhs(N, nrhs, 9)
    ref = gpu_apply(plan, F)
    Fp = torch.zeros((nrhs, ld), dtype=torch.complex64, device="cuda")
    Fp[:, :N] = to_dev(F)
    Gp = torch.zeros((nrhs, ld + 2), dtype=torch.complex64, device="cuda")
    ws = torch.empty(plan.workspace_bytes(3) // 8 + 2, dtype=torch.complex64, device="cuda")
    plan.apply_ex(Fp, ld, Gp, ld + 2, nrhs, workspace=ws, workspace_bytes=plan.workspace_bytes(3))
    torch.cuda.synchronize()
    G = np.asfortranarray(Gp[:, :N].cpu().numpy().T)
    assert np.array_equal(G, ref)
    assert torch.all(Gp[:, N:] == 0)                        # nothing written past N in each column


def test_apply_host_end_to_end():
    plan = _small_plan(nrhs_chunk=2)
    N, nrhs = 1 << 12, 5
    F = W.rhs(N, nrhs, 10)
    ref = gpu_apply(plan, F)
    Fh = torch.from_numpy(np.ascontiguousarray(F.T)).pin_memory()
    Gh = torch.empty_like(Fh).pin_memory()
    plan.apply_host(Fh, Gh, nrhs)
    assert np.array_equal(np.asfortranarray(Gh.numpy().T), ref)


def test_bad_arguments_raise():
    plan = _small_plan()
    N = 1 << 12
    Ft = torch.zeros((2, N), dtype=torch.complex64, device="cuda")
    with pytest.raises(bf.BFError):
        plan.apply(Ft, Ft, 2)                                   # F and G alias
    with pytest.raises(bf.BFError):
        plan.apply_ex(Ft, N - 2, torch.empty_like(Ft), N, 2)    # ld < N


def _host_factors(kernel, amp, LN, l0, r):
    k = bf.fio(kernel, amp, LN, l0, r)
    N = 1 << LN
    a, b = bf.build_amp(k)
    v0 = bf.build_blocks(k, bf.BF_STAGE_V0, 0, N)
    xf = [bf.build_blocks(k, bf.BF_STAGE_XFER0 + i, 0, N) for i in range(LN - 2 * l0)]
    sw = bf.build_blocks(k, bf.BF_STAGE_SW, 0, N)
    u = bf.build_blocks(k, bf.BF_STAGE_U, 0, N)
    return a, b, v0, xf, sw, u


def test_plan_create_from_arrays_and_mutation():
    """bf_plan_create from host arrays == the streaming build (bitwise); perturbing one block of
    one transfer level makes parity fail (the test can fail)."""
    LN, l0, r = 12, 4, 10
    N = 1 << LN
    F = W.rhs(N, 2, 12)
    a, b, v0, xf, sw, u = _host_factors(W.K_FIO, W.A_CFG1, LN, l0, r)
    p1 = bf.Plan.from_arrays(LN, l0, r, a, b, v0, xf, sw, u, max_nrhs_chunk=2)
    p2 = bf.Plan.build_fio(bf.fio(W.K_FIO, W.A_CFG1, LN, l0, r), max_nrhs_chunk=2)
    G1, G2 = gpu_apply(p1, F), gpu_apply(p2, F)
    assert np.array_equal(G1, G2)
    R = oracle.bf_apply(W.K_FIO, W.A_CFG1, LN, l0, r, F)
    assert np.all(per_col_err(G1, R) <= PARITY)
    for lvl in range(len(xf)):
        xm = [x.copy() for x in xf]
        xm[lvl][N // 3] *= -1.0                                 # flip the sign of one block (eqn:2 / eqn:3)
        pm = bf.Plan.from_arrays(LN, l0, r, a, b, v0, xm, sw, u, max_nrhs_chunk=2)
        assert np.all(per_col_err(gpu_apply(pm, F), R) > 1e-3)
        pm.destroy()
    swm = sw.copy()
    swm[7] = swm[7].conj()                                      # a wrong switch block
    pm = bf.Plan.from_arrays(LN, l0, r, a, b, v0, xf, swm, u, max_nrhs_chunk=2)
    assert np.all(per_col_err(gpu_apply(pm, F), R) > 1e-4)


def test_from_device_arrays():
    LN, l0, r = 10, 4, 12
    a, b, v0, xf, sw, u = _host_factors(W.K_FIO, W.A_CFG1, LN, l0, r)
    dev = [torch.from_numpy(x).cuda() for x in (a, b, v0, sw, u)]
    dxf = [torch.from_numpy(x).cuda() for x in xf]
    p = bf.Plan.from_arrays(LN, l0, r, dev[0], dev[1], dev[2], dxf, dev[3], dev[4], max_nrhs_chunk=1,
                            memory=bf.BF_MEM_DEVICE)
    ph = bf.Plan.from_arrays(LN, l0, r, a, b, v0, xf, sw, u, max_nrhs_chunk=1)
    F = W.rhs(1 << LN, 1, 0)
    assert np.array_equal(gpu_apply(p, F), gpu_apply(ph, F))


def test_timing_counts_launches():
    plan = _small_plan(nrhs_chunk=2)
    info = plan.info()
    F = W.rhs(1 << 12, 4, 1)
    plan.set_timing(True)
    gpu_apply(plan, F)
    t = plan.timing()
    n = sum(v[1] for v in t.values())
    assert n == 2 * info["launches_per_chunk"]      # 2 chunks
    assert all(v[0] >= 0 for v in t.values())
    plan.set_timing(False)


@pytest.mark.parametrize("chunk", [5, 7, 9])
@pytest.mark.parametrize("pieces", [2, 3, 4])
def test_apply_host_piece_layouts(chunk, pieces):
    """bf_apply_host's staging ring holds the largest piece of every layout (odd chunks, tapered pieces)."""
    plan = _small_plan(nrhs_chunk=chunk)
    plan.set_option(bf.BF_OPT_HOST_PIECES, pieces)
    N, nrhs = 1 << 12, 2 * chunk + 3
    F = W.rhs(N, nrhs, 20 + chunk)
    ref = gpu_apply(plan, F)
    Fh = torch.from_numpy(np.ascontiguousarray(F.T)).pin_memory()
    Gh = torch.empty_like(Fh).pin_memory()
    plan.apply_host(Fh, Gh, nrhs)
    assert np.array_equal(np.asfortranarray(Gh.numpy().T), ref)


def test_alignment_rejected():
    """F/G must be 16-byte aligned and ld even (bf.h): a view offset by one complex64 is refused with
    BF_ERR_ALIGNMENT instead of faulting the bulk copies of the tensor-core S0."""
    plan = _small_plan()
    N = 1 << 12
    buf = torch.zeros(2 * N + 1, dtype=torch.complex64, device="cuda")
    G = torch.zeros(2 * N, dtype=torch.complex64, device="cuda")
    with pytest.raises(bf.BFError) as e:
        plan.apply(buf[1:], G, 2)
    assert e.value.status == 3
    Fp = torch.zeros(2 * (N + 1), dtype=torch.complex64, device="cuda")
    with pytest.raises(bf.BFError) as e:
        plan.apply_ex(Fp, N + 1, torch.zeros_like(Fp), N + 1, 2)
    assert e.value.status == 3
    plan.apply(buf[2:], G, 2)                                   # 16-byte aligned view: fine
    torch.cuda.synchronize()


def test_upload_coverage():
    """finalize needs every block of every stage: repeating one range does not make up for a missing one."""
    import ctypes
    LN, l0, r = 10, 4, 12
    N = 1 << LN
    a, b, v0, xf, sw, u = _host_factors(W.K_FIO, W.A_CFG1, LN, l0, r)
    L = bf.lib()

    def alloc():
        d = bf.bf_desc_t(bf.BF_ABI_VERSION, LN, l0, r, a.shape[0], bf.BF_MEM_HOST)
        h = ctypes.c_void_p()
        assert L.bf_plan_alloc(ctypes.byref(d), 0, 1, ctypes.byref(h)) == 0
        return h

    def up(h, stage, arr, b0, n):
        assert L.bf_plan_upload(h, stage, b0, n, arr[b0:].ctypes.data, bf.BF_MEM_HOST) == 0

    for overlap in (True, False):
        h = alloc()
        up(h, bf.BF_STAGE_AMP_A, a, 0, a.shape[0])
        up(h, bf.BF_STAGE_AMP_B, b, 0, b.shape[0])
        up(h, bf.BF_STAGE_SW, sw, 0, N)
        up(h, bf.BF_STAGE_U, u, 0, N)
        for i, x in enumerate(xf):
            up(h, bf.BF_STAGE_XFER0 + i, x, 0, N)
        up(h, bf.BF_STAGE_V0, v0, 0, N // 2)
        if overlap:
            up(h, bf.BF_STAGE_V0, v0, 0, N // 2)                 # the same half twice: N blocks counted
            assert L.bf_plan_finalize(h) == 8                    # BF_ERR_STATE
            up(h, bf.BF_STAGE_V0, v0, N // 4, 3 * N // 4)        # overlapping ranges that cover the rest
        else:
            up(h, bf.BF_STAGE_V0, v0, N // 2, N // 2)
        assert L.bf_plan_finalize(h) == 0
        p = bf.Plan(h.value)
        ref = bf.Plan.from_arrays(LN, l0, r, a, b, v0, xf, sw, u, max_nrhs_chunk=1)
        F = W.rhs(N, 1, 3)
        assert np.array_equal(gpu_apply(p, F), gpu_apply(ref, F))


def test_apply_host_async_pipeline():
    """bf_apply_host_async: several calls in flight (distinct host buffers, chunks alternating between the two
    staging slots) give exactly bf_apply's results once bf_apply_host_wait returns."""
    plan = _small_plan(nrhs_chunk=3)
    N = 1 << 12
    calls = [W.rhs(N, n, 30 + n) for n in (7, 3, 5, 1)]     # 3 + 1 + 2 + 1 chunks
    refs = [gpu_apply(plan, F) for F in calls]
    hosts = [(torch.from_numpy(np.ascontiguousarray(F.T)).pin_memory(),
              torch.full((F.shape[1], N), float("nan"), dtype=torch.complex64).pin_memory()) for F in calls]
    for (Fh, Gh), F in zip(hosts, calls):
        plan.apply_host_async(Fh, Gh, F.shape[1])
    plan.apply_host_wait()
    for (_, Gh), ref in zip(hosts, refs):
        assert np.array_equal(np.asfortranarray(Gh.numpy().T), ref)
    plan.destroy()


@pytest.mark.parametrize("world", [4, 8])
def test_cfg4_rhs_shard_launch_configuration(world):
    """cfg4 at full size in the launch configuration one rank of bench.py --gpus 4 / 8 runs (R19): 256/G columns of
    the seeded batch in one chunk (nv = 128 / 64: tensor-core leaf stages on part-filled tiles, precomposed bands),
    sampled columns against the oracle."""
    import bench
    w = W.CONFIGS["cfg4"]
    c0, c1 = bench.rhs_columns(w.nrhs, world, world - 1)      # the last rank's columns
    F = W.rhs(w.n, w.nrhs, w.seed, cols=range(c0, c1))
    plan = bf.Plan.build_fio(bf.fio_of(w), max_nrhs_chunk=c1 - c0)
    info = plan.info()
    assert {"s0", "sl"} <= set(info["tc_classes"]) and any(k.startswith("xfer") for k in info["tc_classes"])
    G = gpu_apply(plan, F)
    plan.destroy()
    cols = [0, c1 - c0 - 1]
    R = oracle.bf_apply(w.kernel, w.amp, w.log2n, w.log2leaf, w.rank, F[:, cols])
    assert np.all(per_col_err(G[:, cols], R) <= PARITY)
