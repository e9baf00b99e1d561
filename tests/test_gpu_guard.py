"""Out-of-bounds write detection without compute-sanitizer (closed on this GPU pool): F, G and the caller
workspace of bf_apply_ex sit inside larger device buffers whose guard zones (64 KB before and after, filled with
a NaN bit pattern) must be untouched after the apply, and F must be unchanged -- for every kernel family (FP32
SIMT, small-batch persistent kernels, tensor-core S0 / composed band / SL, precomposed bands, ragged chunks,
leading dimensions > N)."""
import numpy as np
import pytest

from paper_1803_04128_b200 import bf
from paper_1803_04128_b200 import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GUARD = 8192          # complex64 elements (64 KB) on each side
PATTERN = 0x7FC0DEAD  # a NaN payload no kernel produces


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.init()
    yield


def _guarded(n):
    buf = torch.empty(2 * GUARD + n, dtype=torch.complex64, device="cuda")
    buf.view(torch.int32).fill_(PATTERN)
    return buf, buf[GUARD:GUARD + n]


def _intact(buf, n):
    w = buf.view(torch.int32)
    return bool((w[:2 * GUARD] == PATTERN).all()) and bool((w[2 * (GUARD + n):] == PATTERN).all())


CASES = [
    # kernel, amp, LN, l0, r, nrhs, chunk, ld_pad, tensor cores     what runs
    (W.K_FIO, W.A_CFG1, 10, 4, 12, 1, 1, 0, True),          # cfg1: FP32 SIMT, nv = 2
    (W.K_FIO, W.A_CFG1, 14, 6, 10, 8, 8, 2, True),          # small batch nv = 16 (S0, bands, SL)
    (W.K_FIO, W.A_CFG2, 14, 5, 10, 16, 16, 0, True),        # small batch nv = 32, leaf 32
    (W.K_FIO, W.A_CFG1, 12, 6, 10, 64, 64, 4, True),        # tensor cores nv = 128 (precomposed band)
    (W.K_FIO, W.A_CFG1, 14, 6, 10, 150, 64, 0, True),       # tensor cores, ragged chunks 128 + 128 + 44
    (W.K_FIO, W.A_CFG1, 12, 6, 10, 300, 300, 0, True),      # tensor cores nv = 600: on-chip composed band
    (W.K_FIO_JUMP, W.A_CFG3, 12, 5, 8, 13, 5, 2, False),    # FP32 SIMT, n_amp 4, ragged
]


@pytest.mark.parametrize("kernel,amp,LN,l0,r,nrhs,chunk,pad,tc", CASES)
def test_apply_writes_only_its_outputs(kernel, amp, LN, l0, r, nrhs, chunk, pad, tc):
    N = 1 << LN
    ld = N + pad
    plan = bf.Plan.build_fio(bf.fio(kernel, amp, LN, l0, r), max_nrhs_chunk=chunk)
    plan.set_tensor_cores(tc)
    F = W.rhs(N, nrhs, 3)
    fb, Fv = _guarded(ld * nrhs)
    Fv.view(nrhs, ld)[:, :N] = torch.from_numpy(np.ascontiguousarray(F.T)).cuda()
    F_before = Fv.clone()
    gb, Gv = _guarded(ld * nrhs)
    wsn = plan.workspace_bytes(min(chunk, nrhs)) // 8
    wb, Wv = _guarded(wsn)
    plan.apply_ex(Fv, ld, Gv, ld, nrhs, workspace=Wv, workspace_bytes=wsn * 8)
    torch.cuda.synchronize()
    plan.destroy()
    assert _intact(fb, ld * nrhs) and _intact(gb, ld * nrhs) and _intact(wb, wsn), "a guard zone was written"
    assert torch.equal(Fv.view(torch.int32), F_before.view(torch.int32)), "F was modified"
    G = Gv.view(nrhs, ld)
    if pad:   # the padding between columns is not written either
        assert bool((G[:, N:].view(torch.int32) == PATTERN).all())
    assert bool(torch.isfinite(torch.view_as_real(G[:, :N])).all())
