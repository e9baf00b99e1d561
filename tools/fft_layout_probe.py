"""Probe: cuFFT (through torch.fft) time of the NUFFT's batched inverse FFT in the two layouts -- grids contiguous
([v][l], the plan's layout) vs batch-interleaved ([l][v], vectors fastest)."""
import torch

N, nv = 1 << 20, 512
for layout in ("v_l", "l_v"):
    x = torch.randn(nv, N, dtype=torch.complex64, device="cuda") if layout == "v_l" else \
        torch.randn(N, nv, dtype=torch.complex64, device="cuda")
    dim = 1 if layout == "v_l" else 0
    for _ in range(2):
        y = torch.fft.ifft(x, dim=dim)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        y = torch.fft.ifft(x, dim=dim)
    e1.record()
    torch.cuda.synchronize()
    print(layout, f"{e0.elapsed_time(e1) / 5:.3f} ms per batched FFT ({nv} x 2^20)")
    del x, y
