"""Calibration only (not product code): cuFFT (torch.fft) fp64 timings on the
C2 shapes, to put the fused sweeps' times in context."""
import torch, time
x = torch.randn(2, 2048, 2048, dtype=torch.complex128, device="cuda")
def t(fn, n=20):
    fn(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3
print(f"fft2 (2,2048,2048) c128 fwd:        {t(lambda: torch.fft.fft2(x)):8.1f} us  (2 vector comps, out-of-place)")
print(f"fft along x only:                   {t(lambda: torch.fft.fft(x, dim=-1)):8.1f} us")
print(f"fft along y only:                   {t(lambda: torch.fft.fft(x, dim=-2)):8.1f} us")
y = torch.randn(4, 2048, 2048, dtype=torch.complex128, device="cuda")
print(f"fft2 (4,2048,2048) (r and j fields): {t(lambda: torch.fft.fft2(y)):8.1f} us")
print(f"copy (2,2048,2048) c128:            {t(lambda: x.clone()):8.1f} us  (256 MB moved)")
