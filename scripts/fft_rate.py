"""Rate of the bare transform passes (operator API fftc_fft): one x pass and
one y pass over a (2, n, n) complex128 field, CUDA events, vs HBM time."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch

from paper_2001_08289_b200 import operators as ops

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
t = torch.randn(2, n, n, dtype=torch.complex128, device="cuda")
for mask, name in ((1, "x (rows)"), (2, "y (columns)")):
    for _ in range(3):
        ops.fft_axes(t, mask)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        ops.fft_axes(t, mask)
    e1.record()
    torch.cuda.synchronize()
    us = 1e3 * e0.elapsed_time(e1) / reps
    pts = 2 * n * n
    print(f"{name:12s} {us:8.1f} us/pass  {pts / us / 1e3:6.1f} G points/s  {32 * pts / us / 1e3:6.2f} TB/s (read+write)")
