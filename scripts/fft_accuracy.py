"""FFT accuracy of the CUDA transforms vs numpy/pocketfft, both measured
against scipy.fft in long double (80-bit) as the exact reference."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, scipy.fft as sf
from paper_2001_08289_b200.operators import fft_axes
rng = np.random.default_rng(0)
for n in (8, 64, 256, 1024, 2048, 4096):
    f = rng.standard_normal((2, 4, n)) + 1j*rng.standard_normal((2, 4, n))
    exact = sf.fft(f.astype(np.clongdouble), axis=-1)
    for inv in (False, True):
        exact = sf.ifft(f.astype(np.clongdouble), axis=-1) * n if inv else sf.fft(f.astype(np.clongdouble), axis=-1)
        mine = fft_axes(f, 1, inv).cpu().numpy()
        npy = np.fft.ifft(f, axis=-1) * n if inv else np.fft.fft(f, axis=-1)
        rms = lambda a: float(np.sqrt(np.mean(np.abs(a)**2)))
        e_m = rms(mine - exact) / rms(exact); e_n = rms(npy - exact) / rms(exact)
        print(f"n={n:5d} inv={int(inv)}  cuda rms rel err {e_m:.2e}   numpy {e_n:.2e}   ratio {e_m/e_n:.2f}", flush=True)
