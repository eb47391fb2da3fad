import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
from oracle import fftcond_oracle as O
from paper_2001_08289_b200.operators import gamma1
rng = np.random.default_rng(0)
for shape in [(2,2,2),(4,4,4),(8,8,8),(16,16,16),(2,2,16),(2,16,2),(4,2,2),(2,4,4),(16,8,8),(8,16,8),(16,16,8),(16,8,16),(32,32,32),(8,8,16)]:
    f = rng.standard_normal((3,)+shape) + 1j*rng.standard_normal((3,)+shape)
    got = gamma1(f).cpu().numpy(); ref = O.gamma1(f)
    err = np.abs(got-ref).max()/np.abs(ref).max()
    fg = np.fft.fftn(got, axes=(1,2,3)); fr = np.fft.fftn(ref, axes=(1,2,3))
    bad = np.argwhere(np.abs(fg-fr).max(axis=0) > 1e-9*np.abs(fr).max())
    print(shape, f"{err:.2e}", "bad modes (z,y,x):", bad[:6].tolist(), len(bad), flush=True)
