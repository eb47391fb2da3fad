import sys, os, ctypes as C
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
from paper_2001_08289_b200 import native
from oracle import fftcond_oracle as O
L = native.lib(); L.fftc_debug_project.argtypes=[C.POINTER(native.Problem), C.c_void_p, C.c_void_p]
rng = np.random.default_rng(0)
for shape in [(2,2,2),(8,8,8),(16,16,16),(2,16,16)]:
    f = rng.standard_normal((3,)+shape) + 1j*rng.standard_normal((3,)+shape)
    pre = np.fft.fft(np.fft.fft(f, axis=-1), axis=-2)       # x, y transformed
    ks, inv = O.wave_vectors(shape)
    fh = np.fft.fft(pre, axis=-3)
    dot = (ks[0]*fh[0] + ks[1]*fh[1] + ks[2]*fh[2]) * inv
    ref = np.fft.ifft(np.stack([k*dot for k in ks]), axis=-3) * shape[0]
    t = torch.from_numpy(pre).cuda().contiguous()
    p = native.Problem(); p.d=3; p.n[0]=shape[2]; p.n[1]=shape[1]; p.n[2]=shape[0]
    rc = L.fftc_debug_project(C.byref(p), t.data_ptr(), None); assert rc == 0
    got = t.cpu().numpy()
    bad = np.argwhere(np.abs(got-ref).max(axis=0) > 1e-9*np.abs(ref).max())
    print(shape, np.abs(got-ref).max()/np.abs(ref).max(), bad[:8].tolist(), len(bad))
    if len(bad):
        z,y,x = bad[0]
        print("   got", got[:, z, y, x], "\n   ref", ref[:, z, y, x], "\n   pre", pre[:, z, y, x])
