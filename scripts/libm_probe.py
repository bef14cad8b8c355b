"""How often CUDA's exp / log1p differ from glibc's (the reference's libm) on the
arguments the scan sees (delta*A in [-60, 0], -|x| for softplus in [-40, 0])."""
import ctypes, numpy as np, torch
libm = ctypes.CDLL("libm.so.6")
libm.exp.restype = libm.exp.argtypes = None
libm.exp.restype = ctypes.c_double; libm.exp.argtypes = [ctypes.c_double]
libm.log1p.restype = ctypes.c_double; libm.log1p.argtypes = [ctypes.c_double]
rng = np.random.default_rng(0)
n = 200000
for name, lo, hi in (("exp", -60.0, 0.0), ("exp", -1.0, 1.0)):
    x = rng.uniform(lo, hi, n)
    g = np.array([libm.exp(float(v)) for v in x])
    c = torch.exp(torch.from_numpy(x).cuda()).cpu().numpy()
    print(f"{name} [{lo},{hi}]: differs in {np.mean(g != c) * 100:.4f}% ({np.sum(g != c)} of {n})")
x = np.exp(rng.uniform(-40.0, 0.0, n))
g = np.array([libm.log1p(float(v)) for v in x])
c = torch.log1p(torch.from_numpy(x).cuda()).cpu().numpy()
print(f"log1p(exp(-|x|)): differs in {np.mean(g != c) * 100:.4f}%")
