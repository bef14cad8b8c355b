"""A/B of the K3 scan variants at Vim sizes: scan time per forward and bit-identity.

    python scripts/scan_ab.py E B blocks abits [variants...]

variant 0 = auto, 1 = reference kernel, 2 = exact codes, 3 / 6 = two threads per channel with the f32 / f64
state update, 4 / 5 = one thread per channel with the f64 / f32 state update.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2503_10959_b200 as ob

E, B, blocks, abits = (int(a) for a in sys.argv[1:5])
rho = float(os.environ.get("RHO", "0.01"))
variants = [int(v) for v in sys.argv[5:]] or [0, 3, 4, 5, 2]
ctx = ob.Context(0)
m = ob.Model(ctx, ob.Dims(embed=E, blocks=blocks), 1234)
g = torch.Generator(device="cuda").manual_seed(0)
cal_imgs = torch.randn(8, 224, 224, 3, dtype=torch.float64, device="cuda", generator=g)
imgs = torch.randn(B, 224, 224, 3, dtype=torch.float64, device="cuda", generator=g)
cal = m.calibrate(cal_imgs, ob.QuantSpec(wbits=4, abits=abits, obits=8, n_refresh=10, rho=rho), chunk=8)
res = {}
for v in variants:
    m.set_option("scan_variant", v)
    m.forward_profile(imgs, cal, ob.MODE_DYNAMIC)  # warm-up
    t = []
    for _ in range(3):
        lg, fam = m.forward_profile(imgs, cal, ob.MODE_DYNAMIC)
        t.append(fam["k3_scan"][0])
    torch.cuda.synchronize()
    res[v] = lg.cpu().numpy()
    print(f"variant {v}: scan ms/forward {min(t):.3f} ({min(t) / blocks:.4f} per block)  "
          f"total {sum(x[0] for x in fam.values()):.2f}", flush=True)
base = res[variants[0]]
for v in variants[1:]:
    print(f"variant {variants[0]} == {v}: {np.array_equal(base, res[v])}  max|d| {np.abs(base - res[v]).max()}")
