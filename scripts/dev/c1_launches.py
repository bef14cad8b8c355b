"""Per-launch device times (averaged over blocks) of one C1 forward (Vim-T W4A8 batch 1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2503_10959_b200 as ob
E, abits, B, blocks = 192, 8, 1, 4
ctx = ob.Context(0)
m = ob.Model(ctx, ob.Dims(embed=E, blocks=blocks), 1234)
g = torch.Generator(device="cuda").manual_seed(0)
cal = m.calibrate(torch.randn(8, 224, 224, 3, dtype=torch.float64, device="cuda", generator=g),
                  ob.QuantSpec(wbits=4, abits=abits, obits=8, n_refresh=10, rho=0.01), chunk=8)
x = torch.randn(B, 224, 224, 3, dtype=torch.float64, device="cuda", generator=g)
m.forward(x, cal, ob.MODE_DYNAMIC); torch.cuda.synchronize()
lst = m.forward_profile_launches(x, cal, ob.MODE_DYNAMIC)
print(len(lst), "launches", sum(v for _, v in lst), "ms")
for k, (f, v) in enumerate(lst[:30]):
    print(k, f, round(v * 1e3, 1), "us")
