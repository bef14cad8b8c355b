"""Outlier statistics of the Vim-B quantized forward (mean |O(t)| per linear site, scan outlier-channel fraction)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2503_10959_b200 as ob
E = int(sys.argv[1]); abits = int(sys.argv[2])
ctx = ob.Context(0)
m = ob.Model(ctx, ob.Dims(embed=E, blocks=24), 1234)
g = torch.Generator(device="cuda").manual_seed(0)
cal_imgs = torch.randn(8, 224, 224, 3, dtype=torch.float64, device="cuda", generator=g)
imgs = torch.randn(4, 224, 224, 3, dtype=torch.float64, device="cuda", generator=g).cpu().numpy()
cal = m.calibrate(cal_imgs, ob.QuantSpec(wbits=4, abits=abits, obits=8, n_refresh=10, rho=0.01))
for blk in (0, 11, 23):
    tr = m.trace(imgs, cal, ob.MODE_DYNAMIC, blk)
    s = [tr.get(f"lin{k}.ocnt", np.int32).mean() for k in range(4)]
    sc = [tr.get(f"lin{k}.scanned", np.uint8).mean() for k in range(4)]
    mk = tr.get("dir0.masks", np.uint8).reshape(3, -1).mean(axis=1)
    print(f"block {blk}: mean |O| in/xp0/xp1/out = {np.round(s, 2)}, scanned frac = {np.round(sc, 2)}, "
          f"scan outlier-channel frac abar/bbar/h = {np.round(mk, 4)}")
