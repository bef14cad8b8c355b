"""Fraction of scan steps with the h state in O per (direction, channel) at C1
(Vim-T W4A8 batch 1), from block traces: the small-batch phase B's exact path runs
on every such step. python scripts/dev/h_outlier_stats.py [blocks...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2503_10959_b200 as ob
ctx = ob.Context(0)
m = ob.Model(ctx, ob.Dims(embed=192, blocks=24), 1234)
g = torch.Generator(device="cuda").manual_seed(0)
cal = m.calibrate(torch.randn(8, 224, 224, 3, dtype=torch.float64, device="cuda", generator=g),
                  ob.QuantSpec(wbits=4, abits=8, obits=8, n_refresh=10, rho=0.01), chunk=8)
x = torch.randn(1, 224, 224, 3, dtype=torch.float64, device="cuda", generator=g).cpu().numpy()
E, T = 192, 196
for b in [int(v) for v in sys.argv[1:]] or [0, 6, 12, 18, 23]:
    tr = m.trace(x, cal, ob.MODE_DYNAMIC, b)
    for d in range(2):
        k = f"dir{d}.masks"
        if not tr.has(k):
            print("no", k, [kk for kk in ("masks", "dir0.masks", "scan0.masks") if tr.has(kk)])
            continue
        mk = tr.get(k, np.uint8).reshape(3, 1, T, E)
        h = mk[2, 0].astype(bool)  # [T][E]
        frac = h.mean(axis=0)
        warp = frac.reshape(-1, 2).max(axis=1)  # two channels per warp in phase B
        print(f"block {b} dir {d}: h in O {h.mean():.4f} of steps; channels ever {np.mean(frac > 0):.3f}; "
              f"max per channel {frac.max():.3f}; warps with > 50 % {np.mean(warp > 0.5):.3f}", flush=True)
