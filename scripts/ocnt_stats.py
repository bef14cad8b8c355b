"""|O(t)| per quantized-linear input site at the bench's configuration (Vim-B,
W4A4 dynamic, D1+D2, n_refresh 10, rho 0.01): mean / p50 / p99 / max outlier
channels per token row, read from a trace of block `--block`."""
import argparse
import numpy as np
import torch
import paper_2503_10959_b200 as ob
import bench

ap = argparse.ArgumentParser()
ap.add_argument("--block", type=int, default=0)
ap.add_argument("--batch", type=int, default=8)
a = ap.parse_args()
ctx = ob.Context(0)
dims = ob.Dims(embed=768, blocks=24)
model = ob.Model(ctx, dims, bench.SEED)
spec = ob.QuantSpec(wbits=4, abits=4, obits=8, n_refresh=10, rho=0.01, d1=True, d2=True)
g = torch.Generator(device="cuda").manual_seed(bench.SEED + 7)
cal = model.calibrate(torch.randn(8, dims.image, dims.image, dims.channels, generator=g, device="cuda",
                                  dtype=torch.float64), spec, chunk=8)
g2 = torch.Generator(device="cuda").manual_seed(bench.SEED + 100)
imgs = torch.randn(a.batch, dims.image, dims.image, dims.channels, generator=g2, device="cuda",
                   dtype=torch.float64).cpu().numpy()
for b in sorted({0, a.block, dims.blocks // 2, dims.blocks - 1}):
    tr = model.trace(imgs, cal, ob.MODE_DYNAMIC, b)
    for site in range(4):
        try:
            c = tr.get(f"lin{site}.ocnt", np.int32)
        except Exception:
            continue
        print(f"block {b:2d} site {site}: mean {c.mean():6.2f}  p50 {np.median(c):5.1f}  p99 {np.percentile(c, 99):6.1f}  max {c.max()}")
