"""A/B of the scan-fused out_proj K1 (merge_fuse 1) against the separate k1_channel launch (0):
ms per forward (device, CUDA graphs off), per-family ms and bit-identity."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2503_10959_b200 as ob
E, B = int(sys.argv[1]), int(sys.argv[2])
rho = float(sys.argv[3]) if len(sys.argv) > 3 else 0.01
ctx = ob.Context(0)
m = ob.Model(ctx, ob.Dims(embed=E, blocks=24), 1234)
g = torch.Generator(device="cuda").manual_seed(0)
cal = m.calibrate(torch.randn(8, 224, 224, 3, dtype=torch.float64, device="cuda", generator=g),
                  ob.QuantSpec(wbits=4, abits=4, obits=8, n_refresh=10, rho=rho), chunk=8)
x = torch.randn(B, 224, 224, 3, dtype=torch.float64, device="cuda", generator=g)
out = torch.empty(B, 1000, dtype=torch.float64, device="cuda")
res = {}
for f in (0, 1, 0, 1):
    m.set_option("merge_fuse", f)
    for _ in range(2):
        m.forward(x, cal, ob.MODE_DYNAMIC, logits=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        m.forward(x, cal, ob.MODE_DYNAMIC, logits=out)
    e1.record()
    torch.cuda.synchronize()
    _, fam = m.forward_profile(x, cal, ob.MODE_DYNAMIC)
    res[f] = out.cpu().numpy().copy()
    print(f"merge_fuse {f}: {e0.elapsed_time(e1) / 5:.3f} ms per forward; " +
          " ".join(f"{k} {v[0]:.3f}" for k, v in fam.items()), flush=True)
print("identical", np.array_equal(res[0], res[1]))
