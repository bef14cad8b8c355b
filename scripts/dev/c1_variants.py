"""C1 (Vim-T W4A8 batch 1) forward latency per scan variant (CUDA graphs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2503_10959_b200 as ob
E = int(sys.argv[1]) if len(sys.argv) > 1 else 192
abits = int(sys.argv[2]) if len(sys.argv) > 2 else 8
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1
ctx = ob.Context(0)
m = ob.Model(ctx, ob.Dims(embed=E, blocks=24), 1234)
g = torch.Generator(device="cuda").manual_seed(0)
cal = m.calibrate(torch.randn(8, 224, 224, 3, dtype=torch.float64, device="cuda", generator=g),
                  ob.QuantSpec(wbits=4, abits=abits, obits=8, n_refresh=10, rho=0.01), chunk=8)
x = torch.randn(B, 224, 224, 3, dtype=torch.float64, device="cuda", generator=g)
out = torch.empty(B, 1000, dtype=torch.float64, device="cuda")
res = {}
for v in (0, 3, 4, 5, 6):
    m.set_option("scan_variant", v)
    m.use_graphs(True)
    for _ in range(3):
        m.forward(x, cal, ob.MODE_DYNAMIC, logits=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        m.forward(x, cal, ob.MODE_DYNAMIC, logits=out)
    e1.record()
    torch.cuda.synchronize()
    _, fam = m.forward_profile(x, cal, ob.MODE_DYNAMIC)
    res[v] = out.cpu().numpy().copy()
    print(f"variant {v}: {e0.elapsed_time(e1) / 20:.3f} ms per forward, scan {fam['k3_scan'][0]:.3f} ms", flush=True)
print("identical", all(np.array_equal(res[0], res[v]) for v in res))
