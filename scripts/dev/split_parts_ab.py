"""Forward time per split_parts at a given width / image / batch (W4A4 dynamic):
python scripts/dev/split_parts_ab.py E IMAGE B P1 [P2 ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2503_10959_b200 as ob
E, image, B = (int(v) for v in sys.argv[1:4])
parts = [int(v) for v in sys.argv[4:]]
ctx = ob.Context(0)
m = ob.Model(ctx, ob.Dims(image=image, embed=E, blocks=24), 1234)
g = torch.Generator(device="cuda").manual_seed(0)
cal = m.calibrate(torch.randn(8, image, image, 3, dtype=torch.float64, device="cuda", generator=g),
                  ob.QuantSpec(wbits=4, abits=4, obits=8, n_refresh=10, rho=0.01), chunk=8)
x = torch.randn(B, image, image, 3, dtype=torch.float64, device="cuda", generator=g)
ref = None
for p in parts:
    m.set_option("split_parts", p)
    y = m.forward(x, cal, ob.MODE_DYNAMIC).cpu().numpy()
    ref = y if ref is None else ref
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        m.forward(x, cal, ob.MODE_DYNAMIC)
    e1.record()
    torch.cuda.synchronize()
    print(f"split_parts {p}: {e0.elapsed_time(e1) / 3:.2f} ms per forward, identical {np.array_equal(ref, y)}", flush=True)
