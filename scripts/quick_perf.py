"""Quick device timing of the quantized Vim forward (development aid)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2503_10959_b200 as ob

E = int(sys.argv[1]) if len(sys.argv) > 1 else 768
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
blocks = int(sys.argv[3]) if len(sys.argv) > 3 else 24
ctx = ob.Context(0)
dims = ob.Dims(embed=E, blocks=blocks)
t0 = time.time()
m = ob.Model(ctx, dims, 1234)
print("model init s", time.time() - t0, flush=True)
g = torch.Generator(device="cuda").manual_seed(0)
cal_imgs = torch.randn(8, 224, 224, 3, dtype=torch.float64, device="cuda", generator=g)
imgs = torch.randn(B, 224, 224, 3, dtype=torch.float64, device="cuda", generator=g)
spec = ob.QuantSpec(wbits=4, abits=4, obits=8, n_refresh=10, rho=0.01)
t0 = time.time()
cal = m.calibrate(cal_imgs, spec, chunk=8)
torch.cuda.synchronize()
print("calibrate s", time.time() - t0, flush=True)
for mode, name in ((ob.MODE_DYNAMIC, "dynamic"), (ob.MODE_FP, "fp")):
    logits = m.forward(imgs, cal, mode)
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.time()
    for _ in range(3):
        logits = m.forward(imgs, cal, mode)
    ctx.synchronize()
    dt = (time.time() - t0) / 3
    print(f"{name}: B={B} E={E} blocks={blocks}: {dt*1e3:.1f} ms/forward, {B/dt:.1f} img/s; "
          f"finite={bool(torch.isfinite(logits).all())} max|logit|={logits.abs().max().item():.3f}", flush=True)
