"""One Vim forward inside an NVTX range "fwd" (for ncu --nvtx-include fwd/)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2503_10959_b200 as ob

E = int(sys.argv[1]); B = int(sys.argv[2]); blocks = int(sys.argv[3])
abits = int(sys.argv[4]) if len(sys.argv) > 4 else 4
ctx = ob.Context(0)
m = ob.Model(ctx, ob.Dims(embed=E, blocks=blocks), 1234)
g = torch.Generator(device="cuda").manual_seed(0)
cal_imgs = torch.randn(4, 224, 224, 3, dtype=torch.float64, device="cuda", generator=g)
imgs = torch.randn(B, 224, 224, 3, dtype=torch.float64, device="cuda", generator=g)
cal = m.calibrate(cal_imgs, ob.QuantSpec(wbits=4, abits=abits, obits=8, n_refresh=10, rho=0.01))
m.forward(imgs, cal, ob.MODE_DYNAMIC)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("fwd")
m.forward(imgs, cal, ob.MODE_DYNAMIC)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("ok")
