"""One C1 forward (Vim-T W4A8 batch 1, 24 blocks) between cudaProfilerStart/Stop, for
ncu --profile-from-start off launch lists of the small-batch scan phases."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2503_10959_b200 as ob
ctx = ob.Context(0)
m = ob.Model(ctx, ob.Dims(embed=192, blocks=24), 1234)
g = torch.Generator(device="cuda").manual_seed(0)
cal = m.calibrate(torch.randn(8, 224, 224, 3, dtype=torch.float64, device="cuda", generator=g),
                  ob.QuantSpec(wbits=4, abits=8, obits=8, n_refresh=10, rho=0.01), chunk=8)
x = torch.randn(1, 224, 224, 3, dtype=torch.float64, device="cuda", generator=g)
m.forward(x, cal, ob.MODE_DYNAMIC)
torch.cuda.synchronize()
torch.cuda.profiler.start()
m.forward(x, cal, ob.MODE_DYNAMIC)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")
