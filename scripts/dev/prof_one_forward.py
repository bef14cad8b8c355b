"""One quantized Vim forward between cudaProfilerStart/Stop (ncu --profile-from-start off), after
calibration and a warm-up forward: python prof_one_forward.py E B blocks [split_parts]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2503_10959_b200 as ob
E, B, blocks = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
parts = int(sys.argv[4]) if len(sys.argv) > 4 else 1
ctx = ob.Context(0)
m = ob.Model(ctx, ob.Dims(embed=E, blocks=blocks), 1234)
g = torch.Generator(device="cuda").manual_seed(0)
cal = m.calibrate(torch.randn(8, 224, 224, 3, dtype=torch.float64, device="cuda", generator=g),
                  ob.QuantSpec(wbits=4, abits=4, obits=8, n_refresh=10, rho=0.01), chunk=8)
x = torch.randn(B, 224, 224, 3, dtype=torch.float64, device="cuda", generator=g)
m.set_option("split_parts", parts)
m.forward(x, cal, ob.MODE_DYNAMIC)
torch.cuda.synchronize()
torch.cuda.profiler.start()
m.forward(x, cal, ob.MODE_DYNAMIC)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")
