import sys
import numpy as np, torch
import paper_2503_10959_b200 as ob
ctx = ob.Context(0)
E, T, n_refresh, order, src, lit = [int(v) for v in sys.argv[1:7]]
S = 2
x = torch.randn(S, T, E, dtype=torch.float64, device="cuda")
s_in = torch.full((T,), 0.35, dtype=torch.float64, device="cuda")
r = ctx.detect_quantize(x, S=S, T=T, E=E, theta=2.5, s_in=s_in, s_full=s_in, n_refresh=n_refresh, act_bits=4,
                        outlier_bits=8, mode=1, src=src, order=order, grid=0, literal=bool(lit))
torch.cuda.synchronize()
print("ok", sys.argv[1:])
