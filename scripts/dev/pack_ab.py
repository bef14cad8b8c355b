"""A/B of the packed A4 operand (pack_a4 1) against int8 codes (0): per-family ms per forward and bit-identity."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2503_10959_b200 as ob
E, B = int(sys.argv[1]), int(sys.argv[2])
ctx = ob.Context(0)
m = ob.Model(ctx, ob.Dims(embed=E, blocks=24), 1234)
g = torch.Generator(device="cuda").manual_seed(0)
cal = m.calibrate(torch.randn(8, 224, 224, 3, dtype=torch.float64, device="cuda", generator=g),
                  ob.QuantSpec(wbits=4, abits=4, obits=8, n_refresh=10, rho=0.01), chunk=8)
x = torch.randn(B, 224, 224, 3, dtype=torch.float64, device="cuda", generator=g)
res = {}
for pk in (0, 1, 0, 1):
    m.set_option("pack_a4", pk)
    best = None
    for _ in range(3):
        lg, fam = m.forward_profile(x, cal, ob.MODE_DYNAMIC)
        t = {k: v[0] for k, v in fam.items()}
        best = t if best is None or sum(t.values()) < sum(best.values()) else best
    res[pk] = lg.cpu().numpy()
    print("pack_a4", pk, {k: round(v, 3) for k, v in best.items()}, "total", round(sum(best.values()), 3), flush=True)
print("identical", np.array_equal(res[0], res[1]))
