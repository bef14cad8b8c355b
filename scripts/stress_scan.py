"""Stress: fast K3 path vs exact-code variant vs reference kernel at Vim sizes (bit-exact logits)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2503_10959_b200 as ob
E = int(sys.argv[1]); B = int(sys.argv[2]); blocks = int(sys.argv[3]); abits = int(sys.argv[4])
ctx = ob.Context(0)
m = ob.Model(ctx, ob.Dims(embed=E, blocks=blocks), 1234)
g = torch.Generator(device="cuda").manual_seed(0)
cal_imgs = torch.randn(4, 224, 224, 3, dtype=torch.float64, device="cuda", generator=g)
imgs = torch.randn(B, 224, 224, 3, dtype=torch.float64, device="cuda", generator=g)
cal = m.calibrate(cal_imgs, ob.QuantSpec(wbits=4, abits=abits, obits=8, n_refresh=10, rho=0.01))
res = {}
for v in (0, 2, 1):
    m.set_option("scan_variant", v)
    lg, fam = m.forward_profile(imgs, cal, ob.MODE_DYNAMIC)
    torch.cuda.synchronize()
    res[v] = lg.cpu().numpy()
    print("variant", v, "scan ms", fam["k3_scan"][0], "total ms", sum(x[0] for x in fam.values()), flush=True)
print("fast==exact", np.array_equal(res[0], res[2]), "fast==ref", np.array_equal(res[0], res[1]),
      "max|d|", np.abs(res[0] - res[1]).max())
