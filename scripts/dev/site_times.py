"""Per-site launch times (averaged over blocks) of one Vim-B forward, for pack_a4 0 / 1."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2503_10959_b200 as ob
E, B, blocks = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
ctx = ob.Context(0)
m = ob.Model(ctx, ob.Dims(embed=E, blocks=blocks), 1234)
g = torch.Generator(device="cuda").manual_seed(0)
cal = m.calibrate(torch.randn(8, 224, 224, 3, dtype=torch.float64, device="cuda", generator=g),
                  ob.QuantSpec(wbits=4, abits=4, obits=8, n_refresh=10, rho=0.01), chunk=8)
x = torch.randn(B, 224, 224, 3, dtype=torch.float64, device="cuda", generator=g)
m.set_option("split_parts", 1)
for pk in (0, 1):
    m.set_option("pack_a4", pk)
    m.forward(x, cal, ob.MODE_DYNAMIC); torch.cuda.synchronize()
    lst = m.forward_profile_launches(x, cal, ob.MODE_DYNAMIC)
    per = (len(lst) - 4) // blocks
    body = lst[2:2 + per * blocks]
    print(f"pack_a4={pk}: {len(lst)} launches, {per} per block, total {sum(v for _, v in lst):.2f} ms")
    for i in range(per):
        vals = [body[b * per + i][1] for b in range(blocks)]
        print(f"  {i:2d} {body[i][0]:16s} {np.mean(vals) * 1e3:8.1f} us")
