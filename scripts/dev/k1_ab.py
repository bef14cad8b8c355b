"""Per-site launch times (averaged over blocks) of one Vim forward for each
engine option value given, e.g. k1_variant 0 (register window K1) vs 2 (bulk-copy
staged K1):  python scripts/dev/k1_ab.py E B BLOCKS OPTION V1 [V2 ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2503_10959_b200 as ob
E, B, blocks, opt = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
vals = [int(v) for v in sys.argv[5:]]
ctx = ob.Context(0)
m = ob.Model(ctx, ob.Dims(embed=E, blocks=blocks), 1234)
g = torch.Generator(device="cuda").manual_seed(0)
cal = m.calibrate(torch.randn(8, 224, 224, 3, dtype=torch.float64, device="cuda", generator=g),
                  ob.QuantSpec(wbits=4, abits=4, obits=8, n_refresh=10, rho=0.01), chunk=8)
x = torch.randn(B, 224, 224, 3, dtype=torch.float64, device="cuda", generator=g)
m.set_option("split_parts", 1)
ref = None
for v in vals:
    m.set_option(opt, v)
    y = m.forward(x, cal, ob.MODE_DYNAMIC).cpu().numpy()
    torch.cuda.synchronize()
    same = ref is None or np.array_equal(ref, y)
    ref = y if ref is None else ref
    for rep in range(2):
        lst = m.forward_profile_launches(x, cal, ob.MODE_DYNAMIC)
    per = (len(lst) - 4) // blocks
    body = lst[2:2 + per * blocks]
    print(f"{opt}={v}: {len(lst)} launches, total {sum(t for _, t in lst):.2f} ms, logits identical: {same}")
    for i in range(per):
        ts = [body[b * per + i][1] for b in range(blocks)]
        print(f"  {i:2d} {body[i][0]:16s} {np.mean(ts) * 1e3:8.1f} us")
m.set_option(opt, 0)
