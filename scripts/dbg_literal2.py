import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2503_10959_b200 as ob
from oracle import oracle as O
chk = O.Checker(O.ORACLE_SO)
DIMS = dict(image=32, channels=3, patch=8, embed=64, state=16, blocks=2, classes=10, conv_width=4)
od = O.Dims(**DIMS); om = chk.model(od, 1234)
cimgs = chk.normal(7, 4 * od.pix)
spec = O.Spec(wbits=4, abits=4, obits=8, n_refresh=3, rho=0.1)
ocal = om.calibrate(cimgs, spec).export()
ctx = ob.Context(0)
L, E, N = od.tokens, od.embed, od.state
for S in (1, 2):
  for order in (0, 1):
    g = torch.Generator().manual_seed(5)
    u = torch.randn(S, L, E, dtype=torch.float64, generator=g).cuda()
    proj = (0.5 * torch.randn(S, L, E + 2 * N, dtype=torch.float64, generator=g)).cuda()
    a = torch.from_numpy(om.get("block0.dir0.a")).cuda()
    bd = torch.zeros(E, dtype=torch.float64).cuda()
    tc = [ocal.scan[k] for k in range(3)]
    for t in tc:
        qa = 7.0
        C = np.nextafter(t.theta, np.inf) / qa > t.s_in
        print("C(t) all:", C.all(), "theta", t.theta, "max s_in*qa", (t.s_in*qa).max())
    s_in = [torch.from_numpy(t.s_in).cuda() for t in tc]
    s_full = [torch.from_numpy(t.s_full).cuda() for t in tc]
    outs = []
    for force in (False, True):
        o = torch.zeros(S, L, E, dtype=torch.float64, device="cuda")
        masks = torch.zeros(3, S, L, E, dtype=torch.uint8, device="cuda")
        ctx.quant_scan(S=S, T=L, E=E, order=order, grid=od.grid, u=u, proj=proj, a=a, b_delta=bd, o=o,
                       mode=1, n_refresh=3, act_bits=4, outlier_bits=8,
                       theta=[t.theta for t in tc], s_in=s_in, s_full=s_full, force_literal=force, masks=masks)
        torch.cuda.synchronize()
        outs.append((o.cpu().numpy(), masks.cpu().numpy()))
    d = np.argwhere(outs[0][0] != outs[1][0])
    print("S", S, "order", order, "ndiff", len(d), d[:5], "mask diff", (outs[0][1] != outs[1][1]).sum(),
          "nz fast", (outs[0][0] != 0).sum(), "nz lit", (outs[1][0] != 0).sum())
