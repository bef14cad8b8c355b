import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2503_10959_b200 as ob
ctx = ob.Context(0)
S, L, E, N = 1, 4, 32, 16
g = torch.Generator().manual_seed(5)
u = torch.randn(S, L, E, dtype=torch.float64, generator=g).cuda()
proj = (0.5 * torch.randn(S, L, E + 2 * N, dtype=torch.float64, generator=g)).cuda()
a = -torch.rand(E, N, dtype=torch.float64, generator=g).cuda() - 0.5
bd = torch.zeros(E, dtype=torch.float64).cuda()
for mode in (0, 1):
  outs = []
  for force in (False, True):
    o = torch.zeros(S, L, E, dtype=torch.float64, device="cuda")
    masks = torch.zeros(3, S, L, E, dtype=torch.uint8, device="cuda")
    th = [0.5, 0.5, 0.5]
    s_in = [torch.full((L,), 0.5/7, dtype=torch.float64, device="cuda") for _ in range(3)]
    ctx.quant_scan(S=S, T=L, E=E, order=0, grid=2, u=u, proj=proj, a=a, b_delta=bd, o=o, mode=mode, n_refresh=3,
                   act_bits=4, outlier_bits=8, theta=th, s_in=s_in, s_full=s_in, force_literal=force, masks=masks)
    torch.cuda.synchronize()
    outs.append(o.cpu().numpy())
    print("mode", mode, "force", force, o[0, :, :4].cpu().numpy(), masks.sum().item())
  print("equal", np.array_equal(outs[0], outs[1]))
