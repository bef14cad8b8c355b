"""K2 microbenchmark: hybrid quant-linear at a given shape and outlier count per row."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2503_10959_b200 as ob
M, R, K, n_o = (int(x) for x in sys.argv[1:5])
ctx = ob.Context(0)
g = torch.Generator(device="cuda").manual_seed(0)
codes = torch.randint(-7, 8, (M, K), dtype=torch.int8, device="cuda", generator=g)
w = torch.randint(-7, 8, (R, K), dtype=torch.int8, device="cuda", generator=g)
wt = w.t().contiguous()
ws = torch.rand(R, dtype=torch.float64, device="cuda", generator=g) * 0.01 + 0.005
chans = torch.randperm(K, device="cuda", generator=g)[:n_o].sort().values.cpu().numpy()
words = np.zeros((K + 31) // 32, np.uint32)
for ch in chans:
    words[ch // 32] |= np.uint32(1) << np.uint32(ch % 32)
omask = torch.from_numpy(np.tile(words.view(np.int32), (M, 1))).cuda()
act = dict(codes=codes, s_row=torch.full((M,), 0.01, dtype=torch.float64, device="cuda"),
           ocnt=torch.full((M,), n_o, dtype=torch.int32, device="cuda"), omask=omask,
           ocode=torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda", generator=g),
           oscale=torch.rand(M, K, dtype=torch.float64, device="cuda", generator=g) * 0.01)
out = torch.empty(M, R, dtype=torch.float64, device="cuda")
for _ in range(3):
    ctx.quant_linear(act, w, wt, ws, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 10
e0.record()
for _ in range(n):
    ctx.quant_linear(act, w, wt, ws, out=out)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
byts = M * K + R * K + M * R * 8
print(f"M={M} R={R} K={K} n_o={n_o}: {ms*1e3:.1f} us  {byts/ms/1e6:.0f} GB/s  {2*M*R*K/ms/1e9:.1f} TOPS")
