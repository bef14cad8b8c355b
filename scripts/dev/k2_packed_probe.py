"""Development probe: K2 on the packed operand, one shape at a time (run under `timeout`)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2503_10959_b200 as ob

ctx = ob.Context(0)
post = int(sys.argv[1]) if len(sys.argv) > 1 else 0
for (M, R, K) in [(128, 128, 128), (256, 128, 128), (128, 256, 256), (1000, 800, 768)]:
    rng = np.random.default_rng(M)
    x = rng.integers(-7, 8, size=(M, K), dtype=np.int8)
    w = torch.from_numpy(rng.integers(-7, 8, size=(R, K), dtype=np.int8)).cuda()
    lo = (x[:, 0::2].astype(np.uint8) & 15) | ((x[:, 1::2].astype(np.uint8) & 15) << 4)
    act = dict(codes4=torch.from_numpy(lo).cuda(), s_row=torch.ones(M, dtype=torch.float64, device="cuda"),
               ocnt=torch.zeros(M, dtype=torch.int32, device="cuda"),
               omask=torch.zeros(M, (K + 31) // 32, dtype=torch.int32, device="cuda"),
               ocode=torch.zeros(M, K, dtype=torch.int8, device="cuda"),
               oscale=torch.zeros(M, K, dtype=torch.float64, device="cuda"))
    print("launch", M, R, K, post, flush=True)
    y = ctx.quant_linear(act, w, w.t().contiguous(), torch.ones(R, dtype=torch.float64, device="cuda"), post=post,
                         out=torch.zeros(M, R, dtype=torch.float64, device="cuda"))
    torch.cuda.synchronize()
    ref = x.astype(np.int64) @ w.cpu().numpy().astype(np.int64).T
    print("  ok", np.array_equal(y.cpu().numpy(), ref.astype(np.float64)), flush=True)
