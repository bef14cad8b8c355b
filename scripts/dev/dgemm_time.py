"""Device time of the f64 projection GEMM at the patch-embedding shape (M = 50176, K = 768,
R = 768; ctx.dgemm, CUDA events over 5 calls): python scripts/dev/dgemm_time.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2503_10959_b200 as ob
ctx = ob.Context(0)
g = torch.Generator(device="cuda").manual_seed(0)
for M, K, R in ((50176, 768, 768), (12544, 768, 384), (256, 768, 1000)):
    a = torch.randn(M, K, dtype=torch.float64, device="cuda", generator=g)
    w = torch.randn(R, K, dtype=torch.float64, device="cuda", generator=g)
    out = torch.empty(M, R, dtype=torch.float64, device="cuda")
    ctx.dgemm(a, w, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        ctx.dgemm(a, w, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"M={M} K={K} R={R}: {ms:.3f} ms, {2 * M * K * R / ms / 1e9:.2f} TFLOP/s (mul + add counted)", flush=True)
