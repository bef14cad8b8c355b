"""HBM bandwidth by access pattern (write-only, read-only, copy) with torch ops, CUDA events, best of 10."""
import torch

n = 1 << 27  # 128 Mi doubles = 1 GiB
a = torch.empty(n, dtype=torch.float64, device="cuda")
b = torch.empty(n, dtype=torch.float64, device="cuda")
a.fill_(1.0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def best(fn, nbytes):
    t = 1e30
    for _ in range(10):
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        t = min(t, e0.elapsed_time(e1))
    return nbytes / (t * 1e-3) / 1e9


out = torch.empty(1, dtype=torch.float64, device="cuda")
print(f"write-only (fill): {best(lambda: b.fill_(2.0), 8 * n):.0f} GB/s")
print(f"read-only (sum):   {best(lambda: torch.sum(a, dim=0, out=out.view(())), 8 * n):.0f} GB/s")
print(f"copy (r+w bytes):  {best(lambda: b.copy_(a), 16 * n):.0f} GB/s")
