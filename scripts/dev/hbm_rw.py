import torch
n = 616 * 2**20 // 8
a = torch.empty(n, dtype=torch.float64, device="cuda")
b = torch.empty(n, dtype=torch.float64, device="cuda")
def t(fn, it=20):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it * 1e-3
tw = t(lambda: a.fill_(1.5))
tc = t(lambda: b.copy_(a))
tr = t(lambda: a.sum())
print(f"write-only {n*8/tw/1e9:.0f} GB/s; copy (r+w) {2*n*8/tc/1e9:.0f} GB/s; read-only {n*8/tr/1e9:.0f} GB/s")
