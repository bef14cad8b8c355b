"""Per-launch device times of one Vim forward (CUDA events), grouped by logical op."""
import sys, os, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2503_10959_b200 as ob
E = int(sys.argv[1]); B = int(sys.argv[2]); blocks = int(sys.argv[3]); abits = int(sys.argv[4]) if len(sys.argv) > 4 else 4
ctx = ob.Context(0)
m = ob.Model(ctx, ob.Dims(embed=E, blocks=blocks), 1234)
g = torch.Generator(device="cuda").manual_seed(0)
cal = m.calibrate(torch.randn(4, 224, 224, 3, dtype=torch.float64, device="cuda", generator=g),
                  ob.QuantSpec(wbits=4, abits=abits, obits=8, n_refresh=10, rho=0.01))
imgs = torch.randn(B, 224, 224, 3, dtype=torch.float64, device="cuda", generator=g)
m.forward(imgs, cal, ob.MODE_DYNAMIC); torch.cuda.synchronize()
lst = m.forward_profile_launches(imgs, cal, ob.MODE_DYNAMIC)
names = ["patch_gather", "patch_embed"]
per_block = ["K1 in_proj", "K2 in_proj", "conv", "K1 x_proj d0", "K2 x_proj d0", "K1 x_proj d1", "K2 x_proj d1",
             "K3 scan", "K1 out_proj", "K2 out_proj"]
if (len(lst) - 4) == 8 * blocks:  # conv fused with both x_proj K1s
    per_block = ["K1 in_proj", "K2 in_proj", "conv+K1 x_proj", "K2 x_proj d0", "K2 x_proj d1", "K3 scan",
                 "K1 out_proj", "K2 out_proj"]
for b in range(blocks): names += per_block
names += ["meanpool", "head"]
agg = collections.defaultdict(float)
for (fam, ms), nm in zip(lst, names):
    agg[nm] += ms
tot = sum(ms for _, ms in lst)
print(f"E={E} B={B} blocks={blocks}: {len(lst)} launches, {tot:.2f} ms")
for nm, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"  {nm:14s} {v:8.3f} ms  {v / tot * 100:5.1f}%  per block {v / (blocks if nm in per_block else 1):.3f}")
