import sys, numpy as np, torch
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import paper_2503_10959_b200 as ob
ctx = ob.Context(0)
S, T, E, src = 3, 36, 64, 0
rng = np.random.default_rng(E + src)
x = rng.normal(size=(S, T, E)) * 2.0
x[rng.random((S, T, E)) < 0.02] *= 40.0
x[0, 5, 3] = 1e12
x[1, 7, 10] = -3e11
xd = torch.tensor(x, device="cuda")
s_in = torch.tensor(np.full(T, 0.3) * np.linspace(1.0, 1.3, T), device="cuda")
outs = []
for lit in (0, 2, 1):
    r = ctx.detect_quantize(xd, S=S, T=T, E=E, theta=3.1, s_in=s_in, s_full=s_in, n_refresh=10, act_bits=4,
                            outlier_bits=8, mode=2, src=src, literal=lit)
    torch.cuda.synchronize()
    outs.append(r["codes"].cpu().numpy().reshape(S, T, E))
sf = s_in.cpu().numpy()
for i, nm in ((1, "staged"), (2, "literal")):
    d = np.argwhere(outs[0] != outs[i])
    print(nm, len(d))
    for s, t, e in d[:10]:
        print("  ", s, t, e, x[s, t, e], x[s, t, e] / sf[t], "window", outs[0][s, t, e], nm, outs[i][s, t, e])
