"""BASELINE.json configs C1, C2, C4 (and C3 for reference) measured on one B200.

    python scripts/configs_bench.py OUT.json [--iters N]

* C1 Vim-T W4A8 dynamic, batch 1, 224x224: latency per forward, device
  (CUDA-graph replay, CUDA events) and end to end (forward_host: host image in,
  host logits out);
* C2 Vim-S W4A4 dynamic, batch 64: images/s device and end to end;
* C3 Vim-B W4A4 dynamic, batch 256 (bench.py's workload): images/s device;
* C4 Vim-B 448x448 (L = 784) W4A4 dynamic, batch 64, rho in {0.005, 0.01,
  0.02, 0.05}: images/s and the per-family kernel times of one forward, plus the
  measured outlier fraction of each rho's calibration (channels above theta).

Synthetic N(0,1) images, make_toy_model weights (seed 1234), GPU calibration on
8 disjoint images, D1 + D2, n_refresh 10. Parity at these configs is asserted
by tests/test_gpu_full_config.py (bit-identical logits against the oracle).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2503_10959_b200 as ob

OUT = sys.argv[1] if len(sys.argv) > 1 else "configs.json"
ITERS = int(sys.argv[sys.argv.index("--iters") + 1]) if "--iters" in sys.argv else 20
ctx = ob.Context(0)
res = {}


def model(embed, image=224):
    return ob.Model(ctx, ob.Dims(image=image, embed=embed, blocks=24), 1234)


def images(n, image, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randn(n, image, image, 3, dtype=torch.float64, device="cuda", generator=g)


def dev_time(fn, iters):
    fn()
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def host_time(fn, iters):
    import time
    fn()
    t0 = time.perf_counter()
    for _ in range(iters):
        fn()
    return (time.perf_counter() - t0) * 1e3 / iters


def cal_for(m, image, abits, rho):
    return m.calibrate(images(8, image, 7), ob.QuantSpec(wbits=4, abits=abits, obits=8, n_refresh=10, rho=rho), chunk=8)


# C1: Vim-T W4A8 batch 1 (latency; CUDA graphs)
m = model(192)
cal = cal_for(m, 224, 8, 0.01)
x = images(1, 224, 11)
xh = x.cpu().numpy()
m.use_graphs(True)
out = torch.empty(1, 1000, dtype=torch.float64, device="cuda")
ms = dev_time(lambda: m.forward(x, cal, ob.MODE_DYNAMIC, logits=out), 50)
ms_host = host_time(lambda: m.forward_host(xh, cal, ob.MODE_DYNAMIC), 50)
_, fam = m.forward_profile(x, cal, ob.MODE_DYNAMIC)
res["C1"] = dict(config="Vim-T E=192 W4A8 dynamic, batch 1, 224x224, 24 blocks", device_ms_per_forward=ms,
                 e2e_ms_per_forward=ms_host, images_per_s=1e3 / ms, graphs=True,
                 families_ms={k: v[0] for k, v in fam.items()})
print("C1", res["C1"], flush=True)
del m, cal

# C2: Vim-S W4A4 batch 64
m = model(384)
cal = cal_for(m, 224, 4, 0.01)
x = images(64, 224, 12)
xh = x.cpu().numpy()
ms = dev_time(lambda: m.forward(x, cal, ob.MODE_DYNAMIC), ITERS)
ms_host = host_time(lambda: m.forward_host(xh, cal, ob.MODE_DYNAMIC), max(3, ITERS // 4))
_, fam = m.forward_profile(x, cal, ob.MODE_DYNAMIC)
res["C2"] = dict(config="Vim-S E=384 W4A4 dynamic, batch 64, 224x224, 24 blocks", device_ms_per_forward=ms,
                 images_per_s=64e3 / ms, e2e_images_per_s_pageable=64e3 / ms_host,
                 families_ms={k: v[0] for k, v in fam.items()})
print("C2", res["C2"], flush=True)
del m, cal

# C3: Vim-B W4A4 batch 256 (bench.py's workload, device only here)
m = model(768)
cal = cal_for(m, 224, 4, 0.01)
x = images(256, 224, 13)
ms = dev_time(lambda: m.forward(x, cal, ob.MODE_DYNAMIC), max(3, ITERS // 4))
res["C3"] = dict(config="Vim-B E=768 W4A4 dynamic, batch 256, 224x224, 24 blocks", device_ms_per_forward=ms,
                 images_per_s=256e3 / ms)
print("C3", res["C3"], flush=True)
del m, cal, x

# C4: Vim-B 448x448, rho sweep
m = model(768, image=448)
x = images(64, 448, 14)
c4 = []
for rho in (0.005, 0.01, 0.02, 0.05):
    cal = cal_for(m, 448, 4, rho)
    ms = dev_time(lambda: m.forward(x, cal, ob.MODE_DYNAMIC), max(3, ITERS // 4))
    _, fam = m.forward_profile(x, cal, ob.MODE_DYNAMIC)
    scan, lin = cal.export()
    c4.append(dict(rho=rho, device_ms_per_forward=ms, images_per_s=64e3 / ms,
                   families_ms={k: v[0] for k, v in fam.items()},
                   excluded_channels_mean=float(np.mean([np.mean(np.asarray(t.excluded, dtype=np.float64))
                                                          for t in scan]))))
    print("C4", c4[-1], flush=True)
    del cal
res["C4"] = dict(config="Vim-B E=768 W4A4 dynamic, 448x448 (L=784), batch 64, 24 blocks", sweep=c4)
with open(OUT, "w") as f:
    json.dump(res, f, indent=1)
print("wrote", OUT)
