"""The Python example of INTEGRATION.md section 4, run at a small size (keeps the
documentation honest): every call must succeed."""
import tempfile

import numpy as np
import torch

import paper_2503_10959_b200 as ob

ctx = ob.Context(0)
dims = ob.Dims(image=32, channels=3, patch=8, embed=64, state=16, blocks=2, classes=10, conv_width=4)
m = ob.Model(ctx, dims, seed=1234)
calib_images_cuda = torch.randn(4, 32, 32, 3, dtype=torch.float64, device="cuda")
images_np = np.random.default_rng(0).normal(size=(8, 32, 32, 3))
images_cuda = torch.from_numpy(images_np).cuda()
cal = m.calibrate(calib_images_cuda, ob.QuantSpec(wbits=4, abits=4, obits=8, n_refresh=10, rho=0.01))
with tempfile.TemporaryDirectory() as d:
    cal.save(d)
    cal = m.load_calibration(d)
m.use_graphs(True)
logits = m.forward(images_cuda, cal, ob.MODE_DYNAMIC)
logits_h = m.forward_host(images_np, cal, ob.MODE_DYNAMIC)
torch.cuda.synchronize()
assert np.array_equal(logits.cpu().numpy(), logits_h)
# the reference's own quantized_forward (no D1/D2) needs a calibration recorded the same way
cal_ref = m.calibrate(calib_images_cuda, ob.QuantSpec(wbits=4, abits=4, obits=8, n_refresh=10, rho=0.01, d1=False, d2=False))
res = m.quant_eval(images_np, cal_ref, ob.MODE_DYNAMIC, d1=False, d2=False, spikes=ob.SpikeSettings(rate=0.05, gain=100.0))
sweep = ctx.refresh_sweep((1, 5, 10, 20, 0), steps=50, trials=1)
bench = ctx.gemm_bench((64, 128, 256), trials=1)
m.set_option("split_parts", 2)
print("example ok", logits_h.shape, res["argmax_agree"], [r["mean_o_list"] for r in sweep], len(bench))
