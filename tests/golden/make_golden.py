"""Generate tests/golden/ref_vectors.npz from the REFERENCE build (oracle/_ref:
the reference's own compiled sources under the shared driver, plus its
exported vmm_forward_raw / calibrate / quantized_forward). Run in the build
container (needs /root/reference):  python tests/golden/make_golden.py
The fixtures pin the oracle restatement where the reference build is absent."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

DIMS = dict(image=16, channels=3, patch=4, embed=16, state=4, blocks=2, classes=7, conv_width=3)
SEED = 2024


def main():
    O.build(ref=True)
    ref = O.Checker(O.REF_SO)
    d = O.Dims(**DIMS)
    m = ref.model(d, SEED)
    out = {}
    for name in ("patch_w", "head_w", "block0.w_in", "block1.dir1.a", "block1.dir0.w_delta", "block0.conv"):
        out["w." + name] = m.get(name)
    imgs = ref.normal(5, 3 * d.pix)
    cimgs = ref.normal(6, 4 * d.pix)
    out["images"] = imgs
    out["calib_images"] = cimgs
    # reference end-to-end functions (no extension): FP logits, calibrate, quantized_forward
    out["ref.fp_logits"] = m.ref_fp_forward(imgs)
    spec0 = O.Spec(abits=8, obits=8, n_refresh=3, rho=0.2, d1=False, d2=False)
    rc = m.ref_calibrate(cimgs, spec0)
    e = rc.export()
    out["ref.calib.theta"] = np.array([t.theta for t in e.scan])
    out["ref.calib.s_in"] = np.stack([t.s_in for t in e.scan])
    out["ref.calib.s_full"] = np.stack([t.s_full for t in e.scan])
    for mode in (1, 2):
        lq, lf = m.ref_quantized_forward(imgs, rc, mode)
        out[f"ref.quantized_forward.mode{mode}"] = lq
    # the shared driver on reference primitives with the declared extensions
    for ab in (4, 8):
        spec = O.Spec(abits=ab, obits=8, n_refresh=3, rho=0.1, d1=True, d2=True)
        c = m.calibrate(cimgs, spec)
        ce = c.export()
        out[f"d12.a{ab}.theta_scan"] = np.array([t.theta for t in ce.scan])
        out[f"d12.a{ab}.theta_lin"] = np.array([t.theta for t in ce.lin])
        out[f"d12.a{ab}.s_in_lin"] = np.stack([t.s_in for t in ce.lin])
        for mode in (0, 1, 2):
            out[f"d12.a{ab}.logits.mode{mode}"] = m.forward(imgs, c, mode)
        tr = m.trace(imgs[:d.pix], c, 1, 1)
        for k in ("lin0.codes", "lin0.omask", "lin0.acc_in", "lin3.codes", "lin1.acc_out", "dir0.mask0", "dir1.mask2",
                  "dir0.o", "x_out"):
            out[f"d12.a{ab}.trace.{k}"] = tr.get(k)
    # operator KATs: hybrid_gemm and the per-step detector stream
    rng = np.random.default_rng(7)
    w = rng.integers(-7, 8, size=(9, 24), dtype=np.int8)
    ws = rng.uniform(0.01, 0.1, size=9)
    x = rng.integers(-7, 8, size=(24, 11), dtype=np.int8)
    ch = np.array([2, 5, 17], np.uint64)
    x[ch.astype(int)] = 0
    oc = rng.integers(-127, 128, size=(3, 11), dtype=np.int8)
    osc = rng.uniform(0.01, 0.1, size=3)
    a_in, a_out, y = ref.hybrid_gemm(w, ws, x, 0.05, ch, oc, osc)
    out.update({"op.hg.w": w, "op.hg.ws": ws, "op.hg.x": x, "op.hg.ch": ch, "op.hg.oc": oc, "op.hg.osc": osc,
                "op.hg.acc_in": a_in, "op.hg.acc_out": a_out, "op.hg.out": y})
    xs = rng.normal(size=(2, 30, 16, 4)) * 0.5
    xs[rng.random((2, 30, 16, 4)) < 0.03] *= 20
    s_in = np.full(30, 3.0 / 127)
    fq, masks, scanned = ref.quant_stream(xs, 3.0, s_in, s_in * 1.5, 4, 8, 8, 1)
    out.update({"op.qs.x": xs, "op.qs.fq": fq, "op.qs.masks": masks, "op.qs.scanned": scanned})
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_vectors.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes", len(out), "arrays")


if __name__ == "__main__":
    main()
