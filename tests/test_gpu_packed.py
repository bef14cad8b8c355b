"""The A4 operand nibble-packed between K1 and K2 (north star parts (1) and (2);
pack_int4 / PackedInt4, gemm.cpp:54-83, gemm.hpp:40-49): K1's packed codes ==
the oracle's pack_int4 of its int8 codes (every kernel: staged plain and
RMSNorm, channel-parallel merge, literal), K2 on the packed operand (TMA box of
packed bytes, in-place unpack in shared memory before tcgen05) == K2 on int8
codes == the oracle's hybrid_gemm, integer planes included, and a whole A4
forward with the packed operand == the int8 one bit for bit."""
import numpy as np
import pytest

from test_gpu_ops import _dev, _mask_words

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("src,literal", [(0, False), (0, True), (1, False), (2, False), (2, True)])
def test_detect_quantize_packed_equals_pack_int4(oracle_checker, gpu_ctx, src, literal):
    import torch
    S, T, E = 3, 30, 96
    rng = np.random.default_rng(src * 2 + literal)
    x = rng.normal(size=(S, T, E)) * 2.0
    x[rng.random((S, T, E)) < 0.02] *= 25.0
    x2 = rng.normal(size=(S, T, E))
    gate = rng.normal(size=(S, T, E))
    s_in = _dev(np.full(T, 0.45))
    kw = dict(S=S, T=T, E=E, theta=3.1, s_in=s_in, s_full=s_in, n_refresh=4, act_bits=4, outlier_bits=8, mode=1,
              src=src, x2=_dev(x2), gate=_dev(gate), literal=literal)
    ref = gpu_ctx.detect_quantize(_dev(x), **kw)
    pk = gpu_ctx.detect_quantize(_dev(x), packed=True, **kw)
    torch.cuda.synchronize()
    codes = ref["codes"].cpu().numpy()
    assert codes.min() >= -7 and codes.max() <= 7 and np.any(codes < 0)
    assert np.array_equal(pk["codes4"].cpu().numpy(), oracle_checker.pack_int4(codes))
    for k in ("s_row", "ocnt", "omask"):
        assert np.array_equal(pk[k].cpu().numpy(), ref[k].cpu().numpy()), k
    m = pk["omask"].cpu().numpy().view(np.uint32)
    assert m.any()


def test_detect_quantize_packed_validation(gpu_ctx):
    import paper_2503_10959_b200 as ob
    import torch
    x = torch.zeros(1, 4, 64, dtype=torch.float64, device="cuda")
    s = torch.ones(4, dtype=torch.float64, device="cuda")
    with pytest.raises(ob.ValidationError):  # nibbles hold 4-bit codes only
        gpu_ctx.detect_quantize(x, S=1, T=4, E=64, theta=1.0, s_in=s, s_full=s, n_refresh=2, act_bits=8,
                                outlier_bits=8, packed=True)
    with pytest.raises(ob.ValidationError):  # whole bytes per row
        gpu_ctx.detect_quantize(x[:, :, :63].contiguous(), S=1, T=4, E=63, theta=1.0, s_in=s, s_full=s, n_refresh=2,
                                act_bits=4, outlier_bits=8, packed=True)


@pytest.mark.parametrize("M,R,K,n_o", [(128, 128, 128, 0), (300, 160, 256, 5), (1000, 800, 768, 12),
                                       (77, 1536, 192, 3), (4096, 768, 768, 8), (260, 96, 2048, 40),
                                       (1000, 768, 384, 2)])
def test_quant_linear_packed_bit_exact(oracle_checker, gpu_ctx, M, R, K, n_o):
    """hybrid_gemm on the packed operand: acc_inlier / acc_outlier / output
    bit-exact against the oracle and against the int8-operand kernel, for both
    K2 shapes (8 and 16 epilogue warps), ragged M and partial K-blocks."""
    import torch
    rng = np.random.default_rng(M * 5 + R + K)
    w = rng.integers(-7, 8, size=(R, K), dtype=np.int8)
    ws = rng.uniform(0.005, 0.02, size=R)
    x = rng.integers(-7, 8, size=(M, K), dtype=np.int8)
    chans = np.sort(rng.choice(K, size=n_o, replace=False)).astype(np.int64)
    x[:, chans] = 0
    ocodes = rng.integers(-127, 128, size=(n_o, M), dtype=np.int8)
    oscales = rng.uniform(0.005, 0.02, size=n_o)
    s_in = float(rng.uniform(0.005, 0.02))
    acc_in, acc_out, out = oracle_checker.hybrid_gemm(w, ws, x.T.copy(), s_in, chans.astype(np.uint64), ocodes,
                                                      oscales)
    mask = np.zeros((M, K), np.uint8)
    mask[:, chans] = 1
    dense_code = np.zeros((M, K), np.int8)
    dense_code[:, chans] = ocodes.T
    dense_scale = np.zeros((M, K), np.float64)
    dense_scale[:, chans] = oscales
    common = dict(s_row=_dev(np.full(M, s_in)), ocnt=_dev(np.full(M, n_o, np.int32)),
                  omask=_dev(_mask_words(mask)), ocode=_dev(dense_code), oscale=_dev(dense_scale))
    for post in (0, 2):  # store (8 epilogue warps for wide R) and residual (16 epilogue warps)
        res = []
        for act in (dict(codes=_dev(x), **common), dict(codes4=_dev(oracle_checker.pack_int4(x)), **common)):
            g_in = torch.zeros(M, R, dtype=torch.int32, device="cuda")
            g_out = torch.zeros(M, R, dtype=torch.int32, device="cuda")
            y = torch.zeros(M, R, dtype=torch.float64, device="cuda")
            gpu_ctx.quant_linear(act, _dev(w), _dev(w.T.copy()), _dev(ws), post=post, out=y, acc_in=g_in,
                                 acc_out=g_out)
            y2 = gpu_ctx.quant_linear(act, _dev(w), _dev(w.T.copy()), _dev(ws), post=post,
                                      out=torch.zeros(M, R, dtype=torch.float64, device="cuda"))
            torch.cuda.synchronize()
            res.append((g_in.cpu().numpy(), g_out.cpu().numpy(), y.cpu().numpy(), y2.cpu().numpy()))
        (a_in, a_out, a_y, a_y2), (b_in, b_out, b_y, b_y2) = res
        assert np.array_equal(b_in, acc_in.T) and np.array_equal(b_out, acc_out.T)
        assert np.array_equal(b_y, a_y) and np.array_equal(b_y2, a_y2) and np.array_equal(b_y2, b_y)
        if post == 0:
            assert np.array_equal(b_y, out.T)


@pytest.mark.parametrize("embed", [64, 192])
def test_forward_packed_equals_int8(oracle_checker, gpu_ctx, embed):
    """A4 dynamic / static forwards with the packed operand == the int8 operand
    (the default) == the oracle, bit for bit."""
    import paper_2503_10959_b200 as ob
    from oracle import oracle as O
    dims = dict(image=32, channels=3, patch=8, embed=embed, state=16, blocks=2, classes=10, conv_width=4)
    od = O.Dims(**dims)
    om = oracle_checker.model(od, 5)
    gm = ob.Model(gpu_ctx, ob.Dims(**dims), 5)
    imgs = oracle_checker.normal(51, 4 * od.pix).reshape(4, 32, 32, 3)
    spec = O.Spec(wbits=4, abits=4, obits=8, n_refresh=3, rho=0.05)
    ocal = om.calibrate(oracle_checker.normal(52, 3 * od.pix).reshape(3, 32, 32, 3), spec).export()
    conv = lambda t: ob.TensorCal(t.theta, t.s_in, t.s_full, t.excluded)
    gcal = gm.calibration_from([conv(t) for t in ocal.scan], [conv(t) for t in ocal.lin],
                               ob.QuantSpec(4, 4, 8, 3, 0.05, True, True))
    for mode in (ob.MODE_DYNAMIC, ob.MODE_STATIC):
        outs = []
        for pk in (1, 0):
            gm.set_option("pack_a4", pk)
            outs.append(gm.forward_host(imgs, gcal, mode))
        gm.set_option("pack_a4", 0)
        assert np.array_equal(outs[0], outs[1]), mode
        want = om.forward(imgs, om.calib_from(ocal), mode)
        assert np.array_equal(outs[0], want), mode


def test_trace_packed_codes(oracle_checker, gpu_ctx):
    """Block traces with the packed operand: lin<site>.codes4 == pack_int4 of the
    int8 codes, which equal the int8 forward's, for every quantized linear site."""
    import paper_2503_10959_b200 as ob
    from oracle import oracle as O
    dims = dict(image=32, channels=3, patch=8, embed=64, state=16, blocks=2, classes=10, conv_width=4)
    od = O.Dims(**dims)
    om = oracle_checker.model(od, 6)
    gm = ob.Model(gpu_ctx, ob.Dims(**dims), 6)
    imgs = oracle_checker.normal(61, 2 * od.pix).reshape(2, 32, 32, 3)
    spec = O.Spec(wbits=4, abits=4, obits=8, n_refresh=3, rho=0.05)
    ocal = om.calibrate(oracle_checker.normal(62, 3 * od.pix).reshape(3, 32, 32, 3), spec).export()
    conv = lambda t: ob.TensorCal(t.theta, t.s_in, t.s_full, t.excluded)
    gcal = gm.calibration_from([conv(t) for t in ocal.scan], [conv(t) for t in ocal.lin],
                               ob.QuantSpec(4, 4, 8, 3, 0.05, True, True))
    gm.set_option("pack_a4", 1)
    tp = gm.trace(imgs, gcal, ob.MODE_DYNAMIC, 1)
    gm.set_option("pack_a4", 0)
    ti = gm.trace(imgs, gcal, ob.MODE_DYNAMIC, 1)
    E = dims["embed"]
    for site in range(4):
        p = f"lin{site}."
        codes = ti.get(p + "codes", np.int8).reshape(-1, E)
        assert np.array_equal(tp.get(p + "codes", np.int8).reshape(-1, E), codes), site
        assert np.array_equal(tp.get(p + "codes4", np.uint8).reshape(-1, E // 2), oracle_checker.pack_int4(codes)), site
        for k in ("acc_in", "acc_out"):
            assert np.array_equal(tp.get(p + k, np.int32), ti.get(p + k, np.int32)), (site, k)
    assert np.array_equal(tp.get("logits", np.float64), ti.get("logits", np.float64))


@pytest.mark.parametrize("pack", [0, 1])
def test_merge_fused_into_scan_identical(oracle_checker, gpu_ctx, pack):
    """The out_proj input K1 fused into the f32-state scan's tail (merge_fuse 1)
    == the separate k1_channel launch == the oracle, int8 and packed operands."""
    import paper_2503_10959_b200 as ob
    from oracle import oracle as O
    dims = dict(image=32, channels=3, patch=8, embed=128, state=16, blocks=2, classes=10, conv_width=4)
    od = O.Dims(**dims)
    om = oracle_checker.model(od, 8)
    gm = ob.Model(gpu_ctx, ob.Dims(**dims), 8)
    imgs = oracle_checker.normal(81, 5 * od.pix).reshape(5, 32, 32, 3)
    spec = O.Spec(wbits=4, abits=4, obits=8, n_refresh=3, rho=0.05)
    ocal = om.calibrate(oracle_checker.normal(82, 3 * od.pix).reshape(3, 32, 32, 3), spec).export()
    conv = lambda t: ob.TensorCal(t.theta, t.s_in, t.s_full, t.excluded)
    gcal = gm.calibration_from([conv(t) for t in ocal.scan], [conv(t) for t in ocal.lin],
                               ob.QuantSpec(4, 4, 8, 3, 0.05, True, True))
    gm.set_option("pack_a4", pack)
    for sv in (0, 7):  # 7: the scan kernel's large-grid shape (A in shared memory), as at batch 256
        gm.set_option("scan_variant", sv)
        for mode in (ob.MODE_DYNAMIC, ob.MODE_STATIC):
            outs = []
            for f in (1, 0):
                gm.set_option("merge_fuse", f)
                outs.append(gm.forward_host(imgs, gcal, mode))
            gm.set_option("merge_fuse", 0)
            assert np.array_equal(outs[0], outs[1]), (sv, mode)
            assert np.array_equal(outs[0], om.forward(imgs, om.calib_from(ocal), mode)), (sv, mode)
    gm.set_option("scan_variant", 0)
    gm.set_option("pack_a4", 0)
