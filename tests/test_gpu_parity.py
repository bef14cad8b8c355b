"""GPU parity: the sm_100a path against the CPU oracle (oracle/, pinned to the
reference build) on identical seeded inputs.

Bar: bit-exact outlier masks, quantized codes and int32 accumulators (the
north star), and f64 outputs bit-identical too: every f64 operation follows
the reference's order and the device exp/log1p restate glibc's
(csrc/glibc_math.cuh), so RTOL_F64 is 0 (north star allows 1e-3 on logits).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DIMS = dict(image=32, channels=3, patch=8, embed=64, state=16, blocks=2, classes=10, conv_width=4)
SEED = 1234
B = 3
RTOL_F64 = 0.0


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.fixture(scope="module")
def pair(oracle_checker, gpu_ctx):
    from oracle import oracle as O
    import paper_2503_10959_b200 as ob
    od = O.Dims(**DIMS)
    om = oracle_checker.model(od, SEED)
    gm = ob.Model(gpu_ctx, ob.Dims(**DIMS), SEED)
    imgs = oracle_checker.normal(99, B * od.pix).reshape(B, od.image, od.image, od.channels)
    cimgs = oracle_checker.normal(7, 4 * od.pix).reshape(4, od.image, od.image, od.channels)
    return om, gm, imgs, cimgs


def test_seeded_weights_identical(pair):
    om, gm, _, _ = pair
    for name in om.tensor_names():
        assert np.array_equal(om.get(name), gm.get_tensor(name)), name


@pytest.mark.parametrize("d1", [True, False])
def test_fp_forward_matches_oracle(pair, d1):
    om, gm, imgs, _ = pair
    want = om.forward(imgs, None, 0, d1=d1, d2=True)
    got = gm.forward_host(imgs, None, 0, d1=d1, d2=True)
    assert rel_err(got, want) <= RTOL_F64


def _spec(abits, n_refresh=3, rho=0.05, d1=True, d2=True):
    from oracle import oracle as O
    return O.Spec(wbits=4, abits=abits, obits=8, n_refresh=n_refresh, rho=rho, d1=d1, d2=d2)


def _gspec(s):
    import paper_2503_10959_b200 as ob
    return ob.QuantSpec(s.wbits, s.abits, s.obits, s.n_refresh, s.rho, s.d1, s.d2)


@pytest.mark.parametrize("abits", [4, 8])
def test_gpu_calibration_matches_oracle(pair, abits):
    import torch
    om, gm, _, cimgs = pair
    spec = _spec(abits)
    want = om.calibrate(cimgs, spec).export()
    got_scan, got_lin = gm.calibrate(torch.from_numpy(cimgs).cuda(), _gspec(spec)).export()
    assert len(got_scan) == len(want.scan) and len(got_lin) == len(want.lin)
    for g, w in zip(got_scan + got_lin, want.scan + want.lin):
        assert abs(g.theta - w.theta) <= RTOL_F64 * abs(w.theta)
        assert rel_err(g.s_in, w.s_in) <= RTOL_F64
        assert rel_err(g.s_full, w.s_full) <= RTOL_F64
        assert np.array_equal(g.excluded, w.excluded)


def _import_calib(gm, cal, spec):
    import paper_2503_10959_b200 as ob
    conv = lambda t: ob.TensorCal(t.theta, t.s_in, t.s_full, t.excluded)
    return gm.calibration_from([conv(t) for t in cal.scan], [conv(t) for t in cal.lin], _gspec(spec))


@pytest.mark.parametrize("abits,mode,d1,d2", [(4, 1, True, True), (8, 1, True, True), (4, 2, True, True),
                                              (4, 1, True, False), (8, 2, True, False), (8, 1, False, False),
                                              (8, 2, False, False)])
def test_quantized_forward_logits(pair, abits, mode, d1, d2):
    """d1 = d2 = False is the reference's own quantized pass (quantized_forward,
    quant.cpp:519-526), which the oracle equals bit-for-bit (test_oracle_pin)."""
    om, gm, imgs, cimgs = pair
    spec = _spec(abits, d1=d1, d2=d2)
    ocal = om.calibrate(cimgs, spec)
    gcal = _import_calib(gm, ocal.export(), spec)
    want = om.forward(imgs, ocal, mode, d1=d1, d2=d2)
    got = gm.forward_host(imgs, gcal, mode, d1=d1, d2=d2)
    assert rel_err(got, want) <= RTOL_F64, (got, want)


@pytest.mark.parametrize("abits", [4, 8])
def test_block_trace_bit_exact(pair, abits):
    """Per-block intermediates of sample-level traces: codes, outlier lists,
    masks and accumulators bit-exact; f64 tensors within tolerance."""
    from oracle import oracle as O
    om, gm, imgs, cimgs = pair
    spec = _spec(abits, rho=0.1)
    ocal = om.calibrate(cimgs, spec)
    gcal = _import_calib(gm, ocal.export(), spec)
    d = om.dims
    L, E, N = d.tokens, d.embed, d.state
    nd = 2
    blk = 1
    gt = gm.trace(imgs, gcal, 1, blk)
    n_out_total = 0
    for s in range(B):
        ot = om.trace(imgs[s], ocal, 1, blk)
        rows = slice(s * L, (s + 1) * L)
        for key in ("x_in", "u0", "gate_pre", "u", "x_out"):
            g = gt.get(key, np.float64).reshape(B * L, E)[rows]
            assert rel_err(g, ot.get(key).reshape(L, E)) <= RTOL_F64, key
        for site, R in ((0, 2 * E), (1, E + 2 * N), (2, E + 2 * N), (3, E)):
            p = f"lin{site}."
            g_codes = gt.get(p + "codes", np.int8).reshape(B * L, E)[rows]
            assert np.array_equal(g_codes, ot.get(p + "codes").reshape(L, E)), p + "codes"
            g_cnt = gt.get(p + "ocnt", np.int32)[rows]
            g_ocode = gt.get(p + "ocode", np.int8).reshape(B * L, E)[rows]
            g_osc = gt.get(p + "oscale", np.float64).reshape(B * L, E)[rows]
            o_mask = ot.get(p + "omask").reshape(L, E)
            o_ocode = ot.get(p + "ocode").reshape(L, E)
            o_osc = ot.get(p + "oscale").reshape(L, E)
            for t in range(L):
                chans = np.nonzero(o_mask[t])[0]
                assert g_cnt[t] == len(chans), (p, t)
                assert np.array_equal(g_ocode[t, chans], o_ocode[t, chans]), (p, t)
                assert np.array_equal(g_osc[t, chans], o_osc[t, chans]), (p, t)
                n_out_total += len(chans)
            g_mask_bits = gt.get(p + "omask", np.uint32).reshape(B * L, -1)[rows]
            unpacked = ((g_mask_bits[:, :, None] >> np.arange(32, dtype=np.uint32)) & 1).reshape(L, -1)[:, :E]
            assert np.array_equal(unpacked.astype(np.uint8), o_mask), p + "omask"
            assert np.array_equal(gt.get(p + "scanned", np.uint8)[rows], ot.get(p + "scanned")), p + "scanned"
            assert np.array_equal(gt.get(p + "acc_in", np.int32).reshape(B * L, R)[rows],
                                  ot.get(p + "acc_in").reshape(L, R)), p + "acc_in"
            assert np.array_equal(gt.get(p + "acc_out", np.int32).reshape(B * L, R)[rows],
                                  ot.get(p + "acc_out").reshape(L, R)), p + "acc_out"
        for dd in range(nd):
            perm = np.array([_perm(dd, t, d.grid) for t in range(L)])
            g_proj = gt.get(f"dir{dd}.proj", np.float64).reshape(B * L, E + 2 * N)[rows]
            assert rel_err(g_proj, ot.get(f"lin{1 + dd}.out").reshape(L, E + 2 * N)) <= RTOL_F64
            g_o = gt.get(f"dir{dd}.o", np.float64).reshape(B * L, E)[rows]
            o_o = ot.get(f"dir{dd}.o").reshape(L, E)
            assert rel_err(g_o[perm], o_o) <= RTOL_F64, f"dir{dd}.o"
            g_m = gt.get(f"dir{dd}.masks", np.uint8).reshape(3, B, L, E)
            for k in range(3):
                assert np.array_equal(g_m[k, s], ot.get(f"dir{dd}.mask{k}").reshape(L, E)), (dd, k)
    assert n_out_total > 0, "the fixture must exercise the outlier path"


def _perm(order, t, g):
    m = g * g
    fast, slow = t % g, t // g
    return [slow * g + fast, m - 1 - (slow * g + fast), fast * g + slow, m - 1 - (fast * g + slow)][order]


def test_literal_scan_equals_channel_local(pair, gpu_ctx):
    """The literal detector (cross-channel max, quant.cpp:313-335) and the
    channel-local form agree wherever C(t) holds."""
    import torch
    import paper_2503_10959_b200 as ob
    om, gm, imgs, cimgs = pair
    spec = _spec(4, rho=0.1)
    ocal = om.calibrate(cimgs, spec).export()
    d = om.dims
    L, E, N = d.tokens, d.embed, d.state
    S = 2
    g = torch.Generator().manual_seed(5)
    u = torch.randn(S, L, E, dtype=torch.float64, generator=g).cuda()
    proj = (0.5 * torch.randn(S, L, E + 2 * N, dtype=torch.float64, generator=g)).cuda()
    a = torch.from_numpy(om.get("block0.dir0.a")).cuda()
    bd = torch.zeros(E, dtype=torch.float64).cuda()
    tc = [ocal.scan[k] for k in range(3)]
    s_in = [torch.from_numpy(t.s_in).cuda() for t in tc]
    s_full = [torch.from_numpy(t.s_full).cuda() for t in tc]
    outs = []
    for force in (False, True):
        o = torch.zeros(S, L, E, dtype=torch.float64, device="cuda")
        masks = torch.zeros(3, S, L, E, dtype=torch.uint8, device="cuda")
        gpu_ctx.quant_scan(S=S, T=L, E=E, order=1, grid=d.grid, u=u, proj=proj, a=a, b_delta=bd, o=o,
                           mode=ob.MODE_DYNAMIC, n_refresh=3, act_bits=4, outlier_bits=8,
                           theta=[t.theta for t in tc], s_in=s_in, s_full=s_full, force_literal=force, masks=masks)
        outs.append((o.cpu().numpy(), masks.cpu().numpy()))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("abits", [4, 8])
def test_k1_variants_identical(pair, abits):
    """Channel-parallel K1 (exact under the host-checked condition) and the
    literal detector kernel give bit-identical forwards."""
    om, gm, imgs, cimgs = pair
    spec = _spec(abits, rho=0.05)
    gcal = _import_calib(gm, om.calibrate(cimgs, spec).export(), spec)
    outs = []
    for v in (0, 1):
        gm.set_option("k1_variant", v)
        outs.append(gm.forward_host(imgs, gcal, 1))
    gm.set_option("k1_variant", 0)
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("abits", [4, 8])
def test_scan_variants_identical(pair, abits):
    """K3 fast path (certified f32 codes + exact fallbacks; at this batch the
    small-batch split-phase scan), its all-exact variant, the per-direction
    reference kernel and every fast kernel (one and two threads per channel,
    f32 / f64 state, the large-grid shape with A in shared memory that the
    benchmark batch runs) agree bit-for-bit."""
    om, gm, imgs, cimgs = pair
    spec = _spec(abits, rho=0.05)
    gcal = _import_calib(gm, om.calibrate(cimgs, spec).export(), spec)
    outs = []
    for v in (0, 1, 2, 3, 4, 5, 6, 7):
        gm.set_option("scan_variant", v)
        outs.append(gm.forward_host(imgs, gcal, 1))
    gm.set_option("scan_variant", 0)
    for v in (1, 2, 3, 4, 5, 6, 7):
        assert np.array_equal(outs[0], outs[v]), v


@pytest.mark.parametrize("abits,n_refresh", [(4, 10), (8, 7)])
def test_long_sequence_c4(oracle_checker, gpu_ctx, abits, n_refresh):
    """C4-shaped sequence length (448x448 / 16 -> L = 784, scan grid 28) at a
    small width: FP and quantized logits match the oracle, per-block traces are
    bit-exact for the quantized operands (refresh windows not dividing L)."""
    from oracle import oracle as O
    import paper_2503_10959_b200 as ob
    dims = dict(image=112, channels=3, patch=4, embed=64, state=16, blocks=1, classes=10, conv_width=4)
    om = oracle_checker.model(O.Dims(**dims), SEED)
    gm = ob.Model(gpu_ctx, ob.Dims(**dims), SEED)
    od = O.Dims(**dims)
    assert od.image // od.patch == 28
    imgs = oracle_checker.normal(11, 2 * od.pix).reshape(2, od.image, od.image, od.channels)
    cimgs = oracle_checker.normal(12, 2 * od.pix).reshape(2, od.image, od.image, od.channels)
    assert rel_err(gm.forward_host(imgs, None, 0), om.forward(imgs, None, 0)) <= RTOL_F64
    spec = _spec(abits, n_refresh=n_refresh, rho=0.02)
    ocal = om.calibrate(cimgs, spec)
    gcal = _import_calib(gm, ocal.export(), spec)
    for mode in (1, 2):
        assert rel_err(gm.forward_host(imgs, gcal, mode), om.forward(imgs, ocal, mode)) <= RTOL_F64, mode


@pytest.mark.parametrize("embed,abits", [(192, 8), (384, 4)])
def test_vim_t_s_widths(oracle_checker, gpu_ctx, embed, abits):
    """The C1 (Vim-T, E=192, W4A8) and C2 (Vim-S, E=384, W4A4) channel widths at
    a small image: FP and quantized (dynamic, static) logits vs the oracle, and
    the fast scan == its all-exact variant."""
    from oracle import oracle as O
    import paper_2503_10959_b200 as ob
    dims = dict(image=32, channels=3, patch=8, embed=embed, state=16, blocks=2, classes=10, conv_width=4)
    od = O.Dims(**dims)
    om = oracle_checker.model(od, SEED)
    gm = ob.Model(gpu_ctx, ob.Dims(**dims), SEED)
    imgs = oracle_checker.normal(31, 3 * od.pix).reshape(3, od.image, od.image, od.channels)
    cimgs = oracle_checker.normal(32, 3 * od.pix).reshape(3, od.image, od.image, od.channels)
    assert rel_err(gm.forward_host(imgs, None, 0), om.forward(imgs, None, 0)) <= RTOL_F64
    spec = _spec(abits, n_refresh=4, rho=0.02)
    ocal = om.calibrate(cimgs, spec)
    gcal = _import_calib(gm, ocal.export(), spec)
    for mode in (1, 2):
        assert rel_err(gm.forward_host(imgs, gcal, mode), om.forward(imgs, ocal, mode)) <= RTOL_F64, mode
    a = gm.forward_host(imgs, gcal, 1)
    gm.set_option("scan_variant", 2)
    b = gm.forward_host(imgs, gcal, 1)
    gm.set_option("scan_variant", 0)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("orders,n_refresh", [((2, 3), 4), ((1, 2), 0), ((3,), 5), ((0, 1), 0)])
def test_scan_orders_and_refresh_windows(oracle_checker, gpu_ctx, orders, n_refresh):
    """Column scan orders (scan_perm, ssm.cpp:30-46), a single direction and
    never-refreshing windows (n_refresh 0: the staged K1's row ring refills
    across the whole sequence; the x_proj K1 pair runs unmirrored for orders
    other than (0, 1)): FP and quantized logits bit-identical to the oracle."""
    from oracle import oracle as O
    import paper_2503_10959_b200 as ob
    dims = dict(image=48, channels=3, patch=8, embed=96, state=16, blocks=2, classes=10, conv_width=4)
    od = O.Dims(**dims)
    om = oracle_checker.model(od, SEED, orders=orders)
    gm = ob.Model(gpu_ctx, ob.Dims(**dims), SEED, orders=orders)
    imgs = oracle_checker.normal(41, 2 * od.pix).reshape(2, od.image, od.image, od.channels)
    cimgs = oracle_checker.normal(42, 2 * od.pix).reshape(2, od.image, od.image, od.channels)
    assert rel_err(gm.forward_host(imgs, None, 0), om.forward(imgs, None, 0)) <= RTOL_F64
    for abits in (4, 8):
        spec = _spec(abits, n_refresh=n_refresh, rho=0.02)
        ocal = om.calibrate(cimgs, spec)
        gcal = _import_calib(gm, ocal.export(), spec)
        for mode in (1, 2):
            assert rel_err(gm.forward_host(imgs, gcal, mode), om.forward(imgs, ocal, mode)) <= RTOL_F64, (abits, mode)


@pytest.mark.parametrize("E,T,n_refresh,order,src", [(768, 197, 10, 1, 0), (1024, 60, 0, 2, 0), (32, 33, 7, 3, 1),
                                                     (768, 50, 0, 1, 1), (256, 120, 25, 0, 1)])
def test_staged_k1_equals_literal(gpu_ctx, E, T, n_refresh, order, src):
    """The staged K1 (rows bulk-copied per refresh window, D1 factor from the
    staged rows) == the literal detector kernel, at Vim-B widths, with a ring
    that refills (n_refresh 0 or long windows) and every scan order."""
    import torch
    S = 2
    rng = np.random.default_rng(E + T + order)
    x = rng.normal(size=(S, T, E)) * (3.0 if src == 1 else 1.0)
    x[rng.random((S, T, E)) < 0.01] *= 25.0
    xd = torch.from_numpy(x).cuda()
    s_in = torch.from_numpy(np.full(T, 0.35)).cuda()
    grid = int(T ** 0.5) if order >= 2 else 0
    if order >= 2:
        T2 = grid * grid
        xd, s_in, T = xd[:, :T2].contiguous(), s_in[:T2].contiguous(), T2
    outs = []
    for lit in (False, True):
        r = gpu_ctx.detect_quantize(xd, S=S, T=T, E=E, theta=2.5, s_in=s_in, s_full=s_in, n_refresh=n_refresh,
                                    act_bits=4, outlier_bits=8, mode=1, src=src, order=order, grid=grid, literal=lit)
        torch.cuda.synchronize()
        outs.append({k: v.cpu().numpy() for k, v in r.items()})
    a, b = outs
    for k in ("codes", "s_row", "ocnt", "omask"):
        assert np.array_equal(a[k], b[k]), k
    m = np.unpackbits(a["omask"].view(np.uint8), bitorder="little").reshape(S * T, -1)[:, :E].astype(bool)
    assert m.any()
    assert np.array_equal(a["ocode"][m], b["ocode"][m]) and np.array_equal(a["oscale"][m], b["oscale"][m])


@pytest.mark.parametrize("graphs", [False, True])
def test_split_forward_identical(oracle_checker, gpu_ctx, graphs):
    """A batch split into independent sub-batches on their own streams
    ("split_parts" 2 / 4, uneven halves) gives the single-stream logits bit for
    bit, through the device forward and the host-feed (e2e) path, with and
    without CUDA-graph replay; the quantized logits also equal the oracle's."""
    import torch
    from oracle import oracle as O
    import paper_2503_10959_b200 as ob
    dims = dict(image=32, channels=3, patch=8, embed=64, state=16, blocks=2, classes=10, conv_width=4)
    od = O.Dims(**dims)
    om = oracle_checker.model(od, SEED)
    gm = ob.Model(gpu_ctx, ob.Dims(**dims), SEED)
    B = 130
    imgs = oracle_checker.normal(51, B * od.pix).reshape(B, od.image, od.image, od.channels)
    cimgs = oracle_checker.normal(52, 2 * od.pix).reshape(2, od.image, od.image, od.channels)
    spec = _spec(4, n_refresh=5, rho=0.02)
    ocal = om.calibrate(cimgs, spec)
    gcal = _import_calib(gm, ocal.export(), spec)
    gm.use_graphs(graphs)
    gm.set_option("split_min_rows", 0)  # the toy batch is far below the default part size
    dev = torch.from_numpy(imgs).cuda()
    res = {}
    for parts in (1, 2, 4):
        gm.set_option("split_parts", parts)
        for mode in (0, 1):
            cal = gcal if mode else None
            h = gm.forward_host(imgs, cal, mode)
            d = gm.forward(dev, cal, mode)
            torch.cuda.synchronize()
            res[(parts, mode)] = (h, d.cpu().numpy())
    for mode in (0, 1):
        base = res[(1, mode)][0]
        for parts in (1, 2, 4):
            for got in res[(parts, mode)]:
                assert np.array_equal(got, base), (parts, mode)
    assert rel_err(res[(2, 1)][0], om.forward(imgs, ocal, 1)) <= RTOL_F64
    gm.set_option("split_parts", 2)
    gm.set_option("split_min_rows", 16384)


def test_split_forward_with_spikes_identical(oracle_checker, gpu_ctx):
    """SpikeHook positions use the global sample index, so a spiked batch split
    into sub-batches gives the single-stream logits bit for bit."""
    from oracle import oracle as O
    import paper_2503_10959_b200 as ob
    dims = dict(image=32, channels=3, patch=8, embed=64, state=16, blocks=2, classes=10, conv_width=4)
    od = O.Dims(**dims)
    om = oracle_checker.model(od, SEED)
    gm = ob.Model(gpu_ctx, ob.Dims(**dims), SEED)
    B = 130
    imgs = oracle_checker.normal(61, B * od.pix).reshape(B, od.image, od.image, od.channels)
    cimgs = oracle_checker.normal(62, 2 * od.pix).reshape(2, od.image, od.image, od.channels)
    spec = _spec(4, n_refresh=5, rho=0.02)
    gcal = _import_calib(gm, om.calibrate(cimgs, spec).export(), spec)
    gm.set_spikes(ob.SpikeSettings(rate=0.3, gain=20.0, channels=2, salt=5))
    gm.set_option("split_min_rows", 0)  # the toy batch is far below the default part size
    res = {}
    for parts in (1, 2, 4):
        gm.set_option("split_parts", parts)
        res[parts] = [gm.forward_host(imgs, gcal if mode else None, mode) for mode in (0, 1)]
    # a shard of the batch (as one rank of a multi-GPU run sees it) with its global offset
    gm.set_option("split_parts", 1)
    gm.set_spikes(ob.SpikeSettings(rate=0.3, gain=20.0, channels=2, salt=5, sample0=65))
    shard = [gm.forward_host(imgs[65:], gcal if mode else None, mode) for mode in (0, 1)]
    for a, b in zip(shard, res[1]):
        assert np.array_equal(a, b[65:])
    gm.set_spikes(None)
    gm.set_option("split_parts", 2)
    plain = gm.forward_host(imgs, None, 0)
    assert not np.array_equal(plain, res[1][0])  # the hook fired
    for parts in (2, 4):
        for a, b in zip(res[parts], res[1]):
            assert np.array_equal(a, b), parts
