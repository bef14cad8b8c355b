"""Operator-level GPU parity (K1 detector/quantizer, K2 quant-linear) against
the oracle's restatement of detect_outliers / split_quantize / hybrid_gemm.
Mirrors the reference's own operator tests (tests/test_gemm.cpp,
tests/test_quant.cpp): integer planes bit-exact, output == the reference's
fused epilogue bit-for-bit."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _mask_words(mask_rows: np.ndarray) -> np.ndarray:
    """[M][K] 0/1 -> [M][ceil(K/32)] uint32 words (bit ch%32 of word ch/32)."""
    M, K = mask_rows.shape
    J = (K + 31) // 32
    padded = np.zeros((M, J * 32), np.uint64)
    padded[:, :K] = mask_rows
    w = (padded.reshape(M, J, 32) << np.arange(32, dtype=np.uint64)).sum(axis=2)
    return w.astype(np.uint32).view(np.int32)


def _unpack(words: np.ndarray, K: int) -> np.ndarray:
    w = words.view(np.uint32)
    return ((w[:, :, None] >> np.arange(32, dtype=np.uint32)) & 1).reshape(w.shape[0], -1)[:, :K].astype(np.uint8)


@pytest.mark.parametrize("M,R,K,n_o", [(128, 128, 128, 0), (300, 160, 256, 5), (1000, 800, 768, 12),
                                       (77, 1536, 192, 3), (4096, 768, 768, 8), (260, 96, 2048, 40)])
def test_quant_linear_shared_outliers_bit_exact(oracle_checker, gpu_ctx, M, R, K, n_o):
    """hybrid_gemm with one outlier list for all columns (gemm.cpp:181-225):
    acc_inlier / acc_outlier bit-exact, output bit-exact (same f64 op order)."""
    import torch
    rng = np.random.default_rng(M * 7 + R)
    w = rng.integers(-7, 8, size=(R, K), dtype=np.int8)
    ws = rng.uniform(0.005, 0.02, size=R)
    x = rng.integers(-7, 8, size=(M, K), dtype=np.int8)   # rows = tokens (columns of the reference plane)
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
    act = dict(codes=_dev(x), s_row=_dev(np.full(M, s_in)), ocnt=_dev(np.full(M, n_o, np.int32)),
               omask=_dev(_mask_words(mask)), ocode=_dev(dense_code), oscale=_dev(dense_scale))
    g_in = torch.zeros(M, R, dtype=torch.int32, device="cuda")
    g_out = torch.zeros(M, R, dtype=torch.int32, device="cuda")
    y = gpu_ctx.quant_linear(act, _dev(w), _dev(w.T.copy()), _dev(ws), acc_in=g_in, acc_out=g_out)
    torch.cuda.synchronize()
    assert np.array_equal(g_in.cpu().numpy(), acc_in.T)
    assert np.array_equal(g_out.cpu().numpy(), acc_out.T)
    assert np.array_equal(y.cpu().numpy(), out.T)


def test_quant_linear_validation(gpu_ctx):
    import paper_2503_10959_b200 as ob
    import torch
    act = dict(codes=torch.zeros(4, 20, dtype=torch.int8, device="cuda"),
               s_row=torch.ones(4, dtype=torch.float64, device="cuda"),
               ocnt=torch.zeros(4, dtype=torch.int32, device="cuda"),
               omask=torch.zeros(4, 1, dtype=torch.int32, device="cuda"),
               ocode=torch.zeros(4, 20, dtype=torch.int8, device="cuda"),
               oscale=torch.zeros(4, 20, dtype=torch.float64, device="cuda"))
    w = torch.zeros(32, 20, dtype=torch.int8, device="cuda")
    with pytest.raises(ob.ValidationError):  # K = 20 is not a multiple of 16
        gpu_ctx.quant_linear(act, w, w.t().contiguous(), torch.ones(32, dtype=torch.float64, device="cuda"))


@pytest.mark.parametrize("literal", [False, True])
@pytest.mark.parametrize("abits,n_refresh,mode", [(4, 3, 1), (8, 1, 1), (4, 0, 1), (4, 3, 2)])
def test_detect_quantize_matches_oracle(oracle_checker, gpu_ctx, abits, n_refresh, mode, literal):
    """K1 == maybe_refresh + detect_outliers + split_quantize per (sample,
    token) plane, state carried along the token order (D2); both the
    channel-parallel kernel and the literal one."""
    import torch
    S, T, E = 3, 40, 96
    rng = np.random.default_rng(abits * 10 + n_refresh)
    x = rng.normal(size=(S, T, E))
    spikes = rng.random((S, T, E)) < 0.02
    x[spikes] *= 30.0
    qa = 2 ** (abits - 1) - 1
    clean = np.abs(rng.normal(size=(T, E)))
    theta = float(np.quantile(clean.max(axis=0), 0.99)) * 1.5
    s_in = np.maximum(clean.max(axis=1), 1e-3) / qa
    s_full = s_in * 1.3
    assert np.all(np.nextafter(theta, np.inf) / qa > s_in)  # the channel-local form is exact here
    _, masks, scanned = oracle_checker.quant_stream(x.reshape(S, T, E, 1), theta, s_in, s_full, n_refresh, abits, 8,
                                                    mode)
    sc = torch.zeros(S * T, dtype=torch.uint8, device="cuda") if literal else None
    res = gpu_ctx.detect_quantize(_dev(x), S=S, T=T, E=E, theta=theta, s_in=_dev(s_in), s_full=_dev(s_full),
                                  n_refresh=n_refresh, act_bits=abits, outlier_bits=8, mode=mode, literal=literal,
                                  scanned=sc)
    torch.cuda.synchronize()
    codes = res["codes"].cpu().numpy().reshape(S, T, E)
    ocnt = res["ocnt"].cpu().numpy().reshape(S, T)
    omask = _unpack(res["omask"].cpu().numpy(), E).reshape(S, T, E)
    ocode = res["ocode"].cpu().numpy().reshape(S, T, E)
    osc = res["oscale"].cpu().numpy().reshape(S, T, E)
    s_row = res["s_row"].cpu().numpy().reshape(S, T)
    n_outliers = 0
    assert np.array_equal(omask, masks)
    for s in range(S):
        for t in range(T):
            chans = np.nonzero(masks[s, t])[0]
            S_t = s_in[t] if mode == 1 else s_full[t]
            inl, oc, os_ = oracle_checker.split_quantize(x[s, t].reshape(E, 1), chans, S_t, abits, 8)
            assert np.array_equal(codes[s, t], inl[:, 0]), (s, t)
            assert ocnt[s, t] == len(chans)
            assert np.array_equal(ocode[s, t, chans], oc[:, 0])
            assert np.array_equal(osc[s, t, chans], os_)
            assert s_row[s, t] == S_t
            n_outliers += len(chans)
    if mode == 1:
        if literal:
            assert np.array_equal(sc.cpu().numpy().reshape(S, T), scanned)
        assert n_outliers > 0


@pytest.mark.parametrize("S,E", [(2, 64), (8, 768)])
@pytest.mark.parametrize("src", [1, 2])
def test_detect_quantize_sources(oracle_checker, gpu_ctx, src, S, E):
    """RMSNorm (D1) and merge-gate sources: channel-parallel == literal kernel
    (merge: the lane-per-channel kernel of small batches, S x E <= 148 x 32, and
    the four-channel kernel above that)."""
    import torch
    T = 25
    rng = np.random.default_rng(src)
    x = _dev(rng.normal(size=(S, T, E)) * 3)
    x2 = _dev(rng.normal(size=(S, T, E)))
    gate = _dev(rng.normal(size=(S, T, E)))
    s_in = _dev(np.full(T, 0.4))
    outs = []
    for lit in (False, True):
        r = gpu_ctx.detect_quantize(x, S=S, T=T, E=E, theta=2.9, s_in=s_in, s_full=s_in, n_refresh=4, act_bits=4,
                                    outlier_bits=8, mode=1, src=src, x2=x2, gate=gate, literal=lit)
        torch.cuda.synchronize()
        outs.append({k: v.cpu().numpy() for k, v in r.items()})
    a, b = outs
    for k in ("codes", "s_row", "ocnt", "omask"):
        assert np.array_equal(a[k], b[k]), k
    m = _unpack(a["omask"], E).astype(bool)
    assert m.any()
    assert np.array_equal(a["ocode"][m], b["ocode"][m]) and np.array_equal(a["oscale"][m], b["oscale"][m])


@pytest.mark.parametrize("seed", [0, 1])
def test_detect_quantize_merge_edges(gpu_ctx, seed):
    """Merge source: the certified f32 evaluation of merged * silu(gate) == the
    exact f64 kernel on the cases that stress it: exact zeros (all-zero h codes
    give o = 0), zero gates, gates past +-80 (ex2 flush), subnormals, and values
    placed on / near half-integer quotients and near theta."""
    import torch
    S, T, E = 4, 30, 128
    rng = np.random.default_rng(seed)
    s_val, theta = 0.35, 2.4
    g = rng.normal(size=(S, T, E)) * 2.0
    o0 = rng.normal(size=(S, T, E))
    o1 = rng.normal(size=(S, T, E))
    sig = 1.0 / (1.0 + np.exp(-g))
    silu = g * sig
    kind = rng.integers(0, 8, size=(S, T, E))
    # 1: merged exactly zero; 2: gate zero; 3: gate far negative / positive; 4: subnormal merged
    o1[kind == 1] = -o0[kind == 1]
    g[kind == 2] = 0.0
    g[kind == 3] = rng.choice([-95.0, -81.0, 85.0, 300.0], size=int((kind == 3).sum()))
    o0[kind == 4] = 1e-310
    o1[kind == 4] = 0.0
    # 5/6: merged * silu(gate) / s on a half-integer (+- tiny) -> certification must refuse or be right
    silu = g * (1.0 / (1.0 + np.exp(-g)))
    target = (rng.integers(-6, 7, size=(S, T, E)) + 0.5) * s_val
    off = np.where(kind == 5, 0.0, rng.choice([1e-9, -1e-9, 1e-5, -1e-5, 3e-4], size=(S, T, E)))
    sel = (kind >= 5) & (kind <= 6) & (np.abs(silu) > 1e-3)
    m_target = (target + off * s_val) / np.where(sel, silu, 1.0)
    o0[sel] = m_target[sel]
    o1[sel] = 0.0
    # 7: close to theta
    sel7 = (kind == 7) & (np.abs(silu) > 1e-3)
    o0[sel7] = (theta * (1 + rng.choice([1e-12, -1e-12, 1e-6, -1e-6], size=int(sel7.sum())))) / silu[sel7]
    o1[sel7] = 0.0
    x, x2, gate = _dev(o0), _dev(o1), _dev(g)
    s_in = _dev(np.full(T, s_val))
    outs = []
    for lit in (False, True):
        r = gpu_ctx.detect_quantize(x, S=S, T=T, E=E, theta=theta, s_in=s_in, s_full=s_in, n_refresh=5, act_bits=4,
                                    outlier_bits=8, mode=1, src=2, x2=x2, gate=gate, literal=lit)
        torch.cuda.synchronize()
        outs.append({k: v.cpu().numpy() for k, v in r.items()})
    a, b = outs
    for k in ("codes", "s_row", "ocnt", "omask"):
        assert np.array_equal(a[k], b[k]), k
    m = _unpack(a["omask"], E).astype(bool)
    assert m.any() and (~m).any()
    assert np.array_equal(a["ocode"][m], b["ocode"][m]) and np.array_equal(a["oscale"][m], b["oscale"][m])


def test_scan_order_geometry_validated(gpu_ctx):
    """Column scan orders need T = grid^2; orders outside -1..3 are rejected
    (detect_quantize) before any kernel runs."""
    import torch
    import paper_2503_10959_b200 as ob
    x = torch.zeros(1, 10, 32, dtype=torch.float64, device="cuda")
    s = torch.ones(10, dtype=torch.float64, device="cuda")
    kw = dict(S=1, T=10, E=32, theta=1.0, s_in=s, s_full=s, n_refresh=2, act_bits=4, outlier_bits=8)
    with pytest.raises(ob.ValidationError, match="T = grid"):
        gpu_ctx.detect_quantize(x, order=2, grid=3, **kw)
    with pytest.raises(ob.ValidationError, match="order"):
        gpu_ctx.detect_quantize(x, order=5, grid=0, **kw)
    gpu_ctx.detect_quantize(x, order=1, grid=0, **kw)  # row orders need no grid
    torch.cuda.synchronize()


@pytest.mark.parametrize("S,E", [(3, 64), (3, 192), (3, 768), (8, 768)])
@pytest.mark.parametrize("src", [0, 1])
def test_detect_quantize_window_staged_literal_identical(gpu_ctx, S, E, src):
    """Plain / RMSNorm sources: the default channel-parallel kernel (literal=0:
    the register window kernel for small batches, S x E <= 148 x 32, else the
    bulk-copy staged kernel), the register window kernel (literal=2) and the
    literal detector (literal=1) give identical operands — dynamic (refresh
    windows of 8, 10 and 12+ rows, quotient bound theta/S below and above 2^14)
    and static (quotients up to 1e12, beyond the low-word range), every scan
    order, int8 and packed."""
    import torch
    T = 36  # T = 6^2 for the column orders
    rng = np.random.default_rng(E + src)
    x = rng.normal(size=(S, T, E)) * 2.0
    x[rng.random((S, T, E)) < 0.02] *= 40.0
    x[0, 5, 3] = 1e12  # static mode: |q| >= 2^31
    x[1, 7, 10] = -3e11
    xd = _dev(x)
    # theta / q_a = 0.44 > every S(t) <= 0.3 * 1.3: the channel-local form is exact
    cases = [(1, 4, 0.3, 3.1), (1, 10, 0.3, 3.1), (1, 13, 0.3, 3.1), (1, 10, 1e-5, 3.1), (2, 10, 0.3, 3.1)]
    for mode, n_refresh, sc, theta in cases:
        s_in = _dev(np.full(T, sc) * np.linspace(1.0, 1.3, T))
        for order, grid in ((-1, 0), (1, 0), (2, 6), (3, 6)):
            for packed in (False, True):
                outs = []
                for lit in (0, 2, 1):
                    r = gpu_ctx.detect_quantize(xd, S=S, T=T, E=E, theta=theta, s_in=s_in, s_full=s_in,
                                                n_refresh=n_refresh, act_bits=4, outlier_bits=8, mode=mode, src=src,
                                                order=order, grid=grid, literal=lit, packed=packed)
                    torch.cuda.synchronize()
                    outs.append({k: v.cpu().numpy() for k, v in r.items()})
                tag = (mode, n_refresh, sc, order, packed)
                for b in outs[1:]:
                    for k in ("codes4" if packed else "codes", "s_row", "ocnt", "omask"):
                        assert np.array_equal(outs[0][k], b[k]), (tag, k)
                    m = _unpack(outs[0]["omask"], E).astype(bool)
                    assert np.array_equal(outs[0]["ocode"][m], b["ocode"][m]), tag
                    assert np.array_equal(outs[0]["oscale"][m], b["oscale"][m]), tag
                if mode == 1:
                    assert _unpack(outs[0]["omask"], E).any(), tag
                elif not packed and order == -1:
                    c = outs[0]["codes"].reshape(S, T, E)
                    assert c[0, 5, 3] == 7 and c[1, 7, 10] == -7, tag  # saturated, not wrapped


@pytest.mark.parametrize("M,R,K", [(196, 192, 48), (200, 1000, 32), (1280, 960, 32)])
def test_dgemm_tiles_sequential_k(gpu_ctx, M, R, K):
    """The f64 projection GEMM (detail::mm, tensor.cpp:373-382): every output is
    0.0 + a[m][0] w[r][0] + a[m][1] w[r][1] + ... with separately rounded
    products and sums in ascending k, for both tile shapes (16x16 for problems
    with fewer 128x64 tiles than SMs, 128x64 above), store / bias / residual."""
    import paper_2503_10959_b200 as ob
    import torch
    rng = np.random.default_rng(M + R + K)
    a = rng.normal(size=(M, K))
    w = rng.normal(size=(R, K))
    bias = rng.normal(size=R)
    prev = rng.normal(size=(M, R))
    acc = np.zeros((M, R))
    for k in range(K):
        acc = acc + a[:, k:k + 1] * w[:, k][None, :]
    acc = 0.0 + acc
    for post, want in ((ob.POST_STORE, acc), (ob.POST_BIAS, acc + bias[None, :]), (ob.POST_RESID, prev + acc)):
        out = _dev(prev.copy()) if post == ob.POST_RESID else None
        got = gpu_ctx.dgemm(_dev(a), _dev(w), post=post, out=out, bias=_dev(bias) if post == ob.POST_BIAS else None)
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy(), want), post


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("S,E", [(8, 768), (2, 128)])
def test_detect_quantize_adversarial_values(oracle_checker, gpu_ctx, mode, S, E):
    """K1's branch-free code test against quantize_code's round-half-away on
    values placed on and next to half-integer quotients (S a power of two, so
    (k + 1/2) S is exact), signed zeros, subnormals and quotients far beyond
    the code range, for the staged kernel (S x E above one warp per SM), the
    register window kernel and the literal kernel: every code, mask and
    outlier value equals the oracle's split_quantize."""
    import torch
    T = 12
    rng = np.random.default_rng(S * E + mode)
    s_pow = 0.25
    s_in = np.full(T, s_pow)
    s_full = np.full(T, s_pow)
    theta = 7.5 * s_pow * 1.2  # inlier quotients up to +-8.99: ties at every half-integer in range
    k = rng.integers(-9, 9, size=(S, T, E)).astype(np.float64)
    x = (k + 0.5) * s_pow
    sel = rng.random((S, T, E))
    x = np.where(sel < 0.2, np.nextafter(x, np.inf), x)
    x = np.where((sel >= 0.2) & (sel < 0.4), np.nextafter(x, -np.inf), x)
    x = np.where((sel >= 0.4) & (sel < 0.45), -0.0, x)
    x = np.where((sel >= 0.45) & (sel < 0.5), 0.0, x)
    x = np.where((sel >= 0.5) & (sel < 0.53), 3e-310 * np.sign(k + 0.5), x)
    x = np.where((sel >= 0.53) & (sel < 0.55), 1e300 * np.sign(k + 0.5), x)
    x = np.where((sel >= 0.55) & (sel < 0.57), 3e9 * np.sign(k + 0.5), x)  # |q| >= 2^31 (static: saturate)
    xd = _dev(x)
    _, masks, _ = oracle_checker.quant_stream(x.reshape(S, T, E, 1), theta, s_in, s_full, 4, 4, 8, mode)
    for lit in (0, 2, 1):
        res = gpu_ctx.detect_quantize(xd, S=S, T=T, E=E, theta=theta, s_in=_dev(s_in), s_full=_dev(s_full),
                                      n_refresh=4, act_bits=4, outlier_bits=8, mode=mode, literal=lit)
        torch.cuda.synchronize()
        codes = res["codes"].cpu().numpy().reshape(S, T, E)
        omask = _unpack(res["omask"].cpu().numpy(), E).reshape(S, T, E)
        ocode = res["ocode"].cpu().numpy().reshape(S, T, E)
        osc = res["oscale"].cpu().numpy().reshape(S, T, E)
        assert np.array_equal(omask, masks), lit
        for s in range(S):
            for t in range(T):
                chans = np.nonzero(masks[s, t])[0]
                inl, oc, os_ = oracle_checker.split_quantize(x[s, t].reshape(E, 1), chans, s_pow, 4, 8)
                assert np.array_equal(codes[s, t], inl[:, 0]), (lit, s, t)
                assert np.array_equal(ocode[s, t, chans], oc[:, 0]), (lit, s, t)
                assert np.array_equal(osc[s, t, chans], os_), (lit, s, t)


@pytest.mark.parametrize("post", [0, 1, 4])
def test_quant_linear_full_wave_shapes_match_small_m(gpu_ctx, post):
    """The full-wave K2 shape (16 epilogue warps, one reused staging box, 4
    operand stages: M = 4096, R = 1536, K = 768 -> 384 tiles) against the M <=
    256 dp4a kernel (oracle-checked elsewhere) on the same rows, for the plain
    store, the in_proj split into u0 / gate (POST_INPROJ) and x_proj's
    softplus(y + b_delta) on the first columns (POST_XPROJ), outlier terms and
    the integer planes included."""
    import torch
    M, R, K = 4096, 1536, 768
    rng = np.random.default_rng(post + 7)
    w = rng.integers(-7, 8, size=(R, K), dtype=np.int8)
    ws = rng.uniform(0.005, 0.02, size=R)
    x = rng.integers(-7, 8, size=(M, K), dtype=np.int8)
    mask = (rng.random((M, K)) < 0.01).astype(np.uint8)
    x[mask.astype(bool)] = 0
    ocode = np.where(mask.astype(bool), rng.integers(-127, 128, size=(M, K)), 0).astype(np.int8)
    oscale = np.where(mask.astype(bool), rng.uniform(0.005, 0.02, size=(M, K)), 0.0)
    act = dict(codes=_dev(x), s_row=_dev(rng.uniform(0.005, 0.02, size=M)), ocnt=_dev(mask.sum(axis=1).astype(np.int32)),
               omask=_dev(_mask_words(mask)), ocode=_dev(ocode), oscale=_dev(oscale))
    wd, wtd, wsd = _dev(w), _dev(w.T.copy()), _dev(ws)
    bias = _dev(rng.normal(size=R))

    def run(a, m):
        if post == 1:
            out = torch.zeros(m, R // 2, dtype=torch.float64, device="cuda")
            out2 = torch.zeros(m, R // 2, dtype=torch.float64, device="cuda")
            gpu_ctx.quant_linear(a, wd, wtd, wsd, post=1, out=out, out2=out2, split=R // 2)
            y = torch.cat([out, out2], dim=1)
        elif post == 4:
            y = torch.zeros(m, R, dtype=torch.float64, device="cuda")
            gpu_ctx.quant_linear(a, wd, wtd, wsd, post=4, out=y, split=R // 2, bias=bias)
        else:
            y = torch.zeros(m, R, dtype=torch.float64, device="cuda")
            gpu_ctx.quant_linear(a, wd, wtd, wsd, post=0, out=y)
        ai = torch.zeros(m, R, dtype=torch.int32, device="cuda")
        ao = torch.zeros(m, R, dtype=torch.int32, device="cuda")
        gpu_ctx.quant_linear(a, wd, wtd, wsd, out=torch.zeros(m, R, dtype=torch.float64, device="cuda"),
                             acc_in=ai, acc_out=ao)
        torch.cuda.synchronize()
        return y.cpu().numpy(), ai.cpu().numpy(), ao.cpu().numpy()

    big = run(act, M)
    for m0 in (0, 1920, 3840):
        sub = {k: v[m0:m0 + 256].contiguous() for k, v in act.items()}
        small = run(sub, 256)
        for b, s_ in zip(big, small):
            assert np.array_equal(b[m0:m0 + 256], s_), m0
