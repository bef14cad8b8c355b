"""K1 over streams of K x C planes and the GPU gemm-bench stage against the
reference's own code (oracle/_ref): maybe_refresh + detect_outliers +
split_quantize per step (quant.cpp:303-335, gemm.cpp:106-135) bit for bit, the
hybrid_gemm of every step (gemm.cpp:181-225), and bench_refresh_sweep's
mean |O| and scans per step (gemm.cpp:326-411)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _planes(rng, steps, K, C, n_spike):
    x = rng.normal(size=(steps, K, C))
    for t in range(steps):  # persistent and transient spikes, like the refresh sweep's stream
        for ch in range(n_spike):
            x[t, (7 * ch) % K] *= 40.0
        if rng.uniform() < 0.3:
            x[t, rng.integers(K)] *= 40.0
    s_in = np.array([np.abs(x[t]).max() / 7.0 / 30.0 for t in range(steps)])  # low: the scan fires
    theta = float(np.abs(x).max() / 40.0 * 1.5)
    return x, s_in, theta


def _words(mask_row, Kp):
    J = (Kp + 31) // 32
    w = np.zeros(J, np.uint32)
    for ch in np.flatnonzero(mask_row):
        w[ch // 32] |= np.uint32(1 << (ch % 32))
    return w


@pytest.mark.parametrize("steps,K,C,n_refresh,Kp", [(12, 64, 1, 5, 64), (20, 100, 7, 1, 112), (30, 512, 32, 10, 512),
                                                    (9, 48, 33, 0, 48), (16, 2048, 4, 3, 2048)])
def test_detect_quantize_planes_bit_exact(ref_checker, gpu_ctx, steps, K, C, n_refresh, Kp):
    import torch
    rng = np.random.default_rng(steps * 1000 + K + C)
    x, s_in, theta = _planes(rng, steps, K, C, n_spike=3)
    got = gpu_ctx.detect_quantize_planes(torch.from_numpy(x).cuda(), theta=theta, s_in=torch.from_numpy(s_in).cuda(),
                                         n_refresh=n_refresh, act_bits=4, outlier_bits=8, Kp=Kp)
    torch.cuda.synchronize()
    g = {k: v.cpu().numpy() for k, v in got.items()}
    _, masks, scanned = ref_checker.quant_stream(x[None], theta, s_in, s_in, n_refresh, 4, 8, mode=1)
    assert np.array_equal(g["scanned"], scanned[0])
    assert g["scanned"].any() and masks.any()
    for t in range(steps):
        chans = np.flatnonzero(masks[0, t])
        inl, oc, os_ = ref_checker.split_quantize(x[t], chans, s_in[t], 4, 8)
        rows = slice(t * C, (t + 1) * C)
        codes = g["codes"][rows]
        assert np.array_equal(codes[:, :K], inl.T), t
        assert not codes[:, K:].any()
        assert np.array_equal(g["omask"][rows].view(np.uint32), np.tile(_words(masks[0, t], Kp), (C, 1))), t
        assert np.all(g["ocnt"][rows] == len(chans))
        assert np.all(g["s_row"][rows] == s_in[t])
        for j, ch in enumerate(chans):
            assert np.array_equal(g["ocode"][rows, ch], oc[j]), (t, ch)
            assert np.all(g["oscale"][rows, ch] == os_[j]), (t, ch)


def test_planes_then_quant_linear_equal_hybrid_gemm_per_step(ref_checker, gpu_ctx):
    """The sweep's per-step pipeline: split planes -> K2 over all steps == the
    reference's hybrid_gemm of each step's split operands (output bit for bit)."""
    import torch
    rng = np.random.default_rng(5)
    steps, K, C, M = 14, 256, 24, 32
    x, s_in, theta = _planes(rng, steps, K, C, n_spike=5)
    got = gpu_ctx.detect_quantize_planes(torch.from_numpy(x).cuda(), theta=theta, s_in=torch.from_numpy(s_in).cuda(),
                                         n_refresh=4, act_bits=4, outlier_bits=8)
    w = rng.integers(-7, 8, size=(M, K), dtype=np.int8)
    ws = rng.uniform(0.005, 0.02, size=M)
    act = {k: v for k, v in got.items() if k != "scanned"}
    y = gpu_ctx.quant_linear(act, torch.from_numpy(w).cuda(), torch.from_numpy(np.ascontiguousarray(w.T)).cuda(),
                             torch.from_numpy(ws).cuda())
    torch.cuda.synchronize()
    y = y.cpu().numpy()
    _, masks, _ = ref_checker.quant_stream(x[None], theta, s_in, s_in, 4, 4, 8, mode=1)
    for t in range(steps):
        chans = np.flatnonzero(masks[0, t])
        inl, oc, os_ = ref_checker.split_quantize(x[t], chans, s_in[t], 4, 8)
        _, _, want = ref_checker.hybrid_gemm(w, ws, inl, s_in[t], chans, oc, os_)
        assert np.array_equal(y[t * C:(t + 1) * C], want.T), t


@pytest.mark.parametrize("periods,steps,m,k,c", [((1, 5, 10, 20, 0), 300, 8, 512, 32), ((1, 3, 0), 40, 12, 100, 5)])
def test_refresh_sweep_matches_reference(ref_checker, gpu_ctx, periods, steps, m, k, c):
    got = gpu_ctx.refresh_sweep(periods, steps=steps, m=m, k=k, c=c, trials=2, seed=3)
    mo, sc = ref_checker.ref_refresh_sweep(periods, steps, m, k, c, 6, 0.15, 40.0, 1, 3)
    assert [r["period"] for r in got] == list(periods)
    assert [r["mean_o_list"] for r in got] == mo.tolist()
    assert [r["scans_per_step"] for r in got] == sc.tolist()
    assert all(r["median_total_ns"] > 0 for r in got)


def test_refresh_sweep_outputs_shape_and_finite(gpu_ctx):
    recs, y = gpu_ctx.refresh_sweep((1, 0), steps=10, m=8, k=64, c=4, trials=1, outputs=True)
    assert y.shape == (2, 10, 4, 8) and np.isfinite(y).all() and np.abs(y).sum() > 0


def test_gemm_bench_records_match_reference(ref_checker, gpu_ctx):
    sizes = (64, 200, 512)
    got = gpu_ctx.gemm_bench(sizes, outlier_fraction=0.02, trials=3, seed=2)
    want = ref_checker.ref_gemm_bench(sizes, 0.02, 1, 2)
    assert [(0 if r["path"] == "hybrid" else 1, r["size"]) for r in got] == want
    assert all(r["median_ns"] > 0 for r in got)
    assert gpu_ctx.gemm_bench((64,), trials=1, f16_output=True)[0]["median_ns"] > 0


def test_plane_and_bench_validation(gpu_ctx):
    import torch
    import paper_2503_10959_b200 as ob
    x = torch.zeros(2, 5000, 1, dtype=torch.float64, device="cuda")
    with pytest.raises(ob.ValidationError):
        gpu_ctx.detect_quantize_planes(x, theta=1.0, s_in=torch.ones(2, dtype=torch.float64, device="cuda"),
                                       n_refresh=1)
    with pytest.raises(ob.ValidationError, match="spike gain must exceed 1"):
        gpu_ctx.refresh_sweep((1,), steps=4, spike_gain=1.0)
    with pytest.raises(ob.ValidationError, match="need steps >= 2"):
        gpu_ctx.refresh_sweep((1,), steps=1)
    with pytest.raises(ob.ValidationError, match="outlier fraction"):
        gpu_ctx.gemm_bench((64,), outlier_fraction=1.5)
