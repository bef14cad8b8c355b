"""Operator-level GPU parity (K1 detector/quantizer, K2 quant-linear) against
the oracle's restatement of detect_outliers / split_quantize / hybrid_gemm.
Mirrors the reference's own operator tests (tests/test_gemm.cpp,
tests/test_quant.cpp): integer planes bit-exact, output == scale
decomposition."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("M,R,K,n_o", [(128, 128, 128, 0), (300, 160, 256, 5), (1000, 800, 768, 12),
                                       (77, 1536, 192, 3), (4096, 768, 768, 8)])
def test_quant_linear_shared_outliers_bit_exact(oracle_checker, gpu_ctx, M, R, K, n_o):
    """hybrid_gemm with one outlier list for all columns (gemm.cpp:181-225):
    acc_inlier / acc_outlier bit-exact, output bit-exact (same f64 op order)."""
    import torch
    rng = np.random.default_rng(M * 7 + R)
    w = rng.integers(-7, 8, size=(R, K), dtype=np.int8)
    ws = rng.uniform(0.005, 0.02, size=R)
    x = rng.integers(-7, 8, size=(M, K), dtype=np.int8)   # rows = tokens (columns of the reference plane)
    chans = np.sort(rng.choice(K, size=n_o, replace=False)).astype(np.uint64)
    x[:, chans.astype(np.int64)] = 0
    ocodes = rng.integers(-127, 128, size=(n_o, M), dtype=np.int8)
    oscales = rng.uniform(0.005, 0.02, size=n_o)
    s_in = float(rng.uniform(0.005, 0.02))
    acc_in, acc_out, out = oracle_checker.hybrid_gemm(w, ws, x.T.copy(), s_in, chans, ocodes, oscales)
    act = dict(codes=_dev(x), s_row=_dev(np.full(M, s_in)), ocnt=_dev(np.full(M, n_o, np.int32)),
               och=_dev(np.tile(np.pad(chans.astype(np.int16), (0, K - n_o)), (M, 1))),
               ocode=_dev(np.pad(ocodes.T, ((0, 0), (0, K - n_o)))),
               oscale=_dev(np.tile(np.pad(oscales, (0, K - n_o)), (M, 1))))
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
               och=torch.zeros(4, 20, dtype=torch.int16, device="cuda"),
               ocode=torch.zeros(4, 20, dtype=torch.int8, device="cuda"),
               oscale=torch.zeros(4, 20, dtype=torch.float64, device="cuda"))
    w = torch.zeros(32, 20, dtype=torch.int8, device="cuda")
    with pytest.raises(ob.ValidationError):  # K = 20 is not a multiple of 16
        gpu_ctx.quant_linear(act, w, w.t().contiguous(), torch.ones(32, dtype=torch.float64, device="cuda"))


@pytest.mark.parametrize("abits,n_refresh,mode", [(4, 3, 1), (8, 1, 1), (4, 0, 1), (4, 3, 2)])
def test_detect_quantize_matches_oracle(oracle_checker, gpu_ctx, abits, n_refresh, mode):
    """K1 == maybe_refresh + detect_outliers + split_quantize per (sample,
    token) plane, state carried along the token order (D2)."""
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
    # oracle: detector state per sequence, then split_quantize per token
    _, masks, scanned = oracle_checker.quant_stream(x.reshape(S, T, E, 1), theta, s_in, s_full, n_refresh, abits, 8,
                                                    mode)
    res = gpu_ctx.detect_quantize(_dev(x), S=S, T=T, E=E, theta=theta, s_in=_dev(s_in), s_full=_dev(s_full),
                                  n_refresh=n_refresh, act_bits=abits, outlier_bits=8, mode=mode,
                                  scanned=(sc := torch.zeros(S * T, dtype=torch.uint8, device="cuda")))
    torch.cuda.synchronize()
    codes = res["codes"].cpu().numpy().reshape(S, T, E)
    ocnt = res["ocnt"].cpu().numpy().reshape(S, T)
    och = res["och"].cpu().numpy().view(np.uint16).reshape(S, T, E)
    ocode = res["ocode"].cpu().numpy().reshape(S, T, E)
    osc = res["oscale"].cpu().numpy().reshape(S, T, E)
    s_row = res["s_row"].cpu().numpy().reshape(S, T)
    n_outliers = 0
    for s in range(S):
        for t in range(T):
            chans = np.nonzero(masks[s, t])[0]
            S_t = s_in[t] if mode == 1 else s_full[t]
            inl, oc, os_ = oracle_checker.split_quantize(x[s, t].reshape(E, 1), chans, S_t, abits, 8)
            assert np.array_equal(codes[s, t], inl[:, 0]), (s, t)
            assert ocnt[s, t] == len(chans)
            assert np.array_equal(och[s, t, :len(chans)], chans)
            assert np.array_equal(ocode[s, t, :len(chans)], oc[:, 0])
            assert np.array_equal(osc[s, t, :len(chans)], os_)
            assert s_row[s, t] == S_t
            n_outliers += len(chans)
    if mode == 1:
        assert np.array_equal(sc.cpu().numpy().reshape(S, T), scanned)
        assert n_outliers > 0
