"""The reference's own known-answer tests (tests/test_quant.cpp,
tests/test_gemm.cpp) restated against the oracle's operator entry points."""
import numpy as np
import pytest


def code(chk, x, s, bits):
    """quantize_code through split_quantize on a 1x1 plane (quant.cpp:29-35)."""
    inl, _, _ = chk.split_quantize(np.array([[x]]), [], s, bits, 8 if bits <= 8 else bits)
    return int(inl[0, 0])


def test_rounding_and_clipping(oracle_checker):  # test_quant.cpp:57-81
    c = oracle_checker
    assert code(c, 0.5, 1.0, 8) == 1 and code(c, -0.5, 1.0, 8) == -1
    assert code(c, 2.5, 1.0, 8) == 3 and code(c, -2.5, 1.0, 8) == -3
    assert code(c, 1.49, 1.0, 8) == 1
    assert code(c, 1000.0, 1.0, 4) == 7 and code(c, -1000.0, 1.0, 4) == -7
    assert code(c, 1000.0, 1.0, 8) == 127 and code(c, -1000.0, 1.0, 8) == -127


def test_round_trip_lattice(oracle_checker):  # test_quant.cpp:83-105
    s = 0.37
    xs = np.array([[k * s] for k in range(-7, 8)])
    inl, _, _ = oracle_checker.split_quantize(xs, [], s, 4, 8)
    assert np.array_equal(inl[:, 0] * s, xs[:, 0])
    rng = np.random.default_rng(11)
    x = rng.uniform(-7 * s, 7 * s, size=(2000, 1))
    inl, _, _ = oracle_checker.split_quantize(x, [], s, 4, 8)
    assert np.max(np.abs(inl[:, 0] * s - x[:, 0])) <= s / 2 + 1e-15


def test_pack_int4_layout(oracle_checker):  # test_gemm.cpp:39-64
    codes = np.array([[1, -2, 3], [-7, 7, 0]], np.int8)
    p = oracle_checker.pack_int4(codes)
    assert p.shape == (2, 2)
    assert p[0, 0] == ((1 & 0xF) | ((-2 & 0xF) << 4)) and p[0, 1] == 3  # odd trailing nibble high bits 0
    assert p[1, 0] == ((-7 & 0xF) | (7 << 4))
    from oracle.oracle import OracleError
    with pytest.raises(OracleError):
        oracle_checker.pack_int4(np.array([[-8]], np.int8))


def test_detector_equals_exhaustive_scan(oracle_checker):  # test_quant.cpp:276-315
    e, n, steps, theta = 16, 4, 400, 3.0
    rng = np.random.default_rng(77)
    x = 0.5 * rng.normal(size=(1, steps, e, n))
    for t in range(steps):
        if rng.random() < 0.3:
            for _ in range(1 + rng.integers(3)):
                x[0, t, rng.integers(e), rng.integers(n)] = (1 if rng.random() < 0.5 else -1) * (theta + 5 * rng.random())
    s_in = np.full(steps, theta / 127.0)
    _, masks, _ = oracle_checker.quant_stream(x, theta, s_in, s_in, 1, 8, 8, 1)
    exhaustive = (np.abs(x[0]).max(axis=2) > theta).astype(np.uint8)
    assert np.array_equal(masks[0], exhaustive)
    assert exhaustive.any(axis=1).sum() > 50


def test_detection_trigger_semantics(oracle_checker):  # test_quant.cpp:317-347
    x = np.full((1, 1, 4, 2), 0.1)
    _, m, sc = oracle_checker.quant_stream(x, 3.0, np.array([1 / 127]), np.array([1.0]), 0, 8, 8, 1)
    assert sc[0, 0] == 0 and m.sum() == 0
    x[0, 0, 1, 1] = 5.0
    _, m, sc = oracle_checker.quant_stream(x, 3.0, np.array([1 / 127]), np.array([1.0]), 0, 8, 8, 1)
    assert sc[0, 0] == 1 and list(np.nonzero(m[0, 0])[0]) == [1]


def test_hybrid_decomposition(oracle_checker):  # test_gemm.cpp:193-234
    rng = np.random.default_rng(53)
    m, k, c = 7, 24, 10
    w = rng.integers(-7, 8, size=(m, k), dtype=np.int8)
    ws = rng.uniform(0.01, 0.1, size=m)
    x = rng.integers(-7, 8, size=(k, c), dtype=np.int8)
    ch = np.array([3, 5, 16], np.uint64)
    x[ch.astype(int)] = 0
    oc = rng.integers(-127, 128, size=(3, c), dtype=np.int8)
    osc = rng.uniform(0.01, 0.1, size=3)
    a_in, a_out, y = oracle_checker.hybrid_gemm(w, ws, x, 0.05, ch, oc, osc)
    assert np.array_equal(a_in, w.astype(np.int32) @ x.astype(np.int32))
    assert np.array_equal(a_out, w[:, ch.astype(int)].astype(np.int32) @ oc.astype(np.int32))
    want = 0.05 * a_in + (w[:, ch.astype(int)] * osc) @ oc.astype(np.float64)
    assert np.max(np.abs(ws[:, None] * want - y)) <= 1e-9
