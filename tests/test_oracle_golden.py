"""The oracle restatement against committed vectors generated from the
reference's own compiled code (tests/golden/make_golden.py). Runs on CPU."""
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_vectors.npz")
DIMS = dict(image=16, channels=3, patch=4, embed=16, state=4, blocks=2, classes=7, conv_width=3)
SEED = 2024


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


@pytest.fixture(scope="module")
def model(oracle_checker):
    from oracle import oracle as O
    return oracle_checker.model(O.Dims(**DIMS), SEED)


def test_seeded_weights(gold, model):
    for k, v in gold.items():
        if k.startswith("w."):
            assert np.array_equal(model.get(k[2:]), v), k


def test_normal_images(gold, oracle_checker, model):
    assert np.array_equal(oracle_checker.normal(5, gold["images"].size), gold["images"])


def test_fp_forward_equals_reference_vmm_forward_raw(gold, model):
    assert np.array_equal(model.forward(gold["images"], None, 0, d1=False, d2=False), gold["ref.fp_logits"])


def test_calibrate_equals_reference(gold, model):
    from oracle import oracle as O
    spec = O.Spec(abits=8, obits=8, n_refresh=3, rho=0.2, d1=False, d2=False)
    e = model.calibrate(gold["calib_images"], spec).export()
    assert np.array_equal([t.theta for t in e.scan], gold["ref.calib.theta"])
    assert np.array_equal(np.stack([t.s_in for t in e.scan]), gold["ref.calib.s_in"])
    assert np.array_equal(np.stack([t.s_full for t in e.scan]), gold["ref.calib.s_full"])


@pytest.mark.parametrize("mode", [1, 2])
def test_quantized_forward_equals_reference(gold, model, mode):
    from oracle import oracle as O
    spec = O.Spec(abits=8, obits=8, n_refresh=3, rho=0.2, d1=False, d2=False)
    c = model.calibrate(gold["calib_images"], spec)
    got = model.forward(gold["images"], c, mode, d1=False, d2=False)
    assert np.array_equal(got, gold[f"ref.quantized_forward.mode{mode}"])


@pytest.mark.parametrize("ab", [4, 8])
def test_extended_forward_equals_reference_driver(gold, model, ab):
    from oracle import oracle as O
    spec = O.Spec(abits=ab, obits=8, n_refresh=3, rho=0.1, d1=True, d2=True)
    c = model.calibrate(gold["calib_images"], spec)
    ce = c.export()
    assert np.array_equal([t.theta for t in ce.scan], gold[f"d12.a{ab}.theta_scan"])
    assert np.array_equal([t.theta for t in ce.lin], gold[f"d12.a{ab}.theta_lin"])
    assert np.array_equal(np.stack([t.s_in for t in ce.lin]), gold[f"d12.a{ab}.s_in_lin"])
    for mode in (0, 1, 2):
        assert np.array_equal(model.forward(gold["images"], c, mode), gold[f"d12.a{ab}.logits.mode{mode}"]), mode
    tr = model.trace(gold["images"][:DIMS["image"] ** 2 * 3], c, 1, 1)
    for k in ("lin0.codes", "lin0.omask", "lin0.acc_in", "lin3.codes", "lin1.acc_out", "dir0.mask0", "dir1.mask2",
              "dir0.o", "x_out"):
        assert np.array_equal(tr.get(k), gold[f"d12.a{ab}.trace.{k}"]), k


def test_hybrid_gemm_kat(gold, oracle_checker):
    g = gold
    a_in, a_out, y = oracle_checker.hybrid_gemm(g["op.hg.w"], g["op.hg.ws"], g["op.hg.x"], 0.05, g["op.hg.ch"],
                                                g["op.hg.oc"], g["op.hg.osc"])
    assert np.array_equal(a_in, g["op.hg.acc_in"]) and np.array_equal(a_out, g["op.hg.acc_out"])
    assert np.array_equal(y, g["op.hg.out"])


def test_detector_stream_kat(gold, oracle_checker):
    g = gold
    s_in = np.full(30, 3.0 / 127)
    fq, masks, scanned = oracle_checker.quant_stream(g["op.qs.x"], 3.0, s_in, s_in * 1.5, 4, 8, 8, 1)
    assert np.array_equal(fq, g["op.qs.fq"]) and np.array_equal(masks, g["op.qs.masks"])
    assert np.array_equal(scanned, g["op.qs.scanned"])
