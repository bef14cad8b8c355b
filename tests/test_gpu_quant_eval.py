"""GPU quant-eval == the reference's quantized_forward (quant.cpp:505-579):
FP and quantized logits, logits_mse, argmax agreement and the teacher-forced
per-(block, dir) scan-output MSE (run_quant_eval's metrics,
pipeline.cpp:115-167)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DIMS = dict(image=32, channels=3, patch=8, embed=64, state=16, blocks=2, classes=10, conv_width=4)
SEED = 9


# data seeds (calibration, eval): 31/32 is the case whose block-1 scan put a value
# within an ulp of a code boundary when the device used CUDA's exp; with glibc's
# algorithms on the device every case is bit-identical.
@pytest.mark.parametrize("abits,mode,seeds", [(4, 1, (21, 22)), (4, 2, (21, 22)), (8, 1, (21, 22)),
                                              (4, 1, (31, 32)), (4, 2, (31, 32)), (4, 0, (21, 22))])
def test_quant_eval_matches_reference(ref_checker, gpu_ctx, abits, mode, seeds):
    from oracle import oracle as O
    import paper_2503_10959_b200 as ob
    od = O.Dims(**DIMS)
    rm = ref_checker.model(od, SEED)
    cimgs = ref_checker.normal(seeds[0], 3 * od.pix).reshape(3, od.image, od.image, od.channels)
    imgs = ref_checker.normal(seeds[1], 4 * od.pix).reshape(4, od.image, od.image, od.channels)
    spec = O.Spec(wbits=4, abits=abits, obits=8, n_refresh=5, rho=0.05, d1=False, d2=False)
    rcal = rm.ref_calibrate(cimgs, spec)
    want = rm.ref_quant_eval(imgs, rcal, mode)

    gm = ob.Model(gpu_ctx, ob.Dims(**DIMS), SEED)
    conv = lambda t: ob.TensorCal(t.theta, t.s_in, t.s_full, t.excluded)
    gcal = gm.calibration_from([conv(t) for t in rcal.export().scan], [],
                               ob.QuantSpec(4, abits, 8, 5, 0.05, False, False))
    got = gm.quant_eval(imgs, gcal, mode, d1=False, d2=False)

    assert np.array_equal(np.asarray(got["logits_fp"]), np.asarray(want["logits_fp"]))
    assert np.array_equal(np.asarray(got["logits_q"]), np.asarray(want["logits_q"]))
    assert got["argmax_agree"] == want["argmax_agree"]
    assert abs(got["logits_mse"] - want["logits_mse"]) <= 1e-12 * want["logits_mse"]
    names = [n for n, _ in got["layer_mse"]]
    assert names == [f"block{b}.dir{d}" for b in range(DIMS["blocks"]) for d in range(2)]
    lm = np.array([v for _, v in got["layer_mse"]])
    assert np.all(np.abs(lm - want["layer_mse"]) <= 1e-12 * np.abs(want["layer_mse"]) + 1e-300)


@pytest.mark.parametrize("mode,spikes", [(1, (0.2, 100.0, 1, 0)), (1, (0.5, 30.0, 3, 7)), (2, (0.3, 100.0, 2, 1)),
                                         (0, (0.4, 50.0, 1, 3))])
def test_quant_eval_with_spikes_matches_reference(ref_checker, gpu_ctx, mode, spikes):
    """SpikeHook (quant.cpp:420-446) in all three passes: FP, quantized and the
    teacher-forced re-scan, bit for bit with the reference's quantized_forward."""
    from oracle import oracle as O
    import paper_2503_10959_b200 as ob
    od = O.Dims(**DIMS)
    rm = ref_checker.model(od, SEED)
    cimgs = ref_checker.normal(21, 3 * od.pix).reshape(3, od.image, od.image, od.channels)
    imgs = ref_checker.normal(22, 4 * od.pix).reshape(4, od.image, od.image, od.channels)
    spec = O.Spec(wbits=4, abits=4, obits=8, n_refresh=5, rho=0.05, d1=False, d2=False)
    rcal = rm.ref_calibrate(cimgs, spec)
    want = rm.ref_quant_eval(imgs, rcal, mode, spikes=spikes)

    gm = ob.Model(gpu_ctx, ob.Dims(**DIMS), SEED)
    conv = lambda t: ob.TensorCal(t.theta, t.s_in, t.s_full, t.excluded)
    gcal = gm.calibration_from([conv(t) for t in rcal.export().scan], [], ob.QuantSpec(4, 4, 8, 5, 0.05, False, False))
    got = gm.quant_eval(imgs, gcal, mode, d1=False, d2=False, spikes=ob.SpikeSettings(*spikes))
    assert np.array_equal(np.asarray(got["logits_fp"]), np.asarray(want["logits_fp"]))
    assert np.array_equal(np.asarray(got["logits_q"]), np.asarray(want["logits_q"]))
    assert got["argmax_agree"] == want["argmax_agree"]
    lm = np.array([v for _, v in got["layer_mse"]])
    assert np.all(np.abs(lm - want["layer_mse"]) <= 1e-12 * np.abs(want["layer_mse"]) + 1e-300)
    # spikes move the FP logits (the hook fired) and are switched off again afterwards
    plain = gm.forward_host(imgs, None, ob.MODE_FP, d1=False, d2=False)
    assert not np.array_equal(plain, np.asarray(got["logits_fp"]))
    assert np.array_equal(plain, rm.ref_quant_eval(imgs, rcal, 2)["logits_fp"])
