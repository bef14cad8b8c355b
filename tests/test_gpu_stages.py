"""GPU pipeline stages at the C ABI against the reference's
own stages (pipeline.cpp, compiled in oracle/_ref and driven by a config text
in the reference's format): ouro_b200_calib_stage writes the same calibration
directory as run_calib, and ouro_b200_quant_eval writes a metrics.txt
byte-identical to run_quant_eval's (same run id) — logits_mse, argmax
agreement, every teacher-forced mse_block<b>.dir<d> and the QuantHook timeline —
for the dynamic, static and bypass modes and with SpikeHook."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DIMS = dict(image=32, channels=3, patch=8, embed=64, state=16, blocks=2, classes=10, conv_width=4)
SEED = 9


def _text(mode, abits=4, n_refresh=5, rho=0.05, eval_batch=3, spikes=(0.0, 100.0, 1)):
    m = "\n".join(f"{k} = {v}" for k, v in DIMS.items())
    return (f"[model]\nseed = {SEED}\n{m}\n\n[quant]\nweight_bits = 4\nact_bits = {abits}\noutlier_bits = 8\n"
            f"n_refresh = {n_refresh}\noutlier_quantile = {rho!r}\nmode = {mode}\neval_batch = {eval_batch}\n"
            f"spike_rate = {spikes[0]!r}\nspike_gain = {spikes[1]!r}\nspike_channels = {spikes[2]}\n")


def _cfg(mode, run_id, abits=4, n_refresh=5, rho=0.05, eval_batch=3, spikes=(0.0, 100.0, 1)):
    import paper_2503_10959_b200 as ob
    return ob.StageConfig(dims=ob.Dims(**DIMS), seed=SEED, weight_bits=4, act_bits=abits, outlier_bits=8,
                          n_refresh=n_refresh, outlier_quantile=rho, mode=mode, eval_batch=eval_batch,
                          spike_rate=spikes[0], spike_gain=spikes[1], spike_channels=spikes[2], run_id=run_id)


@pytest.fixture(scope="module")
def files(ref_checker, tmp_path_factory, gpu_ctx):
    import paper_2503_10959_b200 as ob
    d = tmp_path_factory.mktemp("stages")
    pix = DIMS["image"] ** 2 * 3
    ob.tensor_save(d / "calib_images.ouro", ref_checker.normal(41, 4 * pix).reshape(4, pix))
    ob.tensor_save(d / "images.ouro", ref_checker.normal(42, 5 * pix).reshape(5, pix))
    return d


@pytest.mark.parametrize("abits", [4, 8])
def test_calib_stage_matches_reference(ref_checker, files, abits):
    import paper_2503_10959_b200 as ob
    text = _text("dynamic", abits=abits)
    ref_dir, our_dir = files / f"ref_cal{abits}", files / f"our_cal{abits}"
    ref_checker.ref_run_calib(text, files / "calib_images.ouro", ref_dir)
    ob.calib_stage(_cfg("dynamic", ref_checker.ref_run_id(text), abits=abits), files / "calib_images.ouro", our_dir)
    names = sorted(p.name for p in ref_dir.iterdir() if p.name != "manifest.txt")
    assert names == sorted(p.name for p in our_dir.iterdir() if p.name != "manifest.txt")
    for n in names:
        assert (ref_dir / n).read_bytes() == (our_dir / n).read_bytes(), n


@pytest.mark.parametrize("mode,abits,spikes", [("dynamic", 4, (0.0, 100.0, 1)), ("static", 4, (0.0, 100.0, 1)),
                                               ("bypass", 4, (0.0, 100.0, 1)), ("dynamic", 8, (0.0, 100.0, 1)),
                                               ("dynamic", 4, (0.3, 50.0, 2))])
def test_quant_eval_stage_metrics_byte_identical(ref_checker, files, mode, abits, spikes):
    import paper_2503_10959_b200 as ob
    text = _text(mode, abits=abits, spikes=spikes)
    cal = files / f"ref_cal_{abits}"
    if not cal.exists():
        ref_checker.ref_run_calib(_text("dynamic", abits=abits), files / "calib_images.ouro", cal)
    ref_out, our_out = files / f"ref_qe_{mode}_{abits}_{spikes[0]}", files / f"our_qe_{mode}_{abits}_{spikes[0]}"
    ref_checker.ref_run_quant_eval(text, cal, files / "images.ouro", ref_out)
    ob.quant_eval_stage(_cfg(mode, ref_checker.ref_run_id(text), abits=abits, spikes=spikes), cal,
                        files / "images.ouro", our_out)
    want = (ref_out / "metrics.txt").read_text()
    got = (our_out / "metrics.txt").read_text()
    assert "stage=quant-eval" in want and (mode != "dynamic" or "stage=timeline" in want)
    assert got == want
    assert "stage = quant-eval" in (our_out / "manifest.txt").read_text()


def test_quant_eval_stage_errors(ref_checker, files):
    import paper_2503_10959_b200 as ob
    cal = files / "ref_cal_4"
    if not cal.exists():
        ref_checker.ref_run_calib(_text("dynamic"), files / "calib_images.ouro", cal)
    with pytest.raises(ob.ValidationError, match="different quantization settings"):
        ob.quant_eval_stage(_cfg("dynamic", None, n_refresh=7), cal, files / "images.ouro", files / "e1")
    with pytest.raises(ob.ValidationError, match="quant.mode"):
        ob.quant_eval_stage(_cfg("fast", None), cal, files / "images.ouro", files / "e2")
    with pytest.raises(ob.IoError):
        ob.quant_eval_stage(_cfg("dynamic", None), cal, files / "missing.ouro", files / "e3")
    ob.tensor_save(files / "bad_images.ouro", np.zeros((2, 5)))
    with pytest.raises(ob.ValidationError, match="expected shape"):
        ob.quant_eval_stage(_cfg("dynamic", None), cal, files / "bad_images.ouro", files / "e4")
