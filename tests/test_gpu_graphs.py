"""CUDA-graph replay safety of the C ABI forward entry points.

A captured graph holds raw device pointers (workspace, weights, calibration
tables) and by-value kernel parameters (thresholds, literal routing). These
tests interleave every API path that reallocates workspace or edits a
calibration between replays of the same key, and require the replayed logits
to equal an eager (graphs off) forward bit for bit.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DIMS = dict(image=32, channels=3, patch=8, embed=64, state=16, blocks=2, classes=10, conv_width=4)
SEED = 1234


@pytest.fixture(scope="module")
def setup(oracle_checker, gpu_ctx):
    from oracle import oracle as O
    import paper_2503_10959_b200 as ob
    od = O.Dims(**DIMS)
    om = oracle_checker.model(od, SEED)
    B = 130  # >= 64: the forward splits into two sub-batches, forward_profile does not
    imgs = oracle_checker.normal(61, B * od.pix).reshape(B, od.image, od.image, od.channels)
    cimgs = oracle_checker.normal(62, 4 * od.pix).reshape(4, od.image, od.image, od.channels)
    spec = O.Spec(wbits=4, abits=4, obits=8, n_refresh=5, rho=0.02)
    ocal = om.calibrate(cimgs, spec)
    gspec = ob.QuantSpec(4, 4, 8, 5, 0.02, True, True)
    return om, ocal, imgs, cimgs, gspec


def _model(gpu_ctx, ocal, gspec):
    import paper_2503_10959_b200 as ob
    gm = ob.Model(gpu_ctx, ob.Dims(**DIMS), SEED)
    conv = lambda t: ob.TensorCal(t.theta, t.s_in, t.s_full, t.excluded)
    ex = ocal.export()
    gcal = gm.calibration_from([conv(t) for t in ex.scan], [conv(t) for t in ex.lin], gspec)
    return gm, gcal


def test_replay_after_workspace_reallocation(setup, gpu_ctx):
    """use_graphs; forward x3 (eager, capture, replay); then forward_profile,
    a host-feed forward at another batch, a GPU calibration with a larger chunk
    and a trace — each reallocates workspace — and the same-key forward again."""
    import torch
    om, ocal, imgs, cimgs, gspec = setup
    gm, gcal = _model(gpu_ctx, ocal, gspec)
    want = om.forward(imgs, ocal, 1)
    dev = torch.from_numpy(imgs).cuda()
    logits = torch.empty(imgs.shape[0], DIMS["classes"], dtype=torch.float64, device="cuda")
    gm.use_graphs(True)

    def replay_equal():
        for _ in range(3):
            gm.forward(dev, gcal, 1, logits=logits)
            torch.cuda.synchronize()
            assert np.array_equal(logits.cpu().numpy(), want)

    replay_equal()
    gm.forward_profile(dev, gcal, 1)
    replay_equal()
    gm.forward_host(imgs[:7], gcal, 1)
    replay_equal()
    gm.calibrate(torch.from_numpy(np.concatenate([cimgs] * 40)).cuda(), gspec, chunk=160)
    replay_equal()
    gm.trace(imgs[:3], gcal, 1, 1)
    replay_equal()


def test_replay_after_calibration_edit(setup, gpu_ctx):
    """calib_set between replays: every later call (not only the first) uses
    the edited thresholds, through both the device and the host-feed paths."""
    import torch
    import paper_2503_10959_b200 as ob
    om, ocal, imgs, _, gspec = setup
    gm, gcal = _model(gpu_ctx, ocal, gspec)
    gm.use_graphs(True)
    dev = torch.from_numpy(imgs).cuda()
    logits = torch.empty(imgs.shape[0], DIMS["classes"], dtype=torch.float64, device="cuda")
    base = om.forward(imgs, ocal, 1)
    for _ in range(3):
        gm.forward(dev, gcal, 1, logits=logits)
        assert np.array_equal(gm.forward_host(imgs, gcal, 1), base)
    torch.cuda.synchronize()
    assert np.array_equal(logits.cpu().numpy(), base)
    # halve every linear-site threshold: many more outliers, different logits
    ex = ocal.export()
    for i in range(gcal.count(1)):
        t = gcal.get(1, i)
        gcal.set(1, i, ob.TensorCal(t.theta * 0.5, t.s_in, t.s_full, t.excluded))
    from oracle import oracle as O
    edited = O.Calibration(ex.spec, scan=ex.scan,
                           lin=[O.TensorCal(t.theta * 0.5, t.s_in, t.s_full, t.excluded) for t in ex.lin])
    want = om.forward(imgs, om.calib_from(edited), 1)
    assert not np.array_equal(want, base)
    for _ in range(4):
        gm.forward(dev, gcal, 1, logits=logits)
        torch.cuda.synchronize()
        assert np.array_equal(logits.cpu().numpy(), want)
        assert np.array_equal(gm.forward_host(imgs, gcal, 1), want)


def test_host_path_pageable_logits_with_graphs(setup, gpu_ctx):
    """Pinned images with pageable logits: the call must not try to capture a
    pageable D2H copy; repeated calls stay correct."""
    import torch
    om, ocal, imgs, _, gspec = setup
    gm, gcal = _model(gpu_ctx, ocal, gspec)
    gm.use_graphs(True)
    pinned = torch.empty(imgs.shape, dtype=torch.float64, pin_memory=True).numpy()
    pinned[...] = imgs
    want = om.forward(imgs, ocal, 1)
    for _ in range(4):
        out = np.empty((imgs.shape[0], DIMS["classes"]), np.float64)  # pageable
        gm.forward_host(pinned, gcal, 1, logits=out)
        assert np.array_equal(out, want)
    host_logits = torch.empty((imgs.shape[0], DIMS["classes"]), dtype=torch.float64, pin_memory=True).numpy()
    for _ in range(4):  # both pinned: the captured path
        gm.forward_host(pinned, gcal, 1, logits=host_logits)
        assert np.array_equal(host_logits, want)


def test_d1_mismatch_rejected(setup, gpu_ctx):
    """A calibration recorded with D1 cannot drive a d1 = 0 forward."""
    import paper_2503_10959_b200 as ob
    _, ocal, imgs, _, gspec = setup
    gm, gcal = _model(gpu_ctx, ocal, gspec)
    with pytest.raises(ob.OuroError, match="d1"):
        gm.forward_host(imgs[:2], gcal, 1, d1=False)
