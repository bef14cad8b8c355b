"""Calibration directories in the reference's on-disk format:
save_calibration / load_calibration, quant.cpp:179-290, OURO tensor files
tensor_io.hpp:13-19."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DIMS = dict(image=32, channels=3, patch=8, embed=64, state=16, blocks=2, classes=10, conv_width=4)
SEED = 5


def _ref_side(ref_checker, abits, d2):
    from oracle import oracle as O
    od = O.Dims(**DIMS)
    rm = ref_checker.model(od, SEED)
    cimgs = ref_checker.normal(3, 3 * od.pix).reshape(3, od.image, od.image, od.channels)
    imgs = ref_checker.normal(4, 2 * od.pix).reshape(2, od.image, od.image, od.channels)
    spec = O.Spec(wbits=4, abits=abits, obits=8, n_refresh=4, rho=0.05, d1=True, d2=d2)
    return rm, cimgs, imgs, spec


def _gpu_model(gpu_ctx):
    import paper_2503_10959_b200 as ob
    return ob.Model(gpu_ctx, ob.Dims(**DIMS), SEED)


def _gspec(s):
    import paper_2503_10959_b200 as ob
    return ob.QuantSpec(s.wbits, s.abits, s.obits, s.n_refresh, s.rho, s.d1, s.d2)


def _import(gm, cal, spec):
    import paper_2503_10959_b200 as ob
    conv = lambda t: ob.TensorCal(t.theta, t.s_in, t.s_full, t.excluded)
    return gm.calibration_from([conv(t) for t in cal.scan], [conv(t) for t in cal.lin], _gspec(spec))


@pytest.mark.parametrize("abits", [4, 8])
def test_save_is_byte_identical_to_reference(ref_checker, gpu_ctx, tmp_path, abits):
    """The reference's calibrate -> its save_calibration, and the same values
    saved by this library: identical calibration.txt and scale files."""
    rm, cimgs, _, spec = _ref_side(ref_checker, abits, d2=False)
    rcal = rm.ref_calibrate(cimgs, spec)
    rm.ref_save_calibration(rcal, tmp_path / "ref")
    gm = _gpu_model(gpu_ctx)
    gcal = _import(gm, rcal.export(), spec)
    gcal.save(tmp_path / "ours")
    ref_files = sorted(os.listdir(tmp_path / "ref"))
    assert ref_files == sorted(os.listdir(tmp_path / "ours"))
    assert "calibration.txt" in ref_files and len(ref_files) == 1 + DIMS["blocks"] * 2 * 3
    for f in ref_files:
        assert (tmp_path / "ref" / f).read_bytes() == (tmp_path / "ours" / f).read_bytes(), f


def test_load_reference_directory(ref_checker, gpu_ctx, tmp_path):
    """A reference-written directory loads (d2 = False) and drives the same
    forward as the calibration it was written from; asking for the D2 tables
    of a reference directory is a validation error."""
    import paper_2503_10959_b200 as ob
    rm, cimgs, imgs, spec = _ref_side(ref_checker, 4, d2=False)
    rcal = rm.ref_calibrate(cimgs, spec)
    rm.ref_save_calibration(rcal, tmp_path / "ref")
    gm = _gpu_model(gpu_ctx)
    loaded = gm.load_calibration(tmp_path / "ref", d1=True, d2=False)
    assert (loaded.spec.wbits, loaded.spec.abits, loaded.spec.obits, loaded.spec.n_refresh) == (4, 4, 8, 4)
    assert loaded.spec.rho == 0.05 and not loaded.spec.d2
    direct = _import(gm, rcal.export(), spec)
    for mode in (1, 2):
        a = gm.forward_host(imgs, loaded, mode, d1=True, d2=False)
        b = gm.forward_host(imgs, direct, mode, d1=True, d2=False)
        assert np.array_equal(a, b)
    with pytest.raises(ob.ValidationError):
        gm.load_calibration(tmp_path / "ref", d2=True)


def test_d2_round_trip_and_reference_reads_ours(ref_checker, gpu_ctx, tmp_path):
    """Save with the D2 linear-site tables, load back bit-identically; the
    reference loader reads the same directory (it ignores the D2 file)."""
    import torch
    from oracle import oracle as O
    rm, cimgs, _, spec = _ref_side(ref_checker, 4, d2=True)
    gm = _gpu_model(gpu_ctx)
    gcal = gm.calibrate(torch.from_numpy(cimgs).cuda(), _gspec(spec))
    gcal.save(tmp_path / "ours")
    assert os.path.exists(tmp_path / "ours" / "d2_linear_sites.txt")
    back = gm.load_calibration(tmp_path / "ours")
    (s0, l0), (s1, l1) = gcal.export(), back.export()
    assert len(l0) == len(l1) == DIMS["blocks"] * 4
    for a, b in zip(s0 + l0, s1 + l1):
        assert a.theta == b.theta
        assert np.array_equal(a.s_in, b.s_in) and np.array_equal(a.s_full, b.s_full)
        assert np.array_equal(a.excluded, b.excluded)
    rc = rm.ref_load_calibration(tmp_path / "ours", spec).export()
    assert len(rc.scan) == len(s0)
    for a, b in zip(s0, rc.scan):
        assert a.theta == b.theta and np.array_equal(a.s_in, b.s_in) and np.array_equal(a.s_full, b.s_full)


def test_io_errors(gpu_ctx, tmp_path):
    import paper_2503_10959_b200 as ob
    gm = _gpu_model(gpu_ctx)
    with pytest.raises(ob.IoError):
        gm.load_calibration(tmp_path / "missing", d2=False)
    (tmp_path / "bad").mkdir()
    (tmp_path / "bad" / "calibration.txt").write_text("tokens = 16\nthis line is malformed\n")
    with pytest.raises(ob.IoError):
        gm.load_calibration(tmp_path / "bad", d2=False)
    other = ob.Model(gpu_ctx, ob.Dims(**dict(DIMS, embed=32)), SEED)
    cal = other.new_calibration(ob.QuantSpec(4, 4, 8, 4, 0.05, True, False))
    cal.save(tmp_path / "other")
    with pytest.raises(ob.ValidationError):  # made for different model dims
        gm.load_calibration(tmp_path / "other", d2=False)
