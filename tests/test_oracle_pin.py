"""Pins the oracle against the reference build (oracle/_ref, compiled from
the reference's own sources): the reference's unit tests pass under this
repo's doctest shim, and the restatement equals the reference bit-for-bit."""
import os
import subprocess

import numpy as np
import pytest

DIMS = dict(image=16, channels=3, patch=4, embed=12, state=4, blocks=2, classes=7, conv_width=3)


def test_reference_unit_tests_pass(ref_checker):
    from oracle import oracle as O
    here = os.path.dirname(O.ORACLE_SO)
    for t in ("test_quant", "test_gemm", "test_ssm", "test_tensor"):
        exe = os.path.join(here, "_ref", t)
        if not os.path.exists(exe):
            pytest.skip("reference test binaries not built")
        r = subprocess.run([exe], capture_output=True, text=True, cwd=os.path.join(here, "_ref"), timeout=300)
        assert r.returncode == 0, r.stdout + r.stderr
        assert "failed: 0" in r.stdout


@pytest.fixture(scope="module")
def both(oracle_checker, ref_checker):
    from oracle import oracle as O
    d = O.Dims(**DIMS)
    return oracle_checker.model(d, 5), ref_checker.model(d, 5), oracle_checker.normal(21, 4 * d.pix), \
        oracle_checker.normal(77, 3 * d.pix)


def test_weights_identical(both):
    mo, mr, _, _ = both
    for n in mo.tensor_names():
        assert np.array_equal(mo.get(n), mr.get(n)), n


def test_fp_and_quantized_forward_equal_reference_end_to_end(both):
    from oracle import oracle as O
    mo, mr, imgs, cimgs = both
    assert np.array_equal(mo.forward(imgs, None, 0, d1=False, d2=False), mr.ref_fp_forward(imgs))
    spec = O.Spec(abits=8, obits=8, n_refresh=3, rho=0.2, d1=False, d2=False)
    eo, er = mo.calibrate(cimgs, spec).export(), mr.ref_calibrate(cimgs, spec).export()
    for a, b in zip(eo.scan, er.scan):
        assert a.theta == b.theta and np.array_equal(a.s_in, b.s_in) and np.array_equal(a.excluded, b.excluded)
    rc = mr.ref_calibrate(cimgs, spec)
    for mode in (1, 2):
        lq, _ = mr.ref_quantized_forward(imgs, rc, mode)
        assert np.array_equal(mo.forward(imgs, mo.calib_from(er), mode, d1=False, d2=False), lq), mode


@pytest.mark.parametrize("ab", [4, 8])
def test_extended_forward_equals_reference_primitives(both, ab):
    from oracle import oracle as O
    mo, mr, imgs, cimgs = both
    spec = O.Spec(abits=ab, obits=8, n_refresh=3, rho=0.1)
    co, cr = mo.calibrate(cimgs, spec), mr.calibrate(cimgs, spec)
    for a, b in zip(co.export().scan + co.export().lin, cr.export().scan + cr.export().lin):
        assert a.theta == b.theta and np.array_equal(a.s_in, b.s_in)
    for mode in (0, 1, 2):
        assert np.array_equal(mo.forward(imgs, co, mode), mr.forward(imgs, cr, mode)), mode
