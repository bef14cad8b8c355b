"""Device exp / log1p / softplus / SiLU against the host libm the reference calls
(glibc's std::exp / std::log1p; softplus_val / sigmoid_val / silu_val at
tensor.hpp:146-154): bit for bit on the argument ranges the path produces and on
the special values. CUDA's own exp differs from glibc's on ~6% of arguments, so
this is what keeps codes from flipping on a rounding boundary end to end."""
import ctypes
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

_libm = ctypes.CDLL("libm.so.6")
for _f in ("exp", "log1p"):
    getattr(_libm, _f).restype = ctypes.c_double
    getattr(_libm, _f).argtypes = [ctypes.c_double]


def _softplus(x):  # tensor.hpp:152
    return max(x, 0.0) + _libm.log1p(_libm.exp(-abs(x)))


def _silu(x):  # tensor.hpp:146-150, 154
    if x >= 0.0:
        s = 1.0 / (1.0 + _libm.exp(-x))
    else:
        e = _libm.exp(x)
        s = e / (1.0 + e)
    return x * s


HOST = {"exp": _libm.exp, "log1p": _libm.log1p, "softplus": _softplus, "silu": _silu}
RANGES = {"exp": [(-60.0, 0.0), (-1.0, 1.0), (-760.0, 710.0)], "log1p": [(0.0, 1.0), (-1.0, 10.0), (0.0, 1e-6)],
          "softplus": [(-40.0, 40.0), (-3.0, 3.0)], "silu": [(-50.0, 50.0), (-3.0, 3.0)]}
SPECIAL = [0.0, -0.0, math.inf, -math.inf, 709.782712893384, -745.1332191019412, -708.3964185322641, 1e-300,
           -1.0 + 1e-16, 2e-54, 5e-324, -5e-324, 1e-20, 36.0, -36.0]


@pytest.mark.parametrize("fn", ["exp", "log1p", "softplus", "silu"])
def test_device_math_equals_libm(gpu_ctx, fn):
    import torch
    rng = np.random.default_rng(hash(fn) % 1000)
    xs = [rng.uniform(lo, hi, 60000) for lo, hi in RANGES[fn]]
    x = np.concatenate(xs + [np.array(SPECIAL)])
    if fn == "log1p":
        x = x[x >= -1.0]
    y = gpu_ctx.math_eval(fn, torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    got = y.cpu().numpy()
    want = np.array([HOST[fn](float(v)) for v in x])
    same = (got.view(np.uint64) == want.view(np.uint64)) | (np.isnan(got) & np.isnan(want))
    bad = np.flatnonzero(~same)
    assert bad.size == 0, f"{fn}: {bad.size} of {x.size} differ, e.g. x={x[bad[0]]!r} gpu={got[bad[0]]!r} libm={want[bad[0]]!r}"


def test_math_eval_rejects_bad_fn(gpu_ctx):
    import torch
    import paper_2503_10959_b200 as ob
    x = torch.zeros(4, dtype=torch.float64, device="cuda")
    with pytest.raises(ob.ValidationError):
        ob._lib.check(gpu_ctx.lib.ouro_b200_math_eval(gpu_ctx.h, 7, ctypes.c_void_p(x.data_ptr()),
                                                      ctypes.c_void_p(x.data_ptr()), 4))
