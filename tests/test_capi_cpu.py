"""The C-ABI library without a GPU: it loads, exports every symbol that
include/ouro_b200.h declares, and follows the reference's error conventions
(NULL -> validation status + message, never a crash; free(NULL) is a no-op;
tests/test_capi.cpp:71-114)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ouro_b200.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(ouro_b200_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    import paper_2503_10959_b200 as ob
    return ob.load()


def test_header_symbols_exported(lib):
    names = declared()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
    import paper_2503_10959_b200._lib as L
    assert set(names) == set(L.EXPORTED)


def test_null_arguments_are_validation_errors(lib):
    assert lib.ouro_b200_ctx_create(0, None) == 2
    assert b"NULL" in lib.ouro_b200_last_error()
    assert lib.ouro_b200_ctx_synchronize(None) == 2
    assert lib.ouro_b200_model_set_tensor(None, b"x", None, 0) == 2
    assert lib.ouro_b200_forward(None, None, 1, 1, 1, None, 1, None) == 2
    assert lib.ouro_b200_trace_get(None, b"k", None, 0, None) == 2


def test_free_null_is_noop(lib):
    lib.ouro_b200_ctx_free(None)
    lib.ouro_b200_model_free(None)
    lib.ouro_b200_calib_free(None)
    lib.ouro_b200_trace_free(None)


def test_no_device_reports_status_not_crash(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    h = C.c_void_p()
    st = lib.ouro_b200_ctx_create(0, C.byref(h))
    assert st in (2, 3)
    assert lib.ouro_b200_last_error() != b""


def test_version_and_error_slot_cleared(lib):
    assert lib.ouro_b200_version().startswith(b"0.")
    lib.ouro_b200_ctx_free(None)
    assert lib.ouro_b200_ctx_synchronize(None) == 2
    assert lib.ouro_b200_last_error() != b""


def test_null_arguments_newer_entry_points(lib):
    """Every entry point added for the plane stream, the gemm-bench stage, spikes
    and the math diagnostic rejects NULL handles with the validation status."""
    P = None
    assert lib.ouro_b200_math_eval(P, 0, P, P, 4) == 2
    assert lib.ouro_b200_detect_quantize_planes(P, P, 1, 1, 1, C.c_double(1.0), P, 0, 4, 8, 1, P, P, P, P, P, P,
                                                P) == 2
    assert lib.ouro_b200_refresh_sweep(P, P, P, P) == 2
    assert lib.ouro_b200_gemm_bench(P, P, P) == 2
    assert lib.ouro_b200_model_set_spikes(P, P) == 2
    assert lib.ouro_b200_model_set_option(P, b"split_parts", 2) == 2
    assert lib.ouro_b200_quant_scan_spiked(P, 1, 1, 32, 16, 0, 0, P, P, P, P, P, 0, 0, 4, 8, P, P, P, P, 0, 0, 0) == 2
    assert b"NULL" in lib.ouro_b200_last_error()
