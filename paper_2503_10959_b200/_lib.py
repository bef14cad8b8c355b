"""ctypes binding of the C ABI in include/ouro_b200.h (libouro_b200.so).

The library is built in-tree (``make -C paper_2503_10959_b200``). There is no
fallback: if the shared object is missing or the device is not sm_100a, every
entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(HERE, "libouro_b200.so")

_P = C.c_void_p
_SZ = C.c_size_t
_U = C.c_uint
_I = C.c_int
_D = C.c_double

OK, ERR_VALIDATION, ERR_NUMERIC, ERR_IO = 0, 2, 3, 4
MODE_FP, MODE_DYNAMIC, MODE_STATIC = 0, 1, 2
POST_STORE, POST_INPROJ, POST_RESID, POST_BIAS, POST_XPROJ = 0, 1, 2, 3, 4
SRC_PLAIN, SRC_RMSNORM, SRC_MERGE = 0, 1, 2

_SIGS = {
    "ouro_b200_version": ([], C.c_char_p),
    "ouro_b200_last_error": ([], C.c_char_p),
    "ouro_b200_ctx_create": ([_I, C.POINTER(_P)], _I),
    "ouro_b200_ctx_free": ([_P], None),
    "ouro_b200_ctx_set_stream": ([_P, _P], _I),
    "ouro_b200_ctx_synchronize": ([_P], _I),
    "ouro_b200_ctx_num_sms": ([_P, C.POINTER(_I)], _I),
    "ouro_b200_detect_quantize": ([_P, _P, _P, _P, _SZ, _SZ, _SZ, _I, _I, _I, _D, _P, _P, _SZ, _U, _U, _I, _I, _P,
                                   _P, _P, _P, _P, _P, _P, _P], _I),
    "ouro_b200_quant_linear": ([_P, _SZ, _SZ, _SZ, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _P, _SZ, _P, _SZ, _P,
                                _P, _P], _I),
    "ouro_b200_detect_quantize_packed": ([_P, _P, _P, _P, _SZ, _SZ, _SZ, _I, _I, _I, _D, _P, _P, _SZ, _U, _I, _I,
                                          _P, _P, _P, _P, _P, _P, _P], _I),
    "ouro_b200_quant_linear_packed": ([_P, _SZ, _SZ, _SZ, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _P, _SZ, _P, _SZ,
                                       _P, _P, _P], _I),
    "ouro_b200_quant_scan": ([_P, _SZ, _SZ, _SZ, _SZ, _I, _I, _P, _P, _P, _P, _P, _I, _SZ, _U, _U, _P, _P, _P, _P,
                              _I, _P], _I),
    "ouro_b200_dgemm": ([_P, _SZ, _SZ, _SZ, _P, _SZ, _P, _I, _P, _SZ, _P, _SZ, _P], _I),
    "ouro_b200_model_create": ([_P, _P, _P, _SZ, C.c_uint64, C.POINTER(_P)], _I),
    "ouro_b200_model_free": ([_P], None),
    "ouro_b200_model_set_tensor": ([_P, C.c_char_p, _P, _SZ], _I),
    "ouro_b200_model_get_tensor": ([_P, C.c_char_p, _P, _SZ, C.POINTER(_SZ)], _I),
    "ouro_b200_calib_create": ([_P, _P, _SZ, _D, _I, _I, C.POINTER(_P)], _I),
    "ouro_b200_calibrate": ([_P, _P, _SZ, _P, _SZ, _D, _I, _I, _SZ, C.POINTER(_P)], _I),
    "ouro_b200_calib_free": ([_P], None),
    "ouro_b200_calib_count": ([_P, _I, C.POINTER(_SZ)], _I),
    "ouro_b200_calib_get": ([_P, _I, _SZ, C.POINTER(_D), _P, _P, _P], _I),
    "ouro_b200_calib_set": ([_P, _I, _SZ, _D, _P, _P, _P], _I),
    "ouro_b200_forward": ([_P, _P, _I, _I, _I, _P, _SZ, _P], _I),
    "ouro_b200_forward_host": ([_P, _P, _I, _I, _I, _P, _SZ, _P], _I),
    "ouro_b200_model_use_graphs": ([_P, _I], _I),
    "ouro_b200_model_set_option": ([_P, C.c_char_p, C.c_long], _I),
    "ouro_b200_forward_profile":([_P, _P, _I, _I, _I, _P, _SZ, _P, _P, _P], _I),
    "ouro_b200_forward_profile_launches": ([_P, _P, _I, _I, _I, _P, _SZ, _P, _P, _P, _SZ, C.POINTER(_SZ)], _I),
    "ouro_b200_measure_fp64_peak": ([_P, C.POINTER(_D)], _I),
    "ouro_b200_measure_i8_peak": ([_P, C.POINTER(_D)], _I),
    "ouro_b200_launch_count": ([C.POINTER(C.c_longlong)], _I),
    "ouro_b200_tensor_save": ([C.c_char_p, _I, _P, _SZ, _P, _I], _I),
    "ouro_b200_tensor_info": ([C.c_char_p, C.POINTER(_I), _P, _SZ, C.POINTER(_SZ)], _I),
    "ouro_b200_tensor_load": ([C.c_char_p, _I, _P, _SZ, _I], _I),
    "ouro_b200_quant_eval": ([_P, C.c_char_p, C.c_char_p, C.c_char_p], _I),
    "ouro_b200_calib_stage": ([_P, C.c_char_p, C.c_char_p], _I),
    "ouro_b200_math_eval": ([_P, _I, _P, _P, _SZ], _I),
    "ouro_b200_detect_quantize_planes": ([_P, _P, _SZ, _SZ, _SZ, _D, _P, _SZ, C.c_uint, C.c_uint, _SZ, _P, _P, _P,
                                          _P, _P, _P, _P], _I),
    "ouro_b200_refresh_sweep": ([_P, _P, _P, _P], _I),
    "ouro_b200_model_set_spikes": ([_P, _P], _I),
    "ouro_b200_quant_scan_spiked": ([_P, _SZ, _SZ, _SZ, _SZ, _I, _I, _P, _P, _P, _P, _P, _I, _SZ, C.c_uint, C.c_uint,
                                     _P, _P, _P, _P, _SZ, _SZ, _SZ], _I),
    "ouro_b200_gemm_bench": ([_P, _P, _P], _I),
    "ouro_b200_calib_save": ([_P, _P, C.c_char_p], _I),
    "ouro_b200_model_get_qweight": ([_P, C.c_char_p, C.c_uint, _P, C.c_size_t, C.POINTER(C.c_size_t)], _I),
    "ouro_b200_calib_load": ([_P, C.c_char_p, C.c_int, C.c_int, C.POINTER(_P)], _I),
    "ouro_b200_calib_spec": ([_P, C.POINTER(C.c_uint), C.POINTER(C.c_size_t), C.POINTER(_D), C.POINTER(C.c_int),
                              C.POINTER(C.c_int)], _I),
    "ouro_b200_trace_run": ([_P, _P, _I, _I, _I, _P, _SZ, _SZ, C.POINTER(_P)], _I),
    "ouro_b200_trace_get": ([_P, C.c_char_p, _P, _SZ, C.POINTER(_SZ)], _I),
    "ouro_b200_trace_free": ([_P], None),
}

EXPORTED = sorted(_SIGS)


class OuroError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[status {status}] {msg}")
        self.status = status


class ValidationError(OuroError):
    pass


class NumericError(OuroError):
    pass


class IoError(OuroError):
    pass


_lib = None


def load(path: str = SO_PATH):
    """Load libouro_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `make -C {HERE}` (no CPU fallback exists)")
    lib = C.CDLL(path)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


class Spikes(C.Structure):
    """ouro_b200_spikes (SpikeSettings, quant.hpp:105-110)."""
    _fields_ = [("rate", C.c_double), ("gain", C.c_double), ("channels", C.c_size_t), ("salt", C.c_uint64),
                ("sample0", C.c_size_t)]


class StageConfig(C.Structure):
    """ouro_b200_stage_config: the RunConfig settings a pipeline stage reads (config.hpp:17-47)."""
    _fields_ = [("image", C.c_size_t), ("channels", C.c_size_t), ("patch", C.c_size_t), ("embed", C.c_size_t),
                ("state", C.c_size_t), ("blocks", C.c_size_t), ("classes", C.c_size_t), ("conv_width", C.c_size_t),
                ("seed", C.c_uint64), ("weight_bits", C.c_uint), ("act_bits", C.c_uint), ("outlier_bits", C.c_uint),
                ("n_refresh", C.c_size_t), ("outlier_quantile", C.c_double), ("mode", C.c_char_p),
                ("eval_batch", C.c_size_t), ("spike_rate", C.c_double), ("spike_gain", C.c_double),
                ("spike_channels", C.c_size_t), ("d1", C.c_int), ("d2", C.c_int), ("run_id", C.c_char_p),
                ("device", C.c_int)]


class SweepSettings(C.Structure):
    """ouro_b200_sweep_settings (SweepSettings, gemm.hpp:122-131)."""
    _fields_ = [("periods", C.POINTER(C.c_size_t)), ("n_periods", C.c_size_t), ("steps", C.c_size_t),
                ("m", C.c_size_t), ("k", C.c_size_t), ("c", C.c_size_t), ("persistent_channels", C.c_size_t),
                ("transient_rate", C.c_double), ("spike_gain", C.c_double), ("trials", C.c_size_t),
                ("seed", C.c_uint64)]


class SweepRecord(C.Structure):
    _fields_ = [("period", C.c_size_t), ("median_total_ns", C.c_double), ("mean_o_list", C.c_double),
                ("scans_per_step", C.c_double)]


class BenchSettings(C.Structure):
    """ouro_b200_bench_settings (BenchSettings, gemm.hpp:103-110)."""
    _fields_ = [("sizes", C.POINTER(C.c_size_t)), ("n_sizes", C.c_size_t), ("outlier_fraction", C.c_double),
                ("trials", C.c_size_t), ("seed", C.c_uint64), ("f16_output", C.c_int)]


class BenchRecord(C.Structure):
    _fields_ = [("path", C.c_int), ("size", C.c_size_t), ("median_ns", C.c_double)]


def check(status: int) -> None:
    if status == OK:
        return
    msg = _lib.ouro_b200_last_error().decode()
    if status == ERR_VALIDATION:
        raise ValidationError(status, msg)
    if status == ERR_NUMERIC:
        raise NumericError(status, msg)
    if status == ERR_IO:
        raise IoError(status, msg)
    raise OuroError(status, msg)
