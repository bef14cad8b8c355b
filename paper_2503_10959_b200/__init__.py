"""B200-native OuroMamba-Quant quantized Vim inference path.

Python front end over the C ABI of ``include/ouro_b200.h``. Device memory is
managed with torch CUDA tensors (plumbing only); every computation runs in the
sm_100a kernels of ``libouro_b200.so``. Names mirror the reference's C++
operator API (``/root/reference/proj/src/ouro/{quant,gemm,ssm}.hpp``).
"""
from ._lib import (MODE_DYNAMIC, MODE_FP, MODE_STATIC, POST_BIAS, POST_INPROJ, POST_RESID, POST_STORE, SRC_MERGE,
                   SRC_PLAIN, SRC_RMSNORM, IoError, NumericError, OuroError, ValidationError, load)
from .runtime import (DTYPE_F64, DTYPE_I8, DTYPE_U4, Calibration, Context, Dims, Model, QuantSpec, SpikeSettings,
                      StageConfig, TensorCal, Trace, calib_stage, quant_eval_stage, tensor_info, tensor_load, tensor_save)

__all__ = ["Context", "Model", "Calibration", "TensorCal", "QuantSpec", "SpikeSettings", "Dims", "Trace", "load", "OuroError",
           "ValidationError", "NumericError", "IoError", "MODE_FP", "MODE_DYNAMIC", "MODE_STATIC", "POST_STORE", "POST_INPROJ",
           "POST_RESID", "POST_BIAS", "SRC_PLAIN", "SRC_RMSNORM", "SRC_MERGE", "StageConfig", "quant_eval_stage", "calib_stage",
           "tensor_save", "tensor_load", "tensor_info", "DTYPE_F64", "DTYPE_I8", "DTYPE_U4"]
