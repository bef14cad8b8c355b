"""The C++ host API (include/ouro_b200.hpp) against the reference's own
operators: hybrid_gemm / gemm_i4 / gemm_i4xi8 / pack_int4 / round_f16 bit-exact,
calibrate and quantized_forward (logits, argmax agreement, logits and
teacher-forced layer MSE) within tolerance. The test binary links the reference
sources compiled in place (make -C oracle cpp-api-test)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "test_b200_api")


def test_cpp_api_matches_reference(gpu_ctx):
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/test_b200_api not built (needs the reference sources)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
