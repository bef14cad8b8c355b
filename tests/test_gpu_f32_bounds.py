"""The fast scan certifies f32 codes with a relative error bound on its f32
softplus (csrc/scan_f32.cuh). This checks that bound exhaustively: every finite
f32 argument >= -80 against the exact f64 softplus (tests/cpp/softplus_bound_check.cu)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2503_10959_b200", "csrc")


def test_softplus_f32_bound_exhaustive(tmp_path):
    exe = tmp_path / "softplus_bound_check"
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", f"-I{CSRC}",
                    os.path.join(ROOT, "tests", "cpp", "softplus_bound_check.cu"), "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


def test_merge_f32_bound_exhaustive(tmp_path):
    """The merge source's certified v = m * silu(g) (csrc/merge_f32.cuh): every f32
    gate g >= -80 (tests/cpp/merge_bound_check.cu)."""
    exe = tmp_path / "merge_bound_check"
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", f"-I{CSRC}",
                    os.path.join(ROOT, "tests", "cpp", "merge_bound_check.cu"), "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
