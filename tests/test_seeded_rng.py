"""The library's SeededRng mirror (csrc/seeded_rng.h) draws what the reference's
rng.cpp draws: seeded weights and the gemm-bench operands depend on it. CPU test,
linked against the reference's own rng.cpp object (oracle/_ref)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SRC = "/root/reference/proj/src"
RNG_O = os.path.join(ROOT, "oracle", "_ref", "rng.o")


def test_seeded_rng_matches_reference(tmp_path):
    if not (os.path.isdir(REF_SRC) and os.path.exists(RNG_O)):
        pytest.skip("reference sources / oracle/_ref build not available")
    exe = tmp_path / "rng_check"
    subprocess.run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", f"-I{REF_SRC}",
                    f"-I{os.path.join(ROOT, 'paper_2503_10959_b200', 'csrc')}",
                    os.path.join(ROOT, "tests", "cpp", "rng_check.cpp"), RNG_O, "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0 and out.stdout.strip() == "ok", out.stdout
