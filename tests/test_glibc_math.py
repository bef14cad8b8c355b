"""The device exp/log1p (csrc/glibc_math.cuh) restate glibc's algorithms so the
kernels' softplus, SiLU and a_bar = exp(delta*A) equal the reference's bit for bit
(tensor.hpp:146-154, ssm.cpp:157). CPU side: the same source compiled for the host
against the live libm, and the exp table against its generator."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2503_10959_b200", "csrc")


@pytest.fixture(scope="module")
def checker(tmp_path_factory):
    out = tmp_path_factory.mktemp("glibc") / "glibc_math_check"
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-mfma", f"-I{CSRC}",
                    os.path.join(ROOT, "tests", "cpp", "glibc_math_check.cpp"), "-o", str(out), "-lm"], check=True)
    return str(out)


def test_exp_log1p_match_libm(checker):
    res = subprocess.run([checker, "300000"], check=True, capture_output=True, text=True).stdout.split("\n")
    rows = [r.split() for r in res if r.strip()]
    assert len(rows) == 15
    bad = {name: int(m) for name, m, _ in rows if int(m) != 0}
    assert not bad, f"device exp/log1p differ from libm: {bad}"


def test_exp_table_regenerates(tmp_path):
    out = tmp_path / "t.inc"
    subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "gen_exp_table.py"), str(out)], check=True,
                   capture_output=True)
    with open(os.path.join(CSRC, "glibc_exp_table.inc")) as f:
        assert out.read_text() == f.read()
