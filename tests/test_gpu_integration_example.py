"""INTEGRATION.md's Python example (scripts/integration_example.py) runs as documented."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_integration_example_runs():
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "integration_example.py")], capture_output=True,
                       text=True, env=env, timeout=600)
    assert r.returncode == 0 and "example ok" in r.stdout, r.stdout + r.stderr
