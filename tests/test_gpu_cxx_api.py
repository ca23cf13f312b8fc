"""Runs the C++ API test program (tests/cxx/test_leaf_api.cpp) on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_cxx_api_program():
    exe = os.path.join(ROOT, "build", "test_leaf_api")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", ROOT, "cxx_test"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "cxx api ok" in r.stdout
