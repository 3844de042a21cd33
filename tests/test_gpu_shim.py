"""Runs the C++ drop-in shim test (tests/cpp/test_shim.cpp) on the GPU."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def test_cpp_shim_builds():
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp")], check=True)
    assert os.path.exists(os.path.join(HERE, "cpp", "test_shim"))


@pytest.mark.gpu
def test_cpp_shim_runs():
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp")], check=True)
    r = subprocess.run([os.path.join(HERE, "cpp", "test_shim")], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout
