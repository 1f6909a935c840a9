"""The C++ host API (include/parcop_b200.hpp, parcop:: names) end to end on
the GPU: tests/cpp/api_smoke links libparcop_b200.so like a reference caller."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_cpp_api_smoke():
    exe = os.path.join(HERE, "cpp", "api_smoke")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", os.path.join(HERE, "cpp")], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    lines = out.stdout.strip().splitlines()
    assert len(lines) == 8, out.stdout
    for line in lines:
        assert " ok" in line, out.stdout
