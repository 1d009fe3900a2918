"""GPU: the C++ facade (include/voxmap_b200/voxmap.hpp) — reference API shape,
bit-for-bit against the C oracle (tests/cpp/facade_test.cpp)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_facade_parity():
    subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "cpp")], check=True,
                   stdout=subprocess.DEVNULL)
    r = subprocess.run([os.path.join(ROOT, "tests", "cpp", "_bin", "facade_test")],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
