"""Runs the C++ drop-in test (tests/cpp/test_shim.cpp) on the B200."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_shim():
    exe = os.path.join(ROOT, "build", "test_shim")
    if not os.path.exists(exe):
        import sys
        sys.path.insert(0, os.path.join(ROOT, "tests", "cpp"))
        import build_cpp_tests as b  # noqa: E402
        b.build()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
