"""The device restatement of the reference's libm (csrc/libm_port.cuh:
glibc 2.39's sin / cos / atan2 / acos / hypot, generated from the library's
machine code by tools/libm_port.py) pinned bit for bit against the libm
itself: the header is what the tool generates from this image's libm, and
its host build (tests/cpp/libm_port_check.cpp, the same source the device
compiles) returns the libm's exact bits on millions of random inputs --
angles, differences of angles, small and huge magnitudes, raw bit patterns,
arguments near multiples of pi/4 and near +-1 for acos.  CPU only."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_1705_02403_b200", "csrc")
HEADER = os.path.join(CSRC, "libm_port.cuh")


def test_header_is_generated_from_this_libm():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "libm_port.py")], capture_output=True,
                         text=True, check=True).stdout
    with open(HEADER) as f:
        assert f.read() == out


@pytest.fixture(scope="module")
def checker(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("lm") / "libm_port_check")
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-pthread", "-I" + CSRC,
                    os.path.join(ROOT, "tests", "cpp", "libm_port_check.cpp"), "-o", exe], check=True)
    return exe


@pytest.mark.parametrize("fn", ["sin", "cos", "atan2", "acos", "hypot"])
def test_bitwise_against_libm(checker, fn):
    r = subprocess.run([checker, fn, "4000000", "20171005"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout
    assert "mismatches 0" in r.stdout
