"""The double integrator's exact-safe rejection bound (di_cost_exceeds in
csrc/di.cuh, the graph builders' prefilter) never rejects a pair whose exact
minimum cost (di_cost_tau) is within the radius: host build of the same
header, random pairs at five radii (tests/cpp/test_di_reject.cpp)."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_di_reject_bound_is_exact_safe(tmp_path):
    exe = str(tmp_path / "test_di_reject")
    subprocess.run(["g++", "-std=c++17", "-O2", "-ffp-contract=off",
                    "-I" + os.path.join(ROOT, "paper_1705_02403_b200", "csrc"), "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_di_reject.cpp"), "-o", exe], check=True)
    r = subprocess.run([exe, "100000"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "VIOLATION" not in r.stdout
