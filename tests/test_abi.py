"""CPU tests of the drop-in boundary (no GPU needed): the C-ABI library
builds for sm_100a, loads, exports exactly what include/gmt_b200.h declares,
the ctypes signature table covers every entry point, and compute calls fail
loudly (never fall back) without a device."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_1705_02403_b200 import native
from paper_1705_02403_b200.errors import NoDeviceError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gmt_b200.h")


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gmt_[a-z_0-9]+)\s*\(", text)))


def exported():
    out = subprocess.run(["nm", "-D", "--defined-only", native.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    return sorted({ln.split()[-1] for ln in out.splitlines() if " T gmt_" in ln})


def test_library_exports_every_declared_symbol():
    assert os.path.exists(native.LIB_PATH), "run python -m paper_1705_02403_b200.build"
    d, e = declared(), exported()
    assert d, "no declarations parsed"
    missing = sorted(set(d) - set(e))
    assert not missing, f"declared but not exported: {missing}"
    extra = sorted(set(e) - set(d))
    assert not extra, f"exported but not declared: {extra}"


def test_ctypes_table_matches_header():
    assert sorted(n for n, _, _ in native.SIGNATURES) == declared()
    lib = native.load()
    for name, _, _ in native.SIGNATURES:
        assert isinstance(getattr(lib, name), C._CFuncPtr)


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_abi_version_and_scalars():
    lib = native.lib()
    assert lib.gmt_abi_version() == 2
    assert native.Context.connection_radius(2, 1000) == pytest.approx(0.13263, rel=1e-4)


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="a GPU is present")
def test_no_device_fails_loudly():
    with pytest.raises(NoDeviceError):
        native.Context(0)


def test_missing_library_raises(monkeypatch, tmp_path):
    monkeypatch.setattr(native, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(ImportError):
        native.load()


ABI_STRUCTS = ("Scene", "SampleSource", "GraphView", "PlanOut", "PlanSummary", "Problem",
               "DiParams", "BatchHost", "QuadParams", "Scenario", "TrialOutcome", "DubinsParams")


def _sizes(fn):
    out = (C.c_int64 * 16)()
    n = fn(out, 16)
    return list(out)[:n]


def test_struct_layouts_match_bindings():
    """ctypes mirrors of the ABI structs have the C sizes (product library
    and the compiled-reference wrapper, which must be rebuilt when the header
    changes)."""
    from paper_1705_02403_b200 import abi
    want = [C.sizeof(getattr(abi, s)) for s in ABI_STRUCTS]
    assert _sizes(native.lib().gmt_struct_sizes) == want
    import oracle
    if oracle.ref_available():
        f = oracle.ref().lib.ref_struct_sizes
        f.restype, f.argtypes = C.c_int, [C.POINTER(C.c_int64), C.c_int32]
        assert _sizes(f) == want


def test_reference_batch_api():
    """The bench's reference leg: build_instance for many queries and the
    parallel plan loop agree with one-at-a-time planning."""
    import oracle
    if not oracle.ref_available():
        pytest.skip("no compiled reference")
    from paper_1705_02403_b200 import problem as P
    R = oracle.ref()
    specs = [P.random_forest_query(5, q, n=600) for q in range(5)]
    insts = R.instance_build_many(specs, 3)
    sums, sec = R.plan_many(insts, 1.0, 3)
    assert sec > 0
    for s, inst in zip(sums, insts):
        r = inst.plan(1.0)
        assert (s.status, s.cost, s.iterations, s.total_collision_checks) == (
            r.status, r.cost, r.iterations, r.total_collision_checks)
