"""Race evidence for the hand-written kernels.  The reference
relies on worker-count invariance (planner.hpp:57-66); compute-sanitizer is
not available on the GPU pool this suite runs on, so races are hunted the
way the reference hunts them, harder: tools/sanitize_probe.py runs the solve
kernel in every shape (one narrow / wide CTA, 2-, 8- and 16-CTA clusters
with DSMEM; Euclidean and double-integrator; the batched half-warp DI
checks), the batched r-disk grid builder and the shared-pool derivation,
each result compared bit for bit with the single-CTA baseline, and the whole
probe is repeated so that scheduling-dependent races surface as
nondeterminism."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_shapes_and_repeats_are_bitwise_identical():
    outs = []
    for _ in range(3):
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_probe.py"), "--repeats", "20"],
                           capture_output=True, text=True, timeout=1200)
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
        outs.append(r.stdout)
    assert outs[0] == outs[1] == outs[2]
