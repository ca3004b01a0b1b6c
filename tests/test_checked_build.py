"""Bounds-checked build (-m gpu): every kernel of libsks run through the device-side bounds checks of
libsks_checked.so (kernels.h SKS_CHECK: grid cells, polynomial tables, mailbox slots, sort ranks, the fused kernels'
range bound, the planner's footprints).  This pool does not run compute-sanitizer (its runs left GPUs needing a
reset), so these checks stand in for memcheck; tools/sanitize.py is the workload (cfg1-sized cases of every path,
the FP16x2 rerun, many owners, sks_sum_1d, async + graph calls, the fused large-N kernels)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_every_kernel_under_bounds_checks():
    from paper_2401_08260_b200 import build
    lib = build.build(checked=True)
    build.build()
    env = dict(os.environ, SKS_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize.py")], env=env, capture_output=True,
                       text=True, timeout=900)
    out = r.stdout + r.stderr
    assert "SKS_CHECK failed" not in out, out[-3000:]
    assert r.returncode == 0 and "sanitize run OK" in r.stdout, out[-3000:]
