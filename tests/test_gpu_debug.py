"""Every device entry point once more, on the bounds-checked debug build of
the library (CGPU_DEBUG: device traps on out-of-range queue, table, block or
shared-memory indices) -- the stand-in for compute-sanitizer memcheck, which
this GPU pool does not allow."""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DBG = os.path.join(ROOT, "paper_1601_00636_b200", "build_dbg", "libcuboid_gpu.so")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(DBG), reason="debug library not built")
def test_bounds_checked_build_runs_clean():
    env = dict(os.environ, CUBOID_GPU_LIB=DBG)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_case.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "sanitize case ok" in r.stdout
