"""The memcheck stand-in (compute-sanitizer is closed on the
GPU pool): every kernel family run from the bounds-checked build of the
library (libdedisp_b200_checked.so, -DDDB_CHECKED), which counts on the
device every shared-memory window read, bulk copy or output store outside
its bounds.  Small instances, fault-injected tables for the slow paths,
guard rows around the output, and bit-exact results."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_checked_build_reports_no_violations():
    from paper_1601_05052_b200 import api
    if api.device_count() == 0:
        pytest.skip("no CUDA device")
    lib = os.path.join(ROOT, "paper_1601_05052_b200", "libdedisp_b200_checked.so")
    assert os.path.exists(lib), "build(checked=True) first (__graft_entry__.build does)"
    env = dict(os.environ, DDB_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "bounds-checked build: True" in r.stdout
    assert "bounds violations: 0" in r.stdout and "MISMATCH" not in r.stdout
