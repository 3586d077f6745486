"""Bounds-checked runs of the GPU parity suites (compute-sanitizer is closed
on this GPU pool; the pool's operators point to bounds checks and asserts of
our own instead).

`make debug` builds lib/debug/libspttn_b200.so with SPTTN_DEBUG_BOUNDS: every
factor row the packed / piece kernels gather, every staged-window leaf index,
every window's leaf count against its staging buffer and every owner-written
output row is checked on the device; a violation prints the site and traps.
This test runs the golden / fuzz / full-size parity suites against that
library in a child process (a trap poisons the CUDA context) and requires
them to pass with no check firing."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def _run(args):
    env = dict(os.environ, SPTTN_DEBUG_BOUNDS="1")
    return subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                           "-m", "gpu", *args], cwd=ROOT, env=env, capture_output=True,
                          text=True, timeout=1800)


def test_debug_library_is_the_checked_build():
    code = ("import os, paper_2307_05740_b200._native as N; "
            "print(N.engine()._name)")
    env = dict(os.environ, SPTTN_DEBUG_BOUNDS="1")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    assert "/debug/libspttn_b200.so" in out.stdout


def test_parity_suites_under_device_bounds_checks():
    r = _run(["tests/test_gpu_parity.py", "tests/test_gpu_fuzz.py",
              "tests/test_gpu_fullsize.py", "-k", "not item_clock"])
    tail = (r.stdout + r.stderr)[-3000:]
    assert "SPTTN_DCHECK failed" not in r.stdout + r.stderr, tail
    assert r.returncode == 0, tail


def test_device_checks_fire_on_a_bad_coordinate():
    """The checked build really checks: a leaf coordinate planted out of
    range after planning (SPTTN_DEBUG_POISON=1, checked build only) must trap
    the TTMc-3 kernel with the check's message."""
    code = ("import sys; sys.path.insert(0, 'tests'); import numpy as np; "
            "import paper_2307_05740_b200 as P; "
            "from paper_2307_05740_b200.configs import make_workload; "
            "w = make_workload('ttmc3', scale=1e-3); "
            "plan = P.Plan(w.cfg.kind, P.DeviceCsf(w.csf), w.factors, ranks=w.cfg.ranks); "
            "plan.execute(); plan.read_output()")
    env = dict(os.environ, SPTTN_DEBUG_BOUNDS="1", SPTTN_DEBUG_POISON="1")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode != 0
    assert "SPTTN_DCHECK failed" in out.stdout + out.stderr, (out.stdout + out.stderr)[-2000:]
