"""GPU suite: the C++ drop-in under the reference's own API.

* build/tests/test_executor_b200 — the reference executor test cases
  (proj/tests/test_executor.cpp) restated against the device executor, plus
  device-routing checks;
* build/tests/ref_pin — every device route (dedicated kernels, forest
  interpreter, NVRTC-compiled forests, device execute_unfactorized) against
  the reference executor itself (spttn_ref::, compiled from /root/reference
  and linked into the same binary): every admissible order of the
  acceptance fixtures (TTTc-4 sampled in --quick), sampled TTTc-6 orders,
  BASELINE-rank fixtures; bit-identical where the route claims it;
* build/tests/acceptance_b200 — the reference's acceptance harness
  (proj/tests/acceptance.cpp, compiled from /root/reference) linked against
  the device executor instead of proj/src/executor.cpp.
"""
import os
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "build" / "tests"


def run(name, timeout, *args):
    exe = BIN / name
    assert exe.exists(), f"{exe} not built (built from /root/reference headers by build())"
    return subprocess.run([str(exe), *args], capture_output=True, text=True, timeout=timeout)


def test_reference_executor_cases_on_device():
    r = run("test_executor_b200", 600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "0 failures" in r.stdout


def test_every_device_route_pinned_to_the_reference_executor():
    r = run("ref_pin", 1500, "--quick")
    print(r.stdout)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "REF PIN OK" in r.stdout
    assert "failures 0" in r.stdout


@pytest.mark.skipif(not os.environ.get("SPTTN_RUN_ACCEPTANCE"),
                    reason="criterion 6 walks >1e6 admissible orders (TTTc-4) through the "
                           "one-thread device interpreter: ~1 h; opt in with SPTTN_RUN_ACCEPTANCE=1")
def test_reference_acceptance_suite_on_device():
    r = run("acceptance_b200", 7200)
    print(r.stdout)
    lines = [l for l in r.stdout.splitlines() if l.startswith(("PASS", "FAIL"))]
    assert len(lines) == 10, r.stdout
    # executor criteria: 3 (order-4 plan/hooks), 6 (every order vs oracle),
    # 7 (op counters), 10 (round trips + determinism)
    for crit in (3, 6, 7, 10):
        line = [l for l in lines if f"criterion {crit}:" in l][0]
        assert line.startswith("PASS"), r.stdout
    assert r.returncode == 0, r.stdout
