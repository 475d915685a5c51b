"""GPU: the device-checks library (libhsb200_debug.so, -DHS_DEVICE_CHECKS).

compute-sanitizer is closed on this GPU pool (its runs left GPUs needing a
reset), so out-of-bounds accesses and protocol hangs of the dataflow kernels
are caught by the library's own instrumentation: bounds asserts on every
table / map / vector access and a watchdog on every cross-CTA spin-wait
(include/hsb200.h hs_debug_check).  Each workload of tools/device_checks.py
runs in a subprocess with HS_LIB=debug, checks its results against the
reference goldens / the single-RHS kernels, and must report no violation."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEBUG_LIB = os.path.join(ROOT, "paper_2209_10886_b200", "_lib", "libhsb200_debug.so")


@pytest.mark.parametrize("case", ["selftest", "fused", "steps", "zmma", "emu", "gmres", "peer"])
def test_device_checks(case):
    if not os.path.exists(DEBUG_LIB):
        pytest.fail("libhsb200_debug.so missing: python -m paper_2209_10886_b200._build --debug")
    env = dict(os.environ, HS_LIB="debug")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "device_checks.py"), case], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=900)
    recs = [json.loads(l) for l in p.stdout.splitlines() if l.startswith("{")]
    assert recs, p.stderr[-3000:]
    for r in recs:
        assert r["lib"] == "libhsb200_debug.so" and r["checks_enabled"] == 1, r
        assert r["violation"] == 0, r
        assert r["ok"], r
    assert p.returncode == 0, p.stderr[-3000:]
