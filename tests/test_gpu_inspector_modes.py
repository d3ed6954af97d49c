"""The recurrence's alternative schedules on the same parity suite
(tests/test_gpu_inspector.py against the oracle), each in a fresh process
because the knobs are read once per process:
  * GX_INSPECT_CTAS=148: every trace on the multi-CTA grid (small traces
    otherwise take the one-CTA path), so the eviction pool, local pairing and
    small-b* local select run on tiny inputs;
  * + GX_INSPECT_NEVER=2: the NEVER-bucket fast path (maintained id-digit
    histogram + slot-block summary) at every cache size, not only >= 606K slots;
  * GX_INSPECT_CTAS=7: a grid that is neither one CTA nor one per SM;
  * GX_INSPECT_DEFER=0: the ordered (round-1 style) recurrence kept for A/B."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env", [
    {"GX_INSPECT_CTAS": "148"},
    {"GX_INSPECT_CTAS": "148", "GX_INSPECT_NEVER": "2"},
    {"GX_INSPECT_CTAS": "7", "GX_INSPECT_NEVER": "2"},
    {"GX_INSPECT_DEFER": "0"},
], ids=["grid148", "grid148-never", "grid7-never", "ordered"])
def test_inspector_suite_under_schedule(env):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_inspector.py")],
                       cwd=ROOT, env=e, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
