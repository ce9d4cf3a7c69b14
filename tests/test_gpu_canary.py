"""The debug build's canaries (RPD_CANARY=1; the stand-in for compute-sanitizer, closed on this
GPU pool -- profiles/r2/sanitizer_refused.log): a write past the end of a library buffer is
reported by rpd_debug_check.  The whole GPU suite runs with RPD_CANARY=1 in
tools/gpu_canary.sh (every public call followed by the check)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu


def test_canary_detects_an_overrun():
    env = dict(os.environ, RPD_CANARY="1")
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, os.path.join(here, "canary_probe.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "write past the end" in r.stdout
