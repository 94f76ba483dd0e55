"""NEXT-3: custom recordStream (event pair at the simulator's completion op) vs PyTorch's
recordStream with real allocations and stand-in compute: the custom release keeps the
reserved peak at the policy's footprint; recordStream reclaims late and reserves more."""
import subprocess
import sys
import json
import os

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_custom_release_keeps_reserved_at_policy_peak():
    out = subprocess.run([sys.executable, "tools/recordstream_ab.py", "--op-us", "300", "--policy-candidates", "500"],
                         cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    policy_peak = d["config"]["policy_peak_bytes"]
    assert policy_peak < d["config"]["no_swap_peak_bytes"]
    assert d["custom"]["peak_reserved"] <= 1.25 * policy_peak + (64 << 20)
    assert d["naive"]["peak_reserved"] > d["custom"]["peak_reserved"]
    assert d["custom"]["exec_stats"]["bytes_out"] == d["custom"]["exec_stats"]["bytes_in"]
