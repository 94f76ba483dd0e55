"""Algo. 3 in a real training loop (NEXT-4 through the NEXT-2 runtime): under a per-process
memory cap below the model's no-swap peak, plain training runs out of memory; with the runtime
(WarmUp stage, no policy yet) every OOM inside an op is handled by passive swaps of autograd-saved
activations (chm_passive_swap restricted to them), restored by chm_passive_restore when backward
unpacks them -- and training is bit-identical to the uncapped run.  Runs in a child process
(tests/_oom_child.py) so the cap does not leak into other tests."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("frac", [0.6])
def test_runtime_survives_a_memory_cap_with_passive_swaps(frac):
    child = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_oom_child.py")
    r = subprocess.run([sys.executable, child, str(frac)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["plain_under_cap"] == "oom", out
    assert out["losses_equal"] and out["params_equal"], out
    st = out["stats"]
    assert st["oom"] > 0 and st["passive"] > 0 and st["passive_restored"] == st["passive"], st


def test_runtime_policy_under_a_tighter_cap_releases_early():
    """a policy planned for 80% of the activation peak, run under a 50% cap: OOMs inside ops go
    through chm_oom_release first (marked blocks released early), then passive swaps; still
    bit-identical training"""
    child = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_oom_child.py")
    r = subprocess.run([sys.executable, child, "0.5", "0.8"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["losses_equal"] and out["params_equal"], out
    st = out["stats"]
    assert out["plans"] and out["plans"][0]["items"] > 0 and st["release"] > 0, out
    assert st["oom"] > 0 and st["oom_released"] + st["passive"] > 0, st


@pytest.mark.parametrize("frac", [0.6, 0.7])
def test_native_hook_with_defrag_survives_a_memory_cap(frac):
    """Algo. 3 with the C++ hook needs step (iii): Runtime(defrag=True) switches the caching
    allocator to expandable segments, and the passive swaps' freed pages then serve the failed
    requests -- bit-identical training under the cap"""
    child = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_oom_child.py")
    env = dict(os.environ, CHM_OOM_HOOK="native", CHM_OOM_DEFRAG="1")
    env.pop("PYTORCH_CUDA_ALLOC_CONF", None)
    r = subprocess.run([sys.executable, child, str(frac)], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["plain_under_cap"] == "oom", out
    assert out["losses_equal"] and out["params_equal"], out
    st = out["stats"]
    assert st["oom"] > 0 and st["passive"] > 0 and st["passive_restored"] == st["passive"], st

