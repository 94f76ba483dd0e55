"""bench.py's N > 1 path, run end to end as the driver launches it (torchrun, 2 ranks) on the one
GPU a gpurun box has: collectives over gloo on host copies and both ranks on cuda:0 -- a
functional check of the sharding, the trace-digest check, the argmin exchange, the max-over-ranks
timing and rank 0's JSON line, not a measurement (the NCCL exchange itself is covered by
tests/test_gpu_dist.py on a one-rank group)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_two_ranks_functional():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "1", "--config", "C1", "--dist-backend", "gloo",
           "--same-device", "--no-extras", "--c2-steps", "0", "--c1-reps", "0", "--cpu-seconds", "0.5",
           "--alone-steps", "1", "--ce-steps", "1", "--e2e-steps", "1", "--no-clocks"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 2 and d["value"] > 0
    assert d["config"]["candidates_per_rank"] == d["config"]["candidates"] // 2
    assert "gloo" in d["config"]["parallelism"] and "functional" in d["config"]["parallelism"]
    assert d["config"]["policy"]["executed_items"] == d["config"]["policy"]["items"]
    assert d["eval_strong"]["candidates_per_rank"] == d["eval_strong"]["candidates_total"] // 2
    _check_contract(d)


def _check_contract(d):
    """the driver's JSON-line contract: every key it reads, with the right types"""
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert isinstance(d["config"]["workload"], str) and d["higher_is_better"] is True and d["scaling"] == "weak"
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"], k
    assert abs(d["roofline"]["frac"] - d["roofline"]["achieved"] / d["roofline"]["peak"]) < 1e-9
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in d["cpu_baseline"], k
    assert d["cpu_baseline"]["kind"] == "oracle"
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"], k
    assert d["gpu_launches"] > 0
