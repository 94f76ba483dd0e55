"""The C ABI from plain C99 (tests/c/host_abi.c): the header compiles as C, the program links
against libchm.so and drives recording, Algo. 1, the trace build, the generator and the
executor on a host-only ctx -- no Python on the path."""
import os
import re
import subprocess

import pytest

from paper_2509_11076_b200 import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_plain_c_client(tmp_path):
    lib = build.build()
    exe = str(tmp_path / "host_abi")
    cuda_inc = "/usr/local/cuda/include"
    cmd = ["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"), "-I", cuda_inc,
           os.path.join(ROOT, "tests", "c", "host_abi.c"), "-o", exe, "-L", os.path.dirname(lib), "-lchm",
           "-Wl,-rpath," + os.path.dirname(lib)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0 and "cuda_runtime_api.h: No such file" in r.stderr:
        pytest.skip("CUDA headers not available")
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stdout + r.stderr
    out = r.stdout
    assert out.strip().endswith("ok")
    m = re.search(r"trace ops (\d+) swappable (\d+) layers (\d+)", out)
    assert m and int(m.group(1)) == 12 and int(m.group(2)) > 0 and int(m.group(3)) == 12  # 6 + 6 layers
    g = re.search(r"generator items (\d+)", out)
    e = re.search(r"executed items (\d+) matched (\d+) actions (\d+)", out)
    assert int(g.group(1)) > 0 and int(e.group(1)) == int(e.group(2)) == int(g.group(1)) and int(e.group(3)) > 0
    assert "null params -> -1" in out
    assert "descend on a host-only ctx -> -3" in out  # CHM_E_STATE
