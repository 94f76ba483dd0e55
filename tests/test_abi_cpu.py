"""CPU-side checks of the product library: it loads, exports every symbol include/chm.h declares,
and host-only calls behave (no compute without a GPU)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2509_11076_b200 import chm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "chm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(chm_[a-z_0-9]+)\s*\(", src)))


def test_library_builds_and_loads():
    from paper_2509_11076_b200 import build
    path = build.build()
    assert os.path.exists(path)
    chm.load()


def test_exports_every_declared_symbol():
    declared = _declared()
    assert len(declared) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", chm.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (chm_\w+)", out))
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    assert set(declared) == set(chm.EXPORTS)


def test_sm100a_cubin_embedded():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", chm.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_host_only_calls():
    L = chm.load()
    assert b"sm_100a" in L.chm_build_info()
    cfg = chm.Config()
    L.chm_config_default(ctypes.byref(cfg))
    assert (cfg.m, cfg.n, cfg.len_tol, cfg.cos_tol) == (2, 5, 0.05, 0.95)
    keys = np.zeros(3, chm.BEST_DTYPE)
    keys[0] = (5, 0.0, 1, 0, 0)
    keys[1] = (0, 2.0, 9, 1, 0)
    keys[2] = (0, 1.0, 9, 2, 0)
    assert chm.best_reduce(keys).index == 2
    keys[1] = (0, 1.0, 9, 1, 0)
    assert chm.best_reduce(keys).index == 1  # tie on (excess, stall, swapped) -> lowest index
    with pytest.raises(chm.ChmError):
        chm.best_reduce(np.zeros(0, chm.BEST_DTYPE))


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(chm.ChmError):
        chm.Context(device=0)


def test_arena_config_validation():
    """chm_config.arena_mode / arena_numa are validated before any device work (host-only ctx);
    the defaults are AUTO and the GPU's own node (-1)"""
    L = chm.load()
    cfg = chm.Config()
    L.chm_config_default(ctypes.byref(cfg))
    assert (cfg.arena_mode, cfg.arena_numa, cfg.arena_threads) == (chm.ARENA_AUTO, -1, 0)
    for mode, numa in ((3, -1), (chm.ARENA_REGISTER, -3)):
        cfg.device, cfg.arena_mode, cfg.arena_numa = -1, mode, numa
        h = ctypes.c_void_p()
        assert L.chm_create(ctypes.byref(cfg), ctypes.byref(h)) == -1  # CHM_E_INVAL
        assert b"arena" in L.chm_last_error()
    ctx = chm.Context(device=-1)
    assert ctx.arena_placement() == {"numa_node": -1, "mode": -1, "pin_s": 0.0}
    ctx.release_scratch()  # a host-only ctx holds no device scratch: a no-op
    assert chm.load().chm_release_scratch(None) == -1  # CHM_E_INVAL


def test_descend_argument_and_state_errors():
    """chm_descend checks its arguments and refuses a host-only ctx / trace (CHM_E_STATE) before
    it touches any pointer: no CPU fallback"""
    from workloads import traces as W
    tr = W.tiny()
    ctx = chm.Context(device=-1)
    ctx.set_detailed(True)
    chm.record_iteration(ctx, tr)
    ctx.detect_seq_change(tr.t_iter)
    pt = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
    L = chm.load()
    dummy = ctypes.c_void_p(16)
    assert L.chm_descend(ctx.h, pt.h, dummy, 1, 10, dummy, dummy, None, None, None) == -3  # CHM_E_STATE
    assert b"host-only" in L.chm_last_error()
    assert L.chm_descend(ctx.h, pt.h, None, 1, 10, dummy, dummy, None, None, None) == -1  # CHM_E_INVAL
    assert L.chm_descend(ctx.h, pt.h, dummy, 0, 10, dummy, dummy, None, None, None) == -1  # no starts
    assert L.chm_descend(None, pt.h, dummy, 1, 10, dummy, dummy, None, None, None) == -1
    with pytest.raises(chm.ChmError):
        ctx.descend(pt, 16, 1, ends=16, keys=16)
