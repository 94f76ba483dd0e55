"""Test-side construction of small hand-written traces (input data only)."""
import json
import os

import numpy as np

from workloads.traces import Trace

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def _csr(lists):
    ptr = np.zeros(len(lists) + 1, np.int32)
    ptr[1:] = np.cumsum([len(x) for x in lists])
    idx = np.array([x for lst in lists for x in lst], np.int32)
    return ptr, idx


def make_trace(phase, sizes, ins, outs, frees, static_bytes, t_iter, bw, budget, groups_fwd,
               groups_bwd, omega=1.0, name="hand", static=()):
    """sizes: list of tensor sizes (tensor index = position); ins/outs/frees: per-op lists of
    tensor indices.  Tensors listed in `static` are live at start (bytes inside static_bytes)."""
    n = len(phase)
    assert len(ins) == len(outs) == len(frees) == n
    T = len(sizes)
    produced = [t for lst in outs for t in lst]
    ptrs = np.zeros(T, np.uint64)
    for t in range(T):
        ptrs[t] = 0x7F0000000000 + 0x100000 * t
    return Trace(name=name, op_names=[f"op{i}" for i in range(n)],
                 phase=np.array(phase, np.uint8),
                 in_ptr=_csr(ins)[0], in_idx=_csr(ins)[1], out_ptr=_csr(outs)[0], out_idx=_csr(outs)[1],
                 free_ptr=_csr(frees)[0], free_idx=_csr(frees)[1],
                 nbytes=np.array(sizes, np.int64), dtype=np.zeros(T, np.uint8), ptr=ptrs,
                 n_produced=len(produced), static_bytes=static_bytes, t_iter=t_iter, bw=bw,
                 budget=budget, groups_fwd=groups_fwd, groups_bwd=groups_bwd, omega=omega)


def w1_trace(bw, scale=1):
    g = load_golden("w1.json")["trace"]
    names = list(g["tensors"].keys())
    ix = {nm: i for i, nm in enumerate(names)}
    conv = lambda L: [[ix[x] for x in op] for op in L]  # noqa: E731
    return make_trace(g["phase"], [g["tensors"][nm] * scale for nm in names], conv(g["ins"]),
                      conv(g["outs"]), conv(g["frees"]), g["static_bytes"] * scale, g["t_iter"],
                      bw * scale, g["budget"] * scale, g["groups_fwd"], g["groups_bwd"], name="W1"), ix
