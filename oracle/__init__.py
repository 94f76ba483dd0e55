"""CPU ORACLE (test infrastructure only) -- ctypes wrapper over oracle/chm_oracle.c.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference`
leg may import this package.  It shares no code with `paper_2509_11076_b200` (the
product); the product never imports it.  See chm_oracle.h for the citations.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle.so")
_SRC = [os.path.join(_HERE, "chm_oracle.c")]

FWD, BWD, OPT = 0, 1, 2
WARMUP, GENPOLICY, STABLE = 0, 1, 2
EXHAUSTIVE, SEEDED, MASKS = 0, 1, 2


def build(force: bool = False) -> str:
    """gcc -O2 -ffp-contract=off: every FP expression evaluated as written."""
    newest = max(os.path.getmtime(p) for p in _SRC + [os.path.join(_HERE, "chm_oracle.h")])
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < newest:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-std=gnu99", "-O2", "-ffp-contract=off", "-fno-fast-math",
                               "-shared", "-fPIC", "-pthread", "-o", tmp] + _SRC + ["-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


class _Best(C.Structure):
    _fields_ = [("excess", C.c_int64), ("stall", C.c_double), ("swapped", C.c_int64),
                ("index", C.c_uint64), ("peak", C.c_int64)]

    def key(self):
        return (self.excess, self.stall, self.swapped, self.index)


class _Input(C.Structure):
    _fields_ = [("n_ops", C.c_int32), ("n_tensors", C.c_int32), ("phase", C.c_void_p),
                ("in_ptr", C.c_void_p), ("in_idx", C.c_void_p), ("out_ptr", C.c_void_p),
                ("out_idx", C.c_void_p), ("free_ptr", C.c_void_p), ("free_idx", C.c_void_p),
                ("nbytes", C.c_void_p), ("static_bytes", C.c_int64), ("t_iter", C.c_double),
                ("bw", C.c_double), ("omega", C.c_double), ("groups_fwd", C.c_int32),
                ("groups_bwd", C.c_int32)]


class _Stage(C.Structure):
    _fields_ = [("m", C.c_int32), ("n", C.c_int32), ("cos_mode", C.c_int32),
                ("initialized", C.c_int32), ("stable_step", C.c_int32), ("prev_stage", C.c_int32),
                ("len_tol", C.c_double), ("cos_tol", C.c_double), ("prev_len", C.c_int32),
                ("cap", C.c_int32), ("prev_seq", C.c_void_p)]


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        L.orc_build.argtypes = [C.POINTER(_Input), C.POINTER(C.c_void_p)]
        L.orc_error.restype = C.c_char_p
        L.orc_free.argtypes = [C.c_void_p]
        L.orc_dims.argtypes = [C.c_void_p] + [C.POINTER(C.c_int32)] * 4
        L.orc_tensor_table.argtypes = [C.c_void_p] + [C.c_void_p] * 4
        L.orc_layer_table.argtypes = [C.c_void_p] + [C.c_void_p] * 4
        L.orc_swappable.argtypes = [C.c_void_p] + [C.c_void_p] * 6
        L.orc_f0.argtypes = [C.c_void_p, C.c_void_p]
        L.orc_base_mask.argtypes = [C.c_void_p, C.c_void_p]
        L.orc_replay.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.orc_replay.restype = C.c_int64
        L.orc_stall.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_stall.restype = C.c_double
        for fn in (L.orc_stall_dir, L.orc_stall_timeline):
            fn.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]
            fn.restype = C.c_double
        L.orc_reconstruct.argtypes = [C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p]
        L.orc_eval.argtypes = [C.c_void_p, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                               C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                               C.c_void_p, C.POINTER(_Best)]
        L.orc_eval_model.argtypes = [C.c_void_p, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                     C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_void_p, C.POINTER(_Best)]
        L.orc_splitmix64.argtypes = [C.c_uint64]
        L.orc_splitmix64.restype = C.c_uint64
        L.orc_key_less.argtypes = [C.POINTER(_Best), C.POINTER(_Best)]
        L.orc_swap_execute.argtypes = [C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_generate.argtypes = [C.c_void_p, C.c_int64, C.c_double, C.c_double, C.c_int32] + [C.c_void_p] * 5
        L.orc_generate.restype = C.c_int32
        L.orc_eval_explicit.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_int64, C.c_uint64, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.POINTER(_Best)]
        L.orc_stage_init.argtypes = [C.POINTER(_Stage), C.c_int32, C.c_int32, C.c_double,
                                     C.c_double, C.c_int32]
        L.orc_stage_release.argtypes = [C.POINTER(_Stage)]
        L.orc_stage_step.argtypes = [C.POINTER(_Stage), C.c_void_p, C.c_int32,
                                     C.POINTER(C.c_double), C.POINTER(C.c_double),
                                     C.POINTER(C.c_int32)]
        L.orc_stage_step.restype = C.c_int32
        L.orc_compare.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int32,
                                  C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.orc_feature_tables.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]
        L.orc_features_after.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int32,
                                         C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                         C.c_void_p]
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p) if a is not None and a.size else None


def _arr(x, dt):
    return np.ascontiguousarray(np.asarray(x, dtype=dt))


class Model:
    """The oracle's derivation of one trace (tensor table, layers, solo timing, F0)."""

    def __init__(self, trace, t_iter: Optional[float] = None, bw: Optional[float] = None,
                 groups: Optional[Tuple[int, int]] = None, omega: Optional[float] = None,
                 static_bytes: Optional[int] = None):
        L = lib()
        tr = trace
        self.trace = tr
        self._keep = [_arr(tr.phase, np.uint8), _arr(tr.in_ptr, np.int32), _arr(tr.in_idx, np.int32),
                      _arr(tr.out_ptr, np.int32), _arr(tr.out_idx, np.int32),
                      _arr(tr.free_ptr, np.int32), _arr(tr.free_idx, np.int32),
                      _arr(tr.nbytes, np.int64)]
        k = self._keep
        gf, gb = groups if groups is not None else (tr.groups_fwd, tr.groups_bwd)
        self._in = _Input(tr.n_ops, tr.n_tensors, _p(k[0]), _p(k[1]), _p(k[2]), _p(k[3]), _p(k[4]),
                          _p(k[5]), _p(k[6]), _p(k[7]),
                          int(tr.static_bytes if static_bytes is None else static_bytes),
                          float(tr.t_iter if t_iter is None else t_iter),
                          float(tr.bw if bw is None else bw),
                          float(tr.omega if omega is None else omega), int(gf), int(gb))
        h = C.c_void_p()
        if L.orc_build(C.byref(self._in), C.byref(h)) != 0:
            raise ValueError(L.orc_error().decode())
        self._h = h
        n, T, K, Ly = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        L.orc_dims(h, C.byref(n), C.byref(T), C.byref(K), C.byref(Ly))
        self.N, self.T, self.K, self.L = n.value, T.value, K.value, Ly.value
        self.W = (self.K + 63) // 64

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_free(self._h)
            self._h = None

    def tensor_table(self):
        p, f, a, b = (np.zeros(self.T, np.int32) for _ in range(4))
        lib().orc_tensor_table(self._h, _p(p), _p(f), _p(a), _p(b))
        return p, f, a, b

    def layers(self):
        st, n, ty = (np.zeros(self.L, np.int32) for _ in range(3))
        bud = np.zeros(self.L, np.float64)
        lib().orc_layer_table(self._h, _p(st), _p(n), _p(ty), _p(bud))
        return st, n, ty, bud

    def swappable(self):
        out = [np.zeros(self.K, np.int32) for _ in range(6)]
        lib().orc_swappable(self._h, *[_p(x) for x in out])
        return dict(zip(["t", "r", "s", "lin", "lout", "saturated"], out))

    def f0(self):
        f = np.zeros(self.N, np.int64)
        lib().orc_f0(self._h, _p(f))
        return f

    def base_mask(self):
        w = np.zeros(max(self.W, 1), np.uint64)
        lib().orc_base_mask(self._h, _p(w))
        return w[:self.W]

    def replay(self, t: Sequence[int], r: Sequence[int], s: Sequence[int], footprint: bool = True):
        t, r, s = _arr(t, np.int32), _arr(r, np.int32), _arr(s, np.int32)
        F = np.zeros(self.N, np.int64) if footprint else None
        d2h, h2d = C.c_int64(), C.c_int64()
        pk = lib().orc_replay(self._h, len(t), _p(t), _p(r), _p(s), _p(F), C.byref(d2h), C.byref(h2d))
        return dict(peak=pk, footprint=F, d2h=d2h.value, h2d=h2d.value)

    def stall(self, t, r, s) -> float:
        t, r, s = _arr(t, np.int32), _arr(r, np.int32), _arr(s, np.int32)
        return lib().orc_stall(self._h, len(t), _p(t), _p(r), _p(s))

    def stall_dir(self, t, r, s) -> float:
        """Q11 variant: per-direction layer budgets"""
        t, r, s = _arr(t, np.int32), _arr(r, np.int32), _arr(s, np.int32)
        return lib().orc_stall_dir(self._h, len(t), _p(t), _p(r), _p(s))

    def stall_timeline(self, t, r, s) -> float:
        """Q11 variant: max-plus serial-stream timeline"""
        t, r, s = _arr(t, np.int32), _arr(r, np.int32), _arr(s, np.int32)
        return lib().orc_stall_timeline(self._h, len(t), _p(t), _p(r), _p(s))

    def mask_items(self, mask_bits: Sequence[int]):
        """items {t, r, s} of the swappable tensors selected by bit list"""
        sw = self.swappable()
        sel = np.array([k for k in range(self.K) if mask_bits[k]], np.int64)
        return sw["t"][sel], sw["r"][sel], sw["s"][sel]

    def eval(self, kind: int, first: int, count: int, *, seed: int = 0, flip_thr: int = 0,
             words: Optional[np.ndarray] = None, budget: Optional[int] = None, nthreads: int = 1,
             footprint: bool = False, stall_model: int = 0):
        """stall_model 0: R-stall (§8(c).5); 1: the Q11 timeline (stall_timeline of each candidate's
        items in mask-bit order) -- also the stall field of the argmin key"""
        peak = np.zeros(count, np.int64)
        stall = np.zeros(count, np.float64)
        swapped = np.zeros(count, np.int64)
        F = np.zeros((count, self.N), np.int64) if footprint else None
        w = _arr(words, np.uint64) if words is not None else None
        best = _Best()
        rc = lib().orc_eval_model(self._h, kind, first, count, seed, flip_thr, _p(w),
                                  int(self.trace.budget if budget is None else budget), nthreads, stall_model,
                                  _p(peak), _p(stall), _p(swapped), _p(F), C.byref(best))
        if rc != 0:
            raise ValueError(lib().orc_error().decode())
        return dict(peak=peak, stall=stall, swapped=swapped, footprint=F, best=best)


def generate(model: "Model", budget: int = None, C_coef: float = 1.0, rem_scale: float = 1.0):
    """Algo. 2: returns dict(t, r, s, fallback, saturated, feasible)."""
    cap = model.T + 1
    out = [np.zeros(cap, np.int32) for _ in range(5)]
    b = int(model.trace.budget if budget is None else budget)
    n = lib().orc_generate(model._h, b, float(C_coef), float(rem_scale), cap, *[_p(x) for x in out])
    feasible = n >= 0
    n = n if n >= 0 else -1 - n
    return dict(zip(["t", "r", "s", "fallback", "saturated"], [x[:n] for x in out]), feasible=feasible)


def eval_explicit(model: "Model", lists, budget: int = None, first_index: int = 0, footprint: bool = False):
    """lists: sequence of (t, r, s) arrays per candidate"""
    off = np.zeros(len(lists) + 1, np.int64)
    off[1:] = np.cumsum([len(x[0]) for x in lists])
    t = np.concatenate([np.asarray(x[0], np.int32) for x in lists] + [np.zeros(0, np.int32)])
    r = np.concatenate([np.asarray(x[1], np.int32) for x in lists] + [np.zeros(0, np.int32)])
    s = np.concatenate([np.asarray(x[2], np.int32) for x in lists] + [np.zeros(0, np.int32)])
    n = len(lists)
    peak, stall, sw = np.zeros(n, np.int64), np.zeros(n, np.float64), np.zeros(n, np.int64)
    F = np.zeros((n, model.N), np.int64) if footprint else None
    best = _Best()
    lib().orc_eval_explicit(model._h, n, _p(off), _p(t), _p(r), _p(s),
                            int(model.trace.budget if budget is None else budget), first_index,
                            _p(peak), _p(stall), _p(sw), _p(F), C.byref(best))
    return dict(peak=peak, stall=stall, swapped=sw, footprint=F, best=best)


def descend(model: "Model", words, max_rounds: int = 4096, budget: Optional[int] = None, nthreads: int = 16):
    """Steepest single-flip descent from a mask (reading R-search; the planner's
    search around the evaluator, "selects the one with the best runtime performance"),
    written out plainly: each round builds the K masks that differ from the current one in one
    bit, scores them all with the oracle's MASKS evaluation (R-stall, §8(c).5) and takes the
    argmin of (excess, stall, swapped, k) (§8(c).6); it moves there if that key's first three
    fields are lexicographically smaller than the current mask's, else it stops.  Returns
    (end words, end key (excess, stall, swapped), rounds)."""
    K = model.K
    W = (K + 63) // 64
    cur = np.array(words, np.uint64).reshape(W).copy()
    b = int(model.trace.budget if budget is None else budget)
    k0 = model.eval(MASKS, 0, 1, words=cur if W else np.zeros(1, np.uint64), budget=b)["best"]  # K = 0: no bits
    key = (int(k0.excess), float(k0.stall), int(k0.swapped))
    rounds = 0
    while rounds < max_rounds and K > 0:
        nb = np.repeat(cur[None, :], K, axis=0)
        for k in range(K):
            nb[k, k // 64] ^= np.uint64(1 << (k % 64))
        best = model.eval(MASKS, 0, K, words=nb.reshape(-1), budget=b, nthreads=nthreads)["best"]
        nk = (int(best.excess), float(best.stall), int(best.swapped))
        if not nk < key:
            break
        k = int(best.index)
        cur[k // 64] ^= np.uint64(1 << (k % 64))
        key = nk
        rounds += 1
    return cur, key, rounds


def splitmix64(z: int) -> int:
    return lib().orc_splitmix64(z)


def reconstruct(measured, size, r, s):
    measured = _arr(measured, np.int64)
    size, r, s = _arr(size, np.int64), _arr(r, np.int32), _arr(s, np.int32)
    out = np.zeros_like(measured)
    lib().orc_reconstruct(len(measured), _p(measured), len(size), _p(size), _p(r), _p(s), _p(out))
    return out


def compare(a, b, cos_mode: int = 0):
    a, b = _arr(a, np.int32), _arr(b, np.int32)
    ld, cs = C.c_double(), C.c_double()
    if lib().orc_compare(_p(a), len(a), _p(b), len(b), cos_mode, C.byref(ld), C.byref(cs)) != 0:
        raise ValueError(lib().orc_error().decode())
    return ld.value, cs.value


class StageMachine:
    """Algo. 1."""

    def __init__(self, m: int = 2, n: int = 5, len_tol: float = 0.05, cos_tol: float = 0.95,
                 cos_mode: int = 0):
        self._st = _Stage()
        lib().orc_stage_init(C.byref(self._st), m, n, len_tol, cos_tol, cos_mode)

    def step(self, seq):
        seq = _arr(seq, np.int32)
        ld, cs, stable = C.c_double(), C.c_double(), C.c_int32()
        stage = lib().orc_stage_step(C.byref(self._st), _p(seq), len(seq), C.byref(ld), C.byref(cs),
                                     C.byref(stable))
        return dict(stage=stage, len_diff=ld.value, cos=cs.value, stable=bool(stable.value),
                    stable_step=self._st.stable_step)

    def __del__(self):
        if _lib is not None:
            _lib.orc_stage_release(C.byref(self._st))


def tokenize(names: Sequence[str]):
    """an integer per operator name, 1, 2, ... in order of first appearance."""
    table = {}
    return np.array([table.setdefault(nm, len(table) + 1) for nm in names], np.int32), table


def feature_tables(tokens):
    tokens = _arr(tokens, np.int32)
    V = int(tokens.max()) if tokens.size else 0
    idx = np.zeros(V + 1, np.uint8)
    oh = np.zeros(V + 1, np.uint32)
    lib().orc_feature_tables(_p(tokens), len(tokens), V, _p(idx), _p(oh))
    return idx, oh


def features_after(trace, tokens, op_index, op_onehot, after: int):
    """App. A features of every tensor right after op `after`; a tensor used several times
    by one op is updated once for that op."""
    uses = [sorted(set(trace.ins(i).tolist()) | set(trace.outs(i).tolist())) for i in range(trace.n_ops)]
    ptr = np.zeros(trace.n_ops + 1, np.int32)
    ptr[1:] = np.cumsum([len(u) for u in uses])
    idx = np.array([x for u in uses for x in u], np.int32)
    tokens = _arr(tokens, np.int32)
    cnt = np.zeros(trace.n_tensors, np.uint32)
    tag = np.zeros(trace.n_tensors, np.uint32)
    stk = np.zeros(trace.n_tensors, np.uint64)
    lib().orc_features_after(_p(tokens), trace.n_ops, _p(ptr), _p(idx), trace.n_tensors,
                             _p(_arr(op_index, np.uint8)), _p(_arr(op_onehot, np.uint32)), after,
                             _p(cnt), _p(tag), _p(stk))
    return cnt, tag, stk


def swap_execute(dst_ptrs, src_ptrs, nbytes):
    """byte-exact copy of each source range to its destination (host pointers)"""
    n = len(nbytes)
    d = (C.c_void_p * max(n, 1))(*dst_ptrs)
    sp = (C.c_void_p * max(n, 1))(*src_ptrs)
    nb = (C.c_uint64 * max(n, 1))(*[int(x) for x in nbytes])
    lib().orc_swap_execute(n, d, sp, nb)
