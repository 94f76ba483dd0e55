"""Thin ctypes binding of include/chm.h (argument marshalling only).

Every step of the hot path runs inside libchm.so (C++ runtime + sm_100a CUDA kernels).  This
module never computes any part of the method; it converts Python/torch arguments to the
C-ABI's plain pointers and sizes.  If libchm.so is missing it raises -- there is no fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CHM_LIB") or os.path.join(_HERE, "libchm.so")  # CHM_LIB: e.g. libchm_debug.so

CHM_OK, CHM_E_INVAL, CHM_E_PARSE, CHM_E_STATE, CHM_E_NOMEM, CHM_E_CUDA, CHM_E_INFEASIBLE, CHM_E_NOKERNEL = \
    0, -1, -2, -3, -4, -5, -6, -7
FWD, BWD, OPT = 0, 1, 2
WARMUP, GENPOLICY, STABLE = 0, 1, 2
EXHAUSTIVE, SEEDED, MASKS, EXPLICIT, FLIP1 = 0, 1, 2, 3, 4
SWAP_KERNEL, SWAP_CE, SWAP_AUTO = 0, 1, 2


class ChmError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"chm error {code}: {msg}")
        self.code = code


class Config(C.Structure):
    _fields_ = [("m", C.c_uint32), ("n", C.c_uint32), ("len_tol", C.c_double), ("cos_tol", C.c_double),
                ("cos_mode", C.c_uint32), ("detect_bytes", C.c_uint32), ("device", C.c_int32),
                ("host_arena_bytes", C.c_uint64), ("swap_ctas", C.c_uint32), ("eval_ctas_per_sm", C.c_uint32),
                ("match_window", C.c_uint32), ("time_batches", C.c_uint32),
                ("ce_min_bytes", C.c_uint64), ("swap_variant", C.c_uint32), ("arena_mode", C.c_uint32),
                ("arena_numa", C.c_int32), ("arena_threads", C.c_uint32)]

ARENA_AUTO, ARENA_HOSTALLOC, ARENA_REGISTER = 0, 1, 2


class TensorRef(C.Structure):
    _fields_ = [("id", C.c_uint64), ("nbytes", C.c_int64), ("dtype", C.c_uint8)]


class OpRecord(C.Structure):
    _fields_ = [("token", C.c_int32), ("phase", C.c_uint8), ("n_in", C.c_uint32), ("n_out", C.c_uint32),
                ("n_free", C.c_uint32), ("in_", C.POINTER(TensorRef)), ("out", C.POINTER(TensorRef)),
                ("freed", C.POINTER(C.c_uint64)), ("live_bytes", C.c_int64)]


TENSOR_REF_DTYPE = np.dtype([("id", np.uint64), ("nbytes", np.int64), ("dtype", np.uint8)], align=True)


class Recorder:
    """chm_record_op with preallocated argument buffers: the per-op path of a framework hook
    (one ctypes call, no per-op ctypes objects)."""

    def __init__(self, ctx: "Context", cap: int = 64):
        self.ctx = ctx
        self._fn = load().chm_record_op
        self.rec = OpRecord()
        self.act = Actions()
        self._rec_p = C.byref(self.rec)
        self._act_p = C.byref(self.act)
        self._alloc(cap)

    def _alloc(self, cap: int):
        self.cap = cap
        self.ins = np.zeros(cap, TENSOR_REF_DTYPE)
        self.outs = np.zeros(cap, TENSOR_REF_DTYPE)
        self.freed = np.zeros(cap, np.uint64)
        self.rec.in_ = C.cast(self.ins.ctypes.data, C.POINTER(TensorRef))
        self.rec.out = C.cast(self.outs.ctypes.data, C.POINTER(TensorRef))
        self.rec.freed = C.cast(self.freed.ctypes.data, C.POINTER(C.c_uint64))

    def record(self, token: int, phase: int, ins=(), outs=(), freed=(), live_bytes: int = -1) -> "Actions":
        """ins / outs: sequences of (id, nbytes, dtype) tuples"""
        ni, no, nf = len(ins), len(outs), len(freed)
        if max(ni, no, nf) > self.cap:
            self._alloc(2 * max(ni, no, nf))
        r = self.rec
        if ni:
            self.ins[:ni] = ins
        if no:
            self.outs[:no] = outs
        if nf:
            self.freed[:nf] = freed
        r.token, r.phase, r.n_in, r.n_out, r.n_free, r.live_bytes = token, phase, ni, no, nf, live_bytes
        rc = self._fn(self.ctx.h, self._rec_p, self._act_p)
        if rc != CHM_OK:
            _check(rc)
        return self.act


class SwapDesc(C.Structure):
    _fields_ = [("dev", C.c_uint64), ("host_off", C.c_uint64), ("nbytes", C.c_uint64)]


SWAP_DESC_DTYPE = np.dtype([("dev", np.uint64), ("host_off", np.uint64), ("nbytes", np.uint64)])


class Actions(C.Structure):
    _fields_ = [("n_swap_out", C.c_uint32), ("swap_out", C.POINTER(SwapDesc)), ("swap_out_item", C.POINTER(C.c_uint32)),
                ("n_release", C.c_uint32), ("release_item", C.POINTER(C.c_uint32)),
                ("n_swap_in", C.c_uint32), ("swap_in", C.POINTER(SwapDesc)), ("swap_in_item", C.POINTER(C.c_uint32)),
                ("n_wait", C.c_uint32), ("wait_item", C.POINTER(C.c_uint32))]


class TraceParams(C.Structure):
    _fields_ = [("hbm_budget", C.c_int64), ("static_bytes", C.c_int64), ("t_iter_s", C.c_double),
                ("bw_bytes_per_s", C.c_double), ("groups_fwd", C.c_uint32), ("groups_bwd", C.c_uint32),
                ("omega", C.c_double), ("f0_source", C.c_uint32)]


class TraceInfo(C.Structure):
    _fields_ = [("n_ops", C.c_uint32), ("n_tensors", C.c_uint32), ("n_swappable", C.c_uint32),
                ("n_layers", C.c_uint32), ("mask_words", C.c_uint32), ("peak0", C.c_int64),
                ("argmax0", C.c_uint32), ("budget", C.c_int64)]


class Candidates(C.Structure):
    _fields_ = [("kind", C.c_int), ("first_index", C.c_uint64), ("count", C.c_uint64), ("seed", C.c_uint64),
                ("flip_thr", C.c_uint64), ("base_mask", C.c_void_p), ("masks", C.c_void_p),
                ("item_offsets", C.c_void_p), ("items", C.c_void_p)]


class Item(C.Structure):
    _fields_ = [("t", C.c_uint32), ("r", C.c_int32), ("s", C.c_int32), ("flags", C.c_uint32)]


ITEM_DTYPE = np.dtype([("t", np.uint32), ("r", np.int32), ("s", np.int32), ("flags", np.uint32)])


class GenParams(C.Structure):
    _fields_ = [("C", C.c_double), ("rem_scale", C.c_double)]


class Best(C.Structure):
    _fields_ = [("excess", C.c_int64), ("stall", C.c_double), ("swapped_bytes", C.c_int64),
                ("index", C.c_uint64), ("peak", C.c_int64)]

    def key(self):
        return (self.excess, self.stall, self.swapped_bytes, self.index)


BEST_DTYPE = np.dtype([("excess", np.int64), ("stall", np.float64), ("swapped_bytes", np.int64),
                       ("index", np.uint64), ("peak", np.int64)])


class EvalOut(C.Structure):
    _fields_ = [("peak", C.c_void_p), ("stall", C.c_void_p), ("swapped", C.c_void_p), ("footprint", C.c_void_p),
                ("ld", C.c_uint32), ("best", C.c_void_p), ("stall_model", C.c_uint32)]


STALL_LAYER, STALL_TIMELINE = 0, 1


class ExecStats(C.Structure):
    _fields_ = [("n_items", C.c_uint32), ("n_matched", C.c_uint32), ("n_stale", C.c_uint32),
                ("n_collisions", C.c_uint32), ("n_demand_swap_in", C.c_uint32),
                ("bytes_out", C.c_uint64), ("bytes_in", C.c_uint64)]


class Passive(C.Structure):
    _fields_ = [("handle", C.c_uint64), ("id", C.c_uint64), ("nbytes", C.c_int64), ("host_off", C.c_uint64),
                ("batch", C.c_uint64)]


EXPORTS = [
    "chm_config_default", "chm_create", "chm_destroy", "chm_last_error", "chm_build_info", "chm_tokenize",
    "chm_record_op", "chm_set_detailed", "chm_detect_seq_change", "chm_trace_build", "chm_trace_free",
    "chm_trace_get_info", "chm_trace_tables", "chm_trace_digest", "chm_eval_policies", "chm_eval_policies_ex", "chm_best_reduce", "chm_best_reduce_device", "chm_candidate_mask",
    "chm_policy_install", "chm_policy_install_items", "chm_generate_policy", "chm_exec_stats_get", "chm_host_arena", "chm_swap_out", "chm_swap_in",
    "chm_batch_wait", "chm_batch_query", "chm_batch_elapsed", "chm_arena_reserve", "chm_issue_swap_out", "chm_issue_swap_in", "chm_item_wait",
    "chm_oom_release", "chm_passive_swap", "chm_passive_restore", "chm_trace_load", "chm_record_save",
    "chm_stall_models", "chm_record_tokens", "chm_arena_placement", "chm_release_scratch", "chm_descend",
]

_lib = None


def load(path: str = LIB_PATH):
    """Loads libchm.so; raises if it is missing (no CPU fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built: run `python -m paper_2509_11076_b200.build`")
    L = C.CDLL(path)
    vp, u32, u64, i32, i64, dbl = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int32, C.c_int64, C.c_double
    P = C.POINTER
    sig = {
        "chm_config_default": (None, [P(Config)]),
        "chm_arena_placement": (i32, [vp, P(i32), P(i32), P(dbl)]),
        "chm_release_scratch": (i32, [vp]),
        "chm_create": (i32, [P(Config), P(vp)]),
        "chm_destroy": (None, [vp]),
        "chm_last_error": (C.c_char_p, []),
        "chm_build_info": (C.c_char_p, []),
        "chm_tokenize": (i32, [vp, C.c_char_p, P(i32)]),
        "chm_record_op": (i32, [vp, P(OpRecord), P(Actions)]),
        "chm_set_detailed": (i32, [vp, i32]),
        "chm_detect_seq_change": (i32, [vp, dbl, P(i32), P(i32), P(dbl), P(dbl)]),
        "chm_trace_build": (i32, [vp, P(TraceParams), P(vp)]),
        "chm_trace_free": (None, [vp]),
        "chm_trace_get_info": (i32, [vp, P(TraceInfo)]),
        "chm_trace_tables": (i32, [vp] + [vp] * 11),
        "chm_trace_digest": (i32, [vp, P(u64)]),
        "chm_eval_policies": (i32, [vp, vp, P(Candidates), P(EvalOut), vp]),
        "chm_eval_policies_ex": (i32, [vp, vp, P(Candidates), P(EvalOut), vp, P(i64)]),
        "chm_generate_policy": (i32, [vp, P(GenParams), vp, u32, P(u32), P(i32)]),
        "chm_policy_install_items": (i32, [vp, vp, vp, u32]),
        "chm_best_reduce": (i32, [vp, u32, P(Best)]),
        "chm_best_reduce_device": (i32, [vp, vp, u32, vp, vp]),
        "chm_descend": (i32, [vp, vp, vp, u32, u32, vp, vp, vp, vp, vp]),
        "chm_candidate_mask": (i32, [vp, P(Candidates), u64, vp]),
        "chm_policy_install": (i32, [vp, vp, vp]),
        "chm_exec_stats_get": (i32, [vp, P(ExecStats)]),
        "chm_host_arena": (i32, [vp, P(vp), P(u64)]),
        "chm_swap_out": (i32, [vp, vp, u32, vp, vp, u32, P(u64), P(i64)]),
        "chm_swap_in": (i32, [vp, vp, u32, vp, vp, u32, P(u64), P(i64)]),
        "chm_batch_wait": (i32, [vp, u64, vp]),
        "chm_batch_query": (i32, [vp, u64, P(i32)]),
        "chm_batch_elapsed": (i32, [vp, u64, P(C.c_float)]),
        "chm_arena_reserve": (i32, [vp, u64]),
        "chm_issue_swap_out": (i32, [vp, vp, vp, u32, P(u64)]),
        "chm_issue_swap_in": (i32, [vp, vp, vp, vp, u32, P(u64)]),
        "chm_item_wait": (i32, [vp, u32, i32, vp]),
        "chm_oom_release": (i32, [vp, vp, vp, u32, P(u32)]),
        "chm_trace_load": (i32, [vp, C.c_char_p, C.c_size_t, P(TraceParams), P(vp), P(i64)]),
        "chm_record_save": (i32, [vp, vp, C.c_size_t, P(C.c_size_t)]),
        "chm_stall_models": (i32, [vp, vp, u32, vp]),
        "chm_record_tokens": (i32, [vp, vp, vp, u32]),
        "chm_passive_swap": (i32, [vp, i64, vp, u32, vp, u32, vp, vp, P(Passive)]),
        "chm_passive_restore": (i32, [vp, u64, u64, vp, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _check(rc: int):
    if rc != CHM_OK:
        raise ChmError(rc, (load().chm_last_error() or b"").decode())


def _ptr(x) -> Optional[int]:
    """device/host pointer of a torch tensor, numpy array or int"""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    raise TypeError(type(x))


def _stream(s) -> Optional[int]:
    if s is None:
        return None
    if isinstance(s, int):
        return s
    return s.cuda_stream


class Trace:
    def __init__(self, ctx: "Context", handle: C.c_void_p):
        self.ctx = ctx
        self.h = handle
        info = TraceInfo()
        _check(load().chm_trace_get_info(self.h, C.byref(info)))
        self.info = info
        self.N, self.T, self.K, self.L, self.W = (info.n_ops, info.n_tensors, info.n_swappable, info.n_layers,
                                                 info.mask_words)
        self.peak0, self.argmax0, self.budget = info.peak0, info.argmax0, info.budget

    def tables(self):
        N, K, L, W = self.N, self.K, self.L, self.W
        out = dict(f0=np.zeros(N, np.int64), tensor=np.zeros(K, np.uint32), nbytes=np.zeros(K, np.int64),
                   r=np.zeros(K, np.int32), s=np.zeros(K, np.int32), lin=np.zeros(K, np.int32),
                   lout=np.zeros(K, np.int32), lay_start=np.zeros(L, np.int32), lay_count=np.zeros(L, np.int32),
                   bud=np.zeros(L, np.float64), base=np.zeros(max(W, 1), np.uint64))
        keys = ["f0", "tensor", "nbytes", "r", "s", "lin", "lout", "lay_start", "lay_count", "bud", "base"]
        _check(load().chm_trace_tables(self.h, *[out[k].ctypes.data for k in keys]))
        out["base"] = out["base"][:W]
        return out

    def digest(self) -> int:
        """64-bit digest of the evaluated tables (chm_trace_digest)"""
        d = C.c_uint64()
        _check(load().chm_trace_digest(self.h, C.byref(d)))
        return d.value

    def generate_policy(self, C_coef: float = 1.0, rem_scale: float = 1.0):
        """Algo. 2 -> (items ITEM_DTYPE array, feasible)"""
        cap = self.T + 1
        out = np.zeros(cap, ITEM_DTYPE)
        n, feas = C.c_uint32(), C.c_int32()
        _check(load().chm_generate_policy(self.h, C.byref(GenParams(C_coef, rem_scale)), out.ctypes.data, cap,
                                          C.byref(n), C.byref(feas)))
        return out[:n.value], bool(feas.value)

    def stall_models(self, items) -> np.ndarray:
        """[R-stall, per-direction budgets, serial-stream timeline] of one item list (host)"""
        its = np.ascontiguousarray(items, ITEM_DTYPE)
        out = np.zeros(3, np.float64)
        _check(load().chm_stall_models(self.h, _ptr(its) if its.size else None, int(its.size), _ptr(out)))
        return out

    def mask_items(self, words) -> np.ndarray:
        """the item list {t, r, s} (solo timing) of a mask over the swappable set"""
        tb = self.tables()
        ks = [k for k in range(self.K) if (int(words[k // 64]) >> (k % 64)) & 1]
        its = np.zeros(len(ks), ITEM_DTYPE)
        its["t"] = tb["tensor"][ks]
        its["r"] = tb["r"][ks]
        its["s"] = tb["s"][ks]
        return its

    def candidate_mask(self, kind: int, index: int, seed: int = 0, flip_thr: int = 0,
                       base: Optional[np.ndarray] = None) -> np.ndarray:
        w = np.zeros(max(self.W, 1), np.uint64)
        b = np.ascontiguousarray(base, np.uint64) if base is not None else None
        c = Candidates(kind, 0, 1, seed, flip_thr, _ptr(b), None, None, None)
        _check(load().chm_candidate_mask(self.h, C.byref(c), index, w.ctypes.data))
        return w[:self.W]

    def free(self):
        if self.h:
            load().chm_trace_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:  # noqa: BLE001
            pass


class Context:
    """One chm_ctx per device / rank (single owner, not thread-safe)."""

    def __init__(self, device: int = 0, host_arena_bytes: int = 0, swap_ctas: int = 0, eval_ctas_per_sm: int = 0,
                 time_batches: bool = False, swap_variant: int = 0, ce_min_bytes: int = 0,
                 arena_mode: int = ARENA_AUTO, arena_numa: int = -1, arena_threads: int = 0, **algo1):
        L = load()
        cfg = Config()
        L.chm_config_default(C.byref(cfg))
        cfg.device = device
        cfg.host_arena_bytes = host_arena_bytes
        cfg.swap_ctas = swap_ctas
        cfg.eval_ctas_per_sm = eval_ctas_per_sm
        cfg.time_batches = 1 if time_batches else 0
        cfg.swap_variant = swap_variant
        cfg.ce_min_bytes = ce_min_bytes
        cfg.arena_mode = arena_mode
        cfg.arena_numa = arena_numa
        cfg.arena_threads = arena_threads
        for k, v in algo1.items():
            setattr(cfg, k, v)
        h = C.c_void_p()
        _check(L.chm_create(C.byref(cfg), C.byref(h)))
        self.h = h
        self.device = device
        self._actions = Actions()

    def close(self):
        if getattr(self, "h", None):
            load().chm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    # ---------------------------------------------------------------- profiler hook
    def tokenize(self, name: str) -> int:
        t = C.c_int32()
        _check(load().chm_tokenize(self.h, name.encode(), C.byref(t)))
        return t.value

    def set_detailed(self, on: bool = True):
        _check(load().chm_set_detailed(self.h, 1 if on else 0))

    def record_op(self, token: int, phase: int, ins: Sequence = (), outs: Sequence = (), freed: Sequence[int] = (),
                  live_bytes: int = -1) -> Actions:
        """ins/outs: sequences of (id, nbytes, dtype)"""
        ni, no, nf = len(ins), len(outs), len(freed)
        a_in = (TensorRef * max(ni, 1))(*[TensorRef(int(i), int(n), int(d)) for (i, n, d) in ins])
        a_out = (TensorRef * max(no, 1))(*[TensorRef(int(i), int(n), int(d)) for (i, n, d) in outs])
        a_fr = (C.c_uint64 * max(nf, 1))(*[int(x) for x in freed])
        rec = OpRecord(token, phase, ni, no, nf, a_in, a_out, a_fr, live_bytes)
        _check(load().chm_record_op(self.h, C.byref(rec), C.byref(self._actions)))
        return self._actions

    def record_tokens(self, tokens, phases):
        """Lightweight mode in bulk: an iteration's operator tokens and phases at once"""
        t = np.ascontiguousarray(tokens, np.int32)
        ph = np.ascontiguousarray(phases, np.uint8)
        if t.size != ph.size:
            raise ValueError("tokens and phases differ in length")
        _check(load().chm_record_tokens(self.h, _ptr(t) if t.size else None, _ptr(ph) if ph.size else None,
                                        int(t.size)))

    def detect_seq_change(self, t_iter: float):
        st, ch, ld, cs = C.c_int32(), C.c_int32(), C.c_double(), C.c_double()
        _check(load().chm_detect_seq_change(self.h, t_iter, C.byref(st), C.byref(ch), C.byref(ld), C.byref(cs)))
        return dict(stage=st.value, changed=bool(ch.value), len_diff=ld.value, cos=cs.value)

    # ------------------------------------------------------------------ trace build
    def trace_build(self, budget: int, static_bytes: int, bw: float, groups_fwd: int, groups_bwd: int,
                    t_iter: float = 0.0, omega: float = 1.0, f0_source: int = 0) -> Trace:
        p = TraceParams(int(budget), int(static_bytes), float(t_iter), float(bw), int(groups_fwd), int(groups_bwd),
                        float(omega), int(f0_source))
        h = C.c_void_p()
        _check(load().chm_trace_build(self.h, C.byref(p), C.byref(h)))
        return Trace(self, h)

    def trace_load(self, text: bytes, budget: int, static_bytes: int, bw: float, groups_fwd: int, groups_bwd: int,
                   t_iter: float = 0.0, omega: float = 1.0, f0_source: int = 0) -> Trace:
        """builds a trace from a Detailed-record file (chm_trace_load); ChmError.offset = byte
        offset of a parse error"""
        p = TraceParams(int(budget), int(static_bytes), float(t_iter), float(bw), int(groups_fwd), int(groups_bwd),
                        float(omega), int(f0_source))
        h = C.c_void_p()
        off = C.c_int64(-1)
        rc = load().chm_trace_load(self.h, text, len(text), C.byref(p), C.byref(h), C.byref(off))
        if rc != CHM_OK:
            err = ChmError(rc, (load().chm_last_error() or b"").decode())
            err.offset = off.value
            raise err
        return Trace(self, h)

    def record_save(self) -> bytes:
        """the last Detailed iteration as a Detailed-record file (chm_record_save)"""
        n = C.c_size_t()
        rc = load().chm_record_save(self.h, None, 0, C.byref(n))
        if rc not in (CHM_OK, CHM_E_NOMEM):
            _check(rc)
        buf = C.create_string_buffer(n.value)
        _check(load().chm_record_save(self.h, buf, n.value, C.byref(n)))
        return buf.raw[:n.value]

    # ------------------------------------------------------------ policy evaluation
    def eval_policies(self, trace: Trace, kind: int, first: int, count: int, *, best, seed: int = 0,
                      flip_thr: int = 0, base: Optional[np.ndarray] = None, masks=None, peak=None, stall=None,
                      swapped=None, footprint=None, ld: int = 0, stream=None, item_offsets=None, items=None,
                      stall_model: int = STALL_LAYER):
        b = np.ascontiguousarray(base, np.uint64) if base is not None else None
        off = np.ascontiguousarray(item_offsets, np.uint64) if item_offsets is not None else None
        its = np.ascontiguousarray(items, ITEM_DTYPE) if items is not None else None
        c = Candidates(kind, first, count, seed, flip_thr, _ptr(b), _ptr(masks), _ptr(off),
                       _ptr(its) if its is not None and its.size else None)
        o = EvalOut(_ptr(peak), _ptr(stall), _ptr(swapped), _ptr(footprint), ld, _ptr(best), stall_model)
        e = C.c_int64()
        rc = load().chm_eval_policies_ex(self.h, trace.h, C.byref(c), C.byref(o), _stream(stream), C.byref(e))
        if rc != CHM_OK:
            err = ChmError(rc, (load().chm_last_error() or b"").decode())
            err.index = e.value
            raise err

    def policy_install_items(self, trace: Trace, items):
        its = np.ascontiguousarray(items, ITEM_DTYPE)
        _check(load().chm_policy_install_items(self.h, trace.h, its.ctypes.data if its.size else None, len(its)))

    def best_reduce_device(self, keys, n: int, out, stream=None):
        _check(load().chm_best_reduce_device(self.h, _ptr(keys), n, _ptr(out), _stream(stream)))

    def descend(self, trace: Trace, starts, n_starts: int, *, ends, keys, max_rounds: int = 4096, rounds=None,
                best=None, stream=None):
        """chm_descend: steepest single-flip descent from n_starts device masks [n][W] (uint64 /
        int64 tensors); writes the end masks, their keys (chm_best [n]), optional rounds (int32
        [n]) and the best key -- all device buffers, enqueued on `stream`"""
        _check(load().chm_descend(self.h, trace.h, _ptr(starts), n_starts, max_rounds, _ptr(ends), _ptr(keys),
                                  _ptr(rounds), _ptr(best), _stream(stream)))

    # ---------------------------------------------------------------------- swap
    def host_arena(self):
        p, n = C.c_void_p(), C.c_uint64()
        _check(load().chm_host_arena(self.h, C.byref(p), C.byref(n)))
        return p.value or 0, n.value

    def _swap(self, fn, descs, compute, swap, flags):
        d = np.ascontiguousarray(descs, SWAP_DESC_DTYPE)
        b, e = C.c_uint64(), C.c_int64()
        rc = fn(self.h, d.ctypes.data, len(d), _stream(compute), _stream(swap), flags, C.byref(b), C.byref(e))
        if rc != CHM_OK:
            err = ChmError(rc, (load().chm_last_error() or b"").decode())
            err.index = e.value
            raise err
        return b.value

    def swap_out(self, descs, compute=None, swap=None, flags: int = SWAP_KERNEL) -> int:
        return self._swap(load().chm_swap_out, descs, compute, swap, flags)

    def swap_in(self, descs, compute=None, swap=None, flags: int = SWAP_KERNEL) -> int:
        return self._swap(load().chm_swap_in, descs, compute, swap, flags)

    def batch_wait(self, batch: int, stream=None):
        _check(load().chm_batch_wait(self.h, batch, _stream(stream)))

    def batch_elapsed_ms(self, batch: int) -> float:
        ms = C.c_float()
        _check(load().chm_batch_elapsed(self.h, batch, C.byref(ms)))
        return ms.value

    def arena_reserve(self, nbytes: int):
        _check(load().chm_arena_reserve(self.h, int(nbytes)))

    def release_scratch(self):
        """frees the evaluation calls' device scratch (chm_release_scratch); synchronises"""
        _check(load().chm_release_scratch(self.h))

    def arena_placement(self) -> dict:
        """{"numa_node": bound node or -1, "mode": ARENA_HOSTALLOC / ARENA_REGISTER / -1,
        "pin_s": seconds the last allocation + pinning took}"""
        n, m, t = C.c_int32(), C.c_int32(), C.c_double()
        _check(load().chm_arena_placement(self.h, C.byref(n), C.byref(m), C.byref(t)))
        return {"numa_node": n.value, "mode": m.value, "pin_s": t.value}

    def batch_query(self, batch: int) -> bool:
        d = C.c_int32()
        _check(load().chm_batch_query(self.h, batch, C.byref(d)))
        return bool(d.value)

    # ------------------------------------------------------------------ executor
    def policy_install(self, trace: Trace, words: np.ndarray):
        w = np.ascontiguousarray(words, np.uint64)
        _check(load().chm_policy_install(self.h, trace.h, w.ctypes.data if w.size else None))

    def issue_swap_out(self, compute=None, swap=None, flags: int = SWAP_KERNEL) -> int:
        b = C.c_uint64()
        _check(load().chm_issue_swap_out(self.h, _stream(compute), _stream(swap), flags, C.byref(b)))
        return b.value

    def issue_swap_in(self, dev: Sequence[int], compute=None, swap=None, flags: int = SWAP_KERNEL) -> int:
        arr = (C.c_uint64 * max(len(dev), 1))(*[int(x) for x in dev])
        b = C.c_uint64()
        _check(load().chm_issue_swap_in(self.h, arr, _stream(compute), _stream(swap), flags, C.byref(b)))
        return b.value

    def item_wait(self, item: int, swap_in: bool, stream=None):
        _check(load().chm_item_wait(self.h, item, 1 if swap_in else 0, _stream(stream)))

    # ------------------------------------------------------------ OOM handling (Algo. 3)
    def oom_release(self, stream=None, cap: int = 4096) -> list:
        """(i)-(ii): release every marked block (swap-out issued, release point not reached) behind
        an event pair; returns the policy items whose device storage the caller drops now"""
        buf = (C.c_uint32 * cap)()
        n = C.c_uint32()
        _check(load().chm_oom_release(self.h, _stream(stream), buf, cap, C.byref(n)))
        return list(buf[:n.value])

    def passive_swap(self, need: int, exclude=(), compute=None, swap=None, only=None) -> dict:
        """(iv): swap out the resident tensor closest in size to `need` (among `only` if given);
        the caller drops its storage (the compute stream already waits for the copy)"""
        ex = np.ascontiguousarray(list(exclude), np.uint64)
        n_on = 0
        on = None
        if only is not None:
            n_on = len(only)
            on = np.ascontiguousarray(list(only) if n_on else [0], np.uint64)  # empty: nothing eligible
        out = Passive()
        _check(load().chm_passive_swap(self.h, int(need), _ptr(ex) if ex.size else None, int(ex.size),
                                       _ptr(on), n_on, _stream(compute), _stream(swap), C.byref(out)))
        return {k: getattr(out, k) for k, _ in Passive._fields_}

    def passive_restore(self, handle: int, dev: int, compute=None, swap=None):
        """demand swap-in of passive swap `handle` into `dev` before its next use; dev = 0: the
        tensor died while out (drop the host copy)"""
        _check(load().chm_passive_restore(self.h, int(handle), int(dev), _stream(compute), _stream(swap)))

    def exec_stats(self) -> dict:
        s = ExecStats()
        _check(load().chm_exec_stats_get(self.h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in ExecStats._fields_}


def best_reduce(keys: np.ndarray) -> np.void:
    """host lexicographic min of chm_best keys (BEST_DTYPE array)"""
    k = np.ascontiguousarray(keys, BEST_DTYPE)
    out = Best()
    _check(load().chm_best_reduce(k.ctypes.data, len(k), C.byref(out)))
    return out


def actions_view(a: Actions) -> dict:
    """copies the library-owned action arrays of the last record_op into Python lists"""
    def arr(p, n):
        return [p[i] for i in range(n)] if n else []
    def descs(p, n):
        return [(p[i].dev, p[i].host_off, p[i].nbytes) for i in range(n)] if n else []
    return dict(swap_out=descs(a.swap_out, a.n_swap_out), swap_out_item=arr(a.swap_out_item, a.n_swap_out),
                release=arr(a.release_item, a.n_release), swap_in=descs(a.swap_in, a.n_swap_in),
                swap_in_item=arr(a.swap_in_item, a.n_swap_in), wait=arr(a.wait_item, a.n_wait))


def record_iteration(ctx: Context, trace, tokens: Optional[Sequence[int]] = None, on_actions=None):
    """Feeds one iteration of a workloads.traces.Trace through the profiler hook
    (chm_record_op per op, marshalling only).  tokens: per-op token ids (default: ctx tokenizer)."""
    if tokens is None:
        tokens = [ctx.tokenize(nm) for nm in trace.op_names]
    ptr, nb, dt = trace.ptr, trace.nbytes, trace.dtype
    for i in range(trace.n_ops):
        ins = [(ptr[t], nb[t], dt[t]) for t in trace.ins(i)]
        outs = [(ptr[t], nb[t], dt[t]) for t in trace.outs(i)]
        freed = [ptr[t] for t in trace.frees(i)]
        a = ctx.record_op(int(tokens[i]), int(trace.phase[i]), ins, outs, freed)
        if on_actions is not None:
            on_actions(i, a)
    return tokens


class PreparedIteration:
    """Pre-marshalled chm_op_record array for one iteration of a trace (ids chosen by the caller),
    so a replay loop only pays one ctypes call per op."""

    def __init__(self, trace, ids, tokens):
        self.recs = []
        self._keep = []
        nb, dt = trace.nbytes, trace.dtype
        for i in range(trace.n_ops):
            ins = [TensorRef(int(ids[t]), int(nb[t]), int(dt[t])) for t in trace.ins(i)]
            outs = [TensorRef(int(ids[t]), int(nb[t]), int(dt[t])) for t in trace.outs(i)]
            fr = [int(ids[t]) for t in trace.frees(i)]
            a_in = (TensorRef * max(len(ins), 1))(*ins)
            a_out = (TensorRef * max(len(outs), 1))(*outs)
            a_fr = (C.c_uint64 * max(len(fr), 1))(*fr)
            self._keep += [a_in, a_out, a_fr]
            self.recs.append(OpRecord(int(tokens[i]), int(trace.phase[i]), len(ins), len(outs), len(fr),
                                      a_in, a_out, a_fr, -1))
