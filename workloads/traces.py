"""Seeded synthetic eager-mode operator traces (configs C1..C5 of BASELINE.json).

This module is INPUT GENERATION ONLY: it builds what the paper's Detailed-mode
profiler observes for one training iteration ("the name of each
operator, the input tensor arrays, and output tensor arrays ... data_ptr, data
type") plus the refcount releases of eager memory management.  It holds
none of the method's arithmetic: no footprint, no logical layers, no swap
timing, no candidate decoding.  Both the CPU oracle (`oracle/`) and the CUDA
product consume what it returns; neither shares any other code.

Every tensor size is a multiple of 512 B, the caching-allocator block size
(SURVEY.md §8(c) Q16).  Recipes (shapes, sizes, seeds) are stated in DESIGN.md
§"Input recipe".
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

FWD, BWD, OPT = 0, 1, 2
DTYPE_CODE = {"bf16": 0, "f32": 1, "u8": 2, "i64": 3}
DTYPE_SIZE = {"bf16": 2, "f32": 4, "u8": 1, "i64": 8}
GiB = 1 << 30
MiB = 1 << 20
KiB = 1 << 10
B200_HBM_BYTES = 183359 * MiB  # nvidia-smi total on the pool's B200s (B200_PROFILING.md)
B200_BF16_TFLOPS = 1687.8e12  # MEASURED_PEAKS.json, used only for the synthetic T_iter FLOP model


@dataclasses.dataclass
class Trace:
    """One profiled iteration, as raw records.

    Tensor index t = 0..T-1 is the generator's own identity for each tensor
    (what the paper's system lacks across iterations).  `ptr[t]` is a
    simulated `data_ptr` that the allocator may REUSE after a free, which is
    what the C-ABI profiler hook sees (chm_tensor_ref.id).
    Produced tensors are numbered in production order (op order, then output
    slot); static tensors (weights, live at iteration start, bytes inside
    `static_bytes`) come after them.
    """

    name: str
    op_names: List[str]
    phase: np.ndarray  # uint8 [N]
    in_ptr: np.ndarray  # int32 [N+1]   CSR of input tensor indices
    in_idx: np.ndarray  # int32
    out_ptr: np.ndarray  # int32 [N+1]  CSR of output tensor indices (allocations)
    out_idx: np.ndarray
    free_ptr: np.ndarray  # int32 [N+1] CSR of tensors whose refcount hits 0 after op i
    free_idx: np.ndarray
    nbytes: np.ndarray  # int64 [T]
    dtype: np.ndarray  # uint8 [T]
    ptr: np.ndarray  # uint64 [T] simulated data_ptr (reused after free)
    n_produced: int  # tensors 0..n_produced-1 are produced by an op; the rest are static
    static_bytes: int  # M_0: bytes live at iteration start (params, grads, optimizer state)
    t_iter: float  # measured iteration time (s), Eq. 1's T_iter
    bw: float  # host<->device bandwidth B (bytes/s), Eq. 3
    budget: int  # HBM budget (bytes)
    groups_fwd: int
    groups_bwd: int
    omega: float = 1.0
    meta: dict = dataclasses.field(default_factory=dict)

    @property
    def n_ops(self) -> int:
        return len(self.op_names)

    @property
    def n_tensors(self) -> int:
        return len(self.nbytes)

    def ins(self, i: int) -> np.ndarray:
        return self.in_idx[self.in_ptr[i]:self.in_ptr[i + 1]]

    def outs(self, i: int) -> np.ndarray:
        return self.out_idx[self.out_ptr[i]:self.out_ptr[i + 1]]

    def frees(self, i: int) -> np.ndarray:
        return self.free_idx[self.free_ptr[i]:self.free_ptr[i + 1]]


def to_jsonl(trace: Trace) -> bytes:
    """The trace as a Detailed-record file (the format `chm_trace_load` reads, include/chm.h):
    header with the tensor table, then one line per op (format conversion only)."""
    import json
    lines = [json.dumps({"chm_trace": 1, "t_iter_s": float(trace.t_iter),
                         "tensors": [[int(trace.nbytes[t]), int(trace.dtype[t])] for t in range(trace.n_tensors)]},
                        separators=(",", ":"))]
    for i in range(trace.n_ops):
        lines.append(json.dumps({"op": trace.op_names[i], "phase": int(trace.phase[i]),
                                 "in": [int(t) for t in trace.ins(i)], "out": [int(t) for t in trace.outs(i)],
                                 "free": [int(t) for t in trace.frees(i)]}, separators=(",", ":")))
    return ("\n".join(lines) + "\n").encode()


class _Builder:
    """Records ops in dispatch order; frees are the eager refcount releases."""

    def __init__(self) -> None:
        self.ops: List[Tuple[str, int, List[int], List[int]]] = []
        self.nbytes: List[int] = []
        self.dtype: List[int] = []
        self.static: List[bool] = []
        self.persist: List[bool] = []  # survives the iteration (never freed)

    def tensor(self, nbytes: int, dtype: str = "bf16", static: bool = False, persist: bool = False) -> int:
        nbytes = int(nbytes)
        if nbytes <= 0 or nbytes % 512:
            raise ValueError(f"tensor size {nbytes} is not a positive multiple of 512")
        self.nbytes.append(nbytes)
        self.dtype.append(DTYPE_CODE[dtype])
        self.static.append(static)
        self.persist.append(persist or static)
        return len(self.nbytes) - 1

    def op(self, name: str, phase: int, ins: Sequence[int], outs: Sequence[int]) -> int:
        self.ops.append((name, phase, [int(x) for x in ins], [int(x) for x in outs]))
        return len(self.ops) - 1

    def finish(self, name: str, **hdr) -> Trace:
        n = len(self.ops)
        T = len(self.nbytes)
        producer = np.full(T, -1, np.int64)
        last_use = np.full(T, -1, np.int64)
        for i, (_, _, ins, outs) in enumerate(self.ops):
            for t in outs:
                if producer[t] != -1 or self.static[t]:
                    raise ValueError("tensor produced twice / static tensor produced")
                producer[t] = i
                last_use[t] = max(last_use[t], i)
            for t in ins:
                if not self.static[t] and (producer[t] == -1 or producer[t] >= i):
                    raise ValueError(f"op {i} reads tensor {t} before it is produced")
                last_use[t] = max(last_use[t], i)
        # renumber: produced tensors in production order, then static tensors
        order: List[int] = []
        for (_, _, _, outs) in self.ops:
            order.extend(outs)
        n_prod = len(order)
        order.extend([t for t in range(T) if self.static[t]])
        unused = [t for t in range(T) if producer[t] == -1 and not self.static[t]]
        if unused:
            raise ValueError(f"tensors never produced: {unused[:5]}")
        remap = np.empty(T, np.int64)
        remap[np.array(order, np.int64)] = np.arange(T)
        # refcount release after the last op that touches a non-persistent tensor
        frees: List[List[int]] = [[] for _ in range(n)]
        for t in range(T):
            if not self.persist[t]:
                frees[int(last_use[t])].append(int(remap[t]))
        for lst in frees:
            lst.sort()

        def csr(lists):
            ptr = np.zeros(n + 1, np.int32)
            ptr[1:] = np.cumsum([len(x) for x in lists])
            idx = np.array([x for lst in lists for x in lst], np.int32)
            return ptr, idx

        in_ptr, in_idx = csr([[int(remap[t]) for t in ins] for (_, _, ins, _) in self.ops])
        out_ptr, out_idx = csr([[int(remap[t]) for t in outs] for (_, _, _, outs) in self.ops])
        free_ptr, free_idx = csr(frees)
        nbytes = np.array(self.nbytes, np.int64)[np.array(order, np.int64)]
        dtype = np.array(self.dtype, np.uint8)[np.array(order, np.int64)]
        ptr = _simulate_pointers(nbytes, n_prod, out_ptr, out_idx, free_ptr, free_idx)
        return Trace(
            name=name,
            op_names=[o[0] for o in self.ops],
            phase=np.array([o[1] for o in self.ops], np.uint8),
            in_ptr=in_ptr, in_idx=in_idx, out_ptr=out_ptr, out_idx=out_idx,
            free_ptr=free_ptr, free_idx=free_idx,
            nbytes=nbytes, dtype=dtype, ptr=ptr, n_produced=n_prod, **hdr)


def _simulate_pointers(nbytes, n_prod, out_ptr, out_idx, free_ptr, free_idx) -> np.ndarray:
    """A toy size-bucketed caching allocator: a freed block is handed to the next
    allocation of the same size (LIFO), so `data_ptr` values repeat within an
    iteration exactly as they do under PyTorch's allocator."""
    T = len(nbytes)
    ptr = np.zeros(T, np.uint64)
    free_by_size: Dict[int, List[int]] = {}
    bump = 0x7F0000000000
    n = len(out_ptr) - 1
    for i in range(n):
        for t in out_idx[out_ptr[i]:out_ptr[i + 1]]:
            lst = free_by_size.get(int(nbytes[t]))
            if lst:
                ptr[t] = lst.pop()
            else:
                ptr[t] = bump
                bump += int(nbytes[t]) + 512
        for t in free_idx[free_ptr[i]:free_ptr[i + 1]]:
            free_by_size.setdefault(int(nbytes[t]), []).append(int(ptr[t]))
    base = 0x100000000000
    for t in range(n_prod, T):
        ptr[t] = base
        base += int(nbytes[t]) + 512
    return ptr


# ----------------------------------------------------------------------------- C1
def tiny(seed: int = 1) -> Trace:
    """C1: 64 ops (32 FWD, 24 BWD, 8 OPT), 24 saved activations of 4 KiB-4 MiB.

    FWD: 4 "activation layers" x 6 ops, each op saving one activation used by the
    next op and by one backward op; then 2 layers x 4 ops with unsaved temporaries.
    BWD: 6 layers x 4 ops mirroring FWD; FWD layer j's activations are read by
    BWD layer 5-j, round robin over its 4 ops.  OPT: 8 ops on static state.
    """
    rng = np.random.default_rng(seed)
    b = _Builder()
    weights = [b.tensor(256 * KiB, static=True) for _ in range(8)]
    u = rng.random(24)
    act_sizes = [512 * math.ceil(2 ** (12 + 10 * x) / 512) for x in u]
    acts: List[int] = []
    prev: Optional[int] = None
    for j in range(4):
        for m in range(6):
            a = b.tensor(act_sizes[6 * j + m])
            b.op(f"fwd_op{m}", FWD, ([prev] if prev is not None else []) + [weights[j]], [a])
            acts.append(a)
            prev = a
    for j in range(2):
        for m in range(4):
            tmp = b.tensor(512 * KiB)
            b.op(f"fwd_tmp{m}", FWD, [prev, weights[4 + j]], [tmp])
            prev = tmp
    grad = prev
    for k in range(6):
        for q in range(4):
            g = b.tensor(int(512 * math.ceil(2 ** (14 + 6 * rng.random()) / 512)))
            ins = [grad]
            if k >= 2:
                j = 5 - k
                ins += [acts[6 * j + m] for m in range(6) if m % 4 == q]
            b.op(f"bwd_op{q}", BWD, ins, [g])
            grad = g
    for q in range(8):
        tmp = b.tensor(4 * KiB)
        b.op(f"opt_op{q % 4}", OPT, ([grad] if q == 0 else []) + [weights[q]], [tmp])
    static_bytes = 8 * MiB
    total_act = sum(act_sizes)
    budget = static_bytes + (total_act // 2 // 512) * 512
    return b.finish("C1-tiny", static_bytes=static_bytes, t_iter=1e-3, bw=50e9, budget=budget,
                    groups_fwd=6, groups_bwd=6, omega=1.0,
                    meta=dict(config="tiny synthetic eager trace: 64 ops, 24 activation tensors (4 KB-4 MB)",
                              seed=seed, total_act=total_act))


# ----------------------------------------------------------------------- transformers
@dataclasses.dataclass
class ModelShape:
    arch: str  # "gpt2" | "llama"
    layers: int
    hidden: int
    heads: int
    ffn: int
    vocab: int
    batch: int
    seq: int
    params: float  # parameter count (for M_0 and the FLOP model)
    static_bytes_per_param: float
    ce_chunk: int  # tokens per cross-entropy chunk (lm head chunking)


def _transformer(shape: ModelShape, name: str, budget_rule, config: str) -> Trace:
    """Eager trace of one training iteration of a decoder-only transformer.

    FWD per layer follows the PyTorch eager op sequence for the architecture; each
    FWD op declares the tensors autograd saves for it.  BWD emits, per FWD op in
    reverse order, a grad-input op (reads the upstream grad and the op's saved
    tensors, produces the downstream grad) and a grad-weight/accumulate op (reads
    the upstream grad and the op's saved tensors).  OPT: fused optimizer ops over
    static state.
    """
    bsz, s, h, H, f, V = shape.batch, shape.seq, shape.hidden, shape.heads, shape.ffn, shape.vocab
    bs = bsz * s
    B = _Builder()
    n_w = 8
    weights = [B.tensor(512 * KiB, static=True) for _ in range(n_w)]
    fwd_ops: List[Tuple[int, List[int], int]] = []  # (op index, saved tensors, grad-size)

    def fop(opname, ins, outs, saved, grad_bytes):
        i = B.op(opname, FWD, ins + [weights[len(fwd_ops) % n_w]], outs)
        fwd_ops.append((i, list(saved), grad_bytes))
        return i

    def T(nbytes, dtype="bf16"):
        return B.tensor(nbytes, dtype)

    tok = B.tensor(bs * 8, "i64", static=True)
    x = T(bs * h * 2)
    fop("embedding", [tok], [x], [], bs * h * 2)
    for _ in range(shape.layers):
        x_in = x
        if shape.arch == "gpt2":
            ln1, m1, r1 = T(bs * h * 2), T(bs * 4, "f32"), T(bs * 4, "f32")
            fop("native_layer_norm", [x_in], [ln1, m1, r1], [x_in, m1, r1], bs * h * 2)
            qkv = T(bs * 3 * h * 2)
            fop("addmm", [ln1], [qkv], [ln1], bs * h * 2)
            sc = T(bsz * H * s * s * 2)
            fop("bmm", [qkv], [sc], [qkv], bs * 3 * h * 2)
            scm, amask = T(bsz * H * s * s * 2), T(bsz * H * s * s, "u8")
            fop("masked_fill", [sc], [scm, amask], [sc, amask], bsz * H * s * s * 2)
            pr = T(bsz * H * s * s * 2)
            fop("_softmax", [scm], [pr], [pr], bsz * H * s * s * 2)
            prd = T(bsz * H * s * s * 2)
            fop("native_dropout", [pr], [prd], [prd], bsz * H * s * s * 2)
            ctx = T(bs * h * 2)
            fop("bmm", [prd, qkv], [ctx], [prd, qkv], bsz * H * s * s * 2)
            ao = T(bs * h * 2)
            fop("addmm", [ctx], [ao], [ctx], bs * h * 2)
            ad, dm1 = T(bs * h * 2), T(bs * h, "u8")
            fop("native_dropout", [ao], [ad, dm1], [dm1], bs * h * 2)
            h1 = T(bs * h * 2)
            fop("add", [x_in, ad], [h1], [], bs * h * 2)
            ln2, m2, r2 = T(bs * h * 2), T(bs * 4, "f32"), T(bs * 4, "f32")
            fop("native_layer_norm", [h1], [ln2, m2, r2], [h1, m2, r2], bs * h * 2)
            fc = T(bs * f * 2)
            fop("addmm", [ln2], [fc], [ln2], bs * h * 2)
            g1 = T(bs * f * 2)
            fop("mul", [fc], [g1], [fc], bs * f * 2)
            g2 = T(bs * f * 2)
            fop("tanh", [g1], [g2], [g1], bs * f * 2)
            go = T(bs * f * 2)
            fop("gelu_combine", [fc, g2], [go], [g2], bs * f * 2)
            mo = T(bs * h * 2)
            fop("addmm", [go], [mo], [go], bs * f * 2)
            md, dm2 = T(bs * h * 2), T(bs * h, "u8")
            fop("native_dropout", [mo], [md, dm2], [dm2], bs * h * 2)
            x = T(bs * h * 2)
            fop("add", [h1, md], [x], [], bs * h * 2)
        else:  # llama
            n1, rs1 = T(bs * h * 2), T(bs * 4, "f32")
            fop("rms_norm", [x_in], [n1, rs1], [x_in, rs1], bs * h * 2)
            qp = T(bs * h * 2)
            fop("linear", [n1], [qp], [n1], bs * h * 2)
            kp = T(bs * h * 2)
            fop("linear", [n1], [kp], [], bs * h * 2)
            v = T(bs * h * 2)
            fop("linear", [n1], [v], [], bs * h * 2)
            q = T(bs * h * 2)
            fop("rope", [qp], [q], [], bs * h * 2)
            k = T(bs * h * 2)
            fop("rope", [kp], [k], [], bs * h * 2)
            ao, lse = T(bs * h * 2), T(bsz * H * s * 4, "f32")
            fop("flash_attention", [q, k, v], [ao, lse], [q, k, v, ao, lse], bs * h * 2)
            o = T(bs * h * 2)
            fop("linear", [ao], [o], [], bs * h * 2)
            h1 = T(bs * h * 2)
            fop("add", [x_in, o], [h1], [], bs * h * 2)
            n2, rs2 = T(bs * h * 2), T(bs * 4, "f32")
            fop("rms_norm", [h1], [n2, rs2], [h1, rs2], bs * h * 2)
            gate = T(bs * f * 2)
            fop("linear", [n2], [gate], [n2], bs * h * 2)
            up = T(bs * f * 2)
            fop("linear", [n2], [up], [], bs * h * 2)
            sl = T(bs * f * 2)
            fop("silu", [gate], [sl], [gate], bs * f * 2)
            act = T(bs * f * 2)
            fop("mul", [sl, up], [act], [sl, up], bs * f * 2)
            dn = T(bs * h * 2)
            fop("linear", [act], [dn], [act], bs * f * 2)
            x = T(bs * h * 2)
            fop("add", [h1, dn], [x], [], bs * h * 2)
    # final norm + chunked lm head / cross entropy
    if shape.arch == "gpt2":
        xf, mf, rf = T(bs * h * 2), T(bs * 4, "f32"), T(bs * 4, "f32")
        fop("native_layer_norm", [x], [xf, mf, rf], [x, mf, rf], bs * h * 2)
    else:
        xf, rf = T(bs * h * 2), T(bs * 4, "f32")
        fop("rms_norm", [x], [xf, rf], [x, rf], bs * h * 2)
    n_chunks = max(1, s // shape.ce_chunk)
    ct = bsz * (s // n_chunks)
    losses = []
    for c in range(n_chunks):
        lg = T(ct * V * 2)
        fop("linear", [xf], [lg], [xf], bs * h * 2 if c == 0 else ct * V * 2)
        lp = T(ct * V * 2)
        fop("log_softmax", [lg], [lp], [lp], ct * V * 2)
        ls = T(512, "f32")
        fop("nll_loss", [lp], [ls], [], ct * V * 2)
        losses.append(ls)
    loss = T(512, "f32")
    fop("sum", losses, [loss], [], 512)
    # backward: mirror of the forward op list
    grad = loss
    for (i_f, saved, gbytes) in reversed(fwd_ops):
        fname = B.ops[i_f][0]
        g = B.tensor(gbytes)
        B.op(fname + "_backward", BWD, [grad] + saved, [g])
        B.op(fname + "_grad_acc", BWD, [grad] + saved, [])
        grad = g
    # optimizer: fused per-group ops on static state (plus tiny scalar temps)
    for q in range(8):
        tmp = B.tensor(512, "f32")
        B.op(["_foreach_mul_", "_foreach_add_", "_foreach_addcmul_", "_foreach_sqrt"][q % 4], OPT,
             ([grad] if q == 0 else []) + [weights[q % n_w]], [tmp])
    static_bytes = int(round(shape.params * shape.static_bytes_per_param / 512)) * 512
    # synthetic T_iter: FLOP model (6 P tokens + 6 L b s^2 h) at half the measured bf16 peak
    flops = 6 * shape.params * bs + 6 * shape.layers * bsz * s * s * h
    t_iter = flops / (0.5 * B200_BF16_TFLOPS)
    saved_total = 0  # sum of sizes of every produced FWD tensor autograd keeps (peak estimate)
    saved_set = set()
    for (_, saved, _) in fwd_ops:
        saved_set.update(saved)
    saved_total = sum(B.nbytes[t] for t in saved_set if not B.static[t])
    budget = int(budget_rule(static_bytes, saved_total)) // 512 * 512
    tr = B.finish(name, static_bytes=static_bytes, t_iter=t_iter, bw=50e9, budget=budget,
                  groups_fwd=shape.layers, groups_bwd=shape.layers, omega=1.0,
                  meta=dict(config=config, shape=dataclasses.asdict(shape), saved_total=saved_total))
    return tr


def gpt2_xl(seq: int = 1024, batch: int = 8) -> Trace:
    """C2: GPT-2 1.5B (L 48, h 1600, 25 heads, ffn 6400, vocab 50257), seq 1024, b 8,
    HBM budget = 50% of the no-swap peak estimate (static + every saved activation)."""
    shp = ModelShape("gpt2", 48, 1600, 25, 6400, 50257 + 47, batch, seq, 1.558e9, 16.0, seq)
    return _transformer(shp, "C2-gpt2-1.5b", lambda m0, act: 0.5 * (m0 + act),
                        "GPT-2 1.5B single-layer-stack activation trace, seq 1024, HBM budget 50% of peak, 1 B200")


def llama2_7b(seq: int = 4096, batch: int = 18, budget: Optional[int] = None) -> Trace:
    """C3: Llama-2 7B bf16, seq 4096, b 18 (about 2x HBM oversubscription);
    M_0 = bf16 params + grads (ZeRO-2 shards the optimizer)."""
    shp = ModelShape("llama", 32, 4096, 32, 11008, 32000, batch, seq, 6.74e9, 4.0, 2048)
    rule = (lambda m0, act: budget) if budget is not None else (lambda m0, act: B200_HBM_BYTES - 8 * GiB)
    return _transformer(shp, "C3-llama2-7b", rule,
                        "Llama-2 7B trace bf16 seq 4096, 2x HBM oversubscription, swap overlap with compute, 1 B200")


def llama2_7b_2x(batch: int = 6) -> Trace:
    """C3 sized to one box's host RAM: Llama-2 7B bf16, seq 4096, batch b, HBM budget
    = half the no-swap peak estimate (static + every saved activation), i.e. 2x oversubscription of
    the budget.  b = 6: peak0 141 GiB, budget 70 GiB, the SEEDED best swaps ~106 GB each way, which
    fits the 0.6 x ~206 GB pinnable host RAM of the pool's single-socket B200 boxes (b = 18, the
    2x-of-physical-HBM reading, would need ~300 GB pinned)."""
    shp = ModelShape("llama", 32, 4096, 32, 11008, 32000, batch, 4096, 6.74e9, 4.0, 2048)
    return _transformer(shp, f"C3-llama2-7b-b{batch}-2x", lambda m0, act: 0.5 * (m0 + act),
                        "Llama-2 7B trace bf16 seq 4096, 2x HBM oversubscription, swap overlap with compute, 1 B200")


def llama2_13b(seq: int) -> Trace:
    """C4: Llama-2 13B, b 1, seq 2048 or 8192, budget 80 GiB (A100-80GB class)."""
    shp = ModelShape("llama", 40, 5120, 40, 13824, 32000, 1, seq, 13.0e9, 4.0, 2048)
    return _transformer(shp, f"C4-llama2-13b-s{seq}", lambda m0, act: 80 * GiB,
                        "dynamic operator sequence: Llama-2 13B trace switching seq length 2048<->8192 mid-run")


def llama2_7b_rank(batch: int = 4) -> Trace:
    """C5 per-rank trace: Llama-2 7B, s 4096, b 4; budget = M_0 + activations/4 (4x ratio)."""
    shp = ModelShape("llama", 32, 4096, 32, 11008, 32000, batch, 4096, 6.74e9, 2.25, 2048)
    return _transformer(shp, "C5-llama2-7b-rank", lambda m0, act: m0 + act / 4,
                        "8xB200 per-rank swapping at 4x model-to-HBM ratio, 10^5 candidate policies sharded")


CONFIGS = {
    "C1": tiny,
    "C2": gpt2_xl,
    "C3": llama2_7b,
    "C3h": llama2_7b_2x,
    "C4a": lambda: llama2_13b(2048),
    "C4b": lambda: llama2_13b(8192),
    "C5": llama2_7b_rank,
}

# SEEDED candidate sets per config: flip probability 2%, per-config seed.
SEEDED = {
    "C1": dict(seed=1, flip_thr=int(0.02 * 2 ** 64)),
    "C2": dict(seed=2, flip_thr=int(0.02 * 2 ** 64)),
    "C3": dict(seed=3, flip_thr=int(0.02 * 2 ** 64)),
    "C4": dict(seed=4, flip_thr=int(0.02 * 2 ** 64)),
    "C5": dict(seed=5, flip_thr=int(0.02 * 2 ** 64)),
}


def random_trace(seed: int, n_layers: int = 3, ops_per_layer: int = 3, max_kib: int = 64,
                 bw: float = 1e9, t_iter: float = 1e-3) -> Trace:
    """Small random traces for brute-force checks: random saved-activation sizes,
    random reuse patterns, random group counts."""
    rng = np.random.default_rng(seed)
    b = _Builder()
    w = b.tensor(512, static=True)
    acts: List[List[int]] = []
    prev = None
    for j in range(n_layers):
        layer = []
        for m in range(ops_per_layer):
            a = b.tensor(512 * int(rng.integers(1, 2 * max_kib + 1)))
            b.op(f"f{int(rng.integers(0, 4))}", FWD, ([prev] if prev is not None else []) + [w], [a])
            layer.append(a)
            prev = a
        acts.append(layer)
    grad = prev
    for j in reversed(range(n_layers)):
        for m in range(ops_per_layer):
            g = b.tensor(512 * int(rng.integers(1, 9)))
            ins = [grad]
            ins += [a for a in acts[j] if rng.random() < 0.6 or m == ops_per_layer - 1 and a == acts[j][0]]
            b.op(f"b{int(rng.integers(0, 4))}", BWD, sorted(set(ins), key=ins.index), [g])
            grad = g
    if rng.random() < 0.5:
        b.op("opt", OPT, [grad, w], [b.tensor(512)])
    nf = n_layers * ops_per_layer
    gf = int(rng.integers(1, nf + 1))
    gb = int(rng.integers(1, nf + 1))
    static = 512 * int(rng.integers(1, 64))
    total = sum(b.nbytes[t] for L in acts for t in L)
    return b.finish(f"rand{seed}", static_bytes=static, t_iter=t_iter, bw=bw,
                    budget=static + total // 2 // 512 * 512, groups_fwd=gf, groups_bwd=gb, omega=1.0,
                    meta=dict(seed=seed))
