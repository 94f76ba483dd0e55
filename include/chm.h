/*
 * chm.h -- C ABI of the B200-native Chameleon swap hot path (arxiv 2509.11076).
 *
 * Two parts (BASELINE.json north_star):
 *   (X) policy execution: descriptor-driven batched swap-out / swap-in of activation blocks
 *       between HBM and mapped pinned host memory on a dedicated swap stream, event-fenced
 *       against the compute stream, fired at operator indices of the
 *       profiled eager operator sequence;
 *   (V) policy evaluation: replay of the operator sequence's alloc/free/swap events for many
 *       candidate swap sets -> per-operator footprint, peak HBM, estimated stall, argmin
 *       (P:315-340 simulator, P:421 best-of-n).
 * Host steps (recording, sequence-change detection, trace build, triggering) sit behind the
 * same ABI.  Citations "P:<line>" are PAPER.md lines; "§8(c).k" are SURVEY.md readings,
 * restated in DESIGN.md §"Readings".
 *
 * Conventions (all calls):
 *   - Every call returns chm_status: CHM_OK (0) or a negative code.  No C++ exception
 *     crosses the ABI.  chm_last_error() returns a thread-local message for the last failure.
 *   - Pointers marked "host" are host memory; "device" are CUDA device pointers (or mapped
 *     pinned host pointers usable by the device).  Inputs are borrowed for the duration of the
 *     call; the library copies what it keeps.
 *   - A chm_ctx is single-owner and not thread-safe: one ctx per device / rank.
 *   - No call on the hot path synchronises the host with the device.
 */
#ifndef CHM_H
#define CHM_H

#include <stddef.h>
#include <stdint.h>

#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t chm_status;
enum {
  CHM_OK = 0,
  CHM_E_INVAL = -1,      /* invalid argument; *err_index names the offending item if given */
  CHM_E_PARSE = -2,      /* malformed trace file (chm_trace_load); *err_offset = byte offset  */
  CHM_E_STATE = -3,      /* call not valid in the ctx's current state                        */
  CHM_E_NOMEM = -4,      /* host or device allocation failed                                  */
  CHM_E_CUDA = -5,       /* a CUDA runtime call failed; message has cudaGetErrorString        */
  CHM_E_INFEASIBLE = -6, /* reserved for the greedy generator (Algo. 2 "Raise Error")  */
  CHM_E_NOKERNEL = -7    /* the library was built without a kernel image for this device      */
};

typedef enum { CHM_FWD = 0, CHM_BWD = 1, CHM_OPT = 2 } chm_phase;
typedef enum { CHM_WARMUP = 0, CHM_GENPOLICY = 1, CHM_STABLE = 2 } chm_stage; /* Algo. 1  */

typedef struct chm_ctx chm_ctx;
typedef struct chm_trace chm_trace;

/* ------------------------------------------------------------------------------ config */
typedef struct {
  uint32_t m, n;              /* Algo. 1 stable iterations before GenPolicy / Stable;
                                 defaults 2, 5                                      */
  double len_tol, cos_tol;    /* Algo. 1 thresholds, defaults 0.05 / 0.95 */
  uint32_t cos_mode;          /* 0: positional cosine of zero-padded token vectors (default,
                                 reading Q1); 1: cosine of token-count histograms    */
  uint32_t detect_bytes;      /* 1: also require |sum bytes - prev| / max < len_tol (reading
                                 Q4, opt-in); 0: paper-literal (default)                     */
  int32_t device;             /* CUDA device ordinal this ctx drives; -1: host-only ctx
                                 (profiler, detection, trace build and executor tables only;
                                 eval / swap calls return CHM_E_STATE)                       */
  uint64_t host_arena_bytes;  /* pinned + mapped host arena for swapped blocks (0: none)      */
  uint32_t swap_ctas;         /* CTAs of the swap copy kernel (0: default 8: the link is full at
                                 4, fewer CTAs steal less from overlapped compute)           */
  uint32_t eval_ctas_per_sm;  /* resident CTAs per SM for the replay kernel (0: auto)        */
  uint32_t match_window;      /* executor: max recorded ops skipped when aligning a run-time
                                 op to the recorded sequence (0: 32)                         */
  uint32_t time_batches;      /* 1: time every swap batch's copy with CUDA events            */
  uint64_t ce_min_bytes;      /* CHM_SWAP_AUTO threshold (0: 4 MiB)                          */
  uint32_t swap_variant;      /* swap kernel: 0 16 B ld/st (default), 1 + L2::256B prefetch
                                 on loads, 2 TMA bulk copies staged through shared memory
                                 (16 B-aligned batches; others fall back to 0)              */
  uint32_t arena_mode;        /* host arena allocation: CHM_ARENA_AUTO (0) = REGISTER;
                                 CHM_ARENA_HOSTALLOC: cudaHostAlloc(Mapped|Portable), first
                                 touch; CHM_ARENA_REGISTER: mmap + MPOL_PREFERRED node
                                 arena_numa + THP + MADV_DONTFORK + parallel pre-fault +
                                 cudaHostRegister(Mapped|Portable)                           */
  int32_t arena_numa;         /* REGISTER: -1 (default) the GPU's node (its PCIe device's
                                 sysfs numa_node; no binding when that is -1), -2 no binding,
                                 >= 0 prefer that node (falls back to others when full)     */
  uint32_t arena_threads;     /* REGISTER: pre-fault threads (0: min(cores, 32))             */
} chm_config;
enum { CHM_ARENA_AUTO = 0, CHM_ARENA_HOSTALLOC = 1, CHM_ARENA_REGISTER = 2 };

/* fills the paper's defaults */
void chm_config_default(chm_config *cfg);

/* Creates a context (*out, freed by chm_destroy).  A device ctx (cfg->device >= 0) checks for an
 * sm_100 device (else CHM_E_NOKERNEL), loads every kernel of the library now (so the first
 * evaluation or descent after a sequence change pays no module loading), creates its event rings
 * and, if cfg->host_arena_bytes > 0, pins the host arena.  CHM_E_INVAL on a bad config,
 * CHM_E_NOMEM / CHM_E_CUDA when an allocation or CUDA call fails (nothing is left allocated). */
chm_status chm_create(const chm_config *cfg, chm_ctx **out);
void chm_destroy(chm_ctx *ctx);
const char *chm_last_error(void);
/* library version string and the CUDA arch it was compiled for ("sm_100a") */
const char *chm_build_info(void);

/* ---------------------------------------------------------------- profiler hook (a1, a8) */
/* Lightweight-mode tokenisation: an integer per operator name, 1, 2, ... in order
 * of first appearance within this ctx; stable for the ctx lifetime. */
chm_status chm_tokenize(chm_ctx *ctx, const char *name, int32_t *token);

typedef struct {
  uint64_t id;     /* storage data_ptr this iteration (may be reused after a free)   */
  int64_t nbytes;  /* allocated block bytes                                          */
  uint8_t dtype;   /* small dtype code (feature field)                         */
} chm_tensor_ref;

typedef struct {
  int32_t token;                 /* >= 1                                               */
  uint8_t phase;                 /* chm_phase; phases never interleave: FWD* BWD* OPT* */
  uint32_t n_in, n_out, n_free;
  const chm_tensor_ref *in;      /* host: tensors read by the op                       */
  const chm_tensor_ref *out;     /* host: tensors allocated by the op                  */
  const uint64_t *freed;         /* host: ids whose refcount reached 0 after the op    */
  int64_t live_bytes;            /* measured allocator bytes at the op, or -1          */
} chm_op_record;

typedef struct { uint64_t dev, host_off, nbytes; } chm_swap_desc; /* 24 B */

typedef struct {                 /* library-owned; valid until the next chm_record_op  */
  uint32_t n_swap_out;
  const chm_swap_desc *swap_out; /* issue (chm_swap_out) right after this op           */
  const uint32_t *swap_out_item;
  uint32_t n_release;
  const uint32_t *release_item;  /* policy items whose device block may be reclaimed after
                                    this op, once the swap stream reached the out batch
                                    (chm_item_wait on the compute stream)      */
  uint32_t n_swap_in;
  const chm_swap_desc *swap_in;  /* dev == 0: the caller allocates nbytes on the compute
                                    stream, sets dev, then calls chm_swap_in   */
  const uint32_t *swap_in_item;
  uint32_t n_wait;
  const uint32_t *wait_item;     /* compute must wait for these swap-ins before this op */
} chm_actions;

/* Records one dispatched operator (P:219 hook).  Lightweight mode appends the token
 * (P:221); Detailed mode (stage GenPolicy, or forced with chm_set_detailed) also records
 * tensors, frees and live bytes.  If a policy is installed, App. A tensor
 * features are updated and the op's swap actions are returned in *actions (nullable). */
chm_status chm_record_op(chm_ctx *ctx, const chm_op_record *op, chm_actions *actions);
/* Lightweight mode in bulk: appends n operator tokens (and their phases) to the current
 * iteration, as n chm_record_op calls without tensors would -- a hook can buffer an iteration's
 * tokens and hand them over once.  An iteration started this way is recorded Lightweight (the
 * ctx's Detailed request for it is dropped; the last Detailed record is kept).  CHM_E_STATE
 * while a non-empty policy is installed (its actions need chm_record_op per op) or when the
 * iteration already holds Detailed records; CHM_E_INVAL on a token < 1 or a phase out of
 * FWD* BWD* OPT* order (the entries before the bad one are kept). */
chm_status chm_record_tokens(chm_ctx *ctx, const int32_t *tokens, const uint8_t *phases, uint32_t n);
/* force (1) or stop forcing (0) Detailed recording from the next chm_record_op on */
chm_status chm_set_detailed(chm_ctx *ctx, int32_t detailed);

/* Ends the iteration: Algo. 1 on this iteration's token sequence vs the
 * previous one.  t_iter_s is the measured iteration time (kept as Eq. 1's T_iter if the
 * iteration was recorded in Detailed mode).  Outputs are nullable. */
chm_status chm_detect_seq_change(chm_ctx *ctx, double t_iter_s, chm_stage *stage,
                                 int32_t *changed, double *len_diff, double *cos_sim);

/* ----------------------------------------------------------------------- trace build (a3) */
typedef struct {
  int64_t hbm_budget;          /* bytes; excess = max(0, peak - budget)                 */
  int64_t static_bytes;        /* M_0: bytes live at iteration start                    */
  double t_iter_s;             /* T_iter of Eq. 1; <= 0: the recorded iteration's time */
  double bw_bytes_per_s;       /* B of Eq. 3; must be > 0                   */
  uint32_t groups_fwd, groups_bwd; /* logical layers per phase; 0: the phase's
                                  layer count, its length over the token period that best
                                  aligns the sequence with itself (stacked layers)        */
  double omega;                /* overlap factor on layer budgets, 1.0 default  */
  uint32_t f0_source;          /* 0: F0 from the recorded alloc/free events (+ static_bytes);
                                  1: Fig. 3 reconstruction: the recorded
                                  live_bytes of every op plus the bytes that were swapped out
                                  at that op (swap log of the recorded iteration)           */
} chm_trace_params;

/* Builds the evaluation trace from the last iteration recorded in Detailed mode: tensor
 * table (producer p, free op f, last FWD use a, first BWD use b), no-swap footprint F0,
 * logical layers with Eq. 1 budgets, solo swap timing r_t / s_t, the
 * swappable set in mask-bit order (ascending a_t, then production order) and the default
 * SEEDED base (swappable tensors whose window contains the first argmax of F0).  Tables are
 * uploaded to the ctx's device.  The trace is caller-owned: chm_trace_free. */
chm_status chm_trace_build(chm_ctx *ctx, const chm_trace_params *params, chm_trace **out);
void chm_trace_free(chm_trace *t);

/* Detailed records as files (SURVEY §8(b) `chm_trace_load`): one JSON
 * object per line, LF endings --
 *   line 1  {"chm_trace":1,"t_iter_s":T,"tensors":[[nbytes,dtype],...]}
 *   op      {"op":"aten::mm","tok":7,"phase":0,"in":[i,...],"out":[i,...],"free":[i,...],"live":B}
 *   swap    {"swap":[from,to,nbytes]}        (Fig. 3 swap log, to = -1: still out at the end)
 * Tensor ids index the header's table; a tensor no op outputs is live at iteration start.
 * chm_trace_load parses `text` (len bytes, borrowed) and builds a trace exactly as
 * chm_trace_build does from a recorded iteration (op names are tokenized through the ctx; "tok"
 * is used only without a name).  Malformed input: CHM_E_PARSE, *err_offset = byte offset of
 * the offending line or character, no trace.  chm_record_save writes the ctx's last Detailed
 * iteration in this format into buf (cap bytes); *len = bytes needed (CHM_E_NOMEM if > cap, so a
 * first call with cap = 0 sizes the buffer).  load(save(record)) rebuilds identical tables. */
chm_status chm_trace_load(chm_ctx *ctx, const char *text, size_t len, const chm_trace_params *params,
                          chm_trace **out, int64_t *err_offset);
chm_status chm_record_save(chm_ctx *ctx, char *buf, size_t cap, size_t *len);

typedef struct {
  uint32_t n_ops, n_tensors, n_swappable, n_layers, mask_words;
  int64_t peak0;
  uint32_t argmax0;
  int64_t budget;
} chm_trace_info;
/* sizes of a built trace (N, T, K, L, W), its no-swap peak and first argmax, the budget */
chm_status chm_trace_get_info(const chm_trace *t, chm_trace_info *info);
/* Copies host-side tables out (each pointer nullable): f0[n_ops]; per swappable k:
 * tensor[k] (production-order tensor index), nbytes[k], r[k], s[k], lin[k], lout[k];
 * per layer: start[l], count[l], bud[l]; base[mask_words]. */
chm_status chm_trace_tables(const chm_trace *t, int64_t *f0, uint32_t *tensor, int64_t *nbytes,
                            int32_t *r, int32_t *s, int32_t *lin, int32_t *lout,
                            int32_t *lay_start, int32_t *lay_count, double *bud, uint64_t *base);
/* 64-bit FNV-1a digest of everything an evaluation reads from the trace (N, K, L, W, budget, M_0,
 * B, T_iter, F0, the layer table and Eq. 1 budgets, the swappable table, the default base), in a
 * fixed field order.  Ranks that shard one candidate set (SURVEY §8(e), P:421 best-of-n) all-gather
 * it and refuse to proceed on a mismatch.  Host-only; valid on a host-only ctx's trace. */
chm_status chm_trace_digest(const chm_trace *t, uint64_t *digest);

/* ------------------------------------------------------------- policy evaluation (a4-a7) */
/* One swap item of an EXPLICIT candidate: tensor t = production-order index of a produced
 * activation (the trace's tensor numbering), released after op r, swapped in before op s. */
typedef struct {
  uint32_t t;
  int32_t r, s;
  uint32_t flags; /* generator output: bit 0 highest-score fallback, bit 1 saturated
                     swap-out (no layer had T_remaining > T_swap)                      */
} chm_item;

typedef enum {
  CHM_CAND_EXHAUSTIVE = 0, /* swap set of candidate c = bits of c; requires K <= 63        */
  CHM_CAND_SEEDED = 1,     /* bit t = base[t] ^ [f_t < flip_thr >> 48], f_t = 16-bit field
                              t mod 4 of w = mix(seed ^ (c*J + t/4)), J = ceil(K/4),
                              mix = splitmix64 finaliser (reading R-seeded)     */
  CHM_CAND_MASKS = 2,      /* device masks [count][mask_words], little-endian u64 words  */
  CHM_CAND_EXPLICIT = 3,   /* host item lists: candidate c = items[item_offsets[c] ..
                              item_offsets[c+1]); validated (CHM_E_INVAL + err_index = item):
                              t a produced activation, a_t <= r, r + 1 < s <= b_t, no
                              repeated t within a candidate                             */
  CHM_CAND_FLIP1 = 4       /* the one-bit neighbourhood of base_mask: candidate g < K = base
                              with bit g flipped, g = K: base itself (ids 0 .. K); the
                              rounds of a local search (reading R-search)     */
} chm_cand_kind;

typedef struct {
  chm_cand_kind kind;
  uint64_t first_index, count; /* global candidate ids [first_index, first_index + count)  */
  uint64_t seed, flip_thr;     /* SEEDED                                                  */
  const uint64_t *base_mask;   /* SEEDED / FLIP1, host, mask_words words; NULL: the trace's
                                  base                                                    */
  const uint64_t *masks;       /* MASKS, device [count][mask_words]                       */
  const uint64_t *item_offsets;/* EXPLICIT, host [count + 1]                              */
  const chm_item *items;       /* EXPLICIT, host                                          */
} chm_candidates;

/* argmin key, compared lexicographically (excess, stall, swapped_bytes, index): feasibility
 * first, then least estimated stall ("best runtime performance"), then least PCIe
 * traffic, then lowest id -- unique, so any reduction order gives the same winner. */
typedef struct {
  int64_t excess;
  double stall;
  int64_t swapped_bytes;
  uint64_t index;
  int64_t peak;
} chm_best; /* 40 B */

typedef struct {
  int64_t *peak;           /* device [count] or NULL                                    */
  double *stall;           /* device [count] or NULL                                    */
  int64_t *swapped;        /* device [count] or NULL                                    */
  int64_t *footprint;      /* device [count][ld] or NULL (full mode: F_P per op; the
                              entries [n_ops, ld) of a row are unspecified)            */
  uint32_t ld;             /* leading dimension of footprint, >= n_ops, even            */
  chm_best *best;          /* device, 1 element (required)                              */
  uint32_t stall_model;    /* CHM_STALL_LAYER (0, default): R-stall, the per-layer overflow;
                              CHM_STALL_TIMELINE: the max-plus serial-stream timeline of
                              chm_stall_models out[2] over the candidate's items in mask-bit
                              order at their solo (r_t, s_t); `stall` and the argmin key then
                              carry it.  Mask kinds only (EXPLICIT: CHM_E_INVAL).  Needs
                              device scratch of ~8 B x (slots of the trace's event program) per
                              resident thread, capped at 512 MiB (DESIGN.md §5 Timeline);
                              chm_release_scratch frees it                                 */
} chm_eval_out;
enum { CHM_STALL_LAYER = 0, CHM_STALL_TIMELINE = 1 };

/* Evaluates candidates on `stream` (enqueue only).  For candidate P:
 *   F_P[i] = F0[i] - sum_{t in P} S_t [r_t < i < s_t]  (event replay of §8(c).2)
 *   peak = max_i F_P[i]; stall = sum_l max(0, load_l / B - Bud_l) (§8(c).5 terms), summed as a
 *   pairwise tree: terms indexed l = 0..L-1, zero-padded to the next power of two >= L, each
 *   half summed recursively, IEEE double round-to-nearest (reading R-stall);
 * writes the per-candidate outputs and the argmin key of this batch into *best. */
chm_status chm_eval_policies(chm_ctx *ctx, const chm_trace *t, const chm_candidates *c,
                             const chm_eval_out *o, cudaStream_t stream);
/* chm_eval_policies with the index of the offending EXPLICIT item on CHM_E_INVAL */
chm_status chm_eval_policies_ex(chm_ctx *ctx, const chm_trace *t, const chm_candidates *c,
                                const chm_eval_out *o, cudaStream_t stream, int64_t *err_index);
/* Frees the device scratch the evaluation calls keep between launches (per-CTA keys, the
 * timeline kernel's end-time slots -- up to 512 MiB at 10^5 candidates --, internal peak /
 * swapped arrays, EXPLICIT item copies); the next chm_eval_policies allocates again.  Call it
 * after a planning burst (the runtime does) so the HBM goes back to training; it synchronises
 * the device (cudaFree), so not while an evaluation is in flight on another stream. */
chm_status chm_release_scratch(chm_ctx *ctx);
/* host: lexicographic min of n keys (e.g. after an all-gather across ranks) */
chm_status chm_best_reduce(const chm_best *keys, uint32_t n, chm_best *out);
/* device: the same min over n device keys into *out (device), enqueued on `stream` -- the
 * step after the NCCL all-gather of per-rank keys, without a host round trip. */
chm_status chm_best_reduce_device(chm_ctx *ctx, const chm_best *keys, uint32_t n, chm_best *out,
                                  cudaStream_t stream);
/* Steepest single-flip descent over swap masks on the device (reading R-search, DESIGN.md §3;
 * the planner's search around the evaluator), one CTA per start, all rounds on the device.
 * From each start mask a round scores the K masks that differ from it in one bit under R-stall
 * (the chm_eval_policies definitions above, bit for bit) and moves to the argmin of (excess,
 * stall, swapped, k) if its (excess, stall, swapped) is lexicographically smaller than the
 * current mask's; it stops when no flip improves or after max_rounds moves (0: score the starts
 * only).  Enqueued on `stream`; every pointer is device memory, caller-owned:
 *   starts  uint64 [n_starts][W] (W = ceil(K / 64), mask-bit order, bits >= K zero), read;
 *   ends    uint64 [n_starts][W], written: the end masks (may be `starts` itself, in place; any
 *           other overlap is CHM_E_INVAL);
 *   keys    chm_best [n_starts], written: each end mask's key, index = the start's position;
 *   rounds  int32 [n_starts] or NULL: moves made per start;
 *   best    chm_best or NULL: the min of keys (chm_best_reduce_device).
 * CHM_E_STATE on a host-only ctx; CHM_E_INVAL if the trace's tables exceed shared memory. */
chm_status chm_descend(chm_ctx *ctx, const chm_trace *t, const uint64_t *starts, uint32_t n_starts,
                       uint32_t max_rounds, uint64_t *ends, chm_best *keys, int32_t *rounds, chm_best *best,
                       cudaStream_t stream);
/* Algo. 2 policy generation on the trace's recorded iteration: MRL -> candidate
 * list with Eq. 2 scores -> simulated swap-in placement, backward search with the
 * highest-score fallback -> SetFreeTime forward search.  Writes up to
 * `cap` items (sorted by a_t, then t) and *n_items; *feasible = 0 when the MRL could not be
 * cleared (Algo. 2 "Raise Error"; the items chosen so far are still returned).  Host only.
 * C weighs size against MRE coverage in Eq. 2 (the paper gives no value); rem_scale scales
 * every layer's initial T_remaining (1 = Eq. 1 budget x omega).  Readings R-gen in DESIGN.md. */
typedef struct {
  double C;
  double rem_scale;
} chm_gen_params;
chm_status chm_generate_policy(const chm_trace *t, const chm_gen_params *p, chm_item *items,
                               uint32_t cap, uint32_t *n_items, int32_t *feasible);

/* The stall of one explicit item list (host, exact) under the stall models of reading Q11
 * (SURVEY §8(f) NEXT-4), for comparison against measured stalls; out[3]:
 *   out[0] R-stall -- what chm_eval_policies reports: pairwise sum over layers of
 *          max(0, (out_l + in_l)/B - Bud_l), out_l = bytes released in layer lay(r),
 *          in_l = bytes swapped in in layer lay(s);
 *   out[1] per-direction budgets (full-duplex link): max(0, out_l/B - Bud_l) +
 *          max(0, in_l/B - Bud_l) per layer, same pairwise order;
 *   out[2] max-plus serial-stream timeline: ops take T_iter/N each; a swap-out enters the D2H
 *          FIFO after op a_t, a swap-in the H2D FIFO before op s (not before its swap-out
 *          ended); compute waits for the swap-out after op r (the release) and for the swap-in
 *          before op b_t; the total wait.  Event order: before op i swap-ins (s = i) then waits
 *          (b_t = i); after op i swap-outs (a_t = i) then releases (r = i); item order within
 *          a kind.  Items are validated as for chm_policy_install_items. */
chm_status chm_stall_models(const chm_trace *t, const chm_item *items, uint32_t n, double *out);

/* host: the swap set of global candidate `index` as mask words (mask_words u64) */
chm_status chm_candidate_mask(const chm_trace *t, const chm_candidates *c, uint64_t index,
                              uint64_t *words);

/* ----------------------------------------------------------- policy install / trigger (a8) */
/* Installs the swap set `words` of trace t as the active policy: every selected tensor gets
 * an item {App. A feature key after op a_t, release op r_t, swap-in op s_t, host offset in
 * the arena}.  Feature tables (top-32 one-hot, 8-bit index) come from the recorded
 * iteration's token frequencies.  Subsequent chm_record_op calls return the
 * policy's actions.  When the policy's slots do not fit, a device ctx grows its arena to them
 * plus the passive-swap room it kept above the previous policy (chm_arena_reserve; pinning
 * takes time -- reserve ahead to keep it off the re-plan path); CHM_E_STATE while passive swaps
 * are outstanding. */
chm_status chm_policy_install(chm_ctx *ctx, const chm_trace *t, const uint64_t *words);
/* the same for an explicit item list (e.g. chm_generate_policy's output): releases after r,
 * swap-ins before s as given */
chm_status chm_policy_install_items(chm_ctx *ctx, const chm_trace *t, const chm_item *items,
                                    uint32_t n);
typedef struct {
  uint32_t n_items, n_matched, n_stale, n_collisions, n_demand_swap_in;
  uint64_t bytes_out, bytes_in;
} chm_exec_stats;
/* executor counters since the last install: items installed, matched swap-outs, items never
 * matched in an iteration (stale), key collisions, demand swap-ins, bytes out / in */
chm_status chm_exec_stats_get(chm_ctx *ctx, chm_exec_stats *s);

/* ------------------------------------------------ WarmUp OOM handling (NEXT-4, Algo. 3) */
/* Algo. 3, called by the allocator hook when an allocation fails in the
 * WarmUp stage (or when a policy undershoots):
 *   chm_oom_release:   steps (i)-(ii): every policy item whose swap-out was issued but whose
 *                      release point has not come yet is released now -- `compute` waits for its
 *                      swap-out batch (event record/wait, no host sync); *items (cap entries, count
 *                      in *n_items; CHM_E_INVAL if more than cap) receives them; the caller drops
 *                      their device blocks and retries.  CHM_E_STATE on a host-only ctx.
 *   chm_passive_swap:  step (iv): swaps out the resident produced tensor (reported as an output of
 *                      chm_record_op in the current iteration and not freed since; not bound to
 *                      a policy item) whose size
 *                      is closest to `need`: the smallest one of at least `need` bytes, else the
 *                      largest; ties: the older.  `exclude` (n_exclude ids, e.g. the current op's
 *                      inputs) is skipped; `only` (n_only ids, nullable = no restriction) limits
 *                      the choice to those ids (e.g. the tensors a framework can drop).  Copy goes to the arena above the installed policy's
 *                      slots (first fit); `compute` waits for it; *out names the tensor (`id`) and
 *                      a unique `handle`; the caller drops the block and retries.  CHM_E_NOMEM if
 *                      no tensor is eligible or the arena has no room.
 *   chm_passive_restore: demand swap-in (reading Q20) of `handle` into the caller's new block
 *                      `dev` before an op reads it; `compute` waits; from now on the tensor is
 *                      known by id `dev`.  dev == 0: the tensor died while out (its last use has
 *                      been recorded) -- the host copy is dropped, no copy is made.
 * The caller tracks its swapped tensors by handle (a freed block's id may be reused by a new
 * tensor at once).  Passive swaps, their restores and the policy's releases / swap-ins are
 * logged per recorded iteration: the swap log of Fig. 3's reconstruction
 * (chm_trace_params.f0_source = 1).  Policy install fails (CHM_E_STATE) while passive swaps are
 * outstanding.  Use one swap stream for passive swaps: an arena range freed by a restore is
 * rewritten only by later copies in that stream's order. */
typedef struct {
  uint64_t handle;   /* unique per passive swap                                   */
  uint64_t id;       /* the swapped tensor's id (its device address) when it left  */
  int64_t nbytes;
  uint64_t host_off; /* arena offset of the host copy                              */
  uint64_t batch;    /* swap-out batch (chm_batch_wait / query / elapsed)          */
} chm_passive;
chm_status chm_oom_release(chm_ctx *ctx, cudaStream_t compute, uint32_t *items, uint32_t cap,
                           uint32_t *n_items);
chm_status chm_passive_swap(chm_ctx *ctx, int64_t need, const uint64_t *exclude, uint32_t n_exclude,
                            const uint64_t *only, uint32_t n_only, cudaStream_t compute, cudaStream_t swap,
                            chm_passive *out);
chm_status chm_passive_restore(chm_ctx *ctx, uint64_t handle, uint64_t dev, cudaStream_t compute,
                               cudaStream_t swap);

/* ---------------------------------------------------------------- swap execution (a9-a11) */
/* The ctx's pinned, device-mapped host arena (chm_config.arena_mode); device pointer == host
 * pointer (UVA). Swapped bytes land in host DRAM; placing them on the GPU's own
 * NUMA node keeps the DMA off the inter-socket link on multi-socket 8-GPU hosts. */
chm_status chm_host_arena(chm_ctx *ctx, void **host_base, uint64_t *bytes);
/* Where the current arena lives: *numa_node (-1: not bound), *mode (CHM_ARENA_HOSTALLOC /
 * CHM_ARENA_REGISTER, -1: no arena), *pin_seconds (wall time of its allocation + pinning). Any
 * output may be NULL. */
chm_status chm_arena_placement(const chm_ctx *ctx, int32_t *numa_node, int32_t *mode, double *pin_seconds);
/* Grows the arena to at least `bytes` (e.g. to the installed policy's swapped bytes).  The old
 * arena is released: call only while no swap batch is in flight (contents are not kept);
 * CHM_E_STATE while passive swaps hold data in it. */
chm_status chm_arena_reserve(chm_ctx *ctx, uint64_t bytes);

enum {
  CHM_SWAP_KERNEL = 0, /* one multi-tensor gather/scatter kernel launch per <= 64 descriptors */
  CHM_SWAP_CE = 1,     /* baseline: one cudaMemcpyAsync per descriptor on the copy engines   */
  CHM_SWAP_AUTO = 2    /* descriptors >= chm_config.ce_min_bytes on the copy engines (256 B
                          PCIe payloads), the rest in one kernel launch (no per-copy cost)   */
};

/* Swap-out: records an event on `compute` after the last enqueued op, makes
 * `swap` wait on it, copies every descriptor's nbytes from device address dev to
 * arena + host_off, and records the batch's completion event on `swap`.  *batch receives
 * the batch id for chm_batch_wait.  Fails with CHM_E_INVAL (+ *err_index) if nbytes == 0,
 * dev == 0, host_off + nbytes exceeds the arena, or two host ranges of the batch overlap.
 * The device blocks must not be reused until the batch completes: make the consumer stream
 * wait with chm_batch_wait (custom recordStream). */
chm_status chm_swap_out(chm_ctx *ctx, const chm_swap_desc *d, uint32_t n, cudaStream_t compute,
                        cudaStream_t swap, uint32_t flags, uint64_t *batch, int64_t *err_index);
/* Swap-in: the mirror, arena + host_off -> dev, fenced the same way. */
chm_status chm_swap_in(chm_ctx *ctx, const chm_swap_desc *d, uint32_t n, cudaStream_t compute,
                       cudaStream_t swap, uint32_t flags, uint64_t *batch, int64_t *err_index);
/* Stream-ordered wait: `stream` waits for batch completion (no host polling).
 * Batch ids stay valid for the last 4096 batches of the ctx. */
chm_status chm_batch_wait(chm_ctx *ctx, uint64_t batch, cudaStream_t stream);
/* Host query (tests / diagnostics only): *done = 1 if the batch completed. */
chm_status chm_batch_query(chm_ctx *ctx, uint64_t batch, int32_t *done);
/* With chm_config.time_batches = 1, each batch's copy (after its fence wait) is bracketed by
 * timing events on the swap stream; *ms = its device duration.  CHM_E_STATE if the batch has
 * not completed or timing is off. */
chm_status chm_batch_elapsed(chm_ctx *ctx, uint64_t batch, float *ms);
/* Executor helpers for the actions of the last chm_record_op:
 *   chm_issue_swap_out: one swap-out batch of every pending swap-out item;
 *   chm_issue_swap_in:  one swap-in batch of every pending swap-in item; dev[j] is the block
 *                       the caller allocated for actions.swap_in[j] (becomes the tensor's id);
 *   chm_item_wait:      `stream` waits for the swap-out (swap_in = 0: release before reuse)
 *                       or swap-in (swap_in = 1: before the first backward use) of `item`. */
chm_status chm_issue_swap_out(chm_ctx *ctx, cudaStream_t compute, cudaStream_t swap,
                              uint32_t flags, uint64_t *batch);
chm_status chm_issue_swap_in(chm_ctx *ctx, const uint64_t *dev, cudaStream_t compute,
                             cudaStream_t swap, uint32_t flags, uint64_t *batch);
chm_status chm_item_wait(chm_ctx *ctx, uint32_t item, int32_t swap_in, cudaStream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* CHM_H */
