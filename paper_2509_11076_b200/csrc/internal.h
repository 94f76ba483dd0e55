// internal.h -- private structures of libchm (product side; never shared with oracle/).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/chm.h"

// device-side bounds checks of the debug build (build.py --debug): a failed check prints its
// location and traps the kernel; compiled out otherwise
#ifdef CHM_DEBUG
#define CHM_DCHECK(c)                                                                  \
  do {                                                                                 \
    if (!(c)) {                                                                        \
      printf("CHM_DCHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c);                \
      __trap();                                                                        \
    }                                                                                  \
  } while (0)
#else
#define CHM_DCHECK(c) \
  do {                \
  } while (0)
#endif

// NVTX ranges around the ABI's heavier calls (visible to nsys / ncu --nvtx; a no-op without a
// tool attached).  Header-only NVTX v3 from the CUDA toolkit.
#include <nvtx3/nvToolsExt.h>
struct ChmNvtxRange {
  explicit ChmNvtxRange(const char *name) { nvtxRangePushA(name); }
  ~ChmNvtxRange() { nvtxRangePop(); }
};
#define CHM_NVTX(name) ChmNvtxRange chm_nvtx_range_(name)

namespace chm {

// ---------------------------------------------------------------------------- errors
void set_error(const char *fmt, ...);
#define CHM_FAIL(code, ...)          \
  do {                               \
    ::chm::set_error(__VA_ARGS__);   \
    return (code);                   \
  } while (0)
#define CHM_CUDA(call)                                                                  \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      CHM_FAIL(CHM_E_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
               __LINE__);                                                               \
  } while (0)

// Makes `dev` current for the scope of one ABI call and gives the caller's device back on
// return: libchm links its own CUDA runtime, but both runtimes share the driver's per-thread
// current context, so a bare cudaSetDevice would silently move PyTorch's current device.
struct DeviceGuard {
  int prev = -1;
  cudaError_t status = cudaSuccess;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) status = cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard &) = delete;
  DeviceGuard &operator=(const DeviceGuard &) = delete;
};
#define CHM_DEVICE_SCOPE(dev)            \
  ::chm::DeviceGuard chm_dev_guard_(dev); \
  CHM_CUDA(chm_dev_guard_.status)

// ---------------------------------------------------------------- detailed record
struct TensorRec {
  int64_t nbytes = 0;
  uint8_t dtype = 0;
  int32_t producer = -1;  // op index, -1 = live at iteration start
  int32_t freed = -1;     // op after which the refcount hit 0, -1 = survives
};

struct IterRecord {
  std::vector<int32_t> tokens;
  std::vector<uint8_t> phase;
  std::vector<int64_t> live_bytes;
  // per op: CSR of tensor indices it uses (in then out, deduplicated, first-seen order),
  // produced tensors, freed tensors, and which uses are inputs
  std::vector<int32_t> use_ptr{0}, use_idx;
  std::vector<uint8_t> use_is_in;
  std::vector<int32_t> out_ptr{0}, out_idx;
  std::vector<int32_t> free_ptr{0}, free_idx;
  std::vector<TensorRec> tensors;
  int64_t alloc_bytes = 0;  // total bytes allocated by ops (detect_bytes, reading Q4)
  // swap log (Fig. 3): bytes off device over ops [from, to), to = INT32_MAX while still out
  struct SwapSpan { int32_t from, to; int64_t nbytes; uint64_t id; };
  std::vector<SwapSpan> swaps;
  double t_iter = 0.0;
  bool detailed = false;
  void clear() {
    tokens.clear(); phase.clear(); live_bytes.clear();
    use_ptr.assign(1, 0); use_idx.clear(); use_is_in.clear();
    out_ptr.assign(1, 0); out_idx.clear(); free_ptr.assign(1, 0); free_idx.clear();
    tensors.clear(); alloc_bytes = 0; t_iter = 0.0; detailed = false; swaps.clear();
  }
};

// --------------------------------------------------------------------------- executor
struct Feature {  // App. A + argument slot at the latest use (reading in DESIGN.md)
  uint32_t count = 0, tag = 0;
  uint8_t dtype = 0, slot = 0;
  uint64_t stack = 0;
  bool operator==(const Feature &o) const {
    return count == o.count && tag == o.tag && dtype == o.dtype && stack == o.stack && slot == o.slot;
  }
};
struct FeatureHash {
  size_t operator()(const Feature &f) const {
    uint64_t h = f.stack * 0x9E3779B97F4A7C15ull;
    h ^= (uint64_t(f.count) << 32 | f.tag) + 0x7F4A7C15ull + (h << 6) + (h >> 2);
    return size_t(h ^ (uint64_t(f.slot) << 8 | f.dtype));
  }
};

enum ItemState : uint8_t { IT_IDLE = 0, IT_OUT = 1, IT_RELEASED = 2, IT_IN = 3 };

struct PolicyItem {
  Feature key;
  int32_t a = 0, r = 0, s = 0, b = 0;  // recorded op indices
  int64_t nbytes = 0;
  uint64_t host_off = 0;
  // per-iteration state
  uint8_t state = IT_IDLE;
  uint64_t cur_id = 0, cur_bytes = 0, out_batch = 0, in_batch = 0;
  bool has_out = false, has_in = false;
  int32_t span = -1;  // swap-log entry of the current release (Fig. 3)
  int32_t rec_tensor = -1;  // Detailed record's tensor index while released (re-aliased at swap-in)
};

struct FeatureAt {  // policy key: feature right after the recorded op a_t, and a_t itself
  Feature f;
  int32_t a = 0;
  bool operator==(const FeatureAt &o) const { return a == o.a && f == o.f; }
};
struct FeatureAtHash {
  size_t operator()(const FeatureAt &k) const {
    return FeatureHash()(k.f) ^ (size_t(uint32_t(k.a)) * 0x9E3779B1u);
  }
};

struct LiveTensor {
  Feature f;
  int32_t item = -1;  // policy item bound to this storage
};

// ---------------------------------------------------------------------------- trace
// Device image of a trace for the replay kernel: one contiguous, 16 B-aligned block staged
// into each CTA's shared memory with TMA bulk copies.  Search mode stages [0, search_bytes);
// full mode also stages the per-op part [search_bytes, full_bytes).
struct DevTrace {
  const unsigned char *image = nullptr;
  uint32_t search_bytes = 0, full_bytes = 0;
  // byte offsets inside the image
  uint32_t o_mf0 = 0;   // int64 [L]  max F0 over the ops of each logical layer
  uint32_t o_bud = 0;   // double[L]  Eq. 1 budget
  uint32_t o_S = 0;     // int64 [K]  swappable sizes (mask-bit order)
  uint32_t o_lo = 0;    // u16   [K]  lout (release layer) per swappable, mask-bit order
  uint32_t o_li = 0;    // u16   [K]  lin (swap-in layer) per swappable, mask-bit order
  uint32_t o_f0 = 0;    // no-swap footprint (full mode): if f0_narrow int32 units of 2^f0_shift B,
                        // N padded to 128 and lane-swizzled (block of 128 ops: lane l's ops 2l,
                        // 2l+1, 64+2l, 65+2l adjacent); else int64 [N] in op order
  uint32_t o_f0w = 0;   // int64 [N] no-swap footprint, global only (not staged; EXPLICIT replay)
  int32_t f0_shift = 0;
  int32_t f0_narrow = 0;
  uint32_t o_lay = 0;   // u16   [N]  8 x logical layer of each op (byte offset into D, full mode)
  uint32_t o_lay4 = 0;  // u16   [N padded to 128] 8 x layer_slot(layer of each op) (its byte
                        // offset into the warp's padded D row), lane-swizzled like F0 (narrow
                        // only): one 8 B load gives a lane's four ops' offsets
  const uint64_t *base = nullptr;
  int32_t N = 0, K = 0, L = 0, W = 0;
  double bw = 1.0;
  double rbw = 0.0;  // RN(1 / bw) when 2^-500 < bw < 2^500 (div_rn_rcp), else 0 (the kernels divide)
  int64_t budget = 0;
};

// The replay kernel's per-layer shared arrays, bank-conflict free: lane `lane` owns the E
// consecutive layers E lane .. E lane + E - 1 (E = next power of two >= L / 32, 1 .. 8), so a
// lane-blocked access with a stride of E words hits E-way bank conflicts; padding each lane's
// block by one slot (stride E + 1, odd) spreads the lanes over all 32 banks.  Layer l lives at
// layer_slot(l, E); layer_slots(L, E) entries hold all L layers.  Trace build and kernel share it.
#ifdef __CUDACC__
#define CHM_HD __host__ __device__ __forceinline__
#else
#define CHM_HD inline
#endif
CHM_HD int layers_per_lane(int L) {
  int e = 1;
  while (32 * e < L) e *= 2;
  return e;
}
CHM_HD int layer_slot(int l, int E) { return E > 1 ? l + l / E : l; }
// each kernel TU's preload: cudaFuncGetAttributes on every kernel it launches, which loads its
// code now (lazy module loading would otherwise charge the first launch -- e.g. the first
// re-plan -- a few ms); chm_create calls them for a device ctx
cudaError_t preload_replay();
cudaError_t preload_descend();
cudaError_t preload_timeline();
cudaError_t preload_explicit();
cudaError_t preload_swap();
CHM_HD int layer_slots(int L, int E) { return E > 1 ? L + (L + E - 1) / E : L; }

}  // namespace chm

struct chm_trace {
  int device = 0;
  int32_t N = 0, T = 0, K = 0, L = 0, W = 0;
  int64_t budget = 0, M0 = 0, peak0 = 0;
  int32_t argmax0 = 0;
  double bw = 1.0, t_iter = 0.0;
  std::vector<int32_t> p, f, a, b;     // per tensor
  std::vector<int64_t> S_t;            // per tensor
  std::vector<int64_t> F0;             // per op
  std::vector<int32_t> lay_start, lay_n, lay_type, lay_of_op;
  std::vector<double> bud;
  std::vector<uint32_t> sw_t;          // swappable k -> production-order tensor rank
  std::vector<int32_t> sw_tensor_idx;  // swappable k -> recorded tensor index
  std::vector<int32_t> rank_to_tensor;  // production rank -> recorded tensor index
  std::vector<int32_t> tensor_rank;     // recorded tensor index -> production rank (-1: static)
  std::vector<int64_t> sw_S;
  std::vector<int32_t> sw_r, sw_s, sw_lin, sw_lout;
  std::vector<uint64_t> base;
  // recorded iteration (for policy install: features)
  std::vector<int32_t> tokens;
  std::vector<int32_t> use_ptr, use_idx;
  std::vector<uint8_t> dtype;
  // device copies
  void *dev_block = nullptr;
  chm::DevTrace dev;
  // timeline event program (timeline.cu), built on first use by a CHM_STALL_TIMELINE eval
  void *tl_dev = nullptr;          // device: events [tl_events] (8 B each), then cost [K] doubles
  uint32_t tl_events = 0, tl_slots = 0;
  size_t tl_cost_off = 0;
  double tl_tau = 0.0;
};

struct chm_ctx {
  chm_config cfg;
  int device = 0;
  int num_sms = 148;
  // tokenizer
  std::unordered_map<std::string, int32_t> tokens;
  // profiler
  chm::IterRecord cur, last_detailed;
  std::vector<int32_t> prev_tokens;
  int64_t prev_alloc_bytes = -1;
  bool stage_init = false;
  int32_t stable_step = 0;
  chm_stage stage = CHM_WARMUP;
  bool force_detailed = false;
  std::unordered_map<uint64_t, int32_t> id_to_tensor;  // detailed recording
  // executor
  std::vector<chm::PolicyItem> items;
  std::unordered_map<chm::FeatureAt, int32_t, chm::FeatureAtHash> key_to_item;
  std::vector<int32_t> rec_tokens;  // recorded token sequence (alignment of run-time ops)
  int32_t align_cursor = 0;
  std::vector<uint8_t> op_index;   // token -> 8-bit index
  std::vector<uint32_t> op_onehot; // token -> one-hot
  std::unordered_map<uint64_t, chm::LiveTensor> live;
  std::vector<std::vector<int32_t>> release_at, swapin_at, wait_at;  // by op index
  int32_t op_cursor = 0;
  int32_t match_window = 1;
  chm_exec_stats stats{};
  std::vector<chm_swap_desc> act_out, act_in;
  std::vector<uint32_t> act_out_item, act_in_item, act_release, act_wait;
  bool policy_active = false;
  // resident tensors (for passive swaps): id -> bytes, first-seen sequence
  struct Resident { int64_t nbytes; uint64_t seq; };
  std::unordered_map<uint64_t, Resident> resident;
  uint64_t resident_seq = 0;
  // passive swaps: handle -> record; arena region [passive_base, arena_bytes), first-fit free list
  struct Passive {
    uint64_t id;
    int64_t nbytes;
    uint64_t host_off, batch;
    int32_t span;        // swap-log entry of the current iteration
    int32_t tensor;      // Detailed record's tensor index (-1: none)
    bool has_live;       // executor feature state, restored with the tensor
    chm::LiveTensor live;
  };
  std::unordered_map<uint64_t, Passive> passive;
  std::vector<std::pair<uint64_t, uint64_t>> passive_free;  // (offset, bytes), sorted by offset
  uint64_t passive_base = 0;
  uint64_t passive_next = 1;  // next handle
  // swap
  void *arena = nullptr;
  uint64_t arena_bytes = 0;      // usable bytes (as requested)
  uint64_t arena_map_bytes = 0;  // REGISTER: mapped length (2 MiB multiple)
  bool arena_registered = false;
  uint32_t arena_mode = 0, arena_threads = 0;
  int32_t arena_numa = -1;       // requested placement (chm_config.arena_numa)
  int32_t arena_node = -1;       // actual binding
  double arena_pin_s = 0;
  std::atomic<int> arena_busy{0};  // 1 while chm_arena_reserve re-pins (swap calls: CHM_E_STATE)
  std::vector<cudaEvent_t> events;  // ring of batch-completion events
  std::vector<cudaEvent_t> fences;  // ring of compute->swap fence events
  std::vector<cudaEvent_t> t0, t1;  // timing events per batch slot (time_batches)
  uint64_t next_batch = 0;
  std::vector<chm_swap_desc> kernel_descs;  // per-batch scratch (CHM_SWAP_AUTO split)
  // eval scratch
  void *eval_scratch = nullptr;  // per-CTA partial keys + ticket / work counters
  size_t eval_scratch_bytes = 0;
  void *tl_scratch = nullptr;  // timeline: per-thread slot values + internal peak / swapped / key
  size_t tl_scratch_bytes = 0;
  void *tl_aux = nullptr;      // timeline: peak / swapped the caller did not ask for + the replay's key
  size_t tl_aux_bytes = 0;
  void *explicit_scratch = nullptr;  // EXPLICIT candidates: items + offsets + keys (device)
  size_t explicit_scratch_bytes = 0;
  size_t eval_attr_smem[12] = {};  // cached kernel attribute / occupancy per variant (mode x E)
  int eval_per_sm[12] = {};
};

namespace chm {
constexpr int kEventRing = 4096;
constexpr int kMaxDescPerLaunch = 64;
constexpr int kMaxSeededWords = 64;  // SEEDED base mask in kernel params: K <= 4096

// trace.cpp: the trace build from a record (the ctx's last Detailed iteration or a loaded file)
chm_status build_trace(chm_ctx *ctx, const IterRecord &R, const chm_trace_params *P, chm_trace **out);

// executor.cpp: moves a released item's Detailed-record tensor index off its old address
void stash_record(chm_ctx *ctx, PolicyItem &it);

// Raises kernel `f`'s dynamic shared-memory limit on the current device to at least `bytes`.
// The attribute is process-wide per (device, kernel): it is only ever raised, so contexts whose
// traces need different sizes can interleave launches (lowering it under another context's
// launch made that launch fail with an invalid argument).
cudaError_t ensure_dyn_smem(const void *f, size_t bytes);

// arena.cpp: pinned + mapped host arena (sets arena, arena_bytes; frees the mapping)
int device_numa_node(int device);
chm_status arena_alloc(chm_ctx *ctx, uint64_t bytes);
void arena_free(chm_ctx *ctx);

// launchers (swap.cu / replay.cu)
chm_status launch_swap_copy(const chm_swap_desc *d, uint32_t n, char *arena, bool to_host,
                            int ctas, int variant, cudaStream_t stream);
struct EvalLaunch {
  DevTrace tr;
  int kind = 0;
  uint64_t first = 0, count = 0, seed = 0, flip_thr = 0;
  uint64_t base[kMaxSeededWords] = {};
  const uint64_t *masks = nullptr;
  int64_t *peak = nullptr;
  double *stall = nullptr;
  int64_t *swapped = nullptr;
  int64_t *footprint = nullptr;
  uint32_t ld = 0;
  chm_best *best = nullptr;
};
chm_status launch_eval(chm_ctx *ctx, const EvalLaunch &L, cudaStream_t stream);
// timeline.cu: the timeline stall of mask-kind candidates (after launch_eval wrote peak /
// swapped); writes stall and the argmin key
chm_status launch_timeline(chm_ctx *ctx, const chm_trace *t, const EvalLaunch &L, const int64_t *peak,
                           const int64_t *swapped, cudaStream_t stream);
// explicit.cu: generic replay of explicit item lists (arbitrary r, s)
chm_status launch_eval_explicit(chm_ctx *ctx, const chm_trace *t, const chm_candidates *c,
                                const chm_eval_out *o, cudaStream_t stream, int64_t *err_index);
}  // namespace chm
