// timeline.cu -- the timeline stall model in the search (reading Q11's max-plus serial-stream
// variant, chm_stall_models out[2]), one candidate per thread.
//
// The model ("NPU idle periods"): ops take tau = T_iter / N each; a swap-out
// enters the D2H FIFO after op a_t, a swap-in the H2D FIFO before op s_t; compute waits for the
// swap-out after op r_t (the release) and for the swap-in before op b_t; the stall is the total
// wait.  For a mask-kind candidate every item sits at its solo (r_t, s_t), so the sequence of
// events is the same for all candidates -- only which items are selected differs.  The host
// sorts the 4K events of all swappable items once per trace into a program (op, then the
// model's order within an op: swap-ins, waits, [op], swap-outs, releases; item order within a
// kind), with the op ticks between events folded into each event.  Every thread walks the
// program for its own candidate, skipping the items its mask does not select, with the same
// floating-point operations in the same order as the host model (bit-identical to the oracle).
//
// A release needs the end time of its item's swap-out, computed many events earlier (a wait,
// that of its swap-in).  Those values live in per-thread slots in global memory, [warp][slot]
// [lane] so a warp's accesses are one coalesced 256 B line; the host colours the item intervals
// [swap-out, release] and [swap-in, wait] over the program so that items whose intervals do not
// overlap share a slot (C2: 470 slots for 936 items).  A swap-in never waits for its own
// swap-out: the release at r_t < s_t already made `now` >= that end time, and `now` only grows,
// so max(now, h2d, out_end) = max(now, h2d) exactly.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <queue>
#include <vector>

#include "eval_common.cuh"
#include "internal.h"

namespace chm {
namespace {

enum : unsigned { TL_IN = 0, TL_WAIT = 1, TL_OUT = 2, TL_REL = 3 };  // NOP: item K (never selected)
constexpr int kTlThreads = 256;   // CTA size, one candidate per thread
constexpr int kTlThreads2 = 128;  // CTA size, two candidates per thread
constexpr int kTlCpt = 1;         // candidates per thread on the global-memory path
constexpr int kTlGroup = 4;                   // events per group = prefetch distance
constexpr unsigned kTlPrefetch = 1u << 17;    // event flag: its slot value is loaded a group ahead
constexpr size_t kTlSlotCap = 512ull << 20;  // slot scratch at most (C2's 10^5 candidates in one wave: 376 MB;
                                             // chm_release_scratch gives it back after planning)

template <bool kSm>
__device__ __forceinline__ double ld_slot(const double *a) { return kSm ? *a : __ldcg(a); }
template <bool kSm>
__device__ __forceinline__ void st_slot(double *a, double v) {
  if (kSm) *a = v;
  else __stcg(a, v);
}

// event (8 B): x = k (15 bits) | kind << 15 (2) | prefetch flag << 17 | ticks << 18 (14),
//              y = slot | slot to load for the event one group ahead << 16 (0xffff: none)
struct TlParams {
  const uint2 *ev;
  const double *cost;
  uint32_t n_ev, n_slots, ev_bytes, cost_bytes, slot_off;
  double tau;
  int kind, K, W;
  uint64_t first, count, seed, flip_thr;
  uint64_t base[kMaxSeededWords];
  const uint64_t *masks;
  const long long *peak;
  const long long *swapped;
  double *stall;
  long long budget;
  double *slots;
  Key *partial;
  unsigned int *ticket;
  Key *best;
};

// kT threads per CTA; kSm: the end-time slots live in shared memory (one warp per CTA, [slot]
// [lane] after the masks) instead of global memory -- for launches too small to fill the GPU
// (a descent round's FLIP1 neighbourhood), where one chain's latency is the launch's time;
// kC candidates per thread: their chains share the event decode and interleave (ILP)
template <int kT, bool kSm, int kC>
__global__ void __launch_bounds__(kT) timeline_kernel(const __grid_constant__ TlParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ Key s_best[kT / 32];
  __shared__ unsigned int s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, bd = blockDim.x;
  uint2 *s_ev = reinterpret_cast<uint2 *>(smem);
  double *s_cost = reinterpret_cast<double *>(smem + p.ev_bytes);
  unsigned *s_mask = reinterpret_cast<unsigned *>(smem + p.ev_bytes + p.cost_bytes);
  for (uint32_t i = tid; i < p.n_ev; i += bd) s_ev[i] = __ldg(p.ev + i);
  for (int k = tid; k <= p.K; k += bd) s_cost[k] = __ldg(p.cost + k);  // [K] = 0: NOPs
  __syncthreads();
  const uint64_t G = uint64_t(gridDim.x) * bd, gl = uint64_t(blockIdx.x) * bd + tid;
  const int W32 = 2 * p.W, MW = W32 + 1;  // + bit K's word
  char *sbase[kC];
  unsigned *wm[kC];  // 32-bit word w of candidate ci of this thread at wm[ci][w * kT]
#pragma unroll
  for (int ci = 0; ci < kC; ci++) {
    double *slot0 = kSm ? reinterpret_cast<double *>(smem + p.slot_off) + uint64_t(ci) * p.n_slots * 32 + lane
                        : p.slots + ((gl >> 5) * kC + ci) * uint64_t(p.n_slots) * 32 + (gl & 31);
    sbase[ci] = reinterpret_cast<char *>(slot0);
    wm[ci] = s_mask + ci * MW * kT + tid;
  }
  Key best = key_none();
  for (uint64_t q0 = gl; q0 * kC < p.count; q0 += G) {
#pragma unroll
    for (int ci = 0; ci < kC; ci++) {  // decode the masks (a candidate past the range: empty)
      const uint64_t c = q0 * kC + ci, g = p.first + c;
      unsigned *w_ = wm[ci];
      if (c >= p.count) {
        for (int w = 0; w < MW; w++) w_[w * kT] = 0u;
        continue;
      }
      if (p.kind == CHM_CAND_EXHAUSTIVE) {
        w_[0] = unsigned(g);
        w_[kT] = unsigned(g >> 32);
      } else if (p.kind == CHM_CAND_MASKS) {
        for (int w = 0; w < p.W; w++) {
          const uint64_t x = __ldg(p.masks + c * uint64_t(p.W) + w);
          w_[(2 * w) * kT] = unsigned(x);
          w_[(2 * w + 1) * kT] = unsigned(x >> 32);
        }
      } else {  // SEEDED / FLIP1: the base, then the flips (reading R-seeded; FLIP1 one bit)
        for (int w = 0; w < W32; w++) w_[w * kT] = unsigned(p.base[w >> 1] >> (32 * (w & 1)));
        if (p.kind == CHM_CAND_FLIP1) {
          if (g < uint64_t(p.K)) w_[(g >> 5) * kT] ^= 1u << (g & 31);
        } else {
          const uint64_t J = (uint64_t(p.K) + 3) >> 2;
          const unsigned thr16 = unsigned(p.flip_thr >> 48);
          for (uint64_t q = 0; q < J; q++) {
            const uint64_t w = mix64(p.seed ^ (g * J + q));
#pragma unroll
            for (int e = 0; e < 4; e++) {
              const unsigned k = unsigned(4 * q) + e;
              if (k < unsigned(p.K) && unsigned((w >> (16 * e)) & 0xffffull) < thr16)
                w_[(k >> 5) * kT] ^= 1u << (k & 31);
            }
          }
        }
      }
      w_[(p.K >> 5) * kT] &= ~(1u << (p.K & 31));  // bit K: the never-selected item of NOPs
    }
    double now[kC], d2h[kC], h2d[kC], st[kC], pf[kC][kTlGroup];
#pragma unroll
    for (int ci = 0; ci < kC; ci++) {
      now[ci] = d2h[ci] = h2d[ci] = st[ci] = 0.0;
#pragma unroll
      for (int j = 0; j < kTlGroup; j++) pf[ci][j] = 0.0;
    }
    for (uint32_t e0 = 0; e0 < p.n_ev; e0 += kTlGroup) {
      double nx[kC][kTlGroup], cst[kTlGroup];
      uint2 xs[kTlGroup];
      bool sel[kC][kTlGroup];
      // the group's independent work first (event decode, selection, cost, prefetch), then the
      // serial chains over `now` / the FIFOs
#pragma unroll
      for (int j = 0; j < kTlGroup; j++) {
        const uint2 x = s_ev[e0 + j];  // n_ev is a multiple of kTlGroup (NOP padding)
        xs[j] = x;
        const unsigned k = x.x & 0x7fffu, ps = x.y >> 16;
        cst[j] = s_cost[k];  // cost[K] = 0 pads the NOPs
#pragma unroll
        for (int ci = 0; ci < kC; ci++) {
          if (!kSm)  // global slots: load one group ahead (shared-memory slots are close enough)
            nx[ci][j] = ps != 0xffffu ? ld_slot<kSm>(reinterpret_cast<const double *>(sbase[ci] + (ps << 8))) : 0.0;
          sel[ci][j] = (wm[ci][(k >> 5) * kT] >> (k & 31)) & 1u;  // not selected (or a NOP: item K)
        }
      }
#pragma unroll
      for (int j = 0; j < kTlGroup; j++) {
        const uint2 x = xs[j];
        const unsigned kind = (x.x >> 15) & 3u, so = (x.y & 0xffffu) << 8;
        for (unsigned t = x.x >> 18; t; t--) {  // ops between events
#pragma unroll
          for (int ci = 0; ci < kC; ci++) now[ci] = __dadd_rn(now[ci], p.tau);
        }
        CHM_DCHECK((x.y & 0xffffu) < p.n_slots);
#pragma unroll
        for (int ci = 0; ci < kC; ci++) {
          if (!sel[ci][j]) continue;
          double *sl = reinterpret_cast<double *>(sbase[ci] + so);
          if (kind == TL_IN) {  // before op s: the H2D FIFO
            const double v = __dadd_rn(h2d[ci] > now[ci] ? h2d[ci] : now[ci], cst[j]);
            h2d[ci] = v;
            st_slot<kSm>(sl, v);
          } else if (kind == TL_OUT) {  // after op a: the D2H FIFO
            const double v = __dadd_rn(d2h[ci] > now[ci] ? d2h[ci] : now[ci], cst[j]);
            d2h[ci] = v;
            st_slot<kSm>(sl, v);
          } else {  // wait (before op b: swap-in done) / release (after op r: swap-out done)
            const double v = (!kSm && (x.x & kTlPrefetch)) ? pf[ci][j] : ld_slot<kSm>(sl);
            if (v > now[ci]) {
              st[ci] = __dadd_rn(st[ci], __dsub_rn(v, now[ci]));
              now[ci] = v;
            }
          }
        }
      }
      if (!kSm) {
#pragma unroll
        for (int ci = 0; ci < kC; ci++)
#pragma unroll
          for (int j = 0; j < kTlGroup; j++) pf[ci][j] = nx[ci][j];
      }
    }
#pragma unroll
    for (int ci = 0; ci < kC; ci++) {
      const uint64_t c = q0 * kC + ci;
      if (c >= p.count) continue;
      const long long pk = p.peak[c], sw = p.swapped[c];
      if (p.stall) p.stall[c] = st[ci];
      Key kk;
      kk.excess = pk > p.budget ? pk - p.budget : 0;
      kk.stall = st[ci];
      kk.swapped = sw;
      kk.index = p.first + c;
      kk.peak = pk;
      if (key_less(kk, best)) best = kk;
    }
  }
  // thread keys -> warp -> CTA -> the last CTA to finish reduces all CTA keys into *best
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const Key y = key_shfl_xor(best, o);
    if (key_less(y, best)) best = y;
  }
  if (lane == 0) s_best[warp] = best;
  __syncthreads();
  if (tid == 0) {
    Key b = s_best[0];
    for (int w = 1; w < bd / 32; w++) if (key_less(s_best[w], b)) b = s_best[w];
    p.partial[blockIdx.x] = b;
    __threadfence();
    const unsigned int t = atomicAdd(p.ticket, 1u);
    s_last = (t == gridDim.x - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (!s_last || warp != 0) return;
  __threadfence();
  Key b = key_none();
  for (unsigned q = lane; q < gridDim.x; q += 32) {
    Key k;
    k.excess = __ldcg(&p.partial[q].excess);
    k.stall = __ldcg(&p.partial[q].stall);
    k.swapped = __ldcg(&p.partial[q].swapped);
    k.index = __ldcg(&p.partial[q].index);
    k.peak = __ldcg(&p.partial[q].peak);
    if (key_less(k, b)) b = k;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const Key y = key_shfl_xor(b, o);
    if (key_less(y, b)) b = y;
  }
  if (lane == 0) {
    *p.best = b;
    *p.ticket = 0u;
  }
}

// the event program of a trace (host, once per trace): events sorted by (op, phase, item),
// op ticks folded in, slot colouring of the item intervals
chm_status build_program(const chm_trace *tc) {
  chm_trace *t = const_cast<chm_trace *>(tc);  // the program is a cache of the immutable trace
  if (t->tl_dev) return CHM_OK;
  const int32_t K = t->K, N = t->N;
  struct Ev { int32_t op; uint8_t ph; int32_t k; };
  std::vector<Ev> ev;
  ev.reserve(4 * size_t(K));
  for (int32_t k = 0; k < K; k++) {
    const int32_t tid = t->sw_tensor_idx[size_t(k)];
    const int32_t a = t->a[size_t(tid)], b = t->b[size_t(tid)], r = t->sw_r[size_t(k)], s = t->sw_s[size_t(k)];
    if (a < 0 || b < 0 || r < a || !(r + 1 < s) || s > b || b >= N)
      CHM_FAIL(CHM_E_INVAL, "timeline: swappable %d (a %d, r %d, s %d, b %d) breaks a <= r < r + 1 < s <= b", k, a,
               r, s, b);
    ev.push_back({s, TL_IN, k});
    ev.push_back({b, TL_WAIT, k});
    ev.push_back({a, TL_OUT, k});
    ev.push_back({r, TL_REL, k});
  }
  std::sort(ev.begin(), ev.end(), [](const Ev &x, const Ev &y) {
    if (x.op != y.op) return x.op < y.op;
    if (x.ph != y.ph) return x.ph < y.ph;
    return x.k < y.k;
  });
  std::vector<uint32_t> slot_of(2 * size_t(K), 0);  // [k]: out slot, [K + k]: in slot
  std::vector<size_t> store_at(2 * size_t(K), 0);   // program index of the item's swap-out / -in
  std::priority_queue<uint32_t, std::vector<uint32_t>, std::greater<uint32_t>> free_slots;
  uint32_t n_slots = 0;
  std::vector<uint2> prog;
  prog.reserve(ev.size() + 8);
  int64_t done = 0;  // ops executed before the current event
  const uint32_t nop_k = uint32_t(K);  // mask bit K is cleared by the kernel: never selected
  std::vector<uint32_t> pf_slot;       // per program event: its slot if prefetchable, else 0xffff
  for (const Ev &e : ev) {
    int64_t ticks = int64_t(e.op) + (e.ph >= TL_OUT ? 1 : 0) - done;
    done += ticks;
    while (ticks > 0x3fff) {  // long gaps: tick-only events
      prog.push_back(make_uint2(nop_k | (0x3fffu << 18), 0u));
      pf_slot.push_back(0xffffu);
      ticks -= 0x3fff;
    }
    uint32_t slot, flag = 0;
    const size_t key = (e.ph == TL_OUT || e.ph == TL_REL) ? size_t(e.k) : size_t(K) + size_t(e.k);
    const size_t idx = prog.size();
    if (e.ph == TL_IN || e.ph == TL_OUT) {
      if (free_slots.empty()) free_slots.push(n_slots++);
      slot = free_slots.top();
      free_slots.pop();
      slot_of[key] = slot;
      store_at[key] = idx;
    } else {
      slot = slot_of[key];
      free_slots.push(slot);
      // the kernel loads the values of group G at the start of group G - 1 (before any of its
      // events run): the store must precede that group
      const size_t grp = idx / kTlGroup;
      if (grp >= 1 && store_at[key] < kTlGroup * (grp - 1)) flag = kTlPrefetch;
    }
    if (n_slots >= 0xffffu) CHM_FAIL(CHM_E_INVAL, "timeline: more than 65534 concurrent items");
    prog.push_back(make_uint2(uint32_t(e.k) | (uint32_t(e.ph) << 15) | flag | (uint32_t(ticks) << 18), slot));
    pf_slot.push_back(flag ? slot : 0xffffu);
  }
  while (prog.size() % kTlGroup) {  // whole groups
    prog.push_back(make_uint2(nop_k, 0u));
    pf_slot.push_back(0xffffu);
  }
  for (size_t i = 0; i + kTlGroup < prog.size(); i++) prog[i].y |= pf_slot[i + kTlGroup] << 16;
  for (size_t i = prog.size() >= kTlGroup ? prog.size() - kTlGroup : 0; i < prog.size(); i++) prog[i].y |= 0xffffu << 16;
  const size_t ev_bytes = (8 * prog.size() + 15) & ~size_t(15);
  std::vector<double> cost(static_cast<size_t>(K) + 1, 0.0);  // [K] = 0 for the NOP item
  for (int32_t k = 0; k < K; k++) cost[size_t(k)] = double(t->sw_S[size_t(k)]) / t->bw;  // Eq. 3, as the model
  CHM_DEVICE_SCOPE(t->device);
  void *d = nullptr;
  CHM_CUDA(cudaMalloc(&d, ev_bytes + 8 * (size_t(K) + 1)));
  cudaError_t e1 = cudaMemcpy(d, prog.data(), 8 * prog.size(), cudaMemcpyHostToDevice);
  cudaError_t e2 = cudaMemcpy(static_cast<char *>(d) + ev_bytes, cost.data(), 8 * (size_t(K) + 1), cudaMemcpyHostToDevice);
  if (e1 != cudaSuccess || e2 != cudaSuccess) {
    cudaFree(d);
    CHM_FAIL(CHM_E_CUDA, "timeline: program upload failed");
  }
  t->tl_dev = d;
  t->tl_events = uint32_t(prog.size());
  t->tl_slots = std::max<uint32_t>(n_slots, 1);
  t->tl_cost_off = ev_bytes;
  t->tl_tau = N > 0 ? t->t_iter / double(N) : 0.0;
  return CHM_OK;
}

}  // namespace

chm_status launch_timeline(chm_ctx *ctx, const chm_trace *t, const EvalLaunch &L, const int64_t *peak,
                           const int64_t *swapped, cudaStream_t stream) {
  const chm_status st = build_program(t);
  if (st != CHM_OK) return st;
  const size_t ev_bytes = t->tl_cost_off, cost_bytes = (8 * (size_t(t->K) + 1) + 15) & ~size_t(15);
  const size_t mask_words = size_t(2 * t->W + 1);  // + bit K's word
  const size_t per_thread = 8 * size_t(t->tl_slots);
  // small launches (at most one wave of one-warp CTAs, e.g. a descent round's FLIP1
  // neighbourhood): one warp per CTA with its slots in shared memory -- 23-25% less time per
  // launch there (tools/timeline_paths.py); larger ones: 256-thread CTAs, slots in global memory
  const size_t smem_sm = ev_bytes + cost_bytes + mask_words * 32 * 4 + 32 * per_thread;
  bool use_sm = false;
  int per_sm_sm = 0;
  if (smem_sm <= 220 * 1024) {
    CHM_CUDA(ensure_dyn_smem(reinterpret_cast<const void *>(timeline_kernel<32, true, 1>), smem_sm));
    CHM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_sm, timeline_kernel<32, true, 1>, 32, smem_sm));
    use_sm = per_sm_sm > 0 && L.count <= uint64_t(ctx->num_sms) * 32 * uint64_t(per_sm_sm);
  }
  if (const char *f = std::getenv("CHM_TL_SMEM"))  // measurement knob (tools/timeline_paths.py)
    use_sm = f[0] == '1' && per_sm_sm > 0;
  // global path: kC candidates per thread (CHM_TL_CPT, measurement knob; default below)
  int cpt = kTlCpt;
  if (const char *f = std::getenv("CHM_TL_CPT")) cpt = f[0] == '2' ? 2 : 1;
  const int kc = use_sm ? 1 : cpt;
  const int threads = use_sm ? 32 : (kc == 2 ? kTlThreads2 : kTlThreads);
  const size_t smem = use_sm ? smem_sm : ev_bytes + cost_bytes + size_t(kc) * mask_words * threads * 4;
  if (smem > 220 * 1024)
    CHM_FAIL(CHM_E_INVAL, "timeline: event program + masks (%zu B) exceed shared memory", smem);
  auto kern = use_sm ? timeline_kernel<32, true, 1>
                     : (kc == 2 ? timeline_kernel<kTlThreads2, false, 2> : timeline_kernel<kTlThreads, false, 1>);
  int per_sm = per_sm_sm;
  if (!use_sm) {
    CHM_CUDA(ensure_dyn_smem(reinterpret_cast<const void *>(kern), smem));
    CHM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
  }
  if (per_sm < 1) CHM_FAIL(CHM_E_INVAL, "timeline: kernel does not fit an SM");
  const uint64_t units = (L.count + kc - 1) / kc;  // threads' worth of candidates
  uint64_t grid64 = std::min<uint64_t>(uint64_t(ctx->num_sms) * per_sm, (units + threads - 1) / threads);
  size_t cap = kTlSlotCap;
  if (const char *f = std::getenv("CHM_TL_SCRATCH_MIB")) cap = size_t(std::max(1, std::atoi(f))) << 20;  // knob
  if (!use_sm) grid64 = std::min<uint64_t>(grid64, std::max<uint64_t>(1, cap / (per_thread * kc * threads)));
  grid64 = std::max<uint64_t>(1, grid64);
  const int grid = int(grid64);
  const size_t slot_bytes = use_sm ? 0 : size_t(grid) * threads * per_thread * kc;
  if (ctx->tl_scratch_bytes < slot_bytes) {
    if (ctx->tl_scratch) cudaFree(ctx->tl_scratch);
    ctx->tl_scratch = nullptr;
    ctx->tl_scratch_bytes = 0;
    CHM_CUDA(cudaMalloc(&ctx->tl_scratch, slot_bytes));
    ctx->tl_scratch_bytes = slot_bytes;
  }
  const size_t need = size_t(grid) * sizeof(Key) + 256;  // partial keys + ticket (eval scratch)
  if (ctx->eval_scratch_bytes < need) CHM_FAIL(CHM_E_STATE, "timeline: eval scratch too small");
  TlParams p{};
  p.ev = static_cast<const uint2 *>(t->tl_dev);
  p.cost = reinterpret_cast<const double *>(static_cast<const char *>(t->tl_dev) + ev_bytes);
  p.n_ev = t->tl_events;
  p.n_slots = t->tl_slots;
  p.ev_bytes = uint32_t(ev_bytes);
  p.cost_bytes = uint32_t(cost_bytes);
  p.slot_off = uint32_t(ev_bytes + cost_bytes + mask_words * 32 * 4);  // kSm (kC = 1): 16 B aligned
  p.tau = t->tl_tau;
  p.kind = L.kind;
  p.K = t->K;
  p.W = t->W;
  p.first = L.first;
  p.count = L.count;
  p.seed = L.seed;
  p.flip_thr = L.flip_thr;
  std::memcpy(p.base, L.base, sizeof p.base);
  p.masks = L.masks;
  p.peak = reinterpret_cast<const long long *>(peak);
  p.swapped = reinterpret_cast<const long long *>(swapped);
  p.stall = L.stall;
  p.budget = t->budget;
  p.slots = static_cast<double *>(ctx->tl_scratch);
  p.ticket = reinterpret_cast<unsigned int *>(ctx->eval_scratch);
  p.partial = reinterpret_cast<Key *>(static_cast<char *>(ctx->eval_scratch) + 256);
  p.best = reinterpret_cast<Key *>(L.best);
  kern<<<grid, threads, smem, stream>>>(p);
  CHM_CUDA(cudaGetLastError());
  return CHM_OK;
}

}  // namespace chm

namespace chm {
cudaError_t preload_timeline() {
  const void *k[] = {reinterpret_cast<const void *>(timeline_kernel<32, true, 1>),
                     reinterpret_cast<const void *>(timeline_kernel<kTlThreads, false, 1>),
                     reinterpret_cast<const void *>(timeline_kernel<kTlThreads2, false, 2>)};
  cudaFuncAttributes a;
  for (const void *f : k) {
    const cudaError_t e = cudaFuncGetAttributes(&a, f);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}
}  // namespace chm
