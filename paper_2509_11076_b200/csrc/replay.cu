// replay.cu -- policy evaluation (steps a4-a7): one candidate per warp of a persistent grid.
//
// For candidate P (§5.4 simulator; readings SURVEY §8(c).2-.6) the event
// replay gives F_P[i] = F0[i] - sum_{t in P} S_t [r_t < i < s_t].  With the solo timing of the
// trace build every release r_t is the LAST op of layer lout_t ("completed within that
// layer", reading Q6) and every swap-in s_t the FIRST op of layer lin_t (Q7), so the
// offset is constant over each logical layer l (reading R-window):
//   in_l  = sum_{t in P, lin_t = l} S_t,   out_l = sum_{t in P, lout_t = l} S_t
//   D_l   = sum_{l' <= l} in_l' - sum_{l' < l} out_l'          (exact int64)
//   F_P[i] = F0[i] + D_lay(i),   peak = max_l (max_{i in l} F0[i] + D_l)
//   load_l = in_l + out_l,       stall = pairwise sum of max(0, load_l / B - Bud_l)  (R-stall)
// -- the same integers as the event replay, in O(#flips + L) per candidate (+ O(N) to write the
// footprint row in full mode).  Not a contraction: no tensor cores.  Full mode is bound by the
// 8 B/op footprint write to HBM; search mode by the SEEDED hash decode and the layer scans.
//
// Per CTA (512 threads, 2 per SM): the trace image (layer maxima, budgets, sizes, lout/lin, F0 in
// int32 units or int64, op -> layer) is staged once into shared memory by TMA bulk copies
// (cp.async.bulk + mbarrier), and the layer sums of a reference mask R (the SEEDED base) are
// built once.  Per candidate (one warp, handed out by a global atomic counter): the items whose
// bit differs from R add signed deltas to per-layer hi/lo 32-bit shared accumulators (exact),
// warp scans over 32-layer chunks give D_l, the peak and the stall terms (xor-butterfly pairwise
// tree with IEEE _rn intrinsics: bit-identical to the oracle), lane 0 writes peak / stall /
// swapped and keeps the warp's best key; in full mode the warp streams F0 + D_lay out with 16 B
// streaming stores.  Keys: warp -> CTA -> the last CTA to finish reduces (ticket).
#include <algorithm>
#include <climits>
#include <cstring>

#include "eval_common.cuh"
#include "internal.h"

namespace chm {
namespace {

struct EvalParams {
  DevTrace tr;
  int kind;
  uint32_t stage_bytes;
  uint32_t warp_scratch;  // bytes of per-warp scratch after the image
  uint64_t first, count, seed, flip_thr;
  uint64_t base[kMaxSeededWords];
  const uint64_t *masks;
  long long *peak;
  double *stall;
  long long *swapped;
  long long *footprint;
  uint64_t ld;
  int row_pairs;  // 16 B stores per footprint row (ceil(N / 2))
  int lay_per_lane;  // E: layers per lane, next power of two >= L over 32 (1 .. 8)
  uint32_t item_table;  // bytes of the per-item delta / layer table in shared memory
  Key *partial;
  unsigned int *ticket;
  unsigned long long *work;  // candidate counter for dynamic distribution
  Key *best;
};

__device__ __forceinline__ bool cand_bit(const EvalParams &p, uint64_t g, uint64_t c, int k) {
  if (p.kind == CHM_CAND_EXHAUSTIVE) return (g >> k) & 1ull;
  if (p.kind == CHM_CAND_SEEDED) {
    const bool b = (p.base[k >> 6] >> (k & 63)) & 1ull;
    const uint64_t J = (uint64_t(p.tr.K) + 3) >> 2;
    const uint64_t w = mix64(p.seed ^ (g * J + uint64_t(k >> 2)));
    return b != (((w >> (16 * (k & 3))) & 0xffffull) < (p.flip_thr >> 48));
  }
  return (__ldg(p.masks + c * uint64_t(p.tr.W) + uint64_t(k >> 6)) >> (k & 63)) & 1ull;
}

__device__ __forceinline__ void st_cs_v2(long long *dst, long long a, long long b) {
  asm volatile("st.global.cs.v2.s64 [%0], {%1, %2};" ::"l"(dst), "l"(a), "l"(b));
}

// stages [0, bytes) of the trace image into shared memory with TMA bulk copies on one mbarrier
__device__ __forceinline__ void stage_image(unsigned char *dst, const unsigned char *src, uint32_t bytes,
                                            uint64_t *mbar) {
  const unsigned bar = static_cast<unsigned>(__cvta_generic_to_shared(mbar));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    const unsigned sdst = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    for (uint32_t off = 0; off < bytes; off += 32768u) {
      const uint32_t n = min(32768u, bytes - off);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sdst + off),
          "l"(src + off), "r"(n), "r"(bar)
          : "memory");
    }
  }
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(bar)
        : "memory");
  }
}

#ifndef CHM_EVAL_THREADS
#define CHM_EVAL_THREADS 512
#endif
#ifndef CHM_EVAL_MINB
#define CHM_EVAL_MINB 2
#endif
constexpr int kEvalThreads = CHM_EVAL_THREADS;  // 16 warps per CTA, one candidate per warp
constexpr int kChunk = 32;         // consecutive candidates per CTA-level grab

// the warp's next candidate (all lanes get it): lane 0 takes the shared lock, opens a new chunk
// of kChunk from the global counter when the CTA's is used up, takes one, releases the lock
__device__ __forceinline__ uint64_t next_candidate(unsigned long long *work, uint64_t count, int lane, int *lock,
                                                   unsigned long long *cbase, int *left) {
  unsigned long long c = 0;
  if (lane == 0) {
    while (atomicCAS(lock, 0, 1) != 0) {
    }
    __threadfence_block();
    volatile int *vl = left;
    volatile unsigned long long *vb = cbase;
    if (*vl == 0) {
      *vb = *vb >= count ? *vb : atomicAdd(work, (unsigned long long)kChunk);
      *vl = kChunk;
    }
    const int k = *vl;
    c = *vb + (unsigned long long)(kChunk - k);
    if (c < count) *vl = k - 1;  // past the end: keep answering >= count without new grabs
    __threadfence_block();
    atomicExch(lock, 0);
  }
  return __shfl_sync(0xffffffffu, c, 0);
}

__device__ __forceinline__ long long split_sum(unsigned hi, unsigned lo) {  // exact: see trace build
  return (long long)(int)hi * 65536 + (long long)(int)lo;
}

// per-layer hi/lo 32-bit accumulators of signed sizes: exact while |sum S| < 2^47, K < 32768
__device__ __forceinline__ void acc_add(unsigned *hi, unsigned *lo, int l, long long v) {
  const bool neg = v < 0;
  const unsigned long long a = (unsigned long long)(neg ? -v : v);
  const unsigned h = unsigned(a >> 16), w = unsigned(a & 0xffffull);
  atomicAdd(hi + l, neg ? 0u - h : h);
  atomicAdd(lo + l, neg ? 0u - w : w);
}

// kE: layers per lane (1, 2, 4, 8 = the next power of two >= L over 32), a template parameter so
// the per-layer passes have compile-time trip counts and keep the layer deltas in registers
// a flipped item: its precomputed signed split delta into the per-layer accumulators of the
// warp's candidate (swap-in layer lin, release layer lout)
__device__ __forceinline__ void flip_item(const uint2 *dv, const unsigned *lay2, int k, unsigned *dI_hi,
                                          unsigned *dI_lo, unsigned *dO_hi, unsigned *dO_lo) {
  const uint2 v = dv[k];
  const unsigned lz = lay2[k], li = lz & 0xffffu, lo = lz >> 16;
  atomicAdd(dI_hi + li, v.x);
  atomicAdd(dI_lo + li, v.y);
  atomicAdd(dO_hi + lo, v.x);
  atomicAdd(dO_lo + lo, v.y);
}

template <bool kFull, bool kNarrow, int kE>
__global__ void __launch_bounds__(kEvalThreads, CHM_EVAL_MINB) replay_kernel(const __grid_constant__ EvalParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ __align__(8) uint64_t s_mbar;
  __shared__ Key s_best[kEvalThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int K = p.tr.K, L = p.tr.L;
  const int PL = layer_slots(L, kE);  // per-layer arrays: layer l at layer_slot(l, kE) (internal.h)
  unsigned char *img = smem;
  const long long *mf0 = reinterpret_cast<const long long *>(img + p.tr.o_mf0);
  const double *bud = reinterpret_cast<const double *>(img + p.tr.o_bud);
  const long long *S = reinterpret_cast<const long long *>(img + p.tr.o_S);
  const unsigned short *lo_ = reinterpret_cast<const unsigned short *>(img + p.tr.o_lo);
  const unsigned short *li_ = reinterpret_cast<const unsigned short *>(img + p.tr.o_li);
  const unsigned char *f0 = img + p.tr.o_f0;  // int32 units (kNarrow) or int64
  const unsigned short *lay = reinterpret_cast<const unsigned short *>(img + p.tr.o_lay);  // 8 x layer
  // CTA tables of the reference mask R (the SEEDED base; empty for the other kinds):
  // per-layer in / out sums and their cumulative sums, and copies of the image's per-layer max F0
  // and budget, int64 / double [PL] each in the padded slot layout
  long long *s_INR = reinterpret_cast<long long *>(img + p.stage_bytes);
  long long *s_OUTR = s_INR + PL;
  long long *s_DR = s_OUTR + PL;   // D_R(l) = CIR(l) - COR(l) + OUTR(l)
  long long *s_mf0 = s_DR + PL;
  double *s_bud = reinterpret_cast<double *>(s_mf0 + PL);
  long long *s_SWR = reinterpret_cast<long long *>(s_bud + PL);  // [2] (entry 0: total bytes of R)
  unsigned *r_hi = reinterpret_cast<unsigned *>(s_SWR + 2);  // [2L] R accumulators (in, out), dense
  unsigned *r_lo = r_hi + 2 * L;                             // [2L]
  // per item k: its delta against R (-S if R has it, +S else) split as acc_add splits it, and
  // its layers lin | lout << 16 -- a flip is one 8 B + one 4 B shared load and four atomics
  uint2 *s_dv = reinterpret_cast<uint2 *>(r_lo + 2 * L);     // [K]
  unsigned *s_lay2 = reinterpret_cast<unsigned *>(s_dv + K);  // [K]
  // per-warp scratch: D[PL] (int64; padded slots in narrow mode, dense in wide mode, where the
  // image's op -> layer offsets index it) and the candidate's signed deltas vs R, split hi/lo
  // 32-bit, [PL] each in the padded slot layout
  unsigned char *wscr = reinterpret_cast<unsigned char *>(s_dv) + p.item_table + size_t(warp) * p.warp_scratch;
  long long *s_D = reinterpret_cast<long long *>(wscr);
  unsigned *dI_hi = reinterpret_cast<unsigned *>(s_D + PL);
  unsigned *dI_lo = dI_hi + PL;
  unsigned *dO_hi = dI_lo + PL;
  unsigned *dO_lo = dO_hi + PL;

  __shared__ int s_lock, s_left;
  __shared__ unsigned long long s_cbase;
  if (tid == 0) { s_lock = 0; s_left = 0; s_cbase = 0; }
  stage_image(img, p.tr.image, p.stage_bytes, &s_mbar);  // its __syncthreads publishes the above
  for (int l = tid; l < 2 * L; l += blockDim.x) { r_hi[l] = 0u; r_lo[l] = 0u; }
  for (int l = lane; l < PL; l += 32) { dI_hi[l] = 0u; dI_lo[l] = 0u; dO_hi[l] = 0u; dO_lo[l] = 0u; }
  for (int l = tid; l < L; l += blockDim.x) {
    s_mf0[layer_slot(l, kE)] = mf0[l];
    s_bud[layer_slot(l, kE)] = bud[l];
  }
  __syncthreads();
  const bool seeded = p.kind == CHM_CAND_SEEDED, flip1 = p.kind == CHM_CAND_FLIP1;
  for (int k = tid; k < K; k += blockDim.x) {
    const bool in_r = (seeded || flip1) && ((p.base[k >> 6] >> (k & 63)) & 1ull);  // R = base
    if (in_r) {
      acc_add(r_hi, r_lo, li_[k], S[k]);
      acc_add(r_hi + L, r_lo + L, lo_[k], S[k]);
    }
    const long long v = in_r ? -S[k] : S[k];
    const unsigned long long a = (unsigned long long)(v < 0 ? -v : v);
    const unsigned h = unsigned(a >> 16), w = unsigned(a & 0xffffull);
    s_dv[k] = make_uint2(v < 0 ? 0u - h : h, v < 0 ? 0u - w : w);
    s_lay2[k] = unsigned(layer_slot(li_[k], kE)) | (unsigned(layer_slot(lo_[k], kE)) << 16);
  }
  __syncthreads();
  if (warp == 0) {  // cumulative R sums over layers
    long long ci = 0, co = 0;
    for (int l0 = 0; l0 < L; l0 += 32) {
      const int l = l0 + lane;
      long long in_l = 0, out_l = 0;
      if (l < L) { in_l = split_sum(r_hi[l], r_lo[l]); out_l = split_sum(r_hi[L + l], r_lo[L + l]); }
      long long a = in_l, b = out_l;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long ya = __shfl_up_sync(0xffffffffu, a, o), yb = __shfl_up_sync(0xffffffffu, b, o);
        if (lane >= o) { a += ya; b += yb; }
      }
      if (l < L) {
        const int q = layer_slot(l, kE);
        s_INR[q] = in_l;
        s_OUTR[q] = out_l;
        s_DR[q] = (ci + a) - (co + b) + out_l;
      }
      ci += __shfl_sync(0xffffffffu, a, 31);
      co += __shfl_sync(0xffffffffu, b, 31);
    }
    if (lane == 0) s_SWR[0] = co;
  }
  __syncthreads();

  // the warp's best key lives in shared memory (lane 0 updates it once per candidate): ten
  // fewer registers in every thread of the loop
  if (lane == 0) {
    Key b0;
    b0.excess = LLONG_MAX; b0.stall = 0.0; b0.swapped = LLONG_MAX; b0.index = ~0ull; b0.peak = 0;
    s_best[warp] = b0;
  }
  // dynamic distribution in two levels: the CTA takes chunks of kChunk consecutive candidates
  // from a global counter, its warps take single candidates from the CTA's chunk under a
  // shared-memory lock (warps the scheduler favours do more, none idles at the end).  A CTA's
  // rows in flight then lie within a few consecutive rows of the footprint array: measured
  // (tools/write_locality.py) 6.4 vs 3.7 TB/s for 12.6 KB rows and 6.1 vs 5.4 for 20.9 KB
  // rows against one global atomic per candidate, which scatters an SM's rows over every row
  // in flight GPU-wide and serialises 10^5 atomics on one address.
  uint64_t c = next_candidate(p.work, p.count, lane, &s_lock, &s_cbase, &s_left);
  while (c < p.count) {
    CHM_DCHECK(c < p.count);
    const uint64_t g = p.first + c;
    // decode: only the items whose bit differs from R add a signed delta to their layers
    if (seeded) {  // one hash word per 4 items (reading R-seeded); flips are ~flip_thr rare
      const int J = (K + 3) >> 2;
      const unsigned thr16 = unsigned(p.flip_thr >> 48);
      const uint64_t gJ = g * uint64_t(J);  // word q of candidate g hashes g * J + q
      for (int q = lane; q < J; q += 32) {
        const uint64_t w = mix64(p.seed ^ (gJ + uint64_t(q)));
        unsigned f4 = 0;
#pragma unroll
        for (int e = 0; e < 4; e++) f4 |= (unsigned((w >> (16 * e)) & 0xffffull) < thr16 ? 1u : 0u) << e;
        while (f4) {
          const int e = __ffs(f4) - 1;
          f4 &= f4 - 1;
          const int k = 4 * q + e;
          if (k >= K) break;
          flip_item(s_dv, s_lay2, k, dI_hi, dI_lo, dO_hi, dO_lo);
        }
      }
    } else if (flip1) {  // one item differs from R: item g (none for g = K)
      if (lane == 0 && g < uint64_t(K)) flip_item(s_dv, s_lay2, int(g), dI_hi, dI_lo, dO_hi, dO_lo);
    } else {
      for (int k = lane; k < K; k += 32)  // R is empty: the table holds +S
        if (cand_bit(p, g, c, k)) flip_item(s_dv, s_lay2, k, dI_hi, dI_lo, dO_hi, dO_lo);
    }
    __syncwarp();
    // layer l: in_l / out_l = R sums + deltas; D_l = CI(l) - CO(l) + out_l (CI / CO cumulative)
    //   = D_R(l) + sum_{l' <= l} (din_l' - dout_{l'-1}),  D_R(l) = CIR(l) - COR(l) + OUTR(l);
    // term_l = max(0, (in_l + out_l) / B - Bud_l), pairwise tree (reading R-stall).
    // Blocked layers: lane owns E = lay_per_lane (1, 2, 4 or 8) consecutive layers E*lane + j,
    // held at slots (E + 1) lane + j of the padded per-layer arrays (layer_slot: an odd stride,
    // no bank conflicts); its partial sum, one warp scan of the lane totals, then D, peak and the
    // terms per layer.
    // The tree: 8 leaves per lane (zero past E), then the xor butterfly = the pairwise tree over
    // 256 zero-padded leaves, whose value equals R-stall's tree over the next power of two >= L.
    const int lb = kE * lane;
    const int pb = layer_slot(lb, kE);  // = (kE + 1) lane for kE > 1: the lane's padded block
    // this candidate's deltas of the lane's layers, kept in registers between the two passes
    // (kE <= 4; at kE = 8 the second pass reads them again: 32 more registers would spill)
    constexpr bool kKeep = kE <= 4;
    constexpr int kR = kKeep ? kE : 1;
    long long din[kR], dout[kR];
    long long tot = 0, lastd = 0;
#pragma unroll
    for (int j = 0; j < kE; j++) {
      const int l = lb + j, q = pb + j;
      if (l < L) {
        const long long a = split_sum(dI_hi[q], dI_lo[q]), b = split_sum(dO_hi[q], dO_lo[q]);
        if (kKeep) {
          din[j % kR] = a;
          dout[j % kR] = b;
          dI_hi[q] = 0u; dI_lo[q] = 0u; dO_hi[q] = 0u; dO_lo[q] = 0u;  // ready for the next candidate
        }
        tot += a - (j ? lastd : 0);
        lastd = b;
      } else if (kKeep) {
        din[j % kR] = 0;
        dout[j % kR] = 0;
      }
    }
    const long long prev_last = __shfl_up_sync(0xffffffffu, lastd, 1);
    tot -= lane ? prev_last : 0;
    long long inc = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    long long run = inc - tot, pk = LLONG_MIN, swd = 0, prevd = lane ? prev_last : 0;
    double t[kE];  // the lane's leaves of the pairwise tree
#pragma unroll
    for (int j = 0; j < kE; j++) {
      t[j] = 0.0;
      const int l = lb + j, q = pb + j;
      if (l < L) {
        long long a, b;
        if (kKeep) {
          a = din[j % kR];
          b = dout[j % kR];
        } else {
          a = split_sum(dI_hi[q], dI_lo[q]);
          b = split_sum(dO_hi[q], dO_lo[q]);
          dI_hi[q] = 0u; dI_lo[q] = 0u; dO_hi[q] = 0u; dO_lo[q] = 0u;  // ready for the next candidate
        }
        run += a - prevd;
        prevd = b;
        const long long d = s_DR[q] + run;
        if (kFull) s_D[kNarrow ? q : l] = d;
        pk = max(pk, s_mf0[q] + d);
        const double v = double(s_INR[q] + a + s_OUTR[q] + b);
        const double x =
            __dsub_rn(p.tr.rbw != 0.0 ? div_rn_rcp(v, p.tr.bw, p.tr.rbw) : __ddiv_rn(v, p.tr.bw), s_bud[q]);
        t[j] = x > 0.0 ? x : 0.0;
        swd += b;
      }
    }
    // the lane's kE leaves pairwise -- (t0 + t1) + (t2 + t3) ... -- equal to the 8-leaf tree with
    // zero leaves past kE (terms are >= +0, and x + 0 == x); then the xor butterfly over lanes
#pragma unroll
    for (int w = 1; w < kE; w <<= 1)
#pragma unroll
      for (int j = 0; j + w < kE; j += 2 * w) t[j] = __dadd_rn(t[j], t[j + w]);
    const double ta = t[0];
    double st = ta;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) st = __dadd_rn(st, __shfl_xor_sync(0xffffffffu, st, o));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      pk = max(pk, __shfl_xor_sync(0xffffffffu, pk, o));
      swd += __shfl_xor_sync(0xffffffffu, swd, o);
    }
    const long long swp = s_SWR[0] + swd;  // total bytes released = swapped
    if (lane == 0) {
      if (p.peak) p.peak[c] = pk;
      if (p.stall) p.stall[c] = st;
      if (p.swapped) p.swapped[c] = swp;
      Key k;
      k.excess = pk > p.tr.budget ? pk - p.tr.budget : 0;
      k.stall = st;
      k.swapped = swp;
      k.index = g;
      k.peak = pk;
      if (key_less(k, s_best[warp])) s_best[warp] = k;
    }
    if (kFull && kNarrow) {
      __syncwarp();  // s_D visible to the warp
      // F_P[i] = F0[i] + D[lay(i)] over blocks of 128 ops: lane l writes ops (2l, 2l+1) and
      // (64+2l, 65+2l), so each of the warp's two 16 B streaming stores covers 512 contiguous
      // bytes.  Per lane and block: one 16 B shared load of the four ops' F0 (int32 units,
      // swizzled by the trace build), one 8 B load of their D offsets (u16), D of each pair's
      // layer (a second load only when a pair straddles a layer boundary); no store guards but
      // in the ragged last block.  32-bit shared addresses.
      const int nb = (p.tr.N + 127) >> 7, np = p.row_pairs, unit = 1 << p.tr.f0_shift;
      const int nbf = np >> 6;  // blocks whose 64 pairs all lie in the row: no store guards
      const unsigned sD = static_cast<unsigned>(__cvta_generic_to_shared(s_D));
      unsigned sF = static_cast<unsigned>(__cvta_generic_to_shared(f0)) + 16u * lane;
      unsigned sL = static_cast<unsigned>(__cvta_generic_to_shared(img + p.tr.o_lay4)) + 8u * lane;
      long long *out = p.footprint + c * p.ld + 2 * lane;
      // per block: the four ops' F0 (16 B) and D offsets (8 B: u16 8 x layer each), D of each
      // pair (a second load only where a pair straddles a layer boundary), two 16 B stores;
      // the loop runs over whole blocks and one more iteration for the ragged last block
      for (int b = 0; b < nb; b++) {
        int f0x, f0y, f0z, f0w;
        unsigned oa, ob;
        asm("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(f0x), "=r"(f0y), "=r"(f0z), "=r"(f0w) : "r"(sF));
        asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(oa), "=r"(ob) : "r"(sL));
        const unsigned a0 = oa & 0xffffu, a1 = oa >> 16, b0 = ob & 0xffffu, b1 = ob >> 16;
        CHM_DCHECK(a0 < 8u * unsigned(PL) && a1 < 8u * unsigned(PL) && b0 < 8u * unsigned(PL) && b1 < 8u * unsigned(PL));
        long long d0, d1, d2, d3;
        asm("ld.shared.s64 %0, [%1];" : "=l"(d0) : "r"(sD + a0));
        asm("ld.shared.s64 %0, [%1];" : "=l"(d2) : "r"(sD + b0));
        d1 = d0;
        d3 = d2;
        if (a1 != a0) asm("ld.shared.s64 %0, [%1];" : "=l"(d1) : "r"(sD + a1));
        if (b1 != b0) asm("ld.shared.s64 %0, [%1];" : "=l"(d3) : "r"(sD + b1));
        const int pr = 64 * b + lane;
        // IMAD.WIDE, exact: |F0| < 2^31 units
        if (b < nbf || pr < np) st_cs_v2(out, (long long)f0x * unit + d0, (long long)f0y * unit + d1);
        if (b < nbf || pr + 32 < np) st_cs_v2(out + 64, (long long)f0z * unit + d2, (long long)f0w * unit + d3);
        sF += 512u;
        sL += 256u;
        out += 128;
      }
    } else if (kFull) {
      __syncwarp();  // s_D visible to the warp
      // F_P[i] = F0[i] + D[lay(i)], two ops per 16 B streaming store; 32-bit shared addresses
      const int np = p.row_pairs, unit = 1 << p.tr.f0_shift;
      const unsigned sD = static_cast<unsigned>(__cvta_generic_to_shared(s_D));
      unsigned sF = static_cast<unsigned>(__cvta_generic_to_shared(f0)) + (kNarrow ? 8u : 16u) * lane;
      unsigned sL = static_cast<unsigned>(__cvta_generic_to_shared(lay)) + 4u * lane;
      long long *out = p.footprint + c * p.ld + 2 * lane;
      for (int q = lane; q < np; q += 32) {
        long long fx, fy, d0, d1;
        unsigned lz;
        if (kNarrow) {
          int ux, uy;
          asm("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(ux), "=r"(uy) : "r"(sF));
          fx = (long long)ux * unit;  // IMAD.WIDE, exact: |F0| < 2^31 units
          fy = (long long)uy * unit;
        } else {
          asm("ld.shared.v2.s64 {%0, %1}, [%2];" : "=l"(fx), "=l"(fy) : "r"(sF));
        }
        asm("ld.shared.u32 %0, [%1];" : "=r"(lz) : "r"(sL));
        CHM_DCHECK((lz & 0xffffu) < 8u * unsigned(L) && (lz >> 16) < 8u * unsigned(L));
        asm("ld.shared.s64 %0, [%1];" : "=l"(d0) : "r"(sD + (lz & 0xffffu)));
        asm("ld.shared.s64 %0, [%1];" : "=l"(d1) : "r"(sD + (lz >> 16)));
        st_cs_v2(out, fx + d0, fy + d1);
        sF += kNarrow ? 256u : 512u;
        sL += 128u;
        out += 64;
      }
    }
    __syncwarp();  // scratch reuse by the next candidate
    c = next_candidate(p.work, p.count, lane, &s_lock, &s_cbase, &s_left);
  }
  // warp keys -> CTA key -> the last CTA to finish reduces all CTA keys into *best
  __syncthreads();
  __shared__ unsigned int s_last;
  if (tid == 0) {
    Key b = s_best[0];
    for (int w = 1; w < nwarps; w++) if (key_less(s_best[w], b)) b = s_best[w];
    p.partial[blockIdx.x] = b;
    __threadfence();
    const unsigned int t = atomicAdd(p.ticket, 1u);
    s_last = (t == gridDim.x - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (!s_last || warp != 0) return;
  __threadfence();
  Key b;
  b.excess = LLONG_MAX; b.stall = 0.0; b.swapped = LLONG_MAX; b.index = ~0ull; b.peak = 0;
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
    Key y;
    y.excess = __shfl_xor_sync(0xffffffffu, b.excess, o);
    y.stall = __shfl_xor_sync(0xffffffffu, b.stall, o);
    y.swapped = __shfl_xor_sync(0xffffffffu, b.swapped, o);
    y.index = __shfl_xor_sync(0xffffffffu, b.index, o);
    y.peak = __shfl_xor_sync(0xffffffffu, b.peak, o);
    if (key_less(y, b)) b = y;
  }
  if (lane == 0) {
    *p.best = b;
    *p.ticket = 0u;  // ready for the next launch
    *p.work = 0ull;
  }
}

__global__ void best_reduce_kernel(const Key *keys, uint32_t n, Key *out) {
  Key b;
  b.excess = LLONG_MAX; b.stall = 0.0; b.swapped = LLONG_MAX; b.index = ~0ull; b.peak = 0;
  for (uint32_t q = threadIdx.x; q < n; q += 32) if (key_less(keys[q], b)) b = keys[q];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Key y;
    y.excess = __shfl_xor_sync(0xffffffffu, b.excess, o);
    y.stall = __shfl_xor_sync(0xffffffffu, b.stall, o);
    y.swapped = __shfl_xor_sync(0xffffffffu, b.swapped, o);
    y.index = __shfl_xor_sync(0xffffffffu, b.index, o);
    y.peak = __shfl_xor_sync(0xffffffffu, b.peak, o);
    if (key_less(y, b)) b = y;
  }
  if (threadIdx.x == 0) *out = b;
}

}  // namespace

chm_status launch_eval(chm_ctx *ctx, const EvalLaunch &L, cudaStream_t stream) {
  const int N = L.tr.N, Ly = L.tr.L;
  const int threads = kEvalThreads;
  const bool fp = L.footprint != nullptr;
  const uint32_t stage = fp ? L.tr.full_bytes : L.tr.search_bytes;
  const int E = layers_per_lane(Ly), PL = layer_slots(Ly, E);  // padded per-layer slots (internal.h)
  const uint32_t wscr16 = uint32_t((8 * size_t(PL) + 16 * size_t(PL) + 15) & ~size_t(15));
  const size_t cta_tab = 40 * size_t(PL) + 16 + 16 * size_t(Ly);  // R tables, max F0, budget; r_hi / r_lo
  const uint32_t item_table = uint32_t((12 * size_t(L.tr.K) + 15) & ~size_t(15));
  const size_t smem = size_t(stage) + ((cta_tab + 15) & ~size_t(15)) + item_table + size_t(threads / 32) * wscr16;
  if (smem > 220 * 1024)
    CHM_FAIL(CHM_E_INVAL, "chm_eval_policies: trace image + scratch (%zu B) exceeds shared memory", smem);
  const bool narrow = L.tr.f0_narrow != 0;
  int P2 = 32, e_log = 0;
  while (P2 < Ly) { P2 *= 2; e_log++; }  // E = P2 / 32 = 2^e_log (L <= 256: e_log <= 3)
  using KernelFn = void (*)(EvalParams);
  static const KernelFn table[3][4] = {
      {replay_kernel<false, false, 1>, replay_kernel<false, false, 2>, replay_kernel<false, false, 4>,
       replay_kernel<false, false, 8>},
      {replay_kernel<true, false, 1>, replay_kernel<true, false, 2>, replay_kernel<true, false, 4>,
       replay_kernel<true, false, 8>},
      {replay_kernel<true, true, 1>, replay_kernel<true, true, 2>, replay_kernel<true, true, 4>,
       replay_kernel<true, true, 8>}};
  const int base_var = fp ? (narrow ? 2 : 1) : 0;
  auto kern = table[base_var][e_log];
  const int var = base_var * 4 + e_log;
  int per_sm = 0;
  CHM_CUDA(ensure_dyn_smem(reinterpret_cast<const void *>(kern), smem));
  if (ctx->eval_attr_smem[var] == smem) {
    per_sm = ctx->eval_per_sm[var];
  } else {
    CHM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
    ctx->eval_attr_smem[var] = smem;
    ctx->eval_per_sm[var] = per_sm;
  }
  if (per_sm < 1) CHM_FAIL(CHM_E_INVAL, "chm_eval_policies: kernel does not fit an SM");
  if (ctx->cfg.eval_ctas_per_sm) per_sm = std::min(per_sm, int(ctx->cfg.eval_ctas_per_sm));
  const uint64_t grid64 = std::min<uint64_t>(uint64_t(ctx->num_sms) * per_sm, (L.count + threads / 32 - 1) / (threads / 32));
  const int grid = int(std::max<uint64_t>(grid64, 1));
  const size_t need = size_t(grid) * sizeof(Key) + 256;
  if (ctx->eval_scratch_bytes < need) {
    if (ctx->eval_scratch) cudaFree(ctx->eval_scratch);
    ctx->eval_scratch = nullptr;
    ctx->eval_scratch_bytes = 0;
    const size_t bytes = std::max<size_t>(need, size_t(ctx->num_sms) * 32 * sizeof(Key) + 256);
    CHM_CUDA(cudaMalloc(&ctx->eval_scratch, bytes));
    CHM_CUDA(cudaMemset(ctx->eval_scratch, 0, bytes));
    ctx->eval_scratch_bytes = bytes;
  }
  EvalParams p{};
  p.tr = L.tr;
  p.kind = L.kind;
  p.stage_bytes = stage;
  p.warp_scratch = wscr16;
  p.row_pairs = (N + 1) / 2;
  p.lay_per_lane = E;
  if (E != P2 / 32) CHM_FAIL(CHM_E_STATE, "chm_eval_policies: layers per lane %d != %d", E, P2 / 32);
  p.item_table = item_table;
  p.first = L.first;
  p.count = L.count;
  p.seed = L.seed;
  p.flip_thr = L.flip_thr;
  std::memcpy(p.base, L.base, sizeof p.base);
  p.masks = L.masks;
  p.peak = reinterpret_cast<long long *>(L.peak);
  p.stall = L.stall;
  p.swapped = reinterpret_cast<long long *>(L.swapped);
  p.footprint = reinterpret_cast<long long *>(L.footprint);
  p.ld = L.ld;
  p.ticket = reinterpret_cast<unsigned int *>(ctx->eval_scratch);
  p.work = reinterpret_cast<unsigned long long *>(static_cast<char *>(ctx->eval_scratch) + 64);
  p.partial = reinterpret_cast<Key *>(static_cast<char *>(ctx->eval_scratch) + 256);
  p.best = reinterpret_cast<Key *>(L.best);
  kern<<<grid, threads, smem, stream>>>(p);
  CHM_CUDA(cudaGetLastError());
  return CHM_OK;
}

}  // namespace chm

using namespace chm;

extern "C" chm_status chm_eval_policies(chm_ctx *ctx, const chm_trace *t, const chm_candidates *c,
                                        const chm_eval_out *o, cudaStream_t stream) {
  return chm_eval_policies_ex(ctx, t, c, o, stream, nullptr);
}

extern "C" chm_status chm_eval_policies_ex(chm_ctx *ctx, const chm_trace *t, const chm_candidates *c,
                                           const chm_eval_out *o, cudaStream_t stream, int64_t *err_index) {
  CHM_NVTX("chm_eval_policies");
  if (err_index) *err_index = -1;
  if (!ctx || !t || !c || !o) CHM_FAIL(CHM_E_INVAL, "chm_eval_policies: NULL argument");
  if (!o->best) CHM_FAIL(CHM_E_INVAL, "chm_eval_policies: out.best is required");
  if (c->count == 0) CHM_FAIL(CHM_E_INVAL, "chm_eval_policies: empty candidate range");
  if (ctx->device < 0 || !t->dev_block) CHM_FAIL(CHM_E_STATE, "chm_eval_policies: host-only ctx / trace");
  if (t->device != ctx->device) CHM_FAIL(CHM_E_INVAL, "chm_eval_policies: trace on another device");
  if (o->stall_model > CHM_STALL_TIMELINE)
    CHM_FAIL(CHM_E_INVAL, "chm_eval_policies: unknown stall model %u", o->stall_model);
  const bool timeline = o->stall_model == CHM_STALL_TIMELINE;
  if (timeline && c->kind == CHM_CAND_EXPLICIT)
    CHM_FAIL(CHM_E_INVAL, "chm_eval_policies: the timeline stall model takes mask-kind candidates "
             "(EXPLICIT lists: chm_stall_models)");
  EvalLaunch L;
  L.tr = t->dev;
  L.kind = int(c->kind);
  L.first = c->first_index;
  L.count = c->count;
  switch (c->kind) {
    case CHM_CAND_EXHAUSTIVE:
      if (t->K > 63) CHM_FAIL(CHM_E_INVAL, "EXHAUSTIVE candidates need K <= 63 (K = %d)", t->K);
      if (t->K < 64 && (c->first_index + c->count - 1) >> t->K)
        CHM_FAIL(CHM_E_INVAL, "EXHAUSTIVE range exceeds 2^K (K = %d)", t->K);
      break;
    case CHM_CAND_SEEDED:
      if (t->W > kMaxSeededWords) CHM_FAIL(CHM_E_INVAL, "SEEDED candidates need K <= %d", 64 * kMaxSeededWords);
      if (c->base_mask) std::memcpy(L.base, c->base_mask, 8 * size_t(t->W));
      else if (t->W) std::memcpy(L.base, t->base.data(), 8 * size_t(t->W));
      L.seed = c->seed;
      L.flip_thr = c->flip_thr;
      break;
    case CHM_CAND_FLIP1:
      if (t->W > kMaxSeededWords) CHM_FAIL(CHM_E_INVAL, "FLIP1 candidates need K <= %d", 64 * kMaxSeededWords);
      if (c->first_index + c->count > uint64_t(t->K) + 1)
        CHM_FAIL(CHM_E_INVAL, "FLIP1 range exceeds K + 1 = %d candidates", t->K + 1);
      if (c->base_mask) std::memcpy(L.base, c->base_mask, 8 * size_t(t->W));
      else if (t->W) std::memcpy(L.base, t->base.data(), 8 * size_t(t->W));
      break;
    case CHM_CAND_MASKS:
      if (!c->masks && t->W) CHM_FAIL(CHM_E_INVAL, "MASKS candidates need a device mask array");
      L.masks = c->masks;
      break;
    case CHM_CAND_EXPLICIT:
      if (o->footprint && (o->ld < uint32_t(t->N) || (o->ld & 1u)))
        CHM_FAIL(CHM_E_INVAL, "chm_eval_policies: footprint ld %u must be even and >= n_ops %d", o->ld, t->N);
      {
        CHM_DEVICE_SCOPE(ctx->device);
        return launch_eval_explicit(ctx, t, c, o, stream, err_index);
      }
    default:
      CHM_FAIL(CHM_E_INVAL, "chm_eval_policies: unknown candidate kind %d", int(c->kind));
  }
  if (o->footprint) {
    if (o->ld < uint32_t(t->N) || (o->ld & 1u))
      CHM_FAIL(CHM_E_INVAL, "chm_eval_policies: footprint ld %u must be even and >= n_ops %d", o->ld, t->N);
    if (reinterpret_cast<uintptr_t>(o->footprint) & 15)
      CHM_FAIL(CHM_E_INVAL, "chm_eval_policies: footprint must be 16 B aligned");
  }
  L.peak = o->peak;
  L.stall = o->stall;
  L.swapped = o->swapped;
  L.footprint = o->footprint;
  L.ld = o->ld;
  L.best = o->best;
  CHM_DEVICE_SCOPE(ctx->device);
  if (!timeline) return launch_eval(ctx, L, stream);
  // timeline: the replay gives peak / swapped (footprint rows as asked), then timeline.cu the
  // stall of each candidate and the argmin key over (excess, timeline stall, swapped, index)
  const size_t arr = (8 * size_t(c->count) + 255) & ~size_t(255);
  const size_t aux = 256 + (o->peak ? 0 : arr) + (o->swapped ? 0 : arr);
  if (ctx->tl_aux_bytes < aux) {
    if (ctx->tl_aux) cudaFree(ctx->tl_aux);
    ctx->tl_aux = nullptr;
    ctx->tl_aux_bytes = 0;
    CHM_CUDA(cudaMalloc(&ctx->tl_aux, aux));
    ctx->tl_aux_bytes = aux;
  }
  char *ab = static_cast<char *>(ctx->tl_aux);
  int64_t *peak = o->peak ? o->peak : reinterpret_cast<int64_t *>(ab + 256);
  int64_t *swapped = o->swapped ? o->swapped : reinterpret_cast<int64_t *>(ab + 256 + (o->peak ? 0 : arr));
  L.peak = peak;
  L.swapped = swapped;
  L.stall = nullptr;
  L.best = reinterpret_cast<chm_best *>(ab);  // the R-stall key, not reported
  const chm_status st = launch_eval(ctx, L, stream);
  if (st != CHM_OK) return st;
  L.stall = o->stall;
  L.best = o->best;
  return launch_timeline(ctx, t, L, peak, swapped, stream);
}

extern "C" chm_status chm_best_reduce_device(chm_ctx *ctx, const chm_best *keys, uint32_t n, chm_best *out,
                                             cudaStream_t stream) {
  if (!ctx || !keys || !out || n == 0 || ctx->device < 0)
    CHM_FAIL(CHM_E_INVAL, "chm_best_reduce_device: bad argument");
  CHM_DEVICE_SCOPE(ctx->device);
  best_reduce_kernel<<<1, 32, 0, stream>>>(reinterpret_cast<const Key *>(keys), n, reinterpret_cast<Key *>(out));
  CHM_CUDA(cudaGetLastError());
  return CHM_OK;
}

extern "C" chm_status chm_release_scratch(chm_ctx *ctx) {
  if (!ctx) CHM_FAIL(CHM_E_INVAL, "chm_release_scratch: NULL ctx");
  if (ctx->device < 0) return CHM_OK;
  CHM_DEVICE_SCOPE(ctx->device);
  void **bufs[4] = {&ctx->eval_scratch, &ctx->tl_scratch, &ctx->tl_aux, &ctx->explicit_scratch};
  size_t *sizes[4] = {&ctx->eval_scratch_bytes, &ctx->tl_scratch_bytes, &ctx->tl_aux_bytes,
                      &ctx->explicit_scratch_bytes};
  for (int i = 0; i < 4; i++) {
    if (*bufs[i]) CHM_CUDA(cudaFree(*bufs[i]));  // implicit device synchronisation
    *bufs[i] = nullptr;
    *sizes[i] = 0;
  }
  return CHM_OK;
}

namespace chm {
cudaError_t preload_replay() {
  const void *k[] = {
      reinterpret_cast<const void *>(replay_kernel<false, false, 1>), reinterpret_cast<const void *>(replay_kernel<false, false, 2>),
      reinterpret_cast<const void *>(replay_kernel<false, false, 4>), reinterpret_cast<const void *>(replay_kernel<false, false, 8>),
      reinterpret_cast<const void *>(replay_kernel<true, false, 1>), reinterpret_cast<const void *>(replay_kernel<true, false, 2>),
      reinterpret_cast<const void *>(replay_kernel<true, false, 4>), reinterpret_cast<const void *>(replay_kernel<true, false, 8>),
      reinterpret_cast<const void *>(replay_kernel<true, true, 1>), reinterpret_cast<const void *>(replay_kernel<true, true, 2>),
      reinterpret_cast<const void *>(replay_kernel<true, true, 4>), reinterpret_cast<const void *>(replay_kernel<true, true, 8>),
      reinterpret_cast<const void *>(best_reduce_kernel)};
  cudaFuncAttributes a;
  for (const void *f : k) {
    const cudaError_t e = cudaFuncGetAttributes(&a, f);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}
}  // namespace chm
