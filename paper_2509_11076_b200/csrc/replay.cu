// replay.cu -- policy evaluation (steps a4-a7): one candidate per CTA of a persistent grid.
//
// For candidate P (§5.4 simulator; readings SURVEY §8(c).2-.6):
//   d_P[r_t + 1] -= S_t, d_P[s_t] += S_t for t in P      (release after r_t, swap-in before s_t)
//   F_P = F0 + inclusive_scan(d_P)                       (per-op footprint)
//   peak = max F_P, excess = max(0, peak - budget)
//   load_l = sum_{t in P} S_t ([lin_t = l] + [lout_t = l]); stall = sum_l max(0, load_l/B - Bud_l)
// and the argmin key (excess, stall, swapped, index) ("best runtime performance").
//
// Not a contraction: no tensor cores.  The bound is the footprint write (full mode: 8 B per op
// and candidate to HBM) or the SM integer pipe / shared memory (search mode).  Per candidate:
//   zero the shared-memory delta row -> shared-memory int64 atomics for the selected items ->
//   raking scan (each thread sums E contiguous elements, E odd so 8 B accesses are bank-
//   conflict free) + warp shuffle scan of the per-thread sums + block scan of the warp sums ->
//   F0 + prefix written back in place, max-reduced -> one cp.async.bulk (TMA bulk copy engine)
//   shared->global store of the whole row, double-buffered so the next candidate's scan
//   overlaps the previous store.  Stall: warp 0, positive terms only, in ascending layer order
//   (bit-exact with the oracle's sequential sum; IEEE div/sub/add intrinsics, no contraction).
#include <algorithm>
#include <climits>
#include <cstring>

#include "internal.h"

namespace chm {
namespace {

struct Key {
  long long excess;
  double stall;
  long long swapped;
  unsigned long long index;
  long long peak;
};
static_assert(sizeof(Key) == sizeof(chm_best), "key layout");

__device__ __forceinline__ bool key_less(const Key &x, const Key &y) {
  if (x.excess != y.excess) return x.excess < y.excess;
  if (x.stall != y.stall) return x.stall < y.stall;
  if (x.swapped != y.swapped) return x.swapped < y.swapped;
  return x.index < y.index;
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {  // splitmix64 finaliser
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct EvalParams {
  DevTrace tr;
  int kind;
  int E;          // contiguous row elements per thread (odd)
  int row_ld;     // shared row stride in elements (even)
  int fp_elems;   // elements written per footprint row (even, <= ld)
  uint64_t first, count, seed, flip_thr;
  uint64_t base[kMaxSeededWords];
  const uint64_t *masks;
  long long *peak;
  double *stall;
  long long *swapped;
  long long *footprint;
  uint64_t ld;
  Key *partial;
  unsigned int *ticket;
  Key *best;
};

__device__ __forceinline__ bool cand_bit(const EvalParams &p, uint64_t g, uint64_t c, int k) {
  if (p.kind == CHM_CAND_EXHAUSTIVE) return (g >> k) & 1ull;
  if (p.kind == CHM_CAND_SEEDED) {
    const bool b = (p.base[k >> 6] >> (k & 63)) & 1ull;
    const uint64_t h = mix64(p.seed ^ mix64(g * uint64_t(p.tr.K) + uint64_t(k)));
    return b != (h < p.flip_thr);
  }
  return (__ldg(p.masks + c * uint64_t(p.tr.W) + uint64_t(k >> 6)) >> (k & 63)) & 1ull;
}

template <bool kFootprint>
__global__ void __launch_bounds__(256) replay_kernel(const __grid_constant__ EvalParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int N = p.tr.N, K = p.tr.K, L = p.tr.L;
  long long *rows = reinterpret_cast<long long *>(smem);
  long long *s_load = rows + (kFootprint ? 2 : 1) * p.row_ld;
  const int L2 = (L + 1) & ~1;
  long long *s_wtot = s_load + L2;    // [32] warp totals of the scan
  long long *s_rmax = s_wtot + 32;    // [32]
  long long *s_rsum = s_rmax + 32;    // [32]

  Key best;
  best.excess = LLONG_MAX; best.stall = 0.0; best.swapped = LLONG_MAX; best.index = ~0ull; best.peak = 0;
  int j = 0;
  for (uint64_t c = blockIdx.x; c < p.count; c += gridDim.x, j++) {
    const uint64_t g = p.first + c;
    long long *row = rows + (kFootprint ? (j & 1) * p.row_ld : 0);
    if (kFootprint && tid == 0 && j >= 2)  // the store issued 2 candidates ago read this row
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncthreads();  // (A)
    {
      int4 *r4 = reinterpret_cast<int4 *>(row);
      const int4 z = make_int4(0, 0, 0, 0);
      for (int q = tid; q < (p.row_ld >> 1); q += blockDim.x) r4[q] = z;
      for (int q = tid; q < L; q += blockDim.x) s_load[q] = 0;
    }
    __syncthreads();  // (B)
    long long sw = 0;
    for (int k = tid; k < K; k += blockDim.x) {
      if (!cand_bit(p, g, c, k)) continue;
      const long long S = __ldg(p.tr.S + k);
      atomicAdd(reinterpret_cast<unsigned long long *>(row + __ldg(p.tr.r1 + k)), (unsigned long long)(-S));
      atomicAdd(reinterpret_cast<unsigned long long *>(row + __ldg(p.tr.s + k)), (unsigned long long)S);
      atomicAdd(reinterpret_cast<unsigned long long *>(s_load + __ldg(p.tr.lin + k)), (unsigned long long)S);
      atomicAdd(reinterpret_cast<unsigned long long *>(s_load + __ldg(p.tr.lout + k)), (unsigned long long)S);
      sw += S;
    }
    __syncthreads();  // (C)
    // raking scan: thread tid owns [tid*E, tid*E + E) of [0, N)
    const int b0 = tid * p.E, b1 = min(b0 + p.E, N);
    long long tot = 0;
    for (int q = b0; q < b1; q++) tot += row[q];
    long long incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_wtot[warp] = incl;
    __syncthreads();  // (D)
    long long x = incl - tot;
    for (int w = 0; w < warp; w++) x += s_wtot[w];
    long long mx = LLONG_MIN;
    for (int q = b0; q < b1; q++) {
      x += row[q];
      const long long F = __ldg(p.tr.f0 + q) + x;
      if (kFootprint) row[q] = F;
      mx = max(mx, F);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      sw += __shfl_xor_sync(0xffffffffu, sw, o);
    }
    if (lane == 0) { s_rmax[warp] = mx; s_rsum[warp] = sw; }
    if (kFootprint) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();  // (E)
    if (kFootprint && tid == 0) {
      long long *dst = p.footprint + c * p.ld;
      const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(row));
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                   ::"l"(dst), "r"(saddr), "r"(unsigned(p.fp_elems * 8))
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    if (warp == 0) {
      double st = 0.0;
      for (int l0 = 0; l0 < L; l0 += 32) {
        const int l = l0 + lane;
        double term = 0.0;
        if (l < L) term = __dsub_rn(__ddiv_rn(double(s_load[l]), p.tr.bw), __ldg(p.tr.bud + l));
        unsigned m = __ballot_sync(0xffffffffu, term > 0.0);
        while (m) {  // ascending l, positive terms only
          const int bl = __ffs(m) - 1;
          st = __dadd_rn(st, __shfl_sync(0xffffffffu, term, bl));
          m &= m - 1;
        }
      }
      if (lane == 0) {
        long long pk = s_rmax[0], swp = s_rsum[0];
        for (int w = 1; w < nwarps; w++) { pk = max(pk, s_rmax[w]); swp += s_rsum[w]; }
        if (p.peak) p.peak[c] = pk;
        if (p.stall) p.stall[c] = st;
        if (p.swapped) p.swapped[c] = swp;
        Key k;
        k.excess = pk > p.tr.budget ? pk - p.tr.budget : 0;
        k.stall = st;
        k.swapped = swp;
        k.index = g;
        k.peak = pk;
        if (key_less(k, best)) best = k;
      }
    }
  }
  if (kFootprint && tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  // per-CTA key -> the last CTA to finish reduces all of them into *best
  __shared__ unsigned int s_last;
  if (tid == 0) {
    p.partial[blockIdx.x] = best;
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
  const int N = L.tr.N;
  // block size: ~8 row elements per thread, 32..256 threads
  int threads = ((N + 7) / 8 + 31) / 32 * 32;
  threads = std::max(32, std::min(256, threads));
  int E = (N + threads - 1) / threads;
  if (E > 1 && (E & 1) == 0) E += 1;  // odd stride: conflict-free 8 B shared accesses
  const int row_ld = (N + 1) & ~1;
  const bool fp = L.footprint != nullptr;
  const int L2 = (L.tr.L + 1) & ~1;
  const size_t smem = (size_t(fp ? 2 : 1) * row_ld + L2 + 96) * sizeof(long long);
  if (smem > 200 * 1024) CHM_FAIL(CHM_E_INVAL, "chm_eval_policies: N = %d too large for one CTA row", N);
  auto kern = fp ? replay_kernel<true> : replay_kernel<false>;
  CHM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  int per_sm = 0;
  CHM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
  if (per_sm < 1) CHM_FAIL(CHM_E_INVAL, "chm_eval_policies: kernel does not fit an SM");
  if (ctx->cfg.eval_ctas_per_sm) per_sm = std::min(per_sm, int(ctx->cfg.eval_ctas_per_sm));
  const uint64_t grid64 = std::min<uint64_t>(uint64_t(ctx->num_sms) * per_sm, L.count);
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
  p.E = E;
  p.row_ld = row_ld;
  p.fp_elems = fp ? int(std::min<uint64_t>(uint64_t(row_ld), L.ld)) : 0;
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
  if (!ctx || !t || !c || !o) CHM_FAIL(CHM_E_INVAL, "chm_eval_policies: NULL argument");
  if (!o->best) CHM_FAIL(CHM_E_INVAL, "chm_eval_policies: out.best is required");
  if (c->count == 0) CHM_FAIL(CHM_E_INVAL, "chm_eval_policies: empty candidate range");
  if (ctx->device < 0 || !t->dev_block) CHM_FAIL(CHM_E_STATE, "chm_eval_policies: host-only ctx / trace");
  if (t->device != ctx->device) CHM_FAIL(CHM_E_INVAL, "chm_eval_policies: trace on another device");
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
    case CHM_CAND_MASKS:
      if (!c->masks && t->W) CHM_FAIL(CHM_E_INVAL, "MASKS candidates need a device mask array");
      L.masks = c->masks;
      break;
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
  CHM_CUDA(cudaSetDevice(ctx->device));
  return launch_eval(ctx, L, stream);
}

extern "C" chm_status chm_best_reduce_device(chm_ctx *ctx, const chm_best *keys, uint32_t n, chm_best *out,
                                             cudaStream_t stream) {
  if (!ctx || !keys || !out || n == 0 || ctx->device < 0)
    CHM_FAIL(CHM_E_INVAL, "chm_best_reduce_device: bad argument");
  CHM_CUDA(cudaSetDevice(ctx->device));
  best_reduce_kernel<<<1, 32, 0, stream>>>(reinterpret_cast<const Key *>(keys), n, reinterpret_cast<Key *>(out));
  CHM_CUDA(cudaGetLastError());
  return CHM_OK;
}
