// explicit.cu -- replay of EXPLICIT candidates (item lists with arbitrary release / swap-in
// ops, e.g. Algo. 2's policies).  Same result as the layer-segment kernel (replay.cu), without
// its R-window precondition: one CTA per candidate keeps a shared-memory delta row over the ops,
//   d[r_t + 1] -= S_t, d[s_t] += S_t     (release after r_t, swap-in before s_t)
// scans it (raking: each thread E contiguous ops, E odd), F_P = F0 + prefix, peak = max, and
// streams the row out in full mode; per-layer loads (lin = lay(s), lout = lay(r)) give the
// stall with the pairwise tree of reading R-stall.  Explicit sets are few (generator outputs),
// so this kernel favours generality over throughput.
#include <algorithm>
#include <climits>
#include <cstring>
#include <vector>

#include "internal.h"

namespace chm {
namespace {

struct XKey {
  long long excess;
  double stall;
  long long swapped;
  unsigned long long index;
  long long peak;
};

__device__ __forceinline__ bool xkey_less(const XKey &x, const XKey &y) {
  if (x.excess != y.excess) return x.excess < y.excess;
  if (x.stall != y.stall) return x.stall < y.stall;
  if (x.swapped != y.swapped) return x.swapped < y.swapped;
  return x.index < y.index;
}

struct XParams {
  const long long *f0;           // device [N] (trace image)
  const unsigned short *lay8;    // device [N] 8 x layer (trace image)
  const double *bud;             // device [L]
  const long long *S_rank;       // device [n_prod] sizes by production rank
  const unsigned long long *off; // device [count + 1]
  const chm_item *items;         // device
  int N, L, E;
  double bw;
  long long budget;
  unsigned long long first;
  long long *peak;
  double *stall;
  long long *swapped;
  long long *footprint;
  unsigned long long ld;
  XKey *keys;                    // device [count]
};

__global__ void __launch_bounds__(256) replay_explicit_kernel(const __grid_constant__ XParams p) {
  extern __shared__ __align__(16) long long row[];  // [N + 1] deltas, then F
  __shared__ long long s_load[256 * 2];              // per-layer loads (L <= 256 enforced at build)
  __shared__ long long s_wtot[8], s_wmax[8], s_wsum[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int N = p.N, L = p.L;
  const unsigned long long c = blockIdx.x;
  for (int i = tid; i <= N; i += blockDim.x) row[i] = 0;
  for (int l = tid; l < L; l += blockDim.x) s_load[l] = 0;
  __syncthreads();
  long long sw = 0;
  for (unsigned long long q = p.off[c] + tid; q < p.off[c + 1]; q += blockDim.x) {
    const chm_item it = p.items[q];
    CHM_DCHECK(it.r >= 0 && it.r + 1 < it.s && it.s < p.N && (p.lay8[it.s] >> 3) < p.L && (p.lay8[it.r] >> 3) < p.L);
    const long long S = p.S_rank[it.t];
    atomicAdd(reinterpret_cast<unsigned long long *>(row + it.r + 1), (unsigned long long)(-S));
    atomicAdd(reinterpret_cast<unsigned long long *>(row + it.s), (unsigned long long)S);
    atomicAdd(reinterpret_cast<unsigned long long *>(s_load + (p.lay8[it.s] >> 3)), (unsigned long long)S);
    atomicAdd(reinterpret_cast<unsigned long long *>(s_load + (p.lay8[it.r] >> 3)), (unsigned long long)S);
    sw += S;
  }
  __syncthreads();
  const int b0 = tid * p.E, b1 = min(b0 + p.E, N);
  long long tot = 0;
  for (int i = b0; i < b1; i++) tot += row[i];
  long long incl = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_wtot[warp] = incl;
  __syncthreads();
  long long x = incl - tot, mx = LLONG_MIN;
  for (int w = 0; w < warp; w++) x += s_wtot[w];
  for (int i = b0; i < b1; i++) {
    x += row[i];
    const long long F = p.f0[i] + x;
    row[i] = F;
    mx = max(mx, F);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    sw += __shfl_xor_sync(0xffffffffu, sw, o);
  }
  if (lane == 0) { s_wmax[warp] = mx; s_wsum[warp] = sw; }
  __syncthreads();
  if (p.footprint) {
    long long *dst = p.footprint + c * p.ld;
    for (int i = tid; i < N; i += blockDim.x) dst[i] = row[i];
  }
  if (warp == 0) {
    double cs[8];
#pragma unroll
    for (int j = 0; j < 8; j++) {
      double t = 0.0;
      const int l = lane + 32 * j;
      if (l < L) {
        const double v = __dsub_rn(__ddiv_rn(double(s_load[l]), p.bw), p.bud[l]);
        t = v > 0.0 ? v : 0.0;
      }
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) t = __dadd_rn(t, __shfl_xor_sync(0xffffffffu, t, o));
      cs[j] = t;
    }
    const double st = __dadd_rn(__dadd_rn(__dadd_rn(cs[0], cs[1]), __dadd_rn(cs[2], cs[3])),
                                __dadd_rn(__dadd_rn(cs[4], cs[5]), __dadd_rn(cs[6], cs[7])));
    if (lane == 0) {
      long long pk = s_wmax[0], swp = s_wsum[0];
      for (int w = 1; w < int(blockDim.x >> 5); w++) { pk = max(pk, s_wmax[w]); swp += s_wsum[w]; }
      if (p.peak) p.peak[c] = pk;
      if (p.stall) p.stall[c] = st;
      if (p.swapped) p.swapped[c] = swp;
      XKey k;
      k.excess = pk > p.budget ? pk - p.budget : 0;
      k.stall = st;
      k.swapped = swp;
      k.index = p.first + c;
      k.peak = pk;
      p.keys[c] = k;
    }
  }
}

__global__ void xkey_reduce_kernel(const XKey *keys, unsigned long long n, XKey *out) {
  XKey b;
  b.excess = LLONG_MAX; b.stall = 0.0; b.swapped = LLONG_MAX; b.index = ~0ull; b.peak = 0;
  for (unsigned long long q = threadIdx.x; q < n; q += 32) if (xkey_less(keys[q], b)) b = keys[q];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    XKey y;
    y.excess = __shfl_xor_sync(0xffffffffu, b.excess, o);
    y.stall = __shfl_xor_sync(0xffffffffu, b.stall, o);
    y.swapped = __shfl_xor_sync(0xffffffffu, b.swapped, o);
    y.index = __shfl_xor_sync(0xffffffffu, b.index, o);
    y.peak = __shfl_xor_sync(0xffffffffu, b.peak, o);
    if (xkey_less(y, b)) b = y;
  }
  if (threadIdx.x == 0) *out = b;
}

}  // namespace

chm_status launch_eval_explicit(chm_ctx *ctx, const chm_trace *t, const chm_candidates *c,
                                const chm_eval_out *o, cudaStream_t stream, int64_t *err_index) {
  if (!c->item_offsets || (!c->items && c->item_offsets[c->count] > c->item_offsets[0]))
    CHM_FAIL(CHM_E_INVAL, "EXPLICIT candidates need host item_offsets / items");
  const uint64_t base = c->item_offsets[0], n_items = c->item_offsets[c->count] - base;
  // validation: produced activation, a_t <= r, r + 1 < s <= b_t, no repeat
  const int32_t n_prod = int32_t(t->rank_to_tensor.size());
  std::vector<int32_t> seen(static_cast<size_t>(n_prod), -1);
  for (uint64_t cc = 0; cc < c->count; cc++) {
    if (c->item_offsets[cc + 1] < c->item_offsets[cc])
      CHM_FAIL(CHM_E_INVAL, "EXPLICIT item_offsets not ascending at candidate %llu", (unsigned long long)cc);
    for (uint64_t q = c->item_offsets[cc]; q < c->item_offsets[cc + 1]; q++) {
      const chm_item &it = c->items[q];
      bool ok = int64_t(it.t) < n_prod;
      if (ok) {
        const int32_t tid = t->rank_to_tensor[it.t];
        ok = t->a[tid] >= 0 && t->b[tid] >= 0 && t->a[tid] <= it.r && it.r + 1 < it.s && it.s <= t->b[tid] &&
             seen[it.t] != int32_t(cc);
        if (ok) seen[it.t] = int32_t(cc);
      }
      if (!ok) {
        if (err_index) *err_index = int64_t(q - base);
        CHM_FAIL(CHM_E_INVAL, "EXPLICIT item %llu (t %u, r %d, s %d) invalid", (unsigned long long)(q - base),
                 it.t, it.r, it.s);
      }
    }
  }
  // stage sizes-by-rank, offsets, items and keys in ctx scratch
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t b_S = al(8 * size_t(n_prod) + 8), b_off = al(8 * (size_t(c->count) + 1)),
               b_it = al(sizeof(chm_item) * size_t(n_items) + 16), b_key = al(sizeof(XKey) * size_t(c->count));
  const size_t need = b_S + b_off + b_it + b_key;
  if (ctx->explicit_scratch_bytes < need) {
    if (ctx->explicit_scratch) cudaFree(ctx->explicit_scratch);
    ctx->explicit_scratch = nullptr;
    ctx->explicit_scratch_bytes = 0;
    CHM_CUDA(cudaMalloc(&ctx->explicit_scratch, need));
    ctx->explicit_scratch_bytes = need;
  }
  std::vector<unsigned char> host(b_S + b_off + b_it, 0);
  std::vector<int64_t> S_rank(static_cast<size_t>(n_prod));
  for (int32_t rk = 0; rk < n_prod; rk++) S_rank[rk] = t->S_t[t->rank_to_tensor[rk]];
  std::memcpy(host.data(), S_rank.data(), 8 * size_t(n_prod));
  std::vector<uint64_t> off(size_t(c->count) + 1);
  for (uint64_t cc = 0; cc <= c->count; cc++) off[cc] = c->item_offsets[cc] - base;
  std::memcpy(host.data() + b_S, off.data(), 8 * off.size());
  if (n_items) std::memcpy(host.data() + b_S + b_off, c->items + base, sizeof(chm_item) * size_t(n_items));
  unsigned char *d = static_cast<unsigned char *>(ctx->explicit_scratch);
  CHM_CUDA(cudaMemcpyAsync(d, host.data(), host.size(), cudaMemcpyHostToDevice, stream));
  XParams p{};
  p.f0 = reinterpret_cast<const long long *>(t->dev.image + t->dev.o_f0w);
  p.lay8 = reinterpret_cast<const unsigned short *>(t->dev.image + t->dev.o_lay);
  p.bud = reinterpret_cast<const double *>(t->dev.image + t->dev.o_bud);
  p.S_rank = reinterpret_cast<const long long *>(d);
  p.off = reinterpret_cast<const unsigned long long *>(d + b_S);
  p.items = reinterpret_cast<const chm_item *>(d + b_S + b_off);
  p.keys = reinterpret_cast<XKey *>(d + b_S + b_off + b_it);
  p.N = t->N;
  p.L = t->L;
  int E = (t->N + 255) / 256;
  if (E > 1 && (E & 1) == 0) E += 1;
  p.E = E;
  p.bw = t->bw;
  p.budget = t->budget;
  p.first = c->first_index;
  p.peak = reinterpret_cast<long long *>(o->peak);
  p.stall = o->stall;
  p.swapped = reinterpret_cast<long long *>(o->swapped);
  p.footprint = reinterpret_cast<long long *>(o->footprint);
  p.ld = o->ld;
  const size_t smem = 8 * (size_t(t->N) + 2);
  if (smem > 200 * 1024) CHM_FAIL(CHM_E_INVAL, "EXPLICIT replay: N = %d too large for one CTA row", t->N);
  CHM_CUDA(ensure_dyn_smem(reinterpret_cast<const void *>(replay_explicit_kernel), smem));
  replay_explicit_kernel<<<unsigned(c->count), 256, smem, stream>>>(p);
  CHM_CUDA(cudaGetLastError());
  xkey_reduce_kernel<<<1, 32, 0, stream>>>(p.keys, c->count, reinterpret_cast<XKey *>(o->best));
  CHM_CUDA(cudaGetLastError());
  return CHM_OK;
}

}  // namespace chm

namespace chm {
cudaError_t preload_explicit() {
  cudaFuncAttributes a;
  cudaError_t e = cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(replay_explicit_kernel));
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(xkey_reduce_kernel));
  return e;
}
}  // namespace chm
