// swap.cu -- policy execution (steps a9-a11): multi-tensor gather/scatter between HBM and the
// ctx's mapped pinned host arena, on a dedicated swap stream fenced against compute with an
// event record/wait pair (custom recordStream; swap-in pre-trigger P:333).
//
// Kernel design (sm_100a, host-link bound, see DESIGN.md §"Swap kernel"): the descriptor list
// travels in kernel parameter space (<= 64 descriptors + chunk prefix, ~2 KB); the bytes are cut
// into 64 KiB chunks; each 512-thread CTA copies one chunk per grid-stride step with 8
// independent 16 B loads per thread issued before the 8 stores (64 KiB in flight per CTA); the
// default 8 CTAs (512 KiB in flight) already fill the host link and leave the other SMs to the
// overlapped compute (tools/overlap.py, tools/stall_fidelity.py).  Loads use the
// non-coherent path without L1 allocation; stores to HBM are streaming (.cs) so an overlapped
// compute kernel keeps its L2.
#include <algorithm>
#include <cstring>
#include <numeric>
#include <vector>

#include "internal.h"

namespace chm {
namespace {

#ifndef CHM_SWAP_THREADS
#define CHM_SWAP_THREADS 512
#endif
constexpr int kSwapThreads = CHM_SWAP_THREADS;  // threads per swap CTA (A/B knob: tools/build_variant.py)
constexpr int kUnroll = 8;
constexpr int kMisUnroll = 8;  // misaligned views: words per thread per pass
#ifndef CHM_SWAP_MINB
#define CHM_SWAP_MINB 1
#endif
// a chunk is one pass of the CTA: threads x 8 x 16 B (64 KiB at 512 threads)
constexpr int kChunkShift = kSwapThreads == 512 ? 16 : kSwapThreads == 256 ? 15 : 14;
static_assert(kSwapThreads == 512 || kSwapThreads == 256 || kSwapThreads == 128, "swap CTA size");
constexpr uint64_t kChunk = 1ull << kChunkShift;

struct SwapParams {
  uint32_t n;
  uint32_t to_host;
  uint64_t total_chunks;
  uint64_t src[kMaxDescPerLaunch];
  uint64_t dst[kMaxDescPerLaunch];
  uint64_t bytes[kMaxDescPerLaunch];
  uint64_t chunk_begin[kMaxDescPerLaunch + 1];
};

__device__ __forceinline__ int4 ld_nc_na(const void *p) {
  int4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ int4 ld_nc_na_256(const void *p) {  // + 256 B L2 prefetch hint
  int4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st_cs(void *p, int4 v) {
  asm volatile("st.global.cs.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_plain(void *p, int4 v) {
  asm volatile("st.global.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// dest word = bytes [r, r + 16) of the 32 bytes a || b (little endian), r = 4 q + sh / 8
__device__ __forceinline__ int4 shift_combine(const int4 &a, const int4 &b, int q, unsigned sh) {
  unsigned w0, w1, w2, w3, w4;
  switch (q) {  // uniform over the chunk: no divergence
    case 0: w0 = a.x; w1 = a.y; w2 = a.z; w3 = a.w; w4 = b.x; break;
    case 1: w0 = a.y; w1 = a.z; w2 = a.w; w3 = b.x; w4 = b.y; break;
    case 2: w0 = a.z; w1 = a.w; w2 = b.x; w3 = b.y; w4 = b.z; break;
    default: w0 = a.w; w1 = b.x; w2 = b.y; w3 = b.z; w4 = b.w; break;
  }
  int4 v;
  v.x = int(__funnelshift_r(w0, w1, sh));
  v.y = int(__funnelshift_r(w1, w2, sh));
  v.z = int(__funnelshift_r(w2, w3, sh));
  v.w = int(__funnelshift_r(w3, w4, sh));
  return v;
}

// One chunk [s, s + len) -> [d, d + len) where s or d is not 16 B aligned.  A head of
// h < 144 bytes brings d to 16 B alignment (and the host side to 128 B); the body is written in aligned 16 B words, each built
// from the two aligned 16 B source words it straddles (every source word is loaded once: a lane
// takes its right neighbour's word by shuffle, the warp's last lane loads one extra) -- when s
// and d share their misalignment the body is the plain vector copy; a tail of < 16 bytes ends
// it.  An aligned 16 B word holding a byte of the source never crosses a page, so the loads
// stay inside the source's pages.  Stores are 16 B transactions on the link, never single
// bytes.
__device__ __forceinline__ void copy_misaligned(const char *s, char *d, uint64_t len, bool to_host) {
  // the head aligns the host side to 128 B (whole L2 lines, whole PCIe requests): swap-out,
  // the destination; swap-in, the source's aligned words (then a few more bytes bring the
  // device-side destination to 16 B, the source words stay 128 B-grouped)
  const uintptr_t ua = reinterpret_cast<uintptr_t>(d), us = reinterpret_cast<uintptr_t>(s);
  uint64_t h0;
  if (to_host) {
    h0 = (128u - (ua & 127u)) & 127u;
  } else {
    const uint64_t h1 = (128u - (us & 127u)) & 127u;
    h0 = h1 + ((16u - ((ua + h1) & 15u)) & 15u);
  }
  const uint32_t h = uint32_t(h0 < len ? h0 : len);
  for (uint32_t i = threadIdx.x; i < h; i += kSwapThreads) d[i] = s[i];
  const char *sb = s + h;
  char *db = d + h;
  const uint64_t body = len - h;
  const uint32_t nvec = uint32_t(body >> 4);  // <= kSwapThreads x 8 (one chunk)
  const uint32_t r = uint32_t(reinterpret_cast<uintptr_t>(sb) & 15u);
  const int lane = threadIdx.x & 31;
  // kMisUnroll words per thread in flight per pass (zero-copy reads from host memory are
  // latency-bound); words idx = pass + threadIdx.x + k * kSwapThreads.  The word after a
  // warp's last lane is the next warp's lane-0 word (exchanged through shared memory), after
  // the CTA's last thread the next k's thread-0 word; one extra load per pass for the last.
  __shared__ int4 s_edge[kMisUnroll][kSwapThreads / 32];
  const int warp = threadIdx.x >> 5, nwarp = kSwapThreads / 32;
  if (r == 0) {
    for (uint32_t p0 = 0; p0 < nvec; p0 += kMisUnroll * kSwapThreads) {
      int4 v[kMisUnroll];
#pragma unroll
      for (int k = 0; k < kMisUnroll; k++) {
        const uint32_t idx = p0 + threadIdx.x + k * kSwapThreads;
        if (idx < nvec) v[k] = ld_nc_na(sb + 16ull * idx);
      }
#pragma unroll
      for (int k = 0; k < kMisUnroll; k++) {
        const uint32_t idx = p0 + threadIdx.x + k * kSwapThreads;
        if (idx < nvec) st_plain(db + 16ull * idx, v[k]);
      }
    }
  } else {
    const char *as = sb - r;  // aligned source words as[0 .. nvec] hold the body's bytes
    const int q = int(r >> 2);
    const unsigned sh = 8u * (r & 3u);
    for (uint32_t p0 = 0; p0 < nvec; p0 += kMisUnroll * kSwapThreads) {
      int4 a[kMisUnroll];
      int4 last = make_int4(0, 0, 0, 0);
#pragma unroll
      for (int k = 0; k < kMisUnroll; k++) {
        const uint32_t idx = p0 + threadIdx.x + k * kSwapThreads;
        a[k] = make_int4(0, 0, 0, 0);
        if (idx <= nvec) a[k] = ld_nc_na(as + 16ull * idx);
      }
      const uint32_t after = p0 + kMisUnroll * kSwapThreads;  // the word after the pass
      if (threadIdx.x == kSwapThreads - 1 && after <= nvec) last = ld_nc_na(as + 16ull * after);
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < kMisUnroll; k++) s_edge[k][warp] = a[k];
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < kMisUnroll; k++) {
        const uint32_t idx = p0 + threadIdx.x + k * kSwapThreads;
        int4 b;
        b.x = __shfl_down_sync(0xffffffffu, a[k].x, 1);
        b.y = __shfl_down_sync(0xffffffffu, a[k].y, 1);
        b.z = __shfl_down_sync(0xffffffffu, a[k].z, 1);
        b.w = __shfl_down_sync(0xffffffffu, a[k].w, 1);
        if (lane == 31) b = warp + 1 < nwarp ? s_edge[k][warp + 1] : (k + 1 < kMisUnroll ? s_edge[k + 1][0] : last);
        if (idx < nvec) st_plain(db + 16ull * idx, shift_combine(a[k], b, q, sh));
      }
      __syncthreads();  // s_edge is rewritten by the next pass
    }
  }
  const uint32_t tail = uint32_t(body & 15);
  if (threadIdx.x < tail) db[16ull * nvec + threadIdx.x] = sb[16ull * nvec + threadIdx.x];
}

template <bool kPrefetch256>
__global__ void __launch_bounds__(kSwapThreads, CHM_SWAP_MINB) swap_copy_kernel(const __grid_constant__ SwapParams p) {
  for (uint64_t c = blockIdx.x; c < p.total_chunks; c += gridDim.x) {
    uint32_t lo = 0, hi = p.n;  // chunk_begin[lo] <= c < chunk_begin[hi]
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (p.chunk_begin[mid] <= c) lo = mid; else hi = mid;
    }
    const uint64_t off = (c - p.chunk_begin[lo]) << kChunkShift;
    CHM_DCHECK(lo < p.n && c >= p.chunk_begin[lo] && off < p.bytes[lo]);
    const uint64_t len = min(kChunk, p.bytes[lo] - off);
    const char *s = reinterpret_cast<const char *>(p.src[lo]) + off;
    char *d = reinterpret_cast<char *>(p.dst[lo]) + off;
    if (((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d)) & 15) == 0) {
      const uint32_t nvec = uint32_t(len >> 4);
      int4 v[kUnroll];
#pragma unroll
      for (int k = 0; k < kUnroll; k++) {
        const uint32_t idx = threadIdx.x + k * kSwapThreads;
        if (idx < nvec) v[k] = kPrefetch256 ? ld_nc_na_256(s + 16ull * idx) : ld_nc_na(s + 16ull * idx);
      }
#pragma unroll
      for (int k = 0; k < kUnroll; k++) {
        const uint32_t idx = threadIdx.x + k * kSwapThreads;
        if (idx < nvec) {
          if (p.to_host) st_plain(d + 16ull * idx, v[k]);
          else st_cs(d + 16ull * idx, v[k]);
        }
      }
      const uint32_t tail = uint32_t(len & 15);
      if (threadIdx.x < tail) d[16ull * nvec + threadIdx.x] = s[16ull * nvec + threadIdx.x];
    } else {  // misaligned view: aligned 16 B stores fed by aligned 16 B loads (funnel shifts)
      copy_misaligned(s, d, len, p.to_host != 0);
    }
  }
}

// TMA bulk-copy variant: one thread per CTA drives a kBulkStages-deep pipeline of
// cp.async.bulk global->shared (mbarrier completion) and shared->global (bulk group) copies of
// kBulkStage bytes.  Requires 16 B-aligned addresses and sizes (checked by the launcher).
constexpr int kBulkStage = 16384;
constexpr int kBulkStages = 4;

__device__ __forceinline__ void bulk_load(unsigned sdst, const void *src, unsigned n, unsigned bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(n) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sdst),
               "l"(src), "r"(n), "r"(bar)
               : "memory");
}

__device__ __forceinline__ void bulk_wait(unsigned bar, unsigned parity) {
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  }
}

__global__ void __launch_bounds__(32) swap_bulk_kernel(const __grid_constant__ SwapParams p) {
  extern __shared__ __align__(128) unsigned char buf[];
  __shared__ __align__(8) uint64_t mbar[kBulkStages];
  if (threadIdx.x != 0) return;
  const unsigned sbuf = static_cast<unsigned>(__cvta_generic_to_shared(buf));
  unsigned bars[kBulkStages];
  for (int s = 0; s < kBulkStages; s++) {
    bars[s] = static_cast<unsigned>(__cvta_generic_to_shared(&mbar[s]));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bars[s]) : "memory");
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  // this CTA's pieces: piece j = global piece blockIdx.x + j * gridDim.x, pieces of kBulkStage B
  const uint64_t total = p.total_chunks;  // in kBulkStage pieces (launcher)
  const uint64_t n = total > blockIdx.x ? (total - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  auto piece = [&](uint64_t j, const char *&src, char *&dst, unsigned &len) {
    const uint64_t c = blockIdx.x + j * gridDim.x;
    uint32_t lo = 0, hi = p.n;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (p.chunk_begin[mid] <= c) lo = mid; else hi = mid;
    }
    const uint64_t off = (c - p.chunk_begin[lo]) * uint64_t(kBulkStage);
    CHM_DCHECK(lo < p.n && off < p.bytes[lo]);
    len = unsigned(min(uint64_t(kBulkStage), p.bytes[lo] - off));
    src = reinterpret_cast<const char *>(p.src[lo]) + off;
    dst = reinterpret_cast<char *>(p.dst[lo]) + off;
  };
  const char *src;
  char *dst;
  unsigned len;
  for (uint64_t j = 0; j < n && j < kBulkStages - 1; j++) {
    piece(j, src, dst, len);
    bulk_load(sbuf + unsigned(j % kBulkStages) * kBulkStage, src, len, bars[j % kBulkStages]);
  }
  for (uint64_t it = 0; it < n; it++) {
    const int s = int(it % kBulkStages);
    bulk_wait(bars[s], unsigned((it / kBulkStages) & 1));
    piece(it, src, dst, len);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"(sbuf + unsigned(s) * kBulkStage), "r"(len)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    const uint64_t jn = it + kBulkStages - 1;
    if (jn < n) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // store it-1 left its stage
      piece(jn, src, dst, len);
      bulk_load(sbuf + unsigned(jn % kBulkStages) * kBulkStage, src, len, bars[jn % kBulkStages]);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

}  // namespace

chm_status launch_swap_copy(const chm_swap_desc *desc, uint32_t n, char *arena, bool to_host,
                            int ctas, int variant, cudaStream_t stream) {
  for (uint32_t base = 0; base < n; base += kMaxDescPerLaunch) {
    SwapParams p;
    std::memset(&p, 0, sizeof p);
    p.n = std::min<uint32_t>(kMaxDescPerLaunch, n - base);
    p.to_host = to_host ? 1u : 0u;
    bool aligned = true;
    for (uint32_t j = 0; j < p.n; j++) {
      const chm_swap_desc &d = desc[base + j];
      const uint64_t host = reinterpret_cast<uint64_t>(arena) + d.host_off;
      p.src[j] = to_host ? d.dev : host;
      p.dst[j] = to_host ? host : d.dev;
      p.bytes[j] = d.nbytes;
      aligned = aligned && ((p.src[j] | p.dst[j] | p.bytes[j]) & 15) == 0;
    }
    const bool bulk = variant == 2 && aligned;
    const uint64_t piece = bulk ? uint64_t(kBulkStage) : kChunk;
    uint64_t chunks = 0;
    for (uint32_t j = 0; j < p.n; j++) {
      p.chunk_begin[j] = chunks;
      chunks += (p.bytes[j] + piece - 1) / piece;
    }
    p.chunk_begin[p.n] = chunks;
    p.total_chunks = chunks;
    const int grid = int(std::min<uint64_t>(uint64_t(ctas), chunks));
    if (grid == 0) continue;
    if (bulk) {
      CHM_CUDA(ensure_dyn_smem(reinterpret_cast<const void *>(swap_bulk_kernel), size_t(kBulkStage) * kBulkStages));
      swap_bulk_kernel<<<grid, 32, kBulkStage * kBulkStages, stream>>>(p);
    } else if (variant == 1) {
      swap_copy_kernel<true><<<grid, kSwapThreads, 0, stream>>>(p);
    } else {
      swap_copy_kernel<false><<<grid, kSwapThreads, 0, stream>>>(p);
    }
    CHM_CUDA(cudaGetLastError());
  }
  return CHM_OK;
}

}  // namespace chm

using namespace chm;

extern "C" chm_status chm_host_arena(chm_ctx *ctx, void **host_base, uint64_t *bytes) {
  if (!ctx) CHM_FAIL(CHM_E_INVAL, "chm_host_arena: NULL ctx");
  if (ctx->arena_busy.load()) CHM_FAIL(CHM_E_STATE, "chm_host_arena: the arena is being re-pinned");
  if (host_base) *host_base = ctx->arena;
  if (bytes) *bytes = ctx->arena_bytes;
  return CHM_OK;
}

static chm_status validate_batch(chm_ctx *ctx, const chm_swap_desc *d, uint32_t n, int64_t *err) {
  if (err) *err = -1;
  if (n && !d) CHM_FAIL(CHM_E_INVAL, "swap: NULL descriptor list");
  if (n && ctx->arena_busy.load()) CHM_FAIL(CHM_E_STATE, "swap: the host arena is being re-pinned (chm_arena_reserve)");
  if (n && !ctx->arena) CHM_FAIL(CHM_E_STATE, "swap: ctx has no host arena");
  for (uint32_t j = 0; j < n; j++) {
    if (d[j].nbytes == 0 || d[j].dev == 0 || d[j].host_off > ctx->arena_bytes ||
        d[j].nbytes > ctx->arena_bytes - d[j].host_off) {
      if (err) *err = j;
      CHM_FAIL(CHM_E_INVAL, "swap: descriptor %u invalid (dev %llx off %llu bytes %llu, arena %llu)",
               j, (unsigned long long)d[j].dev, (unsigned long long)d[j].host_off,
               (unsigned long long)d[j].nbytes, (unsigned long long)ctx->arena_bytes);
    }
  }
  if (n > 1) {  // host ranges of one batch must not overlap
    std::vector<uint32_t> ord(n);
    std::iota(ord.begin(), ord.end(), 0u);
    std::sort(ord.begin(), ord.end(), [&](uint32_t x, uint32_t y) { return d[x].host_off < d[y].host_off; });
    for (uint32_t j = 1; j < n; j++) {
      const chm_swap_desc &p = d[ord[j - 1]], &q = d[ord[j]];
      if (p.host_off + p.nbytes > q.host_off) {
        if (err) *err = ord[j];
        CHM_FAIL(CHM_E_INVAL, "swap: descriptor %u overlaps descriptor %u in the arena", ord[j], ord[j - 1]);
      }
    }
  }
  return CHM_OK;
}

static chm_status swap_batch(chm_ctx *ctx, const chm_swap_desc *d, uint32_t n, cudaStream_t compute,
                             cudaStream_t swap, uint32_t flags, uint64_t *batch, int64_t *err,
                             bool to_host) {
  CHM_NVTX(to_host ? "chm_swap_out" : "chm_swap_in");
  if (!ctx) CHM_FAIL(CHM_E_INVAL, "swap: NULL ctx");
  if (ctx->device < 0) CHM_FAIL(CHM_E_STATE, "swap: host-only ctx");
  if (flags > CHM_SWAP_AUTO) CHM_FAIL(CHM_E_INVAL, "swap: unknown flags %u", flags);
  chm_status st = validate_batch(ctx, d, n, err);
  if (st != CHM_OK) return st;
  CHM_DEVICE_SCOPE(ctx->device);
  const uint64_t b = ctx->next_batch++;
  const size_t slot = size_t(b % kEventRing);
  if (compute != swap) {  // swap stream starts after everything enqueued on compute so far
    CHM_CUDA(cudaEventRecord(ctx->fences[slot], compute));
    CHM_CUDA(cudaStreamWaitEvent(swap, ctx->fences[slot], 0));
  }
  char *arena = static_cast<char *>(ctx->arena);
  if (!ctx->t0.empty()) CHM_CUDA(cudaEventRecord(ctx->t0[slot], swap));
  const uint64_t ce_min = ctx->cfg.ce_min_bytes ? ctx->cfg.ce_min_bytes : (4ull << 20);
  auto on_ce = [&](const chm_swap_desc &x) {
    return flags == CHM_SWAP_CE || (flags == CHM_SWAP_AUTO && x.nbytes >= ce_min);
  };
  std::vector<chm_swap_desc> &kd = ctx->kernel_descs;
  kd.clear();
  for (uint32_t j = 0; j < n; j++) {
    if (!on_ce(d[j])) { kd.push_back(d[j]); continue; }
    char *host = arena + d[j].host_off;  // copy engine: one transfer per descriptor
    void *dev = reinterpret_cast<void *>(d[j].dev);
    CHM_CUDA(cudaMemcpyAsync(to_host ? (void *)host : dev, to_host ? (const void *)dev : host,
                             d[j].nbytes, to_host ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice, swap));
  }
  if (!kd.empty()) {
    const int ctas = ctx->cfg.swap_ctas ? int(ctx->cfg.swap_ctas) : 8;
    st = launch_swap_copy(kd.data(), uint32_t(kd.size()), arena, to_host, ctas, int(ctx->cfg.swap_variant), swap);
    if (st != CHM_OK) return st;
  }
  if (!ctx->t1.empty()) CHM_CUDA(cudaEventRecord(ctx->t1[slot], swap));
  CHM_CUDA(cudaEventRecord(ctx->events[slot], swap));
  if (batch) *batch = b;
  return CHM_OK;
}

extern "C" chm_status chm_swap_out(chm_ctx *ctx, const chm_swap_desc *d, uint32_t n,
                                   cudaStream_t compute, cudaStream_t swap, uint32_t flags,
                                   uint64_t *batch, int64_t *err_index) {
  return swap_batch(ctx, d, n, compute, swap, flags, batch, err_index, true);
}

extern "C" chm_status chm_swap_in(chm_ctx *ctx, const chm_swap_desc *d, uint32_t n,
                                  cudaStream_t compute, cudaStream_t swap, uint32_t flags,
                                  uint64_t *batch, int64_t *err_index) {
  return swap_batch(ctx, d, n, compute, swap, flags, batch, err_index, false);
}

extern "C" chm_status chm_batch_wait(chm_ctx *ctx, uint64_t batch, cudaStream_t stream) {
  if (!ctx || ctx->device < 0) CHM_FAIL(CHM_E_INVAL, "chm_batch_wait: NULL or host-only ctx");
  if (batch >= ctx->next_batch || batch + kEventRing < ctx->next_batch)
    CHM_FAIL(CHM_E_INVAL, "chm_batch_wait: batch %llu unknown or expired", (unsigned long long)batch);
  CHM_CUDA(cudaStreamWaitEvent(stream, ctx->events[batch % kEventRing], 0));
  return CHM_OK;
}

extern "C" chm_status chm_batch_query(chm_ctx *ctx, uint64_t batch, int32_t *done) {
  if (!ctx || !done || ctx->device < 0) CHM_FAIL(CHM_E_INVAL, "chm_batch_query: NULL argument / host-only ctx");
  if (batch >= ctx->next_batch || batch + kEventRing < ctx->next_batch)
    CHM_FAIL(CHM_E_INVAL, "chm_batch_query: batch unknown or expired");
  cudaError_t e = cudaEventQuery(ctx->events[batch % kEventRing]);
  if (e == cudaErrorNotReady) { *done = 0; return CHM_OK; }
  CHM_CUDA(e);
  *done = 1;
  return CHM_OK;
}

extern "C" chm_status chm_batch_elapsed(chm_ctx *ctx, uint64_t batch, float *ms) {
  if (!ctx || !ms || ctx->device < 0) CHM_FAIL(CHM_E_INVAL, "chm_batch_elapsed: NULL argument / host-only ctx");
  if (ctx->t0.empty()) CHM_FAIL(CHM_E_STATE, "chm_batch_elapsed: ctx created without time_batches");
  if (batch >= ctx->next_batch || batch + kEventRing < ctx->next_batch)
    CHM_FAIL(CHM_E_INVAL, "chm_batch_elapsed: batch unknown or expired");
  const size_t slot = size_t(batch % kEventRing);
  cudaError_t e = cudaEventElapsedTime(ms, ctx->t0[slot], ctx->t1[slot]);
  if (e == cudaErrorNotReady) CHM_FAIL(CHM_E_STATE, "chm_batch_elapsed: batch not complete");
  CHM_CUDA(e);
  return CHM_OK;
}

extern "C" chm_status chm_arena_reserve(chm_ctx *ctx, uint64_t bytes) {
  if (!ctx || ctx->device < 0) CHM_FAIL(CHM_E_INVAL, "chm_arena_reserve: NULL or host-only ctx");
  if (bytes <= ctx->arena_bytes) return CHM_OK;
  if (!ctx->passive.empty())
    CHM_FAIL(CHM_E_STATE, "chm_arena_reserve: %zu passive swaps hold arena data", ctx->passive.size());
  int idle = 0;
  if (!ctx->arena_busy.compare_exchange_strong(idle, 1))
    CHM_FAIL(CHM_E_STATE, "chm_arena_reserve: another reserve is running on this ctx");
  struct Busy { std::atomic<int> &b; ~Busy() { b.store(0); } } busy{ctx->arena_busy};
  ctx->passive_free.clear();  // re-derived from the new size at the next passive swap
  CHM_DEVICE_SCOPE(ctx->device);
  const uint64_t old = ctx->arena_bytes;
  arena_free(ctx);  // arena.cpp; pinning old + new together would double the host footprint
  const chm_status st = arena_alloc(ctx, bytes);
  if (st != CHM_OK && old) {  // keep an arena of the old size: installed plans still fit it
    const std::string msg = chm_last_error();
    if (arena_alloc(ctx, old) != CHM_OK)
      CHM_FAIL(st, "%s (and re-pinning the previous %llu B failed: %s)", msg.c_str(), (unsigned long long)old,
               chm_last_error());
    CHM_FAIL(st, "%s (the previous %llu B arena was re-pinned)", msg.c_str(), (unsigned long long)old);
  }
  return st;
}

namespace chm {
cudaError_t preload_swap() {
  cudaFuncAttributes a;
  cudaError_t e = cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(swap_copy_kernel<true>));
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(swap_copy_kernel<false>));
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(swap_bulk_kernel));
  return e;
}
}  // namespace chm
