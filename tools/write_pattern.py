"""Write-pattern microbenchmark for the replay kernel's full mode (context only): 10^5 rows of
2618 int64 (the C2 footprint rows, 2.09 GB) written (a) as one linear grid-stride stream,
(b) one row per warp, rows handed out by an atomic counter (the replay kernel's pattern),
(c) 16 consecutive rows per CTA written as one linear block by all 512 threads, (d) one row per
warp composed in shared memory and written by TMA bulk stores (1 / 2 / 4 KiB, double-buffered).
16 B streaming stores everywhere; 296 CTAs x 512 threads (2 per SM).  Prints GB/s."""
import torch
from torch.utils.cpp_extension import load_inline

SRC = r"""
#include <torch/extension.h>
__device__ __forceinline__ void st2(long long *d, long long a, long long b) {
  asm volatile("st.global.cs.v2.s64 [%0], {%1, %2};" :: "l"(d), "l"(a), "l"(b));
}
__global__ void linear_k(long long *out, long long n2) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x)
    st2(out + 2 * i, i, i);
}
__global__ void rows_k(long long *out, int rows, int ld, unsigned long long *ctr) {
  int lane = threadIdx.x & 31;
  while (true) {
    unsigned long long c = 0;
    if (lane == 0) c = atomicAdd(ctr, 1ull);
    c = __shfl_sync(0xffffffffu, c, 0);
    if (c >= (unsigned long long)rows) break;
    long long *r = out + c * ld;
    for (int q = lane; q < ld / 2; q += 32) st2(r + 2 * q, c, q);
  }
}
__global__ void block_k(long long *out, int rows, int ld, unsigned long long *ctr) {
  __shared__ unsigned long long c0;
  while (true) {
    if (threadIdx.x == 0) c0 = atomicAdd(ctr, 16ull);
    __syncthreads();
    unsigned long long c = c0;
    __syncthreads();
    if (c >= (unsigned long long)rows) break;
    long long nr = min(16ull, rows - c);
    long long *b = out + c * ld;
    long long n2 = nr * ld / 2;
    for (long long i = threadIdx.x; i < n2; i += blockDim.x) st2(b + 2 * i, c, i);
  }
}
// (d) row per warp, composed in a per-warp shared-memory chunk and written by TMA bulk stores
// (cp.async.bulk.global.shared::cta), double-buffered: CH bytes per bulk store
template <int CH>
__global__ void rows_tma_k(long long *out, int rows, int ld, unsigned long long *ctr) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char *buf = sm + warp * 2 * CH;
  const unsigned sbuf = (unsigned)__cvta_generic_to_shared(buf);
  int flip = 0;
  while (true) {
    unsigned long long c = 0;
    if (lane == 0) c = atomicAdd(ctr, 1ull);
    c = __shfl_sync(0xffffffffu, c, 0);
    if (c >= (unsigned long long)rows) break;
    long long *r = out + c * ld;
    const long long row_bytes = (long long)ld * 8;
    for (long long off = 0; off < row_bytes; off += CH) {
      const int n = (int)min((long long)CH, row_bytes - off);
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      __syncwarp();
      long long *sb = (long long *)(buf + flip * CH);
      for (int q = lane; q < n / 16; q += 32) { sb[2 * q] = c; sb[2 * q + 1] = off / 16 + q; }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     :: "l"((char *)r + off), "r"(sbuf + flip * CH), "r"(n) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      flip ^= 1;
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// (e) groups of G warps: G consecutive rows written as one linear block by the group's threads
// (named barrier per group), i.e. 4736 / G concurrent write streams
template <int G>
__global__ void group_k(long long *out, int rows, int ld, unsigned long long *ctr) {
  __shared__ unsigned long long c0[16];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, grp = warp / G, gt = threadIdx.x - grp * G * 32;
  while (true) {
    if (gt == 0) c0[grp] = atomicAdd(ctr, (unsigned long long)G);
    asm volatile("bar.sync %0, %1;" :: "r"(grp + 1), "r"(G * 32) : "memory");
    const unsigned long long c = c0[grp];
    asm volatile("bar.sync %0, %1;" :: "r"(grp + 1), "r"(G * 32) : "memory");
    if (c >= (unsigned long long)rows) break;
    const long long nr = min((unsigned long long)G, rows - c);
    long long *b = out + c * ld;
    const long long n2 = nr * ld / 2;
    for (long long i = gt; i < n2; i += G * 32) st2(b + 2 * i, c, i);
  }
  (void)lane;
}
// (f) row per warp with 256-bit stores (st.global.cs.v4.s64, sm_100): 1 KiB per warp instruction
__device__ __forceinline__ void st4(long long *d, long long a, long long b, long long c, long long e) {
  asm volatile("st.global.cs.v4.s64 [%0], {%1, %2, %3, %4};" :: "l"(d), "l"(a), "l"(b), "l"(c), "l"(e));
}
__global__ void rows256_k(long long *out, int rows, int ld, unsigned long long *ctr) {
  int lane = threadIdx.x & 31;
  while (true) {
    unsigned long long c = 0;
    if (lane == 0) c = atomicAdd(ctr, 1ull);
    c = __shfl_sync(0xffffffffu, c, 0);
    if (c >= (unsigned long long)rows) break;
    long long *r = out + c * ld;
    const int h = (reinterpret_cast<unsigned long long>(r) & 31) ? 2 : 0;  // 16 B head to 32 B alignment
    if (h && lane == 0) st2(r, c, c);
    const int n4 = (ld - h) / 4;
    for (int q = lane; q < n4; q += 32) st4(r + h + 4 * q, c, q, c, q);
    for (int q = h + 4 * n4 + lane; q < ld; q += 32) r[q] = c;  // tail
  }
}
// (g) row per warp, default write-back stores (no .cs) / L2 evict_last hint
template <int kHint>
__global__ void rows_wb_k(long long *out, int rows, int ld, unsigned long long *ctr) {
  int lane = threadIdx.x & 31;
  while (true) {
    unsigned long long c = 0;
    if (lane == 0) c = atomicAdd(ctr, 1ull);
    c = __shfl_sync(0xffffffffu, c, 0);
    if (c >= (unsigned long long)rows) break;
    long long *r = out + c * ld;
    for (int q = lane; q < ld / 2; q += 32) {
      if (kHint == 0) asm volatile("st.global.v2.s64 [%0], {%1, %2};" :: "l"(r + 2 * q), "l"((long long)c), "l"((long long)q));
      else asm volatile("st.global.L1::no_allocate.v2.s64 [%0], {%1, %2};" :: "l"(r + 2 * q), "l"((long long)c), "l"((long long)q));
    }
  }
}
// (h) one warp writes R consecutive rows as one linear block (no inter-warp sync)
template <int R>
__global__ void warp_rows_k(long long *out, int rows, int ld, unsigned long long *ctr) {
  int lane = threadIdx.x & 31;
  while (true) {
    unsigned long long c = 0;
    if (lane == 0) c = atomicAdd(ctr, (unsigned long long)R);
    c = __shfl_sync(0xffffffffu, c, 0);
    if (c >= (unsigned long long)rows) break;
    const long long nr = min((unsigned long long)R, rows - c);
    long long *b = out + c * ld;
    const long long n2 = nr * ld / 2;
    for (long long i = lane; i < n2; i += 32) st2(b + 2 * i, c, i);
  }
}
void run(torch::Tensor out, int rows, int ld, torch::Tensor ctr, int mode) {
  auto *o = (long long *)out.data_ptr();
  auto *k = (unsigned long long *)ctr.data_ptr();
  if (mode == 0) linear_k<<<296, 512>>>(o, (long long)rows * ld / 2);
  else if (mode == 1) rows_k<<<296, 512>>>(o, rows, ld, k);
  else if (mode == 2) block_k<<<296, 512>>>(o, rows, ld, k);
  else if (mode == 3) {
    cudaFuncSetAttribute(rows_tma_k<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 2 * 1024);
    rows_tma_k<1024><<<296, 512, 16 * 2 * 1024>>>(o, rows, ld, k);
  } else if (mode == 4) {
    cudaFuncSetAttribute(rows_tma_k<2048>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 2 * 2048);
    rows_tma_k<2048><<<296, 512, 16 * 2 * 2048>>>(o, rows, ld, k);
  } else if (mode == 6) group_k<2><<<296, 512>>>(o, rows, ld, k);
  else if (mode == 7) group_k<4><<<296, 512>>>(o, rows, ld, k);
  else if (mode == 8) group_k<8><<<296, 512>>>(o, rows, ld, k);
  else if (mode == 9) rows256_k<<<296, 512>>>(o, rows, ld, k);
  else if (mode == 12) rows_k<<<296, 256>>>(o, rows, ld, k);
  else if (mode == 14) warp_rows_k<2><<<296, 512>>>(o, rows, ld, k);
  else if (mode == 15) warp_rows_k<4><<<296, 512>>>(o, rows, ld, k);
  else if (mode == 13) rows_k<<<296, 128>>>(o, rows, ld, k);
  else if (mode == 10) rows_wb_k<0><<<296, 512>>>(o, rows, ld, k);
  else if (mode == 11) rows_wb_k<1><<<296, 512>>>(o, rows, ld, k);
  else {
    cudaFuncSetAttribute(rows_tma_k<4096>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 2 * 4096);
    rows_tma_k<4096><<<296, 512, 16 * 2 * 4096>>>(o, rows, ld, k);
  }
}
"""
mod = load_inline("write_pattern", cpp_sources="void run(torch::Tensor out, int rows, int ld, torch::Tensor ctr, int mode);",
                  cuda_sources=SRC, functions=["run"], extra_cuda_cflags=["-O3", "-gencode", "arch=compute_100a,code=sm_100a"],
                  verbose=False)
rows = 100_000
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ctr = torch.zeros(1, dtype=torch.int64, device="cuda")
for ld in (2618, 2620):  # C2's row: 20,944 B (a 32 B sector split between rows) vs padded to 32 B
    out = torch.empty(rows * ld, dtype=torch.int64, device="cuda")
    print(f"-- ld = {ld} ({ld * 8} B rows, {'32 B-aligned' if ld % 4 == 0 else 'rows split 32 B sectors'})")
    modes = ((0, "linear grid-stride"), (1, "row per warp (replay pattern)"), (2, "16 rows per CTA, linear"),
             (3, "row per warp, TMA bulk 1 KiB"), (4, "row per warp, TMA bulk 2 KiB"),
             (5, "row per warp, TMA bulk 4 KiB"), (6, "2-warp groups, 2 rows linear"),
             (7, "4-warp groups, 4 rows linear"), (8, "8-warp groups, 8 rows linear"),
             (9, "row per warp, 256-bit stores"), (10, "row per warp, write-back stores"),
             (11, "row per warp, L1::no_allocate stores"), (12, "row per warp, 8 warps/CTA (2368 streams)"),
             (13, "row per warp, 4 warps/CTA (1184 streams)"), (14, "one warp, 2 rows linear"),
             (15, "one warp, 4 rows linear"))
    if ld % 4 == 0:
        modes = tuple(m for m in modes if m[0] in (0, 1, 2, 6, 14))
    for mode, name in modes:
        best = 1e9
        for it in range(8):
            ctr.zero_()
            torch.cuda._sleep(1_000_000)
            s.record()
            mod.run(out, rows, ld, ctr, mode)
            e.record()
            torch.cuda.synchronize()
            if it >= 2:
                best = min(best, s.elapsed_time(e))
        print(f"{name:42s} {rows * ld * 8 / (best * 1e-3) / 1e9:8.1f} GB/s  {best:.3f} ms")
    del out
