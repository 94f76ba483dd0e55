"""Write-pattern microbenchmark for the replay kernel's full mode (context only): 10^5 rows of
2618 int64 (the C2 footprint rows, 2.09 GB) written (a) as one linear grid-stride stream,
(b) one row per warp, rows handed out by an atomic counter (the replay kernel's pattern),
(c) 16 consecutive rows per CTA written as one linear block by all 512 threads.
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
void run(torch::Tensor out, int rows, int ld, torch::Tensor ctr, int mode) {
  auto *o = (long long *)out.data_ptr();
  auto *k = (unsigned long long *)ctr.data_ptr();
  if (mode == 0) linear_k<<<296, 512>>>(o, (long long)rows * ld / 2);
  else if (mode == 1) rows_k<<<296, 512>>>(o, rows, ld, k);
  else block_k<<<296, 512>>>(o, rows, ld, k);
}
"""
mod = load_inline("write_pattern", cpp_sources="void run(torch::Tensor out, int rows, int ld, torch::Tensor ctr, int mode);",
                  cuda_sources=SRC, functions=["run"], extra_cuda_cflags=["-O3", "-gencode", "arch=compute_100a,code=sm_100a"],
                  verbose=False)
rows, ld = 100_000, 2618
out = torch.empty(rows * ld, dtype=torch.int64, device="cuda")
ctr = torch.zeros(1, dtype=torch.int64, device="cuda")
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for mode, name in ((0, "linear grid-stride"), (1, "row per warp (replay pattern)"), (2, "16 rows per CTA, linear")):
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
    print(f"{name:34s} {rows * ld * 8 / (best * 1e-3) / 1e9:8.1f} GB/s  {best:.3f} ms")
