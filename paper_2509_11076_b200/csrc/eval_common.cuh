// eval_common.cuh -- device pieces shared by the evaluation kernels (replay.cu, timeline.cu):
// the argmin key and the splitmix64 finaliser of SEEDED candidates.
#pragma once

#include "internal.h"

namespace chm {

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

__device__ __forceinline__ Key key_none() {
  Key b;
  b.excess = LLONG_MAX; b.stall = 0.0; b.swapped = LLONG_MAX; b.index = ~0ull; b.peak = 0;
  return b;
}

__device__ __forceinline__ Key key_shfl_xor(const Key &b, int o) {
  Key y;
  y.excess = __shfl_xor_sync(0xffffffffu, b.excess, o);
  y.stall = __shfl_xor_sync(0xffffffffu, b.stall, o);
  y.swapped = __shfl_xor_sync(0xffffffffu, b.swapped, o);
  y.index = __shfl_xor_sync(0xffffffffu, b.index, o);
  y.peak = __shfl_xor_sync(0xffffffffu, b.peak, o);
  return y;
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {  // splitmix64 finaliser
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// x / b rounded to nearest (bit-equal to __ddiv_rn(x, b) and to the oracle's C division) for
// x >= 0 an integer below 2^53 (a layer's swap bytes) and y = RN(1/b) with 2^-500 < b < 2^500
// (the host sets y, else 0 and the caller divides): q = RN(x y) is within one ulp of x / b,
// r = x - b q is exact under the FMA, and RN(q + r y) = RN(x / b) (Markstein's correction
// theorem).  Three FP64 operations instead of the division's reciprocal refinement and the
// out-of-line slow path it takes whenever x = 0, i.e. for every layer without swap traffic
// (ncu, r02: 2 slow-path calls per candidate on C3h).  Checked against the division on 3 x 10^9
// random (x, b) pairs, mantissa edge cases included (tools/div_check.c).
__device__ __forceinline__ double div_rn_rcp(double x, double b, double y) {
  const double q = __dmul_rn(x, y);
  const double r = __fma_rn(-q, b, x);
  return __fma_rn(r, y, q);
}

}  // namespace chm
