// descend.cu -- chm_descend: steepest single-flip descent over swap masks on the device (reading
// R-search: the planner's search around the evaluator, "generates five
// different policies and selects the one with the best runtime performance"), one CTA per start
// mask, every round on the device.
//
// A round scores the K masks that differ from the current one in one bit under R-stall and
// moves to the argmin of (excess, stall, swapped, k) if its first three fields are smaller than
// the current mask's; the same trajectory as the host loop of FLIP1 launches
// (runtime.descend) and the oracle's descend, bit for bit.  A neighbour is scored from per-round
// tables instead of a replay: flipping item k (layers lout_k < lin_k, lin_k >= lout_k + 2 by the
// trace build's swappable rule) changes D by -/+S_k on the layers strictly between lout_k and
// lin_k only (F_P[i] = F0[i] - sum S_t [r_t < i < s_t], §8(c).2, with r_t the last op of lout and
// s_t the first op of lin), the loads of layers lin_k and lout_k by +/-S_k, swapped by +/-S_k:
//   peak'  = max(prefix max of P up to lout, suffix max from lin, range max over (lout, lin) + dD)
//            with P_l = max F0 over layer l + D_l (a sparse table answers the range max);
//   stall' = the pairwise tree of the L terms (zero-padded to a power of two) with the two
//            changed leaves re-summed along their paths (the other nodes are this round's);
// the same integers and the same IEEE additions in the same tree order as the replay kernel.
#include <climits>

#include "eval_common.cuh"

namespace chm {
namespace {

constexpr int kDescThreads = 256;

struct DescParams {
  DevTrace tr;
  uint32_t stage_bytes;
  const uint64_t *starts;
  uint64_t *ends;
  Key *keys;
  int32_t *rounds;
  uint32_t n_starts, max_rounds;
  int P2, LG;  // leaves of the stall tree (power of two >= L), sparse-table levels above P
  uint32_t o_mask, o_in, o_out, o_p, o_pm, o_sm, o_st, o_tree, o_acc;  // shared-memory offsets
};

__device__ __forceinline__ long long split_sum2(unsigned hi, unsigned lo) {
  return (long long)(int)hi * 65536 + (long long)(int)lo;
}

__device__ __forceinline__ double stall_term(long long load, const DevTrace &tr, double bud) {
  const double v = double(load);
  const double x = __dsub_rn(tr.rbw != 0.0 ? div_rn_rcp(v, tr.bw, tr.rbw) : __ddiv_rn(v, tr.bw), bud);
  return x > 0.0 ? x : 0.0;
}

__device__ __forceinline__ long long max64(long long a, long long b) { return a > b ? a : b; }

__global__ void __launch_bounds__(kDescThreads) descend_kernel(const __grid_constant__ DescParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ Key s_wkey[kDescThreads / 32];
  __shared__ long long s_swapped;
  __shared__ int s_move;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int K = p.tr.K, L = p.tr.L, W = p.tr.W, P2 = p.P2;
  // the trace image's search part (per-layer max F0, budgets, S, lout, lin), staged once
  for (uint32_t o = 16u * tid; o < p.stage_bytes; o += 16u * blockDim.x)
    *reinterpret_cast<uint4 *>(smem + o) = __ldg(reinterpret_cast<const uint4 *>(p.tr.image + o));
  const long long *mf0 = reinterpret_cast<const long long *>(smem + p.tr.o_mf0);
  const double *bud = reinterpret_cast<const double *>(smem + p.tr.o_bud);
  const long long *S = reinterpret_cast<const long long *>(smem + p.tr.o_S);
  const unsigned short *lo_ = reinterpret_cast<const unsigned short *>(smem + p.tr.o_lo);
  const unsigned short *li_ = reinterpret_cast<const unsigned short *>(smem + p.tr.o_li);
  uint64_t *mask = reinterpret_cast<uint64_t *>(smem + p.o_mask);   // [W]
  long long *IN = reinterpret_cast<long long *>(smem + p.o_in);     // [L] bytes swapped in at l
  long long *OUT = reinterpret_cast<long long *>(smem + p.o_out);   // [L] bytes released at l
  long long *P = reinterpret_cast<long long *>(smem + p.o_p);       // [L] max F0 + D
  long long *PM = reinterpret_cast<long long *>(smem + p.o_pm);     // [L] prefix max of P
  long long *SM = reinterpret_cast<long long *>(smem + p.o_sm);     // [L] suffix max of P
  long long *ST = reinterpret_cast<long long *>(smem + p.o_st);     // [LG][L] level j: max P[l, l + 2^j)
  double *tree = reinterpret_cast<double *>(smem + p.o_tree);       // [2 P2] heap, leaves at P2 + l
  unsigned *acc = reinterpret_cast<unsigned *>(smem + p.o_acc);     // [4L] hi / lo accumulators
  auto st_at = [&](int j, int l) -> long long { return j == 0 ? P[l] : ST[(j - 1) * L + l]; };

  for (uint32_t sidx = blockIdx.x; sidx < p.n_starts; sidx += gridDim.x) {
    __syncthreads();  // the previous start's tables are done with (and the image staged)
    for (int w = tid; w < W; w += blockDim.x) mask[w] = p.starts[uint64_t(sidx) * W + w];
    for (int l = tid; l < 4 * L; l += blockDim.x) acc[l] = 0u;
    __syncthreads();
    // per-layer in / out sums of the start mask (exact split accumulators, as the replay's)
    for (int k = tid; k < K; k += blockDim.x) {
      if (!((mask[k >> 6] >> (k & 63)) & 1ull)) continue;
      const long long s = S[k];
      const unsigned h = unsigned(s >> 16), w = unsigned(s & 0xffff);
      atomicAdd(acc + li_[k], h);
      atomicAdd(acc + L + li_[k], w);
      atomicAdd(acc + 2 * L + lo_[k], h);
      atomicAdd(acc + 3 * L + lo_[k], w);
    }
    __syncthreads();
    for (int l = tid; l < L; l += blockDim.x) {
      IN[l] = split_sum2(acc[l], acc[L + l]);
      OUT[l] = split_sum2(acc[2 * L + l], acc[3 * L + l]);
    }
    __syncthreads();
    if (warp == 0) {  // swapped = every selected item's bytes, once (at its release layer)
      long long sw = 0;
      for (int l = lane; l < L; l += 32) sw += OUT[l];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sw += __shfl_xor_sync(0xffffffffu, sw, o);
      if (lane == 0) s_swapped = sw;
    }
    uint32_t round = 0;
    Key cur;
    while (true) {
      // ---- this mask's tables, warp-synchronous (one CTA barrier per rebuild): warp 0 builds D,
      // P, its prefix / suffix maxima and the sparse table, warp 1 the stall tree
      if (warp == 0) {
        long long ci = 0, co = 0, pmax = LLONG_MIN;
        for (int l0 = 0; l0 < L; l0 += 32) {
          const int l = l0 + lane;
          const long long in_l = l < L ? IN[l] : 0, out_l = l < L ? OUT[l] : 0;
          long long a = in_l, b = out_l;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const long long ya = __shfl_up_sync(0xffffffffu, a, o), yb = __shfl_up_sync(0xffffffffu, b, o);
            if (lane >= o) { a += ya; b += yb; }
          }
          // D_l = CI(l) - CO(l) + out_l (the replay's layer-segment form)
          const long long pl = l < L ? mf0[l] + ((ci + a) - (co + b) + out_l) : LLONG_MIN;
          long long m = pl;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, m, o);
            if (lane >= o) m = max64(m, y);
          }
          if (l < L) { P[l] = pl; PM[l] = max64(pmax, m); }
          ci += __shfl_sync(0xffffffffu, a, 31);
          co += __shfl_sync(0xffffffffu, b, 31);
          pmax = max64(pmax, __shfl_sync(0xffffffffu, m, 31));
        }
        __syncwarp();
        long long smax = LLONG_MIN;
        for (int l0 = ((L - 1) >> 5) << 5; l0 >= 0; l0 -= 32) {
          const int l = l0 + lane;
          long long m = l < L ? P[l] : LLONG_MIN;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_down_sync(0xffffffffu, m, o);
            if (lane + o < 32) m = max64(m, y);
          }
          if (l < L) SM[l] = max64(smax, m);
          smax = max64(smax, __shfl_sync(0xffffffffu, m, 0));
        }
        __syncwarp();
        // the sparse table of P, level by level inside the warp (no CTA barrier per level)
        for (int it = 1; it <= p.LG; it++) {
          const int half = 1 << (it - 1), n = L - (1 << it) + 1;
          for (int l = lane; l < n; l += 32) ST[(it - 1) * L + l] = max64(st_at(it - 1, l), st_at(it - 1, l + half));
          __syncwarp();
        }
      } else if (warp == 1) {  // the stall tree: leaves, then the pairwise levels (left + right)
        for (int l = lane; l < P2; l += 32) tree[P2 + l] = l < L ? stall_term(IN[l] + OUT[l], p.tr, bud[l]) : 0.0;
        __syncwarp();
        for (int h = P2 >> 1; h >= 1; h >>= 1) {
          for (int i = lane; i < h; i += 32) tree[h + i] = __dadd_rn(tree[2 * (h + i)], tree[2 * (h + i) + 1]);
          __syncwarp();
        }
      }
      __syncthreads();
      const long long pk0 = PM[L - 1], sw0 = s_swapped;
      cur.excess = pk0 > p.tr.budget ? pk0 - p.tr.budget : 0;
      cur.stall = P2 > 0 ? tree[1] : 0.0;
      cur.swapped = sw0;
      cur.index = sidx;
      cur.peak = pk0;
      if (round >= p.max_rounds || K == 0) break;
      // ---- every single-flip neighbour
      Key b = key_none();
      for (int k = tid; k < K; k += blockDim.x) {
        const bool in_mask = (mask[k >> 6] >> (k & 63)) & 1ull;
        const long long dS = in_mask ? -S[k] : S[k];  // swapped, load of lin and of lout
        const int lo = lo_[k], li = li_[k];
        CHM_DCHECK(lo + 2 <= li && li < L);
        long long pk = max64(PM[lo], SM[li]);
        {
          const int a = lo + 1, len = li - 1 - a + 1, j = 31 - __clz(len);
          pk = max64(pk, max64(st_at(j, a), st_at(j, li - (1 << j))) - dS);
        }
        // the two changed leaves' paths to the root
        int ia = P2 + li, ib = P2 + lo;
        double va = stall_term(IN[li] + dS + OUT[li], p.tr, bud[li]);
        double vb = stall_term(IN[lo] + OUT[lo] + dS, p.tr, bud[lo]);
        bool two = true;
        while (ia > 1) {
          if (two && (ia ^ 1) == ib) {
            va = (ia & 1) ? __dadd_rn(vb, va) : __dadd_rn(va, vb);
            two = false;
          } else {
            const double sa = tree[ia ^ 1];
            va = (ia & 1) ? __dadd_rn(sa, va) : __dadd_rn(va, sa);
            if (two) {
              const double sb = tree[ib ^ 1];
              vb = (ib & 1) ? __dadd_rn(sb, vb) : __dadd_rn(vb, sb);
              ib >>= 1;
            }
          }
          ia >>= 1;
        }
        Key n;
        n.excess = pk > p.tr.budget ? pk - p.tr.budget : 0;
        n.stall = va;
        n.swapped = sw0 + dS;
        n.index = uint64_t(k);
        n.peak = pk;
        if (key_less(n, b)) b = n;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const Key y = key_shfl_xor(b, o);
        if (key_less(y, b)) b = y;
      }
      if (lane == 0) s_wkey[warp] = b;
      __syncthreads();
      if (tid == 0) {
        Key m = s_wkey[0];
        for (int w = 1; w < kDescThreads / 32; w++) if (key_less(s_wkey[w], m)) m = s_wkey[w];
        const bool better = m.excess != cur.excess ? m.excess < cur.excess
                            : m.stall != cur.stall ? m.stall < cur.stall
                                                   : m.swapped < cur.swapped;
        s_move = better ? 1 : 0;
        if (better) {  // move: the mask bit, the two layers' loads, swapped
          const int k = int(m.index);
          const bool in_mask = (mask[k >> 6] >> (k & 63)) & 1ull;
          const long long dS = in_mask ? -S[k] : S[k];
          mask[k >> 6] ^= 1ull << (k & 63);
          IN[li_[k]] += dS;
          OUT[lo_[k]] += dS;
          s_swapped += dS;
        }
      }
      __syncthreads();
      if (!s_move) break;
      round++;
    }
    for (int w = tid; w < W; w += blockDim.x) p.ends[uint64_t(sidx) * W + w] = mask[w];
    if (tid == 0) {
      p.keys[sidx] = cur;
      if (p.rounds) p.rounds[sidx] = int32_t(round);
    }
  }
}

}  // namespace
}  // namespace chm

using namespace chm;

extern "C" chm_status chm_descend(chm_ctx *ctx, const chm_trace *t, const uint64_t *starts, uint32_t n_starts,
                                  uint32_t max_rounds, uint64_t *ends, chm_best *keys, int32_t *rounds,
                                  chm_best *best, cudaStream_t stream) {
  CHM_NVTX("chm_descend");
  if (!ctx || !t || !starts || !ends || !keys || n_starts == 0) CHM_FAIL(CHM_E_INVAL, "chm_descend: bad argument");
  if (ctx->device < 0 || !t->dev_block) CHM_FAIL(CHM_E_STATE, "chm_descend: host-only ctx / trace");
  if (t->device != ctx->device) CHM_FAIL(CHM_E_INVAL, "chm_descend: trace on another device");
  if (starts != ends && reinterpret_cast<const char *>(starts) < reinterpret_cast<const char *>(ends + size_t(n_starts) * t->W) &&
      reinterpret_cast<const char *>(ends) < reinterpret_cast<const char *>(starts + size_t(n_starts) * t->W))
    CHM_FAIL(CHM_E_INVAL, "chm_descend: starts and ends overlap without being the same array");
  const DevTrace &tr = t->dev;
  const int L = tr.L;
  if (L < 1) CHM_FAIL(CHM_E_INVAL, "chm_descend: trace without layers");
  DescParams p{};
  p.tr = tr;
  p.stage_bytes = tr.search_bytes;
  p.starts = starts;
  p.ends = ends;
  p.keys = reinterpret_cast<Key *>(keys);
  p.rounds = rounds;
  p.n_starts = n_starts;
  p.max_rounds = max_rounds;
  int P2 = 1;
  while (P2 < L) P2 *= 2;
  int LG = 0;
  while ((2 << LG) <= L) LG++;  // levels 1 .. LG: windows of 2 .. 2^LG <= L
  p.P2 = P2;
  p.LG = LG;
  auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
  size_t o = al(tr.search_bytes);
  p.o_mask = uint32_t(o); o += al(8 * size_t(tr.W) + 8);
  p.o_in = uint32_t(o); o += al(8 * size_t(L));
  p.o_out = uint32_t(o); o += al(8 * size_t(L));
  p.o_p = uint32_t(o); o += al(8 * size_t(L));
  p.o_pm = uint32_t(o); o += al(8 * size_t(L));
  p.o_sm = uint32_t(o); o += al(8 * size_t(L));
  p.o_st = uint32_t(o); o += al(8 * size_t(L) * size_t(LG) + 8);
  p.o_tree = uint32_t(o); o += al(16 * size_t(P2));
  p.o_acc = uint32_t(o); o += al(16 * size_t(L));
  const size_t smem = o;
  if (smem > 220 * 1024) CHM_FAIL(CHM_E_INVAL, "chm_descend: trace tables (%zu B) exceed shared memory", smem);
  CHM_DEVICE_SCOPE(ctx->device);
  auto kern = descend_kernel;
  CHM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  int per_sm = 0;
  CHM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kDescThreads, smem));
  if (per_sm < 1) CHM_FAIL(CHM_E_INVAL, "chm_descend: kernel does not fit an SM");
  const uint32_t grid = std::min<uint32_t>(n_starts, uint32_t(ctx->num_sms) * uint32_t(per_sm));
  kern<<<grid, kDescThreads, smem, stream>>>(p);
  CHM_CUDA(cudaGetLastError());
  if (best) return chm_best_reduce_device(ctx, keys, n_starts, best, stream);
  return CHM_OK;
}

namespace chm {
cudaError_t preload_descend() {
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(descend_kernel));
}
}  // namespace chm
