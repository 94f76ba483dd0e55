// trace.cpp -- trace build (step a3): tensor table, no-swap footprint F0, logical layers
// (Eq. 1), solo swap timing (Eq. 3, P:333 swap-in placement, P:340 swap-out completion),
// swappable set, default SEEDED base; upload of the device tables for the replay kernel.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <numeric>

#include "internal.h"

using namespace chm;

enum { kFWD = 0, kBWD = 1, kOPT = 2 };

// Logical layers when the caller gives no group count: the paper groups each phase evenly and
// finds the estimate reliable up to the model's layer count; a stacked model repeats
// one layer's operators, so the count is the phase length over the period p that best aligns the
// token sequence with itself shifted by p (the smallest p within 0.5% of the best match rate;
// embedding / head ops at the ends only lower every rate a little).
static int32_t auto_groups(const int32_t *tok, int32_t n) {
  if (n < 4) return 1;
  const int32_t pmax = std::min(n / 2, 4096);
  std::vector<double> rate(size_t(pmax) + 1, 0.0);
  double best = 0.0;
  for (int32_t p = 1; p <= pmax; p++) {
    int32_t m = 0;
    for (int32_t i = 0; i + p < n; i++) m += tok[i] == tok[i + p];
    rate[p] = double(m) / double(n - p);
    best = std::max(best, rate[p]);
  }
  if (best < 0.5) return 1;  // no repeated structure
  for (int32_t p = 1; p <= pmax; p++)
    if (rate[p] >= best - 0.005) return std::max(1, n / p);
  return 1;
}

extern "C" chm_status chm_trace_build(chm_ctx *ctx, const chm_trace_params *P, chm_trace **out) {
  CHM_NVTX("chm_trace_build");
  if (!ctx || !P || !out) CHM_FAIL(CHM_E_INVAL, "chm_trace_build: NULL argument");
  *out = nullptr;
  if (ctx->last_detailed.tokens.empty()) CHM_FAIL(CHM_E_STATE, "chm_trace_build: no Detailed-mode iteration recorded");
  return build_trace(ctx, ctx->last_detailed, P, out);
}

// the build proper, from the ctx's last Detailed record or a loaded file (trace_io.cpp)
chm_status chm::build_trace(chm_ctx *ctx, const IterRecord &R, const chm_trace_params *P, chm_trace **out) {
  *out = nullptr;
  if (!(P->bw_bytes_per_s > 0.0)) CHM_FAIL(CHM_E_INVAL, "chm_trace_build: B must be > 0 (Eq. 3)");
  const double t_iter = P->t_iter_s > 0.0 ? P->t_iter_s : R.t_iter;
  if (!(t_iter >= 0.0)) CHM_FAIL(CHM_E_INVAL, "chm_trace_build: T_iter < 0");
  const double omega = P->omega > 0.0 ? P->omega : 1.0;

  chm_trace *tr = new (std::nothrow) chm_trace();
  if (!tr) CHM_FAIL(CHM_E_NOMEM, "chm_trace_build: out of host memory");
  const int32_t N = int32_t(R.tokens.size()), T = int32_t(R.tensors.size());
  tr->device = ctx->device;
  tr->N = N;
  tr->T = T;
  tr->budget = P->hbm_budget;
  tr->M0 = P->static_bytes;
  tr->bw = P->bw_bytes_per_s;
  tr->t_iter = t_iter;

  // tensor table: producer p, refcount release f (N: survives), last FWD use a (production
  // counts), first BWD input use b
  tr->p.assign(T, -1); tr->f.assign(T, N); tr->a.assign(T, -1); tr->b.assign(T, -1);
  tr->S_t.resize(T);
  for (int32_t t = 0; t < T; t++) {
    tr->p[t] = R.tensors[t].producer;
    tr->f[t] = R.tensors[t].freed >= 0 ? R.tensors[t].freed : N;
    tr->S_t[t] = R.tensors[t].nbytes;
  }
  for (int32_t i = 0; i < N; i++) {
    for (int32_t u = R.use_ptr[i]; u < R.use_ptr[i + 1]; u++) {
      const int32_t t = R.use_idx[u];
      if (R.phase[i] == kFWD) tr->a[t] = std::max(tr->a[t], i);
      if (R.phase[i] == kBWD && R.use_is_in[u] && tr->b[t] < 0) tr->b[t] = i;
    }
  }
  // F0 by a difference array: a produced tensor is live on ops [p_t, f_t]; a static tensor
  // released during the iteration leaves after op f_t
  {
    std::vector<int64_t> d(size_t(N) + 1, 0);
    for (int32_t t = 0; t < T; t++) {
      if (tr->p[t] >= 0) {
        d[tr->p[t]] += tr->S_t[t];
        d[tr->f[t] + (tr->f[t] < N ? 1 : 0)] -= tr->S_t[t];
      } else if (tr->f[t] < N) {
        d[tr->f[t] + 1] -= tr->S_t[t];
      }
    }
    tr->F0.resize(N);
    int64_t acc = P->static_bytes;
    for (int32_t i = 0; i < N; i++) { acc += d[i]; tr->F0[i] = acc; }
  }
  if (P->f0_source == 1) {
    // Fig. 3: the no-swap footprint is the measured footprint of every op plus
    // the bytes the swap log has off the device at that op (span [from, to))
    if (R.live_bytes.size() != size_t(N)) { delete tr; CHM_FAIL(CHM_E_STATE, "chm_trace_build: no live bytes recorded"); }
    std::vector<int64_t> d(size_t(N) + 1, 0);
    for (const auto &sp : R.swaps) {
      const int32_t a = std::max(sp.from, 0), b = std::min(sp.to, N);
      if (a >= b) continue;
      d[a] += sp.nbytes;
      d[b] -= sp.nbytes;
    }
    int64_t acc = 0;
    for (int32_t i = 0; i < N; i++) {
      if (R.live_bytes[i] < 0) { delete tr; CHM_FAIL(CHM_E_INVAL, "chm_trace_build: op %d has live_bytes < 0", i); }
      acc += d[i];
      tr->F0[i] = R.live_bytes[i] + acc;
    }
  } else if (P->f0_source != 0) {
    delete tr;
    CHM_FAIL(CHM_E_INVAL, "chm_trace_build: f0_source %u", P->f0_source);
  }
  tr->argmax0 = 0;
  for (int32_t i = 1; i < N; i++) if (tr->F0[i] > tr->F0[tr->argmax0]) tr->argmax0 = i;
  tr->peak0 = tr->F0[tr->argmax0];

  // logical layers: near-even contiguous groups per phase (first n mod G groups one larger),
  // OPT one group; budget Bud = ((T_iter / N) * n_l) * omega (Eq. 1)
  int32_t nph[3] = {0, 0, 0};
  for (int32_t i = 0; i < N; i++) nph[R.phase[i]]++;
  int32_t G[3] = {int32_t(P->groups_fwd), int32_t(P->groups_bwd), nph[kOPT] > 0 ? 1 : 0};
  for (int ph = 0; ph < 2; ph++) {  // 0 groups: the phase's layer count, from its period
    if (G[ph] == 0 && nph[ph] > 0) G[ph] = auto_groups(R.tokens.data() + (ph ? nph[0] : 0), nph[ph]);
  }
  for (int ph = 0; ph < 2; ph++) {
    if (nph[ph] == 0) G[ph] = 0;
    else if (G[ph] < 1 || G[ph] > nph[ph]) {
      delete tr;
      CHM_FAIL(CHM_E_INVAL, "chm_trace_build: %d groups for %d ops of phase %d", G[ph], nph[ph], ph);
    }
  }
  tr->L = G[0] + G[1] + G[2];
  tr->lay_of_op.resize(N);
  int32_t op = 0, last_fwd = -1;
  for (int ph = 0; ph < 3; ph++) {
    for (int32_t g = 0; g < G[ph]; g++) {
      const int32_t n = nph[ph] / G[ph] + (g < nph[ph] % G[ph] ? 1 : 0);
      tr->lay_start.push_back(op);
      tr->lay_n.push_back(n);
      tr->lay_type.push_back(ph);
      tr->bud.push_back(((t_iter / double(N)) * double(n)) * omega);
      for (int32_t k = op; k < op + n; k++) tr->lay_of_op[k] = int32_t(tr->lay_start.size()) - 1;
      if (ph == kFWD) last_fwd = int32_t(tr->lay_start.size()) - 1;
      op += n;
    }
  }

  // solo timing + swappable set
  std::vector<int32_t> prod_rank(T, -1);
  {
    int32_t rk = 0;
    for (int32_t i = 0; i < N; i++)
      for (int32_t j = R.out_ptr[i]; j < R.out_ptr[i + 1]; j++) prod_rank[R.out_idx[j]] = rk++;
  }
  struct Cand { int32_t t, r, s; };
  std::vector<Cand> cands;
  for (int32_t t = 0; t < T; t++) {
    if (tr->p[t] < 0 || tr->a[t] < 0 || tr->b[t] < 0) continue;  // activations only
    const double tswap = double(tr->S_t[t]) / tr->bw;  // Eq. 3
    int32_t r = -1;
    for (int32_t l = tr->lay_of_op[tr->a[t]]; l <= last_fwd; l++)  // P:340, forward search
      if (tr->bud[l] > tswap) { r = tr->lay_start[l] + tr->lay_n[l] - 1; break; }
    if (r < 0) r = tr->lay_start[last_fwd] + tr->lay_n[last_fwd] - 1;  // saturated
    const int32_t lb = tr->lay_of_op[tr->b[t]];
    if (lb < 1) continue;
    const int32_t s = tr->lay_start[lb - 1];  // previous layer of the first BWD use
    if (!(r + 1 < s)) continue;               // empty off-device window
    cands.push_back({t, r, s});
  }
  std::sort(cands.begin(), cands.end(), [&](const Cand &x, const Cand &y) {
    if (tr->a[x.t] != tr->a[y.t]) return tr->a[x.t] < tr->a[y.t];
    return prod_rank[x.t] < prod_rank[y.t];
  });
  tr->K = int32_t(cands.size());
  tr->W = (tr->K + 63) / 64;
  tr->base.assign(size_t(tr->W), 0);
  for (int32_t k = 0; k < tr->K; k++) {
    const Cand &c = cands[k];
    tr->sw_t.push_back(uint32_t(prod_rank[c.t]));
    tr->sw_S.push_back(tr->S_t[c.t]);
    tr->sw_r.push_back(c.r);
    tr->sw_s.push_back(c.s);
    tr->sw_lin.push_back(tr->lay_of_op[c.s]);
    tr->sw_lout.push_back(tr->lay_of_op[c.r]);
    if (c.r < tr->argmax0 && tr->argmax0 < c.s) tr->base[k / 64] |= 1ull << (k % 64);
  }
  // keep what policy install needs (App. A features over the recorded iteration)
  tr->tokens = R.tokens;
  tr->use_ptr = R.use_ptr;
  tr->use_idx = R.use_idx;
  tr->dtype.resize(T);
  for (int32_t t = 0; t < T; t++) tr->dtype[t] = R.tensors[t].dtype;
  tr->tensor_rank = prod_rank;
  tr->rank_to_tensor.assign(size_t(R.out_idx.size()), -1);
  for (int32_t t = 0; t < T; t++) if (prod_rank[t] >= 0) tr->rank_to_tensor[prod_rank[t]] = t;
  // swappable k -> product tensor index (kept for install)
  std::vector<int32_t> sw_tensor(tr->K);
  for (int32_t k = 0; k < tr->K; k++) sw_tensor[k] = cands[k].t;
  tr->sw_tensor_idx = std::move(sw_tensor);

  // replay image (see DevTrace): with solo timing every release r_t is the last op of layer
  // lout_t and every swap-in s_t the first op of layer lin_t, so a candidate's footprint offset
  // is constant per logical layer; the image holds what the kernel needs for that form
  // bounds of the kernel's exact 32-bit partial sums (hi = S >> 16, lo = S & 0xffff)
  int64_t sum_S = 0;
  for (int32_t k = 0; k < tr->K; k++) sum_S += tr->sw_S[k];
  if (tr->K > 32767 || tr->L > 256 || sum_S >= (int64_t(1) << 47)) {
    chm_trace_free(tr);
    CHM_FAIL(CHM_E_INVAL, "chm_trace_build: K = %d, L = %d, sum S = %lld exceed the replay image bounds "
             "(K < 32768, L <= 256, sum S < 2^47)", tr->K, tr->L, (long long)sum_S);
  }
  auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
  DevTrace &D = tr->dev;
  size_t o = 0;
  D.o_mf0 = uint32_t(o); o += al(8 * size_t(tr->L));
  D.o_bud = uint32_t(o); o += al(8 * size_t(tr->L));
  D.o_S = uint32_t(o); o += al(8 * size_t(tr->K));
  D.o_lo = uint32_t(o); o += al(2 * size_t(tr->K));
  D.o_li = uint32_t(o); o += al(2 * size_t(tr->K));
  D.search_bytes = uint32_t(o);
  // F0 in int32 units of 2^g bytes when every value is a multiple of 2^g (g <= 9, the allocator
  // block) and fits: halves the row stream's shared-memory reads
  int g = 9;
  int64_t fmax = 0;
  bool nonneg = true;
  for (int32_t i = 0; i < N; i++) {
    while (g > 0 && (tr->F0[i] & ((int64_t(1) << g) - 1))) g--;
    fmax = std::max(fmax, tr->F0[i]);
    nonneg = nonneg && tr->F0[i] >= 0;
  }
  D.f0_narrow = nonneg && (fmax >> g) < (int64_t(1) << 31) ? 1 : 0;
  D.f0_shift = g;
  // narrow: F0 and the ops' layers lane-swizzled for the row stream (see replay.cu): in each
  // block of 128 ops, lane l's four ops 2l, 2l+1, 64+2l, 65+2l are stored together (one 16 B
  // load of F0, one 32-bit load of the u8 layers); wide: F0 int64 and u16 8 x layer in op order
  const size_t n128 = (size_t(N) + 127) / 128 * 128;
  if (D.f0_narrow) {
    D.o_f0 = uint32_t(o); o += al(4 * n128);
    D.o_lay4 = uint32_t(o); o += al(2 * n128);  // per (block, lane): two pairs' D offsets
    D.full_bytes = uint32_t(o);
    D.o_lay = uint32_t(o); o += al(2 * size_t(N));  // EXPLICIT replay only (global memory)
  } else {
    D.o_f0 = uint32_t(o); o += al(8 * size_t(N));
    D.o_lay = uint32_t(o); o += al(2 * size_t(N));
    D.o_lay4 = 0;
    D.full_bytes = uint32_t(o);
  }
  D.o_f0w = uint32_t(o); o += al(8 * size_t(N));
  const size_t o_base = al(o);
  const size_t total = o_base + al(8 * size_t(tr->W) + 8);
  std::vector<unsigned char> host(total, 0);
  unsigned char *h = host.data();
  std::vector<int64_t> mf0(size_t(tr->L), INT64_MIN);
  for (int32_t i = 0; i < N; i++) mf0[tr->lay_of_op[i]] = std::max(mf0[tr->lay_of_op[i]], tr->F0[i]);
  std::memcpy(h + D.o_mf0, mf0.data(), 8 * size_t(tr->L));
  std::memcpy(h + D.o_bud, tr->bud.data(), 8 * size_t(tr->L));
  if (tr->K) std::memcpy(h + D.o_S, tr->sw_S.data(), 8 * size_t(tr->K));
  std::vector<uint16_t> lo16(tr->K), li16(tr->K);
  for (int32_t k = 0; k < tr->K; k++) {
    lo16[k] = uint16_t(tr->sw_lout[k]);
    li16[k] = uint16_t(tr->sw_lin[k]);
  }
  if (tr->K) {
    std::memcpy(h + D.o_lo, lo16.data(), 2 * size_t(tr->K));
    std::memcpy(h + D.o_li, li16.data(), 2 * size_t(tr->K));
  }
  if (D.f0_narrow) {  // swizzled position of op i: block i / 128, lane (i % 64) / 2, slot
    const int E = chm::layers_per_lane(tr->L);
    std::vector<int32_t> f0u(n128, 0);
    for (size_t i = 0; i < n128; i++) {
      const size_t blk = i / 128, w = i % 128, lane = (w % 64) / 2, slot = (w / 64) * 2 + (w % 2);
      const size_t at = blk * 128 + 4 * lane + slot;
      const size_t src = std::min(i, size_t(N) - 1);  // padding: the last op's layer, F0 0
      f0u[at] = i < size_t(N) ? int32_t(tr->F0[i] >> D.f0_shift) : 0;
      // u16 byte offset of op i's layer into the warp's padded D row, at (block, lane, slot)
      const uint16_t off = uint16_t(8 * chm::layer_slot(tr->lay_of_op[src], E));  // L <= 256 (checked above)
      std::memcpy(h + D.o_lay4 + 2 * at, &off, 2);
    }
    std::memcpy(h + D.o_f0, f0u.data(), 4 * n128);
  } else {
    std::memcpy(h + D.o_f0, tr->F0.data(), 8 * size_t(N));
  }
  std::memcpy(h + D.o_f0w, tr->F0.data(), 8 * size_t(N));
  std::vector<uint16_t> lay16(N);
  for (int32_t i = 0; i < N; i++) lay16[i] = uint16_t(8 * tr->lay_of_op[i]);  // byte offset into D[L]
  std::memcpy(h + D.o_lay, lay16.data(), 2 * size_t(N));
  if (tr->W) std::memcpy(h + o_base, tr->base.data(), 8 * size_t(tr->W));
  D.N = N;
  D.K = tr->K;
  D.L = tr->L;
  D.W = tr->W;
  D.bw = tr->bw;
  D.rbw = (tr->bw > std::ldexp(1.0, -500) && tr->bw < std::ldexp(1.0, 500)) ? 1.0 / tr->bw : 0.0;
  D.budget = tr->budget;
  if (ctx->device < 0) {  // host-only ctx: tables stay on the host
    *out = tr;
    return CHM_OK;
  }
  DeviceGuard dg(ctx->device);
  cudaError_t e = dg.status;
  if (e == cudaSuccess) e = cudaMalloc(&tr->dev_block, total);
  if (e == cudaSuccess) e = cudaMemcpy(tr->dev_block, host.data(), total, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    chm_trace_free(tr);
    CHM_FAIL(CHM_E_CUDA, "chm_trace_build: device upload failed: %s", cudaGetErrorString(e));
  }
  D.image = static_cast<const unsigned char *>(tr->dev_block);
  D.base = reinterpret_cast<const uint64_t *>(static_cast<char *>(tr->dev_block) + o_base);
  *out = tr;
  return CHM_OK;
}

extern "C" void chm_trace_free(chm_trace *t) {
  if (!t) return;
  if ((t->dev_block || t->tl_dev) && t->device >= 0) {
    DeviceGuard dg(t->device);
    if (t->dev_block) cudaFree(t->dev_block);
    if (t->tl_dev) cudaFree(t->tl_dev);
  }
  delete t;
}

extern "C" chm_status chm_trace_get_info(const chm_trace *t, chm_trace_info *info) {
  if (!t || !info) CHM_FAIL(CHM_E_INVAL, "chm_trace_get_info: NULL argument");
  info->n_ops = uint32_t(t->N);
  info->n_tensors = uint32_t(t->T);
  info->n_swappable = uint32_t(t->K);
  info->n_layers = uint32_t(t->L);
  info->mask_words = uint32_t(t->W);
  info->peak0 = t->peak0;
  info->argmax0 = uint32_t(t->argmax0);
  info->budget = t->budget;
  return CHM_OK;
}

extern "C" chm_status chm_trace_tables(const chm_trace *t, int64_t *f0, uint32_t *tensor,
                                       int64_t *nbytes, int32_t *r, int32_t *s, int32_t *lin,
                                       int32_t *lout, int32_t *lay_start, int32_t *lay_count,
                                       double *bud, uint64_t *base) {
  if (!t) CHM_FAIL(CHM_E_INVAL, "chm_trace_tables: NULL trace");
  if (f0) std::copy(t->F0.begin(), t->F0.end(), f0);
  if (tensor) std::copy(t->sw_t.begin(), t->sw_t.end(), tensor);
  if (nbytes) std::copy(t->sw_S.begin(), t->sw_S.end(), nbytes);
  if (r) std::copy(t->sw_r.begin(), t->sw_r.end(), r);
  if (s) std::copy(t->sw_s.begin(), t->sw_s.end(), s);
  if (lin) std::copy(t->sw_lin.begin(), t->sw_lin.end(), lin);
  if (lout) std::copy(t->sw_lout.begin(), t->sw_lout.end(), lout);
  if (lay_start) std::copy(t->lay_start.begin(), t->lay_start.end(), lay_start);
  if (lay_count) std::copy(t->lay_n.begin(), t->lay_n.end(), lay_count);
  if (bud) std::copy(t->bud.begin(), t->bud.end(), bud);
  if (base) std::copy(t->base.begin(), t->base.end(), base);
  return CHM_OK;
}

namespace {
struct Fnv64 {  // FNV-1a over the bytes of each field, in a fixed order
  uint64_t h = 0xcbf29ce484222325ull;
  void bytes(const void *p, size_t n) {
    const unsigned char *c = static_cast<const unsigned char *>(p);
    for (size_t i = 0; i < n; i++) { h ^= c[i]; h *= 0x100000001b3ull; }
  }
  template <class T> void pod(const T &v) { bytes(&v, sizeof v); }
  template <class T> void vec(const std::vector<T> &v) { pod(uint64_t(v.size())); bytes(v.data(), v.size() * sizeof(T)); }
};
}  // namespace

extern "C" chm_status chm_trace_digest(const chm_trace *t, uint64_t *digest) {
  if (!t || !digest) CHM_FAIL(CHM_E_INVAL, "chm_trace_digest: NULL argument");
  Fnv64 f;
  f.pod(t->N); f.pod(t->K); f.pod(t->L); f.pod(t->W);
  f.pod(t->budget); f.pod(t->M0); f.pod(t->bw); f.pod(t->t_iter);
  f.vec(t->F0); f.vec(t->lay_start); f.vec(t->lay_n); f.vec(t->bud);
  f.vec(t->sw_S); f.vec(t->sw_r); f.vec(t->sw_s); f.vec(t->sw_lin); f.vec(t->sw_lout); f.vec(t->base);
  *digest = f.h;
  return CHM_OK;
}
