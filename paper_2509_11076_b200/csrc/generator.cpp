// generator.cpp -- NEXT-1: the paper's policy generator, Algo. 2, on the
// host, over a built trace.  Its policies are EXPLICIT candidates for chm_eval_policies (the
// GPU replay gives their true footprint / peak / stall) and for chm_policy_install_items.
//
//   MRL        per-op required reduction, F0[i] - budget where positive        (§5.2)
//   CL         unselected activations whose [a_t, b_t) holds an MRE, scored
//              N_MRE / max + C * S / max (Eq. 2), descending                   (§5.3)
//   swap-in    per candidate: from the layer before lay(b_t) backward, not past the layer of the
//              first MRE it covers nor into its swap-out layer, the first layer with
//              T_remaining > T_swap = S/B (Eq. 3); else the next candidate; if none fits, the
//              highest-score candidate goes to the layer before lay(b_t)    (§5.4.1)
//              then T_remaining -= T_swap and the MREs of the ops it is off device for shrink
//   SetFreeTime in swap-out order, from lay(a_t) forward to two layers before the swap-in layer,
//              the first layer with T_remaining > T_swap; release after its last op (§5.4.2)
#include <algorithm>
#include <cstring>
#include <vector>

#include "internal.h"

using namespace chm;

namespace {

struct Cand {
  int32_t rank;  // production-order tensor index (the EXPLICIT item's t)
  int32_t tid;   // recorded tensor index
  double score;
};

}  // namespace

extern "C" chm_status chm_generate_policy(const chm_trace *tr, const chm_gen_params *gp, chm_item *items,
                                          uint32_t cap, uint32_t *n_items, int32_t *feasible) {
  CHM_NVTX("chm_generate_policy");
  if (!tr || !gp || !n_items || (cap && !items)) CHM_FAIL(CHM_E_INVAL, "chm_generate_policy: NULL argument");
  if (!(gp->rem_scale >= 0.0)) CHM_FAIL(CHM_E_INVAL, "chm_generate_policy: rem_scale < 0");
  const int32_t N = tr->N, L = tr->L;
  const std::vector<int32_t> &lay = tr->lay_of_op;
  std::vector<int64_t> mre(N);
  int64_t n_pos = 0;  // MREs still > 0
  for (int32_t i = 0; i < N; i++) {
    mre[i] = tr->F0[i] > tr->budget ? tr->F0[i] - tr->budget : 0;
    n_pos += mre[i] > 0;
  }
  // next_pos: first op >= i whose MRE is still > 0 (N: none); MREs only ever drop to 0, so a
  // path-compressed "next" forest answers it in near-constant time
  std::vector<int32_t> nxt(size_t(N) + 1);
  for (int32_t i = 0; i <= N; i++) nxt[i] = (i < N && mre[i] <= 0) ? i + 1 : i;
  auto next_pos = [&](int32_t i) {
    int32_t r = i;
    while (nxt[r] != r) r = nxt[r];
    while (nxt[i] != r) { const int32_t t = nxt[i]; nxt[i] = r; i = t; }
    return r;
  };
  std::vector<double> rem(L);
  for (int32_t l = 0; l < L; l++) rem[l] = tr->bud[l] * gp->rem_scale;
  auto mrl_empty = [&]() { return n_pos == 0; };
  auto credit = [&](int32_t tid, int32_t sp) {  // the tensor is off device for ops (a_t, s_t)
    for (int32_t i = tr->a[tid] + 1; i < sp; i++) {
      if (mre[i] <= 0) continue;
      mre[i] = std::max<int64_t>(0, mre[i] - tr->S_t[tid]);
      if (mre[i] == 0) { n_pos--; nxt[i] = i + 1; }
    }
  };
  std::vector<int32_t> pos_prefix(size_t(N) + 1, 0);  // # MREs > 0 in ops [0, i), per round
  const int32_t n_prod = int32_t(tr->rank_to_tensor.size());
  std::vector<char> selected(n_prod, 0);
  struct Placed { int32_t rank, tid, s; uint32_t flags; };
  std::vector<Placed> placed;
  bool ok = true;
  while (!mrl_empty()) {
    std::vector<Cand> cl;
    int32_t max_n = 0;
    int64_t max_s = 0;
    for (int32_t i = 0; i < N; i++) pos_prefix[i + 1] = pos_prefix[i] + (mre[i] > 0);
    for (int32_t rk = 0; rk < n_prod; rk++) {
      const int32_t tid = tr->rank_to_tensor[rk];
      if (selected[rk] || tr->a[tid] < 0 || tr->b[tid] < 0) continue;
      const int32_t cnt = tr->b[tid] > tr->a[tid] ? pos_prefix[tr->b[tid]] - pos_prefix[tr->a[tid]] : 0;
      if (!cnt) continue;
      cl.push_back({rk, tid, double(cnt)});
      max_n = std::max(max_n, cnt);
      max_s = std::max(max_s, tr->S_t[tid]);
    }
    if (cl.empty()) { ok = false; break; }  // Algo. 2 "Raise Error"
    for (Cand &c : cl) c.score = c.score / double(max_n) + gp->C * (double(tr->S_t[c.tid]) / double(max_s));
    std::stable_sort(cl.begin(), cl.end(), [&](const Cand &x, const Cand &y) {
      if (x.score != y.score) return x.score > y.score;
      if (tr->S_t[x.tid] != tr->S_t[y.tid]) return tr->S_t[x.tid] > tr->S_t[y.tid];
      if (tr->a[x.tid] != tr->a[y.tid]) return tr->a[x.tid] < tr->a[y.tid];
      return x.rank < y.rank;
    });
    bool any = false;
    for (const Cand &c : cl) {
      const int32_t tid = c.tid;
      const double tswap = double(tr->S_t[tid]) / tr->bw;
      const int32_t first = next_pos(tr->a[tid]);
      if (first >= tr->b[tid]) continue;
      const int32_t lo = std::max(lay[first], lay[tr->a[tid]] + 1);
      int32_t found = -1;
      for (int32_t l = lay[tr->b[tid]] - 1; l >= lo; l--) if (rem[l] > tswap) { found = l; break; }
      if (found < 0) continue;
      const int32_t sp = tr->lay_start[found];
      rem[found] -= tswap;
      selected[c.rank] = 1;
      placed.push_back({c.rank, tid, sp, 0u});
      credit(tid, sp);
      any = true;
      if (mrl_empty()) break;
    }
    if (!any) {  // schedule the highest-score candidate in the layer before its first BWD use
      const Cand &c = cl.front();
      const int32_t l = lay[tr->b[c.tid]] - 1;
      selected[c.rank] = 1;
      if (l > lay[tr->a[c.tid]]) {
        const int32_t sp = tr->lay_start[l];
        rem[l] -= double(tr->S_t[c.tid]) / tr->bw;
        placed.push_back({c.rank, c.tid, sp, 1u});
        credit(c.tid, sp);
      }
    }
  }
  // SetFreeTime in swap-out order
  std::stable_sort(placed.begin(), placed.end(), [&](const Placed &x, const Placed &y) {
    if (tr->a[x.tid] != tr->a[y.tid]) return tr->a[x.tid] < tr->a[y.tid];
    return x.rank < y.rank;
  });
  uint32_t w = 0;
  for (const Placed &pl : placed) {
    const double tswap = double(tr->S_t[pl.tid]) / tr->bw;
    const int32_t la = lay[tr->a[pl.tid]], lhi = lay[pl.s] - 2;
    int32_t r = -1;
    uint32_t flags = pl.flags;
    for (int32_t l = la; l <= lhi; l++)
      if (rem[l] > tswap) { r = tr->lay_start[l] + tr->lay_n[l] - 1; rem[l] -= tswap; break; }
    if (r < 0) {
      flags |= 2u;
      r = lhi >= la ? tr->lay_start[lhi] + tr->lay_n[lhi] - 1 : pl.s - 2;
    }
    if (r < tr->a[pl.tid] || !(r + 1 < pl.s)) continue;  // no off-device window
    if (w < cap) items[w] = {uint32_t(pl.rank), r, pl.s, flags};
    w++;
  }
  *n_items = w;
  if (feasible) *feasible = ok ? 1 : 0;
  if (w > cap) CHM_FAIL(CHM_E_INVAL, "chm_generate_policy: %u items exceed cap %u", w, cap);
  return CHM_OK;
}
