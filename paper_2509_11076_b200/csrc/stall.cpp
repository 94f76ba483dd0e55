// stall.cpp -- the stall of one explicit policy under the three models of reading Q11 (SURVEY
// §8(f) NEXT-4): R-stall (the model the replay kernels evaluate), per-direction layer budgets,
// and the max-plus serial-stream timeline.  Host-side: for comparing the models against
// measured stalls (tools/stall_fidelity.py), not on the search path.
#include <algorithm>
#include <vector>

#include "internal.h"

using namespace chm;

namespace {
double pairwise(const std::vector<double> &v, size_t lo, size_t n) {
  if (n == 1) return v[lo];
  return pairwise(v, lo, n / 2) + pairwise(v, lo + n / 2, n / 2);
}
}  // namespace

extern "C" chm_status chm_stall_models(const chm_trace *t, const chm_item *items, uint32_t n, double *out) {
  if (!t || !out || (n && !items)) CHM_FAIL(CHM_E_INVAL, "chm_stall_models: NULL argument");
  const int32_t n_prod = int32_t(t->rank_to_tensor.size());
  std::vector<int32_t> tid(n), r(n), s(n), a(n), b(n);
  std::vector<int64_t> S(n);
  for (uint32_t k = 0; k < n; k++) {
    const chm_item &it = items[k];
    if (int64_t(it.t) >= n_prod) CHM_FAIL(CHM_E_INVAL, "chm_stall_models: item %u: bad tensor", k);
    tid[k] = t->rank_to_tensor[it.t];
    a[k] = t->a[tid[k]];
    b[k] = t->b[tid[k]];
    r[k] = it.r;
    s[k] = it.s;
    S[k] = t->S_t[tid[k]];
    if (a[k] < 0 || b[k] < 0 || r[k] < a[k] || !(r[k] + 1 < s[k]) || s[k] > b[k] || s[k] >= t->N)
      CHM_FAIL(CHM_E_INVAL, "chm_stall_models: item %u (t %u, r %d, s %d) invalid", k, it.t, it.r, it.s);
  }
  const int32_t L = t->L;
  size_t P = 1;
  while (P < size_t(L)) P *= 2;
  // R-stall: one budget per layer for both directions; per-direction: one each
  std::vector<int64_t> load_o(size_t(L), 0), load_i(size_t(L), 0);
  for (uint32_t k = 0; k < n; k++) {
    load_o[size_t(t->lay_of_op[r[k]])] += S[k];
    load_i[size_t(t->lay_of_op[s[k]])] += S[k];
  }
  std::vector<double> t0(P, 0.0), t1(P, 0.0);
  for (int32_t l = 0; l < L; l++) {
    const double x = double(load_o[l] + load_i[l]) / t->bw - t->bud[l];
    t0[l] = x > 0.0 ? x : 0.0;
    const double xo = double(load_o[l]) / t->bw - t->bud[l];
    const double xi = double(load_i[l]) / t->bw - t->bud[l];
    t1[l] = (xo > 0.0 ? xo : 0.0) + (xi > 0.0 ? xi : 0.0);
  }
  out[0] = pairwise(t0, 0, P);
  out[1] = pairwise(t1, 0, P);
  // timeline: op-indexed event lists, item order within a kind
  const int32_t N = t->N;
  auto bucket = [&](const std::vector<int32_t> &key, std::vector<int32_t> &ptr, std::vector<int32_t> &idx) {
    ptr.assign(size_t(N) + 1, 0);
    for (uint32_t k = 0; k < n; k++) ptr[size_t(key[k]) + 1]++;
    for (int32_t i = 0; i < N; i++) ptr[size_t(i) + 1] += ptr[size_t(i)];
    idx.assign(n, 0);
    std::vector<int32_t> fill(ptr.begin(), ptr.end() - 1);
    for (uint32_t k = 0; k < n; k++) idx[size_t(fill[size_t(key[k])]++)] = int32_t(k);
  };
  std::vector<int32_t> pa, ia, pr, ir, ps, is, pb, ib;
  bucket(a, pa, ia);
  bucket(r, pr, ir);
  bucket(s, ps, is);
  bucket(b, pb, ib);
  const double tau = N > 0 ? t->t_iter / double(N) : 0.0;
  double now = 0.0, d2h = 0.0, h2d = 0.0, stall = 0.0;
  std::vector<double> out_end(n, 0.0), in_end(n, 0.0);
  for (int32_t i = 0; i < N; i++) {
    for (int32_t q = ps[i]; q < ps[i + 1]; q++) {
      const int32_t k = is[q];
      double start = now;
      if (h2d > start) start = h2d;
      if (out_end[k] > start) start = out_end[k];
      in_end[k] = start + double(S[k]) / t->bw;
      h2d = in_end[k];
    }
    for (int32_t q = pb[i]; q < pb[i + 1]; q++) {
      const int32_t k = ib[q];
      if (in_end[k] > now) { stall += in_end[k] - now; now = in_end[k]; }
    }
    now += tau;
    for (int32_t q = pa[i]; q < pa[i + 1]; q++) {
      const int32_t k = ia[q];
      double start = now;
      if (d2h > start) start = d2h;
      out_end[k] = start + double(S[k]) / t->bw;
      d2h = out_end[k];
    }
    for (int32_t q = pr[i]; q < pr[i + 1]; q++) {
      const int32_t k = ir[q];
      if (out_end[k] > now) { stall += out_end[k] - now; now = out_end[k]; }
    }
  }
  out[2] = stall;
  return CHM_OK;
}
