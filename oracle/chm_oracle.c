/*
 * chm_oracle.c -- CPU ORACLE for the Chameleon swap hot path.  TEST INFRASTRUCTURE ONLY
 * (see chm_oracle.h).  Plain C99, built with -O2 -ffp-contract=off so every floating-point
 * expression is evaluated exactly as written (no FMA contraction).
 *
 * Nothing here is blocked, fused or reordered for speed: each function walks the paper's
 * definition in the paper's order.
 */
#define _GNU_SOURCE
#include "chm_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

enum { FWD = 0, BWD = 1, OPT = 2 };

static __thread char g_err[256];
const char *orc_error(void) { return g_err; }
#define FAIL(...)                                        \
  do {                                                   \
    snprintf(g_err, sizeof g_err, __VA_ARGS__);          \
    return -1;                                           \
  } while (0)

struct orc_model {
  int32_t N, T, K, L;
  int64_t M0;
  double t_iter, bw, omega;
  const orc_input *in; /* borrowed for the lifetime of the model */
  /* tensor table */
  int32_t *p, *f, *a, *b;
  int64_t *S;
  /* logical layers: start op, op count, type, budget (Eq. 1) */
  int32_t *lay_start, *lay_n, *lay_type, *lay_of_op;
  double *bud;
  int32_t last_fwd_layer;
  /* swappable set in mask-bit order */
  int32_t *sw_t, *sw_r, *sw_s, *sw_lin, *sw_lout, *sw_sat;
  int64_t *F0;
  uint64_t *base; /* W words */
  int32_t W;
};

static void *xcalloc(size_t n, size_t sz) {
  void *p = calloc(n ? n : 1, sz);
  if (!p) abort();
  return p;
}

/* ---------------------------------------------------------------------------------------
 * Event-by-event replay, following the eager semantics of P:160 (host-side
 * alloc/free, refcount release) and the custom recordStream release of P:393.
 * For op i, in this order:
 *   1. swap-ins dispatched before op i (s_t == i) allocate their block     (Q7)
 *   2. op i's outputs are allocated
 *   3. record F[i] = live   -- the op's execution-point usage, the MRL quantity
 *   4. refcount releases after op i (f_t == i) free their blocks
 *   5. swap-outs that complete during op i are reclaimed after it (r_t == i) (Q6)
 * ------------------------------------------------------------------------------------- */
typedef struct {
  int32_t *head_s, *head_r, *next_s, *next_r; /* per-op item buckets */
} replay_scratch;

static void scratch_init(replay_scratch *w, int32_t N, int32_t max_items) {
  w->head_s = xcalloc((size_t)N, sizeof(int32_t));
  w->head_r = xcalloc((size_t)N, sizeof(int32_t));
  w->next_s = xcalloc((size_t)max_items + 1, sizeof(int32_t));
  w->next_r = xcalloc((size_t)max_items + 1, sizeof(int32_t));
}
static void scratch_free(replay_scratch *w) {
  free(w->head_s); free(w->head_r); free(w->next_s); free(w->next_r);
}

static int64_t replay_items(const orc_model *m, replay_scratch *w, int32_t n_items,
                            const int32_t *t, const int32_t *r, const int32_t *s,
                            int64_t *footprint, int64_t *d2h, int64_t *h2d) {
  const orc_input *in = m->in;
  int32_t N = m->N;
  for (int32_t i = 0; i < N; i++) { w->head_s[i] = -1; w->head_r[i] = -1; }
  int64_t out_bytes = 0, in_bytes = 0;
  for (int32_t k = 0; k < n_items; k++) {
    w->next_s[k] = w->head_s[s[k]]; w->head_s[s[k]] = k;
    w->next_r[k] = w->head_r[r[k]]; w->head_r[r[k]] = k;
    out_bytes += m->S[t[k]]; /* swap-out issued after op a_t: no memory effect, D2H log */
    in_bytes += m->S[t[k]];  /* swap-in issued before op s_t: H2D log */
  }
  int64_t live = m->M0, peak = INT64_MIN;
  for (int32_t i = 0; i < N; i++) {
    for (int32_t k = w->head_s[i]; k >= 0; k = w->next_s[k]) live += m->S[t[k]];          /* 1 */
    for (int32_t j = in->out_ptr[i]; j < in->out_ptr[i + 1]; j++) live += m->S[in->out_idx[j]]; /* 2 */
    if (footprint) footprint[i] = live;                                                   /* 3 */
    if (live > peak) peak = live;
    for (int32_t j = in->free_ptr[i]; j < in->free_ptr[i + 1]; j++) live -= m->S[in->free_idx[j]]; /* 4 */
    for (int32_t k = w->head_r[i]; k >= 0; k = w->next_r[k]) live -= m->S[t[k]];          /* 5 */
  }
  if (d2h) *d2h = out_bytes;
  if (h2d) *h2d = in_bytes;
  return N > 0 ? peak : m->M0;
}

/* ---------------------------------------------------------------------------------------
 * Estimated stall, SURVEY §8(c).5 / DESIGN.md reading R-stall (the paper gives no formula,
 * reading Q11).
 *   load_l = sum over items of S_t*([lin_t == l] + [lout_t == l])  (swap-in charged to its
 *            placement layer; swap-out to its completion layer)
 *   term_l = max(0, load_l / B - Bud_l)                               ("introduce latency")
 *   stall  = pairwise sum of term_0 .. term_{L-1}: the index range, padded with +0.0 to a power
 *            of two, is halved recursively and the two halves' sums are added.  A fixed order,
 *            so every implementation rounds identically.
 * ------------------------------------------------------------------------------------- */
static double pairwise_sum(const double *v, int32_t lo, int32_t n) {
  if (n == 1) return v[lo];
  return pairwise_sum(v, lo, n / 2) + pairwise_sum(v, lo + n / 2, n / 2);
}

static double stall_items(const orc_model *m, int64_t *load, int32_t n_items, const int32_t *t,
                          const int32_t *r, const int32_t *s) {
  for (int32_t l = 0; l < m->L; l++) load[l] = 0;
  for (int32_t k = 0; k < n_items; k++) {
    load[m->lay_of_op[s[k]]] += m->S[t[k]];
    load[m->lay_of_op[r[k]]] += m->S[t[k]];
  }
  int32_t P = 1;
  while (P < m->L) P *= 2;
  double *term = xcalloc((size_t)P, sizeof(double)); /* zero padded */
  for (int32_t l = 0; l < m->L; l++) {
    double x = (double)load[l] / m->bw - m->bud[l];
    term[l] = x > 0.0 ? x : 0.0;
  }
  double stall = pairwise_sum(term, 0, P);
  free(term);
  return stall;
}

/* --------------------------------------------------------------------------------------- */
int orc_build(const orc_input *in, orc_model **out) {
  int32_t N = in->n_ops, T = in->n_tensors;
  if (N < 0 || T < 0) FAIL("negative sizes");
  if (!(in->bw > 0.0)) FAIL("bandwidth B must be > 0 (Eq. 3)");
  if (!(in->t_iter >= 0.0)) FAIL("T_iter must be >= 0");
  orc_model *m = xcalloc(1, sizeof *m);
  m->N = N; m->T = T; m->M0 = in->static_bytes; m->t_iter = in->t_iter; m->bw = in->bw;
  m->omega = in->omega; m->in = in;
  m->p = xcalloc((size_t)T, sizeof(int32_t)); m->f = xcalloc((size_t)T, sizeof(int32_t));
  m->a = xcalloc((size_t)T, sizeof(int32_t)); m->b = xcalloc((size_t)T, sizeof(int32_t));
  m->S = xcalloc((size_t)T, sizeof(int64_t));
  for (int32_t t = 0; t < T; t++) {
    m->p[t] = -1; m->f[t] = N; m->a[t] = -1; m->b[t] = -1; m->S[t] = in->nbytes[t];
    if (in->nbytes[t] <= 0) { orc_free(m); FAIL("tensor %d has size <= 0", t); }
  }
  /* phases must be FWD* BWD* OPT* (P:160 dispatch order) */
  for (int32_t i = 1; i < N; i++)
    if (in->phase[i] < in->phase[i - 1]) { orc_free(m); FAIL("phases interleave at op %d", i); }
  /* tensor table: producer, refcount release, last FWD use (production counts), first BWD
   * input use ("long lifetimes and extended idle periods") */
  for (int32_t i = 0; i < N; i++) {
    for (int32_t j = in->out_ptr[i]; j < in->out_ptr[i + 1]; j++) {
      int32_t t = in->out_idx[j];
      m->p[t] = i;
      if (in->phase[i] == FWD) m->a[t] = i;
    }
    for (int32_t j = in->in_ptr[i]; j < in->in_ptr[i + 1]; j++) {
      int32_t t = in->in_idx[j];
      if (in->phase[i] == FWD && i > m->a[t]) m->a[t] = i;
      if (in->phase[i] == BWD && m->b[t] < 0) m->b[t] = i;
    }
    for (int32_t j = in->free_ptr[i]; j < in->free_ptr[i + 1]; j++) m->f[in->free_idx[j]] = i;
  }
  /* logical layers, P:283-288 + P:316-325: FWD ops in groups_fwd near-even contiguous groups,
   * BWD likewise, OPT one group; the first (n mod G) groups take one extra op */
  int32_t nph[3] = {0, 0, 0};
  for (int32_t i = 0; i < N; i++) nph[in->phase[i]]++;
  int32_t G[3] = {in->groups_fwd, in->groups_bwd, nph[OPT] > 0 ? 1 : 0};
  for (int ph = 0; ph < 2; ph++) {
    if (nph[ph] == 0) G[ph] = 0;
    else if (G[ph] < 1 || G[ph] > nph[ph]) { orc_free(m); FAIL("group count %d invalid for %d ops", G[ph], nph[ph]); }
  }
  m->L = G[0] + G[1] + G[2];
  m->lay_start = xcalloc((size_t)m->L, sizeof(int32_t)); m->lay_n = xcalloc((size_t)m->L, sizeof(int32_t));
  m->lay_type = xcalloc((size_t)m->L, sizeof(int32_t)); m->bud = xcalloc((size_t)m->L, sizeof(double));
  m->lay_of_op = xcalloc((size_t)N, sizeof(int32_t));
  int32_t l = 0, op = 0;
  m->last_fwd_layer = -1;
  for (int ph = 0; ph < 3; ph++) {
    for (int32_t g = 0; g < G[ph]; g++) {
      int32_t n = nph[ph] / G[ph] + (g < nph[ph] % G[ph] ? 1 : 0);
      m->lay_start[l] = op; m->lay_n[l] = n; m->lay_type[l] = ph;
      /* Eq. 1: T_group = T_iter / N_iter * N_group; times the overlap factor */
      m->bud[l] = ((m->t_iter / (double)N) * (double)n) * m->omega;
      for (int32_t i = op; i < op + n; i++) m->lay_of_op[i] = l;
      if (ph == FWD) m->last_fwd_layer = l;
      op += n; l++;
    }
  }
  /* no-swap footprint F0 = replay with an empty swap set */
  m->F0 = xcalloc((size_t)N, sizeof(int64_t));
  {
    replay_scratch w; scratch_init(&w, N > 0 ? N : 1, 1);
    replay_items(m, &w, 0, NULL, NULL, NULL, m->F0, NULL, NULL);
    scratch_free(&w);
  }
  /* solo timing per candidate tensor:
   *   T_swap = S / B                                                          (Eq. 3)
   *   r_t: from lay(a_t) forward over FWD layers, first layer with Bud > T_swap;
   *        release after its last op; none -> end of last FWD layer, saturated
   *   s_t: start of the layer before the one holding the first BWD use       (Q8)
   * swappable iff the off-device window (r_t, s_t) holds at least one op. */
  int32_t *cand = xcalloc((size_t)T + 1, sizeof(int32_t));
  int32_t *cr = xcalloc((size_t)T + 1, sizeof(int32_t)), *cs = xcalloc((size_t)T + 1, sizeof(int32_t));
  int32_t *csat = xcalloc((size_t)T + 1, sizeof(int32_t));
  int32_t K = 0;
  for (int32_t t = 0; t < T; t++) {
    if (m->p[t] < 0 || m->a[t] < 0 || m->b[t] < 0) continue; /* activations only */
    double tswap = (double)m->S[t] / m->bw;
    int32_t r = -1, sat = 0;
    for (int32_t ll = m->lay_of_op[m->a[t]]; ll <= m->last_fwd_layer; ll++) {
      if (m->bud[ll] > tswap) { r = m->lay_start[ll] + m->lay_n[ll] - 1; break; }
    }
    if (r < 0) {
      r = m->lay_start[m->last_fwd_layer] + m->lay_n[m->last_fwd_layer] - 1;
      sat = 1;
    }
    int32_t lb = m->lay_of_op[m->b[t]];
    if (lb - 1 < 0) continue;
    int32_t s = m->lay_start[lb - 1];
    if (!(r + 1 < s)) continue;
    cand[K] = t; cr[K] = r; cs[K] = s; csat[K] = sat; K++;
  }
  /* mask-bit order: ascending a_t, ties by production order (tensor index) -- insertion sort */
  for (int32_t i = 1; i < K; i++) {
    int32_t ct = cand[i], rr = cr[i], ss = cs[i], sa = csat[i], j = i - 1;
    while (j >= 0 && (m->a[cand[j]] > m->a[ct] || (m->a[cand[j]] == m->a[ct] && cand[j] > ct))) {
      cand[j + 1] = cand[j]; cr[j + 1] = cr[j]; cs[j + 1] = cs[j]; csat[j + 1] = csat[j]; j--;
    }
    cand[j + 1] = ct; cr[j + 1] = rr; cs[j + 1] = ss; csat[j + 1] = sa;
  }
  m->K = K;
  m->sw_t = cand; m->sw_r = cr; m->sw_s = cs; m->sw_sat = csat;
  m->sw_lin = xcalloc((size_t)K + 1, sizeof(int32_t)); m->sw_lout = xcalloc((size_t)K + 1, sizeof(int32_t));
  for (int32_t k = 0; k < K; k++) { m->sw_lin[k] = m->lay_of_op[cs[k]]; m->sw_lout[k] = m->lay_of_op[cr[k]]; }
  /* default SEEDED base: swappable tensors whose window contains the first argmax of F0 */
  m->W = (K + 63) / 64;
  m->base = xcalloc((size_t)m->W + 1, sizeof(uint64_t));
  int32_t imax = 0;
  for (int32_t i = 1; i < N; i++) if (m->F0[i] > m->F0[imax]) imax = i;
  for (int32_t k = 0; k < K; k++)
    if (N > 0 && cr[k] < imax && imax < cs[k]) m->base[k / 64] |= 1ull << (k % 64);
  *out = m;
  return 0;
}

void orc_free(orc_model *m) {
  if (!m) return;
  free(m->p); free(m->f); free(m->a); free(m->b); free(m->S);
  free(m->lay_start); free(m->lay_n); free(m->lay_type); free(m->lay_of_op); free(m->bud);
  free(m->sw_t); free(m->sw_r); free(m->sw_s); free(m->sw_lin); free(m->sw_lout); free(m->sw_sat);
  free(m->F0); free(m->base); free(m);
}

void orc_dims(const orc_model *m, int32_t *n_ops, int32_t *n_tensors, int32_t *n_swappable,
              int32_t *n_layers) {
  *n_ops = m->N; *n_tensors = m->T; *n_swappable = m->K; *n_layers = m->L;
}
void orc_tensor_table(const orc_model *m, int32_t *p, int32_t *f, int32_t *a, int32_t *b) {
  for (int32_t t = 0; t < m->T; t++) { p[t] = m->p[t]; f[t] = m->f[t]; a[t] = m->a[t]; b[t] = m->b[t]; }
}
void orc_layer_table(const orc_model *m, int32_t *start, int32_t *count, int32_t *type, double *bud) {
  for (int32_t l = 0; l < m->L; l++) { start[l] = m->lay_start[l]; count[l] = m->lay_n[l]; type[l] = m->lay_type[l]; bud[l] = m->bud[l]; }
}
void orc_swappable(const orc_model *m, int32_t *t, int32_t *r, int32_t *s, int32_t *lin,
                   int32_t *lout, int32_t *saturated) {
  for (int32_t k = 0; k < m->K; k++) {
    t[k] = m->sw_t[k]; r[k] = m->sw_r[k]; s[k] = m->sw_s[k]; lin[k] = m->sw_lin[k];
    lout[k] = m->sw_lout[k]; saturated[k] = m->sw_sat[k];
  }
}
void orc_f0(const orc_model *m, int64_t *f0) { for (int32_t i = 0; i < m->N; i++) f0[i] = m->F0[i]; }
void orc_base_mask(const orc_model *m, uint64_t *w) { for (int32_t i = 0; i < m->W; i++) w[i] = m->base[i]; }

int64_t orc_replay(const orc_model *m, int32_t n_items, const int32_t *t, const int32_t *r,
                   const int32_t *s, int64_t *footprint, int64_t *d2h, int64_t *h2d) {
  replay_scratch w; scratch_init(&w, m->N > 0 ? m->N : 1, n_items);
  int64_t pk = replay_items(m, &w, n_items, t, r, s, footprint, d2h, h2d);
  scratch_free(&w);
  return pk;
}

double orc_stall(const orc_model *m, int32_t n_items, const int32_t *t, const int32_t *r,
                 const int32_t *s) {
  int64_t *load = xcalloc((size_t)m->L + 1, sizeof(int64_t));
  double st = stall_items(m, load, n_items, t, r, s);
  free(load);
  return st;
}

/* Q11 variant: per-direction budgets (the host link is full duplex) */
double orc_stall_dir(const orc_model *m, int32_t n_items, const int32_t *t, const int32_t *r,
                     const int32_t *s) {
  int64_t *out = xcalloc((size_t)m->L + 1, sizeof(int64_t));
  int64_t *in = xcalloc((size_t)m->L + 1, sizeof(int64_t));
  for (int32_t k = 0; k < n_items; k++) {
    out[m->lay_of_op[r[k]]] += m->S[t[k]];
    in[m->lay_of_op[s[k]]] += m->S[t[k]];
  }
  int32_t P = 1;
  while (P < m->L) P *= 2;
  double *term = xcalloc((size_t)P, sizeof(double));
  for (int32_t l = 0; l < m->L; l++) {
    double xo = (double)out[l] / m->bw - m->bud[l];
    double xi = (double)in[l] / m->bw - m->bud[l];
    term[l] = (xo > 0.0 ? xo : 0.0) + (xi > 0.0 ? xi : 0.0);
  }
  double stall = pairwise_sum(term, 0, P);
  free(term); free(in); free(out);
  return stall;
}

/* Q11 variant: max-plus serial-stream timeline, walked op by op */
double orc_stall_timeline(const orc_model *m, int32_t n_items, const int32_t *t, const int32_t *r,
                          const int32_t *s) {
  const double tau = m->N > 0 ? m->t_iter / (double)m->N : 0.0;
  double now = 0.0, d2h_free = 0.0, h2d_free = 0.0, stall = 0.0;
  double *out_end = xcalloc((size_t)n_items + 1, sizeof(double));
  double *in_end = xcalloc((size_t)n_items + 1, sizeof(double));
  for (int32_t i = 0; i < m->N; i++) {
    /* before op i: swap-ins issued for s = i, then waits for b = i */
    for (int32_t k = 0; k < n_items; k++) {
      if (s[k] != i) continue;
      double start = now;
      if (h2d_free > start) start = h2d_free;
      if (out_end[k] > start) start = out_end[k];
      in_end[k] = start + (double)m->S[t[k]] / m->bw;
      h2d_free = in_end[k];
    }
    for (int32_t k = 0; k < n_items; k++) {
      if (m->b[t[k]] != i) continue;
      if (in_end[k] > now) { stall += in_end[k] - now; now = in_end[k]; }
    }
    now += tau; /* op i */
    /* after op i: swap-outs of a = i, then releases of r = i */
    for (int32_t k = 0; k < n_items; k++) {
      if (m->a[t[k]] != i) continue;
      double start = now;
      if (d2h_free > start) start = d2h_free;
      out_end[k] = start + (double)m->S[t[k]] / m->bw;
      d2h_free = out_end[k];
    }
    for (int32_t k = 0; k < n_items; k++) {
      if (r[k] != i) continue;
      if (out_end[k] > now) { stall += out_end[k] - now; now = out_end[k]; }
    }
  }
  free(out_end); free(in_end);
  return stall;
}

/* Fig. 3: actual usage = measured usage + bytes swapped out and not yet back */
void orc_reconstruct(int32_t n_ops, const int64_t *measured, int32_t n_items, const int64_t *size,
                     const int32_t *r, const int32_t *s, int64_t *actual) {
  for (int32_t i = 0; i < n_ops; i++) {
    int64_t off = 0;
    for (int32_t k = 0; k < n_items; k++)
      if (r[k] < i && i < s[k]) off += size[k];
    actual[i] = measured[i] + off;
  }
}

/* ---------------------------------------------------------------------------------------
 * Candidates and the argmin key (§8(c).6, "selects the one with the
 * best runtime performance"): key = (excess, stall, swapped bytes, global index), lexicographic.
 * ------------------------------------------------------------------------------------- */
uint64_t orc_splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int orc_key_less(const orc_best *x, const orc_best *y) {
  if (x->excess != y->excess) return x->excess < y->excess;
  if (x->stall != y->stall) return x->stall < y->stall;
  if (x->swapped != y->swapped) return x->swapped < y->swapped;
  return x->index < y->index;
}

typedef struct {
  const orc_model *m;
  int kind;
  uint64_t first, lo, hi, seed, flip_thr;
  const uint64_t *words;
  int64_t budget;
  int64_t *peak, *swapped, *footprint;
  double *stall;
  int stall_model;  /* 0: stall_items (R-stall, §8(c).5); 1: orc_stall_timeline (Q11 variant) */
  orc_best best;
  int have_best;
} eval_job;

static int cand_bit(const eval_job *j, uint64_t c, uint64_t idx, int32_t k) {
  const orc_model *m = j->m;
  if (j->kind == ORC_EXHAUSTIVE) return (int)((c >> k) & 1ull);
  if (j->kind == ORC_SEEDED) {
    /* DESIGN.md reading R-seeded: candidate c draws J = ceil(K/4) words
     * w_q = mix(seed ^ mix(c*J + q)); item k flips iff its 16-bit field
     * (w_{k/4} >> 16*(k mod 4)) & 0xffff is below flip_thr >> 48 */
    const uint64_t *base = j->words ? j->words : m->base;
    int b = (int)((base[k / 64] >> (k % 64)) & 1ull);
    uint64_t J = ((uint64_t)m->K + 3) / 4;
    uint64_t w = orc_splitmix64(j->seed ^ (c * J + (uint64_t)(k / 4)));  /* reading R-seeded (r02: one mix) */
    uint64_t field = (w >> (16 * (k % 4))) & 0xffffull;
    return b ^ (field < (j->flip_thr >> 48) ? 1 : 0);
  }
  return (int)((j->words[idx * (uint64_t)m->W + (uint64_t)(k / 64)] >> (k % 64)) & 1ull);
}

static void *eval_range(void *arg) {
  eval_job *j = arg;
  const orc_model *m = j->m;
  replay_scratch w; scratch_init(&w, m->N > 0 ? m->N : 1, m->K);
  int32_t *t = xcalloc((size_t)m->K + 1, sizeof(int32_t)), *r = xcalloc((size_t)m->K + 1, sizeof(int32_t));
  int32_t *s = xcalloc((size_t)m->K + 1, sizeof(int32_t));
  int64_t *load = xcalloc((size_t)m->L + 1, sizeof(int64_t));
  for (uint64_t idx = j->lo; idx < j->hi; idx++) {
    uint64_t c = j->first + idx;
    int32_t n = 0;
    for (int32_t k = 0; k < m->K; k++)
      if (cand_bit(j, c, idx, k)) { t[n] = m->sw_t[k]; r[n] = m->sw_r[k]; s[n] = m->sw_s[k]; n++; }
    int64_t out_b;
    int64_t pk = replay_items(m, &w, n, t, r, s, j->footprint ? j->footprint + idx * (uint64_t)m->N : NULL, &out_b, NULL);
    double st = j->stall_model ? orc_stall_timeline(m, n, t, r, s) : stall_items(m, load, n, t, r, s);
    if (j->peak) j->peak[idx] = pk;
    if (j->stall) j->stall[idx] = st;
    if (j->swapped) j->swapped[idx] = out_b;
    orc_best key = { pk > j->budget ? pk - j->budget : 0, st, out_b, c, pk };
    if (!j->have_best || orc_key_less(&key, &j->best)) { j->best = key; j->have_best = 1; }
  }
  free(t); free(r); free(s); free(load); scratch_free(&w);
  return NULL;
}

int orc_eval(const orc_model *m, int kind, uint64_t first, uint64_t count, uint64_t seed,
             uint64_t flip_thr, const uint64_t *words, int64_t budget, int nthreads,
             int64_t *peak, double *stall, int64_t *swapped, int64_t *footprint, orc_best *best) {
  return orc_eval_model(m, kind, first, count, seed, flip_thr, words, budget, nthreads, 0, peak, stall,
                        swapped, footprint, best);
}

/* orc_eval with the candidate's stall under stall_model 1 = the timeline (orc_stall_timeline of
 * its items in mask-bit order): the stall and the key's second field change, nothing else */
int orc_eval_model(const orc_model *m, int kind, uint64_t first, uint64_t count, uint64_t seed,
                   uint64_t flip_thr, const uint64_t *words, int64_t budget, int nthreads, int stall_model,
                   int64_t *peak, double *stall, int64_t *swapped, int64_t *footprint, orc_best *best) {
  if (kind == ORC_EXHAUSTIVE && m->K > 63) FAIL("EXHAUSTIVE needs K <= 63 (K = %d)", m->K);
  if (kind == ORC_MASKS && !words) FAIL("MASKS needs masks");
  if (nthreads < 1) nthreads = 1;
  if ((uint64_t)nthreads > count) nthreads = count ? (int)count : 1;
  eval_job *jobs = xcalloc((size_t)nthreads, sizeof(eval_job));
  pthread_t *th = xcalloc((size_t)nthreads, sizeof(pthread_t));
  for (int i = 0; i < nthreads; i++) {
    eval_job *j = &jobs[i];
    j->m = m; j->kind = kind; j->first = first; j->seed = seed; j->flip_thr = flip_thr;
    j->words = words; j->budget = budget; j->peak = peak; j->stall = stall; j->swapped = swapped;
    j->footprint = footprint;
    j->stall_model = stall_model;
    j->lo = count * (uint64_t)i / (uint64_t)nthreads;
    j->hi = count * (uint64_t)(i + 1) / (uint64_t)nthreads;
    if (nthreads == 1) eval_range(j);
    else pthread_create(&th[i], NULL, eval_range, j);
  }
  int have = 0;
  orc_best b = {0, 0.0, 0, 0, 0};
  for (int i = 0; i < nthreads; i++) {
    if (nthreads > 1) pthread_join(th[i], NULL);
    if (jobs[i].have_best && (!have || orc_key_less(&jobs[i].best, &b))) { b = jobs[i].best; have = 1; }
  }
  if (best) *best = b;
  free(jobs); free(th);
  return 0;
}

void orc_swap_execute(int32_t n, void *const *dst, const void *const *src, const uint64_t *nbytes) {
  for (int32_t j = 0; j < n; j++) memcpy(dst[j], src[j], (size_t)nbytes[j]);
}

/* ---------------------------------------------------------------------------------------
 * Algo. 1, stage adjusting, with the readings of SURVEY §8(c).8 / Q1-Q3:
 *   len_diff = |n - n'| / max(n, n');  cos = positional cosine of the zero-padded token
 *   vectors (cos_mode 0) or of token-count histograms (cos_mode 1);
 *   stable iff len_diff < len_tol and cos > cos_tol (strict).
 * ------------------------------------------------------------------------------------- */
int orc_compare(const int32_t *a, int32_t na, const int32_t *b, int32_t nb, int32_t cos_mode,
                double *len_diff, double *cos_sim) {
  if (na <= 0 || nb <= 0) FAIL("empty operator sequence");
  int32_t mx = na > nb ? na : nb;
  int64_t diff = (int64_t)na - (int64_t)nb;
  if (diff < 0) diff = -diff;
  *len_diff = (double)diff / (double)mx;
  int64_t dot = 0, aa = 0, bb = 0;
  if (cos_mode == 0) {
    for (int32_t i = 0; i < mx; i++) {
      int64_t x = i < na ? a[i] : 0, y = i < nb ? b[i] : 0;
      dot += x * y; aa += x * x; bb += y * y;
    }
  } else {
    int32_t V = 0;
    for (int32_t i = 0; i < na; i++) if (a[i] > V) V = a[i];
    for (int32_t i = 0; i < nb; i++) if (b[i] > V) V = b[i];
    int64_t *ha = xcalloc((size_t)V + 1, sizeof(int64_t)), *hb = xcalloc((size_t)V + 1, sizeof(int64_t));
    for (int32_t i = 0; i < na; i++) ha[a[i]]++;
    for (int32_t i = 0; i < nb; i++) hb[b[i]]++;
    for (int32_t v = 0; v <= V; v++) { dot += ha[v] * hb[v]; aa += ha[v] * ha[v]; bb += hb[v] * hb[v]; }
    free(ha); free(hb);
  }
  *cos_sim = (double)dot / sqrt((double)aa * (double)bb);
  return 0;
}

void orc_stage_init(orc_stage_state *st, int32_t m, int32_t n, double len_tol, double cos_tol,
                    int32_t cos_mode) {
  memset(st, 0, sizeof *st);
  st->m = m; st->n = n; st->len_tol = len_tol; st->cos_tol = cos_tol; st->cos_mode = cos_mode;
  st->prev_stage = 0;
}
void orc_stage_release(orc_stage_state *st) { free(st->prev_seq); st->prev_seq = NULL; }

int32_t orc_stage_step(orc_stage_state *st, const int32_t *seq, int32_t len, double *len_diff,
                       double *cos_sim, int32_t *stable_out) {
  enum { WARMUP = 0, GENPOLICY = 1, STABLE = 2 };
  if (!st->initialized) { /* "static PrevOpSeq <- OpSeq ... initialized only once" */
    st->stable_step = 0; st->prev_stage = WARMUP;
    st->prev_seq = xcalloc((size_t)len + 1, sizeof(int32_t));
    memcpy(st->prev_seq, seq, sizeof(int32_t) * (size_t)len);
    st->prev_len = len; st->cap = len; st->initialized = 1;
  }
  double ld = 1.0, cs = 0.0;
  int stable = 0;
  if (orc_compare(seq, len, st->prev_seq, st->prev_len, st->cos_mode, &ld, &cs) == 0)
    stable = ld < st->len_tol && cs > st->cos_tol;
  int32_t stage;
  if (stable) {
    st->stable_step += 1;
    if (st->prev_stage == WARMUP && st->stable_step > st->m) { stage = GENPOLICY; st->stable_step = 0; }
    else if (st->prev_stage == GENPOLICY && st->stable_step > st->n) stage = STABLE;
    else stage = st->prev_stage; /* reading Q3: Stage unassigned -> keep PrevStage */
  } else {
    stage = WARMUP; st->stable_step = 0;
  }
  st->prev_stage = stage;
  if (len > st->cap) { free(st->prev_seq); st->prev_seq = xcalloc((size_t)len + 1, sizeof(int32_t)); st->cap = len; }
  memcpy(st->prev_seq, seq, sizeof(int32_t) * (size_t)len);
  st->prev_len = len;
  if (len_diff) *len_diff = ld;
  if (cos_sim) *cos_sim = cs;
  if (stable_out) *stable_out = stable;
  return stage;
}

/* ---------------------------------------------------------------------------------------
 * App. A: the 32 most frequent operators get a one-hot bit; every operator an
 * 8-bit index by frequency; per tensor on every op that uses it:
 *   opCount++; opTag |= opOneHot; opCallStack = (opCallStack << 8) + opIndex.
 * Frequency ties are broken by first appearance (reading Q19); index clamps at 255.
 * ------------------------------------------------------------------------------------- */
void orc_feature_tables(const int32_t *tokens, int32_t n, int32_t max_token, uint8_t *op_index,
                        uint32_t *op_onehot) {
  int64_t *cnt = xcalloc((size_t)max_token + 1, sizeof(int64_t));
  int32_t *first = xcalloc((size_t)max_token + 1, sizeof(int32_t));
  for (int32_t v = 0; v <= max_token; v++) first[v] = -1;
  for (int32_t i = 0; i < n; i++) { cnt[tokens[i]]++; if (first[tokens[i]] < 0) first[tokens[i]] = i; }
  for (int32_t v = 0; v <= max_token; v++) { op_index[v] = 0; op_onehot[v] = 0; }
  for (int32_t v = 0; v <= max_token; v++) {
    if (cnt[v] == 0) continue;
    int32_t rank = 0; /* number of tokens strictly before v in (count desc, first asc) order */
    for (int32_t u = 0; u <= max_token; u++) {
      if (cnt[u] == 0 || u == v) continue;
      if (cnt[u] > cnt[v] || (cnt[u] == cnt[v] && first[u] < first[v])) rank++;
    }
    op_index[v] = (uint8_t)(rank + 1 < 255 ? rank + 1 : 255);
    op_onehot[v] = rank < 32 ? (1u << rank) : 0u;
  }
  free(cnt); free(first);
}

void orc_features_after(const int32_t *tokens, int32_t n_ops, const int32_t *use_ptr,
                        const int32_t *use_idx, int32_t n_tensors, const uint8_t *op_index,
                        const uint32_t *op_onehot, int32_t after, uint32_t *count, uint32_t *tag,
                        uint64_t *stack) {
  for (int32_t t = 0; t < n_tensors; t++) { count[t] = 0; tag[t] = 0; stack[t] = 0; }
  for (int32_t i = 0; i < n_ops && i <= after; i++) {
    for (int32_t j = use_ptr[i]; j < use_ptr[i + 1]; j++) {
      int32_t t = use_idx[j];
      count[t] += 1;
      tag[t] |= op_onehot[tokens[i]];
      stack[t] = (stack[t] << 8) + (uint64_t)op_index[tokens[i]];
    }
  }
}

/* ---------------------------------------------------------------------------------------
 * Algo. 2, policy generation, step by step:
 *   MRL <- per-op required reduction F0[i] - budget where positive
 *   while MRL not empty:
 *     CL <- unselected activations whose span [a_t, b_t) holds an MRE
 *           Score = N_MRE/max N_MRE + C * S/max S, descending                  (Eq. 2)
 *           (ties: larger S, smaller a_t, smaller t)
 *     if CL empty: Raise Error
 *     simulate swap-in: per candidate, T_swap = S/B (Eq. 3); from the layer before the one
 *       holding b_t, search backward, not past the layer of the first MRE op in the span nor
 *       into the swap-out layer, for a layer with T_remaining > T_swap; place the swap-in at
 *       its first op, T_remaining -= T_swap, decrement S from the MREs of the ops the tensor is
 *       off device for (a_t, s_t)
 *       if no candidate fits: the highest-score one goes to the layer before its first BWD use
 *   SetFreeTime: in swap-out order, from the layer of a_t search forward (up to two layers
 *     before the swap-in layer) for T_remaining > T_swap; release after its last op, charge
 *     T_swap; none fits: the last such layer (saturated)
 * ------------------------------------------------------------------------------------- */
typedef struct { int32_t t; double score; } gen_cand;

static int gen_cand_before(const orc_model *m, const gen_cand *x, const gen_cand *y) {
  if (x->score != y->score) return x->score > y->score;
  if (m->S[x->t] != m->S[y->t]) return m->S[x->t] > m->S[y->t];
  if (m->a[x->t] != m->a[y->t]) return m->a[x->t] < m->a[y->t];
  return x->t < y->t;
}

int32_t orc_generate(const orc_model *m, int64_t budget, double C, double rem_scale, int32_t cap,
                     int32_t *t_out, int32_t *r_out, int32_t *s_out, int32_t *fb_out, int32_t *sat_out) {
  int32_t N = m->N, T = m->T, L = m->L;
  int64_t *mre = xcalloc((size_t)N + 1, sizeof(int64_t));
  double *rem = xcalloc((size_t)L + 1, sizeof(double));
  int32_t *sel = xcalloc((size_t)T + 1, sizeof(int32_t));
  gen_cand *cl = xcalloc((size_t)T + 1, sizeof(gen_cand));
  int32_t *it_t = xcalloc((size_t)T + 1, sizeof(int32_t)), *it_s = xcalloc((size_t)T + 1, sizeof(int32_t));
  int32_t *it_fb = xcalloc((size_t)T + 1, sizeof(int32_t));
  int32_t n = 0, status = 0;
  for (int32_t i = 0; i < N; i++) mre[i] = m->F0[i] > budget ? m->F0[i] - budget : 0;
  for (int32_t l = 0; l < L; l++) rem[l] = m->bud[l] * rem_scale;
  for (;;) {
    int32_t mrl_empty = 1;
    for (int32_t i = 0; i < N; i++) if (mre[i] > 0) { mrl_empty = 0; break; }
    if (mrl_empty) break;
    /* candidate list with Eq. 2 scores */
    int32_t ncl = 0, max_n = 0;
    int64_t max_s = 0;
    for (int32_t t = 0; t < T; t++) {
      if (sel[t] || m->p[t] < 0 || m->a[t] < 0 || m->b[t] < 0) continue;
      int32_t cnt = 0;
      for (int32_t i = m->a[t]; i < m->b[t]; i++) if (mre[i] > 0) cnt++;
      if (cnt == 0) continue;
      cl[ncl].t = t; cl[ncl].score = (double)cnt; ncl++;
      if (cnt > max_n) max_n = cnt;
      if (m->S[t] > max_s) max_s = m->S[t];
    }
    if (ncl == 0) { status = -1; break; }
    for (int32_t k = 0; k < ncl; k++)
      cl[k].score = cl[k].score / (double)max_n + C * ((double)m->S[cl[k].t] / (double)max_s);
    for (int32_t k = 1; k < ncl; k++) { /* insertion sort, descending score */
      gen_cand x = cl[k];
      int32_t j = k - 1;
      while (j >= 0 && gen_cand_before(m, &x, &cl[j])) { cl[j + 1] = cl[j]; j--; }
      cl[j + 1] = x;
    }
    /* simulate swap-in */
    int32_t placed = 0;
    for (int32_t k = 0; k < ncl; k++) {
      int32_t t = cl[k].t;
      double tswap = (double)m->S[t] / m->bw;
      int32_t first_mre = -1;
      for (int32_t i = m->a[t]; i < m->b[t]; i++) if (mre[i] > 0) { first_mre = i; break; }
      if (first_mre < 0) continue; /* its MREs were cleared by an earlier candidate */
      int32_t lo = m->lay_of_op[first_mre];
      if (lo < m->lay_of_op[m->a[t]] + 1) lo = m->lay_of_op[m->a[t]] + 1;
      int32_t found = -1;
      for (int32_t l = m->lay_of_op[m->b[t]] - 1; l >= lo; l--)
        if (rem[l] > tswap) { found = l; break; }
      if (found < 0) continue;
      int32_t sp = m->lay_start[found];
      rem[found] -= tswap;
      sel[t] = 1;
      it_t[n] = t; it_s[n] = sp; it_fb[n] = 0; n++;
      for (int32_t i = m->a[t] + 1; i < sp; i++) { mre[i] -= m->S[t]; if (mre[i] < 0) mre[i] = 0; }
      placed = 1;
      int32_t empty = 1;
      for (int32_t i = 0; i < N; i++) if (mre[i] > 0) { empty = 0; break; }
      if (empty) break;
    }
    if (!placed) { /* prioritise the highest-score candidate anyway */
      int32_t t = cl[0].t;
      double tswap = (double)m->S[t] / m->bw;
      int32_t l = m->lay_of_op[m->b[t]] - 1;
      sel[t] = 1;
      if (l > m->lay_of_op[m->a[t]]) {
        int32_t sp = m->lay_start[l];
        rem[l] -= tswap;
        it_t[n] = t; it_s[n] = sp; it_fb[n] = 1; n++;
        for (int32_t i = m->a[t] + 1; i < sp; i++) { mre[i] -= m->S[t]; if (mre[i] < 0) mre[i] = 0; }
      }
    }
  }
  /* SetFreeTime, in swap-out order (a_t, t) */
  int32_t *ord = xcalloc((size_t)n + 1, sizeof(int32_t));
  for (int32_t k = 0; k < n; k++) ord[k] = k;
  for (int32_t k = 1; k < n; k++) {
    int32_t x = ord[k], j = k - 1;
    while (j >= 0 && (m->a[it_t[ord[j]]] > m->a[it_t[x]] ||
                      (m->a[it_t[ord[j]]] == m->a[it_t[x]] && it_t[ord[j]] > it_t[x]))) {
      ord[j + 1] = ord[j]; j--;
    }
    ord[j + 1] = x;
  }
  int32_t w = 0;
  for (int32_t q = 0; q < n; q++) {
    int32_t k = ord[q], t = it_t[k], sp = it_s[k];
    double tswap = (double)m->S[t] / m->bw;
    int32_t lhi = m->lay_of_op[sp] - 2, r = -1, sat = 0;
    for (int32_t l = m->lay_of_op[m->a[t]]; l <= lhi; l++)
      if (rem[l] > tswap) { r = m->lay_start[l] + m->lay_n[l] - 1; rem[l] -= tswap; break; }
    if (r < 0) {
      sat = 1;
      r = lhi >= m->lay_of_op[m->a[t]] ? m->lay_start[lhi] + m->lay_n[lhi] - 1 : sp - 2;
    }
    if (r < m->a[t] || !(r + 1 < sp)) continue; /* no off-device window */
    if (w < cap) { t_out[w] = t; r_out[w] = r; s_out[w] = sp; fb_out[w] = it_fb[k]; sat_out[w] = sat; }
    w++;
  }
  free(ord); free(mre); free(rem); free(sel); free(cl); free(it_t); free(it_s); free(it_fb);
  return status < 0 ? -1 - w : w;
}

int orc_eval_explicit(const orc_model *m, int32_t count, const int64_t *off, const int32_t *t,
                      const int32_t *r, const int32_t *s, int64_t budget, uint64_t first_index,
                      int64_t *peak, double *stall, int64_t *swapped, int64_t *footprint,
                      orc_best *best) {
  int have = 0;
  orc_best b = {0, 0.0, 0, 0, 0};
  for (int32_t c = 0; c < count; c++) {
    int32_t n = (int32_t)(off[c + 1] - off[c]);
    const int32_t *tt = t + off[c], *rr = r + off[c], *ss = s + off[c];
    int64_t out_b;
    int64_t pk = orc_replay(m, n, tt, rr, ss, footprint ? footprint + (size_t)c * (size_t)m->N : NULL, &out_b, NULL);
    double st = orc_stall(m, n, tt, rr, ss);
    if (peak) peak[c] = pk;
    if (stall) stall[c] = st;
    if (swapped) swapped[c] = out_b;
    orc_best key = { pk > budget ? pk - budget : 0, st, out_b, first_index + (uint64_t)c, pk };
    if (!have || orc_key_less(&key, &b)) { b = key; have = 1; }
  }
  if (best) *best = b;
  return 0;
}
