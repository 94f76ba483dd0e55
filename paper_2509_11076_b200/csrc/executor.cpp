// executor.cpp -- policy install + trigger tables (step a8): App. A multi-feature fuzzy
// matching, swap-out right after the last FWD use, stream-
// ordered release at the simulator's completion op (custom recordStream),
// swap-in pre-triggered at the chosen layer start.
#include <algorithm>
#include <climits>
#include <cstring>

#include "internal.h"

using namespace chm;

static uint64_t splitmix64(uint64_t z) {  // SEEDED candidate decode, SURVEY §8(c).4
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

extern "C" chm_status chm_candidate_mask(const chm_trace *t, const chm_candidates *c,
                                         uint64_t index, uint64_t *words) {
  if (!t || !c || !words) CHM_FAIL(CHM_E_INVAL, "chm_candidate_mask: NULL argument");
  const int32_t K = t->K, W = t->W;
  std::fill(words, words + W, 0ull);
  switch (c->kind) {
    case CHM_CAND_EXHAUSTIVE:
      if (K > 63) CHM_FAIL(CHM_E_INVAL, "EXHAUSTIVE needs K <= 63");
      if (W) words[0] = index & ((K == 64) ? ~0ull : ((1ull << K) - 1));
      return CHM_OK;
    case CHM_CAND_SEEDED: {
      const uint64_t *base = c->base_mask ? c->base_mask : t->base.data();
      const uint64_t J = (uint64_t(K) + 3) / 4, thr16 = c->flip_thr >> 48;
      for (int32_t k = 0; k < K; k++) {
        uint64_t bit = (base[k / 64] >> (k % 64)) & 1ull;
        const uint64_t w = splitmix64(c->seed ^ (index * J + uint64_t(k / 4)));
        bit ^= ((w >> (16 * (k % 4))) & 0xffffull) < thr16 ? 1ull : 0ull;
        words[k / 64] |= bit << (k % 64);
      }
      return CHM_OK;
    }
    case CHM_CAND_FLIP1: {
      if (index > uint64_t(K)) CHM_FAIL(CHM_E_INVAL, "chm_candidate_mask: FLIP1 index %llu > K", (unsigned long long)index);
      const uint64_t *base = c->base_mask ? c->base_mask : t->base.data();
      std::copy(base, base + W, words);
      if (index < uint64_t(K)) words[index / 64] ^= 1ull << (index % 64);
      return CHM_OK;
    }
    default:
      CHM_FAIL(CHM_E_INVAL, "chm_candidate_mask: MASKS candidates live on the device");
  }
}

// App. A tables from the recorded iteration's token frequencies: rank by count descending,
// ties by first appearance; index = min(rank + 1, 255); one-hot for the 32 most frequent.
static void feature_tables(const std::vector<int32_t> &tokens, std::vector<uint8_t> &index,
                           std::vector<uint32_t> &onehot) {
  int32_t V = 0;
  for (auto x : tokens) V = std::max(V, x);
  std::vector<int64_t> cnt(size_t(V) + 1, 0);
  std::vector<int32_t> first(size_t(V) + 1, -1);
  for (size_t i = 0; i < tokens.size(); i++) {
    cnt[tokens[i]]++;
    if (first[tokens[i]] < 0) first[tokens[i]] = int32_t(i);
  }
  std::vector<int32_t> order;
  for (int32_t v = 0; v <= V; v++) if (cnt[v]) order.push_back(v);
  std::sort(order.begin(), order.end(), [&](int32_t x, int32_t y) {
    return cnt[x] != cnt[y] ? cnt[x] > cnt[y] : first[x] < first[y];
  });
  index.assign(size_t(V) + 1, 0);
  onehot.assign(size_t(V) + 1, 0);
  for (size_t rk = 0; rk < order.size(); rk++) {
    index[order[rk]] = uint8_t(std::min<size_t>(rk + 1, 255));
    onehot[order[rk]] = rk < 32 ? (1u << rk) : 0u;
  }
}

static inline void feature_update(Feature &f, int32_t token, uint8_t dtype, uint32_t slot,
                                  const chm_ctx *ctx) {
  uint8_t idx = 0;
  uint32_t oh = 0;
  if (token >= 0 && size_t(token) < ctx->op_index.size()) {
    idx = ctx->op_index[token];
    oh = ctx->op_onehot[token];
  }
  f.count += 1;                       // opCount++
  f.tag |= oh;                        // opTag |= opOneHot
  f.stack = (f.stack << 8) + idx;     // opCallStack = (opCallStack << 8) + opIndex
  f.dtype = dtype;
  f.slot = uint8_t(slot < 255 ? slot : 255);  // position among the op's distinct tensors
}

namespace {
struct InstallItem {
  int32_t tid, r, s;
  int64_t nbytes;
};
}  // namespace

static chm_status install_items(chm_ctx *ctx, const chm_trace *t, const std::vector<InstallItem> &sel) {
  uint64_t need = 0;
  for (const InstallItem &x : sel) need += (uint64_t(x.nbytes) + 511) & ~uint64_t(511);
  if (!ctx->passive.empty())
    CHM_FAIL(CHM_E_STATE, "policy install: %zu passive swaps outstanding (restore them first)", ctx->passive.size());
  if (ctx->device >= 0 && need > ctx->arena_bytes) {  // a host-only ctx plans offsets only
    // grow to the policy's slots plus the passive-swap room kept above the previous policy
    const uint64_t room = (ctx->policy_active && ctx->arena_bytes > ctx->passive_base)
                              ? ctx->arena_bytes - ctx->passive_base : 0;
    const chm_status st = chm_arena_reserve(ctx, need + room);
    if (st != CHM_OK) return st;
  }
  feature_tables(t->tokens, ctx->op_index, ctx->op_onehot);
  // feature key of every selected tensor right after op a_t (replay of the recorded uses)
  std::vector<int32_t> item_of_tensor(size_t(t->T), -1);
  ctx->items.assign(sel.size(), PolicyItem());
  uint64_t off = 0;
  for (size_t j = 0; j < sel.size(); j++) {
    const int32_t tid = sel[j].tid;
    PolicyItem &it = ctx->items[j];
    it.a = t->a[tid];
    it.b = t->b[tid];
    it.r = sel[j].r;
    it.s = sel[j].s;
    it.nbytes = sel[j].nbytes;
    it.host_off = off;
    off += (uint64_t(it.nbytes) + 511) & ~uint64_t(511);
    item_of_tensor[tid] = int32_t(j);
  }
  ctx->passive_base = off;  // passive swaps (Algo. 3) use the arena above the policy's slots
  ctx->passive_free.clear();
  std::vector<Feature> feat(size_t(t->T));
  for (int32_t i = 0; i < t->N; i++) {
    for (int32_t u = t->use_ptr[i]; u < t->use_ptr[i + 1]; u++) {
      const int32_t tid = t->use_idx[u];
      feature_update(feat[tid], t->tokens[i], t->dtype[tid], uint32_t(u - t->use_ptr[i]), ctx);
      const int32_t j = item_of_tensor[tid];
      if (j >= 0 && ctx->items[j].a == i) ctx->items[j].key = feat[tid];
    }
  }
  // key = (App. A feature after a_t, a_t): the same tensor role repeats in every layer of a
  // stacked model with identical features, so the recorded op index is part of the key and
  // run-time ops are aligned to the recorded sequence (align_op)
  ctx->key_to_item.clear();
  ctx->stats = chm_exec_stats{};
  ctx->stats.n_items = uint32_t(sel.size());
  for (size_t j = 0; j < ctx->items.size(); j++) {
    FeatureAt k;
    k.f = ctx->items[j].key;
    k.a = ctx->items[j].a;
    if (!ctx->key_to_item.emplace(k, int32_t(j)).second) ctx->stats.n_collisions++;
  }
  ctx->rec_tokens = t->tokens;
  ctx->align_cursor = 0;
  // index-keyed tables: actions returned by chm_record_op(op i) happen between op i and i+1
  const size_t N = size_t(t->N);
  ctx->release_at.assign(N, {});
  ctx->swapin_at.assign(N, {});
  ctx->wait_at.assign(N, {});
  for (size_t j = 0; j < ctx->items.size(); j++) {
    const PolicyItem &it = ctx->items[j];
    ctx->release_at[it.r].push_back(int32_t(j));                       // after op r_t
    if (it.s >= 1) ctx->swapin_at[it.s - 1].push_back(int32_t(j));     // before op s_t
    if (it.b >= 1) ctx->wait_at[it.b - 1].push_back(int32_t(j));       // before op b_t
  }
  ctx->match_window = ctx->cfg.match_window ? int32_t(ctx->cfg.match_window) : 32;
  ctx->live.clear();
  ctx->op_cursor = 0;
  ctx->policy_active = true;
  return CHM_OK;
}

extern "C" chm_status chm_policy_install(chm_ctx *ctx, const chm_trace *t, const uint64_t *words) {
  if (!ctx || !t || (!words && t->W)) CHM_FAIL(CHM_E_INVAL, "chm_policy_install: NULL argument");
  std::vector<InstallItem> sel;
  for (int32_t k = 0; k < t->K; k++)
    if ((words[k / 64] >> (k % 64)) & 1ull)
      sel.push_back({t->sw_tensor_idx[k], t->sw_r[k], t->sw_s[k], t->sw_S[k]});
  return install_items(ctx, t, sel);
}

extern "C" chm_status chm_policy_install_items(chm_ctx *ctx, const chm_trace *t, const chm_item *items,
                                               uint32_t n) {
  if (!ctx || !t || (n && !items)) CHM_FAIL(CHM_E_INVAL, "chm_policy_install_items: NULL argument");
  const int32_t n_prod = int32_t(t->rank_to_tensor.size());
  std::vector<InstallItem> sel;
  std::vector<char> seen(size_t(n_prod), 0);
  for (uint32_t j = 0; j < n; j++) {
    const chm_item &it = items[j];
    if (int64_t(it.t) >= n_prod) CHM_FAIL(CHM_E_INVAL, "chm_policy_install_items: item %u: bad tensor", j);
    const int32_t tid = t->rank_to_tensor[it.t];
    if (t->a[tid] < 0 || t->b[tid] < 0 || it.r < t->a[tid] || !(it.r + 1 < it.s) || it.s > t->b[tid] || seen[it.t])
      CHM_FAIL(CHM_E_INVAL, "chm_policy_install_items: item %u (t %u, r %d, s %d) invalid", j, it.t, it.r, it.s);
    seen[it.t] = 1;
    sel.push_back({tid, it.r, it.s, t->S_t[tid]});
  }
  std::stable_sort(sel.begin(), sel.end(), [&](const InstallItem &x, const InstallItem &y) {
    if (t->a[x.tid] != t->a[y.tid]) return t->a[x.tid] < t->a[y.tid];
    return t->tensor_rank[x.tid] < t->tensor_rank[y.tid];
  });
  return install_items(ctx, t, sel);
}

// Aligns run-time op i to a recorded op index: the next recorded op if its token matches; else
// the first match within `match_window` recorded ops ahead (recorded ops were skipped); else -1
// (an inserted op, e.g. on-the-fly validation or a conditional branch).
static int32_t align_op(chm_ctx *ctx, int32_t token) {
  const int32_t n = int32_t(ctx->rec_tokens.size());
  const int32_t j0 = ctx->align_cursor;
  for (int32_t j = j0; j < n && j <= j0 + ctx->match_window; j++) {
    if (ctx->rec_tokens[j] == token) {
      ctx->align_cursor = j + 1;
      return j;
    }
  }
  return -1;
}

// A released block's address may name a new tensor at once: the Detailed record keeps the
// swapped tensor's index on the item until its swap-in re-aliases it to the new address.
void chm::stash_record(chm_ctx *ctx, PolicyItem &it) {
  auto tt = ctx->id_to_tensor.find(it.cur_id);
  if (tt == ctx->id_to_tensor.end()) return;
  it.rec_tensor = tt->second;
  ctx->id_to_tensor.erase(tt);
}

chm_status executor_on_op(chm_ctx *ctx, const chm_op_record *op, int32_t i) {
  ctx->act_out.clear(); ctx->act_out_item.clear(); ctx->act_in.clear(); ctx->act_in_item.clear();
  ctx->act_release.clear(); ctx->act_wait.clear();
  const int32_t ra = align_op(ctx, op->token);
  uint64_t seen[64];
  uint32_t n_seen = 0;
  auto visit = [&](const chm_tensor_ref &ref, bool is_out) {
    for (uint32_t q = 0; q < n_seen && q < 64; q++) if (seen[q] == ref.id) return;
    const uint32_t slot = n_seen;
    if (n_seen < 64) seen[n_seen++] = ref.id;
    LiveTensor *lt;
    if (is_out) {
      lt = &(ctx->live[ref.id] = LiveTensor());
    } else {
      lt = &ctx->live[ref.id];
    }
    feature_update(lt->f, op->token, ref.dtype, slot, ctx);
    if (op->phase != CHM_FWD || lt->item >= 0 || ra < 0) return;
    FeatureAt key;
    key.f = lt->f;
    key.a = ra;
    auto m = ctx->key_to_item.find(key);
    if (m == ctx->key_to_item.end()) return;
    const int32_t j = m->second;
    PolicyItem &it = ctx->items[j];
    if (it.state != IT_IDLE) { ctx->stats.n_collisions++; return; }  // first one wins
    const uint64_t slot_bytes = (uint64_t(it.nbytes) + 511) & ~uint64_t(511);
    if (uint64_t(ref.nbytes) > slot_bytes) return;  // larger than its arena slot: cannot swap
    it.state = IT_OUT;
    it.cur_id = ref.id;
    it.cur_bytes = uint64_t(ref.nbytes);
    it.has_out = it.has_in = false;
    it.span = -1;
    it.rec_tensor = -1;
    lt->item = j;
    ctx->stats.n_matched++;
    ctx->act_out.push_back({ref.id, it.host_off, uint64_t(ref.nbytes)});
    ctx->act_out_item.push_back(uint32_t(j));
  };
  for (uint32_t j = 0; j < op->n_in; j++) visit(op->in[j], false);
  for (uint32_t j = 0; j < op->n_out; j++) visit(op->out[j], true);
  for (uint32_t j = 0; j < op->n_free; j++) ctx->live.erase(op->freed[j]);
  if (ra >= 0 && size_t(ra) < ctx->release_at.size()) {
    for (int32_t j : ctx->release_at[ra]) {
      PolicyItem &it = ctx->items[j];
      if (it.state != IT_OUT) continue;
      it.state = IT_RELEASED;
      ctx->live.erase(it.cur_id);  // the caller drops the device storage after the wait
      ctx->resident.erase(it.cur_id);
      stash_record(ctx, it);
      ctx->cur.swaps.push_back({i + 1, INT32_MAX, int64_t(it.cur_bytes), it.cur_id});  // off from op i+1
      it.span = int32_t(ctx->cur.swaps.size()) - 1;
      ctx->act_release.push_back(uint32_t(j));
    }
    for (int32_t j : ctx->swapin_at[ra]) {
      PolicyItem &it = ctx->items[j];
      if (it.state != IT_RELEASED) continue;
      if (it.span >= 0 && size_t(it.span) < ctx->cur.swaps.size()) ctx->cur.swaps[it.span].to = i + 1;
      ctx->act_in.push_back({0, it.host_off, it.cur_bytes});
      ctx->act_in_item.push_back(uint32_t(j));
    }
    for (int32_t j : ctx->wait_at[ra]) {
      PolicyItem &it = ctx->items[j];
      if (it.state == IT_IN) ctx->act_wait.push_back(uint32_t(j));  // s_t < b_t: issued
    }
  }
  ctx->op_cursor = i + 1;
  return CHM_OK;
}

void executor_end_iteration(chm_ctx *ctx) {
  if (!ctx->policy_active) return;
  for (PolicyItem &it : ctx->items) {
    if (it.state == IT_IDLE) ctx->stats.n_stale++;  // never matched: diagnostic
    it.state = IT_IDLE;
  }
  ctx->live.clear();
  ctx->op_cursor = 0;
  ctx->align_cursor = 0;
}

extern "C" chm_status chm_exec_stats_get(chm_ctx *ctx, chm_exec_stats *s) {
  if (!ctx || !s) CHM_FAIL(CHM_E_INVAL, "chm_exec_stats_get: NULL argument");
  *s = ctx->stats;
  return CHM_OK;
}

extern "C" chm_status chm_issue_swap_out(chm_ctx *ctx, cudaStream_t compute, cudaStream_t swap,
                                         uint32_t flags, uint64_t *batch) {
  if (!ctx) CHM_FAIL(CHM_E_INVAL, "chm_issue_swap_out: NULL ctx");
  if (ctx->act_out.empty()) { if (batch) *batch = ~0ull; return CHM_OK; }
  uint64_t b = 0;
  int64_t err = -1;
  chm_status st = chm_swap_out(ctx, ctx->act_out.data(), uint32_t(ctx->act_out.size()), compute,
                               swap, flags, &b, &err);
  if (st != CHM_OK) return st;
  for (uint32_t j : ctx->act_out_item) {
    ctx->items[j].out_batch = b;
    ctx->items[j].has_out = true;
    ctx->stats.bytes_out += ctx->items[j].cur_bytes;
  }
  ctx->act_out.clear();
  if (batch) *batch = b;
  return CHM_OK;
}

extern "C" chm_status chm_issue_swap_in(chm_ctx *ctx, const uint64_t *dev, cudaStream_t compute,
                                        cudaStream_t swap, uint32_t flags, uint64_t *batch) {
  if (!ctx) CHM_FAIL(CHM_E_INVAL, "chm_issue_swap_in: NULL ctx");
  if (ctx->act_in.empty()) { if (batch) *batch = ~0ull; return CHM_OK; }
  if (!dev) CHM_FAIL(CHM_E_INVAL, "chm_issue_swap_in: NULL destination list");
  for (size_t j = 0; j < ctx->act_in.size(); j++) ctx->act_in[j].dev = dev[j];
  uint64_t b = 0;
  int64_t err = -1;
  chm_status st = chm_swap_in(ctx, ctx->act_in.data(), uint32_t(ctx->act_in.size()), compute,
                              swap, flags, &b, &err);
  if (st != CHM_OK) return st;
  for (size_t j = 0; j < ctx->act_in_item.size(); j++) {
    PolicyItem &it = ctx->items[ctx->act_in_item[j]];
    it.in_batch = b;
    it.has_in = true;
    it.state = IT_IN;
    it.cur_id = dev[j];
    if (it.rec_tensor >= 0) ctx->id_to_tensor[dev[j]] = it.rec_tensor;  // same recorded tensor
    LiveTensor &lt = ctx->live[dev[j]];
    lt.item = int32_t(ctx->act_in_item[j]);
    ctx->stats.bytes_in += it.cur_bytes;
  }
  ctx->act_in.clear();
  if (batch) *batch = b;
  return CHM_OK;
}

extern "C" chm_status chm_item_wait(chm_ctx *ctx, uint32_t item, int32_t swap_in, cudaStream_t stream) {
  if (!ctx || item >= ctx->items.size()) CHM_FAIL(CHM_E_INVAL, "chm_item_wait: bad item");
  const PolicyItem &it = ctx->items[item];
  if (swap_in ? !it.has_in : !it.has_out)
    CHM_FAIL(CHM_E_STATE, "chm_item_wait: item %u has no %s batch", item, swap_in ? "swap-in" : "swap-out");
  return chm_batch_wait(ctx, swap_in ? it.in_batch : it.out_batch, stream);
}
