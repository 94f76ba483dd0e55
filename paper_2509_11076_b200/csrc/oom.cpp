// oom.cpp -- NEXT-4: WarmUp-stage OOM handling, Algo. 3 of the paper:
//   (i)-(ii)  release every block marked by the custom recordStream (swap-outs issued, release
//             point not reached) behind an event record/wait between swap and compute streams;
//   (iv)      passive swap of the resident tensor whose size is closest to the failed request,
//             again fenced by an event pair -- no host synchronisation;
// plus the demand swap-in a passively swapped tensor needs before its next use (reading Q20).
// Every release / swap-in is logged per recorded iteration: the swap log of Fig. 3.
// (Step (iii), GMLake defragmentation, is out of scope: DESIGN.md §8.)
#include <algorithm>
#include <climits>

#include "internal.h"

using namespace chm;

static int32_t current_op(const chm_ctx *ctx) { return int32_t(ctx->cur.tokens.size()); }

extern "C" chm_status chm_oom_release(chm_ctx *ctx, cudaStream_t compute, uint32_t *items, uint32_t cap,
                                      uint32_t *n_items) {
  if (!ctx || !n_items || (cap && !items)) CHM_FAIL(CHM_E_INVAL, "chm_oom_release: NULL argument");
  if (ctx->device < 0) CHM_FAIL(CHM_E_STATE, "chm_oom_release: host-only ctx");
  uint32_t n = 0;
  for (size_t j = 0; j < ctx->items.size(); j++) {
    PolicyItem &it = ctx->items[j];
    if (it.state != IT_OUT || !it.has_out) continue;
    chm_status st = chm_batch_wait(ctx, it.out_batch, compute);  // event pair
    if (st != CHM_OK) return st;
    it.state = IT_RELEASED;
    ctx->live.erase(it.cur_id);
    ctx->resident.erase(it.cur_id);
    stash_record(ctx, it);
    ctx->cur.swaps.push_back({current_op(ctx), INT32_MAX, int64_t(it.cur_bytes), it.cur_id});
    it.span = int32_t(ctx->cur.swaps.size()) - 1;
    if (n < cap) items[n] = uint32_t(j);
    n++;
  }
  *n_items = n;
  if (n > cap) CHM_FAIL(CHM_E_INVAL, "chm_oom_release: %u items exceed cap %u", n, cap);
  return CHM_OK;
}

static bool passive_alloc(chm_ctx *ctx, uint64_t bytes, uint64_t *off) {
  if (ctx->passive_free.empty() && ctx->passive.empty() && ctx->passive_base < ctx->arena_bytes)
    ctx->passive_free.push_back({ctx->passive_base, ctx->arena_bytes - ctx->passive_base});
  bytes = (bytes + 511) & ~uint64_t(511);
  for (size_t j = 0; j < ctx->passive_free.size(); j++) {
    auto &f = ctx->passive_free[j];
    if (f.second < bytes) continue;
    *off = f.first;
    f.first += bytes;
    f.second -= bytes;
    if (!f.second) ctx->passive_free.erase(ctx->passive_free.begin() + long(j));
    return true;
  }
  return false;
}

static void passive_free_range(chm_ctx *ctx, uint64_t off, uint64_t bytes) {
  bytes = (bytes + 511) & ~uint64_t(511);
  auto &fl = ctx->passive_free;
  auto pos = std::lower_bound(fl.begin(), fl.end(), std::make_pair(off, uint64_t(0)));
  pos = fl.insert(pos, {off, bytes});
  if (pos + 1 != fl.end() && pos->first + pos->second == (pos + 1)->first) {  // merge right
    pos->second += (pos + 1)->second;
    fl.erase(pos + 1);
  }
  if (pos != fl.begin() && (pos - 1)->first + (pos - 1)->second == pos->first) {  // merge left
    (pos - 1)->second += pos->second;
    fl.erase(pos);
  }
}

extern "C" chm_status chm_passive_swap(chm_ctx *ctx, int64_t need, const uint64_t *exclude, uint32_t n_exclude,
                                       const uint64_t *only, uint32_t n_only, cudaStream_t compute,
                                       cudaStream_t swap, chm_passive *out) {
  if (!ctx || !out || (n_exclude && !exclude) || (n_only && !only))
    CHM_FAIL(CHM_E_INVAL, "chm_passive_swap: NULL argument");
  if (ctx->device < 0) CHM_FAIL(CHM_E_STATE, "chm_passive_swap: host-only ctx");
  // closest size to the request: the smallest resident tensor >= need, else the largest; ties
  // by age (older first)
  uint64_t best = 0;
  int64_t bsz = 0;
  uint64_t bseq = 0;
  bool found = false, above = false;
  for (const auto &kv : ctx->resident) {
    const uint64_t id = kv.first;
    const int64_t sz = kv.second.nbytes;
    if (std::find(exclude, exclude + n_exclude, id) != exclude + n_exclude) continue;
    if (only && std::find(only, only + n_only, id) == only + n_only) continue;
    auto lt = ctx->live.find(id);
    if (lt != ctx->live.end() && lt->second.item >= 0) continue;  // bound to a policy item
    const bool ab = sz >= need;
    bool better;
    if (!found) better = true;
    else if (ab != above) better = ab;
    else if (sz != bsz) better = ab ? sz < bsz : sz > bsz;
    else better = kv.second.seq < bseq;
    if (better) { best = id; bsz = sz; bseq = kv.second.seq; above = ab; found = true; }
  }
  if (!found) CHM_FAIL(CHM_E_NOMEM, "chm_passive_swap: no resident tensor to swap (need %lld B)", (long long)need);
  uint64_t off = 0;
  if (!passive_alloc(ctx, uint64_t(bsz), &off))
    CHM_FAIL(CHM_E_NOMEM, "chm_passive_swap: arena has no room for %lld B", (long long)bsz);
  chm_swap_desc d{best, off, uint64_t(bsz)};
  uint64_t b = 0;
  int64_t err = -1;
  chm_status st = chm_swap_out(ctx, &d, 1, compute, swap, CHM_SWAP_KERNEL, &b, &err);
  if (st != CHM_OK) { passive_free_range(ctx, off, uint64_t(bsz)); return st; }
  st = chm_batch_wait(ctx, b, compute);  // the block is reusable once the copy is done (P:410 (iv))
  if (st != CHM_OK) return st;
  chm_ctx::Passive p{};
  p.id = best;
  p.nbytes = bsz;
  p.host_off = off;
  p.batch = b;
  ctx->cur.swaps.push_back({current_op(ctx), INT32_MAX, bsz, best});
  p.span = int32_t(ctx->cur.swaps.size()) - 1;
  // the freed block's address may name a new tensor at once: stash the tensor's identity
  p.tensor = -1;
  auto tt = ctx->id_to_tensor.find(best);
  if (tt != ctx->id_to_tensor.end()) { p.tensor = tt->second; ctx->id_to_tensor.erase(tt); }
  auto lt = ctx->live.find(best);
  p.has_live = lt != ctx->live.end();
  if (p.has_live) { p.live = lt->second; ctx->live.erase(lt); }
  ctx->resident.erase(best);
  const uint64_t h = ctx->passive_next++;
  ctx->passive[h] = p;
  out->handle = h;
  out->id = best;
  out->nbytes = bsz;
  out->host_off = off;
  out->batch = b;
  return CHM_OK;
}

extern "C" chm_status chm_passive_restore(chm_ctx *ctx, uint64_t handle, uint64_t dev, cudaStream_t compute,
                                          cudaStream_t swap) {
  if (!ctx) CHM_FAIL(CHM_E_INVAL, "chm_passive_restore: NULL ctx");
  auto it = ctx->passive.find(handle);
  if (it == ctx->passive.end())
    CHM_FAIL(CHM_E_INVAL, "chm_passive_restore: %llu is not a passive swap", (unsigned long long)handle);
  chm_ctx::Passive &p = it->second;
  const int32_t i = current_op(ctx);
  IterRecord &R = ctx->cur;
  if (dev) {
    chm_swap_desc d{dev, p.host_off, uint64_t(p.nbytes)};
    uint64_t b = 0;
    int64_t err = -1;
    chm_status st = chm_swap_in(ctx, &d, 1, compute, swap, CHM_SWAP_KERNEL, &b, &err);
    if (st != CHM_OK) return st;
    st = chm_batch_wait(ctx, b, compute);  // demand swap-in: the op waits (a stall, reading Q20)
    if (st != CHM_OK) return st;
    if (p.span >= 0 && size_t(p.span) < R.swaps.size()) R.swaps[p.span].to = i;  // back for op i
    ctx->resident[dev] = {p.nbytes, ctx->resident_seq++};
    if (p.tensor >= 0) ctx->id_to_tensor[dev] = p.tensor;
    if (p.has_live) ctx->live[dev] = p.live;
    ctx->stats.n_demand_swap_in++;
  } else {
    // died while out: its last use was op i-1; off the device until then
    if (p.span >= 0 && size_t(p.span) < R.swaps.size()) R.swaps[p.span].to = i;
    if (p.tensor >= 0 && R.detailed && i > 0) R.tensors[p.tensor].freed = i - 1;
  }
  passive_free_range(ctx, p.host_off, uint64_t(p.nbytes));
  ctx->passive.erase(it);
  return CHM_OK;
}
