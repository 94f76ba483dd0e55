// core.cpp -- ctx lifecycle, errors, tokenizer, profiler hook (a1) and Algo. 1 (a2).
//
// PAPER.md citations: P:219 (hook at op dispatch), P:221 (Lightweight mode: operator names
// -> integer tensor), P:250-252 (Detailed mode: tensors, data_ptr, dtype, iteration time),
// P:263 (memory in use per op), P:224-248 (Algo. 1 stage adjusting), P:421 (m = 2, n = 5).
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>

#include "internal.h"

#include <map>
#include <mutex>

namespace chm {
static thread_local char g_err[512];
void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
}
}  // namespace chm

using namespace chm;

extern "C" const char *chm_last_error(void) { return g_err; }

extern "C" const char *chm_build_info(void) {
  return "libchm 0.1 (arxiv 2509.11076 swap hot path) sm_100a";
}

extern "C" void chm_config_default(chm_config *c) {
  std::memset(c, 0, sizeof *c);
  c->m = 2;
  c->n = 5;
  c->len_tol = 0.05;
  c->cos_tol = 0.95;
  c->cos_mode = 0;
  c->detect_bytes = 0;
  c->device = 0;
  c->host_arena_bytes = 0;
  c->swap_ctas = 0;
  c->eval_ctas_per_sm = 0;
  c->match_window = 0;
  c->time_batches = 0;
  c->swap_variant = 0;
  c->ce_min_bytes = 0;
  c->arena_mode = CHM_ARENA_AUTO;
  c->arena_numa = -1;
  c->arena_threads = 0;
}

extern "C" chm_status chm_create(const chm_config *cfg, chm_ctx **out) {
  if (!out) CHM_FAIL(CHM_E_INVAL, "chm_create: out is NULL");
  *out = nullptr;
  chm_config c;
  if (cfg) c = *cfg; else chm_config_default(&c);
  if (c.len_tol <= 0 || c.cos_tol <= 0 || c.cos_tol > 1 || c.cos_mode > 1 || c.swap_variant > 2)
    CHM_FAIL(CHM_E_INVAL, "chm_create: invalid Algo. 1 thresholds / cos_mode");
  if (c.arena_mode > CHM_ARENA_REGISTER || c.arena_numa < -2)
    CHM_FAIL(CHM_E_INVAL, "chm_create: arena_mode %u / arena_numa %d", c.arena_mode, c.arena_numa);
  if (c.device < 0) {  // host-only ctx: profiler, detection, trace build, executor tables
    if (c.host_arena_bytes) CHM_FAIL(CHM_E_INVAL, "chm_create: a host-only ctx has no arena");
    chm_ctx *ctx = new (std::nothrow) chm_ctx();
    if (!ctx) CHM_FAIL(CHM_E_NOMEM, "chm_create: out of host memory");
    ctx->cfg = c;
    ctx->device = -1;
    *out = ctx;
    return CHM_OK;
  }
  int ndev = 0;
  CHM_CUDA(cudaGetDeviceCount(&ndev));
  if (c.device >= ndev) CHM_FAIL(CHM_E_INVAL, "chm_create: device %d of %d", c.device, ndev);
  CHM_DEVICE_SCOPE(c.device);
  cudaDeviceProp prop;
  CHM_CUDA(cudaGetDeviceProperties(&prop, c.device));
  if (prop.major != 10 || prop.minor != 0)
    CHM_FAIL(CHM_E_NOKERNEL, "chm_create: libchm is built for sm_100a only, device is sm_%d%d",
             prop.major, prop.minor);
  chm_ctx *ctx = new (std::nothrow) chm_ctx();
  if (!ctx) CHM_FAIL(CHM_E_NOMEM, "chm_create: out of host memory");
  ctx->cfg = c;
  ctx->device = c.device;
  ctx->num_sms = prop.multiProcessorCount;
  ctx->arena_mode = c.arena_mode;
  ctx->arena_numa = c.arena_numa;
  ctx->arena_threads = c.arena_threads;
  {
    cudaError_t (*pre[])() = {preload_swap, preload_replay, preload_descend, preload_timeline, preload_explicit};
    for (auto f : pre) {
      const cudaError_t e = f();
      if (e != cudaSuccess) {
        delete ctx;
        CHM_FAIL(CHM_E_CUDA, "chm_create: loading the kernels: %s", cudaGetErrorString(e));
      }
    }
  }
  ctx->events.resize(kEventRing, nullptr);
  ctx->fences.resize(kEventRing, nullptr);
  for (int i = 0; i < kEventRing; i++) {
    if (cudaEventCreateWithFlags(&ctx->events[i], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->fences[i], cudaEventDisableTiming) != cudaSuccess) {
      chm_destroy(ctx);
      CHM_FAIL(CHM_E_CUDA, "chm_create: cudaEventCreate failed");
    }
  }
  if (c.time_batches) {
    ctx->t0.resize(kEventRing, nullptr);
    ctx->t1.resize(kEventRing, nullptr);
    for (int i = 0; i < kEventRing; i++) {
      if (cudaEventCreate(&ctx->t0[i]) != cudaSuccess || cudaEventCreate(&ctx->t1[i]) != cudaSuccess) {
        chm_destroy(ctx);
        CHM_FAIL(CHM_E_CUDA, "chm_create: cudaEventCreate (timing) failed");
      }
    }
  }
  if (c.host_arena_bytes) {
    chm_status st = arena_alloc(ctx, c.host_arena_bytes);  // arena.cpp
    if (st != CHM_OK) {
      std::string msg = chm_last_error();
      chm_destroy(ctx);
      CHM_FAIL(st, "chm_create: %s", msg.c_str());
    }
  }
  *out = ctx;
  return CHM_OK;
}

extern "C" void chm_destroy(chm_ctx *ctx) {
  if (!ctx) return;
  if (ctx->device < 0) { delete ctx; return; }
  DeviceGuard dg(ctx->device);
  for (auto e : ctx->events) if (e) cudaEventDestroy(e);
  for (auto e : ctx->fences) if (e) cudaEventDestroy(e);
  for (auto e : ctx->t0) if (e) cudaEventDestroy(e);
  for (auto e : ctx->t1) if (e) cudaEventDestroy(e);
  arena_free(ctx);
  if (ctx->eval_scratch) cudaFree(ctx->eval_scratch);
  if (ctx->tl_scratch) cudaFree(ctx->tl_scratch);
  if (ctx->tl_aux) cudaFree(ctx->tl_aux);
  delete ctx;
}

extern "C" chm_status chm_tokenize(chm_ctx *ctx, const char *name, int32_t *token) {
  if (!ctx || !name || !token) CHM_FAIL(CHM_E_INVAL, "chm_tokenize: NULL argument");
  auto it = ctx->tokens.find(name);
  if (it == ctx->tokens.end())
    it = ctx->tokens.emplace(name, int32_t(ctx->tokens.size() + 1)).first;
  *token = it->second;
  return CHM_OK;
}

extern "C" chm_status chm_set_detailed(chm_ctx *ctx, int32_t detailed) {
  if (!ctx) CHM_FAIL(CHM_E_INVAL, "chm_set_detailed: NULL ctx");
  ctx->force_detailed = detailed != 0;
  if (ctx->cur.tokens.empty()) ctx->cur.detailed = ctx->force_detailed || ctx->stage == CHM_GENPOLICY;
  return CHM_OK;
}

chm_status executor_on_op(chm_ctx *ctx, const chm_op_record *op, int32_t i);  // executor.cpp
void executor_end_iteration(chm_ctx *ctx);

extern "C" chm_status chm_record_op(chm_ctx *ctx, const chm_op_record *op, chm_actions *act) {
  if (!ctx || !op) CHM_FAIL(CHM_E_INVAL, "chm_record_op: NULL argument");
  if (op->token < 1) CHM_FAIL(CHM_E_INVAL, "chm_record_op: token %d < 1", op->token);
  if (op->phase > CHM_OPT) CHM_FAIL(CHM_E_INVAL, "chm_record_op: bad phase %u", op->phase);
  if ((op->n_in && !op->in) || (op->n_out && !op->out) || (op->n_free && !op->freed))
    CHM_FAIL(CHM_E_INVAL, "chm_record_op: NULL ref array");
  IterRecord &R = ctx->cur;
  if (!R.phase.empty() && op->phase < R.phase.back())
    CHM_FAIL(CHM_E_INVAL, "chm_record_op: phases interleave (FWD* BWD* OPT* required)");
  if (R.tokens.empty()) R.detailed = ctx->force_detailed || ctx->stage == CHM_GENPOLICY;
  const int32_t i = int32_t(R.tokens.size());
  R.tokens.push_back(op->token);
  R.phase.push_back(op->phase);
  for (uint32_t j = 0; j < op->n_out; j++) R.alloc_bytes += op->out[j].nbytes;
  if (R.detailed) {
    R.live_bytes.push_back(op->live_bytes);
    const size_t use_begin = R.use_idx.size();
    auto add_use = [&](int32_t t, bool is_in) {
      for (size_t u = use_begin; u < R.use_idx.size(); u++)
        if (R.use_idx[u] == t) return;  // one feature update per op and tensor
      R.use_idx.push_back(t);
      R.use_is_in.push_back(is_in ? 1 : 0);
    };
    for (uint32_t j = 0; j < op->n_in; j++) {
      const chm_tensor_ref &ref = op->in[j];
      auto it = ctx->id_to_tensor.find(ref.id);
      int32_t t;
      if (it == ctx->id_to_tensor.end()) {  // never produced in this iteration: static
        t = int32_t(R.tensors.size());
        TensorRec tr;
        tr.nbytes = ref.nbytes;
        tr.dtype = ref.dtype;
        R.tensors.push_back(tr);
        ctx->id_to_tensor.emplace(ref.id, t);
      } else {
        t = it->second;
      }
      add_use(t, true);
    }
    for (uint32_t j = 0; j < op->n_out; j++) {
      const chm_tensor_ref &ref = op->out[j];
      if (ref.nbytes <= 0) CHM_FAIL(CHM_E_INVAL, "chm_record_op: output %u has nbytes <= 0", j);
      int32_t t = int32_t(R.tensors.size());
      TensorRec tr;
      tr.nbytes = ref.nbytes;
      tr.dtype = ref.dtype;
      tr.producer = i;
      R.tensors.push_back(tr);
      ctx->id_to_tensor[ref.id] = t;  // a reused data_ptr is a new tensor
      R.out_idx.push_back(t);
      add_use(t, false);
    }
    for (uint32_t j = 0; j < op->n_free; j++) {
      auto it = ctx->id_to_tensor.find(op->freed[j]);
      if (it == ctx->id_to_tensor.end()) continue;  // block not seen in this iteration
      R.tensors[it->second].freed = i;
      R.free_idx.push_back(it->second);
      ctx->id_to_tensor.erase(it);
    }
    R.use_ptr.push_back(int32_t(R.use_idx.size()));
    R.out_ptr.push_back(int32_t(R.out_idx.size()));
    R.free_ptr.push_back(int32_t(R.free_idx.size()));
  }
  // resident produced tensors: the candidates of a passive swap (Algo. 3 (iv))
  for (uint32_t j = 0; j < op->n_out; j++) ctx->resident[op->out[j].id] = {op->out[j].nbytes, ctx->resident_seq++};
  for (uint32_t j = 0; j < op->n_free; j++) ctx->resident.erase(op->freed[j]);
  if (act) std::memset(act, 0, sizeof *act);
  if (ctx->policy_active) {
    chm_status st = executor_on_op(ctx, op, i);
    if (st != CHM_OK) return st;
    if (act) {
      act->n_swap_out = uint32_t(ctx->act_out.size());
      act->swap_out = ctx->act_out.data();
      act->swap_out_item = ctx->act_out_item.data();
      act->n_release = uint32_t(ctx->act_release.size());
      act->release_item = ctx->act_release.data();
      act->n_swap_in = uint32_t(ctx->act_in.size());
      act->swap_in = ctx->act_in.data();
      act->swap_in_item = ctx->act_in_item.data();
      act->n_wait = uint32_t(ctx->act_wait.size());
      act->wait_item = ctx->act_wait.data();
    }
  }
  return CHM_OK;
}

extern "C" chm_status chm_record_tokens(chm_ctx *ctx, const int32_t *tokens, const uint8_t *phases, uint32_t n) {
  if (!ctx || (n && (!tokens || !phases))) CHM_FAIL(CHM_E_INVAL, "chm_record_tokens: NULL argument");
  if (ctx->policy_active && !ctx->items.empty())
    CHM_FAIL(CHM_E_STATE, "chm_record_tokens: a policy is installed (chm_record_op per op)");
  IterRecord &R = ctx->cur;
  if (R.detailed && !R.tokens.empty() && n)
    CHM_FAIL(CHM_E_STATE, "chm_record_tokens: this iteration is being recorded in Detailed mode");
  if (R.tokens.empty()) R.detailed = false;  // a bulk-recorded iteration is Lightweight
  for (uint32_t j = 0; j < n; j++) {
    if (tokens[j] < 1) CHM_FAIL(CHM_E_INVAL, "chm_record_tokens: token %d < 1 at %u", tokens[j], j);
    if (phases[j] > CHM_OPT || (!R.phase.empty() && phases[j] < R.phase.back()))
      CHM_FAIL(CHM_E_INVAL, "chm_record_tokens: bad or interleaved phase at %u", j);
    R.tokens.push_back(tokens[j]);
    R.phase.push_back(phases[j]);
  }
  return CHM_OK;
}

// Positional (cos_mode 0) or histogram (cos_mode 1) cosine similarity of two token
// sequences: dot and squared norms are exact int64 sums, then one double divide + sqrt.
static bool seq_compare(const std::vector<int32_t> &a, const std::vector<int32_t> &b,
                        uint32_t cos_mode, double *len_diff, double *cos_sim) {
  const size_t na = a.size(), nb = b.size();
  if (na == 0 || nb == 0) { *len_diff = 1.0; *cos_sim = 0.0; return false; }
  const size_t mx = std::max(na, nb);
  *len_diff = double(na > nb ? na - nb : nb - na) / double(mx);
  int64_t dot = 0, aa = 0, bb = 0;
  if (cos_mode == 0) {
    const size_t mn = std::min(na, nb);
    for (size_t i = 0; i < mn; i++) {
      dot += int64_t(a[i]) * b[i];
      aa += int64_t(a[i]) * a[i];
      bb += int64_t(b[i]) * b[i];
    }
    for (size_t i = mn; i < na; i++) aa += int64_t(a[i]) * a[i];
    for (size_t i = mn; i < nb; i++) bb += int64_t(b[i]) * b[i];
  } else {
    int32_t V = 0;
    for (auto x : a) V = std::max(V, x);
    for (auto x : b) V = std::max(V, x);
    std::vector<int64_t> ha(size_t(V) + 1, 0), hb(size_t(V) + 1, 0);
    for (auto x : a) ha[x]++;
    for (auto x : b) hb[x]++;
    for (int32_t v = 0; v <= V; v++) {
      dot += ha[v] * hb[v];
      aa += ha[v] * ha[v];
      bb += hb[v] * hb[v];
    }
  }
  *cos_sim = double(dot) / std::sqrt(double(aa) * double(bb));
  return true;
}

extern "C" chm_status chm_detect_seq_change(chm_ctx *ctx, double t_iter_s, chm_stage *stage,
                                            int32_t *changed, double *len_diff, double *cos_sim) {
  if (!ctx) CHM_FAIL(CHM_E_INVAL, "chm_detect_seq_change: NULL ctx");
  IterRecord &R = ctx->cur;
  // Algo. 1: static variables initialised once with the first sequence
  if (!ctx->stage_init) {
    ctx->prev_tokens = R.tokens;
    ctx->prev_alloc_bytes = R.alloc_bytes;
    ctx->stage = CHM_WARMUP;
    ctx->stable_step = 0;
    ctx->stage_init = true;
  }
  double ld = 1.0, cs = 0.0;
  bool ok = seq_compare(R.tokens, ctx->prev_tokens, ctx->cfg.cos_mode, &ld, &cs);
  bool stable = ok && ld < ctx->cfg.len_tol && cs > ctx->cfg.cos_tol;  // P:235-236, strict
  if (stable && ctx->cfg.detect_bytes) {  // reading Q4 (opt-in): shape-only changes
    const int64_t x = R.alloc_bytes, y = ctx->prev_alloc_bytes;
    const int64_t mx = std::max(x, y);
    const double bd = mx > 0 ? double(x > y ? x - y : y - x) / double(mx) : 0.0;
    stable = bd < ctx->cfg.len_tol;
  }
  if (stable) {
    ctx->stable_step += 1;
    if (ctx->stage == CHM_WARMUP && ctx->stable_step > int32_t(ctx->cfg.m)) {
      ctx->stage = CHM_GENPOLICY;
      ctx->stable_step = 0;
    } else if (ctx->stage == CHM_GENPOLICY && ctx->stable_step > int32_t(ctx->cfg.n)) {
      ctx->stage = CHM_STABLE;
    }  // else: Stage keeps PrevStage (reading Q3)
  } else {
    ctx->stage = CHM_WARMUP;
    ctx->stable_step = 0;
  }
  ctx->prev_tokens = R.tokens;  // PrevOpSeq <- OpSeq
  ctx->prev_alloc_bytes = R.alloc_bytes;
  if (R.detailed) {
    R.t_iter = t_iter_s;
    ctx->last_detailed = std::move(R);
  }
  ctx->cur.clear();
  ctx->id_to_tensor.clear();
  ctx->resident.clear();  // passive-swap candidates are this iteration's produced tensors
  for (auto &kv : ctx->passive) {  // still passively out: off the device from op 0 on
    ctx->cur.swaps.push_back({0, INT32_MAX, kv.second.nbytes, kv.second.id});
    kv.second.span = int32_t(ctx->cur.swaps.size()) - 1;
    kv.second.tensor = -1;  // a tensor of the previous iteration's record
    kv.second.has_live = false;
  }
  executor_end_iteration(ctx);
  if (stage) *stage = ctx->stage;
  if (changed) *changed = stable ? 0 : 1;
  if (len_diff) *len_diff = ld;
  if (cos_sim) *cos_sim = cs;
  return CHM_OK;
}

extern "C" chm_status chm_best_reduce(const chm_best *keys, uint32_t n, chm_best *out) {
  if (!keys || !out || n == 0) CHM_FAIL(CHM_E_INVAL, "chm_best_reduce: empty input");
  chm_best b = keys[0];
  for (uint32_t i = 1; i < n; i++) {
    const chm_best &k = keys[i];
    bool less = k.excess != b.excess ? k.excess < b.excess
              : k.stall != b.stall   ? k.stall < b.stall
              : k.swapped_bytes != b.swapped_bytes ? k.swapped_bytes < b.swapped_bytes
              : k.index < b.index;
    if (less) b = k;
  }
  *out = b;
  return CHM_OK;
}

namespace chm {
cudaError_t ensure_dyn_smem(const void *f, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void *>, size_t> set;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  size_t &cur = set[{dev, f}];
  if (bytes <= cur) return cudaSuccess;
  e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
  if (e == cudaSuccess) cur = bytes;
  return e;
}
}  // namespace chm
