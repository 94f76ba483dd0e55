/* A plain C99 client of the C ABI (no Python, no CUDA device): a host-only ctx records three
 * iterations of a small stacked model through chm_record_op, runs Algo. 1, builds the trace
 * from the Detailed iteration, runs the Algo. 2 generator, installs its policy and replays one
 * more iteration, printing one line per check.  Built and run by tests/test_c_abi_cpu.py. */
#include <stdio.h>
#include <string.h>

#include "chm.h"

#define CHECK(call)                                                          \
  do {                                                                       \
    chm_status st_ = (call);                                                 \
    if (st_ != CHM_OK) {                                                     \
      fprintf(stderr, "%s failed (%d): %s\n", #call, st_, chm_last_error()); \
      return 1;                                                              \
    }                                                                        \
  } while (0)

enum { LAYERS = 6 };

/* one iteration: per layer FWD op producing a 1 MiB activation saved for its BWD op, then the
 * BWD ops in reverse order; ids are the (simulated) storage addresses of this iteration */
static int iteration(chm_ctx *ctx, int32_t tf, int32_t tb, uint64_t base, int *n_actions) {
  chm_actions act;
  for (int l = 0; l < LAYERS; l++) {
    chm_tensor_ref in = {base + (uint64_t)(l ? l - 1 : 100) * 4096, 1 << 20, 2};
    chm_tensor_ref out = {base + (uint64_t)l * 4096, 1 << 20, 2};
    chm_op_record op;
    memset(&op, 0, sizeof op);
    op.token = tf;
    op.phase = CHM_FWD;
    op.n_in = l ? 1 : 0;
    op.in = &in;
    op.n_out = 1;
    op.out = &out;
    op.live_bytes = -1;
    CHECK(chm_record_op(ctx, &op, &act));
    *n_actions += (int)(act.n_swap_out + act.n_release + act.n_swap_in);
  }
  for (int l = LAYERS - 1; l >= 0; l--) {
    chm_tensor_ref in = {base + (uint64_t)l * 4096, 1 << 20, 2};
    uint64_t freed = in.id;
    chm_op_record op;
    memset(&op, 0, sizeof op);
    op.token = tb;
    op.phase = CHM_BWD;
    op.n_in = 1;
    op.in = &in;
    op.n_free = 1;
    op.freed = &freed;
    op.live_bytes = -1;
    CHECK(chm_record_op(ctx, &op, &act));
    *n_actions += (int)(act.n_swap_out + act.n_release + act.n_swap_in);
  }
  return 0;
}

int main(void) {
  chm_config cfg;
  chm_config_default(&cfg);
  cfg.device = -1;  /* host-only: recording, Algo. 1, trace build, generator, executor */
  chm_ctx *ctx = NULL;
  CHECK(chm_create(&cfg, &ctx));
  int32_t tf, tb;
  CHECK(chm_tokenize(ctx, "aten::linear", &tf));
  CHECK(chm_tokenize(ctx, "aten::linear_backward", &tb));
  int n_actions = 0;
  chm_stage stage = CHM_WARMUP;
  for (int it = 0; it < 4; it++) {
    if (it == 3) CHECK(chm_set_detailed(ctx, 1));
    if (iteration(ctx, tf, tb, 0x10000000ull * (uint64_t)(it + 1), &n_actions)) return 1;
    int32_t changed;
    double len_diff, cos_sim;
    CHECK(chm_detect_seq_change(ctx, 1e-3, &stage, &changed, &len_diff, &cos_sim));
    printf("iteration %d stage %d changed %d cos %.3f\n", it, (int)stage, changed, cos_sim);
  }
  CHECK(chm_set_detailed(ctx, 0));
  chm_trace_params tp;
  memset(&tp, 0, sizeof tp);
  tp.hbm_budget = 3 << 20;
  tp.static_bytes = 0;
  tp.bw_bytes_per_s = 1e9;
  tp.groups_fwd = 0; /* layer count from the token period */
  tp.groups_bwd = 0;
  tp.omega = 1.0;
  chm_trace *t = NULL;
  CHECK(chm_trace_build(ctx, &tp, &t));
  chm_trace_info info;
  CHECK(chm_trace_get_info(t, &info));
  printf("trace ops %u swappable %u layers %u peak0 %lld budget %lld\n", info.n_ops, info.n_swappable,
         info.n_layers, (long long)info.peak0, (long long)info.budget);
  chm_gen_params gp = {1.0, 1.0};
  chm_item items[64];
  uint32_t n_items = 0;
  int32_t feasible = 0;
  CHECK(chm_generate_policy(t, &gp, items, 64, &n_items, &feasible));
  printf("generator items %u feasible %d\n", n_items, feasible);
  CHECK(chm_policy_install_items(ctx, t, items, n_items));
  n_actions = 0;
  if (iteration(ctx, tf, tb, 0x90000000ull, &n_actions)) return 1;
  CHECK(chm_detect_seq_change(ctx, 1e-3, &stage, NULL, NULL, NULL));
  chm_exec_stats es;
  CHECK(chm_exec_stats_get(ctx, &es));
  printf("executed items %u matched %u actions %d\n", es.n_items, es.n_matched, n_actions);
  /* errors come back as codes with a message, never as a crash */
  chm_status bad = chm_trace_build(ctx, NULL, &t);
  printf("null params -> %d (%s)\n", bad, chm_last_error());
  /* device-only calls on this host-only ctx: a state error, no CPU fallback */
  uint64_t w[2] = {0, 0};
  chm_best k[2];
  bad = chm_descend(ctx, t, w, 1, 8, w, k, NULL, NULL, NULL);
  printf("descend on a host-only ctx -> %d\n", bad);
  chm_trace_free(t);
  chm_destroy(ctx);
  printf("ok\n");
  return 0;
}
