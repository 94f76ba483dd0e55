/*
 * chm_oracle.h -- CPU ORACLE for the Chameleon swap hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load this library.  It shares no code, header, table or constant with the
 * product under paper_2509_11076_b200/ and include/; neither imports the other.
 *
 * It is a plain, slow, literal implementation of what PAPER.md (arxiv 2509.11076)
 * defines, with the readings of SURVEY.md §8(c) / DESIGN.md §"Readings" where the
 * paper is silent.  Every function cites the passage it follows ("P:<line>").
 *
 * Parity status: every function below is pinned by tests/test_oracle_*.py
 * (worked example W1, SPEC examples, brute force against a closed form, invariants)
 * EXCEPT the fidelity of the stall model to real stalls ("parity unpinned": the paper
 * gives no formula or number for it, DESIGN.md §"Unpinned").
 */
#ifndef CHM_ORACLE_H
#define CHM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One profiled iteration (Detailed mode) with tensors already identified by
 * the generator's index (the oracle does not need fuzzy matching to know them). */
typedef struct {
  int32_t n_ops, n_tensors;
  const uint8_t *phase;               /* [n_ops] 0 FWD, 1 BWD, 2 OPT                      */
  const int32_t *in_ptr, *in_idx;     /* CSR: tensors read by op i                        */
  const int32_t *out_ptr, *out_idx;   /* CSR: tensors allocated (produced) by op i        */
  const int32_t *free_ptr, *free_idx; /* CSR: refcount releases right after op i */
  const int64_t *nbytes;              /* [n_tensors] block bytes                          */
  int64_t static_bytes;               /* M_0, bytes live when the iteration starts        */
  double t_iter, bw, omega;           /* T_iter (Eq. 1), B (Eq. 3), overlap factor        */
  int32_t groups_fwd, groups_bwd;     /* logical-layer counts                 */
} orc_input;

typedef struct orc_model orc_model;

/* returns 0, or a negative code with a message in orc_error() */
int orc_build(const orc_input *in, orc_model **out);
void orc_free(orc_model *m);
const char *orc_error(void);

void orc_dims(const orc_model *m, int32_t *n_ops, int32_t *n_tensors, int32_t *n_swappable,
              int32_t *n_layers);
/* per tensor: producer p (-1 static), free op f (N if it survives), last FWD use a, first BWD
 * input use b (-1 if none) */
void orc_tensor_table(const orc_model *m, int32_t *p, int32_t *f, int32_t *a, int32_t *b);
void orc_layer_table(const orc_model *m, int32_t *start, int32_t *count, int32_t *type,
                     double *bud);
/* swappable set in mask-bit order: tensor, solo release op r, solo swap-in op s, lin, lout,
 * saturated flag */
void orc_swappable(const orc_model *m, int32_t *t, int32_t *r, int32_t *s, int32_t *lin,
                   int32_t *lout, int32_t *saturated);
void orc_f0(const orc_model *m, int64_t *f0);
void orc_base_mask(const orc_model *m, uint64_t *words);

/* Event-by-event replay of an explicit item list {t, r, s}.
 * footprint may be NULL.  Returns peak. */
int64_t orc_replay(const orc_model *m, int32_t n_items, const int32_t *t, const int32_t *r,
                   const int32_t *s, int64_t *footprint, int64_t *d2h, int64_t *h2d);
double orc_stall(const orc_model *m, int32_t n_items, const int32_t *t, const int32_t *r,
                 const int32_t *s);
/* Stall-model variants of reading Q11, same items:
 *  orc_stall_dir: per-direction budgets -- each layer's swap-out and swap-in loads are charged
 *    against Bud_l separately (a full-duplex link): pairwise sum over l of
 *    max(0, out_l/B - Bud_l) + max(0, in_l/B - Bud_l), out_l at lay(r), in_l at lay(s).
 *  orc_stall_timeline: max-plus serial-stream timeline -- ops take T_iter/N each; a swap-out
 *    enters the D2H FIFO after op a_t, a swap-in the H2D FIFO before op s_t (not before its
 *    swap-out ended); compute waits for the swap-out after op r_t (release) and for the swap-in
 *    before op b_t.  Returns the total wait, events handled in op order (after op i: swap-outs,
 *    releases; before op i+1: swap-ins, waits; item order within a kind). */
double orc_stall_dir(const orc_model *m, int32_t n_items, const int32_t *t, const int32_t *r,
                     const int32_t *s);
double orc_stall_timeline(const orc_model *m, int32_t n_items, const int32_t *t, const int32_t *r,
                          const int32_t *s);

/* Fig. 3 reconstruction: measured[i] + bytes that are off device at op i */
void orc_reconstruct(int32_t n_ops, const int64_t *measured, int32_t n_items,
                     const int64_t *size, const int32_t *r, const int32_t *s, int64_t *actual);

enum { ORC_EXHAUSTIVE = 0, ORC_SEEDED = 1, ORC_MASKS = 2 };
typedef struct {
  int64_t excess;
  double stall;
  int64_t swapped;
  uint64_t index;
  int64_t peak;
} orc_best;

/* Evaluate candidates [first, first+count) of the given kind.  words: SEEDED base mask
 * (W words, NULL -> default base) or MASKS [count][W].  Outputs may be NULL.
 * footprint: [count][N] or NULL.  nthreads >= 1. */
int orc_eval(const orc_model *m, int kind, uint64_t first, uint64_t count, uint64_t seed,
             uint64_t flip_thr, const uint64_t *words, int64_t budget, int nthreads,
             int64_t *peak, double *stall, int64_t *swapped, int64_t *footprint, orc_best *best);
int orc_eval_model(const orc_model *m, int kind, uint64_t first, uint64_t count, uint64_t seed,
                   uint64_t flip_thr, const uint64_t *words, int64_t budget, int nthreads, int stall_model,
                   int64_t *peak, double *stall, int64_t *swapped, int64_t *footprint, orc_best *best);
uint64_t orc_splitmix64(uint64_t z);
int orc_key_less(const orc_best *x, const orc_best *y);

/* Algo. 2 policy generation with the simulator of P:315-340; readings R-gen in
 * DESIGN.md.  Items are (tensor, release op r, swap-in op s) sorted by (a_t, t).  Returns the
 * number of items, or -1 if the MRL cannot be cleared ("Raise Error") -- the items chosen
 * so far are still written.  fallback[k] = 1 if item k was placed by the highest-score fallback
 * (P:333), saturated[k] = 1 if its swap-out found no layer with enough remaining time.
 * rem_scale scales the layers' initial T_remaining (1 = Eq. 1 budgets x omega). */
int32_t orc_generate(const orc_model *m, int64_t budget, double C, double rem_scale, int32_t cap,
                     int32_t *t, int32_t *r, int32_t *s, int32_t *fallback, int32_t *saturated);
/* Evaluate explicit item lists: candidate c = items [off[c], off[c+1]); outputs nullable */
int orc_eval_explicit(const orc_model *m, int32_t count, const int64_t *off, const int32_t *t,
                      const int32_t *r, const int32_t *s, int64_t budget, uint64_t first_index,
                      int64_t *peak, double *stall, int64_t *swapped, int64_t *footprint,
                      orc_best *best);

/* Swap execution oracle: after a swap the destination range equals the
 * source range byte for byte.  Executed literally on host buffers (memcpy per descriptor). */
void orc_swap_execute(int32_t n, void *const *dst, const void *const *src, const uint64_t *nbytes);

/* Algo. 1 */
typedef struct {
  int32_t m, n, cos_mode, initialized, stable_step, prev_stage;
  double len_tol, cos_tol;
  int32_t prev_len, cap;
  int32_t *prev_seq;
} orc_stage_state;
void orc_stage_init(orc_stage_state *st, int32_t m, int32_t n, double len_tol, double cos_tol,
                    int32_t cos_mode);
void orc_stage_release(orc_stage_state *st);
/* returns the stage; *stable = the Algo. 1 condition */
int32_t orc_stage_step(orc_stage_state *st, const int32_t *seq, int32_t len, double *len_diff,
                       double *cos_sim, int32_t *stable);
int orc_compare(const int32_t *a, int32_t na, const int32_t *b, int32_t nb, int32_t cos_mode,
                double *len_diff, double *cos_sim);

/* App. A features: ranks from token frequencies, then per-tensor updates */
void orc_feature_tables(const int32_t *tokens, int32_t n, int32_t max_token, uint8_t *op_index,
                        uint32_t *op_onehot);
/* feature of every tensor right after op `after` (uses of ops 0..after) */
void orc_features_after(const int32_t *tokens, int32_t n_ops, const int32_t *use_ptr,
                        const int32_t *use_idx, int32_t n_tensors, const uint8_t *op_index,
                        const uint32_t *op_onehot, int32_t after, uint32_t *count, uint32_t *tag,
                        uint64_t *stack);

#ifdef __cplusplus
}
#endif
#endif
