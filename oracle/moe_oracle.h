/*
 * moe_oracle.h -- CPU restatement of the reference's activation-sparse MoE
 * FFN layer (moe-sparsekit, /root/reference/proj).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the shipped product path
 * (paper_2605_08575_b200/, include/) may include, link or call this file;
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs use it, and there only as the checker.
 *
 * Parity status: PINNED.  tests/test_oracle_cpu.py checks this restatement
 * against (a) the reference's own golden vector and hand cases
 * (proj/tests/golden/..., router_test.cpp, activation_test.cpp,
 * linalg_test.cpp, engine_test.cpp) and (b) the unmodified reference compiled
 * into oracle/_ref/libsparsekit_ref.so (bit-for-bit on random models).
 *
 * All reductions: float accumulator, ascending index, no FMA contraction
 * (build with -ffp-contract=off; proj/CMakeLists.txt:26-27).
 *
 * Weight layout (contiguous restatement of MoELayerWeights, model.hpp:34-43):
 *   router [E][D]; gate, up, down_t each [E][N][D]; shared_* [S][D].
 */
#ifndef MOE_ORACLE_H
#define MOE_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORK_PAD_INDEX (-1)
#define ORK_TILE 64

enum { ORK_OK = 0, ORK_ESHAPE = 1, ORK_ECONFIG = 2, ORK_EINDEX = 3, ORK_EINTERNAL = 4 };

typedef struct ork_config {
  int32_t n_experts, top_k, d_model, d_ffn;
  int32_t has_shared, d_shared, renormalize, align_block;
} ork_config;

typedef struct ork_weights {
  ork_config cfg;
  const float *router;
  const float *gate, *up, *down_t;
  const float *shared_gate, *shared_up, *shared_down_t;
} ork_weights;

typedef struct ork_report {
  uint64_t gate_macs, up_macs, down_macs, other_macs;
  uint64_t active_neurons_total;
  double achieved_routed_sparsity;
  uint64_t tiles_total, tiles_skipped;
  int32_t path_used; /* 0 dense, 1 sparse */
} ork_report;

/* rng.hpp:16-61 */
uint64_t ork_splitmix_next(uint64_t *state);
void ork_fill_symmetric(float *dst, uint64_t count, uint64_t seed, uint64_t draw_offset, float scale);
void ork_fill_gaussian(float *dst, uint64_t count, uint64_t seed);
/* draw offsets of each matrix inside generate_synthetic's stream (model.cpp:129-166) */
uint64_t ork_synth_offset_router(const ork_config *c);
uint64_t ork_synth_offset_expert(const ork_config *c, int e, int which /*0 gate 1 up 2 down_t*/);
uint64_t ork_synth_offset_shared(const ork_config *c, int which);

/* round-to-nearest-even float -> bf16 -> float, in place (operand preparation) */
void ork_round_bf16(float *v, uint64_t count);

int ork_config_validate(const ork_config *c);

/* linalg.cpp */
float ork_dot(const float *a, const float *b, int n);
void ork_matvec(const float *w, int rows, int cols, const float *x, float *y);
int ork_gathered_matvec_t(const float *w_t, int rows, int cols, const int32_t *idx, const float *h,
                          int m, float *y);

/* router.cpp */
int ork_route(const float *logits, int batch, int n_experts, int top_k, int renorm, int32_t *ids,
              float *weights);
/* sorted_out needs batch*top_k + n_experts*(block-1) entries; expert_of_block the same / block */
int ork_align_dispatch(const int32_t *ids, int batch, int top_k, int n_experts, int block,
                       int32_t *sorted_out, int32_t *expert_of_block, int32_t *n_padded,
                       int32_t *n_blocks);
void ork_combine(const float *slot_outputs, const float *weights, int batch, int top_k, int d_model,
                 float *y);

/* activation.cpp */
float ork_silu(float x);
void ork_swiglu_rows(const float *gate_out, const float *up_out, int n, float *h);
int ork_n_off(double s, int n);
void ork_mask_smallest(const float *h, int n, int count, uint8_t *mask);
int ork_topk_mask(const float *h, int n, double s, uint8_t *mask);
int ork_threshold_mask(const float *gate_out, int n, float threshold, uint8_t *mask);
int ork_default_capacity(int top_k, int d_ffn);
int ork_compact_active(const uint8_t *masks, const int32_t *topk_ids, int n_slots, int d_ffn,
                       int capacity, int32_t *flat, int32_t *active_per_slot,
                       int32_t *total_active);

/* profiler.cpp:101-150; mode 0 = routed only, 1 = routed+shared. shared_masks may be NULL. */
int ork_build_topk_masks(const ork_weights *w, const float *x, int batch, double s, int mode,
                         uint8_t *routed_masks, uint8_t *shared_masks);

/* engine.cpp:94-191. routed_masks/shared_masks NULL => forward_dense.
 * Optional captures (may be NULL): ids/weights [B*K], h_routed [B*K*N] (pre-mask SwiGLU
 * output, slot-major), h_shared [B*S]. */
int ork_forward_masked(const ork_weights *w, const float *x, int batch, const uint8_t *routed_masks,
                       const uint8_t *shared_masks, float *y, ork_report *rep, int32_t *ids_out,
                       float *weights_out, float *h_routed_out, float *h_shared_out);

/* engine.cpp:229-369 */
int ork_forward_sparse(const ork_weights *w, const float *x, int batch, float threshold, float *y,
                       ork_report *rep);

/* tests/support.hpp:55-152 -- double-accumulating independent check */
int ork_scalar_forward(const ork_weights *w, const float *x, int batch, const uint8_t *routed_masks,
                       const uint8_t *shared_masks, float *y);
double ork_max_rel_diff(const float *a, const float *b, uint64_t count);

#ifdef __cplusplus
}
#endif
#endif
