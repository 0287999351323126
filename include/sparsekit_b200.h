/*
 * sparsekit_b200.h -- C ABI of the B200-native activation-sparse MoE FFN layer.
 *
 * Drop-in boundary for the hot path of the reference `sparsekit` library
 * (/root/reference/proj): the reference exposes this path as C++ free
 * functions over value types and has no FFI of its own, so each entry point
 * below names the reference interface it stands in for (file:line).  The C++
 * facade in sparsekit_b200.hpp re-creates those reference signatures on top
 * of this ABI; INTEGRATION.md shows the binding a maintainer adds.
 *
 * Conventions
 *   - plain pointers and sizes only; no C++ or torch types.
 *   - every function returns an skb_status; skb_last_error() gives the
 *     thread-local message.  Codes map 1:1 onto the reference exception types
 *     (proj/include/sparsekit/errors.hpp:12-43).
 *   - "host" pointers are ordinary (pageable or pinned) CPU memory borrowed
 *     for the duration of the call.  "device" pointers are CUDA device memory
 *     on the layer's device.
 *   - there is no CPU fallback: without a CUDA device every compute entry
 *     point fails with SKB_ECUDA.
 *
 * Numeric contract: expert weights are rounded once to
 * bf16 at layer creation, tokens are rounded to bf16 for the gate/up
 * contraction, all accumulation is fp32, h = silu(g)*u stays fp32.  The
 * router keeps fp32 weights and fp32 tokens and, unless
 * SKB_FLAG_FAST_ROUTER is set, reproduces the reference's ascending-index
 * float accumulation bit for bit, so expert ids equal the reference's.
 */
#ifndef SPARSEKIT_B200_H
#define SPARSEKIT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SKB_ABI_VERSION 3

typedef enum skb_status {
  SKB_OK = 0,
  SKB_ESHAPE = 1,    /* sparsekit::ShapeError    */
  SKB_ECONFIG = 2,   /* sparsekit::ConfigError   */
  SKB_EINDEX = 3,    /* sparsekit::IndexError    */
  SKB_EINTERNAL = 4, /* sparsekit::InternalError */
  SKB_ECUDA = 5,     /* no reference analogue: CUDA runtime/driver failure */
  SKB_EFORMAT = 6,   /* sparsekit::FormatError; byte offset in skb_last_error_offset() */
  SKB_EIO = 7        /* sparsekit::IoError       */
} skb_status;

/* MoEConfig, proj/include/sparsekit/model.hpp:15-29, as fixed-width ints. */
typedef struct skb_config {
  int32_t n_experts;   /* E */
  int32_t top_k;       /* K */
  int32_t d_model;     /* D */
  int32_t d_ffn;       /* N */
  int32_t has_shared;  /* bool */
  int32_t d_shared;    /* S, 0 when absent */
  int32_t renormalize; /* bool */
  int32_t align_block; /* dispatch padding granularity (plan export only) */
} skb_config;

/* ForwardReport minus the output matrix, proj/include/sparsekit/engine.hpp:19-27,
 * with MacCounter (linalg.hpp:51-70) flattened in. */
typedef struct skb_report {
  uint64_t gate_macs, up_macs, down_macs, other_macs;
  uint64_t active_neurons_total;
  double achieved_routed_sparsity;
  uint64_t tiles_total, tiles_skipped;
  int32_t path_used; /* ExecPath: 0 dense, 1 sparse */
  int32_t reserved;
} skb_report;

/* Execution modes of skb_layer_forward*. */
enum {
  SKB_MODE_DENSE = 0,  /* forward_dense,        engine.hpp:38-39  */
  SKB_MODE_TOPK = 1,   /* forward_masked_dense(build_topk_masks(s)) fused; skips masked W_down rows */
  SKB_MODE_MASKED = 2, /* forward_masked_dense with caller masks, engine.hpp:43-44 */
  SKB_MODE_ROUTE_ONLY = 3, /* route_logits + route only (engine.cpp:121-122): x -> ids_out, weights_out;
                              the home-rank half of expert parallelism */
  SKB_MODE_THRESHOLD = 4   /* forward_sparse, engine.hpp:46-51 / engine.cpp:229-369: a routed neuron
                              is kept iff |silu(gate)| >= tau (threshold_mask, activation.cpp:62-72);
                              the shared expert stays dense; ForwardReport carries the 64-neuron tile
                              accounting of the reference (engine.cpp:341-348) */
};

/* Flags. */
#define SKB_FLAG_FAST_ROUTER 0x1u  /* warp-parallel router dot products (not order-faithful) */
#define SKB_FLAG_SIMT_GATEUP 0x2u  /* verification only: CUDA-core gate/up instead of tcgen05 */
#define SKB_FLAG_TIME_STAGES 0x4u  /* record CUDA events around every stage; disables PDL */
#define SKB_FLAG_NO_PDL 0x8u       /* disable programmatic dependent launch between stages */
#define SKB_FLAG_GATHER_DOWN 0x10u /* force the row-gather down projection (decode path) */
#define SKB_FLAG_DENSE_DOWN 0x20u  /* force the dense masked tcgen05 down projection (batch path) */
#define SKB_FLAG_BF16_H 0x40u      /* dense down projection: h rounded to bf16 (1e-2 mode) instead
                                      of the exact three-term bf16 split (1e-5 mode) */

#define SKB_FLAG_NO_FUSED_DECODE 0x80u /* batches <= 16: use the staged kernels instead of the
                                          single persistent decode kernel */

#define SKB_FLAG_FUSED_DECODE 0x100u   /* batches <= 16: take the persistent decode kernel even where
                                          the cost model prefers the staged kernels */

#define SKB_FLAG_NO_PAIRED_BLOCKS 0x200u /* batch GEMMs: one 128-row weight block per CTA instead of
                                           two sharing each token tile (A/B measurements) */

#define SKB_FLAG_PAIRED_BLOCKS 0x400u    /* batch GEMMs: pair weight blocks whenever the token tile is
                                           >= 64 rows, whatever the grid-size heuristic says (tests) */

#define SKB_N_STAGES 6 /* router, dispatch, gateup, select, down, combine */

typedef struct skb_forward_args {
  int32_t batch; /* B >= 1 */
  int32_t mode;  /* SKB_MODE_* */
  uint32_t flags;
  int32_t reserved;
  double s_routed; /* SparsityLevel for routed experts, [0,1] (TOPK mode) */
  double s_shared; /* SparsityLevel for the shared expert, [0,1] (TOPK mode) */
  const float* x;  /* [B][D] tokens */
  float* y;        /* [B][D] outputs */
  /* MASKED mode inputs (MaskSet, engine.hpp:31-34); shared may be NULL/0 => dense shared expert */
  const uint8_t* routed_mask_in;
  uint64_t routed_mask_len; /* must be B*K*N */
  const uint8_t* shared_mask_in;
  uint64_t shared_mask_len; /* 0 or B*S */
  /* Optional captures (NULL to skip).  Host pointers for skb_layer_forward,
   * ignored by skb_layer_forward_device. */
  int32_t* ids_out;         /* [B][K]  RouteResult::ids,     router.hpp:20-32 */
  float* weights_out;       /* [B][K]  RouteResult::weights */
  uint8_t* routed_mask_out; /* [B][K][N] slot-major, 1 = kept (MaskSet::routed) */
  uint8_t* shared_mask_out; /* [B][S] */
  float* h_routed_out;      /* [B][K][N] pre-mask SwiGLU output */
  float* h_shared_out;      /* [B][S] */
  /* External routing (expert parallelism: the owner rank computes slots routed elsewhere).
   * When ids_in is non-NULL the router stage is skipped: ids_in [B][K] are expert ids of THIS
   * layer, weights_in [B][K] the combine weights (NULL = 1.0, i.e. un-weighted slot outputs
   * for K = 1).  Host pointers for skb_layer_forward, device pointers for
   * skb_layer_forward_device (which then also honours ids_out / weights_out as device
   * pointers in SKB_MODE_ROUTE_ONLY). */
  const int32_t* ids_in;
  const float* weights_in;
  float tau;        /* SKB_MODE_THRESHOLD: the activation threshold, >= 0 (NaN is rejected) */
  int32_t reserved2;
  /* SKB_MODE_TOPK with neuron budgets (budget.hpp:31-44 + the analysis mode of the reference CLI,
   * tools/main.cpp:271-345): slot_n_off [K] (host pointer) gives, per routing slot, how many of
   * the smallest-|h| neurons are dropped (d_ffn - keep_count of apply_budget) in place of
   * n_off(s_routed).  Slots are in descending router weight, so slot s IS rank s of
   * group_experts.  NULL = plain top-k.  skb_layer_forward only. */
  const int32_t* slot_n_off;
} skb_forward_args;

typedef struct skb_layer skb_layer;

const char* skb_last_error(void);
int skb_abi_version(void);
/* Number of CUDA devices visible (0 when none); never fails. */
int skb_device_count(void);

/* MoEConfig::validate, proj/src/model.cpp:113-127 (same order, same messages). */
int skb_config_validate(const skb_config* cfg);

/* Builds the device weight image from a MoELayerWeights (model.hpp:34-43):
 * router [E][D]; gate/up/down_t[e] each [N][D] row-major fp32 (down stored
 * transposed exactly as the reference does); shared_* [S][D] or NULL. */
int skb_layer_create(const skb_config* cfg, const float* router, const float* const* gate,
                     const float* const* up, const float* const* down_t,
                     const float* shared_gate, const float* shared_up,
                     const float* shared_down_t, int device, skb_layer** out);

/* generate_synthetic(cfg, seed, scale), proj/src/model.cpp:129-166, evaluated
 * on the device with SplitMix64 jump-ahead: the image is bit-identical to
 * uploading the reference's matrices, without materialising them on the host. */
int skb_layer_create_synthetic(const skb_config* cfg, uint64_t seed, float scale, int device,
                               skb_layer** out);

/* Expert-parallel slices of generate_synthetic(full, seed, scale), built on the device with
 * the same SplitMix64 jump-ahead (bit-identical to slicing the full model):
 *   which = 0: experts [e_lo, e_hi) of the full model as a layer with
 *              {n_experts = e_hi - e_lo, top_k = 1, no shared expert};
 *   which = 1: the shared expert as a layer with {n_experts = 1, top_k = 1, d_ffn = d_shared}.
 * Either slice also carries the FULL router (E x D, top_k of the full model) for
 * SKB_MODE_ROUTE_ONLY. */
int skb_layer_create_synthetic_slice(const skb_config* full, uint64_t seed, float scale, int e_lo,
                                     int e_hi, int which, int device, skb_layer** out);

/* Attaches a router for SKB_MODE_ROUTE_ONLY that differs from the layer's own (expert-parallel
 * slices built with skb_layer_create from real weights): router is host fp32 [n_experts][D]. */
int skb_layer_set_router(skb_layer* layer, const float* router, int n_experts, int top_k,
                         int renormalize);

void skb_layer_destroy(skb_layer* layer);

/* Pre-sizes every workspace for batches up to max_batch (so that
 * skb_layer_forward_device never allocates and can be stream-captured). */
int skb_layer_reserve(skb_layer* layer, int max_batch);

/* The layer forward with HOST buffers: copies x in, runs the stages, copies
 * y (and any requested captures) out, synchronises.  Replaces
 * forward_dense / forward_masked_dense (proj/src/engine.cpp:94-191, 219-227)
 * and, in TOPK mode, build_topk_masks + forward_masked_dense
 * (proj/src/profiler.cpp:101-150). */
int skb_layer_forward(skb_layer* layer, const skb_forward_args* args, skb_report* report);

/* Same stages with DEVICE x/y, enqueued asynchronously on `stream`
 * (a cudaStream_t passed as void*; NULL = the layer's own stream -- pass
 * cudaStreamLegacy / cudaStreamPerThread to name a default stream).  No
 * allocation, no synchronisation: safe inside CUDA-graph capture after
 * skb_layer_reserve.  Capture pointers in args are ignored. */
int skb_layer_forward_device(skb_layer* layer, const skb_forward_args* args, void* stream,
                             skb_report* report);
/* The same with one destination per output row: row t of the result goes to y_rows[t] (device
 * array of device pointers, each d_model floats; args->y is ignored).  Expert parallelism passes
 * rows of the home ranks' peer-mapped buffers (skb_ep_back_ptrs), so that the layer's last kernel
 * writes its outputs where they are combined -- no copy pass.  Dense and top-k modes. */
int skb_layer_forward_device_rows(skb_layer* layer, const skb_forward_args* args, void* stream,
                                  float* const* y_rows);

/* Per-stage milliseconds of the last forward call (host or device entry) that
 * carried SKB_FLAG_TIME_STAGES; waits for that forward to finish.  ms must
 * hold SKB_N_STAGES floats. */
int skb_layer_stage_times(skb_layer* layer, float* ms);

/* Kernel launches issued by the last forward call on this layer. */
int skb_layer_last_launches(skb_layer* layer);

/* Device bytes held by the weight image. */
uint64_t skb_layer_weight_bytes(skb_layer* layer);

/* ---- stage entry points (host buffers in and out; used by the parity tests) ---- */

/* route(), proj/src/router.cpp:13-68: softmax + top-k, ties to the lower id. */
int skb_route(const float* logits, int batch, int n_experts, int top_k, int renormalize,
              int32_t* ids, float* weights);

/* align_dispatch(), proj/src/router.cpp:70-107.  sorted_out needs
 * batch*top_k + n_experts*(block-1) entries, expert_of_block the same / block. */
int skb_align_dispatch(const int32_t* ids, int batch, int top_k, int n_experts, int block,
                       int32_t* sorted_out, int32_t* expert_of_block, int32_t* n_padded,
                       int32_t* n_blocks);

/* combine(), proj/src/router.cpp:109-132. */
int skb_combine(const float* slot_outputs, const float* weights, int batch, int top_k,
                int d_model, float* y);

/* mask_smallest_magnitudes(), proj/src/activation.cpp:31-52, row-wise:
 * h is [rows][n]; counts is per-row (length rows) -- apply_budget's per-slot
 * budgets (proj/src/budget.cpp:78-85) are the same call.  kept_idx (optional)
 * is [rows][n] ascending survivors padded with -1; kept_count (optional) [rows]. */
int skb_mask_smallest(const float* h, int rows, int n, const int32_t* counts, uint8_t* mask,
                      int32_t* kept_idx, int32_t* kept_count);

/* topk_mask(), proj/src/activation.cpp:54-60: count = floor(s*n + 0.5) in double. */
int skb_topk_mask(const float* h, int rows, int n, double s, uint8_t* mask);

/* round-half-up count used by topk_mask (host arithmetic, no device needed). */
int skb_n_off(double s, int n, int32_t* out);

/* The threshold variant's stage functions (proj/include/sparsekit/activation.hpp:41-60).
 * skb_threshold_mask: threshold_mask (proj/src/activation.cpp:62-72) over rows*n gate
 *   pre-activations: keep iff |silu(g)| >= tau; tau < 0 or NaN -> SKB_ECONFIG.
 * skb_default_capacity: default_capacity (activation.cpp:74-77): top_k*d_ffn rounded up to 32.
 * skb_compact_active: compact_active (activation.cpp:79-114), one ActiveIndexRow per token:
 *   masks [batch][top_k][d_ffn] (masks_len bytes; a mismatch is SKB_ESHAPE as in the reference),
 *   topk_ids [batch][top_k] -> flat [batch][capacity] of expert*d_ffn+neuron in (slot ascending,
 *   neuron ascending) order padded with -1, active_per_slot [batch][top_k] (clamped where the
 *   list is full), total_active [batch].  capacity < 0 -> SKB_ECONFIG. */
int skb_threshold_mask(const float* gate_raw, int rows, int n, float tau, uint8_t* mask);
int skb_default_capacity(int top_k, int d_ffn);
int skb_compact_active(const uint8_t* masks, uint64_t masks_len, const int32_t* topk_ids, int batch,
                       int top_k, int d_ffn, int capacity, int32_t* flat, int32_t* active_per_slot,
                       int32_t* total_active);

/* The "MOE1" weight file (save_weights / load_weights / weight_file_size,
 * proj/src/model.cpp:180-282): magic "MOE1", six little-endian u32 (n_experts, top_k, d_model,
 * d_ffn, d_shared, flags: bit 0 has_shared, bit 1 renormalize), then fp32 little-endian
 * matrices: router, per expert gate / up / down_t, then the shared expert's three.
 * skb_layer_load maps the file and builds the device image straight from it (no host copy of
 * the fp32 weights); header checks, their order, messages and byte offsets follow load_weights.
 * Errors: SKB_EIO (cannot open), SKB_EFORMAT (+ skb_last_error_offset()).  align_block = 64. */
int skb_layer_load(const char* path, int device, skb_config* cfg_out, skb_layer** out);
int skb_save_weights(const skb_config* cfg, const float* router, const float* const* gate,
                     const float* const* up, const float* const* down_t, const float* shared_gate,
                     const float* shared_up, const float* shared_down_t, const char* path);
uint64_t skb_weight_file_size(const skb_config* cfg);
/* Byte offset carried by the last SKB_EFORMAT on this thread (FormatError::offset). */
uint64_t skb_last_error_offset(void);

/* generate_tokens(), proj/src/model.cpp:168-178 over SplitMix64::next_gaussian
 * (proj/include/sparsekit/rng.hpp:42-55): batch*d_model standard normals, Box-Muller in double
 * (pairs: cos value first, the sin value on the next draw), cast to float.  Host arithmetic with
 * the host's libm, no device needed; used by profile_tipping for its probe batches. */
int skb_generate_tokens(int32_t batch, int32_t d_model, uint64_t seed, float* out);

/* ---- expert-parallel data plane (device pointers, one process per GPU) --------------------
 * The reference is single-process; these are the device halves of the exchange
 * that shards its experts over ranks (proj/src/engine.cpp:132-165: experts are independent
 * given their routed tokens; proj/src/router.cpp:119-130: the combine is a per-token sum over
 * slots).  paper_2605_08575_b200/ep.py drives them around two NCCL all-to-all-v calls.
 *
 * skb_ep_plan: from the all-gathered routing ids_all [world][slots_per_rank] (flat slot
 *   t*top_k+s per rank; ids < 0 pad a short batch) and the expert range starts expert_lo
 *   [world+1]: counts [world][world] (slots src sends to dst), and for THIS rank's slots their
 *   position in its send buffer (grouped by destination, ascending flat slot inside a group;
 *   -1 for padding) and the expert id local to the destination.
 * skb_ep_pack: token rows as bf16 into the packed send buffer, row stride skb_ep_row_stride():
 *   [d_model bf16][int32 local expert id][pad to 16 bytes].
 * skb_ep_unpack: received packed rows -> fp32 rows + ids (inputs of skb_layer_forward_device
 *   with external routing).
 * skb_ep_combine: y[t] = sum_s weights[t][s] * back[pos[t*top_k+s]] (+ shared[t]), slots
 *   ascending, multiply and add rounded separately (router.cpp:119-130, engine.cpp:168-173). */
int skb_ep_row_stride(int d_model);
int skb_ep_plan(const int32_t* ids_all, int world, int slots_per_rank, const int32_t* expert_lo,
                int rank, int32_t* counts, int32_t* pos, int32_t* local_ids, void* stream);
int skb_ep_pack(const float* x, const int32_t* pos, const int32_t* local_ids, int slots, int top_k,
                int d_model, uint8_t* send, void* stream);
int skb_ep_unpack(const uint8_t* recv, int rows, int d_model, float* x, int32_t* ids, void* stream);
int skb_ep_combine(const float* back, const int32_t* pos, const float* weights, const float* shared,
                   int batch, int top_k, int d_model, float* y, void* stream);

/* Combine without the second collective (combine direction): buffers that
 * peers map through CUDA IPC (skb_ep_symm_alloc / _ipc_export / _ipc_import); the expert rank
 * pushes its un-weighted row outputs into every home rank's `back` buffer at the positions that
 * rank's plan expects and bumps a cumulative counter there (skb_ep_push_back; `expect` is this
 * rank's own running total per expert rank, advanced by the same call from its counts row); the
 * home rank's combine waits on its counters instead of on an all-to-all (skb_ep_combine_symm).
 * With world == 1 the "peer" is the rank itself: the same kernels, checked against skb_ep_combine. */
int skb_ep_symm_alloc(uint64_t bytes, void** ptr);
int skb_ep_symm_free(void* ptr);
int skb_ep_ipc_export(void* ptr, uint8_t* handle64);
int skb_ep_ipc_import(const uint8_t* handle64, void** peer_ptr);
int skb_ep_ipc_close(void* peer_ptr);
int skb_ep_push_back(const float* out_rows, int rows, int d_model, const int32_t* counts, int world,
                     int rank, float* const* peer_back, unsigned long long* const* peer_flag,
                     unsigned long long* expect, uint32_t* done_ctr, void* stream);
/* The dispatch direction the same way (no first all-to-all either): the home rank packs its token
 * rows straight into the owner ranks' receive buffers (peer-mapped, `skb_ep_row_stride` bytes per
 * row) at the rows the owners' view of the plan expects, and bumps cumulative counters there
 * (skb_ep_push_rows); the owner's unpack waits on its counters (skb_ep_unpack_symm; `expect` is
 * the owner's own running total per source rank, advanced by the call). */
int skb_ep_push_rows(const float* x, const int32_t* pos, const int32_t* local_ids, int slots, int top_k,
                     int d_model, const int32_t* counts, int world, int rank, uint8_t* const* peer_recv,
                     unsigned long long* const* peer_flag, uint32_t* done_ctr, void* stream);
int skb_ep_unpack_symm(const uint8_t* recv, const unsigned long long* flag, unsigned long long* expect,
                       const int32_t* counts, int world, int rank, int rows, int d_model, float* x,
                       int32_t* ids, void* stream);
/* Outputs pushed by the expert layer itself: skb_ep_back_ptrs fills ptrs[r] with the address of
 * received row r's output in its home rank's `back` buffer (pass them to
 * skb_layer_forward_device_rows); skb_ep_signal_back, enqueued after the layer, fences at system
 * scope and bumps the home ranks' counters (it also advances `expect`, like skb_ep_push_back). */
int skb_ep_back_ptrs(const int32_t* counts, int world, int rank, int rows, int d_model,
                     float* const* peer_back, float** ptrs, void* stream);
int skb_ep_signal_back(const int32_t* counts, int world, int rank,
                       unsigned long long* const* peer_flag, unsigned long long* expect, void* stream);
int skb_ep_combine_symm(const float* back, const unsigned long long* flag,
                        const unsigned long long* expect, int world, const int32_t* pos,
                        const float* weights, const float* shared, int batch, int top_k, int d_model,
                        float* y, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPARSEKIT_B200_H */
