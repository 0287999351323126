// skb_internal.cuh -- shared declarations of the sm_100a kernels behind include/sparsekit_b200.h.
//
// Row space used by every stage after dispatch ("rows"):
//   rows [0, B*K)        routed token-slots in expert-major order (the order
//                        align_dispatch produces, proj/src/router.cpp:80-104,
//                        without the padding entries)
//   rows [B*K, B*K + B)  the shared expert, one row per token, when has_shared
// perm[row] = flat slot t*K+s, inv[flat slot] = row.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace skb {

constexpr int kNeuronBlock = 64;   // neurons per gate/up tile (64 gate + 64 up rows = UMMA M 128)
constexpr int kBlockK = 64;        // bf16 elements per TMA/UMMA K block (one 128-byte swizzle row)
constexpr int kSelectThreads = 256;
constexpr int kMaxExperts = 1024;
constexpr int kSmallSlots = 64;    // B*K up to which the router kernel builds the dispatch itself  // 32 probabilities per lane in the warp top-k

__host__ __device__ inline int round_up(int v, int m) { return (v + m - 1) / m * m; }

// GEMM operand images are stored TILED: 128-row x 64-column tiles (one TMA box = one UMMA
// A tile), each tile 16 KB contiguous, tiles of one 128-row block consecutive along K.  A TMA
// tile load is then one contiguous HBM read instead of 128 segments of 128 B at a row-stride
// apart.  Element (r, d) of an image whose rows have Kp (multiple of 64) columns:
__host__ __device__ inline size_t tiled_index(size_t r, int d, int Kp) {
  return ((r / 128) * static_cast<size_t>(Kp / 64) + static_cast<size_t>(d / 64)) * (128 * 64) +
         (r % 128) * 64 + static_cast<size_t>(d % 64);
}
__host__ __device__ inline int ceil_div(int a, int b) { return (a + b - 1) / b; }

// Geometry of one layer's device image.
struct Geometry {
  int E, K, D, N, S;
  int has_shared, renorm;
  int Dp;  // D rounded up to kBlockK (zero padded)
  int Dp128;  // D rounded up to 128: rows per expert of the W_down^T image
  int Np;  // N rounded up to kNeuronBlock
  int Sp;  // S rounded up to kNeuronBlock (0 when no shared expert)
  int Nh;  // row stride of h / kept lists: max(Np, Sp)
};

// Per-call dispatch outputs (device pointers).
struct DispatchBuffers {
  int32_t* perm;         // [B*K]
  int32_t* inv;          // [B*K]
  int32_t* row_expert;   // [B*K + B]   expert id, E for shared rows
  int32_t* expert_off;   // [E + 1]
  int32_t* tile_expert;  // [max_tiles]
  int32_t* tile_row0;    // [max_tiles]
  int32_t* tile_nrows;   // [max_tiles]
  int32_t* n_tiles;      // [1]
  int32_t* tile_colrow;  // [max_tiles][16] token-indexed tiles (decode): h row of column c, or -1
};

// ---- launchers (one per stage; each returns the number of kernels it launched) ----
struct LaunchCtx {
  cudaStream_t stream;
  bool pdl;  // programmatic dependent launch between stages
};

// Router stage: logits (x == nullptr: `logits` already holds them), route(), and -- when
// `dispatch` is given -- the dispatch (inside the router kernel for B*K <= kSmallSlots, else by
// dispatch_kernel).  `counters` is 1 + ceil(B / 4) zero-initialised words that the kernel
// leaves zeroed.
struct RouterLaunch {
  const float* x;
  const float* router;
  int B, E, D, K, renorm;
  bool fast;
  float* logits;
  int32_t* ids;
  float* weights;
  unsigned* counters;
  const DispatchBuffers* dispatch;
  int has_shared, tile_tokens;
  // decode (B <= 16, dispatch built inside the router kernel): extra CTAs convert the tokens to
  // bf16 rows xb[B][Dp] while the chains run, and the tile list is token-indexed -- the gate/up
  // GEMM reads token rows directly, no expert-sorted copy (no permute kernel)
  __nv_bfloat16* xb;
  int Dp;
  // batches: route + dispatch + token permutation as one kernel (router.cu: route_dispatch_kernel)
  // when the expert-sorted token copy `xs` and the two grid-barrier words are given
  __nv_bfloat16* xs;
  unsigned* grid_bar;  // [0] barrier word, [1] "tile list written" flag (polled by the gate/up CTAs)
};
// true when launch_router() will also write the expert-sorted token copy (no permute kernel)
bool router_fuses_permute(const RouterLaunch& r);
// true when launch_router() will build token-indexed tiles for this call
bool router_token_tiles(int B, int K, bool want);
int launch_router(const LaunchCtx& ctx, const RouterLaunch& r);
int launch_dispatch(const LaunchCtx& ctx, const int32_t* ids, int B, int K, int E, int has_shared,
                    int tile_tokens, const DispatchBuffers& d);
int launch_permute_tokens(const LaunchCtx& ctx, const float* x, const int32_t* perm, int B, int K,
                          int D, int Dp, int has_shared, __nv_bfloat16* xs);
int launch_plan_export(const LaunchCtx& ctx, const int32_t* perm, const int32_t* expert_off, int E,
                       int block, int32_t* sorted_out, int32_t* expert_of_block, int32_t* counts2);

int launch_gateup_tc(const LaunchCtx& ctx, const CUtensorMap* tmap_w, const CUtensorMap* tmap_x,
                     const CUtensorMap* tmap_x32 /*32-row boxes*/, int tile_tokens, const DispatchBuffers& d, int max_tiles, const Geometry& g,
                     float* h, bool token_tiles, float* sg = nullptr, bool pair_blocks = false,
                     bool precise = false, bool early_tiles = false, const void* w_image = nullptr,
                     const int* tiles_flag = nullptr);
int launch_down_tc(const LaunchCtx& ctx, const CUtensorMap* tmap_wdt,
                   const CUtensorMap* tmap_wdt_shared, const CUtensorMap* tmap_hb /*[3]*/,
                   const CUtensorMap* tmap_hb32 /*[3], 32-row boxes*/, int nsplit, int tile_tokens, const DispatchBuffers& d, int max_tiles,
                   const Geometry& g, float* slot_out, bool pair_blocks = false,
                   bool precise = false, bool early_tiles = false, const void* wdt_image = nullptr,
                   const void* wdt_shared_image = nullptr, float* const* out_rows = nullptr,
                   const int32_t* out_perm = nullptr);
int launch_combine_rows(const LaunchCtx& ctx, const float* slot_out, const int32_t* inv,
                        const float* weights, int B, const Geometry& g, float* y,
                        float* const* y_rows = nullptr);
int launch_gateup_simt(const LaunchCtx& ctx, const __nv_bfloat16* wgu, const __nv_bfloat16* xs,
                       const int32_t* row_expert, int rows, const Geometry& g, float* h);

// select modes
enum { kSelectTopk = 0, kSelectAll = 1, kSelectGiven = 2, kSelectThreshold = 3 };
struct SelectArgs {
  const float* h;  // [rows][Nh]
  int rows, BK, N, S, Nh, K;
  int mode;
  int n_off_routed, n_off_shared;
  const float* sg;               // kSelectThreshold: silu(gate) [rows][Nh]; a routed neuron is kept
  float tau;                     //   iff |sg| >= tau (activation.cpp:62-72); shared rows keep all
  const int32_t* counts;         // optional per-row n_off override (stage API), else NULL
  const int32_t* slot_counts;    // optional per-slot n_off of routed rows, [K] (neuron budgets)
  const int32_t* perm;           // row -> flat slot (masks are slot-major); NULL = identity
  const uint8_t* mask_in_routed; // kSelectGiven: [B*K][N] slot-major
  const uint8_t* mask_in_shared; // kSelectGiven: [B][S] or NULL (=> keep all)
  uint8_t* mask_out_routed;      // optional [B*K][N] slot-major
  uint8_t* mask_out_shared;      // optional [B][S]
  int32_t* kept_idx;             // optional [rows][Nh]
  float* kept_val;               // optional [rows][Nh]
  int32_t* kept_cnt;             // optional [rows]
  // dense down projection: masked activations as nsplit bf16 terms, [nsplit][rows][Nh]
  __nv_bfloat16* hb;
  size_t hb_split_stride;        // rows * Nh
  int nsplit;
  int kext_routed, kext_shared;  // columns written per row (Np / Sp; pad columns are zeros)
};
int launch_select(const LaunchCtx& ctx, const SelectArgs& a);
// threshold variant, stage API (activation.cpp:62-114)
int launch_threshold_mask(cudaStream_t s, const float* g, size_t n, float tau, uint8_t* mask);
int launch_compact_active(cudaStream_t s, const uint8_t* masks, const int32_t* ids, int batch, int K,
                          int N, int capacity, int32_t* flat, int32_t* per_slot, int32_t* total);

struct DownArgs {
  const __nv_bfloat16* wd;         // [E][Np][Dp]
  const __nv_bfloat16* wd_shared;  // [Sp][Dp] or NULL
  const int32_t* row_expert;       // [rows]
  const int32_t* inv;              // [B*K] flat slot -> row
  const float* weights;            // [B*K] router weights
  int B, K, BK, has_shared;
  const float* h;  // [rows][Nh]
  int Nh, N, S;
  // selection (kSelect*), done inside the kernel
  int sel_mode, n_off_routed, n_off_shared;
  const uint8_t* mask_in_routed;  // kSelectGiven: [B*K][N] slot-major
  const uint8_t* mask_in_shared;  // kSelectGiven: [B][S] or NULL (=> keep all)
  int max_keep;                   // upper bound of survivors per row
  float* y;                       // [B][D]
};
int launch_down(const LaunchCtx& ctx, const DownArgs& a, const Geometry& g);
int launch_combine_slots(const LaunchCtx& ctx, const float* slot_outputs, const float* weights,
                         int B, int K, int D, float* y);

// Fused decode kernel (decode.cu): the whole layer for B <= 4 in one persistent launch.
struct DecodeLaunch {
  const float* x;                  // [B][D]
  const float* router;             // [E][D]
  const __nv_bfloat16* wd;         // [E][Np][Dp]
  const __nv_bfloat16* wd_shared;  // [Sp][Dp] or NULL
  int B;
  int sel_mode, n_off_r, n_off_s;  // kSelect*
  float tau;                       // kSelectThreshold
  const __nv_bfloat16* wu;         // W_up rows [E][Np][Dp] (threshold mode gathers them)
  int32_t* kcnt;                   // kSelectThreshold: survivors per flat slot [B*K]
  const uint8_t* mask_r;           // kSelectGiven: [B*K][N]
  const uint8_t* mask_s;           // kSelectGiven: [B][S] or NULL
  int CH;                          // row chunks per (token, slot): decode_chunks()
  bool capture;                    // also write h / inv / perm / row_expert in slot order
  float* p0;                       // decode_p0_words() words: tagged partial fast logits
  float* logits;                   // [B][E] exact logits
  int32_t* ids;                    // [B][K]
  float* wts;                      // [B][K]
  float* hc;                       // [16 * CM + 16][Nh] activations of the candidate rows
  float* part;                     // [B][R][CH][Dp]
  unsigned* ctr;                   // decode_counter_words() zeroed words
  float* y;                        // [B][D]
  float* h_cap;                    // capture: [B*K + B][Nh]
  int32_t* inv;
  int32_t* perm;
  int32_t* row_expert;
};
bool decode_fused_eligible(const Geometry& g, int B);
int decode_counter_words();
int decode_cand_rows(int K);
int decode_p0_words(const Geometry& g);
int decode_chunks(const Geometry& g, int B, int keep_max, int n_sms);
// tmap_w3: the gate/up image as {64 columns, 128 rows, tiles}, box {64, 32, 4}, no swizzle;
// tmap_w3g: the same view with box {64, 16, 4} (the gate rows of one tile quarter)
int launch_decode_fused(const LaunchCtx& ctx, const CUtensorMap* tmap_w3, const CUtensorMap* tmap_w3g,
                        const DecodeLaunch& d, const Geometry& g, int n_sms);

// weight image construction
int launch_pack_gateup(cudaStream_t s, const float* gate, const float* up, int n_rows, int D, int Dp,
                       __nv_bfloat16* dst_block_base);
int launch_pack_rows(cudaStream_t s, const float* src, int n_rows, int D, int Dp,
                     __nv_bfloat16* dst);
int launch_synth_gateup(cudaStream_t s, uint64_t seed, float scale, uint64_t off_gate,
                        uint64_t off_up, int n_rows, int n_rows_padded, int D, int Dp,
                        __nv_bfloat16* dst);
int launch_synth_rows_bf16(cudaStream_t s, uint64_t seed, float scale, uint64_t off, int n_rows,
                           int n_rows_padded, int D, int Dp, __nv_bfloat16* dst);
int launch_pack_down_t(cudaStream_t s, const float* down_t, int n_rows, int D, int Kp,
                       __nv_bfloat16* dst);
int launch_synth_down_t(cudaStream_t s, uint64_t seed, float scale, uint64_t off, int n_rows, int D,
                        int Kp, __nv_bfloat16* dst);
int launch_fill_f32(cudaStream_t s, float* dst, float value, size_t count);
int launch_synth_f32(cudaStream_t s, uint64_t seed, float scale, uint64_t off, uint64_t count,
                     float* dst);

// ---- device helpers ----
#if defined(__CUDACC__)

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier / bulk-copy (TMA) wrappers ----
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_LOOP:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra WAIT_DONE;\n"
      "bra WAIT_LOOP;\n"
      "WAIT_DONE:\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// 1-D bulk copy global -> shared (TMA engine, no tensor map): `bytes` and both addresses are
// multiples of 16; completion is signalled on `bar` as complete_tx(bytes).
__device__ __forceinline__ void bulk_copy_g2s(uint32_t dst_smem, const void* src, uint32_t bytes,
                                              uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst_smem),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

// Position of neuron j of a 64-neuron block inside the interleaved 128-row
// gate/up tile: 16 gate rows then 16 up rows per TMEM lane quarter, so that a
// warp's 32 TMEM lanes hold gate (lanes 0-15) and up (lanes 16-31) of the
// same 16 neurons.
__host__ __device__ inline int gateup_row(int j /*0..63*/, int is_up) {
  return 32 * (j >> 4) + 16 * is_up + (j & 15);
}

#endif  // __CUDACC__

}  // namespace skb
