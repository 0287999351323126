// api.cu -- the C ABI of include/sparsekit_b200.h: host-side validation (same order and
// messages as the reference), device weight image, workspaces, stage sequencing.
#include <cstdarg>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>
#include <cstdio>
#include <cstring>
#include <cmath>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include <cudaTypedefs.h>

#include "../../include/sparsekit_b200.h"
#include "skb_internal.cuh"

using namespace skb;

namespace {

thread_local std::string g_err;
thread_local uint64_t g_err_offset = 0;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define SKB_CUDA(expr)                                                                       \
  do {                                                                                       \
    cudaError_t _e = (expr);                                                                 \
    if (_e != cudaSuccess)                                                                   \
      return fail(SKB_ECUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, \
                  __LINE__);                                                                 \
  } while (0)

PFN_cuTensorMapEncodeTiled g_encode = nullptr;

int load_encode() {
  if (g_encode) return SKB_OK;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  SKB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (q != cudaDriverEntryPointSuccess || fn == nullptr)
    return fail(SKB_ECUDA, "cuTensorMapEncodeTiled not available from the driver");
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
  return SKB_OK;
}

// 2D bf16 tensor [rows][cols] row-major, box = {kBlockK cols, box_rows}, 128-byte swizzle.
int encode_bf16_2d(CUtensorMap* map, void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  int rc = load_encode();
  if (rc) return rc;
  cuuint64_t gdim[2] = {cols, rows};
  cuuint64_t gstride[1] = {cols * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(kBlockK), box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, gdim, gstride, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SKB_ECUDA, "cuTensorMapEncodeTiled failed with CUresult %d", (int)r);
  return SKB_OK;
}

// 3-D view for the fused decode kernel: {64 bf16 columns, rows, planes}, row and plane strides in
// bytes, box = {64, box_rows, box_planes}; 128-byte swizzle, or none (plain 128-byte rows for
// consumers that read the stage with ordinary shared-memory loads).
int encode_bf16_3d(CUtensorMap* map, void* base, uint64_t rows, uint64_t planes, uint64_t row_stride,
                   uint64_t plane_stride, uint32_t box_rows, uint32_t box_planes, bool swizzle = true) {
  int rc = load_encode();
  if (rc) return rc;
  cuuint64_t gdim[3] = {static_cast<cuuint64_t>(kBlockK), rows, planes};
  cuuint64_t gstride[2] = {row_stride, plane_stride};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(kBlockK), box_rows, box_planes};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, gdim, gstride, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SKB_ECUDA, "cuTensorMapEncodeTiled (3-D) failed with CUresult %d", (int)r);
  return SKB_OK;
}

int n_off_of(double s, int n) {
  // topk_mask, proj/src/activation.cpp:54-60
  const long raw = static_cast<long>(std::floor(s * n + 0.5));
  long c = raw < 0 ? 0 : raw;
  if (c > n) c = n;
  return static_cast<int>(c);
}

const int kTileCases[5] = {16, 32, 64, 128, 256};


}  // namespace

struct skb_layer {
  skb_config cfg{};
  Geometry g{};
  int device = 0;
  cudaStream_t stream = nullptr;
  int l2_bytes = 0;
  std::mutex mu;

  // router used by the router stage: the layer's own, or the full model's for EP slices
  int route_E = 0, route_K = 0, route_renorm = 1;
  // weight image
  float* d_router = nullptr;
  __nv_bfloat16* d_wgu = nullptr;
  __nv_bfloat16* d_wd = nullptr;
  __nv_bfloat16* d_wu = nullptr;          // W_up rows [E][Np][Dp], row-major like W_down: the
                                          // threshold mode of the fused decode kernel gathers them
  __nv_bfloat16* d_wd_shared = nullptr;
  __nv_bfloat16* d_wdt = nullptr;         // W_down^T image [E][Dp128][Np] (dense down projection)
  __nv_bfloat16* d_wdt_shared = nullptr;  // [Dp128][Sp]
  uint64_t weight_bytes = 0;
  CUtensorMap tmap_w{};
  CUtensorMap tmap_w3{};  // fused decode kernel: quarter-tile pieces of the same image
  CUtensorMap tmap_w3g{};  // ... and the 16 gate rows of a quarter (threshold mode)
  CUtensorMap tmap_wdt{}, tmap_wdt_shared{};

  // workspaces, sized for cap_batch
  int cap_batch = 0;
  float* d_x = nullptr;
  float* d_y = nullptr;
  float* d_logits = nullptr;
  int32_t* d_ids = nullptr;
  float* d_wts = nullptr;
  DispatchBuffers disp{};
  unsigned* d_counters = nullptr;
  int32_t* d_ids_stage = nullptr;  // host-API staging of external routing
  float* d_wts_stage = nullptr;
  __nv_bfloat16* d_xs = nullptr;
  uint64_t xs_rows = 0;
  CUtensorMap tmap_x[5]{};
  __nv_bfloat16* d_xb = nullptr;  // decode: bf16 token rows [max(cap,16)][Dp] (token-indexed tiles)
  CUtensorMap tmap_xb{};
  float* d_h = nullptr;
  float* d_sg = nullptr;  // silu(gate) of every row (threshold selection, forward_sparse)
  __nv_bfloat16* d_hb = nullptr;  // masked activations, [3][rows][Nh] bf16 terms
  CUtensorMap tmap_hb[5][3]{};
  float* d_slot_out = nullptr;    // [rows][Dp]
  int32_t* d_kidx = nullptr;
  float* d_kval = nullptr;
  int32_t* d_kcnt = nullptr;
  int32_t* d_slot_noff = nullptr;  // [K] per-slot drop counts (neuron budgets)
  uint8_t* d_mask_in_r = nullptr;
  uint8_t* d_mask_in_s = nullptr;
  uint8_t* d_mask_out_r = nullptr;
  uint8_t* d_mask_out_s = nullptr;

  // fused decode kernel (decode.cu)
  int n_sms = 0;
  float* d_dec_p0 = nullptr;
  float* d_dec_hc = nullptr;
  float* d_dec_part = nullptr;
  unsigned* d_dec_ctr = nullptr;

  cudaEvent_t ev[SKB_N_STAGES + 1]{};
  float stage_ms[SKB_N_STAGES]{};
  bool have_stage_ms = false;
  bool stage_ms_pending = false;
  int last_launches = 0;
};

namespace {

void free_workspace(skb_layer* L) {
  void* ptrs[] = {L->d_x,        L->d_y,         L->d_logits,       L->d_ids,
                  L->d_wts,      L->disp.perm,   L->disp.inv,       L->disp.row_expert,
                  L->disp.expert_off, L->disp.tile_expert, L->disp.tile_row0, L->disp.tile_nrows,
                  L->disp.n_tiles, L->d_xs,      L->d_h,            L->d_kidx,
                  L->d_kval,     L->d_kcnt,      L->d_mask_in_r,
                  L->d_mask_in_s, L->d_mask_out_r, L->d_mask_out_s, L->d_counters,
                  L->d_hb,       L->d_slot_out,  L->d_ids_stage,    L->d_wts_stage,
                  L->d_xb,       L->disp.tile_colrow, L->d_dec_p0,
                  L->d_dec_hc,   L->d_dec_part,  L->d_dec_ctr,      L->d_sg,
                  L->d_slot_noff};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  L->d_x = L->d_y = L->d_logits = L->d_wts = L->d_h = L->d_kval = nullptr;
  L->d_ids = L->d_kidx = L->d_kcnt = L->d_slot_noff = nullptr;
  L->disp = DispatchBuffers{};
  L->d_xs = nullptr;
  L->d_counters = nullptr;
  L->d_hb = nullptr;
  L->d_slot_out = nullptr;
  L->d_ids_stage = nullptr;
  L->d_wts_stage = nullptr;
  L->d_xb = nullptr;
  L->d_dec_p0 = L->d_dec_hc = L->d_dec_part = nullptr;
  L->d_dec_ctr = nullptr;
  L->d_sg = nullptr;
  L->d_mask_in_r = L->d_mask_in_s = L->d_mask_out_r = L->d_mask_out_s = nullptr;
  L->cap_batch = 0;
}

template <typename T>
int dmalloc(T** p, size_t count) {
  SKB_CUDA(cudaMalloc(reinterpret_cast<void**>(p), (count ? count : 1) * sizeof(T)));
  return SKB_OK;
}

int max_tiles_for(const Geometry& g, int B, int tn) {
  const int BK = B * g.K;
  return (g.E < BK ? g.E : BK) + BK / tn + (g.has_shared ? ceil_div(B, tn) : 0);
}

int reserve_locked(skb_layer* L, int B) {
  if (B <= L->cap_batch) return SKB_OK;
  SKB_CUDA(cudaSetDevice(L->device));
  SKB_CUDA(cudaStreamSynchronize(L->stream));
  free_workspace(L);
  const Geometry& g = L->g;
  int cap = 1;
  while (cap < B) cap <<= 1;
  const size_t BK = static_cast<size_t>(cap) * g.K;
  const size_t rows = BK + (g.has_shared ? cap : 0);
  int rc;
#define SKB_TRY(x) \
  if ((rc = (x)) != SKB_OK) return rc
  SKB_TRY(dmalloc(&L->d_x, static_cast<size_t>(cap) * g.D));
  SKB_TRY(dmalloc(&L->d_y, static_cast<size_t>(cap) * g.D));
  SKB_TRY(dmalloc(&L->d_logits, static_cast<size_t>(cap) * (L->route_E > g.E ? L->route_E : g.E)));
  {
    const size_t rk = static_cast<size_t>(cap) * (L->route_K > g.K ? L->route_K : g.K);
    SKB_TRY(dmalloc(&L->d_ids, rk));
    SKB_TRY(dmalloc(&L->d_wts, rk));
  }
  SKB_TRY(dmalloc(&L->d_ids_stage, BK));
  SKB_TRY(dmalloc(&L->d_wts_stage, BK));
  SKB_TRY(dmalloc(&L->disp.perm, BK));
  SKB_TRY(dmalloc(&L->disp.inv, BK));
  SKB_TRY(dmalloc(&L->disp.row_expert, rows));
  SKB_TRY(dmalloc(&L->disp.expert_off, static_cast<size_t>(g.E) + 2));
  const size_t max_tiles = static_cast<size_t>(max_tiles_for(g, cap, 16)) + 1;
  SKB_TRY(dmalloc(&L->disp.tile_expert, max_tiles));
  SKB_TRY(dmalloc(&L->disp.tile_row0, max_tiles));
  SKB_TRY(dmalloc(&L->disp.tile_nrows, max_tiles));
  SKB_TRY(dmalloc(&L->disp.n_tiles, 1));
  SKB_TRY(dmalloc(&L->disp.tile_colrow, max_tiles * 16));
  {
    const size_t xb_rows = cap > 16 ? cap : 16;
    SKB_TRY(dmalloc(&L->d_xb, xb_rows * g.Dp));
    SKB_CUDA(cudaMemsetAsync(L->d_xb, 0, xb_rows * g.Dp * sizeof(__nv_bfloat16), L->stream));
    SKB_TRY(encode_bf16_2d(&L->tmap_xb, L->d_xb, xb_rows, g.Dp, 16));
  }
  {
    const size_t n_counters = 4 + static_cast<size_t>(cap);  // router counters + grid-barrier pair
    SKB_TRY(dmalloc(&L->d_counters, n_counters));
    SKB_CUDA(cudaMemsetAsync(L->d_counters, 0, n_counters * sizeof(unsigned), L->stream));
  }
  if (decode_fused_eligible(g, 1)) {
    const size_t crow = 16 * static_cast<size_t>(decode_cand_rows(g.K)) + 16;
    SKB_TRY(dmalloc(&L->d_dec_p0, static_cast<size_t>(decode_p0_words(g))));
    SKB_CUDA(cudaMemsetAsync(L->d_dec_p0, 0, decode_p0_words(g) * sizeof(float), L->stream));
    SKB_TRY(dmalloc(&L->d_dec_hc, crow * g.Nh));
    SKB_CUDA(cudaMemsetAsync(L->d_dec_hc, 0, crow * g.Nh * sizeof(float), L->stream));
    SKB_TRY(dmalloc(&L->d_dec_part,
                    16 * static_cast<size_t>(decode_cand_rows(g.K) + 1) *
                        decode_chunks(g, 1, g.N > g.S ? g.N : g.S, L->n_sms) * g.Dp));
    SKB_TRY(dmalloc(&L->d_dec_ctr, static_cast<size_t>(decode_counter_words())));
    SKB_CUDA(cudaMemsetAsync(L->d_dec_ctr, 0, decode_counter_words() * sizeof(unsigned), L->stream));
  }
  L->xs_rows = rows;
  SKB_TRY(dmalloc(&L->d_xs, rows * g.Dp));
  SKB_CUDA(cudaMemsetAsync(L->d_xs, 0, rows * g.Dp * sizeof(__nv_bfloat16), L->stream));
  for (int i = 0; i < 5; ++i)
    SKB_TRY(encode_bf16_2d(&L->tmap_x[i], L->d_xs, rows, g.Dp, kTileCases[i]));
  SKB_TRY(dmalloc(&L->d_h, rows * g.Nh));
  SKB_TRY(dmalloc(&L->d_sg, rows * g.Nh));
  SKB_TRY(dmalloc(&L->d_hb, 3 * rows * g.Nh));
  SKB_CUDA(cudaMemsetAsync(L->d_hb, 0, 3 * rows * g.Nh * sizeof(__nv_bfloat16), L->stream));
  for (int i = 0; i < 5; ++i)
    for (int sp = 0; sp < 3; ++sp)
      SKB_TRY(encode_bf16_2d(&L->tmap_hb[i][sp], L->d_hb + sp * rows * g.Nh, rows, g.Nh,
                             kTileCases[i]));
  SKB_TRY(dmalloc(&L->d_slot_out, rows * g.Dp));
  SKB_TRY(dmalloc(&L->d_kidx, rows * g.Nh));
  SKB_TRY(dmalloc(&L->d_kval, rows * g.Nh));
  SKB_TRY(dmalloc(&L->d_kcnt, rows));
  SKB_TRY(dmalloc(&L->d_slot_noff, static_cast<size_t>(g.K)));
  SKB_TRY(dmalloc(&L->d_mask_in_r, BK * g.N));
  SKB_TRY(dmalloc(&L->d_mask_out_r, BK * g.N));
  if (g.has_shared) {
    SKB_TRY(dmalloc(&L->d_mask_in_s, static_cast<size_t>(cap) * g.S));
    SKB_TRY(dmalloc(&L->d_mask_out_s, static_cast<size_t>(cap) * g.S));
  }
#undef SKB_TRY
  SKB_CUDA(cudaStreamSynchronize(L->stream));
  L->cap_batch = cap;
  return SKB_OK;
}

int validate_cfg(const skb_config* c) {
  // MoEConfig::validate, proj/src/model.cpp:113-127
  if (c == nullptr) return fail(SKB_ECONFIG, "config is null");
  if (c->n_experts < 1) return fail(SKB_ECONFIG, "n_experts must be >= 1");
  if (c->top_k < 1 || c->top_k > c->n_experts)
    return fail(SKB_ECONFIG, "top_k must satisfy 1 <= K <= E, got K=%d E=%d", c->top_k,
                c->n_experts);
  if (c->d_model < 1) return fail(SKB_ECONFIG, "d_model must be >= 1");
  if (c->d_ffn < 1) return fail(SKB_ECONFIG, "d_ffn must be >= 1");
  if (c->d_shared < 0) return fail(SKB_ECONFIG, "d_shared must be >= 0");
  if ((c->has_shared != 0) != (c->d_shared > 0))
    return fail(SKB_ECONFIG, "has_shared must match d_shared > 0");
  if (c->align_block < 1) return fail(SKB_ECONFIG, "align_block must be >= 1");
  return SKB_OK;
}

int new_layer(const skb_config* cfg, int device, skb_layer** out, int route_E = 0, int route_K = 0) {
  int rc = validate_cfg(cfg);
  if (rc) return rc;
  if (out == nullptr) return fail(SKB_EINTERNAL, "out pointer is null");
  if (cfg->n_experts > kMaxExperts)
    return fail(SKB_ECONFIG, "n_experts=%d exceeds the device router limit %d", cfg->n_experts,
                kMaxExperts);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1)
    return fail(SKB_ECUDA, "no CUDA device: this library has no CPU path");
  if (device < 0 || device >= ndev) return fail(SKB_ECUDA, "device %d outside [0, %d)", device, ndev);
  SKB_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  SKB_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(SKB_ECUDA, "device %d is sm_%d%d; this library is built for sm_100a only", device,
                prop.major, prop.minor);
  skb_layer* L = new skb_layer();
  L->cfg = *cfg;
  L->device = device;
  L->n_sms = prop.multiProcessorCount;
  Geometry& g = L->g;
  g.E = cfg->n_experts;
  g.K = cfg->top_k;
  g.D = cfg->d_model;
  g.N = cfg->d_ffn;
  g.S = cfg->has_shared ? cfg->d_shared : 0;
  g.has_shared = cfg->has_shared ? 1 : 0;
  g.renorm = cfg->renormalize ? 1 : 0;
  g.Dp = round_up(g.D, kBlockK);
  g.Dp128 = round_up(g.D, 128);
  g.Np = round_up(g.N, kNeuronBlock);
  g.Sp = g.has_shared ? round_up(g.S, kNeuronBlock) : 0;
  g.Nh = g.Np > g.Sp ? g.Np : g.Sp;
  L->route_E = route_E > 0 ? route_E : g.E;
  L->route_K = route_K > 0 ? route_K : g.K;
  L->route_renorm = g.renorm;
  if (L->route_E > kMaxExperts) {
    delete L;
    return fail(SKB_ECONFIG, "n_experts=%d exceeds the device router limit %d", route_E, kMaxExperts);
  }
  cudaError_t e = cudaStreamCreateWithFlags(&L->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete L;
    return fail(SKB_ECUDA, "cudaStreamCreate failed: %s", cudaGetErrorString(e));
  }
  for (auto& ev : L->ev) cudaEventCreate(&ev);
  cudaDeviceGetAttribute(&L->l2_bytes, cudaDevAttrL2CacheSize, device);
  const size_t gu_rows = static_cast<size_t>(g.E) * 2 * g.Np + 2 * static_cast<size_t>(g.Sp);
  const size_t wd_rows = static_cast<size_t>(g.E) * g.Np + g.Sp;
  rc = dmalloc(&L->d_router, static_cast<size_t>(L->route_E) * g.D);
  if (!rc) rc = dmalloc(&L->d_wgu, gu_rows * g.Dp);
  if (!rc) rc = dmalloc(&L->d_wd, wd_rows * g.Dp);
  if (!rc && decode_fused_eligible(g, 1)) rc = dmalloc(&L->d_wu, static_cast<size_t>(g.E) * g.Np * g.Dp);
  if (rc) {
    skb_layer_destroy(L);
    return rc;
  }
  const size_t wdt_elems = static_cast<size_t>(g.E) * g.Dp128 * g.Np + static_cast<size_t>(g.Dp128) * g.Sp;
  if (!rc) rc = dmalloc(&L->d_wdt, wdt_elems);
  if (rc) {
    skb_layer_destroy(L);
    return rc;
  }
  L->d_wd_shared = g.has_shared ? L->d_wd + static_cast<size_t>(g.E) * g.Np * g.Dp : nullptr;
  L->d_wdt_shared = g.has_shared ? L->d_wdt + static_cast<size_t>(g.E) * g.Dp128 * g.Np : nullptr;
  L->weight_bytes = static_cast<uint64_t>(g.E) * g.D * 4 + (gu_rows + wd_rows) * g.Dp * 2 + wdt_elems * 2 +
                    (L->d_wu ? static_cast<uint64_t>(g.E) * g.Np * g.Dp * 2 : 0);
  cudaMemsetAsync(L->d_wdt, 0, wdt_elems * 2, L->stream);
  cudaMemsetAsync(L->d_wgu, 0, gu_rows * g.Dp * 2, L->stream);
  cudaMemsetAsync(L->d_wd, 0, wd_rows * g.Dp * 2, L->stream);
  if (L->d_wu) cudaMemsetAsync(L->d_wu, 0, static_cast<size_t>(g.E) * g.Np * g.Dp * 2, L->stream);
  // tiled images: the tensor maps see them as [n_tiles * 128][64] (tiled_index())
  rc = encode_bf16_2d(&L->tmap_w, L->d_wgu, gu_rows * (g.Dp / kBlockK), kBlockK, 128);
  if (!rc)  // the same image as planes of 128 x 64 tiles: a box is 32 rows of 4 consecutive tiles
    rc = encode_bf16_3d(&L->tmap_w3, L->d_wgu, 128, gu_rows / 128 * (g.Dp / kBlockK), kBlockK * 2,
                        128 * kBlockK * 2, 32, 4, /*swizzle=*/false);
  if (!rc)
    rc = encode_bf16_3d(&L->tmap_w3g, L->d_wgu, 128, gu_rows / 128 * (g.Dp / kBlockK), kBlockK * 2,
                        128 * kBlockK * 2, 16, 4, /*swizzle=*/false);
  if (!rc)
    rc = encode_bf16_2d(&L->tmap_wdt, L->d_wdt,
                        static_cast<uint64_t>(g.E) * g.Dp128 * (g.Np / kBlockK), kBlockK, 128);
  if (!rc && g.has_shared)
    rc = encode_bf16_2d(&L->tmap_wdt_shared, L->d_wdt_shared,
                        static_cast<uint64_t>(g.Dp128) * (g.Sp / kBlockK), kBlockK, 128);
  if (rc) {
    skb_layer_destroy(L);
    return rc;
  }
  *out = L;
  return SKB_OK;
}

struct StageTimer {
  skb_layer* L;
  bool on;
  cudaStream_t s;
  int i = 0;
  void mark() {
    if (on) cudaEventRecord(L->ev[i++], s);
  }
};

// Fused decode kernel or staged kernels for a batch <= 4?  Both are correct for every eligible
// shape; which is faster depends on how much the per-(token, slot) row gather of the fused
// kernel moves against one pass over the routed experts' W_down.  Linear models fitted to
// measurements on B200 (tools/fused_vs_staged.py: Granite, OLMoE, Qwen3.5 and GPT-OSS shapes,
// batches 1-4, s = 0.5, clean L2): microseconds from MB.  One and two tokens: the fused kernel
// by 20-40 %; three: a tie; four: the staged kernels by 5-25 %.
bool decode_fused_preferred(const Geometry& g, int B, double keep_r, double keep_s) {
  const double E = g.E, K = g.K;
  const double U = E * (1.0 - std::pow(1.0 - K / E, B));  // expected distinct routed experts
  const double row_mb = g.Dp * 2.0 / 1e6;
  const double gup = (U * 2.0 * g.N + (g.has_shared ? 2.0 * g.S : 0.0)) * row_mb;
  const double vg = (B * K * keep_r + (g.has_shared ? B * keep_s : 0.0)) * row_mb;
  const double vd = (U * g.N + (g.has_shared ? g.S : 0.0)) * row_mb;
  const double R = K + (g.has_shared ? 1.0 : 0.0);
  double fused = 24.0 + 0.20 * gup + 0.30 * vg + 0.53 * B * R;
  if (B >= 3) fused += 4.0 + 0.025 * gup;  // four tokens per consumer lane: slower per byte
  // staged kernels: a fixed chain of launches whose router part grows with d_model (the exact
  // logit chains are d_model dependent adds long), plus one pass over the routed experts
  const double staged = 32.0 + 10.34 * (g.Dp / 1024.0) + 0.1814 * (gup + 0.5 * vd);
  return fused <= staged;
}

// Enqueues every stage of one forward on `stream`.  x/y (and masks in MASKED mode) are device
// pointers.  No allocation, no synchronisation.
int forward_core(skb_layer* L, const skb_forward_args* a, const float* d_x, float* d_y,
                 const uint8_t* d_mask_r, const uint8_t* d_mask_s, uint8_t* d_mask_out_r,
                 uint8_t* d_mask_out_s, cudaStream_t stream, bool timing,
                 const int32_t* d_ids_in = nullptr, const float* d_w_in = nullptr,
                 int32_t* d_ids_out = nullptr, float* d_w_out = nullptr, bool capture_h = false,
                 float* const* d_y_rows = nullptr) {
  const Geometry& g = L->g;
  const int B = a->batch;
  const int BK = B * g.K;
  const int rows = BK + (g.has_shared ? B : 0);
  LaunchCtx ctx{stream, !timing && !(a->flags & SKB_FLAG_NO_PDL)};
  StageTimer tm{L, timing, stream};
  int launches = 0;

  if (a->mode == SKB_MODE_ROUTE_ONLY) {
    RouterLaunch r{};
    r.x = d_x;
    r.router = L->d_router;
    r.B = B;
    r.E = L->route_E;
    r.D = g.D;
    r.K = L->route_K;
    r.renorm = L->route_renorm;
    r.fast = (a->flags & SKB_FLAG_FAST_ROUTER) != 0;
    r.logits = L->d_logits;
    r.ids = d_ids_out ? d_ids_out : L->d_ids;
    r.weights = d_w_out ? d_w_out : L->d_wts;
    r.counters = L->d_counters;
    r.dispatch = nullptr;
    launches += launch_router(ctx, r);
    L->last_launches = launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SKB_ECUDA, "kernel launch failed: %s", cudaGetErrorString(e));
    return SKB_OK;
  }

  const bool budget = a->mode == SKB_MODE_TOPK && a->slot_n_off != nullptr;
  int sel_mode, n_off_r = 0, n_off_s = 0;
  int max_keep = g.N > g.S ? g.N : g.S;
  if (a->mode == SKB_MODE_DENSE) {
    sel_mode = kSelectAll;
  } else if (a->mode == SKB_MODE_TOPK) {
    sel_mode = kSelectTopk;
    n_off_r = n_off_of(a->s_routed, g.N);
    n_off_s = g.has_shared ? n_off_of(a->s_shared, g.S) : 0;
    int kr = g.N - n_off_r;
    const int ks = g.S - n_off_s;
    if (budget)  // per-slot counts: the largest survivor count bounds the lists
      for (int sl = 0; sl < g.K; ++sl) kr = kr > g.N - a->slot_n_off[sl] ? kr : g.N - a->slot_n_off[sl];
    max_keep = kr > ks ? kr : ks;
  } else if (a->mode == SKB_MODE_THRESHOLD) {
    sel_mode = kSelectThreshold;
  } else {
    sel_mode = kSelectGiven;
  }

  // Down-projection path of the staged kernels (batches above 4; smaller ones take the fused
  // decode kernel, which gathers).  Gathering surviving rows per (token, slot) moves B*K*keep rows
  // through L2; the dense masked GEMM streams each routed expert's W_down once.  Measured on B200
  // (tools/path_probe.py, tools/fused_vs_staged.py, tools/ep_probe.py; us, gather / dense):
  // Qwen3.5 shape B=64 s=.5 482 / 353, s=.9 463 / 371; B=32 295 / 278; OLMoE shape B=32 261 / 232,
  // B=8 158 / 140, B=5 116 / 100; Granite shape B=32 99 / 69, B=8 58 / 52; GPT-OSS shape B=8
  // 257 / 211; Llama-4-Maverick shape, 64 rows with external routing at s=.9 (the expert-parallel
  // step, gather volume 10 % of the dense one) 1931 / 631 -- the cluster gather kernel loses at
  // every staged batch size, so the masked GEMM is the default and the gather a forced option
  // (SKB_FLAG_GATHER_DOWN; the tests keep it honest).  The decision is identical for
  // forward_dense and forward_topk_sparse at s = 0.
  bool dense_down = true;
  {
    if (a->flags & SKB_FLAG_GATHER_DOWN) dense_down = false;
    if (a->flags & SKB_FLAG_DENSE_DOWN) dense_down = true;
    // threshold selection: the survivor count is data dependent; the masked GEMM covers every case
    if (sel_mode == kSelectThreshold) dense_down = true;
    // per-slot counts: the stand-alone selection kernel is the one that takes them
    if (budget) dense_down = true;
  }
  // masked activations of the dense down projection as bf16 terms: one (1e-2 mode), or two --
  // 16 mantissa bits, measured 3e-7..1e-6 of the output on every BASELINE shape
  // (tools/h_err_probe.py); a third term (exact) bought nothing the 1e-5 bar can see and cost a
  // third of the GEMM's MMA steps and token-tile traffic
  const int nsplit = (a->flags & SKB_FLAG_BF16_H) ? 1 : 2;
  // 1e-5 parity mode: the tensor-core GEMMs fold long contractions chunk by chunk (gateup.cu)
  const bool precise = !(a->flags & SKB_FLAG_BF16_H);

  if (d_y_rows != nullptr && !dense_down)
    return fail(SKB_ECONFIG, "forward: per-row output destinations need the dense down projection");
  // Decode batches: the whole layer as one persistent launch (decode.cu).
  if (d_y_rows == nullptr && d_ids_in == nullptr && L->d_dec_ctr != nullptr && decode_fused_eligible(g, B) &&
      !budget && (sel_mode != kSelectThreshold || L->d_wu != nullptr) &&
      !(a->flags & (SKB_FLAG_FAST_ROUTER | SKB_FLAG_SIMT_GATEUP | SKB_FLAG_DENSE_DOWN |
                    SKB_FLAG_GATHER_DOWN | SKB_FLAG_NO_FUSED_DECODE)) &&
      ((a->flags & SKB_FLAG_FUSED_DECODE) ||
       decode_fused_preferred(g, B,
                              sel_mode == kSelectTopk ? g.N - n_off_r
                                                      : (sel_mode == kSelectThreshold ? g.N / 2 : g.N),
                              sel_mode == kSelectTopk ? g.S - n_off_s : g.S))) {
    const bool want_masks = d_mask_out_r != nullptr || d_mask_out_s != nullptr;
    DecodeLaunch dl{};
    dl.x = d_x;
    dl.router = L->d_router;
    dl.wd = L->d_wd;
    dl.wd_shared = L->d_wd_shared;
    dl.B = B;
    dl.sel_mode = sel_mode;
    dl.n_off_r = n_off_r;
    dl.n_off_s = n_off_s;
    dl.tau = a->tau;
    dl.wu = L->d_wu;
    dl.kcnt = L->d_kcnt;
    dl.mask_r = d_mask_r;
    dl.mask_s = d_mask_s;
    dl.CH = decode_chunks(g, B, max_keep, L->n_sms);
    dl.capture = capture_h || want_masks;
    dl.p0 = L->d_dec_p0;
    dl.logits = L->d_logits;
    dl.ids = L->d_ids;
    dl.wts = L->d_wts;
    dl.hc = L->d_dec_hc;
    dl.part = L->d_dec_part;
    dl.ctr = L->d_dec_ctr;
    dl.y = d_y;
    dl.h_cap = L->d_h;
    dl.inv = L->disp.inv;
    dl.perm = L->disp.perm;
    dl.row_expert = L->disp.row_expert;
    tm.mark();
    tm.mark();
    tm.mark();
    launches += launch_decode_fused(ctx, &L->tmap_w3, &L->tmap_w3g, dl, g, L->n_sms);
    tm.mark();
    if (want_masks) {
      SelectArgs sa{};
      sa.h = L->d_h;
      sa.rows = rows;
      sa.BK = BK;
      sa.N = g.N;
      sa.S = g.S;
      sa.Nh = g.Nh;
      sa.K = g.K;
      sa.perm = L->disp.perm;
      sa.mask_out_routed = d_mask_out_r;
      sa.mask_out_shared = d_mask_out_s;
      sa.mode = sel_mode;
      sa.n_off_routed = n_off_r;
      sa.n_off_shared = n_off_s;
      sa.mask_in_routed = d_mask_r;
      sa.mask_in_shared = d_mask_s;
      if (sel_mode == kSelectThreshold) {
        // the fused kernel's routed rows hold silu(gate) in this mode (the up projection is
        // only ever computed for the survivors)
        sa.sg = L->d_h;
        sa.tau = a->tau;
      }
      LaunchCtx plain{stream, false};
      launches += launch_select(plain, sa);
    }
    tm.mark();
    tm.mark();
    tm.mark();
    L->last_launches = launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SKB_ECUDA, "kernel launch failed: %s", cudaGetErrorString(e));
    return SKB_OK;
  }

  // tile size for the grouped GEMMs: ~1.5x the mean tokens per expert, power of two in
  // [16, 256] (at most 128 when the dense down projection shares the tile list)
  int tn = 16;
  {
    const double want = 1.5 * static_cast<double>(BK) / g.E;
    // (and when the fp32-accumulation mode folds long contractions chunk by chunk: its master
    // accumulator shares the TMEM with two chunk buffers, gateup.cu)
    const int cap = (dense_down || precise) ? 128 : 256;
    while (tn < cap && tn < want) tn <<= 1;
  }
  // decode: token-indexed tiles built inside the router kernel (no expert-sorted token copy)
  // (the dense down projection walks the same tile list and needs it expert-sorted)
  const bool token_tiles = d_ids_in == nullptr && tn == 16 && !dense_down &&
                           !(a->flags & SKB_FLAG_SIMT_GATEUP) &&
                           !(a->flags & SKB_FLAG_FAST_ROUTER) && router_token_tiles(B, g.K, true);
  int tn_idx = 0;
  while (kTileCases[tn_idx] != tn) ++tn_idx;
  const int max_tiles = max_tiles_for(g, B, tn);

  // Paired weight blocks (gateup.cu): worth it once the tile list alone covers most SMs with
  // half as many CTAs; below that the extra CTAs' parallelism is worth more than the bytes.
  const int est_tiles = (g.E < BK ? g.E : BK) + (g.has_shared ? 1 : 0);
  const auto pair_for = [&](int mblocks) {
    return tn >= 64 && !(a->flags & SKB_FLAG_NO_PAIRED_BLOCKS) &&
           ((a->flags & SKB_FLAG_PAIRED_BLOCKS) ||
            est_tiles * ceil_div(mblocks, 2) * 4 >= L->n_sms * 3);
  };
  // gate/up: slower paired while the grid is about one CTA per SM (Granite shape batch 256: 25.5 ->
  // 29.7 us stage time; GPT-OSS shape prefill with one CTA per SM: 0.77 -> 0.87 ms -- nothing hides a
  // tile's ramp and epilogue); with two CTAs per SM on a two-stage ring each, a grid of several
  // waves gains (GPT-OSS shape, 4096 tokens: 0.77 -> 0.71 ms).  Hence: only for such grids.
  const long paired_gateup_ctas =
      static_cast<long>(est_tiles + BK / tn) * ceil_div(g.Np / kNeuronBlock, 2);
  const bool pair_gateup =
      !(a->flags & SKB_FLAG_NO_PAIRED_BLOCKS) && tn >= 64 &&
      ((a->flags & SKB_FLAG_PAIRED_BLOCKS) || (tn == 128 && paired_gateup_ctas >= 4L * L->n_sms));
  const bool pair_down = pair_for(g.Dp128 / 128);

  bool permuted = false;  // the router stage wrote the expert-sorted token copy itself
  tm.mark();
  if (d_ids_in != nullptr) {
    // external routing: ids (and weights, default 1) are given; only the dispatch runs
    ctx.pdl = false;  // memcpy nodes in between: plain stream order for this call
    cudaMemcpyAsync(L->d_ids, d_ids_in, static_cast<size_t>(BK) * 4, cudaMemcpyDeviceToDevice, stream);
    if (d_w_in != nullptr)
      cudaMemcpyAsync(L->d_wts, d_w_in, static_cast<size_t>(BK) * 4, cudaMemcpyDeviceToDevice, stream);
    else
      launches += launch_fill_f32(stream, L->d_wts, 1.0f, static_cast<size_t>(BK));
    launches += launch_dispatch(ctx, L->d_ids, B, g.K, g.E, g.has_shared, tn, L->disp);
  } else {
    RouterLaunch r{};
    r.x = d_x;
    r.router = L->d_router;
    r.B = B;
    r.E = g.E;
    r.D = g.D;
    r.K = g.K;
    r.renorm = g.renorm;
    r.fast = (a->flags & SKB_FLAG_FAST_ROUTER) != 0;
    r.logits = L->d_logits;
    r.ids = L->d_ids;
    r.weights = L->d_wts;
    r.counters = L->d_counters;
    r.dispatch = &L->disp;
    r.has_shared = g.has_shared;
    r.tile_tokens = tn;
    r.xb = token_tiles ? L->d_xb : nullptr;
    r.Dp = g.Dp;
    if (!token_tiles && !(a->flags & SKB_FLAG_FAST_ROUTER)) {
      r.xs = L->d_xs;
      r.grid_bar = L->d_counters + 2 + L->cap_batch;
    }
    permuted = router_fuses_permute(r);
    launches += launch_router(ctx, r);
  }
  tm.mark();
  if (!token_tiles && !permuted)
    launches += launch_permute_tokens(ctx, d_x, L->disp.perm, B, g.K, g.D, g.Dp, g.has_shared,
                                      L->d_xs);
  tm.mark();
  if (a->flags & SKB_FLAG_SIMT_GATEUP)
    launches += launch_gateup_simt(ctx, L->d_wgu, L->d_xs, L->disp.row_expert, rows, g, L->d_h);
  else
    launches += launch_gateup_tc(ctx, &L->tmap_w, token_tiles ? &L->tmap_xb : &L->tmap_x[tn_idx],
                                 &L->tmap_x[1], tn, L->disp, max_tiles, g, L->d_h, token_tiles,
                                 sel_mode == kSelectThreshold ? L->d_sg : nullptr, pair_gateup,
                                 precise, /*early_tiles=*/!token_tiles && !permuted,
                                 /*prefetch image=*/nullptr,
                                 permuted ? reinterpret_cast<const int*>(L->d_counters + 3 + L->cap_batch)
                                          : nullptr);
  tm.mark();

  // Gather path: the selection runs inside the down kernel; the stand-alone selection kernel
  // then only serves mask captures (MaskSet export).  Dense path: it writes the masked
  // activations the GEMM consumes.
  if (dense_down || d_mask_out_r != nullptr || d_mask_out_s != nullptr) {
    SelectArgs sa{};
    sa.h = L->d_h;
    sa.rows = rows;
    sa.BK = BK;
    sa.N = g.N;
    sa.S = g.S;
    sa.Nh = g.Nh;
    sa.K = g.K;
    sa.perm = L->disp.perm;
    sa.mask_out_routed = d_mask_out_r;
    sa.mask_out_shared = d_mask_out_s;
    sa.mode = sel_mode;
    sa.n_off_routed = n_off_r;
    sa.n_off_shared = n_off_s;
    sa.mask_in_routed = d_mask_r;
    sa.mask_in_shared = d_mask_s;
    if (budget) sa.slot_counts = L->d_slot_noff;
    if (sel_mode == kSelectThreshold) {
      sa.sg = L->d_sg;
      sa.tau = a->tau;
      sa.kept_cnt = L->d_kcnt;  // per-row survivor counts: the report's tile accounting
    }
    if (dense_down) {
      sa.hb = L->d_hb;
      sa.hb_split_stride = static_cast<size_t>(L->xs_rows) * g.Nh;
      sa.nsplit = nsplit;
      sa.kext_routed = g.Np;
      sa.kext_shared = g.Sp;
    }
    launches += launch_select(ctx, sa);
  }
  tm.mark();

  // Per-row destinations with one expert per row, weight 1 and no shared expert (the expert
  // rank of expert parallelism): the combine would copy -- the GEMM's epilogue stores there itself.
  const bool direct_rows = d_y_rows != nullptr && g.K == 1 && !g.has_shared && d_ids_in != nullptr &&
                           d_w_in == nullptr;
  if (dense_down) {
    // W_down^T blocks prefetched into the L2 while the CTAs wait for the selection kernel: pays
    // when the image is small enough to sit there (Granite shape batch 256: the down stage starts
    // 2.5 us earlier); on a long stream the prefetches only queue ahead of the demand loads
    // (Qwen3.5 shape batch 64: stage time 79 -> 93 us)
    const bool prefetch_wdt =
        static_cast<size_t>(g.E) * g.Dp128 * g.Np * 2 <= static_cast<size_t>(L->l2_bytes) / 2;
    launches += launch_down_tc(ctx, &L->tmap_wdt, g.has_shared ? &L->tmap_wdt_shared : nullptr,
                               L->tmap_hb[tn_idx], L->tmap_hb[1], nsplit, tn, L->disp, max_tiles, g,
                               L->d_slot_out, pair_down, precise, /*early_tiles=*/true,
                               prefetch_wdt ? L->d_wdt : nullptr,
                               prefetch_wdt ? L->d_wdt_shared : nullptr,
                               direct_rows ? d_y_rows : nullptr, direct_rows ? L->disp.perm : nullptr);
    tm.mark();
    if (!direct_rows)
      launches += launch_combine_rows(ctx, L->d_slot_out, L->disp.inv, L->d_wts, B, g, d_y, d_y_rows);
    tm.mark();
  } else {
    DownArgs da{};
    da.wd = L->d_wd;
    da.wd_shared = L->d_wd_shared;
    da.row_expert = L->disp.row_expert;
    da.inv = L->disp.inv;
    da.weights = L->d_wts;
    da.B = B;
    da.K = g.K;
    da.BK = BK;
    da.has_shared = g.has_shared;
    da.h = L->d_h;
    da.Nh = g.Nh;
    da.N = g.N;
    da.S = g.S;
    da.sel_mode = sel_mode;
    da.n_off_routed = n_off_r;
    da.n_off_shared = n_off_s;
    da.mask_in_routed = d_mask_r;
    da.mask_in_shared = d_mask_s;
    da.max_keep = max_keep;
    da.y = d_y;
    const int n = launch_down(ctx, da, g);
    if (n < 0)
      return fail(SKB_ECONFIG, "forward: top_k * d_ffn too large for the down-projection kernel's "
                               "shared-memory lists (K=%d, N=%d, S=%d)", g.K, g.N, g.S);
    launches += n;
    tm.mark();
    tm.mark();
  }
  L->last_launches = launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(SKB_ECUDA, "kernel launch failed: %s", cudaGetErrorString(e));
  return SKB_OK;
}

int check_args(const skb_layer* L, const skb_forward_args* a, bool y_elsewhere = false) {
  if (L == nullptr) return fail(SKB_EINTERNAL, "layer is null");
  if (a == nullptr) return fail(SKB_EINTERNAL, "args is null");
  const Geometry& g = L->g;
  if (a->x == nullptr || (a->y == nullptr && a->mode != SKB_MODE_ROUTE_ONLY && !y_elsewhere))
    return fail(SKB_ESHAPE, "forward: x and y must be non-null");
  if (a->batch < 1) return fail(SKB_ESHAPE, "route: empty batch");  // router.cpp:16-18
  if (a->mode != SKB_MODE_DENSE && a->mode != SKB_MODE_TOPK && a->mode != SKB_MODE_MASKED &&
      a->mode != SKB_MODE_ROUTE_ONLY && a->mode != SKB_MODE_THRESHOLD)
    return fail(SKB_ECONFIG, "forward: unknown mode %d", a->mode);
  if (a->mode == SKB_MODE_ROUTE_ONLY && (a->ids_out == nullptr || a->weights_out == nullptr))
    return fail(SKB_ESHAPE, "route-only forward: ids_out and weights_out must be non-null");
  if (a->mode != SKB_MODE_ROUTE_ONLY && a->ids_in == nullptr && L->route_E != g.E)
    return fail(SKB_ECONFIG, "forward: an expert-parallel slice needs external routing (ids_in)");
  if (a->mode == SKB_MODE_MASKED) {
    // engine.cpp:107-117
    const uint64_t want = static_cast<uint64_t>(a->batch) * g.K * g.N;
    if (a->routed_mask_in == nullptr || a->routed_mask_len != want)
      return fail(SKB_ESHAPE, "forward_masked_dense: routed masks must be B*K*d_ffn");
    if (a->shared_mask_len != 0 &&
        (a->shared_mask_in == nullptr ||
         a->shared_mask_len != static_cast<uint64_t>(a->batch) * static_cast<uint64_t>(g.S)))
      return fail(SKB_ESHAPE, "forward_masked_dense: shared masks must be B*d_shared");
  }
  if (a->mode == SKB_MODE_THRESHOLD) {
    // engine.cpp:238-240 (NaN fails the comparison as well)
    if (!(a->tau >= 0.0f)) return fail(SKB_ECONFIG, "forward_sparse: threshold must be >= 0");
    if (a->flags & SKB_FLAG_SIMT_GATEUP)
      return fail(SKB_ECONFIG, "forward_sparse: the verification gate/up kernel has no threshold mode");
  }
  if (a->mode == SKB_MODE_TOPK) {
    // SparsityLevel, activation.hpp:18-22
    if (!(a->s_routed >= 0.0 && a->s_routed <= 1.0) || !(a->s_shared >= 0.0 && a->s_shared <= 1.0))
      return fail(SKB_ECONFIG, "sparsity must lie in [0, 1]");
    if (a->slot_n_off != nullptr)
      for (int sl = 0; sl < g.K; ++sl)  // budget.cpp:80-82
        if (a->slot_n_off[sl] < 0 || a->slot_n_off[sl] > g.N)
          return fail(SKB_ECONFIG, "apply_budget: keep_count outside [0, N]");
  }
  return SKB_OK;
}

void fill_report(const skb_layer* L, const skb_forward_args* a, skb_report* r,
                 const uint8_t* host_routed_mask, const uint8_t* host_shared_mask) {
  if (r == nullptr) return;
  const Geometry& g = L->g;
  const uint64_t B = a->batch, K = g.K, D = g.D, N = g.N, S = g.S, E = g.E;
  const uint64_t routed_neurons = B * K * N;
  std::memset(r, 0, sizeof(*r));
  uint64_t active = routed_neurons, active_sh = B * S;
  if (a->mode == SKB_MODE_TOPK) {
    active = B * K * (N - n_off_of(a->s_routed, g.N));
    if (a->slot_n_off != nullptr) {
      active = 0;
      for (uint64_t sl = 0; sl < K; ++sl) active += B * (N - static_cast<uint64_t>(a->slot_n_off[sl]));
    }
    if (g.has_shared) active_sh = B * (S - n_off_of(a->s_shared, g.S));
  } else if (a->mode == SKB_MODE_MASKED && host_routed_mask != nullptr) {
    active = 0;
    for (uint64_t i = 0; i < routed_neurons; ++i) active += host_routed_mask[i] ? 1 : 0;
    if (host_shared_mask != nullptr) {
      active_sh = 0;
      for (uint64_t i = 0; i < B * S; ++i) active_sh += host_shared_mask[i] ? 1 : 0;
    }
  }
  r->gate_macs = B * K * D * N;
  r->up_macs = B * K * D * N;
  r->other_macs = B * E * D;
  if (a->mode == SKB_MODE_TOPK) {
    // executed work: only surviving W_down rows are touched
    r->down_macs = active * D;
    if (g.has_shared) r->other_macs += B * 2 * S * D + active_sh * D;
    r->path_used = 1;
  } else {
    // forward_dense / forward_masked_dense charge full dense MACs (engine.hpp:41-42)
    r->down_macs = B * K * D * N;
    if (g.has_shared) r->other_macs += B * 3 * S * D;
    r->path_used = 0;
  }
  r->active_neurons_total = active;
  r->achieved_routed_sparsity =
      1.0 - static_cast<double>(active) / static_cast<double>(routed_neurons);
}

// ForwardReport of forward_sparse (engine.cpp:341-368) from the per-row survivor counts: the
// reference charges its gathered up/down stage in 64-neuron tiles of the compacted index list.
void fill_report_threshold(const skb_layer* L, const skb_forward_args* a, skb_report* r,
                           const int32_t* kcnt, const int32_t* inv) {
  if (r == nullptr) return;
  const Geometry& g = L->g;
  const uint64_t B = a->batch, K = g.K, D = g.D, N = g.N, S = g.S, E = g.E;
  std::memset(r, 0, sizeof(*r));
  const uint64_t capacity = (K * N + 31) / 32 * 32;  // default_capacity, activation.cpp:74-77
  const uint64_t token_tiles = (capacity + 63) / 64;   // tiles_per_token, engine.cpp:209-212
  uint64_t active = 0, padded = 0, skipped = 0;
  if (kcnt != nullptr) {
    for (uint64_t t = 0; t < B; ++t) {
      uint64_t at = 0;
      for (uint64_t s = 0; s < K; ++s) at += static_cast<uint64_t>(kcnt[inv[t * K + s]]);
      const uint64_t tiles = (at + 63) / 64;  // tiles_executed, engine.cpp:214-217
      active += at;
      padded += tiles * 64;
      skipped += token_tiles - tiles;
    }
  }
  r->gate_macs = B * K * D * N;
  r->up_macs = padded * D;
  r->down_macs = padded * D;
  r->other_macs = B * E * D + (g.has_shared ? B * 3 * S * D : 0);
  r->active_neurons_total = active;
  r->tiles_total = B * token_tiles;
  r->tiles_skipped = skipped;
  r->achieved_routed_sparsity =
      1.0 - static_cast<double>(active) / static_cast<double>(B * K * N);
  r->path_used = 1;
}

}  // namespace

extern "C" {

const char* skb_last_error(void) { return g_err.c_str(); }
int skb_abi_version(void) { return SKB_ABI_VERSION; }

int skb_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int skb_config_validate(const skb_config* cfg) { return validate_cfg(cfg); }

int skb_n_off(double s, int n, int32_t* out) {
  if (!(s >= 0.0 && s <= 1.0)) return fail(SKB_ECONFIG, "sparsity must lie in [0, 1]");
  if (n < 0 || out == nullptr) return fail(SKB_ESHAPE, "n_off: bad arguments");
  *out = n_off_of(s, n);
  return SKB_OK;
}

// ---- "MOE1" weight files (proj/src/model.cpp:180-282) ---------------------------------------

uint64_t skb_last_error_offset(void) { return g_err_offset; }

// Size of the file in 128-bit arithmetic (header fields are 31-bit values: their product wraps
// 64 bits); false when it does not fit in 64 bits or a field is negative.
static bool weight_file_size_checked(const skb_config* c, uint64_t* out) {
  if (c->d_model < 0 || c->n_experts < 0 || c->d_ffn < 0 || c->d_shared < 0) return false;
  const unsigned __int128 D = static_cast<unsigned __int128>(c->d_model) * sizeof(float);
  unsigned __int128 n = 28 + static_cast<unsigned __int128>(c->n_experts) * D +
                        static_cast<unsigned __int128>(3) * c->n_experts * c->d_ffn * D;
  if (c->has_shared) n += static_cast<unsigned __int128>(3) * c->d_shared * D;
  if (n > static_cast<unsigned __int128>(UINT64_MAX)) return false;
  *out = static_cast<uint64_t>(n);
  return true;
}

uint64_t skb_weight_file_size(const skb_config* c) {
  uint64_t n = 0;
  if (c == nullptr || !weight_file_size_checked(c, &n)) return 0;
  return n;
}

static int format_error(uint64_t at, const char* what) {
  g_err_offset = at;
  return fail(SKB_EFORMAT, "%s (offset %llu)", what, static_cast<unsigned long long>(at));
}

static bool host_is_little_endian() {
  const uint32_t probe = 1;
  unsigned char b;
  std::memcpy(&b, &probe, 1);
  return b == 1;
}

int skb_layer_load(const char* path, int device, skb_config* cfg_out, skb_layer** out) {
  if (path == nullptr || out == nullptr) return fail(SKB_EINTERNAL, "layer_load: null argument");
  if (!host_is_little_endian())
    return fail(SKB_EINTERNAL, "layer_load: the mapped-file loader needs a little-endian host");
  const int fd = ::open(path, O_RDONLY);
  if (fd < 0) return fail(SKB_EIO, "cannot open for reading: %s", path);
  struct stat st {};
  if (::fstat(fd, &st) != 0) {
    ::close(fd);
    return fail(SKB_EIO, "cannot open for reading: %s", path);
  }
  const uint64_t size = static_cast<uint64_t>(st.st_size);
  const unsigned char* base = nullptr;
  if (size > 0) {
    void* m = ::mmap(nullptr, size, PROT_READ, MAP_PRIVATE, fd, 0);
    if (m == MAP_FAILED) {
      ::close(fd);
      return fail(SKB_EIO, "cannot open for reading: %s", path);
    }
    base = static_cast<const unsigned char*>(m);
  }
  ::close(fd);
  auto done = [&](int rc) {
    if (base != nullptr) ::munmap(const_cast<unsigned char*>(base), size);
    return rc;
  };
  // the reference reads 4 bytes at a time: a short file stops at the last whole word
  const uint64_t whole = size / 4 * 4;
  if (size < 4) return done(format_error(0, "truncated file"));
  if (std::memcmp(base, "MOE1", 4) != 0) return done(format_error(0, "bad magic, expected MOE1"));
  if (size < 28) return done(format_error(whole, "truncated file"));
  auto u32 = [&](uint64_t off) {
    return static_cast<uint32_t>(base[off]) | (static_cast<uint32_t>(base[off + 1]) << 8) |
           (static_cast<uint32_t>(base[off + 2]) << 16) | (static_cast<uint32_t>(base[off + 3]) << 24);
  };
  skb_config c{};
  c.n_experts = static_cast<int32_t>(u32(4));
  c.top_k = static_cast<int32_t>(u32(8));
  c.d_model = static_cast<int32_t>(u32(12));
  c.d_ffn = static_cast<int32_t>(u32(16));
  c.d_shared = static_cast<int32_t>(u32(20));
  const uint32_t flags = u32(24);
  c.has_shared = (flags & 1u) ? 1 : 0;
  c.renormalize = (flags & 2u) ? 1 : 0;
  c.align_block = 64;
  if (c.n_experts < 1) return done(format_error(4, "header: n_experts < 1"));
  if (c.top_k < 1 || c.top_k > c.n_experts)
    return done(format_error(8, "header: top_k outside [1, n_experts]"));
  if (c.d_model < 1) return done(format_error(12, "header: d_model < 1"));
  if (c.d_ffn < 1) return done(format_error(16, "header: d_ffn < 1"));
  if ((c.has_shared != 0) != (c.d_shared > 0))
    return done(format_error(20, "header: shared flag disagrees with d_shared"));
  uint64_t want = 0;
  if (!weight_file_size_checked(&c, &want))  // a payload no file can hold: the file is short
    return done(format_error(whole, "truncated file"));
  if (size < want) return done(format_error(whole, "truncated file"));
  if (size > want) return done(format_error(want, "trailing bytes after weight payload"));

  const size_t E = static_cast<size_t>(c.n_experts);
  const uint64_t mat = static_cast<uint64_t>(c.d_ffn) * c.d_model * sizeof(float);
  const unsigned char* p = base + 28;
  const float* router = reinterpret_cast<const float*>(p);  // 28 is a multiple of 4
  p += E * c.d_model * sizeof(float);
  std::vector<const float*> gate, up, down;
  try {  // no exception may cross the C boundary
    gate.resize(E);
    up.resize(E);
    down.resize(E);
  } catch (const std::bad_alloc&) {
    return done(fail(SKB_EINTERNAL, "layer_load: out of host memory for %zu expert pointers", E));
  }
  for (size_t e = 0; e < E; ++e) {
    gate[e] = reinterpret_cast<const float*>(p);
    up[e] = reinterpret_cast<const float*>(p + mat);
    down[e] = reinterpret_cast<const float*>(p + 2 * mat);
    p += 3 * mat;
  }
  const float *sg = nullptr, *su = nullptr, *sd = nullptr;
  if (c.has_shared) {
    const uint64_t smat = static_cast<uint64_t>(c.d_shared) * c.d_model * sizeof(float);
    sg = reinterpret_cast<const float*>(p);
    su = reinterpret_cast<const float*>(p + smat);
    sd = reinterpret_cast<const float*>(p + 2 * smat);
  }
  if (cfg_out != nullptr) *cfg_out = c;
  return done(skb_layer_create(&c, router, gate.data(), up.data(), down.data(), sg, su, sd, device, out));
}

int skb_save_weights(const skb_config* cfg, const float* router, const float* const* gate,
                     const float* const* up, const float* const* down_t, const float* shared_gate,
                     const float* shared_up, const float* shared_down_t, const char* path) {
  int rc = validate_cfg(cfg);  // save_weights validates first (model.cpp:191)
  if (rc) return rc;
  if (path == nullptr || router == nullptr || gate == nullptr || up == nullptr || down_t == nullptr ||
      (cfg->has_shared && (shared_gate == nullptr || shared_up == nullptr || shared_down_t == nullptr)))
    return fail(SKB_EINTERNAL, "save_weights: null argument");
  FILE* f = std::fopen(path, "wb");
  if (f == nullptr) return fail(SKB_EIO, "cannot open for writing: %s", path);
  auto put_u32 = [&](uint32_t v) {
    const unsigned char b[4] = {static_cast<unsigned char>(v), static_cast<unsigned char>(v >> 8),
                                static_cast<unsigned char>(v >> 16), static_cast<unsigned char>(v >> 24)};
    std::fwrite(b, 1, 4, f);
  };
  const bool le = host_is_little_endian();
  auto put_matrix = [&](const float* m, size_t count) {
    if (le) {
      std::fwrite(m, sizeof(float), count, f);
    } else {
      for (size_t i = 0; i < count; ++i) {
        uint32_t bits;
        std::memcpy(&bits, m + i, 4);
        put_u32(bits);
      }
    }
  };
  std::fwrite("MOE1", 1, 4, f);
  put_u32(static_cast<uint32_t>(cfg->n_experts));
  put_u32(static_cast<uint32_t>(cfg->top_k));
  put_u32(static_cast<uint32_t>(cfg->d_model));
  put_u32(static_cast<uint32_t>(cfg->d_ffn));
  put_u32(static_cast<uint32_t>(cfg->d_shared));
  put_u32((cfg->has_shared ? 1u : 0u) | (cfg->renormalize ? 2u : 0u));
  const size_t D = static_cast<size_t>(cfg->d_model);
  put_matrix(router, static_cast<size_t>(cfg->n_experts) * D);
  for (int e = 0; e < cfg->n_experts; ++e) {
    put_matrix(gate[e], static_cast<size_t>(cfg->d_ffn) * D);
    put_matrix(up[e], static_cast<size_t>(cfg->d_ffn) * D);
    put_matrix(down_t[e], static_cast<size_t>(cfg->d_ffn) * D);
  }
  if (cfg->has_shared) {
    put_matrix(shared_gate, static_cast<size_t>(cfg->d_shared) * D);
    put_matrix(shared_up, static_cast<size_t>(cfg->d_shared) * D);
    put_matrix(shared_down_t, static_cast<size_t>(cfg->d_shared) * D);
  }
  const bool bad = std::ferror(f) != 0;
  if (std::fclose(f) != 0 || bad) return fail(SKB_EIO, "write failed");
  return SKB_OK;
}

int skb_generate_tokens(int32_t batch, int32_t d_model, uint64_t seed, float* out) {
  if (batch < 1 || d_model < 1)
    return fail(SKB_ECONFIG, "token batch needs batch >= 1 and d_model >= 1");
  if (out == nullptr) return fail(SKB_ESHAPE, "generate_tokens: null output");
  uint64_t state = seed;
  auto unit = [&state]() {  // SplitMix64 step, top 53 bits as a double in [0, 1)
    uint64_t z = (state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return static_cast<double>(z >> 11) * 0x1.0p-53;
  };
  const size_t n = static_cast<size_t>(batch) * static_cast<size_t>(d_model);
  for (size_t i = 0; i < n; i += 2) {
    double u1 = unit();
    const double u2 = unit();
    if (u1 <= 0.0) u1 = 0x1.0p-53;
    const double radius = std::sqrt(-2.0 * std::log(u1));
    const double angle = 2.0 * 3.14159265358979323846 * u2;
    const double second = radius * std::sin(angle);
    out[i] = static_cast<float>(radius * std::cos(angle));
    if (i + 1 < n) out[i + 1] = static_cast<float>(second);
  }
  return SKB_OK;
}

int skb_layer_create(const skb_config* cfg, const float* router, const float* const* gate,
                     const float* const* up, const float* const* down_t, const float* shared_gate,
                     const float* shared_up, const float* shared_down_t, int device,
                     skb_layer** out) {
  int rc = validate_cfg(cfg);
  if (rc) return rc;
  if (router == nullptr || gate == nullptr || up == nullptr || down_t == nullptr)
    return fail(SKB_ESHAPE, "layer_create: router/gate/up/down_t must be non-null");
  if (cfg->has_shared && (shared_gate == nullptr || shared_up == nullptr || shared_down_t == nullptr))
    return fail(SKB_ESHAPE, "layer_create: shared matrices missing while has_shared is set");
  skb_layer* L = nullptr;
  rc = new_layer(cfg, device, &L);
  if (rc) return rc;
  const Geometry& g = L->g;
  const int rmax = g.N > g.S ? g.N : g.S;
  float *sa = nullptr, *sb = nullptr;  // fp32 staging for one matrix pair
  const size_t mat = static_cast<size_t>(rmax) * g.D;
  if ((rc = dmalloc(&sa, mat)) || (rc = dmalloc(&sb, mat))) {
    if (sa) cudaFree(sa);
    skb_layer_destroy(L);
    return rc;
  }
  cudaError_t e = cudaMemcpyAsync(L->d_router, router, static_cast<size_t>(g.E) * g.D * 4,
                                  cudaMemcpyHostToDevice, L->stream);
  for (int ex = 0; ex < g.E && e == cudaSuccess; ++ex) {
    const size_t bytes = static_cast<size_t>(g.N) * g.D * 4;
    e = cudaMemcpyAsync(sa, gate[ex], bytes, cudaMemcpyHostToDevice, L->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(sb, up[ex], bytes, cudaMemcpyHostToDevice, L->stream);
    launch_pack_gateup(L->stream, sa, sb, g.N, g.D, g.Dp,
                       L->d_wgu + static_cast<size_t>(ex) * 2 * g.Np * g.Dp);
    if (L->d_wu)
      launch_pack_rows(L->stream, sb, g.N, g.D, g.Dp, L->d_wu + static_cast<size_t>(ex) * g.Np * g.Dp);
    if (e == cudaSuccess) e = cudaMemcpyAsync(sa, down_t[ex], bytes, cudaMemcpyHostToDevice, L->stream);
    launch_pack_rows(L->stream, sa, g.N, g.D, g.Dp, L->d_wd + static_cast<size_t>(ex) * g.Np * g.Dp);
    launch_pack_down_t(L->stream, sa, g.N, g.D, g.Np,
                       L->d_wdt + static_cast<size_t>(ex) * g.Dp128 * g.Np);
  }
  if (g.has_shared && e == cudaSuccess) {
    const size_t bytes = static_cast<size_t>(g.S) * g.D * 4;
    e = cudaMemcpyAsync(sa, shared_gate, bytes, cudaMemcpyHostToDevice, L->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(sb, shared_up, bytes, cudaMemcpyHostToDevice, L->stream);
    launch_pack_gateup(L->stream, sa, sb, g.S, g.D, g.Dp,
                       L->d_wgu + static_cast<size_t>(g.E) * 2 * g.Np * g.Dp);
    if (e == cudaSuccess) e = cudaMemcpyAsync(sa, shared_down_t, bytes, cudaMemcpyHostToDevice, L->stream);
    launch_pack_rows(L->stream, sa, g.S, g.D, g.Dp, L->d_wd_shared);
    launch_pack_down_t(L->stream, sa, g.S, g.D, g.Sp, L->d_wdt_shared);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(L->stream);
  if (e == cudaSuccess) e = cudaGetLastError();
  cudaFree(sa);
  cudaFree(sb);
  if (e != cudaSuccess) {
    skb_layer_destroy(L);
    return fail(SKB_ECUDA, "layer_create: upload failed: %s", cudaGetErrorString(e));
  }
  *out = L;
  return SKB_OK;
}

int skb_layer_create_synthetic(const skb_config* cfg, uint64_t seed, float scale, int device,
                               skb_layer** out) {
  int rc = validate_cfg(cfg);
  if (rc) return rc;
  if (!(scale > 0.0f)) return fail(SKB_ECONFIG, "scale must be > 0");  // model.cpp:132-134
  skb_layer* L = nullptr;
  rc = new_layer(cfg, device, &L);
  if (rc) return rc;
  const Geometry& g = L->g;
  const uint64_t ED = static_cast<uint64_t>(g.E) * g.D;
  const uint64_t ND = static_cast<uint64_t>(g.N) * g.D;
  const uint64_t SD = static_cast<uint64_t>(g.S) * g.D;
  launch_synth_f32(L->stream, seed, scale, 0, ED, L->d_router);
  for (int ex = 0; ex < g.E; ++ex) {
    const uint64_t base = ED + static_cast<uint64_t>(ex) * 3 * ND;
    launch_synth_gateup(L->stream, seed, scale, base, base + ND, g.N, g.Np, g.D, g.Dp,
                        L->d_wgu + static_cast<size_t>(ex) * 2 * g.Np * g.Dp);
    launch_synth_rows_bf16(L->stream, seed, scale, base + 2 * ND, g.N, g.Np, g.D, g.Dp,
                           L->d_wd + static_cast<size_t>(ex) * g.Np * g.Dp);
    if (L->d_wu)
      launch_synth_rows_bf16(L->stream, seed, scale, base + ND, g.N, g.Np, g.D, g.Dp,
                             L->d_wu + static_cast<size_t>(ex) * g.Np * g.Dp);
    launch_synth_down_t(L->stream, seed, scale, base + 2 * ND, g.N, g.D, g.Np,
                        L->d_wdt + static_cast<size_t>(ex) * g.Dp128 * g.Np);
  }
  if (g.has_shared) {
    const uint64_t base = ED + static_cast<uint64_t>(g.E) * 3 * ND;
    launch_synth_gateup(L->stream, seed, scale, base, base + SD, g.S, g.Sp, g.D, g.Dp,
                        L->d_wgu + static_cast<size_t>(g.E) * 2 * g.Np * g.Dp);
    launch_synth_rows_bf16(L->stream, seed, scale, base + 2 * SD, g.S, g.Sp, g.D, g.Dp,
                           L->d_wd_shared);
    launch_synth_down_t(L->stream, seed, scale, base + 2 * SD, g.S, g.D, g.Sp, L->d_wdt_shared);
  }
  cudaError_t e = cudaStreamSynchronize(L->stream);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    skb_layer_destroy(L);
    return fail(SKB_ECUDA, "layer_create_synthetic failed: %s", cudaGetErrorString(e));
  }
  *out = L;
  return SKB_OK;
}

int skb_layer_create_synthetic_slice(const skb_config* full, uint64_t seed, float scale, int e_lo,
                                     int e_hi, int which, int device, skb_layer** out) {
  int rc = validate_cfg(full);
  if (rc) return rc;
  if (!(scale > 0.0f)) return fail(SKB_ECONFIG, "scale must be > 0");
  if (which != 0 && which != 1) return fail(SKB_ECONFIG, "slice: which must be 0 or 1");
  if (which == 0 && (e_lo < 0 || e_hi <= e_lo || e_hi > full->n_experts))
    return fail(SKB_EINDEX, "slice: expert range [%d, %d) outside [0, %d)", e_lo, e_hi,
                full->n_experts);
  if (which == 1 && !full->has_shared)
    return fail(SKB_ECONFIG, "slice: the model has no shared expert");
  skb_config loc = *full;
  loc.n_experts = which == 0 ? e_hi - e_lo : 1;
  loc.top_k = 1;
  loc.d_ffn = which == 0 ? full->d_ffn : full->d_shared;
  loc.has_shared = 0;
  loc.d_shared = 0;
  skb_layer* L = nullptr;
  rc = new_layer(&loc, device, &L, full->n_experts, full->top_k);
  if (rc) return rc;
  const Geometry& g = L->g;
  const uint64_t ED = static_cast<uint64_t>(full->n_experts) * g.D;
  const uint64_t ND = static_cast<uint64_t>(full->d_ffn) * g.D;
  const uint64_t SD = static_cast<uint64_t>(full->d_shared) * g.D;
  launch_synth_f32(L->stream, seed, scale, 0, ED, L->d_router);
  for (int j = 0; j < g.E; ++j) {
    // draw offsets inside generate_synthetic's stream (model.cpp:129-166)
    uint64_t og, ou, od;
    if (which == 0) {
      const uint64_t base = ED + static_cast<uint64_t>(e_lo + j) * 3 * ND;
      og = base;
      ou = base + ND;
      od = base + 2 * ND;
    } else {
      const uint64_t base = ED + static_cast<uint64_t>(full->n_experts) * 3 * ND;
      og = base;
      ou = base + SD;
      od = base + 2 * SD;
    }
    launch_synth_gateup(L->stream, seed, scale, og, ou, g.N, g.Np, g.D, g.Dp,
                        L->d_wgu + static_cast<size_t>(j) * 2 * g.Np * g.Dp);
    launch_synth_rows_bf16(L->stream, seed, scale, od, g.N, g.Np, g.D, g.Dp,
                           L->d_wd + static_cast<size_t>(j) * g.Np * g.Dp);
    if (L->d_wu)
      launch_synth_rows_bf16(L->stream, seed, scale, ou, g.N, g.Np, g.D, g.Dp,
                             L->d_wu + static_cast<size_t>(j) * g.Np * g.Dp);
    launch_synth_down_t(L->stream, seed, scale, od, g.N, g.D, g.Np,
                        L->d_wdt + static_cast<size_t>(j) * g.Dp128 * g.Np);
  }
  cudaError_t e = cudaStreamSynchronize(L->stream);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    skb_layer_destroy(L);
    return fail(SKB_ECUDA, "layer_create_synthetic_slice failed: %s", cudaGetErrorString(e));
  }
  *out = L;
  return SKB_OK;
}

int skb_layer_set_router(skb_layer* L, const float* router, int n_experts, int top_k,
                         int renormalize) {
  if (L == nullptr || router == nullptr) return fail(SKB_EINTERNAL, "set_router: null argument");
  if (n_experts < 1 || top_k < 1 || top_k > n_experts)
    return fail(SKB_ECONFIG, "set_router: top_k must satisfy 1 <= K <= E, got K=%d E=%d", top_k,
                n_experts);
  if (n_experts > kMaxExperts)
    return fail(SKB_ECONFIG, "set_router: n_experts=%d exceeds the device router limit %d",
                n_experts, kMaxExperts);
  std::lock_guard<std::mutex> lk(L->mu);
  SKB_CUDA(cudaSetDevice(L->device));
  SKB_CUDA(cudaStreamSynchronize(L->stream));
  float* nr = nullptr;
  int rc = dmalloc(&nr, static_cast<size_t>(n_experts) * L->g.D);
  if (rc) return rc;
  SKB_CUDA(cudaMemcpy(nr, router, static_cast<size_t>(n_experts) * L->g.D * 4, cudaMemcpyHostToDevice));
  cudaFree(L->d_router);
  L->d_router = nr;
  L->route_E = n_experts;
  L->route_K = top_k;
  L->route_renorm = renormalize ? 1 : 0;
  free_workspace(L);  // logits / ids workspaces depend on the router shape
  return SKB_OK;
}

void skb_layer_destroy(skb_layer* L) {
  if (L == nullptr) return;
  cudaSetDevice(L->device);
  if (L->stream) cudaStreamSynchronize(L->stream);
  free_workspace(L);
  if (L->d_router) cudaFree(L->d_router);
  if (L->d_wgu) cudaFree(L->d_wgu);
  if (L->d_wd) cudaFree(L->d_wd);
  if (L->d_wu) cudaFree(L->d_wu);
  if (L->d_wdt) cudaFree(L->d_wdt);
  for (auto& ev : L->ev)
    if (ev) cudaEventDestroy(ev);
  if (L->stream) cudaStreamDestroy(L->stream);
  delete L;
}

int skb_layer_reserve(skb_layer* L, int max_batch) {
  if (L == nullptr) return fail(SKB_EINTERNAL, "layer is null");
  if (max_batch < 1) return fail(SKB_ESHAPE, "reserve: max_batch must be >= 1");
  std::lock_guard<std::mutex> lk(L->mu);
  return reserve_locked(L, max_batch);
}

int skb_layer_forward(skb_layer* L, const skb_forward_args* a, skb_report* report) {
  int rc = check_args(L, a);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(L->mu);
  SKB_CUDA(cudaSetDevice(L->device));
  rc = reserve_locked(L, a->batch);
  if (rc) return rc;
  const Geometry& g = L->g;
  const size_t B = a->batch, BK = B * g.K;
  cudaStream_t s = L->stream;
  SKB_CUDA(cudaMemcpyAsync(L->d_x, a->x, B * g.D * 4, cudaMemcpyHostToDevice, s));
  const uint8_t *mr = nullptr, *ms = nullptr;
  if (a->mode == SKB_MODE_MASKED) {
    SKB_CUDA(cudaMemcpyAsync(L->d_mask_in_r, a->routed_mask_in, BK * g.N, cudaMemcpyHostToDevice, s));
    mr = L->d_mask_in_r;
    if (a->shared_mask_len != 0 && g.has_shared) {
      SKB_CUDA(cudaMemcpyAsync(L->d_mask_in_s, a->shared_mask_in, B * g.S, cudaMemcpyHostToDevice, s));
      ms = L->d_mask_in_s;
    }
  }
  if (a->mode == SKB_MODE_TOPK && a->slot_n_off != nullptr)
    SKB_CUDA(cudaMemcpyAsync(L->d_slot_noff, a->slot_n_off, static_cast<size_t>(g.K) * 4,
                             cudaMemcpyHostToDevice, s));
  const bool timing = (a->flags & SKB_FLAG_TIME_STAGES) != 0;
  if (a->mode == SKB_MODE_ROUTE_ONLY) {
    rc = forward_core(L, a, L->d_x, nullptr, nullptr, nullptr, nullptr, nullptr, s, false);
    if (rc) return rc;
    const size_t rk = B * static_cast<size_t>(L->route_K);
    SKB_CUDA(cudaMemcpyAsync(a->ids_out, L->d_ids, rk * 4, cudaMemcpyDeviceToHost, s));
    SKB_CUDA(cudaMemcpyAsync(a->weights_out, L->d_wts, rk * 4, cudaMemcpyDeviceToHost, s));
    SKB_CUDA(cudaStreamSynchronize(s));
    if (report) std::memset(report, 0, sizeof(*report));
    return SKB_OK;
  }
  const int32_t* d_ids_in = nullptr;
  const float* d_w_in = nullptr;
  if (a->ids_in != nullptr) {
    for (size_t i = 0; i < BK; ++i)
      if (a->ids_in[i] < 0 || a->ids_in[i] >= g.E)
        return fail(SKB_EINDEX, "forward: external expert id %d outside [0, %d)", a->ids_in[i], g.E);
    // staged through the mask-input buffer's neighbours: ids/weights workspaces are the targets
    SKB_CUDA(cudaMemcpyAsync(L->d_ids_stage, a->ids_in, BK * 4, cudaMemcpyHostToDevice, s));
    d_ids_in = L->d_ids_stage;
    if (a->weights_in != nullptr) {
      SKB_CUDA(cudaMemcpyAsync(L->d_wts_stage, a->weights_in, BK * 4, cudaMemcpyHostToDevice, s));
      d_w_in = L->d_wts_stage;
    }
  }
  // Small pinned (page-locked, device-mapped) output buffers are written by the last kernel
  // directly: no device-to-host copy to launch and wait for after the layer (measured: OLMoE
  // shape batch 1, 75.1 -> 72.2 us end to end; at 1 MB the copy engine is faster than the
  // kernel's stores over PCIe, 166 vs 194 us, hence the size limit).
  float* y_target = L->d_y;
  if (B * g.D * 4 <= 64 * 1024) {
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, a->y) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
        pa.devicePointer != nullptr && (reinterpret_cast<uintptr_t>(pa.devicePointer) & 15) == 0)
      y_target = static_cast<float*>(pa.devicePointer);
    else
      cudaGetLastError();  // unregistered host memory reports an error on older drivers: not ours
  }
  rc = forward_core(L, a, L->d_x, y_target, mr, ms, a->routed_mask_out ? L->d_mask_out_r : nullptr,
                    (a->shared_mask_out && g.has_shared) ? L->d_mask_out_s : nullptr, s, timing,
                    d_ids_in, d_w_in, nullptr, nullptr,
                    a->h_routed_out != nullptr || a->h_shared_out != nullptr);
  if (rc) return rc;
  if (y_target == L->d_y)
    SKB_CUDA(cudaMemcpyAsync(a->y, L->d_y, B * g.D * 4, cudaMemcpyDeviceToHost, s));
  if (a->ids_out) SKB_CUDA(cudaMemcpyAsync(a->ids_out, L->d_ids, BK * 4, cudaMemcpyDeviceToHost, s));
  if (a->weights_out)
    SKB_CUDA(cudaMemcpyAsync(a->weights_out, L->d_wts, BK * 4, cudaMemcpyDeviceToHost, s));
  if (a->routed_mask_out)
    SKB_CUDA(cudaMemcpyAsync(a->routed_mask_out, L->d_mask_out_r, BK * g.N, cudaMemcpyDeviceToHost, s));
  if (a->shared_mask_out && g.has_shared)
    SKB_CUDA(cudaMemcpyAsync(a->shared_mask_out, L->d_mask_out_s, B * g.S, cudaMemcpyDeviceToHost, s));
  std::vector<int32_t> kcnt_host, inv_host;
  if (a->mode == SKB_MODE_THRESHOLD) {
    kcnt_host.resize(BK + (g.has_shared ? B : 0));
    inv_host.resize(BK);
    SKB_CUDA(cudaMemcpyAsync(kcnt_host.data(), L->d_kcnt, kcnt_host.size() * 4, cudaMemcpyDeviceToHost, s));
    SKB_CUDA(cudaMemcpyAsync(inv_host.data(), L->disp.inv, BK * 4, cudaMemcpyDeviceToHost, s));
  }
  std::vector<float> hbuf;
  std::vector<int32_t> inv;
  if (a->h_routed_out || (a->h_shared_out && g.has_shared)) {
    const size_t rows = BK + (g.has_shared ? B : 0);
    hbuf.resize(rows * g.Nh);
    inv.resize(BK);
    SKB_CUDA(cudaMemcpyAsync(hbuf.data(), L->d_h, rows * g.Nh * 4, cudaMemcpyDeviceToHost, s));
    SKB_CUDA(cudaMemcpyAsync(inv.data(), L->disp.inv, BK * 4, cudaMemcpyDeviceToHost, s));
  }
  SKB_CUDA(cudaStreamSynchronize(s));
  if (a->h_routed_out)
    for (size_t i = 0; i < BK; ++i)
      std::memcpy(a->h_routed_out + i * g.N, hbuf.data() + static_cast<size_t>(inv[i]) * g.Nh,
                  static_cast<size_t>(g.N) * 4);
  if (a->h_shared_out && g.has_shared)
    for (size_t t = 0; t < B; ++t)
      std::memcpy(a->h_shared_out + t * g.S, hbuf.data() + (BK + t) * g.Nh,
                  static_cast<size_t>(g.S) * 4);
  if (timing) L->stage_ms_pending = true;
  if (a->mode == SKB_MODE_THRESHOLD)
    fill_report_threshold(L, a, report, kcnt_host.data(), inv_host.data());
  else
    fill_report(L, a, report, a->routed_mask_in,
                (a->shared_mask_len != 0) ? a->shared_mask_in : nullptr);
  return SKB_OK;
}

int skb_layer_forward_device(skb_layer* L, const skb_forward_args* a, void* stream,
                             skb_report* report) {
  int rc = check_args(L, a);
  if (rc) return rc;
  if (a->batch > L->cap_batch)
    return fail(SKB_ESHAPE, "forward_device: batch %d exceeds reserved capacity %d; call skb_layer_reserve",
                a->batch, L->cap_batch);
  if (a->mode == SKB_MODE_TOPK && a->slot_n_off != nullptr)
    return fail(SKB_ECONFIG, "forward_device: per-slot neuron budgets need skb_layer_forward");
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : L->stream;
  const bool timing = (a->flags & SKB_FLAG_TIME_STAGES) != 0;
  rc = forward_core(L, a, a->x, a->y, a->mode == SKB_MODE_MASKED ? a->routed_mask_in : nullptr,
                    (a->mode == SKB_MODE_MASKED && a->shared_mask_len) ? a->shared_mask_in : nullptr,
                    nullptr, nullptr, s, timing, a->ids_in, a->weights_in,
                    a->mode == SKB_MODE_ROUTE_ONLY ? a->ids_out : nullptr,
                    a->mode == SKB_MODE_ROUTE_ONLY ? a->weights_out : nullptr);
  if (rc) return rc;
  if (timing) L->stage_ms_pending = true;
  if (a->mode == SKB_MODE_THRESHOLD)
    fill_report_threshold(L, a, report, nullptr, nullptr);  // data-dependent fields need the host entry
  else if (a->mode != SKB_MODE_ROUTE_ONLY)
    fill_report(L, a, report, nullptr, nullptr);
  return SKB_OK;
}

int skb_layer_forward_device_rows(skb_layer* L, const skb_forward_args* a, void* stream,
                                  float* const* y_rows) {
  int rc = check_args(L, a, /*y_elsewhere=*/true);
  if (rc) return rc;
  if (y_rows == nullptr) return fail(SKB_EINTERNAL, "forward_device_rows: y_rows is null");
  if (a->batch > L->cap_batch)
    return fail(SKB_ESHAPE, "forward_device_rows: batch %d exceeds reserved capacity %d; call skb_layer_reserve",
                a->batch, L->cap_batch);
  if (a->mode != SKB_MODE_TOPK && a->mode != SKB_MODE_DENSE)
    return fail(SKB_ECONFIG, "forward_device_rows: dense and top-k modes only");
  if (a->mode == SKB_MODE_TOPK && a->slot_n_off != nullptr)
    return fail(SKB_ECONFIG, "forward_device_rows: per-slot neuron budgets need skb_layer_forward");
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : L->stream;
  return forward_core(L, a, a->x, nullptr, nullptr, nullptr, nullptr, nullptr, s, false, a->ids_in,
                      a->weights_in, nullptr, nullptr, false, y_rows);
}

int skb_layer_stage_times(skb_layer* L, float* ms) {
  if (L == nullptr || ms == nullptr) return fail(SKB_EINTERNAL, "stage_times: null argument");
  if (L->stage_ms_pending) {
    // waits for the last stage of the timed forward (the device entry point does not synchronise)
    SKB_CUDA(cudaEventSynchronize(L->ev[SKB_N_STAGES]));
    for (int i = 0; i < SKB_N_STAGES; ++i)
      SKB_CUDA(cudaEventElapsedTime(&L->stage_ms[i], L->ev[i], L->ev[i + 1]));
    L->stage_ms_pending = false;
    L->have_stage_ms = true;
  }
  if (!L->have_stage_ms) return fail(SKB_EINTERNAL, "stage_times: no timed forward yet");
  std::memcpy(ms, L->stage_ms, sizeof(L->stage_ms));
  return SKB_OK;
}

int skb_layer_last_launches(skb_layer* L) { return L ? L->last_launches : 0; }
uint64_t skb_layer_weight_bytes(skb_layer* L) { return L ? L->weight_bytes : 0; }

// ---- stage entry points ----------------------------------------------------------------------

static int stage_device_ready() {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
    cudaGetLastError();
    return fail(SKB_ECUDA, "no CUDA device: this library has no CPU path");
  }
  return SKB_OK;
}

int skb_route(const float* logits, int batch, int n_experts, int top_k, int renormalize,
              int32_t* ids, float* weights) {
  if (batch < 1) return fail(SKB_ESHAPE, "route: empty batch");
  if (top_k < 1 || top_k > n_experts)
    return fail(SKB_ECONFIG, "route: top_k=%d outside [1, %d]", top_k, n_experts);
  if (n_experts > kMaxExperts)
    return fail(SKB_ECONFIG, "route: n_experts=%d exceeds the device router limit %d", n_experts,
                kMaxExperts);
  if (logits == nullptr || ids == nullptr || weights == nullptr)
    return fail(SKB_ESHAPE, "route: null buffer");
  int rc = stage_device_ready();
  if (rc) return rc;
  const size_t BE = static_cast<size_t>(batch) * n_experts, BK = static_cast<size_t>(batch) * top_k;
  float *dl = nullptr, *dw = nullptr;
  int32_t* di = nullptr;
  unsigned* dc = nullptr;
  const size_t n_counters = 2 + static_cast<size_t>(batch);
  if ((rc = dmalloc(&dl, BE)) || (rc = dmalloc(&dw, BK)) || (rc = dmalloc(&di, BK)) ||
      (rc = dmalloc(&dc, n_counters)))
    return rc;
  cudaMemcpy(dl, logits, BE * 4, cudaMemcpyHostToDevice);
  cudaMemset(dc, 0, n_counters * sizeof(unsigned));
  LaunchCtx ctx{nullptr, false};
  RouterLaunch r{};
  r.B = batch;
  r.E = n_experts;
  r.K = top_k;
  r.renorm = renormalize;
  r.logits = dl;
  r.ids = di;
  r.weights = dw;
  r.counters = dc;
  launch_router(ctx, r);
  cudaMemcpy(ids, di, BK * 4, cudaMemcpyDeviceToHost);
  cudaError_t e = cudaMemcpy(weights, dw, BK * 4, cudaMemcpyDeviceToHost);
  cudaFree(dl);
  cudaFree(dw);
  cudaFree(di);
  cudaFree(dc);
  if (e != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess)
    return fail(SKB_ECUDA, "route: %s", cudaGetErrorString(e));
  return SKB_OK;
}

int skb_align_dispatch(const int32_t* ids, int batch, int top_k, int n_experts, int block,
                       int32_t* sorted_out, int32_t* expert_of_block, int32_t* n_padded,
                       int32_t* n_blocks) {
  if (block < 1) return fail(SKB_ECONFIG, "align_dispatch: block must be >= 1");
  if (batch < 0 || top_k < 1 || n_experts < 1 || n_experts > kMaxExperts)
    return fail(SKB_ESHAPE, "align_dispatch: bad shape");
  const size_t BK = static_cast<size_t>(batch) * top_k;
  for (size_t i = 0; i < BK; ++i)
    if (ids[i] < 0 || ids[i] >= n_experts)
      return fail(SKB_EINDEX, "align_dispatch: expert id %d outside [0, %d)", ids[i], n_experts);
  int rc = stage_device_ready();
  if (rc) return rc;
  DispatchBuffers d{};
  int32_t *dids = nullptr, *dsorted = nullptr, *deob = nullptr, *dcounts = nullptr;
  const size_t cap = BK + static_cast<size_t>(n_experts) * (block - 1) + 1;
  const size_t max_tiles = static_cast<size_t>(n_experts) + BK / 16 + 2;
  if ((rc = dmalloc(&dids, BK)) || (rc = dmalloc(&d.perm, BK)) || (rc = dmalloc(&d.inv, BK)) ||
      (rc = dmalloc(&d.row_expert, BK)) || (rc = dmalloc(&d.expert_off, (size_t)n_experts + 2)) ||
      (rc = dmalloc(&d.tile_expert, max_tiles)) || (rc = dmalloc(&d.tile_row0, max_tiles)) ||
      (rc = dmalloc(&d.tile_nrows, max_tiles)) || (rc = dmalloc(&d.n_tiles, 1)) ||
      (rc = dmalloc(&dsorted, cap)) || (rc = dmalloc(&deob, cap)) || (rc = dmalloc(&dcounts, 2)))
    return rc;
  cudaMemcpy(dids, ids, BK * 4, cudaMemcpyHostToDevice);
  LaunchCtx ctx{nullptr, false};
  launch_dispatch(ctx, dids, batch, top_k, n_experts, 0, 16, d);
  launch_plan_export(ctx, d.perm, d.expert_off, n_experts, block, dsorted, deob, dcounts);
  int32_t counts[2] = {0, 0};
  cudaError_t e = cudaMemcpy(counts, dcounts, 8, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && counts[0] > 0)
    e = cudaMemcpy(sorted_out, dsorted, static_cast<size_t>(counts[0]) * 4, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && counts[1] > 0)
    e = cudaMemcpy(expert_of_block, deob, static_cast<size_t>(counts[1]) * 4, cudaMemcpyDeviceToHost);
  void* ptrs[] = {dids, d.perm, d.inv, d.row_expert, d.expert_off, d.tile_expert, d.tile_row0,
                  d.tile_nrows, d.n_tiles, dsorted, deob, dcounts};
  for (void* p : ptrs) cudaFree(p);
  if (e != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess)
    return fail(SKB_ECUDA, "align_dispatch: %s", cudaGetErrorString(e));
  *n_padded = counts[0];
  *n_blocks = counts[1];
  return SKB_OK;
}

int skb_combine(const float* slot_outputs, const float* weights, int batch, int top_k, int d_model,
                float* y) {
  if (batch < 1 || top_k < 1 || d_model < 1) return fail(SKB_ESHAPE, "combine: bad shape");
  int rc = stage_device_ready();
  if (rc) return rc;
  const size_t BK = static_cast<size_t>(batch) * top_k;
  float *ds = nullptr, *dw = nullptr, *dy = nullptr;
  if ((rc = dmalloc(&ds, BK * d_model)) || (rc = dmalloc(&dw, BK)) ||
      (rc = dmalloc(&dy, static_cast<size_t>(batch) * d_model)))
    return rc;
  cudaMemcpy(ds, slot_outputs, BK * d_model * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dw, weights, BK * 4, cudaMemcpyHostToDevice);
  LaunchCtx ctx{nullptr, false};
  launch_combine_slots(ctx, ds, dw, batch, top_k, d_model, dy);
  cudaError_t e = cudaMemcpy(y, dy, static_cast<size_t>(batch) * d_model * 4, cudaMemcpyDeviceToHost);
  cudaFree(ds);
  cudaFree(dw);
  cudaFree(dy);
  if (e != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess)
    return fail(SKB_ECUDA, "combine: %s", cudaGetErrorString(e));
  return SKB_OK;
}

int skb_mask_smallest(const float* h, int rows, int n, const int32_t* counts, uint8_t* mask,
                      int32_t* kept_idx, int32_t* kept_count) {
  if (rows < 1 || n < 1) return fail(SKB_ESHAPE, "mask_smallest: rows and n must be >= 1");
  if (h == nullptr || counts == nullptr || mask == nullptr)
    return fail(SKB_ESHAPE, "mask_smallest: null buffer");
  int rc = stage_device_ready();
  if (rc) return rc;
  const size_t total = static_cast<size_t>(rows) * n;
  float* dh = nullptr;
  int32_t *dc = nullptr, *dki = nullptr, *dkc = nullptr;
  uint8_t* dm = nullptr;
  if ((rc = dmalloc(&dh, total)) || (rc = dmalloc(&dc, (size_t)rows)) || (rc = dmalloc(&dki, total)) ||
      (rc = dmalloc(&dkc, (size_t)rows)) || (rc = dmalloc(&dm, total)))
    return rc;
  cudaMemcpy(dh, h, total * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dc, counts, static_cast<size_t>(rows) * 4, cudaMemcpyHostToDevice);
  cudaMemset(dki, 0xFF, total * 4);
  SelectArgs sa{};
  sa.h = dh;
  sa.rows = rows;
  sa.BK = rows;
  sa.N = n;
  sa.S = 0;
  sa.Nh = n;
  sa.K = 1;
  sa.mode = kSelectTopk;
  sa.counts = dc;
  sa.mask_out_routed = dm;
  sa.kept_idx = dki;
  sa.kept_cnt = dkc;
  LaunchCtx ctx{nullptr, false};
  launch_select(ctx, sa);
  cudaError_t e = cudaMemcpy(mask, dm, total, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && kept_idx) e = cudaMemcpy(kept_idx, dki, total * 4, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && kept_count)
    e = cudaMemcpy(kept_count, dkc, static_cast<size_t>(rows) * 4, cudaMemcpyDeviceToHost);
  cudaFree(dh);
  cudaFree(dc);
  cudaFree(dki);
  cudaFree(dkc);
  cudaFree(dm);
  if (e != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess)
    return fail(SKB_ECUDA, "mask_smallest: %s", cudaGetErrorString(e));
  return SKB_OK;
}

int skb_threshold_mask(const float* gate_raw, int rows, int n, float tau, uint8_t* mask) {
  if (!(tau >= 0.0f)) return fail(SKB_ECONFIG, "threshold must be >= 0");
  if (rows < 0 || n < 0) return fail(SKB_ESHAPE, "threshold_mask: negative size");
  const size_t total = static_cast<size_t>(rows) * n;
  if (total == 0) return SKB_OK;
  if (gate_raw == nullptr || mask == nullptr) return fail(SKB_ESHAPE, "threshold_mask: null buffer");
  int rc = stage_device_ready();
  if (rc) return rc;
  float* dg = nullptr;
  uint8_t* dm = nullptr;
  if ((rc = dmalloc(&dg, total)) || (rc = dmalloc(&dm, total))) return rc;
  cudaMemcpy(dg, gate_raw, total * 4, cudaMemcpyHostToDevice);
  launch_threshold_mask(nullptr, dg, total, tau, dm);
  cudaError_t e = cudaMemcpy(mask, dm, total, cudaMemcpyDeviceToHost);
  cudaFree(dg);
  cudaFree(dm);
  if (e != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess)
    return fail(SKB_ECUDA, "threshold_mask: %s", cudaGetErrorString(e));
  return SKB_OK;
}

int skb_default_capacity(int top_k, int d_ffn) { return (top_k * d_ffn + 31) / 32 * 32; }

int skb_compact_active(const uint8_t* masks, uint64_t masks_len, const int32_t* topk_ids, int batch,
                       int top_k, int d_ffn, int capacity, int32_t* flat, int32_t* active_per_slot,
                       int32_t* total_active) {
  if (capacity < 0) return fail(SKB_ECONFIG, "compact_active: capacity must be >= 0");
  if (batch < 0 || top_k < 0 || d_ffn < 0) return fail(SKB_ESHAPE, "compact_active: negative size");
  const size_t slots = static_cast<size_t>(batch) * top_k;
  if (masks_len != slots * static_cast<size_t>(d_ffn))
    return fail(SKB_ESHAPE, "compact_active: mask size %llu != slots * d_ffn",
                static_cast<unsigned long long>(masks_len));
  if (batch == 0) return SKB_OK;
  int rc = stage_device_ready();
  if (rc) return rc;
  uint8_t* dm = nullptr;
  int32_t *di = nullptr, *df = nullptr, *dp = nullptr, *dt = nullptr;
  const size_t fl = static_cast<size_t>(batch) * (capacity > 0 ? capacity : 1);
  if ((rc = dmalloc(&dm, masks_len ? masks_len : 1)) || (rc = dmalloc(&di, slots ? slots : 1)) ||
      (rc = dmalloc(&df, fl)) || (rc = dmalloc(&dp, slots ? slots : 1)) ||
      (rc = dmalloc(&dt, static_cast<size_t>(batch))))
    return rc;
  if (masks_len) cudaMemcpy(dm, masks, masks_len, cudaMemcpyHostToDevice);
  if (slots) cudaMemcpy(di, topk_ids, slots * 4, cudaMemcpyHostToDevice);
  launch_compact_active(nullptr, dm, di, batch, top_k, d_ffn, capacity, df, dp, dt);
  cudaError_t e = cudaSuccess;
  if (capacity > 0)
    e = cudaMemcpy(flat, df, static_cast<size_t>(batch) * capacity * 4, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && slots) e = cudaMemcpy(active_per_slot, dp, slots * 4, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess)
    e = cudaMemcpy(total_active, dt, static_cast<size_t>(batch) * 4, cudaMemcpyDeviceToHost);
  cudaFree(dm);
  cudaFree(di);
  cudaFree(df);
  cudaFree(dp);
  cudaFree(dt);
  if (e != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess)
    return fail(SKB_ECUDA, "compact_active: %s", cudaGetErrorString(e));
  return SKB_OK;
}

int skb_topk_mask(const float* h, int rows, int n, double s, uint8_t* mask) {
  if (!(s >= 0.0 && s <= 1.0)) return fail(SKB_ECONFIG, "sparsity must lie in [0, 1]");
  if (rows < 1 || n < 1) return fail(SKB_ESHAPE, "topk_mask: rows and n must be >= 1");
  std::vector<int32_t> counts(static_cast<size_t>(rows), n_off_of(s, n));
  return skb_mask_smallest(h, rows, n, counts.data(), mask, nullptr, nullptr);
}

}  // extern "C"
