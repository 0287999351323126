// down.cu -- subsystem (4): the down projection as a gather over the surviving W_down rows,
// plus the router-weighted combine.  Only rows named in the survivor list are ever addressed,
// so dropped neurons cost no HBM bytes.
//
// Replaces gathered_matvec_t (proj/src/linalg.cpp:56-81), combine (proj/src/router.cpp:109-132)
// and the shared-expert accumulation (proj/src/engine.cpp:55-84).
//
// Reduction tree (fixed, independent of batch size and grid shape, no float atomics):
//   micro-chunk  16 consecutive survivors, accumulated in ascending order by one warp
//   chunk        8 micro-chunks (128 survivors) summed in ascending order -> one partial row
//   slot output  partial rows summed in ascending chunk order
//   y[t]         slots ascending, weight * slot output (multiply and add rounded separately,
//                as router.cpp:119-130 does), then the shared expert's output last
//                (engine.cpp:168-173).
#include "skb_internal.cuh"

namespace skb {

namespace {

__device__ __forceinline__ uint4 ldg_stream_16B(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void fma_bf16x8(const uint4& w, float hk, float (&acc)[8]) {
  const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    // bf16 -> fp32 is a 16-bit shift
    acc[2 * i] = fmaf(__uint_as_float(u[i] << 16), hk, acc[2 * i]);
    acc[2 * i + 1] = fmaf(__uint_as_float(u[i] & 0xffff0000u), hk, acc[2 * i + 1]);
  }
}

constexpr int kDownWarps = 8;
constexpr int kMicro = kDownChunk / kDownWarps;  // 16 survivors per warp

}  // namespace

// grid (chunk, column segment, row); 256 threads.  Warp w handles survivors
// [chunk*128 + 16w, +16) of `row` for the 256 columns of the segment (16 B per lane per row).
__global__ void __launch_bounds__(256) gather_down_kernel(DownArgs a, int E, int Np, int Dp,
                                                          int Nh) {
  __shared__ float red[kDownWarps][kDownSeg];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int chunk = blockIdx.x, seg = blockIdx.y, row = blockIdx.z;

  pdl_wait();
  pdl_launch_dependents();

  const int cnt = a.kept_cnt[row];
  const int k0 = chunk * kDownChunk;
  if (k0 >= cnt) return;
  const int e = a.row_expert[row];
  const __nv_bfloat16* w =
      (e < E) ? a.wd + static_cast<size_t>(e) * Np * Dp : a.wd_shared;
  const int col = seg * kDownSeg + lane * 8;
  const bool col_ok = col < Dp;

  const int kb = k0 + warp * kMicro;
  int my_idx = 0;
  float my_h = 0.0f;
  if (lane < kMicro && kb + lane < cnt) {
    my_idx = a.kept_idx[static_cast<size_t>(row) * Nh + kb + lane];
    my_h = a.kept_val[static_cast<size_t>(row) * Nh + kb + lane];
  }
  const int m = min(kMicro, cnt - kb);  // survivors in this micro-chunk (<= 0: none)

  float acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.0f;

  uint4 wv[kMicro];
#pragma unroll
  for (int j = 0; j < kMicro; ++j) {
    const int idx = __shfl_sync(0xffffffffu, my_idx, j);
    wv[j] = make_uint4(0u, 0u, 0u, 0u);
    if (j < m && col_ok) wv[j] = ldg_stream_16B(w + static_cast<size_t>(idx) * Dp + col);
  }
#pragma unroll
  for (int j = 0; j < kMicro; ++j) {
    const float hk = __shfl_sync(0xffffffffu, my_h, j);
    if (j < m) fma_bf16x8(wv[j], hk, acc);
  }

#pragma unroll
  for (int i = 0; i < 8; ++i) red[warp][lane * 8 + i] = acc[i];
  __syncthreads();
  const int c = seg * kDownSeg + tid;
  if (c < Dp) {
    float s = red[0][tid];
#pragma unroll
    for (int wq = 1; wq < kDownWarps; ++wq) s = __fadd_rn(s, red[wq][tid]);
    a.partial[(static_cast<size_t>(row) * a.n_chunks + chunk) * Dp + c] = s;
  }
}

int launch_down(const LaunchCtx& ctx, const DownArgs& a, const Geometry& g) {
  if (a.max_keep <= 0 || a.rows <= 0) return 0;
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = ctx.pdl ? 1 : 0;
  cfg.stream = ctx.stream;
  cfg.gridDim = dim3(ceil_div(a.max_keep, kDownChunk), ceil_div(g.Dp, kDownSeg), a.rows);
  cfg.blockDim = dim3(256);
  cudaLaunchKernelEx(&cfg, gather_down_kernel, a, g.E, g.Np, g.Dp, g.Nh);
  return 1;
}

// y[t][d]: chunks ascending per slot, slots ascending with router weights, shared expert last.
__global__ void __launch_bounds__(256) combine_kernel(const float* __restrict__ partial,
                                                      int n_chunks, const int32_t* __restrict__ inv,
                                                      const int32_t* __restrict__ kept_cnt,
                                                      const float* __restrict__ weights, int B,
                                                      int K, int D, int Dp, int has_shared,
                                                      float* __restrict__ y) {
  pdl_wait();
  pdl_launch_dependents();
  const int t = blockIdx.y;
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= D) return;
  float acc = 0.0f;
  for (int s = 0; s <= K; ++s) {
    int row;
    float wgt = 1.0f;
    if (s < K) {
      row = inv[t * K + s];
      wgt = weights[t * K + s];
    } else {
      if (!has_shared) break;
      row = B * K + t;
    }
    const int nch = ceil_div(kept_cnt[row], kDownChunk);
    const float* p = partial + static_cast<size_t>(row) * n_chunks * Dp + d;
    float o = 0.0f;
    for (int c = 0; c < nch; ++c) o = __fadd_rn(o, p[static_cast<size_t>(c) * Dp]);
    acc = (s < K) ? __fadd_rn(acc, __fmul_rn(wgt, o)) : __fadd_rn(acc, o);
  }
  y[static_cast<size_t>(t) * D + d] = acc;
}

int launch_combine(const LaunchCtx& ctx, const float* partial, int n_chunks, const int32_t* inv,
                   const int32_t* kept_cnt, const float* weights, int B, const Geometry& g,
                   float* y) {
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = ctx.pdl ? 1 : 0;
  cfg.stream = ctx.stream;
  cfg.gridDim = dim3(ceil_div(g.D, 256), B);
  cfg.blockDim = dim3(256);
  cudaLaunchKernelEx(&cfg, combine_kernel, partial, n_chunks, inv, kept_cnt, weights, B, g.K, g.D,
                     g.Dp, g.has_shared, y);
  return 1;
}

}  // namespace skb
