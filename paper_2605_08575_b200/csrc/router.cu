// router.cu -- subsystem (1): router logits, softmax + warp-level top-k, counting sort by
// expert (token permutation) and the tile list the grouped GEMM walks.
//
// Reference behaviour reproduced here:
//   route_logits / matvec   proj/src/engine.cpp:43-53, proj/src/linalg.cpp:22-40
//   route                   proj/src/router.cpp:13-68
//   align_dispatch          proj/src/router.cpp:70-107
#include "skb_internal.cuh"

namespace skb {

// ---------------------------------------------------------------------------------------------
// Router logits, order-faithful: logits[t][e] = sum_d router[e][d] * x[t][d] with a float
// accumulator, d ascending, multiply and add rounded separately (the reference is built with
// -ffp-contract=off, proj/CMakeLists.txt:26-27).  One thread per expert, TT tokens per CTA so
// that TT independent dependent-add chains fill the 4-cycle FADD latency.
// ---------------------------------------------------------------------------------------------
constexpr int kLogitChunk = 1024;

template <int TT>
__global__ void __launch_bounds__(1024) router_logits_exact_kernel(const float* __restrict__ x,
                                                                  const float* __restrict__ router,
                                                                  int B, int E, int D,
                                                                  float* __restrict__ logits) {
  __shared__ float xs[TT][kLogitChunk];
  const int e = threadIdx.x;
  const int t0 = blockIdx.x * TT;
  float acc[TT];
#pragma unroll
  for (int tt = 0; tt < TT; ++tt) acc[tt] = 0.0f;
  pdl_wait();
  pdl_launch_dependents();
  const bool vec_ok = (D % 4) == 0;
  for (int d0 = 0; d0 < D; d0 += kLogitChunk) {
    const int len = min(kLogitChunk, D - d0);
    __syncthreads();
#pragma unroll
    for (int tt = 0; tt < TT; ++tt) {
      const int t = t0 + tt;
      for (int i = threadIdx.x; i < len; i += blockDim.x)
        xs[tt][i] = (t < B) ? x[static_cast<size_t>(t) * D + d0 + i] : 0.0f;
    }
    __syncthreads();
    if (e < E) {
      const float* wr = router + static_cast<size_t>(e) * D + d0;
      int i = 0;
      if (vec_ok) {
        const float4* wr4 = reinterpret_cast<const float4*>(wr);
        const int n4 = len / 4;
#pragma unroll 4
        for (int q = 0; q < n4; ++q) {
          const float4 w = __ldg(wr4 + q);
#pragma unroll
          for (int tt = 0; tt < TT; ++tt) {
            const float4 xv = *reinterpret_cast<const float4*>(&xs[tt][4 * q]);
            acc[tt] = __fadd_rn(acc[tt], __fmul_rn(w.x, xv.x));
            acc[tt] = __fadd_rn(acc[tt], __fmul_rn(w.y, xv.y));
            acc[tt] = __fadd_rn(acc[tt], __fmul_rn(w.z, xv.z));
            acc[tt] = __fadd_rn(acc[tt], __fmul_rn(w.w, xv.w));
          }
        }
        i = n4 * 4;
      }
      for (; i < len; ++i) {
        const float w = __ldg(wr + i);
#pragma unroll
        for (int tt = 0; tt < TT; ++tt) acc[tt] = __fadd_rn(acc[tt], __fmul_rn(w, xs[tt][i]));
      }
    }
  }
  if (e < E) {
#pragma unroll
    for (int tt = 0; tt < TT; ++tt)
      if (t0 + tt < B) logits[static_cast<size_t>(t0 + tt) * E + e] = acc[tt];
  }
}

// Fast variant (SKB_FLAG_FAST_ROUTER): one warp per (token, expert), lanes stride d, fp32 FMA,
// shuffle tree.  Not order-faithful: ids can differ from the reference when two probabilities
// sit within float summation noise of each other.
__global__ void __launch_bounds__(256) router_logits_fast_kernel(const float* __restrict__ x,
                                                                 const float* __restrict__ router,
                                                                 int B, int E, int D,
                                                                 float* __restrict__ logits) {
  pdl_wait();
  pdl_launch_dependents();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= B * E) return;
  const int t = warp / E, e = warp % E;
  const float* xr = x + static_cast<size_t>(t) * D;
  const float* wr = router + static_cast<size_t>(e) * D;
  float acc = 0.0f;
  if ((D % 4) == 0) {
    const float4* x4 = reinterpret_cast<const float4*>(xr);
    const float4* w4 = reinterpret_cast<const float4*>(wr);
    for (int q = lane; q < D / 4; q += 32) {
      const float4 a = __ldg(w4 + q), b = __ldg(x4 + q);
      acc = fmaf(a.x, b.x, acc);
      acc = fmaf(a.y, b.y, acc);
      acc = fmaf(a.z, b.z, acc);
      acc = fmaf(a.w, b.w, acc);
    }
  } else {
    for (int d = lane; d < D; d += 32) acc = fmaf(__ldg(wr + d), __ldg(xr + d), acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) logits[static_cast<size_t>(t) * E + e] = acc;
}

int launch_router_logits(const LaunchCtx& ctx, const float* x, const float* router, int B, int E,
                         int D, bool fast, float* logits) {
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = ctx.pdl ? 1 : 0;
  cfg.stream = ctx.stream;
  if (fast) {
    const long warps = static_cast<long>(B) * E;
    cfg.gridDim = dim3(static_cast<unsigned>((warps * 32 + 255) / 256));
    cfg.blockDim = dim3(256);
    cudaLaunchKernelEx(&cfg, router_logits_fast_kernel, x, router, B, E, D, logits);
    return 1;
  }
  cfg.blockDim = dim3(round_up(E, 32));
  if (B == 1) {
    cfg.gridDim = dim3(1);
    cudaLaunchKernelEx(&cfg, router_logits_exact_kernel<1>, x, router, B, E, D, logits);
  } else {
    cfg.gridDim = dim3(ceil_div(B, 2));
    cudaLaunchKernelEx(&cfg, router_logits_exact_kernel<2>, x, router, B, E, D, logits);
  }
  return 1;
}

// ---------------------------------------------------------------------------------------------
// route(): one warp per token.  Softmax with max subtraction, exp evaluated in double and
// rounded to float (what glibc's expf does internally), ascending float sum for the
// denominator, IEEE division, then K rounds of warp arg-max under the reference's total order
// (probability descending, expert id ascending on ties).
// ---------------------------------------------------------------------------------------------
template <int EPL>  // experts per lane, E <= 32 * EPL
__global__ void __launch_bounds__(128) route_topk_kernel(const float* __restrict__ logits, int B,
                                                         int E, int K, int renorm,
                                                         int32_t* __restrict__ ids,
                                                         float* __restrict__ weights) {
  extern __shared__ float smem_probs[];  // [warps][E]
  const int warp_in_block = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * (blockDim.x >> 5) + warp_in_block;
  pdl_wait();
  pdl_launch_dependents();
  if (t >= B) return;
  float* ex_s = smem_probs + static_cast<size_t>(warp_in_block) * E;
  const float* row = logits + static_cast<size_t>(t) * E;

  float l[EPL];
  float mx = -INFINITY;
#pragma unroll
  for (int j = 0; j < EPL; ++j) {
    const int e = j * 32 + lane;
    l[j] = (e < E) ? row[e] : -INFINITY;
    mx = fmaxf(mx, l[j]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));

  float p[EPL];
#pragma unroll
  for (int j = 0; j < EPL; ++j) {
    const int e = j * 32 + lane;
    if (e < E) {
      p[j] = static_cast<float>(exp(static_cast<double>(__fsub_rn(l[j], mx))));
      ex_s[e] = p[j];
    } else {
      p[j] = 0.0f;
    }
  }
  __syncwarp();
  float denom = 0.0f;
  if (lane == 0) {
    for (int e = 0; e < E; ++e) denom = __fadd_rn(denom, ex_s[e]);
  }
  denom = __shfl_sync(0xffffffffu, denom, 0);
#pragma unroll
  for (int j = 0; j < EPL; ++j) {
    const int e = j * 32 + lane;
    p[j] = (e < E) ? __fdiv_rn(p[j], denom) : -2.0f;
  }

  int32_t* out_ids = ids + static_cast<size_t>(t) * K;
  float* out_w = weights + static_cast<size_t>(t) * K;
  float selected_sum = 0.0f;
  for (int s = 0; s < K; ++s) {
    float bp = -3.0f;
    int be = 0x7fffffff;
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      if (p[j] > bp) {  // j ascending => lowest id kept on equal probability
        bp = p[j];
        be = j * 32 + lane;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float op = __shfl_xor_sync(0xffffffffu, bp, o);
      const int oe = __shfl_xor_sync(0xffffffffu, be, o);
      if (op > bp || (op == bp && oe < be)) {
        bp = op;
        be = oe;
      }
    }
#pragma unroll
    for (int j = 0; j < EPL; ++j)
      if (j * 32 + lane == be) p[j] = -1.0f;  // selected: never wins again (probabilities >= 0)
    selected_sum = __fadd_rn(selected_sum, bp);
    if (lane == 0) {
      out_ids[s] = be;
      out_w[s] = bp;
    }
  }
  __syncwarp();
  if (renorm) {
    for (int s = lane; s < K; s += 32) out_w[s] = __fdiv_rn(out_w[s], selected_sum);
  }
}

int launch_route_topk(const LaunchCtx& ctx, const float* logits, int B, int E, int K, int renorm,
                      int32_t* ids, float* weights) {
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = ctx.pdl ? 1 : 0;
  cfg.stream = ctx.stream;
  const int warps = (E > 256) ? 1 : 4;  // keep dynamic smem small for wide routers
  cfg.blockDim = dim3(32 * warps);
  cfg.gridDim = dim3(ceil_div(B, warps));
  cfg.dynamicSmemBytes = static_cast<size_t>(warps) * E * sizeof(float);
  const int epl = ceil_div(E, 32);
#define SKB_ROUTE_CASE(N)                                                                       \
  cudaLaunchKernelEx(&cfg, route_topk_kernel<N>, logits, B, E, K, renorm, ids, weights)
  if (epl <= 1) SKB_ROUTE_CASE(1);
  else if (epl <= 2) SKB_ROUTE_CASE(2);
  else if (epl <= 4) SKB_ROUTE_CASE(4);
  else if (epl <= 8) SKB_ROUTE_CASE(8);
  else if (epl <= 16) SKB_ROUTE_CASE(16);
  else SKB_ROUTE_CASE(32);
#undef SKB_ROUTE_CASE
  return 1;
}

// ---------------------------------------------------------------------------------------------
// Dispatch: stable counting sort of the B*K flat slots by expert id.  One CTA; W warps each own
// a contiguous segment of slots, so "ascending flat slot inside an expert bucket"
// (proj/src/router.cpp:80-87) falls out of (segment order, in-segment order).
// ---------------------------------------------------------------------------------------------
constexpr int kDispatchThreads = 1024;

__global__ void __launch_bounds__(kDispatchThreads) dispatch_kernel(
    const int32_t* __restrict__ ids, int B, int K, int E, int has_shared, int tile_tokens, int W,
    DispatchBuffers d) {
  extern __shared__ int32_t sm[];
  int32_t* whist = sm;                 // [W][E] per-warp counts, later exclusive bases
  int32_t* cnt = whist + W * E;        // [E]
  int32_t* off = cnt + E;              // [E + 1]
  int32_t* tile_off = off + E + 1;     // [E + 1]
  __shared__ int32_t warp_sums[32];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int BK = B * K;
  const int seg = round_up(ceil_div(BK, W), 32);  // slots per warp segment

  for (int i = tid; i < W * E; i += blockDim.x) whist[i] = 0;
  pdl_wait();
  pdl_launch_dependents();
  __syncthreads();

  if (warp < W) {
    const int lo = warp * seg, hi = min(BK, lo + seg);
    for (int i = lo + lane; i < hi; i += 32) atomicAdd(&whist[warp * E + ids[i]], 1);
  }
  __syncthreads();

  for (int e = tid; e < E; e += blockDim.x) {
    int run = 0;
    for (int w = 0; w < W; ++w) {
      const int c = whist[w * E + e];
      whist[w * E + e] = run;
      run += c;
    }
    cnt[e] = run;
  }
  __syncthreads();

  // exclusive scans over experts (E <= 1024 = blockDim): token offsets and tile offsets
  {
    const int c = (tid < E) ? cnt[tid] : 0;
    const int tl = ceil_div(c, tile_tokens);
    int a = c, b = tl;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int ua = __shfl_up_sync(0xffffffffu, a, o);
      const int ub = __shfl_up_sync(0xffffffffu, b, o);
      if (lane >= o) {
        a += ua;
        b += ub;
      }
    }
    if (lane == 31) warp_sums[warp] = (a << 0);
    __syncthreads();
    // pack-free: two passes through the same scratch
    int base_a = 0;
    for (int w = 0; w < warp; ++w) base_a += warp_sums[w];
    __syncthreads();
    if (lane == 31) warp_sums[warp] = b;
    __syncthreads();
    int base_b = 0;
    for (int w = 0; w < warp; ++w) base_b += warp_sums[w];
    if (tid < E) {
      off[tid] = base_a + a - c;
      tile_off[tid] = base_b + b - tl;
      if (tid == E - 1) {
        off[E] = base_a + a;
        tile_off[E] = base_b + b;
      }
    }
  }
  __syncthreads();

  for (int e = tid; e <= E; e += blockDim.x) d.expert_off[e] = off[e];

  if (warp < W) {
    const int lo = warp * seg, hi = min(BK, lo + seg);
    for (int base = lo; base < hi; base += 32) {
      const int i = base + lane;
      const int e = (i < hi) ? ids[i] : -1 - lane;  // distinct negatives: no false matches
      const unsigned peers = __match_any_sync(0xffffffffu, e);
      const int rank = __popc(peers & ((1u << lane) - 1u));
      if (i < hi) {
        const int pos = off[e] + whist[warp * E + e] + rank;
        d.perm[pos] = i;
        d.inv[i] = pos;
        d.row_expert[pos] = e;
      }
      __syncwarp();
      if (i < hi && rank == 0) whist[warp * E + e] += __popc(peers);
      __syncwarp();
    }
  }

  // tile list: expert-major, tile_tokens rows per tile, then the shared expert's tiles
  for (int e = tid; e < E; e += blockDim.x) {
    const int c = cnt[e];
    const int nt = ceil_div(c, tile_tokens);
    for (int j = 0; j < nt; ++j) {
      const int ti = tile_off[e] + j;
      d.tile_expert[ti] = e;
      d.tile_row0[ti] = off[e] + j * tile_tokens;
      d.tile_nrows[ti] = min(tile_tokens, c - j * tile_tokens);
    }
  }
  int n_tiles = tile_off[E];
  if (has_shared) {
    const int nsh = ceil_div(B, tile_tokens);
    for (int j = tid; j < nsh; j += blockDim.x) {
      d.tile_expert[n_tiles + j] = E;
      d.tile_row0[n_tiles + j] = BK + j * tile_tokens;
      d.tile_nrows[n_tiles + j] = min(tile_tokens, B - j * tile_tokens);
    }
    for (int t = tid; t < B; t += blockDim.x) d.row_expert[BK + t] = E;
    n_tiles += nsh;
  }
  if (tid == 0) *d.n_tiles = n_tiles;
}

static int dispatch_warps(int E) {
  int w = 8192 / (E > 0 ? E : 1);
  if (w > 32) w = 32;
  if (w < 1) w = 1;
  return w;
}

int launch_dispatch(const LaunchCtx& ctx, const int32_t* ids, int B, int K, int E, int has_shared,
                    int tile_tokens, const DispatchBuffers& d) {
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = ctx.pdl ? 1 : 0;
  cfg.stream = ctx.stream;
  const int W = dispatch_warps(E);
  cfg.blockDim = dim3(kDispatchThreads);
  cfg.gridDim = dim3(1);
  cfg.dynamicSmemBytes = (static_cast<size_t>(W) * E + 3 * E + 2) * sizeof(int32_t);
  cudaLaunchKernelEx(&cfg, dispatch_kernel, ids, B, K, E, has_shared, tile_tokens, W, d);
  return 1;
}

// Token permutation: xs[row] = bf16(x[token(row)]); pad columns [D, Dp) stay zero (memset once).
__global__ void __launch_bounds__(256) permute_tokens_kernel(const float* __restrict__ x,
                                                             const int32_t* __restrict__ perm,
                                                             int BK, int K, int D, int Dp,
                                                             __nv_bfloat16* __restrict__ xs) {
  pdl_wait();
  pdl_launch_dependents();
  const int row = blockIdx.x;
  const int t = (row < BK) ? perm[row] / K : row - BK;
  const float* src = x + static_cast<size_t>(t) * D;
  __nv_bfloat16* dst = xs + static_cast<size_t>(row) * Dp;
  if ((D % 4) == 0) {
    const float4* s4 = reinterpret_cast<const float4*>(src);
    uint2* d2 = reinterpret_cast<uint2*>(dst);
    for (int q = threadIdx.x; q < D / 4; q += blockDim.x) {
      const float4 v = __ldg(s4 + q);
      __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y);
      __nv_bfloat162 hi = __floats2bfloat162_rn(v.z, v.w);
      uint2 o;
      o.x = *reinterpret_cast<uint32_t*>(&lo);
      o.y = *reinterpret_cast<uint32_t*>(&hi);
      d2[q] = o;
    }
  } else {
    for (int dd = threadIdx.x; dd < D; dd += blockDim.x) dst[dd] = __float2bfloat16_rn(src[dd]);
  }
}

int launch_permute_tokens(const LaunchCtx& ctx, const float* x, const int32_t* perm, int B, int K,
                          int D, int Dp, int has_shared, __nv_bfloat16* xs) {
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = ctx.pdl ? 1 : 0;
  cfg.stream = ctx.stream;
  cfg.blockDim = dim3(256);
  cfg.gridDim = dim3(B * K + (has_shared ? B : 0));
  cudaLaunchKernelEx(&cfg, permute_tokens_kernel, x, perm, B * K, K, D, Dp, xs);
  return 1;
}

// DispatchPlan export (align_dispatch's padded view): experts ascending, each non-empty bucket
// padded with -1 to a multiple of `block`.  counts2 = {n_padded, n_blocks}.
__global__ void __launch_bounds__(1024) plan_export_kernel(const int32_t* __restrict__ perm,
                                                           const int32_t* __restrict__ expert_off,
                                                           int E, int block,
                                                           int32_t* __restrict__ sorted_out,
                                                           int32_t* __restrict__ expert_of_block,
                                                           int32_t* __restrict__ counts2) {
  extern __shared__ int32_t pad_off[];  // [E + 1]
  if (threadIdx.x == 0) {
    int run = 0;
    for (int e = 0; e < E; ++e) {
      pad_off[e] = run;
      run += round_up(expert_off[e + 1] - expert_off[e], block);
    }
    pad_off[E] = run;
    counts2[0] = run;
    counts2[1] = run / block;
  }
  __syncthreads();
  for (int e = 0; e < E; ++e) {
    const int lo = expert_off[e], c = expert_off[e + 1] - lo;
    const int padded = pad_off[e + 1] - pad_off[e];
    for (int i = threadIdx.x; i < padded; i += blockDim.x) {
      sorted_out[pad_off[e] + i] = (i < c) ? perm[lo + i] : -1;
      if ((i % block) == 0) expert_of_block[(pad_off[e] + i) / block] = e;
    }
  }
}

int launch_plan_export(const LaunchCtx& ctx, const int32_t* perm, const int32_t* expert_off, int E,
                       int block, int32_t* sorted_out, int32_t* expert_of_block,
                       int32_t* counts2) {
  plan_export_kernel<<<1, 1024, (E + 1) * sizeof(int32_t), ctx.stream>>>(
      perm, expert_off, E, block, sorted_out, expert_of_block, counts2);
  return 1;
}

// combine() as a stage of its own (proj/src/router.cpp:109-132): y = sum_s w * out, s ascending,
// multiply and add rounded separately => bit-identical to the reference.
__global__ void __launch_bounds__(256) combine_slots_kernel(const float* __restrict__ slot_outputs,
                                                            const float* __restrict__ weights,
                                                            int K, int D, float* __restrict__ y) {
  const int t = blockIdx.y;
  const int dd = blockIdx.x * blockDim.x + threadIdx.x;
  if (dd >= D) return;
  float acc = 0.0f;
  for (int s = 0; s < K; ++s) {
    const float w = weights[static_cast<size_t>(t) * K + s];
    const float v = slot_outputs[(static_cast<size_t>(t) * K + s) * D + dd];
    acc = __fadd_rn(acc, __fmul_rn(w, v));
  }
  y[static_cast<size_t>(t) * D + dd] = acc;
}

int launch_combine_slots(const LaunchCtx& ctx, const float* slot_outputs, const float* weights,
                         int B, int K, int D, float* y) {
  combine_slots_kernel<<<dim3(ceil_div(D, 256), B), 256, 0, ctx.stream>>>(slot_outputs, weights,
                                                                          K, D, y);
  return 1;
}

}  // namespace skb
