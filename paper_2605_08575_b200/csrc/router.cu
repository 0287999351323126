// router.cu -- subsystem (1): router logits, softmax + warp-level top-k, counting sort by
// expert (token permutation) and the tile list the grouped GEMM walks.
//
// Reference behaviour reproduced here:
//   route_logits / matvec   proj/src/engine.cpp:43-53, proj/src/linalg.cpp:22-40
//   route                   proj/src/router.cpp:13-68
//   align_dispatch          proj/src/router.cpp:70-107
#include "skb_internal.cuh"
#include "route_device.cuh"

namespace skb {

// ---------------------------------------------------------------------------------------------
// Fused router: logits (order-faithful) -> softmax/top-k -> dispatch, one launch.
//
// logits[t][e] = sum_d router[e][d] * x[t][d] with a float accumulator, d ascending, multiply
// and add rounded separately (the reference is built with -ffp-contract=off,
// proj/CMakeLists.txt:26-27).  That chain is inherently serial (D dependent FADDs), so the
// kernel is organised around it: one single-warp CTA per (8 experts x 4 tokens) runs 32
// chains, one per lane, fed by a second warp through a 4-deep ring of 512-float sub-chunks
// (1-D TMA bulk copies, mbarrier hand-off, no block barriers in the loop).  Measured on B200: a
// dependent fp32 add chain advances one element per ~5.5-6.5 cycles (tools/micro/chain_lat.cu).  The CTA that completes a token block's logits
// ("last arriver" on a global counter) runs route() for those tokens; the CTA that completes
// the last token block builds the dispatch when B*K is small (decode).
// ---------------------------------------------------------------------------------------------
constexpr int kRfEB = 8;        // experts per CTA
constexpr int kRfTB = 4;        // tokens per CTA
constexpr int kRfSub = 512;     // floats per sub-chunk (one mbarrier wait costs ~300 cycles of the
                                // chain: measured 18.0k cycles at 128, so waits are kept rare)
constexpr int kRfStages = 4;    // ring depth (maximum; large grids run with 2, see launch_router)
constexpr int kRfRow = kRfSub + 4;  // padded row stride (floats): conflict-free LDS.128
constexpr int kRfRows = kRfEB + kRfTB;
constexpr int kRfSmemFloats = kRfStages * kRfRows * kRfRow;
constexpr int kRfSmemBytes = kRfSmemFloats * 4 + 2 * kRfStages * 8;  // ring + full/empty barriers

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Dispatch for B*K <= kSmallSlots by one warp: stable counting sort by expert and the tile list,
// by direct counting (O((B*K)^2 / 32), no scans).  Same outputs as dispatch_kernel.
__device__ void warp_small_dispatch(const int32_t* __restrict__ ids, int B, int K, int E,
                                    int has_shared, int tile_tokens, const DispatchBuffers& d,
                                    int32_t* sc /* >= 4 * kSmallSlots ints */, bool token_tiles) {
  const int lane = threadIdx.x & 31;
  const int BK = B * K;
  int32_t* ids_s = sc;
  int32_t* rank_s = sc + kSmallSlots;
  int32_t* pos_s = sc + 2 * kSmallSlots;
  int32_t* cnt_s = sc + 3 * kSmallSlots;
  for (int i = lane; i < BK; i += 32) ids_s[i] = __ldcg(ids + i);
  __syncwarp();
  for (int i = lane; i < BK; i += 32) {
    const int e = ids_s[i];
    int lower = 0, before = 0, cnt = 0;
    for (int j = 0; j < BK; ++j) {
      const int ej = ids_s[j];
      lower += (ej < e);
      before += (ej == e && j < i);
      cnt += (ej == e);
    }
    const int pos = lower + before;
    rank_s[i] = before;
    pos_s[i] = pos;
    cnt_s[i] = ((before % tile_tokens) == 0) ? cnt : -cnt;  // sign marks tile heads
    d.perm[pos] = i;
    d.inv[i] = pos;
    d.row_expert[pos] = e;
  }
  __syncwarp();
  if (token_tiles) {
    // Token-indexed tiles (B <= 16): one tile per distinct expert; column c of the tile is
    // token c, tile_colrow names the h row of (token c, this expert) or -1.  The GEMM reads
    // the bf16 token rows directly.
    int heads = 0;
    for (int i = lane; i < BK; i += 32) {
      if (rank_s[i] == 0) {  // first slot of its expert
        const int e = ids_s[i];
        int ti = 0;
        for (int j = 0; j < BK; ++j) ti += (rank_s[j] == 0 && ids_s[j] < e);
        d.tile_expert[ti] = e;
        d.tile_row0[ti] = 0;
        d.tile_nrows[ti] = B;
        for (int c = 0; c < 16; ++c) {
          int r = -1;
          if (c < B)
            for (int s2 = 0; s2 < K; ++s2)
              if (ids_s[c * K + s2] == e) r = pos_s[c * K + s2];
          d.tile_colrow[ti * 16 + c] = r;
        }
        ++heads;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) heads += __shfl_xor_sync(0xffffffffu, heads, o);
    int n_tiles = heads;
    if (has_shared) {
      if (lane < 16) d.tile_colrow[n_tiles * 16 + lane] = lane < B ? BK + lane : -1;
      if (lane == 0) {
        d.tile_expert[n_tiles] = E;
        d.tile_row0[n_tiles] = 0;
        d.tile_nrows[n_tiles] = B;
      }
      for (int t = lane; t < B; t += 32) d.row_expert[BK + t] = E;
      n_tiles += 1;
    }
    if (lane == 0) *d.n_tiles = n_tiles;
    return;
  }
  int heads = 0;
  for (int i = lane; i < BK; i += 32) {
    if (cnt_s[i] > 0) {
      const int e = ids_s[i], r = rank_s[i];
      int ti = 0;
      for (int j = 0; j < BK; ++j)
        ti += (cnt_s[j] > 0 && (ids_s[j] < e || (ids_s[j] == e && rank_s[j] < r)));
      d.tile_expert[ti] = e;
      d.tile_row0[ti] = pos_s[i];
      d.tile_nrows[ti] = min(tile_tokens, cnt_s[i] - r);
      ++heads;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) heads += __shfl_xor_sync(0xffffffffu, heads, o);
  int n_tiles = heads;
  if (has_shared) {
    const int nsh = ceil_div(B, tile_tokens);
    for (int j = lane; j < nsh; j += 32) {
      d.tile_expert[n_tiles + j] = E;
      d.tile_row0[n_tiles + j] = BK + j * tile_tokens;
      d.tile_nrows[n_tiles + j] = min(tile_tokens, B - j * tile_tokens);
    }
    for (int t = lane; t < B; t += 32) d.row_expert[BK + t] = E;
    n_tiles += nsh;
  }
  if (lane == 0) *d.n_tiles = n_tiles;
}

// route() for batches: one warp per token, 4 tokens per CTA.
__global__ void __launch_bounds__(128) route_tokens_kernel(const float* __restrict__ logits, int B,
                                                           int E, int K, int renorm,
                                                           int32_t* __restrict__ ids,
                                                           float* __restrict__ weights) {
  extern __shared__ __align__(16) float rt_smem[];  // [4][round_up(E, 4) + round_up(K, 4)]
  const int warp = threadIdx.x >> 5;
  const int t = blockIdx.x * 4 + warp;
  pdl_wait();
  pdl_launch_dependents();
  if (t >= B) return;
  warp_route_token(logits + static_cast<size_t>(t) * E, E, K, renorm,
                   rt_smem + static_cast<size_t>(warp) * (round_up(E, 4) + round_up(K, 4)),
                   ids + static_cast<size_t>(t) * K,
                   weights + static_cast<size_t>(t) * K);
}

// ---------------------------------------------------------------------------------------------
// route() + dispatch + token permutation of a batch as ONE kernel (batches whose CTAs are all
// resident): a warp per token, 4 tokens per CTA.
//   1. every warp routes its token (ids, weights to global memory);
//   2. grid barrier (arrive counter + generation word, self-resetting: graph-replay safe);
//   3. every CTA reads all B*K expert ids (L2) into two shared-memory histograms -- slots of the
//      whole batch and slots before its own first slot -- so that it can place its own 4*K slots
//      of the stable counting sort without any other CTA: pos = off[e] + before[e] + rank;
//      CTA 0 also writes the expert offsets and the tile list;
//   4. every warp converts its token to bf16 ONCE and writes the K (+1 shared) expert-sorted
//      copies the gate/up GEMM reads.
// Same perm / inv / tile list as dispatch_kernel, bit for bit.  Replaces three launches
// (route_tokens_kernel, dispatch_chunks_kernel: a single CTA, permute_tokens_kernel) whose
// boundaries and single-CTA latency were ~10 us of the Granite-shape batch-256 step.
// ---------------------------------------------------------------------------------------------
struct RouteDispatchArgs {
  const float* logits;
  const float* x;
  int B, E, K, renorm, D, Dp, has_shared, tile_tokens;
  int32_t* ids;
  float* weights;
  DispatchBuffers d;
  __nv_bfloat16* xs;
  unsigned* bar;  // grid-barrier word: arrivals | generation << 16
};

__device__ __forceinline__ uint2 pack_bf16x4(float4 v) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y);
  __nv_bfloat162 hi = __floats2bfloat162_rn(v.z, v.w);
  uint2 o;
  o.x = *reinterpret_cast<uint32_t*>(&lo);
  o.y = *reinterpret_cast<uint32_t*>(&hi);
  return o;
}
__device__ __forceinline__ unsigned ld_acquire_gpu_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

#ifdef SKB_DEBUG_TIMING
__device__ long long g_rd_dbg[16];
#define RD_T(i) do { if (blockIdx.x == gridDim.x / 2 && threadIdx.x == 0) g_rd_dbg[i] = clock64(); } while (0)
extern "C" void skb_debug_rd(long long* out) { cudaMemcpyFromSymbol(out, g_rd_dbg, sizeof(g_rd_dbg)); }
#else
#define RD_T(i) do { } while (0)
#endif

// 4 token warps + 4 helper warps (16 warps: the kernel itself 0.4 us shorter, the step 2 us
// longer -- the big CTAs keep the next kernel's CTAs from becoming resident beside them)
constexpr int kRdThreads = 256;
constexpr int kRdGroups = kRdThreads / 128;
template <int RV>  // route() variant: warp_route_token_v
__global__ void __launch_bounds__(kRdThreads) route_dispatch_kernel(RouteDispatchArgs a) {
  extern __shared__ __align__(16) float rd_smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int E = a.E, K = a.K, BK = a.B * a.K;
  const int rt_words = round_up(E, 4) + round_up(K, 4);
  float* rt = rd_smem + static_cast<size_t>(warp & 3) * rt_words;
  int32_t* tot = reinterpret_cast<int32_t*>(rd_smem + 4 * static_cast<size_t>(rt_words));  // [E]
  int32_t* bef = tot + E;           // [E] slots before this CTA's first slot, per expert
  int32_t* off = bef + E;           // [E + 1]
  int32_t* tile_off = off + E + 1;  // [E + 1]
  int32_t* pos_s = tile_off + E + 1;  // [4 * K] rows of this CTA's slots
  // warps 0-3 own the CTA's four tokens; the other warps help with the histograms and write
  // their share of each token's copies
  const int tw = warp & 3, half = warp >> 2;
  const int t = blockIdx.x * 4 + tw;
  for (int i = tid; i < 2 * E; i += kRdThreads) tot[i] = 0;

  RD_T(0);
  // the token row is an input of the layer, not of the previous kernel: loaded and converted
  // before the programmatic-launch wait (first 1024 columns; longer rows stream later)
  const bool vec_row = (a.D % 4) == 0;
  const int nq = a.D / 4;
  uint2 o0[8];
  if (t < a.B && vec_row) {
    const float4* s4 = reinterpret_cast<const float4*>(a.x + static_cast<size_t>(t) * a.D);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int q = u * 32 + lane;
      if (q < nq) o0[u] = pack_bf16x4(__ldg(s4 + q));
    }
  }
  pdl_wait();
  pdl_launch_dependents();
  RD_T(1);
  if (t < a.B && half == 0)
    warp_route_token_v<RV>(a.logits + static_cast<size_t>(t) * E, E, K, a.renorm, rt,
                           a.ids + static_cast<size_t>(t) * K, a.weights + static_cast<size_t>(t) * K);

  // ---- grid barrier ----
  RD_T(2);
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    // one word: arrivals in the low 16 bits, generation above.  The last arriver's single add
    // clears the arrivals and bumps the generation; everybody else learnt the generation from
    // its own arrival and spins until it changes.  At rest the low bits are 0 again.
    const unsigned old = atomicAdd(a.bar, 1u);
    if ((old & 0xffffu) == gridDim.x - 1) {
      atomicAdd(a.bar, 0x10000u - gridDim.x);
    } else {
      while ((ld_acquire_gpu_u32(a.bar) >> 16) == (old >> 16)) {
      }
    }
  }
  __syncthreads();

  // ---- histograms over all slots ----
  RD_T(3);
  const int s0 = blockIdx.x * 4 * K;  // first flat slot of this CTA
  for (int i = tid; i < BK; i += kRdThreads) {
    const int e = __ldcg(a.ids + i);
    atomicAdd(&tot[e], 1);
    if (i < s0) atomicAdd(&bef[e], 1);
  }
  __syncthreads();
  RD_T(4);
  if (warp == 0) {
    int run = 0, trun = 0;
    for (int e0 = 0; e0 < E; e0 += 32) {
      const int e = e0 + lane;
      const int c = e < E ? tot[e] : 0;
      const int tl = ceil_div(c, a.tile_tokens);
      int ia = c, ib = tl;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int ua = __shfl_up_sync(0xffffffffu, ia, o);
        const int ub = __shfl_up_sync(0xffffffffu, ib, o);
        if (lane >= o) {
          ia += ua;
          ib += ub;
        }
      }
      if (e < E) {
        off[e] = run + ia - c;
        tile_off[e] = trun + ib - tl;
      }
      run += __shfl_sync(0xffffffffu, ia, 31);
      trun += __shfl_sync(0xffffffffu, ib, 31);
    }
    if (lane == 0) {
      off[E] = run;
      tile_off[E] = trun;
    }
    __syncwarp();
    // ---- this CTA's slots, in flat order, 32 at a time ----
    const int n_own = max(0, min(4 * K, BK - s0));
    for (int j0 = 0; j0 < n_own; j0 += 32) {
      const int j = j0 + lane;
      const int i = s0 + j;
      const int e = j < n_own ? __ldcg(a.ids + i) : -1 - lane;  // distinct negatives: no matches
      const unsigned peers = __match_any_sync(0xffffffffu, e);
      const int rank = __popc(peers & ((1u << lane) - 1u));
      if (j < n_own) {
        const int pos = off[e] + bef[e] + rank;
        a.d.perm[pos] = i;
        a.d.inv[i] = pos;
        a.d.row_expert[pos] = e;
        pos_s[j] = pos;
      }
      __syncwarp();
      if (j < n_own && rank == 0) bef[e] += __popc(peers);
      __syncwarp();
    }
  }
  __syncthreads();
  RD_T(5);

  if (blockIdx.x == 0) {
    for (int e = tid; e <= E; e += kRdThreads) a.d.expert_off[e] = off[e];
    // tile list: expert-major, tile_tokens rows per tile, then the shared expert's tiles
    for (int e = tid; e < E; e += kRdThreads) {
      const int c = tot[e];
      const int nt = ceil_div(c, a.tile_tokens);
      for (int j = 0; j < nt; ++j) {
        const int ti = tile_off[e] + j;
        a.d.tile_expert[ti] = e;
        a.d.tile_row0[ti] = off[e] + j * a.tile_tokens;
        a.d.tile_nrows[ti] = min(a.tile_tokens, c - j * a.tile_tokens);
      }
    }
    int n_tiles = tile_off[E];
    if (a.has_shared) {
      const int nsh = ceil_div(a.B, a.tile_tokens);
      for (int j = tid; j < nsh; j += kRdThreads) {
        a.d.tile_expert[n_tiles + j] = E;
        a.d.tile_row0[n_tiles + j] = BK + j * a.tile_tokens;
        a.d.tile_nrows[n_tiles + j] = min(a.tile_tokens, a.B - j * a.tile_tokens);
      }
      n_tiles += nsh;
    }
    if (tid == 0) *a.d.n_tiles = n_tiles;
    // the gate/up CTAs, resident behind this kernel, may read the list from here on
    __threadfence();
    __syncthreads();
    if (tid == 0) atomicExch(a.bar + 1, 1u);
  }

  // ---- token permutation: the token's bf16 row, K (+1) copies ----
  RD_T(6);
  if (t < a.B) {
    if (a.has_shared && lane == 0 && half == 0) a.d.row_expert[BK + t] = E;
    const float* src = a.x + static_cast<size_t>(t) * a.D;
    const int copies = K + (a.has_shared ? 1 : 0);
    if (vec_row) {
      const float4* s4 = reinterpret_cast<const float4*>(src);
      for (int q0 = 0; q0 < nq; q0 += 256) {
        uint2 o[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int q = q0 + u * 32 + lane;
          if (q0 == 0) o[u] = o0[u];
          else if (q < nq) o[u] = pack_bf16x4(__ldg(s4 + q));
        }
        for (int k = half; k < copies; k += kRdGroups) {
          const int row = k < K ? pos_s[tw * K + k] : BK + t;
          uint2* d2 = reinterpret_cast<uint2*>(a.xs + static_cast<size_t>(row) * a.Dp);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int q = q0 + u * 32 + lane;
            if (q < nq) d2[q] = o[u];
          }
        }
      }
    } else {
      for (int k = half; k < copies; k += kRdGroups) {
        const int row = k < K ? pos_s[tw * K + k] : BK + t;
        __nv_bfloat16* dst = a.xs + static_cast<size_t>(row) * a.Dp;
        for (int dd = lane; dd < a.D; dd += 32) dst[dd] = __float2bfloat16_rn(src[dd]);
      }
    }
  }
  RD_T(7);
}

struct RouterFusedArgs {
  const float* x;
  const float* router;
  int B, E, D, K, renorm;
  int logits_ready;   // 1: logits were produced by the fast kernel; skip the chains
  int fuse_route;     // 1: the last CTA of a token block runs route() (decode); 0: route_tokens_kernel
  int fuse_dispatch;  // 1: the last CTA also builds the dispatch (B*K <= kSmallSlots)
  int has_shared, tile_tokens;
  int n_eb;            // expert blocks (CTAs per token block that run chains)
  int stages;          // ring depth of this launch
  __nv_bfloat16* xb;   // token tiles: bf16 copy of x, [B][Dp]; written by CTA column n_eb
  int Dp;
  float* logits;
  int32_t* ids;
  float* weights;
  unsigned* counters;  // [0] = finished token blocks, [1 + tb] = finished expert blocks of tb
  unsigned* tiles_flag;  // see route_dispatch_kernel, or nullptr
  DispatchBuffers d;
};

// clock64() timestamps of the kernel's phases, read back by tools/dbg_rf.py; compiled in only
// with -DSKB_DEBUG_TIMING (SKB_DEBUG_TIMING=1 python -m paper_2605_08575_b200.build --force)
#ifdef SKB_DEBUG_TIMING
__device__ long long g_rf_dbg[16];
#define RF_T(i) do { if (lane == 0 && warp == 0) g_rf_dbg[i] = clock64(); } while (0)
#else
#define RF_T(i) do { } while (0)
#endif

__global__ void __launch_bounds__(64) router_fused_kernel(RouterFusedArgs a) {
  extern __shared__ __align__(16) float rf_smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int e0 = blockIdx.x * kRfEB, t0 = blockIdx.y * kRfTB;
  const int D = a.D;
  const int nst = a.stages;  // ring depth of this launch (2 .. kRfStages)
  const uint32_t bar_base = smem_u32(rf_smem + nst * kRfRows * kRfRow);
  auto full_bar = [&](int s) { return bar_base + 8u * s; };
  auto empty_bar = [&](int s) { return bar_base + 8u * (nst + s); };

  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    fence_barrier_init();
  }
  RF_T(0);
  __syncthreads();
  pdl_wait();
  pdl_launch_dependents();
  RF_T(1);
  // "tile list written" flag of this step's route_dispatch_kernel: down again (every reader of
  // the previous step finished kernels ago)
  if (a.tiles_flag != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *a.tiles_flag = 0u;

  if (a.xb != nullptr && static_cast<int>(blockIdx.x) == a.n_eb) {
    // conversion CTAs (token tiles): xb[t] = bf16(x[t]) for this token block, in parallel with
    // the chains of the other CTAs; pad columns [D, Dp) stay zero
    for (int tt = 0; tt < kRfTB; ++tt) {
      const int t = t0 + tt;
      if (t >= a.B) break;
      const float* src = a.x + static_cast<size_t>(t) * D;
      __nv_bfloat16* dst = a.xb + static_cast<size_t>(t) * a.Dp;
      for (int d = threadIdx.x; d < D; d += 64) dst[d] = __float2bfloat16_rn(__ldg(src + d));
    }
    return;
  }

  if (!a.logits_ready) {
    const int nsub = ceil_div(D, kRfSub);
    const bool vec_ok = (D % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0) &&
                        ((reinterpret_cast<uintptr_t>(a.router) & 15) == 0);
    const int n_e = min(kRfEB, a.E - e0), n_t = min(kRfTB, a.B - t0);  // valid rows
    if (warp == 1) {
      // ---- producer: the ring is fed with 1-D bulk copies (TMA engine), one row per lane -- a
      // copy costs its issuing thread ~40 ns + bytes / 30 GB/s, so twelve 2 KB rows issued by one
      // lane (1.3 us per sub-chunk) starved the chains (1.05 us per sub-chunk); the chain warp
      // never spends an issue slot on staging ----
      if (vec_ok) {
        // ring row of this lane: lanes [0, n_e) a router row, lanes [kRfEB, kRfEB + n_t) a token
        const bool w_lane = lane < n_e, x_lane = lane >= kRfEB && lane - kRfEB < n_t;
        const float* src = w_lane ? a.router + static_cast<size_t>(e0 + lane) * D
                                  : a.x + static_cast<size_t>(t0 + (x_lane ? lane - kRfEB : 0)) * D;
#pragma unroll 1
        for (int sc = 0; sc < nsub; ++sc) {
          const int slot = sc % nst;
          const int d0 = sc * kRfSub;
          const uint32_t bytes = static_cast<uint32_t>(min(kRfSub, D - d0)) * 4u;
          if (lane == 0) {
            mbar_wait(empty_bar(slot), ((sc / nst) & 1u) ^ 1u);
            mbar_arrive_expect_tx(full_bar(slot), bytes * static_cast<uint32_t>(n_e + n_t));
          }
          __syncwarp();
          const uint32_t dst = smem_u32(rf_smem + slot * kRfRows * kRfRow);
          if (w_lane || x_lane)
            bulk_copy_g2s(dst + lane * kRfRow * 4, src + d0, bytes, full_bar(slot));
        }
      } else {
        // unaligned / odd d_model: plain loads by the whole producer warp, handed over with two
        // block barriers per sub-chunk (generic-proxy stores; rare path, kept simple)
#pragma unroll 1
        for (int sc = 0; sc < nsub; ++sc) {
          const int slot = sc % nst;
          const int d0 = sc * kRfSub;
          const int n = min(kRfSub, D - d0);
          float* dst = rf_smem + slot * kRfRows * kRfRow;
#pragma unroll 1
          for (int r = 0; r < n_e + n_t; ++r) {
            const float* src = (r < n_e) ? a.router + static_cast<size_t>(e0 + r) * D + d0
                                         : a.x + static_cast<size_t>(t0 + r - n_e) * D + d0;
            float* drow = dst + ((r < n_e) ? r : kRfEB + r - n_e) * kRfRow;
#pragma unroll 1
            for (int i = lane; i < n; i += 32) drow[i] = __ldg(src + i);
          }
          __syncthreads();  // filled
          __syncthreads();  // consumed
        }
      }
      return;
    }

    // ---- consumer: 32 chains, one per lane ----
    const int e_i = lane / kRfTB, t_j = lane % kRfTB;
    const bool valid = (e_i < n_e) && (t_j < n_t);
    float acc = 0.0f;
#ifdef SKB_DEBUG_TIMING
    long long t_wait = 0;
#endif
#pragma unroll 1
    for (int sc = 0; sc < nsub; ++sc) {
      const int slot = sc % nst;
#ifdef SKB_DEBUG_TIMING
      const long long tw0 = clock64();
#endif
      if (vec_ok) mbar_wait(full_bar(slot), (sc / nst) & 1u);
      else __syncthreads();  // filled (fallback path)
#ifdef SKB_DEBUG_TIMING
      t_wait += clock64() - tw0;
#endif
      if (sc == 0) RF_T(8);
      const float* base = rf_smem + slot * kRfRows * kRfRow;
      const float* wr = base + e_i * kRfRow;
      const float* xr = base + (kRfEB + t_j) * kRfRow;
      const int n = min(kRfSub, D - sc * kRfSub);
      const int n4 = n >> 2;
#pragma unroll 8
      for (int q = 0; q < n4; ++q) {
        const float4 w = *reinterpret_cast<const float4*>(wr + 4 * q);
        const float4 xv = *reinterpret_cast<const float4*>(xr + 4 * q);
        acc = __fadd_rn(acc, __fmul_rn(w.x, xv.x));
        acc = __fadd_rn(acc, __fmul_rn(w.y, xv.y));
        acc = __fadd_rn(acc, __fmul_rn(w.z, xv.z));
        acc = __fadd_rn(acc, __fmul_rn(w.w, xv.w));
      }
#pragma unroll 1
      for (int i = 4 * n4; i < n; ++i) acc = __fadd_rn(acc, __fmul_rn(wr[i], xr[i]));
      if (vec_ok) {
        __syncwarp();
        if (lane == 0) mbar_arrive(empty_bar(slot));
      } else {
        __syncthreads();  // consumed (fallback path)
      }
    }
    RF_T(2);
#ifdef SKB_DEBUG_TIMING
    if (lane == 0) g_rf_dbg[9] = t_wait;
#endif
    if (valid) a.logits[static_cast<size_t>(t0 + t_j) * a.E + e0 + e_i] = acc;

    if (!a.fuse_route) return;
    // last arriver of this token block runs route() for its tokens
    __threadfence();
    __syncwarp();
    unsigned prev = 0;
    if (lane == 0) prev = atomicAdd(&a.counters[1 + blockIdx.y], 1u);
    prev = __shfl_sync(0xffffffffu, prev, 0);
    RF_T(3);
    if (prev != static_cast<unsigned>(a.n_eb - 1)) return;
    if (lane == 0) a.counters[1 + blockIdx.y] = 0;  // at rest again for the next forward
    __threadfence();
    RF_T(4);
  } else if (warp == 1) {
    return;
  }

  for (int tt = 0; tt < kRfTB; ++tt) {
    const int t = t0 + tt;
    if (t >= a.B) break;
    warp_route_token(a.logits + static_cast<size_t>(t) * a.E, a.E, a.K, a.renorm, rf_smem,
                     a.ids + static_cast<size_t>(t) * a.K, a.weights + static_cast<size_t>(t) * a.K);
  }
  RF_T(5);
  if (!a.fuse_dispatch) return;

  if (gridDim.y > 1) {  // a single token block is its own last arriver
    __threadfence();
    __syncwarp();
    unsigned prev = 0;
    if (lane == 0) prev = atomicAdd(&a.counters[0], 1u);
    prev = __shfl_sync(0xffffffffu, prev, 0);
    if (prev != gridDim.y - 1) return;
    if (lane == 0) a.counters[0] = 0;
    __threadfence();
  }
  __syncwarp();
  RF_T(6);
  warp_small_dispatch(a.ids, a.B, a.K, a.E, a.has_shared, a.tile_tokens, a.d,
                      reinterpret_cast<int32_t*>(rf_smem), a.xb != nullptr);
  RF_T(7);
}

#ifdef SKB_DEBUG_TIMING
extern "C" void skb_debug_rf(long long* out) { cudaMemcpyFromSymbol(out, g_rf_dbg, sizeof(g_rf_dbg)); }
#endif

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

// Batches up to this size run route() and the dispatch inside the router kernel (its last CTA);
// above it they are parallel kernels of their own.  Measured (tools/fused_vs_staged.py, staged
// column): the in-kernel tail costs ~2.8 us per token (one warp per token block routes its tokens
// one after the other, one warp sorts all slots), so it only pays for one or two tokens.
// (Granite shape batch 8: 66.7 -> 54.3 us, OLMoE shape batch 8: 146 -> 130-143 us with the limit at 2.)
static constexpr int fuse_route_max_batch() { return 2; }

static size_t route_dispatch_smem(int E, int K) {
  return (4 * static_cast<size_t>(round_up(E, 4) + round_up(K, 4)) + 4 * static_cast<size_t>(E) + 2 +
          4 * static_cast<size_t>(K)) * 4;
}

// One launch for route + dispatch + permutation: the grid barrier inside needs every CTA resident
// (4 tokens per CTA, 256 threads, a few KB of shared memory: 8 CTAs per SM), and every CTA reads
// all B*K ids, which stops paying on large batches.
bool router_fuses_permute(const RouterLaunch& r) {
  if (r.xs == nullptr || r.grid_bar == nullptr || r.dispatch == nullptr || r.x == nullptr) return false;
  if (r.B <= fuse_route_max_batch()) return false;
  if (static_cast<long>(r.B) * r.K > 4096) return false;
  if (route_dispatch_smem(r.E, r.K) > 40 * 1024) return false;
  // every CTA of the grid must be resident at once: asked of the runtime, per device and
  // expert-count class, with the largest shared-memory request the limit above allows
  static int resident[64][4] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  const int cls = r.E <= 32 ? 0 : (r.E <= 64 ? 1 : (r.E <= 128 ? 2 : 3));
  int cap = __atomic_load_n(&resident[dev & 63][cls], __ATOMIC_ACQUIRE);
  if (cap == 0) {
    int per_sm = 0, sms = 0;
    const size_t smem = 40 * 1024;
    cudaError_t e = cudaSuccess;
    switch (cls) {
      case 0: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, route_dispatch_kernel<1>, kRdThreads, smem); break;
      case 1: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, route_dispatch_kernel<2>, kRdThreads, smem); break;
      case 2: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, route_dispatch_kernel<4>, kRdThreads, smem); break;
      default: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, route_dispatch_kernel<0>, kRdThreads, smem); break;
    }
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cap = (e == cudaSuccess && per_sm > 0 && sms > 0) ? per_sm * sms : -1;
    __atomic_store_n(&resident[dev & 63][cls], cap, __ATOMIC_RELEASE);
  }
  // (half of it: the previous kernel's last CTAs and the next kernel's first share the SMs)
  return cap > 0 && ceil_div(r.B, 4) <= cap / 2;
}

bool router_token_tiles(int B, int K, bool want) {
  return want && B <= 16 && B <= fuse_route_max_batch() && B * K <= kSmallSlots;
}

int launch_router(const LaunchCtx& ctx, const RouterLaunch& r) {
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = ctx.pdl ? 1 : 0;
  cfg.stream = ctx.stream;
  int launches = 0;
  if (r.fast && r.x != nullptr) {
    const long warps = static_cast<long>(r.B) * r.E;
    cfg.gridDim = dim3(static_cast<unsigned>((warps * 32 + 255) / 256));
    cfg.blockDim = dim3(256);
    cudaLaunchKernelEx(&cfg, router_logits_fast_kernel, r.x, r.router, r.B, r.E, r.D, r.logits);
    ++launches;
  }
  // per device (function attributes and the SM count are per device; the C ABI takes a device)
  static bool attr_set[64] = {};
  static int sms_of[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  const int di = dev & 63;
  constexpr int smem = kRfSmemBytes;
  if (!__atomic_load_n(&attr_set[di], __ATOMIC_ACQUIRE)) {
    cudaFuncSetAttribute(router_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    sms_of[di] = n;
    __atomic_store_n(&attr_set[di], true, __ATOMIC_RELEASE);
  }
  const int n_sms = sms_of[di];
  RouterFusedArgs a{};
  a.x = r.x;
  a.router = r.router;
  a.B = r.B;
  a.E = r.E;
  a.D = r.D;
  a.K = r.K;
  a.renorm = r.renorm;
  a.logits_ready = (r.fast || r.x == nullptr) ? 1 : 0;
  // decode batches: everything in the router kernel (no launch boundaries); larger batches:
  // route() and the dispatch are parallel kernels of their own
  a.fuse_route = (r.B <= fuse_route_max_batch()) ? 1 : 0;
  a.fuse_dispatch = (a.fuse_route && r.dispatch != nullptr && r.B * r.K <= kSmallSlots) ? 1 : 0;
  a.has_shared = r.has_shared;
  a.tile_tokens = r.tile_tokens;
  a.logits = r.logits;
  a.ids = r.ids;
  a.weights = r.weights;
  a.counters = r.counters;
  a.tiles_flag = router_fuses_permute(r) ? r.grid_bar + 1 : nullptr;
  if (r.dispatch) a.d = *r.dispatch;
  a.n_eb = a.logits_ready ? 1 : ceil_div(r.E, kRfEB);
  const bool token_tiles = a.fuse_dispatch && router_token_tiles(r.B, r.K, r.xb != nullptr);
  a.xb = token_tiles ? r.xb : nullptr;
  a.Dp = r.Dp;
  if (!(a.logits_ready && !a.fuse_route)) {
    cfg.gridDim = dim3(a.n_eb + (token_tiles ? 1 : 0), ceil_div(r.B, kRfTB));
    cfg.blockDim = dim3(64);
    // One chain warp per CTA is latency-bound (a dependent add every 4 cycles), so what matters
    // for a grid of many CTAs is how many are resident: a ring of 2 instead of 4 sub-chunks
    // halves the shared memory and doubles the CTAs per SM (prefill: 4096 CTAs, 14 waves -> 7).
    const long n_ctas = static_cast<long>(cfg.gridDim.x) * cfg.gridDim.y;
    a.stages = n_ctas > 2L * n_sms ? 2 : kRfStages;
    cfg.dynamicSmemBytes = static_cast<size_t>(a.stages) * kRfRows * kRfRow * 4 + 2 * a.stages * 8;
    cudaLaunchKernelEx(&cfg, router_fused_kernel, a);
    ++launches;
  }
  if (!a.fuse_route && router_fuses_permute(r)) {
    RouteDispatchArgs rd{};
    rd.logits = r.logits;
    rd.x = r.x;
    rd.B = r.B;
    rd.E = r.E;
    rd.K = r.K;
    rd.renorm = r.renorm;
    rd.D = r.D;
    rd.Dp = r.Dp;
    rd.has_shared = r.has_shared;
    rd.tile_tokens = r.tile_tokens;
    rd.ids = r.ids;
    rd.weights = r.weights;
    rd.d = *r.dispatch;
    rd.xs = r.xs;
    rd.bar = r.grid_bar;
    cfg.gridDim = dim3(ceil_div(r.B, 4));
    cfg.blockDim = dim3(kRdThreads);
    cfg.dynamicSmemBytes = route_dispatch_smem(r.E, r.K);
    if (r.E <= 32) cudaLaunchKernelEx(&cfg, route_dispatch_kernel<1>, rd);
    else if (r.E <= 64) cudaLaunchKernelEx(&cfg, route_dispatch_kernel<2>, rd);
    else if (r.E <= 128) cudaLaunchKernelEx(&cfg, route_dispatch_kernel<4>, rd);
    else cudaLaunchKernelEx(&cfg, route_dispatch_kernel<0>, rd);
    return launches + 1;
  }
  if (!a.fuse_route) {
    cfg.gridDim = dim3(ceil_div(r.B, 4));
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = 4 * static_cast<size_t>(round_up(r.E, 4) + round_up(r.K, 4)) * sizeof(float);
    cudaLaunchKernelEx(&cfg, route_tokens_kernel, (const float*)r.logits, r.B, r.E, r.K, r.renorm,
                       r.ids, r.weights);
    ++launches;
  }
  if (r.dispatch != nullptr && !a.fuse_dispatch)
    launches += launch_dispatch(ctx, r.ids, r.B, r.K, r.E, r.has_shared, r.tile_tokens, *r.dispatch);
  return launches;
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

// Same outputs by 32-slot chunks: every chunk of 32 consecutive flat slots is its own segment, so
// the per-segment counts need no atomics (one __match_any per chunk), the bases are one warp scan
// per expert over the chunks, and ids are read from global memory once (expert id and in-chunk
// rank stay in registers for the scatter).  4 block barriers instead of 7; used whenever the
// [chunks][E + 1] table fits shared memory and each warp owns at most kDcPerWarp chunks.
constexpr int kDcPerWarp = 4;

__global__ void __launch_bounds__(kDispatchThreads) dispatch_chunks_kernel(
    const int32_t* __restrict__ ids, int B, int K, int E, int has_shared, int tile_tokens,
    DispatchBuffers d) {
  extern __shared__ int32_t sm[];
  const int BK = B * K;
  const int chunks = ceil_div(BK, 32);
  const int ES = E + 1;                 // padded row: column walks hit distinct banks
  int32_t* chist = sm;                  // [chunks][ES] counts, later exclusive bases
  int32_t* cnt = chist + chunks * ES;   // [E]
  int32_t* off = cnt + E;               // [E + 1]
  int32_t* tile_off = off + E + 1;      // [E + 1]
  __shared__ int32_t wsum_a[32], wsum_b[32];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < chunks * ES; i += kDispatchThreads) chist[i] = 0;
  pdl_wait();
  pdl_launch_dependents();
  __syncthreads();

  int my_e[kDcPerWarp], my_rank[kDcPerWarp];
#pragma unroll
  for (int r = 0; r < kDcPerWarp; ++r) {
    const int i = (warp + 32 * r) * 32 + lane;
    my_e[r] = (i < BK) ? __ldcg(ids + i) : -1 - lane;  // distinct negatives: no false matches
  }
#pragma unroll
  for (int r = 0; r < kDcPerWarp; ++r) {
    const int c = warp + 32 * r;
    if (c < chunks) {  // warp-uniform
      const unsigned peers = __match_any_sync(0xffffffffu, my_e[r]);
      my_rank[r] = __popc(peers & ((1u << lane) - 1u));
      if (my_e[r] >= 0 && my_rank[r] == 0) chist[c * ES + my_e[r]] = __popc(peers);
    }
  }
  __syncthreads();

  // per expert: exclusive scan of the chunk counts (chunk order = flat slot order)
  for (int e = warp; e < E; e += 32) {
    int run = 0;
    for (int c0 = 0; c0 < chunks; c0 += 32) {
      const int c = c0 + lane;
      const int v = (c < chunks) ? chist[c * ES + e] : 0;
      int incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      if (c < chunks) chist[c * ES + e] = run + incl - v;
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) cnt[e] = run;
  }
  __syncthreads();

  // exclusive scans over experts (E <= 1024 = blockDim): row offsets and tile offsets
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
    if (E > 32) {  // block-uniform
      if (lane == 31) {
        wsum_a[warp] = a;
        wsum_b[warp] = b;
      }
      __syncthreads();
      for (int w = 0; w < warp; ++w) {
        a += wsum_a[w];
        b += wsum_b[w];
      }
    }
    if (tid < E) {
      off[tid] = a - c;
      tile_off[tid] = b - tl;
      if (tid == E - 1) {
        off[E] = a;
        tile_off[E] = b;
      }
    }
  }
  __syncthreads();

#pragma unroll
  for (int r = 0; r < kDcPerWarp; ++r) {
    const int c = warp + 32 * r;
    const int i = c * 32 + lane;
    if (i < BK) {
      const int e = my_e[r];
      const int pos = off[e] + chist[c * ES + e] + my_rank[r];
      d.perm[pos] = i;
      d.inv[i] = pos;
      d.row_expert[pos] = e;
    }
  }
  for (int e = tid; e <= E; e += kDispatchThreads) d.expert_off[e] = off[e];

  // tile list: expert-major, tile_tokens rows per tile, then the shared expert's tiles
  for (int e = tid; e < E; e += kDispatchThreads) {
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
    for (int j = tid; j < nsh; j += kDispatchThreads) {
      d.tile_expert[n_tiles + j] = E;
      d.tile_row0[n_tiles + j] = BK + j * tile_tokens;
      d.tile_nrows[n_tiles + j] = min(tile_tokens, B - j * tile_tokens);
    }
    for (int t = tid; t < B; t += kDispatchThreads) d.row_expert[BK + t] = E;
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
  cfg.blockDim = dim3(kDispatchThreads);
  cfg.gridDim = dim3(1);
  const int chunks = ceil_div(B * K, 32);
  const size_t chunk_smem = (static_cast<size_t>(chunks) * (E + 1) + 3 * E + 2) * sizeof(int32_t);
  if (chunks <= 32 * kDcPerWarp && chunk_smem <= 48 * 1024) {
    cfg.dynamicSmemBytes = chunk_smem;
    cudaLaunchKernelEx(&cfg, dispatch_chunks_kernel, ids, B, K, E, has_shared, tile_tokens, d);
    return 1;
  }
  const int W = dispatch_warps(E);
  cfg.dynamicSmemBytes = (static_cast<size_t>(W) * E + 3 * E + 2) * sizeof(int32_t);
  cudaLaunchKernelEx(&cfg, dispatch_kernel, ids, B, K, E, has_shared, tile_tokens, W, d);
  return 1;
}

// Token permutation: xs[row] = bf16(x[token(row)]); pad columns [D, Dp) stay zero (memset once).
// One warp per row, 8 rows per CTA, eight 128-bit loads in flight per lane (a CTA per row was
// 2048 tiny CTAs at batch 256: launch- and latency-bound).
__global__ void __launch_bounds__(256) permute_tokens_kernel(const float* __restrict__ x,
                                                             const int32_t* __restrict__ perm,
                                                             int BK, int rows, int K, int D, int Dp,
                                                             __nv_bfloat16* __restrict__ xs) {
  pdl_wait();
  pdl_launch_dependents();
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int t = (row < BK) ? perm[row] / K : row - BK;
  const float* src = x + static_cast<size_t>(t) * D;
  __nv_bfloat16* dst = xs + static_cast<size_t>(row) * Dp;
  if ((D % 4) == 0) {
    const float4* s4 = reinterpret_cast<const float4*>(src);
    uint2* d2 = reinterpret_cast<uint2*>(dst);
    const int nq = D / 4;
    for (int q0 = 0; q0 < nq; q0 += 256) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int q = q0 + u * 32 + lane;
        if (q < nq) v[u] = __ldg(s4 + q);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int q = q0 + u * 32 + lane;
        if (q < nq) {
          __nv_bfloat162 lo = __floats2bfloat162_rn(v[u].x, v[u].y);
          __nv_bfloat162 hi = __floats2bfloat162_rn(v[u].z, v[u].w);
          uint2 o;
          o.x = *reinterpret_cast<uint32_t*>(&lo);
          o.y = *reinterpret_cast<uint32_t*>(&hi);
          d2[q] = o;
        }
      }
    }
  } else {
    for (int dd = lane; dd < D; dd += 32) dst[dd] = __float2bfloat16_rn(src[dd]);
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
  const int rows = B * K + (has_shared ? B : 0);
  cfg.gridDim = dim3(ceil_div(rows, 8));
  cudaLaunchKernelEx(&cfg, permute_tokens_kernel, x, perm, B * K, rows, K, D, Dp, xs);
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

// Combine after the dense down projection: y[t] = sum_s w(t,s) * slot_out[row(t,s)] (slots
// ascending, multiply and add rounded separately, router.cpp:119-130), shared expert last
// (engine.cpp:168-173).  One thread per (token, 4 columns).
__global__ void __launch_bounds__(256) combine_rows_kernel(const float* __restrict__ slot_out,
                                                           const int32_t* __restrict__ inv,
                                                           const float* __restrict__ weights,
                                                           int B, int K, int D, int Dp,
                                                           int has_shared, float* __restrict__ y,
                                                           float* const* __restrict__ y_rows) {
  // The token's row indices and weights first (one round trip for all slots), then the slot
  // rows eight at a time with every load in flight before the first add: the kernel is two or
  // three memory round trips long instead of two per slot.
  // (Rows and weights come from the router stage, kernels upstream of the down projection this
  // kernel waits for: they are read BEFORE the programmatic-launch wait.)
  __shared__ int32_t rs[kMaxExperts + 1];
  __shared__ float ws[kMaxExperts + 1];
  const int t = blockIdx.y;
  const int R = K + has_shared;
  for (int s = threadIdx.x; s < R; s += blockDim.x) {
    rs[s] = s < K ? __ldcg(inv + t * K + s) : B * K + t;
    ws[s] = s < K ? __ldcg(weights + t * K + s) : 1.0f;
  }
  __syncthreads();
  pdl_wait();
  pdl_launch_dependents();
  const int c4 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (c4 >= D) return;
  float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  const bool vec = (c4 + 3 < D);
#pragma unroll 1
  for (int s0 = 0; s0 < R; s0 += 8) {
    float v[8][4];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      v[u][0] = v[u][1] = v[u][2] = v[u][3] = 0.0f;
      if (s0 + u < R) {
        const float* p = slot_out + static_cast<size_t>(rs[s0 + u]) * Dp + c4;
        if (vec) {
          const float4 q = __ldg(reinterpret_cast<const float4*>(p));
          v[u][0] = q.x; v[u][1] = q.y; v[u][2] = q.z; v[u][3] = q.w;
        } else {
          for (int i = 0; i < 4; ++i) if (c4 + i < D) v[u][i] = p[i];
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (s0 + u < R) {
        const float w = ws[s0 + u];
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i] = __fadd_rn(acc[i], __fmul_rn(w, v[u][i]));
      }
    }
  }
  // (y_rows: every token's output row has its own destination -- expert parallelism writes it
  // straight into the home rank's peer-mapped buffer)
  float* yo = y_rows != nullptr ? y_rows[t] : y + static_cast<size_t>(t) * D;
  for (int i = 0; i < 4; ++i) if (c4 + i < D) yo[c4 + i] = acc[i];
}

int launch_combine_rows(const LaunchCtx& ctx, const float* slot_out, const int32_t* inv,
                        const float* weights, int B, const Geometry& g, float* y,
                        float* const* y_rows) {
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = ctx.pdl ? 1 : 0;
  cfg.stream = ctx.stream;
  cfg.gridDim = dim3(ceil_div(ceil_div(g.D, 4), 256), B);
  cfg.blockDim = dim3(256);
  cudaLaunchKernelEx(&cfg, combine_rows_kernel, slot_out, inv, weights, B, g.K, g.D, g.Dp,
                     g.has_shared, y, y_rows);
  return 1;
}

int launch_combine_slots(const LaunchCtx& ctx, const float* slot_outputs, const float* weights,
                         int B, int K, int D, float* y) {
  combine_slots_kernel<<<dim3(ceil_div(D, 256), B), 256, 0, ctx.stream>>>(slot_outputs, weights,
                                                                          K, D, y);
  return 1;
}

}  // namespace skb
