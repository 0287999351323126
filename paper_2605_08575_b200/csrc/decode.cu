// decode.cu -- the whole layer for decode batches (B <= 16) as ONE persistent launch.
//
// Why one kernel: at decode sizes the layer moves ~10-100 MB, i.e. 10-20 us of HBM time, and
// every kernel boundary (launch, drain, refill of the memory pipeline) costs 2-5 us of that.
// The stages of the reference path (proj/src/engine.cpp:94-191) map onto phases of one grid of
// numSMs CTAs (one per SM, all co-resident), chained by counters in global memory:
//
//   P0  fast router logits.  lf[t][e] = x[t].router[e] by a parallel (not order-faithful)
//       reduction, together with A[t][e] = sum |x.router|.  The reference's logit (ascending-index
//       float accumulation, proj/src/linalg.cpp:22-40) differs from lf by at most
//       m = 2*gamma_D*A (gamma_D = D*u/(1-D*u), u = 2^-24: the standard recursive-summation
//       bound, applied to both sums).  Every expert whose interval [lf-m, lf+m] reaches the K-th
//       largest lower end is a CANDIDATE of the token; the reference's top-K set is provably a
//       subset.  Typically K candidates, sometimes K+1.  (More than K+4, non-finite values, or
//       a threshold more than 60 below the maximum -- the exp underflow region where
//       probabilities tie -- and the CTA simply waits for the exact routing instead.)
//   CH  exact routing, concurrently.  Two dedicated warps per CTA run the order-faithful logit
//       chains (the D dependent float adds of the reference, ~6 cycles each) while the gate/up
//       stream runs; the last chain to finish a token block runs route() (proj/src/router.cpp:
//       13-68) for it.  Expert ids, slot order and weights are therefore the reference's bit for
//       bit, and their latency (5-10 us) is hidden behind P1.
//   P1  gate/up + SwiGLU for the union of candidate experts: work item = (expert, 64 neurons);
//       tcgen05.mma 128x16x16 (gate and up rows interleaved on M, the <=16 tokens on N),
//       TMEM accumulators double-buffered, weights streamed once by TMA through a 9-stage ring
//       (~160 KB in flight per SM).  The epilogue stores h and, in top-k mode, adds each value
//       to a 512-bin histogram of its row (bins = exponent + 3 mantissa bits of |h|).
//   P2  neuron selection + down projection.  Work unit = (token, slot, row chunk).  The unit
//       loads its h row, locates the pivot bucket from the histogram, ranks only the bucket's
//       members (bit-exact mask_smallest_magnitudes, proj/src/activation.cpp:31-52, including the
//       lower-index-first tie rule), takes its share of the survivors in ascending index order
//       and streams exactly those W_down rows (coalesced 128-bit loads, fp32 accumulation in
//       registers).  Dropped neurons cost no HBM bytes.
//   P3  combine: y[t] = sum_s w(t,s) * (sum_chunks partial), slots ascending, shared expert
//       last with weight 1 (proj/src/router.cpp:109-132, engine.cpp:168-173), fixed order.
//
// No float atomics anywhere: results are deterministic and, for a given (shape, batch), do not
// depend on timing.
#include "route_device.cuh"
#include "select_device.cuh"
#include "tc_ptx.cuh"

namespace skb {

namespace {

constexpr int kDecThreads = 256;
constexpr int kDecTokens = 16;                     // MMA N
constexpr int kDecATile = 128 * kBlockK * 2;       // 16 KB
constexpr int kDecBTile = kDecTokens * kBlockK * 2;  // 2 KB
constexpr int kDecStageBytes = kDecATile + kDecBTile;
constexpr int kDecStages = 9;
constexpr int kDecWork = kDecStages * kDecStageBytes;  // 165888 B, reused by P0 / P2 scratch
constexpr int kHistBins = 512;
constexpr int kHistBase = (135 << 3) - (kHistBins - 1);  // top bin = |h| >= 2^8
constexpr int kMemberCap = 1024;
constexpr int kMaxKpt = 32;  // keys per thread: N, S <= 8192
constexpr int kMaxChunkRows = 2048;  // survivors per (row, chunk) unit
constexpr int kGBatches = 8;         // W_down row batches (mbarriers) of the gather ring

// exact-chain ring (per CTA): 8 experts + 4 tokens per unit, 256-float sub-chunks
constexpr int kChEB = 8, kChTB = 4, kChSub = 256, kChStages = 4;
constexpr int kChRow = kChSub + 4;
constexpr int kChRows = kChEB + kChTB;
constexpr int kChBytes = kChStages * kChRows * kChRow * 4;  // 49920

constexpr int kDecMaxE = 256;
constexpr int kDecMaxU = 256;  // union of candidate experts

// counters (unsigned words)
enum { kCtrP0 = 0, kCtrExit = 1, kCtrRoute = 2, kCtrP2 = 3, kCtrChain = 4 /*[4]*/, kCtrH = 8 };

struct DecSmem {
  // offsets from the 1024-aligned base
  static constexpr int work = 0;
  static constexpr int chain = kDecWork;
  static constexpr int rowtab = chain + kChBytes;                  // int16 [kDecMaxU + 1][16]
  static constexpr int uidx = rowtab + (kDecMaxU + 1) * 16 * 2;    // int16 [kDecMaxE]
  static constexpr int ulist = uidx + kDecMaxE * 2;                // int16 [kDecMaxU]
  static constexpr int cande = ulist + kDecMaxU * 2;               // int16 [16][20] candidate experts
  static constexpr int cmask = cande + 16 * 20 * 2;                // uint32 [kDecMaxE]
  static constexpr int rscr = cmask + kDecMaxE * 4;                // float [E + K + 8] route() scratch
  static constexpr int bars = rscr + 1152;                         // 8-byte aligned
  static constexpr int n_bars = 2 * kDecStages + 4 + 2 * kChStages + kGBatches;
  static constexpr int misc = bars + n_bars * 8;                   // ints
  static constexpr int total = misc + 64 * 4;
};
static_assert(DecSmem::bars % 8 == 0, "barrier alignment");
constexpr int kDecSmemBytes = DecSmem::total + 1024;

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void spin_until(const unsigned* p, unsigned target) {
  while (ld_acquire_u32(p) < target) {
  }
}
__device__ __forceinline__ uint2 ld_volatile_u2(const uint2* p) {
  uint2 v;
  asm volatile("ld.volatile.global.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_proxy_async_all() {
  asm volatile("fence.proxy.async;" ::: "memory");
}
__device__ __forceinline__ int hist_bin(uint32_t key) {
  const int b = static_cast<int>(key >> 20) - kHistBase;
  return b < 0 ? 0 : (b > kHistBins - 1 ? kHistBins - 1 : b);
}
__device__ __forceinline__ void fma8(const uint4& u, float hk, float* a) {
  a[0] = fmaf(__uint_as_float(u.x << 16), hk, a[0]);
  a[1] = fmaf(__uint_as_float(u.x & 0xffff0000u), hk, a[1]);
  a[2] = fmaf(__uint_as_float(u.y << 16), hk, a[2]);
  a[3] = fmaf(__uint_as_float(u.y & 0xffff0000u), hk, a[3]);
  a[4] = fmaf(__uint_as_float(u.z << 16), hk, a[4]);
  a[5] = fmaf(__uint_as_float(u.z & 0xffff0000u), hk, a[5]);
  a[6] = fmaf(__uint_as_float(u.w << 16), hk, a[6]);
  a[7] = fmaf(__uint_as_float(u.w & 0xffff0000u), hk, a[7]);
}

}  // namespace

#ifdef SKB_DEBUG_TIMING
__device__ long long g_dec_dbg[160 * 24];
__device__ __forceinline__ long long dec_gtime() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// the dummy shared-memory load makes a stamp placed after a barrier wait for the barrier's
// release (BAR.SYNC blocks at the next dependent instruction, not at issue)
#define DEC_T(i) do { if (threadIdx.x == 0) { unsigned dmy; asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(dmy) : "r"(sm_u32 + DecSmem::misc + 252)); g_dec_dbg[blockIdx.x * 24 + (i) + (dmy & 0u)] = dec_gtime(); } } while (0)
#define DEC_TW(w, i) do { if (threadIdx.x == (w) * 32) g_dec_dbg[blockIdx.x * 24 + (i)] = dec_gtime(); } while (0)
#define DEC_G(i) do { if (threadIdx.x == 0) g_dec_dbg[blockIdx.x * 24 + (i)] = dec_gtime(); } while (0)
extern "C" void skb_debug_dec(long long* out) { cudaMemcpyFromSymbol(out, g_dec_dbg, sizeof(g_dec_dbg)); }
#else
#define DEC_T(i) do { } while (0)
#define DEC_TW(w, i) do { } while (0)
#define DEC_G(i) do { } while (0)
#endif

// One staged W_down row (bf16, in shared memory) times its activation, accumulated into the
// thread's columns: column tile nt covers columns (nt * 256 + l) * 8 .. + 7.
template <int NT>
__device__ __forceinline__ void consume_row(const uint8_t* rowp, float hv, int LPR, int l,
                                            float (&acc)[NT][8]) {
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int c8 = nt * 256 + l;
    if (c8 < LPR) {
      const uint4 u = *reinterpret_cast<const uint4*>(rowp + static_cast<size_t>(c8) * 16);
      fma8(u, hv, acc[nt]);
    }
  }
}

struct DecodeArgs {
  const float* x;
  const float* router;
  const __nv_bfloat16* wd;
  const __nv_bfloat16* wd_shared;
  int B, E, K, D, Dp, N, Np, S, Sp, Nh, has_shared, renorm;
  int sel_mode, n_off_r, n_off_s;
  const uint8_t* mask_r;
  const uint8_t* mask_s;
  int CM, CH, capture;
  __nv_bfloat16* xb;
  float* lf;
  float* lm;
  float* logits;
  int32_t* ids;
  float* wts;
  uint2* hc;  // [16 * CM + 16][Nh] of {bits of h, launch epoch}: data and flag in one 8-byte word
  float* part;
  unsigned* ctr;
  float* y;
  float* h_cap;
  int32_t* inv;
  int32_t* perm;
  int32_t* row_expert;
};

// order-preserving map float -> uint32 (so that warp REDUX max works on floats) and back
__device__ __forceinline__ uint32_t f2ord(float f) {
  const uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// Candidate experts of one token (one warp): every expert whose interval [lf - m, lf + m] reaches
// the K-th largest lower end.  Returns true when the bound cannot be used (non-finite values,
// the exp-underflow region, or more than CM candidates): the caller then waits for the exact
// routing.  VPL = experts per lane.
template <int VPL>
__device__ __forceinline__ bool cand_token(const float* lf, const float* lm, int E, int K, int CM,
                                           int t, uint32_t* cmask) {
  const int lane = threadIdx.x & 31;
  uint32_t lo[VPL];
  float hi[VPL];
  bool bad = false;
  uint32_t mxk = 0u;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int e = i * 32 + lane;
    if (e < E) {
      const float f = __ldcg(lf + e), m = __ldcg(lm + e);
      lo[i] = f2ord(f - m);
      hi[i] = f + m;
      mxk = max(mxk, f2ord(f));
      bad |= !(fabsf(f) < 1e30f) || !(m < 1e30f);
    } else {
      lo[i] = 0u;
      hi[i] = -INFINITY;
    }
  }
  const float mx = ord2f(__reduce_max_sync(0xffffffffu, mxk));
  // K-th largest lower end: K rounds of warp max, all instances of the maximum removed per round
  // (duplicates can only lower the threshold, i.e. enlarge the candidate set)
  uint32_t thrk = 0u;
#pragma unroll 1
  for (int s = 0; s < K; ++s) {
    uint32_t m = 0u;
#pragma unroll
    for (int i = 0; i < VPL; ++i) m = max(m, lo[i]);
    thrk = __reduce_max_sync(0xffffffffu, m);
#pragma unroll
    for (int i = 0; i < VPL; ++i)
      if (lo[i] == thrk) lo[i] = 0u;
  }
  const float thr = thrk == 0u ? -INFINITY : ord2f(thrk);
  int cnt = 0;
  unsigned mine = 0;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const bool c = hi[i] >= thr && (i * 32 + lane) < E;
    cnt += __popc(__ballot_sync(0xffffffffu, c));
    if (c) mine |= 1u << i;
  }
  bad = __any_sync(0xffffffffu, bad) || !(thr > -1e30f) || (thr < mx - 60.0f) || cnt > CM || cnt < K;
  if (!bad) {
#pragma unroll
    for (int i = 0; i < VPL; ++i)
      if (mine & (1u << i)) atomicOr(&cmask[i * 32 + lane], 1u << t);
  }
  return bad;
}

__global__ void __launch_bounds__(kDecThreads, 1)
decode_fused_kernel(const __grid_constant__ CUtensorMap tmap_w,
                    const __grid_constant__ CUtensorMap tmap_xb, const DecodeArgs a) {
  extern __shared__ uint8_t dsm_raw[];
  uint8_t* sm = dsm_raw + ((1024u - (smem_u32(dsm_raw) & 1023u)) & 1023u);
  const uint32_t sm_u32 = smem_u32(sm);
  uint8_t* work = sm + DecSmem::work;
  int16_t* rowtab = reinterpret_cast<int16_t*>(sm + DecSmem::rowtab);
  int16_t* uidx = reinterpret_cast<int16_t*>(sm + DecSmem::uidx);
  int16_t* ulist = reinterpret_cast<int16_t*>(sm + DecSmem::ulist);
  int16_t* cande = reinterpret_cast<int16_t*>(sm + DecSmem::cande);
  uint32_t* cmask = reinterpret_cast<uint32_t*>(sm + DecSmem::cmask);
  int* misc = reinterpret_cast<int*>(sm + DecSmem::misc);
  // misc: 0 tmem ptr, 1 overflow flag, 2 n_u, 8.. P2 scalars, 24.. ncand[16], 40.. pairoff[17]
  int* ncand = misc + 24;
  int* pairoff = misc + 40;
  const uint32_t bar0 = sm_u32 + DecSmem::bars;
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 8u * (kDecStages + s); };
  auto tfull_bar = [&](int b) { return bar0 + 8u * (2 * kDecStages + b); };
  auto tempty_bar = [&](int b) { return bar0 + 8u * (2 * kDecStages + 2 + b); };
  auto cfull_bar = [&](int s) { return bar0 + 8u * (2 * kDecStages + 4 + s); };
  auto cempty_bar = [&](int s) { return bar0 + 8u * (2 * kDecStages + 4 + kChStages + s); };
  auto gbar = [&](int h) { return bar0 + 8u * (2 * kDecStages + 4 + 2 * kChStages + h); };
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grid = gridDim.x, bid = blockIdx.x;
  const int B = a.B, E = a.E, K = a.K, D = a.D, Dp = a.Dp, CM = a.CM;
  const int n_tb = ceil_div(B, kChTB), n_eb = ceil_div(E, kChEB);
  const bool vec_ok = (D % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0) &&
                      ((reinterpret_cast<uintptr_t>(a.router) & 15) == 0);

  DEC_T(0);
  DEC_G(16);
  // the P2 barrier counter is monotonic: this launch waits for base + grid.  Read first thing
  // (nobody can have passed P0 yet); the latency hides behind the prologue.
  unsigned p2_base = 0;
  if (tid == 0) {
    p2_base = *reinterpret_cast<volatile const unsigned*>(&a.ctr[kCtrP2]);
    misc[3] = static_cast<int>(p2_base + 1u);
  }
  // ---- prologue ----
  if (tid == 0) {
    tma_prefetch_desc(&tmap_w);
    tma_prefetch_desc(&tmap_xb);
    for (int s = 0; s < kDecStages; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull_bar(b), 1);
      mbar_init(tempty_bar(b), 4);
    }
    for (int s = 0; s < kChStages; ++s) {
      mbar_init(cfull_bar(s), 1);
      mbar_init(cempty_bar(s), 1);
    }
    for (int b = 0; b < kGBatches; ++b) mbar_init(gbar(b), 1);
    fence_barrier_init();
    misc[1] = 0;
  }
  if (warp == 1) tmem_alloc(sm_u32 + DecSmem::misc, 32);
  for (int e = tid; e < kDecMaxE; e += kDecThreads) cmask[e] = 0u;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t*>(misc);
  // Tag of this launch's activations: h values travel from the P1 epilogue to P2 as 8-byte
  // {bits, epoch} words, so a consumer that reads the right epoch has the value -- no fence, no
  // counter, no polling thread between the two phases.
  const uint32_t epoch = static_cast<uint32_t>(misc[3]);

  // =====================================================================================
  // P0: histogram zeroing, bf16 token rows, fast logits with error bounds
  // =====================================================================================
  for (int t = (bid - E % grid + grid) % grid; t < B; t += grid) {
    const float* src = a.x + static_cast<size_t>(t) * D;
    __nv_bfloat16* dst = a.xb + static_cast<size_t>(t) * Dp;
    for (int d = tid; d < D; d += kDecThreads) dst[d] = __float2bfloat16_rn(__ldg(src + d));
  }
  {
    float* red = reinterpret_cast<float*>(work);  // [8 warps][4 tokens][2]
    // margin = 2 * gamma_D * A, a little inflated for the rounding of A itself
    const double u24 = 5.9604644775390625e-8;
    const float mfac = static_cast<float>(2.02 * (D * u24) / (1.0 - D * u24));
#pragma unroll 1
    for (int e = bid; e < E; e += grid) {
      const float* wr = a.router + static_cast<size_t>(e) * D;
#pragma unroll 1
      for (int t0 = 0; t0 < B; t0 += 4) {
        float pl[4] = {0.0f, 0.0f, 0.0f, 0.0f}, pa[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        if (vec_ok) {
          const float4* w4 = reinterpret_cast<const float4*>(wr);
#pragma unroll 2
          for (int q = tid; q < D / 4; q += kDecThreads) {
            const float4 w = __ldg(w4 + q);
#pragma unroll
            for (int tt = 0; tt < 4; ++tt) {
              if (t0 + tt < B) {
                const float4 xv =
                    __ldg(reinterpret_cast<const float4*>(a.x + static_cast<size_t>(t0 + tt) * D) + q);
                pl[tt] = fmaf(w.x, xv.x, pl[tt]);
                pl[tt] = fmaf(w.y, xv.y, pl[tt]);
                pl[tt] = fmaf(w.z, xv.z, pl[tt]);
                pl[tt] = fmaf(w.w, xv.w, pl[tt]);
                pa[tt] = fmaf(fabsf(w.x), fabsf(xv.x), pa[tt]);
                pa[tt] = fmaf(fabsf(w.y), fabsf(xv.y), pa[tt]);
                pa[tt] = fmaf(fabsf(w.z), fabsf(xv.z), pa[tt]);
                pa[tt] = fmaf(fabsf(w.w), fabsf(xv.w), pa[tt]);
              }
            }
          }
        } else {
#pragma unroll 1
          for (int d = tid; d < D; d += kDecThreads) {
            const float w = __ldg(wr + d);
#pragma unroll
            for (int tt = 0; tt < 4; ++tt) {
              if (t0 + tt < B) {
                const float xv = __ldg(a.x + static_cast<size_t>(t0 + tt) * D + d);
                pl[tt] = fmaf(w, xv, pl[tt]);
                pa[tt] = fmaf(fabsf(w), fabsf(xv), pa[tt]);
              }
            }
          }
        }
#pragma unroll
        for (int tt = 0; tt < 4; ++tt) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            pl[tt] += __shfl_xor_sync(0xffffffffu, pl[tt], o);
            pa[tt] += __shfl_xor_sync(0xffffffffu, pa[tt], o);
          }
          if (lane == 0) {
            red[(warp * 4 + tt) * 2 + 0] = pl[tt];
            red[(warp * 4 + tt) * 2 + 1] = pa[tt];
          }
        }
        __syncthreads();
        if (tid < 4 && t0 + tid < B) {
          float s = 0.0f, sa = 0.0f;
#pragma unroll
          for (int w = 0; w < kDecThreads / 32; ++w) {
            s += red[(w * 4 + tid) * 2 + 0];
            sa += red[(w * 4 + tid) * 2 + 1];
          }
          a.lf[static_cast<size_t>(t0 + tid) * E + e] = s;
          a.lm[static_cast<size_t>(t0 + tid) * E + e] = sa * mfac + 2e-5f;
        }
        __syncthreads();
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    fence_proxy_async_all();
    atomicAdd(&a.ctr[kCtrP0], 1u);
  }
  DEC_T(1);

  // =====================================================================================
  // Exact routing chains: warps 6 (consumer) and 7 (producer), on the LAST CTAs of the grid
  // (the first ones carry the logit units and, at decode sizes, all the gate/up items).  They
  // only read x and the router, so they start right away; their result is needed by P3.
  // =====================================================================================
  if (warp >= 6) {
    float* ring = reinterpret_cast<float*>(sm + DecSmem::chain);
    const int n_cu = n_eb * n_tb;
    const int nsub = ceil_div(D, kChSub);
    int gsc = 0;  // ring position, continues across units
#pragma unroll 1
    for (int cu = grid - 1 - bid; cu < n_cu; cu += grid) {
      const int eb = cu % n_eb, tb = cu / n_eb;
      const int e0 = eb * kChEB, t0 = tb * kChTB;
      const int n_e = min(kChEB, E - e0), n_t = min(kChTB, B - t0);
      if (warp == 7) {
        const float* wsrc = a.router + static_cast<size_t>(e0) * D;
        const float* xsrc = a.x + static_cast<size_t>(t0) * D;
        int psc = gsc;
        if (vec_ok) {
          if (lane == 0) {
#pragma unroll 1
            for (int sc = 0; sc < nsub; ++sc, ++psc) {
              const int slot = psc % kChStages;
              mbar_wait(cempty_bar(slot), ((psc / kChStages) & 1u) ^ 1u);
              const int d0 = sc * kChSub;
              const uint32_t bytes = static_cast<uint32_t>(min(kChSub, D - d0)) * 4u;
              mbar_arrive_expect_tx(cfull_bar(slot), bytes * static_cast<uint32_t>(n_e + n_t));
              const uint32_t dst = smem_u32(ring + slot * kChRows * kChRow);
#pragma unroll 1
              for (int r = 0; r < n_e; ++r)
                bulk_copy_g2s(dst + r * kChRow * 4, wsrc + static_cast<size_t>(r) * D + d0, bytes,
                              cfull_bar(slot));
#pragma unroll 1
              for (int r = 0; r < n_t; ++r)
                bulk_copy_g2s(dst + (kChEB + r) * kChRow * 4, xsrc + static_cast<size_t>(r) * D + d0,
                              bytes, cfull_bar(slot));
            }
          }
        } else {
#pragma unroll 1
          for (int sc = 0; sc < nsub; ++sc, ++psc) {
            const int slot = psc % kChStages;
            mbar_wait(cempty_bar(slot), ((psc / kChStages) & 1u) ^ 1u);
            const int d0 = sc * kChSub;
            const int n = min(kChSub, D - d0);
            float* dst = ring + slot * kChRows * kChRow;
#pragma unroll 1
            for (int r = 0; r < n_e + n_t; ++r) {
              const float* src = (r < n_e) ? wsrc + static_cast<size_t>(r) * D + d0
                                           : xsrc + static_cast<size_t>(r - n_e) * D + d0;
              float* drow = dst + ((r < n_e) ? r : kChEB + r - n_e) * kChRow;
#pragma unroll 1
              for (int i = lane; i < n; i += 32) drow[i] = __ldg(src + i);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(cfull_bar(slot));
          }
        }
      } else {
        const int e_i = lane / kChTB, t_j = lane % kChTB;
        const bool valid = (e_i < n_e) && (t_j < n_t);
        float acc = 0.0f;
        int csc = gsc;
        DEC_TW(6, 14);
#pragma unroll 1
        for (int sc = 0; sc < nsub; ++sc, ++csc) {
          const int slot = csc % kChStages;
          mbar_wait(cfull_bar(slot), (csc / kChStages) & 1u);
          const float* base = ring + slot * kChRows * kChRow;
          const float* wr = base + e_i * kChRow;
          const float* xr = base + (kChEB + t_j) * kChRow;
          const int n = min(kChSub, D - sc * kChSub);
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
          __syncwarp();
          if (lane == 0) mbar_arrive(cempty_bar(slot));
        }
        DEC_TW(6, 15);
        if (valid) a.logits[static_cast<size_t>(t0 + t_j) * E + e0 + e_i] = acc;
        __threadfence();
        __syncwarp();
        unsigned prev = 0;
        if (lane == 0) prev = atomicAdd(&a.ctr[kCtrChain + tb], 1u);
        prev = __shfl_sync(0xffffffffu, prev, 0);
        if (prev == static_cast<unsigned>(n_eb - 1)) {
          // last chain of this token block: route() for its tokens
          __threadfence();
          float* scr = reinterpret_cast<float*>(sm + DecSmem::rscr);
#pragma unroll 1
          for (int tt = 0; tt < n_t; ++tt) {
            const int t = t0 + tt;
            warp_route_token(a.logits + static_cast<size_t>(t) * E, E, K, a.renorm, scr,
                             a.ids + static_cast<size_t>(t) * K, a.wts + static_cast<size_t>(t) * K);
          }
          __threadfence();
          __syncwarp();
          if (lane == 0) atomicAdd(&a.ctr[kCtrRoute], 1u);
        }
      }
      gsc += nsub;
    }
    DEC_TW(6, 10);
  }

  // =====================================================================================
  // P0 barrier, candidates (every CTA computes the same tables), P1
  // =====================================================================================
  if (warp < 6) {
    if (tid == 0) {
      spin_until(&a.ctr[kCtrP0], static_cast<unsigned>(grid));
      fence_proxy_async_all();
    }
    asm volatile("bar.sync 2, 192;" ::: "memory");
    DEC_T(2);
#pragma unroll 1
    for (int t = warp; t < B; t += 6) {
      bool bad;
      if (E <= 64)
        bad = cand_token<2>(a.lf + t * E, a.lm + t * E, E, K, CM, t, cmask);
      else if (E <= 128)
        bad = cand_token<4>(a.lf + t * E, a.lm + t * E, E, K, CM, t, cmask);
      else
        bad = cand_token<8>(a.lf + t * E, a.lm + t * E, E, K, CM, t, cmask);
      if (bad && lane == 0) misc[1] = 1;
    }
    asm volatile("bar.sync 2, 192;" ::: "memory");
    if (misc[1] != 0) {
      // rare: the bound could not separate the candidates -- wait for the exact routing
      if (tid == 0) spin_until(&a.ctr[kCtrRoute], static_cast<unsigned>(n_tb));
      for (int e = tid; e < E; e += 192) cmask[e] = 0u;
      asm volatile("bar.sync 2, 192;" ::: "memory");
      for (int i = tid; i < B * K; i += 192) atomicOr(&cmask[__ldcg(a.ids + i)], 1u << (i / K));
      asm volatile("bar.sync 2, 192;" ::: "memory");
    }
    // union list (ascending expert id) by warp 0
    if (warp == 0) {
      int run = 0;
#pragma unroll 1
      for (int base = 0; base < E; base += 32) {
        const int e = base + lane;
        const bool f = e < E && cmask[e] != 0u;
        const unsigned b = __ballot_sync(0xffffffffu, f);
        const int pos = run + __popc(b & ((1u << lane) - 1u));
        if (e < E) uidx[e] = f ? static_cast<int16_t>(pos) : static_cast<int16_t>(-1);
        if (f) ulist[pos] = static_cast<int16_t>(e);
        run += __popc(b);
      }
      if (lane == 0) misc[2] = run;
    }
    asm volatile("bar.sync 2, 192;" ::: "memory");
    const int n_u = misc[2];
    // The TMA warp only needs the union list: it starts streaming now.  Warps 1-5 build the
    // per-token tables (row table column, candidate list and count) meanwhile; the MMA issuer
    // and the epilogue warps take up their roles after barrier 3.
    if (warp != 0) {
#pragma unroll 1
      for (int t = warp - 1; t < kDecTokens; t += 5) {
        for (int u = lane; u <= n_u; u += 32) rowtab[u * 16 + t] = -1;
        __syncwarp();
        if (t < B) {
          int run = 0;
#pragma unroll 1
          for (int base = 0; base < E; base += 32) {
            const int e = base + lane;
            const bool f = e < E && ((cmask[e] >> t) & 1u);
            const unsigned b = __ballot_sync(0xffffffffu, f);
            if (f) {
              const int r = run + __popc(b & ((1u << lane) - 1u));
              rowtab[uidx[e] * 16 + t] = static_cast<int16_t>(t * CM + r);
              cande[t * CM + r] = static_cast<int16_t>(e);
            }
            run += __popc(b);
          }
          if (lane == 0) {
            ncand[t] = run;
            if (a.has_shared) rowtab[n_u * 16 + t] = static_cast<int16_t>(kDecTokens * CM + t);
          }
        }
      }
      asm volatile("bar.sync 3, 160;" ::: "memory");
      if (tid == 32) {
        int run = 0;
        for (int t = 0; t < B; ++t) {
          pairoff[t] = run;
          run += ncand[t] + (a.has_shared ? 1 : 0);
        }
        pairoff[B] = run;
      }
    }
    DEC_T(3);

    // ---- P1: gate/up + SwiGLU over (union expert, 64-neuron block) items ----
    const int NB = a.Np / kNeuronBlock, NBs = a.has_shared ? a.Sp / kNeuronBlock : 0;
    const int n_items = n_u * NB + NBs;
    const int KB = Dp / kBlockK;
    if (warp == 0) {
      if (lane == 0) {
        int gk = 0;
#pragma unroll 1
        for (int it = bid; it < n_items; it += grid) {
          const bool sh = it >= n_u * NB;
          const int u = sh ? n_u : it / NB;
          const int nb = sh ? it - n_u * NB : it % NB;
          const int e = sh ? E : ulist[u];
          const int a_row = e * 2 * a.Np + nb * 128;
#pragma unroll 1
          for (int kb = 0; kb < KB; ++kb, ++gk) {
            const int s = gk % kDecStages;
            mbar_wait(empty_bar(s), ((gk / kDecStages) & 1u) ^ 1u);
            mbar_arrive_expect_tx(full_bar(s), kDecStageBytes);
            const uint32_t dst = sm_u32 + s * kDecStageBytes;
            tma_load_2d(dst, &tmap_w, 0, ((a_row >> 7) * KB + kb) * 128, full_bar(s),
                        kPolicyEvictFirst);
            tma_load_2d(dst + kDecATile, &tmap_xb, kb * kBlockK, 0, full_bar(s), kPolicyEvictLast);
          }
        }
      }
    } else if (warp == 1) {
      if (lane == 0) {
        constexpr uint32_t kIdesc = make_idesc_bf16(128, kDecTokens);
        int gk = 0, li = 0;
#pragma unroll 1
        for (int it = bid; it < n_items; it += grid, ++li) {
          const int buf = li & 1;
          mbar_wait(tempty_bar(buf), (((li >> 1) & 1u) ^ 1u));
          tc_fence_after();
#pragma unroll 1
          for (int kb = 0; kb < KB; ++kb, ++gk) {
            const int s = gk % kDecStages;
            mbar_wait(full_bar(s), (gk / kDecStages) & 1u);
            tc_fence_after();
            const uint32_t a_smem = sm_u32 + s * kDecStageBytes;
            const uint64_t a_desc = make_smem_desc_sw128(a_smem);
            const uint64_t b_desc = make_smem_desc_sw128(a_smem + kDecATile);
#pragma unroll
            for (int k = 0; k < kBlockK / 16; ++k)
              umma_bf16(tmem_base + buf * kDecTokens, a_desc + 2u * k, b_desc + 2u * k, kIdesc,
                        (kb | k) != 0 ? 1u : 0u);
            umma_commit(empty_bar(s));
          }
          umma_commit(tfull_bar(buf));
        }
      }
    } else {
      const int q = warp & 3;
      const bool is_gate_lane = lane < 16;
      int li = 0;
#pragma unroll 1
      for (int it = bid; it < n_items; it += grid, ++li) {
        const bool sh = it >= n_u * NB;
        const int u = sh ? n_u : it / NB;
        const int nb = sh ? it - n_u * NB : it % NB;
        const int m_valid = sh ? a.S : a.N;
        const int buf = li & 1;
        mbar_wait(tfull_bar(buf), (li >> 1) & 1u);
        tc_fence_after();
        uint32_t v[16];
        tmem_ld_32x32b_x16(tmem_base + (static_cast<uint32_t>(32 * q) << 16) + buf * kDecTokens, v);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty_bar(buf));
        const int n = nb * kNeuronBlock + 16 * q + (lane & 15);
#pragma unroll
        for (int c = 0; c < 16; c += 2) {
          if (c < B) {
            const float mine0 = __uint_as_float(v[c]);
            const float mine1 = __uint_as_float(v[c + 1]);
            const float send = is_gate_lane ? mine1 : mine0;
            const float recv = __shfl_xor_sync(0xffffffffu, send, 16);
            const float g = is_gate_lane ? mine0 : recv;
            const float up = is_gate_lane ? recv : mine1;
            const int col = c + (is_gate_lane ? 0 : 1);
            if (col < B && n < m_valid) {
              const int r = rowtab[u * 16 + col];
              if (r >= 0) {
                const float hval = silu_f(g) * up;
                a.hc[static_cast<size_t>(r) * a.Nh + n] = make_uint2(__float_as_uint(hval), epoch);
              }
            }
          }
        }
      }
    }
  }
  __syncthreads();
  DEC_T(4);
  DEC_G(17);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 32);
  }

  // =====================================================================================
  // P2: selection + down projection over (token, candidate, row chunk) units.  Units are dealt
  // in contiguous ranges, chunk index fastest, so a CTA that holds several chunks of one row
  // selects once.  The chunking depends on the shape only -- not on the batch -- so the
  // reduction tree of a token does not depend on what else is in the batch.  Candidates that the
  // exact routing later rejects (rare) are computed and ignored by P3.
  // =====================================================================================
  const int n_u = misc[2];
  const int CH = a.CH;
  {
        const int n_units = pairoff[B] * CH;
    // scratch inside the (now idle) GEMM stage area, sized by the shape so that as many W_down
    // rows as possible can be in flight
    const int nmax_pad = round_up(a.N > a.S ? a.N : a.S, 256);
    int so = 0;
    uint16_t* lst_idx = reinterpret_cast<uint16_t*>(work + so);  // [nmax_pad] survivors of a run
    so += nmax_pad * 2;
    uint32_t* mlist = reinterpret_cast<uint32_t*>(work + so);  // [kMemberCap + 4] pivot bucket
    so += 4352;
    int* wc = reinterpret_cast<int*>(work + so);               // [kMaxKpt * 8] + [8]
    so += 1280;
    float* gred = reinterpret_cast<float*>(work + so);         // [G][Dp] <= 8 KB (NT == 1)
    so += 8192;
    int* hist_s = reinterpret_cast<int*>(work + so);           // [kHistBins] histogram of the row
    so += kHistBins * 4;
    uint32_t* keys_s = reinterpret_cast<uint32_t*>(work + so); // [nmax_pad] raw bits of h
    so += nmax_pad * 4;
    uint8_t* kf = work + so;                                   // [nmax_pad] keep flags
    so += nmax_pad;
    so = round_up(so, 1024);
    uint8_t* rows_s = work + so;                               // TMA-staged W_down rows
    const int row_bytes = Dp * 2;
    const int n_slots = (kDecWork - so) / row_bytes;
    int gb = 0;                                                    // batches issued so far (phase)
    __shared__ SelScratch sel_sc;
    int* p2 = misc + 8;  // 0 row, 1 e, 2 b*, 3 below_bins, 4 M, 5 pivot, 6 below, 7 equal, 8 mcount, 9 total, 10 slot
    bool route_ready = false;
    const int LPR = Dp >> 3;
    const int NT = ceil_div(LPR, 256);
    const int G = NT == 1 ? (256 / LPR > 0 ? 256 / LPR : 1) : 1;
    // CTAs that host exact-routing chains (the last ones) take units only when the others
    // cannot hold them all in one wave: their P2 would start after the chains
    const int n_chain_ctas = min(n_eb * n_tb, grid);
    const int gp = (n_units <= grid - n_chain_ctas) ? grid - n_chain_ctas : grid;
    const int v0 = bid < gp ? static_cast<int>(static_cast<long long>(bid) * n_units / gp) : 0;
    const int v1 = bid < gp ? static_cast<int>(static_cast<long long>(bid + 1) * n_units / gp) : 0;

    int e = 0, n = 0, kpt = 0, cnt = 0, t = 0, q = 0;
    bool routed = true;

    // A CTA's units are consecutive: they form RUNS of chunks [c_a, c_b) of one row.  A run
    // selects once and streams its rows through the gather ring without draining it between
    // chunks; every chunk still produces its own partial, so the reduction tree is the same
    // whatever the batch (and the run boundaries) -- only the latency of a chunk is paid once
    // per run instead of once per chunk.
#pragma unroll 1
    for (int v = v0; v < v1;) {
      const int pr = v / CH;
      const int c_a = v % CH;
      const int vb = min(v1, (pr + 1) * CH);
      const int c_b = c_a + (vb - v);
      v = vb;
      {
        t = 0;
        while (t + 1 < B && pairoff[t + 1] <= pr) ++t;
        q = pr - pairoff[t];
        routed = q < ncand[t];
        if (tid == 0) {
          int ee, rr, slot = -1;
          if (routed) {
            ee = cande[t * CM + q];
            rr = t * CM + q;
            if (a.sel_mode == kSelectGiven) {
              // caller masks are indexed by slot: the exact routing is needed here
              if (!route_ready) spin_until(&a.ctr[kCtrRoute], static_cast<unsigned>(n_tb));
              for (int j = 0; j < K; ++j)
                if (__ldcg(a.ids + t * K + j) == ee) slot = t * K + j;
            }
          } else {
            ee = E;
            rr = kDecTokens * CM + t;
            slot = t;
          }
          p2[0] = rr;
          p2[1] = ee;
          p2[8] = 0;
          p2[10] = slot;
        }
        route_ready = true;
        __syncthreads();
        DEC_T(8);
        DEC_G(18);
        const int row = p2[0];
        e = p2[1];
        const int slot = p2[10];
        n = routed ? a.N : a.S;
        int mode = a.sel_mode;
        const uint8_t* min_ = nullptr;
        if (mode == kSelectGiven) {
          if (routed) {
            min_ = slot >= 0 ? a.mask_r + static_cast<size_t>(slot) * n : nullptr;
            if (slot < 0) mode = -1;  // a candidate the exact routing rejected: nothing to do
          } else {
            min_ = a.mask_s ? a.mask_s + static_cast<size_t>(slot) * n : nullptr;
            if (min_ == nullptr) mode = kSelectAll;
          }
        }
        int n_off = 0;
        if (mode == kSelectTopk) {
          n_off = routed ? a.n_off_r : a.n_off_s;
          if (n_off <= 0) mode = kSelectAll;
        }
        kpt = ceil_div(n, kDecThreads);
        const uint2* hrow = a.hc + static_cast<size_t>(row) * a.Nh;
        const bool want_hist = mode == kSelectTopk && n_off < n;
        hist_s[2 * tid] = 0;
        hist_s[2 * tid + 1] = 0;
        __syncthreads();
        // every element is read until it carries this launch's epoch (usually at once: the
        // loads of a thread are issued back to back, four in flight)
#pragma unroll 1
        for (int i0 = tid; i0 < n; i0 += 4 * kDecThreads) {
          uint2 v4[4];
#pragma unroll
          for (int u4 = 0; u4 < 4; ++u4) {
            const int i = i0 + u4 * kDecThreads;
            v4[u4] = i < n ? ld_volatile_u2(hrow + i) : make_uint2(0u, epoch);
          }
#pragma unroll
          for (int u4 = 0; u4 < 4; ++u4) {
            const int i = i0 + u4 * kDecThreads;
            if (i < n) {
              while (v4[u4].y != epoch) v4[u4] = ld_volatile_u2(hrow + i);
              keys_s[i] = v4[u4].x;
              if (want_hist) atomicAdd(&hist_s[hist_bin(v4[u4].x & 0x7fffffffu)], 1);
            }
          }
        }
        __syncthreads();
        const uint2 hh = want_hist ? make_uint2(static_cast<unsigned>(hist_s[2 * tid]),
                                                static_cast<unsigned>(hist_s[2 * tid + 1]))
                                   : make_uint2(0u, 0u);

        RowPick pk{0u, 0, true};
        if (mode == kSelectAll) {
          cnt = n;
        } else if (mode == kSelectGiven) {
          cnt = 0;  // counted by the prefix below
        } else if (mode < 0) {
          cnt = 0;
        } else {
          cnt = n_off >= n ? 0 : n - n_off;
          if (cnt > 0) {
            // ---- pivot bucket from the row's histogram ----
            int incl = static_cast<int>(hh.x + hh.y);
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int up = __shfl_up_sync(0xffffffffu, incl, o);
              if (lane >= o) incl += up;
            }
            if (lane == 31) wc[warp] = incl;
            for (int i = tid; i < kMemberCap + 4; i += kDecThreads) mlist[i] = 0xffffffffu;
            __syncthreads();
            int base = 0;
#pragma unroll
            for (int w = 0; w < 8; ++w)
              if (w < warp) base += wc[w];
            incl += base;
            const int excl = incl - static_cast<int>(hh.x + hh.y);
            if (excl < n_off && n_off <= incl) {
              const bool first = n_off <= excl + static_cast<int>(hh.x);
              p2[2] = 2 * tid + (first ? 0 : 1);
              p2[3] = first ? excl : excl + static_cast<int>(hh.x);
              p2[4] = first ? static_cast<int>(hh.x) : static_cast<int>(hh.y);
            }
            __syncthreads();
            const int bstar = p2[2], below_bins = p2[3], M = p2[4];
            if (M <= kMemberCap) {
#pragma unroll 1
              for (int i = tid; i < n; i += kDecThreads) {
                const uint32_t k = keys_s[i] & 0x7fffffffu;
                if (hist_bin(k) == bstar) mlist[atomicAdd(&p2[8], 1)] = k;
              }
              __syncthreads();
              const int rr = n_off - below_bins;  // 1-based rank inside the bucket
              const int M4 = (M + 3) >> 2;
              // one member per thread (the bucket rarely holds more than a few dozen keys)
#pragma unroll 1
              for (int mi = tid; mi < M; mi += kDecThreads) {
                const uint32_t k = mlist[mi];
                int lt = 0, le = 0;
#pragma unroll 1
                for (int q4 = 0; q4 < M4; ++q4) {
                  const uint4 mm = *reinterpret_cast<const uint4*>(mlist + 4 * q4);
                  lt += (mm.x < k) + (mm.y < k) + (mm.z < k) + (mm.w < k);
                  le += (mm.x <= k) + (mm.y <= k) + (mm.z <= k) + (mm.w <= k);
                }
                if (lt < rr && rr <= le) {
                  p2[5] = static_cast<int>(k);
                  p2[6] = below_bins + lt;
                  p2[7] = le - lt;
                }
              }
              __syncthreads();
              pk.pivot = static_cast<uint32_t>(p2[5]);
              pk.ties_to_drop = n_off - p2[6];
              pk.drop_all_ties = (pk.ties_to_drop == p2[7]);
            } else {
              // huge bucket (many equal / clamped values): the general search
#pragma unroll 1
              for (int i = tid; i < n; i += kDecThreads) keys_s[i] &= 0x7fffffffu;
              __syncthreads();
              pk = sel_kary_pick(keys_s, n, n_off, sel_sc);
              __syncthreads();
#pragma unroll 1
              for (int i = tid; i < n; i += kDecThreads) keys_s[i] = ld_volatile_u2(hrow + i).x;
            }
          }
        }
        __syncthreads();
        DEC_T(9);

        // ---- keep flags kf[i] and their exclusive prefix in index order (wc[jj * 8 + warp]) ----
        if (cnt > 0 || mode == kSelectGiven) {
          const bool need_ties = (mode == kSelectTopk) && !pk.drop_all_ties;
#pragma unroll 1
          for (int pass = need_ties ? 0 : 1; pass < 2; ++pass) {
            // pass 0: prefix over tie flags (only when some but not all ties are dropped);
            // pass 1: prefix over keep flags
#pragma unroll 1
            for (int jj = 0; jj < kpt; ++jj) {
              const int i = jj * kDecThreads + tid;
              const bool valid = i < n;
              const uint32_t k = valid ? (keys_s[i] & 0x7fffffffu) : 0u;
              bool f;
              if (pass == 0) {
                f = valid && k == pk.pivot;
              } else if (mode == kSelectAll) {
                f = valid;
              } else if (mode == kSelectGiven) {
                f = valid && min_[i] != 0;
              } else if (pk.drop_all_ties) {
                f = valid && k > pk.pivot;
              } else {
                f = valid && (k > pk.pivot || (k == pk.pivot && kf[i] != 0));
              }
              const unsigned bal = __ballot_sync(0xffffffffu, f);
              if (lane == 0) wc[jj * 8 + warp] = __popc(bal);
              if (pass == 1 && valid) kf[i] = f ? 1 : 0;
            }
            __syncthreads();
            {
              // exclusive scan of wc[0 .. kpt*8) in (jj, warp) order: one entry per thread
              const int ne = kpt * 8;
              const int val = tid < ne ? wc[tid] : 0;
              int incl = val;
#pragma unroll
              for (int o = 1; o < 32; o <<= 1) {
                const int up = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += up;
              }
              if (lane == 31) wc[kMaxKpt * 8 + warp] = incl;
              __syncthreads();
              int base = 0;
#pragma unroll
              for (int w = 0; w < 8; ++w)
                if (w < warp) base += wc[kMaxKpt * 8 + w];
              if (tid < ne) wc[tid] = base + incl - val;
              if (tid == kDecThreads - 1) p2[9] = base + incl;  // total
              __syncthreads();
            }
            if (pass == 0) {
              // a tie survives when its rank among the ties (ascending index) >= ties_to_drop
#pragma unroll 1
              for (int jj = 0; jj < kpt; ++jj) {
                const int i = jj * kDecThreads + tid;
                const bool f = i < n && (keys_s[i] & 0x7fffffffu) == pk.pivot;
                const unsigned bal = __ballot_sync(0xffffffffu, f);
                const int rank = wc[jj * 8 + warp] + __popc(bal & ((1u << lane) - 1u));
                if (f) kf[i] = rank >= pk.ties_to_drop ? 1 : 0;
              }
              __syncthreads();
            } else if (mode == kSelectGiven) {
              cnt = p2[9];
            }
          }
        }
      }
      DEC_T(11);

      // ---- survivors of the run's chunks, ascending index: ranks [c_a * C, min(cnt, c_b * C)) ----
      const int C = ceil_div(cnt > 0 ? cnt : 1, CH);
      const int lo = c_a * C;
      const int hi_ = min(cnt, c_b * C);
      const int m = hi_ > lo ? hi_ - lo : 0;
      if (m > 0) {
#pragma unroll 1
        for (int jj = 0; jj < kpt; ++jj) {
          const int i = jj * kDecThreads + tid;
          const bool f = i < n && kf[i] != 0;
          const unsigned bal = __ballot_sync(0xffffffffu, f);
          const int rank = wc[jj * 8 + warp] + __popc(bal & ((1u << lane) - 1u));
          if (f && rank >= lo && rank < hi_) lst_idx[rank - lo] = static_cast<uint16_t>(i);
        }
      }
      __syncthreads();
      DEC_T(12);

      // ---- gather: one 1-D bulk copy (TMA engine) per surviving W_down row into a ring of
      // kGBatches batches of H rows (one mbarrier each) in shared memory, accumulated from there.
      // Batches never straddle a chunk; the ring runs ahead across the chunks of the run.
      // (Measured alternatives for a 32-row chunk: 32 direct 128-bit loads per thread, all in
      // flight: 7.7 us; two-batch ring: 7.3 us; this ring: 6.9 us.  16-byte cp.async by all
      // threads instead of bulk copies for 2 KB rows: 106 vs 96 us at Granite shape, batch 16.)
      const __nv_bfloat16* wb = routed ? a.wd + static_cast<size_t>(e) * a.Np * Dp : a.wd_shared;
      const int H = max(1, min(C, n_slots / kGBatches));
      const int nb_c = ceil_div(C, H);                 // batches of a full chunk
      const int n_ch = ceil_div(m, C);                 // chunks of the run that have rows
      const int Q = n_ch > 0 ? (n_ch - 1) * nb_c + ceil_div(m - (n_ch - 1) * C, H) : 0;
      auto batch_rows = [&](int qq, int& p0, int& p1) {
        const int j = min(qq / nb_c, n_ch - 1);
        const int b = qq - j * nb_c;
        p0 = j * C + b * H;
        p1 = min(min(m, (j + 1) * C), p0 + H);
      };
      auto issue = [&](int qq) {
        const int pos = (gb + qq) % kGBatches;
        int p0, p1;
        batch_rows(qq, p0, p1);
        if (tid == 0) mbar_arrive_expect_tx(gbar(pos), static_cast<uint32_t>((p1 - p0) * row_bytes));
        // convergent issue: lane l of warp w copies row p0 + w + 8 * l
        for (int p = p0 + warp + 8 * lane; p < p1; p += kDecThreads)
          bulk_copy_g2s(smem_u32(rows_s + static_cast<size_t>(pos * H + (p - p0)) * row_bytes),
                        wb + static_cast<size_t>(lst_idx[p]) * Dp, static_cast<uint32_t>(row_bytes),
                        gbar(pos));
        __syncwarp();
      };
      const int g = NT == 1 ? tid / LPR : 0, l = NT == 1 ? tid % LPR : tid;
      const bool lane_ok = g < G;
      for (int qq = 0; qq < Q && qq < kGBatches; ++qq) issue(qq);
      int qn = 0;  // next batch to consume
#pragma unroll 1
      for (int j = 0; j < c_b - c_a; ++j) {
        float acc[4][8];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[nt][i] = 0.0f;
        const int cbase = j * C;  // first row of this chunk in the run's list
        const int nb_j = j < n_ch ? ceil_div(min(C, m - cbase), H) : 0;
#pragma unroll 1
        for (int b = 0; b < nb_j; ++b, ++qn) {
          const int pos = (gb + qn) % kGBatches;
          mbar_wait(gbar(pos), ((gb + qn) / kGBatches) & 1u);
          int p0, p1;
          batch_rows(qn, p0, p1);
          const uint8_t* base = rows_s + static_cast<size_t>(pos * H) * row_bytes;
          if (NT == 1) {
            // group g owns the chunk's rows r with r % G == g (ascending); 4 rows are loaded
            // before their FMAs so that the shared-memory latency is paid once per 4 rows
            if (lane_ok) {
              const int r0 = p0 - cbase;
#pragma unroll 1
              for (int p = p0 + ((g - r0 % G) + G) % G; p < p1; p += 4 * G) {
                uint4 v4[4];
                float hv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  const int pp = p + u * G;
                  const bool ok = pp < p1;
                  hv[u] = ok ? __uint_as_float(keys_s[lst_idx[pp]]) : 0.0f;
                  v4[u] = ok ? *reinterpret_cast<const uint4*>(base + static_cast<size_t>(pp - p0) * row_bytes +
                                                              static_cast<size_t>(l) * 16)
                             : make_uint4(0u, 0u, 0u, 0u);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) fma8(v4[u], hv[u], acc[0]);
              }
            }
          } else {
#pragma unroll 2
            for (int p = p0; p < p1; ++p)
              consume_row<4>(base + static_cast<size_t>(p - p0) * row_bytes,
                             __uint_as_float(keys_s[lst_idx[p]]), LPR, l, acc);
          }
          if (qn + kGBatches < Q) {
            __syncthreads();  // this ring position is free again
            issue(qn + kGBatches);
          }
        }
        // ---- this chunk's partial ----
        float* pout =
            a.part + (static_cast<size_t>(t * (CM + 1) + (routed ? q : CM)) * CH + (c_a + j)) * Dp;
        if (NT == 1) {
          if (G > 1) {
            __syncthreads();  // gred of the previous chunk has been read
            if (lane_ok) {
              float4* d4 = reinterpret_cast<float4*>(gred + static_cast<size_t>(g) * Dp + l * 8);
              d4[0] = make_float4(acc[0][0], acc[0][1], acc[0][2], acc[0][3]);
              d4[1] = make_float4(acc[0][4], acc[0][5], acc[0][6], acc[0][7]);
            }
            __syncthreads();
            for (int d = tid; d < Dp; d += kDecThreads) {
              float sacc = gred[d];
              for (int gg = 1; gg < G; ++gg) sacc = __fadd_rn(sacc, gred[gg * Dp + d]);
              pout[d] = sacc;
            }
          } else if (lane_ok) {
            float4* d4 = reinterpret_cast<float4*>(pout + l * 8);
            d4[0] = make_float4(acc[0][0], acc[0][1], acc[0][2], acc[0][3]);
            d4[1] = make_float4(acc[0][4], acc[0][5], acc[0][6], acc[0][7]);
          }
        } else {
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) {
            const int c8 = nt * 256 + tid;
            if (c8 < LPR) {
              float4* d4 = reinterpret_cast<float4*>(pout + c8 * 8);
              d4[0] = make_float4(acc[nt][0], acc[nt][1], acc[nt][2], acc[nt][3]);
              d4[1] = make_float4(acc[nt][4], acc[nt][5], acc[nt][6], acc[nt][7]);
            }
          }
        }
      }
      gb += Q;
      DEC_T(13);
      __syncthreads();  // scratch is reused by the next run
    }
  }
  DEC_T(5);

  // =====================================================================================
  // P3: grid barrier (partials + exact routing), then the ordered combine.  Each CTA owns a
  // contiguous range of (token, 4 columns) outputs: all partials of a batch of 8 outputs are
  // fetched at once into shared memory, summed per slot over the chunks (ascending), then over
  // the slots (ascending, shared expert last with weight 1: router.cpp:109-132,
  // engine.cpp:168-173).
  // =====================================================================================
  __syncthreads();
  int* srow = reinterpret_cast<int*>(work);          // [B][R] candidate rank of every slot
  float* swt = reinterpret_cast<float*>(work + 2048);  // [B][R] combine weights
  {
    const int R = K + (a.has_shared ? 1 : 0);
    if (tid == 0) {
      __threadfence();
      atomicAdd(&a.ctr[kCtrP2], 1u);
      spin_until(&a.ctr[kCtrRoute], static_cast<unsigned>(n_tb));
    }
    __syncthreads();
    // slot tables (the exact routing is known now); overlaps the wait for the other CTAs
    for (int i = tid; i < B * R; i += kDecThreads) {
      const int t = i / R, j = i % R;
      if (j < K) {
        const int ee = __ldcg(a.ids + t * K + j);
        srow[i] = rowtab[uidx[ee] * 16 + t] - t * CM;
        swt[i] = __ldcg(a.wts + t * K + j);
      } else {
        srow[i] = CM;
        swt[i] = 1.0f;
      }
    }
    if (tid == 0) {
      while (ld_acquire_u32(&a.ctr[kCtrP2]) - p2_base < static_cast<unsigned>(grid)) {
      }
      if (bid == 0) {
        // every CTA is past its last read of these: back to rest for the next forward
        a.ctr[kCtrP0] = 0u;
        a.ctr[kCtrRoute] = 0u;
        for (int i = 0; i < 4; ++i) a.ctr[kCtrChain + i] = 0u;
      }
    }
    __syncthreads();
    DEC_T(6);
    const int RC = R * CH;
    const int D4 = Dp / 4;
    const int total4 = B * D4;
    constexpr int QB = 8;
    float4* buf = reinterpret_cast<float4*>(work + 4096);  // [QB][R][CH]
    float4* sj = buf + QB * RC;                            // [QB][R]
    const bool y_vec = (D % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.y) & 15) == 0);
    const int q0 = static_cast<int>(static_cast<long long>(bid) * total4 / grid);
    const int q1 = static_cast<int>(static_cast<long long>(bid + 1) * total4 / grid);
#pragma unroll 1
    for (int qb = q0; qb < q1; qb += QB) {
      const int nq = min(QB, q1 - qb);
#pragma unroll 2
      for (int idx = tid; idx < nq * RC; idx += kDecThreads) {
        const int qi = idx / RC, rem = idx % RC;
        const int j = rem / CH, c = rem % CH;
        const int qq = qb + qi;
        const int t = qq / D4, d4 = qq % D4;
        const int r = srow[t * R + j];
        buf[idx] = __ldcg(reinterpret_cast<const float4*>(
            a.part + (static_cast<size_t>(t * (CM + 1) + r) * CH + c) * Dp + d4 * 4));
      }
      __syncthreads();
      for (int idx = tid; idx < nq * R; idx += kDecThreads) {
        const float4* pb = buf + static_cast<size_t>(idx) * CH;
        float4 sacc = pb[0];
#pragma unroll 1
        for (int c = 1; c < CH; ++c) {
          const float4 pv = pb[c];
          sacc.x = __fadd_rn(sacc.x, pv.x);
          sacc.y = __fadd_rn(sacc.y, pv.y);
          sacc.z = __fadd_rn(sacc.z, pv.z);
          sacc.w = __fadd_rn(sacc.w, pv.w);
        }
        sj[idx] = sacc;
      }
      __syncthreads();
      if (tid < nq) {
        const int qq = qb + tid;
        const int t = qq / D4, d4 = qq % D4;
        float4 acc = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll 1
        for (int j = 0; j < R; ++j) {
          const float w = swt[t * R + j];
          const float4 sv = sj[tid * R + j];
          acc.x = __fadd_rn(acc.x, __fmul_rn(w, sv.x));
          acc.y = __fadd_rn(acc.y, __fmul_rn(w, sv.y));
          acc.z = __fadd_rn(acc.z, __fmul_rn(w, sv.z));
          acc.w = __fadd_rn(acc.w, __fmul_rn(w, sv.w));
        }
        float* yo = a.y + static_cast<size_t>(t) * D + d4 * 4;
        if (y_vec && d4 * 4 + 3 < D) {
          *reinterpret_cast<float4*>(yo) = acc;
        } else {
          if (d4 * 4 + 0 < D) yo[0] = acc.x;
          if (d4 * 4 + 1 < D) yo[1] = acc.y;
          if (d4 * 4 + 2 < D) yo[2] = acc.z;
          if (d4 * 4 + 3 < D) yo[3] = acc.w;
        }
      }
      __syncthreads();
    }
    if (a.capture) {
      // h in slot order for the MaskSet / activation captures of the host API
      const int BK = B * K;
#pragma unroll 1
      for (int sl = bid; sl < BK + (a.has_shared ? B : 0); sl += grid) {
        const bool rt = sl < BK;
        const int t = rt ? sl / K : sl - BK;
        const int ee = rt ? __ldcg(a.ids + sl) : E;
        const int row = rt ? rowtab[uidx[ee] * 16 + t] : kDecTokens * CM + t;
        const int n = rt ? a.N : a.S;
        const uint2* src = a.hc + static_cast<size_t>(row) * a.Nh;
        float* dst = a.h_cap + static_cast<size_t>(sl) * a.Nh;
        for (int i = tid; i < n; i += kDecThreads) dst[i] = __uint_as_float(ld_volatile_u2(src + i).x);
        if (tid == 0) {
          a.row_expert[sl] = ee;
          if (rt) {
            a.inv[sl] = sl;
            a.perm[sl] = sl;
          }
        }
      }
    }
  }
  DEC_T(7);
  DEC_G(19);
}

bool decode_fused_eligible(const Geometry& g, int B) {
  const int nmax = g.N > g.S ? g.N : g.S;
  if (!(B >= 1 && B <= kDecTokens && g.E <= kDecMaxE && g.K <= 16 && nmax <= kMaxKpt * kDecThreads &&
        g.Dp <= 8192 && (g.Dp % 64) == 0 && g.E + g.K + 8 <= 288 &&
        ceil_div(nmax, 32) <= kMaxChunkRows))
    return false;
  // the gather ring needs at least kGBatches W_down rows of shared memory (P2 scratch layout)
  const int nmax_pad = round_up(nmax, 256);
  const int so = round_up(2 * nmax_pad + 4352 + 1280 + 8192 + kHistBins * 4 + 5 * nmax_pad, 1024);
  return (kDecWork - so) / (g.Dp * 2) >= kGBatches;
}

int decode_counter_words() { return kCtrH + kDecMaxU + 8; }
int decode_cand_rows(int K) { return K + 4; }
int decode_chunks(const Geometry& g, int B, int keep_max, int n_sms) {
  // Batch-invariant by design (B is ignored): one token's units fill the grid once.
  (void)B;
  const int R = g.K + (g.has_shared ? 1 : 0);
  int ch = n_sms / (R + 1);  // room for one extra candidate per token in a single wave
  int cap = keep_max / 8;  // at least ~8 rows per unit
  if (cap < 1) cap = 1;
  if (ch > cap) ch = cap;
  if (ch > 32) ch = 32;
  if (ch < 1) ch = 1;
  while (ch < 32 && ceil_div(keep_max, ch) > kMaxChunkRows) ++ch;  // survivor list capacity
  return ch;
}

int launch_decode_fused(const LaunchCtx& ctx, const CUtensorMap* tmap_w, const CUtensorMap* tmap_xb,
                        const DecodeLaunch& d, const Geometry& g, int n_sms) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(decode_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kDecSmemBytes);
    attr_set = true;
  }
  DecodeArgs a{};
  a.x = d.x;
  a.router = d.router;
  a.wd = d.wd;
  a.wd_shared = d.wd_shared;
  a.B = d.B;
  a.E = g.E;
  a.K = g.K;
  a.D = g.D;
  a.Dp = g.Dp;
  a.N = g.N;
  a.Np = g.Np;
  a.S = g.S;
  a.Sp = g.Sp;
  a.Nh = g.Nh;
  a.has_shared = g.has_shared;
  a.renorm = g.renorm;
  a.sel_mode = d.sel_mode;
  a.n_off_r = d.n_off_r;
  a.n_off_s = d.n_off_s;
  a.mask_r = d.mask_r;
  a.mask_s = d.mask_s;
  a.CM = decode_cand_rows(g.K);
  a.CH = d.CH;
  a.capture = d.capture ? 1 : 0;
  a.xb = d.xb;
  a.lf = d.lf;
  a.lm = d.lm;
  a.logits = d.logits;
  a.ids = d.ids;
  a.wts = d.wts;
  a.hc = reinterpret_cast<uint2*>(d.hc);
  a.part = d.part;
  a.ctr = d.ctr;
  a.y = d.y;
  a.h_cap = d.h_cap;
  a.inv = d.inv;
  a.perm = d.perm;
  a.row_expert = d.row_expert;
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.stream = ctx.stream;
  cfg.gridDim = dim3(n_sms);
  cfg.blockDim = dim3(kDecThreads);
  cfg.dynamicSmemBytes = kDecSmemBytes;
  cudaLaunchKernelEx(&cfg, decode_fused_kernel, *tmap_w, *tmap_xb, a);
  return 1;
}

}  // namespace skb
