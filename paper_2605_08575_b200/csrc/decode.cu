// decode.cu -- the whole layer for decode batches (B <= 4) as ONE persistent launch, software
// pipelined: the down projection of an expert runs while the gate/up weights of the next
// experts are still streaming.
//
// Why one kernel: at decode sizes the layer moves ~10-100 MB, i.e. 10-20 us of HBM time; every
// kernel boundary costs 2-3 us of drain + launch + refill, and a cold burst out of HBM ramps for
// ~3 us before it reaches full rate (tools/micro/burst.cu: 64 MB in 14 us, 16 MB in 5.5 us, by
// every access method).  So the stages of the reference path (proj/src/engine.cpp:94-191) are
// ROLES of one grid of numSMs CTAs (one per SM, all co-resident), each role on its own warps,
// chained through global memory:
//
//   warps 6-13 "D role" (256 threads)
//     P0  fast router logits, split over (expert, d_model slice) units on all CTAs: partial
//         lf = x.router and A = sum |x.router| per slice, published as {bits, epoch} words that the
//         readers poll (all words of a CTA in flight at once) -- no grid barrier.  The reference's
//         logit (ascending-index float accumulation, proj/src/linalg.cpp:22-40) differs from lf
//         by at most m = 2*gamma_D*A (gamma_D = D*u/(1-D*u), u = 2^-24).  Every expert whose
//         interval [lf-m, lf+m] reaches the K-th largest lower end is a CANDIDATE of the token;
//         the reference's top-K set is provably a subset.  Typically K candidates, sometimes K+1.
//         (More than K+4, non-finite values, or a threshold more than 60 below the maximum -- the
//         exp underflow region where probabilities tie -- and the CTA waits for the exact routing
//         instead.)
//     P2  neuron selection + down projection.  Work unit = (token, candidate, neuron-index
//         chunk), dealt round-robin in the order the experts finish.  The unit waits (one polite
//         poller) for its expert's piece counter, loads the h row, finds the pivot bucket from a
//         512-bin histogram and ranks only the bucket's members (bit-exact
//         mask_smallest_magnitudes, proj/src/activation.cpp:31-52, lower index first on ties),
//         and streams exactly the surviving W_down rows of its chunk with direct 128-bit loads,
//         16 in flight per thread, fp32 accumulation in registers.  Dropped neurons cost no HBM
//         bytes.
//     P3  combine: y[t] = sum_s w(t,s) * (sum_chunks partial), slots ascending, shared expert
//         last with weight 1 (proj/src/router.cpp:109-132, engine.cpp:168-173), fixed order.
//   warp 0 + warps 2-5 "G role": TMA producer, four consumer warps
//     gate/up + SwiGLU for the shared expert (streams from the first microsecond: it does not
//     depend on the routing) and then for the union of candidate experts, in EXPERT-MAJOR order
//     over all CTAs: a piece = 16 neurons (their 16 gate + 16 up rows) x all of d_model, read as
//     one 3-D TMA box {64 columns, 32 rows, 4 K-blocks} (16 KB) per ring stage out of the
//     128-row tiled image.  With at most 4 tokens the contraction is a GEMV: a tensor-core tile
//     would be 1/16 full and its operand staging (token tile TMA, UMMA issue, TMEM round trip)
//     only adds latency to a stream whose cost is HBM bytes, so the consumers are plain fp32 FMAs
//     straight out of the ring -- consumer warp w owns K-block w of every stage, lane l the
//     16-byte column piece l%8 of rows l/8 + 4i; the tokens sit in shared memory as bf16.  (The
//     batch kernels, gateup.cu, are the tcgen05 path.)  Expert u is complete -- and its down
//     projection starts -- after 1/n_u of the stream, not at its end.
//   warp 1 "CH role": exact routing.  The order-faithful logit chains (the D dependent float
//     adds of the reference) run on the last CTAs from the first microsecond; the last chain of
//     a token block runs route() (proj/src/router.cpp:13-68).  Ids, slot order and weights are
//     the reference's bit for bit; only P3 needs them.
//
// No float atomics anywhere: results are deterministic and, for a given shape, a token's result
// does not depend on the rest of the batch (the same FMA sequence per token for every batch size).
#include <cstdlib>
#include <mutex>

#include "route_device.cuh"
#include "select_device.cuh"
#include "tc_ptx.cuh"

namespace skb {

namespace {

constexpr int kDecThreads = 448;  // 14 warps
constexpr int kDThreads = 256;    // the D role: warps 6..13
constexpr int kWarpTma = 0, kWarpChain = 1, kWarpG0 = 2, kNumGWarps = 4, kWarpD0 = 6;
constexpr int kGThreads = kNumGWarps * 32;
constexpr int kDecMaxB = 4;  // more tokens per consumer lane than this spill (and the staged kernels win anyway)
constexpr int kDecTokens = 16;             // token stride of the row tables and of hc / part
constexpr int kKBox = 4;                   // K blocks per ring stage = consumer warps
constexpr int kStageBytes = kKBox * 32 * 128;  // 16 KB: 32 rows x 64 bf16 per K block
constexpr int kMaxStages = 8;
constexpr int kMinStages = 5;  // the exact-chain ring of the chain CTAs lives in the stage ring
constexpr int kHistBins = 512;
constexpr int kHistBase = (135 << 3) - (kHistBins - 1);  // top bin = |h| >= 2^8
constexpr int kMemberCap = 1024;
constexpr int kMaxN = 8192;  // N, S <= 8192

// exact-chain ring (chain CTAs only, in the stage ring's space): a unit is 8 experts x 4 tokens,
// 512-float sub-chunks as 1-D bulk copies of 2 KB (the TMA engine spends ~40 ns + 1 ns per 30
// bytes on a copy: short rows cost more than the chain they feed)
constexpr int kChSub = 512, kChStages = 3;
constexpr int kChRow = kChSub + 4;
constexpr int kChBytes = kChStages * 12 * kChRow * 4;  // 74304
static_assert(kChBytes <= kMinStages * kStageBytes, "the chain rings live in the stage ring");
constexpr int kMaxChainCtas = 16;

constexpr int kDecMaxE = 256;
constexpr int kDecMaxU = 256;  // union of candidate experts
constexpr int kMaxND = 8;      // d_model slices of the fast logits

// counters (unsigned words); everything but the epoch is back to zero when a launch ends
enum {
  kCtrEpoch = 0,
  kCtrDone = 1,
  kCtrExit = 2,
  kCtrRoute = 3,
  kCtrChain = 4,   // [4]
  kCtrCnt = 40,    // [1 + kDecMaxU] finished gate/up pieces: [0] shared expert, [1 + u] union expert u
  kCtrKept = kCtrCnt + 1 + kDecMaxU + 7,  // [16 * 20] threshold mode: survivors per candidate row
  kCtrWords = kCtrKept + 16 * 20
};

struct DecSmem {
  int ring, chain, gbuf, xs, gpart, keys, lst, hist, mlist, scr, gred, rowtab, uidx, ulist, cande,
      cmask, plist, rscr, bars, misc, total;
};
constexpr int kNumBars = 2 * kMaxStages + kChStages;
__host__ __device__ inline DecSmem dec_smem_layout(int stages, int gb_rows, int nmax, int tb, int Dp) {
  DecSmem m;
  const int nmax_pad = round_up(nmax, 256);
  int o = 0;
  m.ring = o;
  o += stages * kStageBytes;
  m.chain = m.ring;  // chain CTAs take no gate/up pieces
  m.gbuf = o;        // gb_rows rows of W_down staged by cp.async for the gather
  o += gb_rows * Dp * 2;
  m.xs = o;  // bf16 token rows [tb][Dp]
  o += round_up(tb * Dp * 2, 128);
  m.gpart = o;  // [2][4 warps][tb][32] partial gate/up sums of a piece
  o += 2 * kNumGWarps * tb * 32 * 4;
  m.keys = o;
  o += nmax_pad * 4;
  m.lst = o;
  o += nmax_pad * 2;
  m.hist = o;
  o += kHistBins * 4;
  m.mlist = o;
  o += (kMemberCap + 8) * 4;
  m.scr = o;
  o += 1024;
  m.gred = o;  // gather reduction [G][Dp] floats (8 KB); P0: polled partials [B*E*ND] float2
  o += 16384;
  m.rowtab = o;
  o += (kDecMaxU + 1) * 16 * 2 + 32;
  m.uidx = o;
  o += kDecMaxE * 2;
  m.ulist = o;
  o += kDecMaxU * 2;
  m.cande = o;
  o += 16 * 20 * 2;
  m.cmask = o;
  o += kDecMaxE * 4;
  m.plist = o;
  o += 352 * 2;
  m.rscr = o;
  o += 1152;
  m.bars = o;  // 8-byte aligned: every term above is a multiple of 8
  o += kNumBars * 8;
  m.misc = o;
  o += 64 * 4;
  m.total = o;
  return m;
}
// dynamic shared memory: 227 KB minus the kernel's static shared memory (< 1 KB) and the
// 1 KB alignment slack
constexpr int kSmemBudget = 227 * 1024 - 1024 - 1024;
inline int dec_tb_for(int B) { return B <= 1 ? 1 : (B <= 2 ? 2 : 4); }
// Split of what the fixed regions leave: a staging buffer of up to 80 KB of gathered W_down rows
// and kMinStages..kMaxStages ring stages (deeper rings only lengthen every other request's queue:
// 96 KB in flight per SM already saturates HBM, tools/micro/burst.cu).
struct DecPlan {
  int stages, gb_rows;
};
constexpr int kGbufMax = 80 * 1024;
inline DecPlan dec_plan(int nmax, int tb, int Dp) {
  const int room = kSmemBudget - dec_smem_layout(0, 0, nmax, tb, Dp).total;
  int st = (room - kGbufMax) / kStageBytes;
  if (st > kMaxStages) st = kMaxStages;
  if (st < kMinStages) st = kMinStages;
  int gb = room - st * kStageBytes;
  if (gb > kGbufMax) gb = kGbufMax;
  DecPlan p;
  p.stages = st;
  p.gb_rows = gb > 0 ? gb / (Dp * 2) : 0;
  return p;
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// One poller per CTA, probes back to back: a probe is an L2 round trip (~0.6 us) and 148 of them
// in flight are no load, while __nanosleep -- whatever its argument -- was measured to put the
// poller away for microseconds (the candidate exchange waited 3-6 us instead of ~1).
__device__ __forceinline__ void spin_until(const unsigned* p, unsigned target) {
  while (ld_acquire_u32(p) < target) {
  }
}
__device__ __forceinline__ uint2 ld_volatile_u2(const uint2* p) {
  uint2 v;
  asm volatile("ld.volatile.global.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_volatile_u2(uint2* p, uint32_t x, uint32_t y) {
  asm volatile("st.volatile.global.v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ uint4 ld_stream_u4(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* m, int c0, int c1, int c2,
                                            uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "l"(policy)
      : "memory");
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

// 8 bf16 -> 8 floats, element order
__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
  f[0] = __uint_as_float(u.x << 16);
  f[1] = __uint_as_float(u.x & 0xffff0000u);
  f[2] = __uint_as_float(u.y << 16);
  f[3] = __uint_as_float(u.y & 0xffff0000u);
  f[4] = __uint_as_float(u.z << 16);
  f[5] = __uint_as_float(u.z & 0xffff0000u);
  f[6] = __uint_as_float(u.w << 16);
  f[7] = __uint_as_float(u.w & 0xffff0000u);
}

// the D role's own barrier (256 threads, id 1); id 2 hands the candidate tables to the G role;
// id 3 is the consumer warps' barrier
__device__ __forceinline__ void d_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
__device__ __forceinline__ void g_sync() { asm volatile("bar.sync 3, 128;" ::: "memory"); }
struct SelDRole {
  __device__ static __forceinline__ int tid() { return threadIdx.x - kWarpD0 * 32; }
  __device__ static __forceinline__ void sync() { d_sync(); }
};
// (two barriers, so that the producer does not wait for the consumers' token staging)
__device__ __forceinline__ void tables_arrive() {
  asm volatile("bar.arrive 2, %0;" ::"n"(kDThreads + 32) : "memory");
  asm volatile("bar.arrive 4, %0;" ::"n"(kDThreads + kGThreads) : "memory");
}
__device__ __forceinline__ void tables_wait_producer() {
  asm volatile("bar.sync 2, %0;" ::"n"(kDThreads + 32) : "memory");
}
__device__ __forceinline__ void tables_wait_consumers() {
  asm volatile("bar.sync 4, %0;" ::"n"(kDThreads + kGThreads) : "memory");
}

}  // namespace

#ifdef SKB_DEBUG_TIMING
__device__ long long g_dec_dbg[160 * 32];
__device__ __forceinline__ long long dec_gtime() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// stamp i of this CTA, by thread `thr`: the SM's cycle counter (reading %globaltimer costs about a
// microsecond); stamp 0 records {globaltimer, clock64} once, which places the CTA on the common axis
#define DEC_STAMP(thr, i) do { if (threadIdx.x == (thr)) { if ((i) == 0) { g_dec_dbg[blockIdx.x * 32] = dec_gtime(); g_dec_dbg[blockIdx.x * 32 + 31] = clock64(); } else g_dec_dbg[blockIdx.x * 32 + (i)] = clock64(); } } while (0)
extern "C" void skb_debug_dec(long long* out) { cudaMemcpyFromSymbol(out, g_dec_dbg, sizeof(g_dec_dbg)); }
#else
#define DEC_STAMP(thr, i) do { } while (0)
#endif

struct DecodeArgs {
  const float* x;
  const float* router;
  const __nv_bfloat16* wd;
  const __nv_bfloat16* wd_shared;
  int B, E, K, D, Dp, N, Np, S, Sp, Nh, has_shared, renorm;
  int sel_mode, n_off_r, n_off_s;
  float tau;                     // kSelectThreshold: a routed neuron is kept iff |silu(g)| >= tau
  const __nv_bfloat16* wu;       // W_up rows [E][Np][Dp], row-major (threshold mode gathers them)
  int32_t* kcnt;                 // kSelectThreshold: survivors per flat slot [B*K]
  const uint8_t* mask_r;
  const uint8_t* mask_s;
  int CM, CH, capture, stages, gb_rows, ND, DS;
  int n_ch;  // dedicated chain CTAs (the last n_ch of the grid): no gate/up pieces, no P2 units
  uint2* p0;  // [B][E][ND][2] of {bits, epoch}: partial fast logit and partial sum of |products|
  float* logits;
  int32_t* ids;
  float* wts;
  float* hc;  // [16 * CM + 16][Nh] activations of the candidate rows
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
// the K-th largest lower end.  pf[e * stride + j] = {fast logit, sum of |products|} partials of
// the token's `stride` d_model slices, summed here in slice order (every CTA forms the same
// sums, hence the same candidate sets).  Returns true when the bound cannot be used (non-finite values, the exp-underflow
// region, or more than CM candidates): the caller then waits for the exact routing.
// VPL = experts per lane.
template <int VPL>
__device__ __forceinline__ bool cand_token(const float2* pf, int stride, int E, float mfac, int K,
                                           int CM, int t, uint32_t* cmask) {
  const int lane = threadIdx.x & 31;
  uint32_t lo[VPL];
  float hi[VPL];
  bool bad = false;
  uint32_t mxk = 0u;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int e = i * 32 + lane;
    if (e < E) {
      float f = 0.0f, sa = 0.0f;  // slice partials summed in slice order
#pragma unroll 1
      for (int j = 0; j < stride; ++j) {
        const float2 v = pf[static_cast<size_t>(e) * stride + j];
        f = __fadd_rn(f, v.x);
        sa = __fadd_rn(sa, v.y);
      }
      const float m = sa * mfac + 2e-5f;
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

// the general search behind the histogram pick (huge pivot buckets only): out of line, so that the
// path every launch takes stays short
__device__ __noinline__ RowPick kary_pick_cold(const uint32_t* keys, int n, int n_off, SelScratch& sc) {
  return sel_kary_pick<SelDRole>(keys, n, n_off, sc);
}

template <int TB>
__global__ void __launch_bounds__(kDecThreads, 1)
decode_fused_kernel(const __grid_constant__ CUtensorMap tmap_w3,
                    const __grid_constant__ CUtensorMap tmap_w3g, const DecodeArgs a) {
  extern __shared__ uint8_t dsm_raw[];
  uint8_t* sm = dsm_raw + ((1024u - (smem_u32(dsm_raw) & 1023u)) & 1023u);
  const uint32_t sm_u32 = smem_u32(sm);
  const int nmax = a.N > a.S ? a.N : a.S;
  const DecSmem L = dec_smem_layout(a.stages, a.gb_rows, nmax, TB, a.Dp);
  int16_t* rowtab = reinterpret_cast<int16_t*>(sm + L.rowtab);
  int16_t* uidx = reinterpret_cast<int16_t*>(sm + L.uidx);
  int16_t* ulist = reinterpret_cast<int16_t*>(sm + L.ulist);
  int16_t* cande = reinterpret_cast<int16_t*>(sm + L.cande);
  uint32_t* cmask = reinterpret_cast<uint32_t*>(sm + L.cmask);
  int16_t* plist = reinterpret_cast<int16_t*>(sm + L.plist);
  int* misc = reinterpret_cast<int*>(sm + L.misc);
  // misc: 1 overflow flag, 2 n_u, 3 n_pairs, 8.. unit scalars, 24.. ncand[16]
  int* ncand = misc + 24;
  const uint32_t bar0 = sm_u32 + L.bars;
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 8u * (kMaxStages + s); };
  auto cfull_bar = [&](int s) { return bar0 + 8u * (2 * kMaxStages + s); };
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grid = gridDim.x, bid = blockIdx.x;
  const int B = a.B, E = a.E, K = a.K, D = a.D, Dp = a.Dp, CM = a.CM, CH = a.CH;
  constexpr int ch_tb = 4, ch_eb = 8;  // chain unit shape (lane = expert * 4 + token)
  const int n_tb = ceil_div(B, ch_tb), n_eb = ceil_div(E, ch_eb);
  const int gwn = grid - a.n_ch;       // worker CTAs: gate/up pieces and P2 units
  const bool worker = bid < gwn;
  const int stages = a.stages;
  const bool vec_ok = (D % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0) &&
                      ((reinterpret_cast<uintptr_t>(a.router) & 15) == 0);
  // tag of this launch's P0 partials; issued first, consumed late
  const uint32_t epoch = *reinterpret_cast<volatile const unsigned*>(&a.ctr[kCtrEpoch]) + 1u;

  DEC_STAMP(0, 0);
  // ---- prologue ----
  if (tid < stages) {
    mbar_init(full_bar(tid), 1);
    mbar_init(empty_bar(tid), kNumGWarps);
    if (tid < kChStages) mbar_init(cfull_bar(tid), 1);
    fence_barrier_init();
    if (tid == 0) {
      tma_prefetch_desc(&tmap_w3);
      misc[1] = 0;
      misc[4] = 0;  // consumer warps that are through with the ring (threshold mode reuses it)
    }
  }
  for (int e = tid; e < kDecMaxE; e += kDecThreads) cmask[e] = 0u;
  {
    // row table: -1 = (expert, token) is not a candidate pair; at most B * CM union experts
    uint32_t* rt32 = reinterpret_cast<uint32_t*>(rowtab);
    for (int i = tid; i < (kDecMaxB * 20 + 1) * 8; i += kDecThreads) rt32[i] = 0xffffffffu;
  }
  __syncthreads();

  const int NB = a.Np / kNeuronBlock, NBs = a.has_shared ? a.Sp / kNeuronBlock : 0;
  const int KB = Dp / kBlockK;
  const int KX = ceil_div(KB, kKBox);       // ring stages per piece
  const int PE = 4 * NB;                    // pieces per routed expert
  const int n_sh = 4 * NBs;                 // pieces of the shared expert (come first)
  constexpr int kStoreWarps = (16 * TB + 31) / 32;  // consumer warps that store h of a piece
  // Threshold mode (forward_sparse, engine.cpp:229-369): the routed experts stream their GATE
  // rows only -- a piece is the 2 x 16 gate rows of two tile quarters (32 neurons), two TMA boxes
  // of 16 rows per stage; the up rows are gathered later, only for the surviving neurons.
  const bool thr = a.sel_mode == kSelectThreshold;
  const int PEr = thr ? 2 * NB : PE;                 // pieces per routed expert
  constexpr int kStoreWarpsG = TB;                   // threshold pieces: 32 x TB outputs

  if (warp == kWarpTma) {
    // =====================================================================================
    // G role, producer: one 3-D box of the weight image per stage
    // =====================================================================================
    int gk = 0, p = worker ? bid : 0x3fffffff;
    auto produce = [&](int rb, int q) {
#pragma unroll 1
      for (int kx = 0; kx < KX; ++kx, ++gk) {
        const int s = gk % stages;
        mbar_wait(empty_bar(s), ((gk / stages) & 1u) ^ 1u);
        mbar_arrive_expect_tx(full_bar(s), kStageBytes);
        tma_load_3d(sm_u32 + L.ring + s * kStageBytes, &tmap_w3, 0, q * 32, rb * KB + kx * kKBox,
                    full_bar(s), kPolicyEvictFirst);
      }
    };
    if (lane == 0) {
#pragma unroll 1
      for (; p < n_sh; p += gwn) produce(E * NB + (p >> 2), p & 3);
    }
    __syncwarp();
    tables_wait_producer();
    if (lane == 0) {
      const int n_u = misc[2];
      DEC_STAMP(0, 11);
#pragma unroll 1
      for (; p < n_sh + n_u * PEr; p += gwn) {
        const int pr = p - n_sh;
        const int u = pr / PEr, qq = pr % PEr;
        if (!thr) {
          produce(static_cast<int>(ulist[u]) * NB + (qq >> 2), qq & 3);
        } else {
          const int rb = static_cast<int>(ulist[u]) * NB + (qq >> 1), hq = qq & 1;
#pragma unroll 1
          for (int kx = 0; kx < KX; ++kx, ++gk) {
            const int s = gk % stages;
            mbar_wait(empty_bar(s), ((gk / stages) & 1u) ^ 1u);
            mbar_arrive_expect_tx(full_bar(s), kStageBytes);
            const uint32_t dst = sm_u32 + L.ring + s * kStageBytes;
            tma_load_3d(dst, &tmap_w3g, 0, (2 * hq) * 32, rb * KB + kx * kKBox, full_bar(s),
                        kPolicyEvictFirst);
            tma_load_3d(dst + kStageBytes / 2, &tmap_w3g, 0, (2 * hq + 1) * 32, rb * KB + kx * kKBox,
                        full_bar(s), kPolicyEvictFirst);
          }
        }
      }
      DEC_STAMP(0, 3);
    }
  } else if (warp >= kWarpG0 && warp < kWarpG0 + kNumGWarps) {
    // =====================================================================================
    // G role, consumers: warp gw owns K block gw of every stage; lane l holds the 16-byte
    // column piece l % 8 of the rows l / 8 + 4 i (i < 8; rows 0-15 gate, 16-31 up).  Per token
    // the FMA sequence is the same for every batch size.
    // =====================================================================================
    const int gw = warp - kWarpG0, gtid = tid - kWarpG0 * 32;
    __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(sm + L.xs);
    if (!worker) {
      // chain CTA: nothing to stage
    } else if (vec_ok) {
      // four 16-byte loads in flight per thread (a dependent load per element would cost a cold
      // miss each)
      const int q4 = Dp / 4, tot4 = TB * q4;
#pragma unroll 1
      for (int i0 = gtid; i0 < tot4; i0 += 4 * kGThreads) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + u * kGThreads;
          const int t = i / q4, d = (i - t * q4) * 4;
          v[u] = (i < tot4 && t < B && d < D)
                     ? __ldg(reinterpret_cast<const float4*>(a.x + static_cast<size_t>(t) * D + d))
                     : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + u * kGThreads;
          if (i < tot4) {
            __nv_bfloat162* dst = reinterpret_cast<__nv_bfloat162*>(xs) + 2 * i;
            dst[0] = __floats2bfloat162_rn(v[u].x, v[u].y);
            dst[1] = __floats2bfloat162_rn(v[u].z, v[u].w);
          }
        }
      }
    } else {
      for (int i = gtid; i < TB * Dp; i += kGThreads) {
        const int t = i / Dp, d = i - t * Dp;
        const float v = (t < B && d < D) ? __ldg(a.x + static_cast<size_t>(t) * D + d) : 0.0f;
        xs[i] = __float2bfloat16_rn(v);
      }
    }
    g_sync();
    DEC_STAMP(kWarpG0 * 32, 16);
    float* gpart = reinterpret_cast<float*>(sm + L.gpart);
    const int c8 = lane & 7, rq = lane >> 3;
    constexpr int TG = TB < 4 ? TB : 4;
    int gk = 0, li = 0, p = worker ? bid : 0x3fffffff;
    auto do_piece = [&](int u /* -1: shared */, int nb, int q, int m_valid, bool gate_only) {
      // stage layout: one box of 32 rows per plane, or two boxes of 16 gate rows
      const int plane_stride = gate_only ? 2048 : 4096, half_stride = gate_only ? kStageBytes / 2 : 2048;
      float acc[8][TB];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int t = 0; t < TB; ++t) acc[i][t] = 0.0f;
#pragma unroll 1
      for (int kx = 0; kx < KX; ++kx, ++gk) {
        const int s = gk % stages;
        mbar_wait(full_bar(s), (gk / stages) & 1u);
        const int kb = kx * kKBox + gw;
        if (kb < KB) {
          const uint8_t* wp = sm + L.ring + s * kStageBytes + gw * plane_stride + lane * 16;
          uint4 wv[8];
#pragma unroll
          for (int i = 0; i < 8; ++i)
            wv[i] = *reinterpret_cast<const uint4*>(wp + (i >> 2) * half_stride + (i & 3) * 512);
#pragma unroll
          for (int tg = 0; tg < TB; tg += TG) {
            float xf[TG][8];
#pragma unroll
            for (int tt = 0; tt < TG; ++tt) {
              const uint4 xv = *reinterpret_cast<const uint4*>(xs + static_cast<size_t>(tg + tt) * Dp +
                                                               kb * kBlockK + c8 * 8);
              unpack8(xv, xf[tt]);
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              float wf[8];
              unpack8(wv[i], wf);
#pragma unroll
              for (int tt = 0; tt < TG; ++tt)
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[i][tg + tt] = fmaf(wf[e], xf[tt][e], acc[i][tg + tt]);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty_bar(s));
      }
      // sum over the 8 lanes of a row: butterfly that leaves row 4*b2 + 2*b1 + b0 on lane bits
      // (b2 b1 b0) of every group of 8 -- 7 shuffles per token instead of 24, fixed order
      const int buf = li & 1;
      const bool b2 = (lane & 4) != 0, b1 = (lane & 2) != 0, b0 = (lane & 1) != 0;
      const int myrow = 4 * ((b2 ? 4 : 0) + (b1 ? 2 : 0) + (b0 ? 1 : 0)) + rq;
#pragma unroll
      for (int t = 0; t < TB; ++t) {
        float v4[4], v2[2];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float keep = b2 ? acc[4 + k][t] : acc[k][t];
          const float send = b2 ? acc[k][t] : acc[4 + k][t];
          v4[k] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const float keep = b1 ? v4[2 + k] : v4[k];
          const float send = b1 ? v4[k] : v4[2 + k];
          v2[k] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
        }
        const float keep = b0 ? v2[1] : v2[0];
        const float send = b0 ? v2[0] : v2[1];
        gpart[((buf * kNumGWarps + gw) * TB + t) * 32 + myrow] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
      }
      g_sync();
      if (gate_only) {
        // 32 gate rows = 32 consecutive neurons: store silu(g), the value the mask is taken of
        if (gw < kStoreWarpsG) {
          const int j = lane, t = gw;
          const float* gp = gpart + (buf * kNumGWarps * TB + t) * 32;
          float g = gp[j];
#pragma unroll
          for (int w = 1; w < kNumGWarps; ++w) g = __fadd_rn(g, gp[w * TB * 32 + j]);
          const int n = nb * kNeuronBlock + 32 * q + j;
          if (t < B && n < m_valid) {
            const int r = rowtab[u * 16 + t];
            if (r >= 0) a.hc[static_cast<size_t>(r) * a.Nh + n] = silu_f(g);
          }
          __threadfence();
          __syncwarp();
          if (lane == 0) atomicAdd(&a.ctr[kCtrCnt + 1 + u], 1u);
        }
      } else if (gw < kStoreWarps) {
        if (gtid < 16 * TB) {
          const int j = gtid & 15, t = gtid >> 4;
          const float* gp = gpart + (buf * kNumGWarps * TB + t) * 32;
          float g = gp[j], up = gp[16 + j];
#pragma unroll
          for (int w = 1; w < kNumGWarps; ++w) {
            g = __fadd_rn(g, gp[w * TB * 32 + j]);
            up = __fadd_rn(up, gp[w * TB * 32 + 16 + j]);
          }
          const int n = nb * kNeuronBlock + 16 * q + j;
          if (t < B && n < m_valid) {
            const int r = u < 0 ? kDecTokens * CM + t : rowtab[u * 16 + t];
            if (r >= 0) a.hc[static_cast<size_t>(r) * a.Nh + n] = silu_f(g) * up;
          }
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(&a.ctr[kCtrCnt + 1 + u], 1u);
      }
      ++li;
    };
#pragma unroll 1
    for (; p < n_sh; p += gwn) do_piece(-1, p >> 2, p & 3, a.S, false);
    tables_wait_consumers();
    DEC_STAMP(kWarpG0 * 32, 17);
    const int n_u = misc[2];
#pragma unroll 1
    for (; p < n_sh + n_u * PEr; p += gwn) {
      const int pr = p - n_sh;
      const int u = pr / PEr, qq = pr % PEr;
      if (thr)
        do_piece(u, qq >> 1, qq & 1, a.N, true);
      else
        do_piece(u, qq >> 2, qq & 3, a.N, false);
      if (p == bid + ((n_sh + gwn - 1 - bid) / gwn) * gwn) DEC_STAMP(kWarpG0 * 32, 18);
    }
    // this warp has read its last ring stage: once all consumer warps say so, the D role may
    // stage gathered rows in the ring (threshold mode, below)
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      atomicAdd(&misc[4], 1);
    }
    DEC_STAMP(kWarpG0 * 32, 4);
  } else if (warp == kWarpChain) {
    // =====================================================================================
    // Exact routing chains on the LAST n_ch CTAs of the grid, which do nothing else (next to
    // streaming warps a dependent-add chain runs three times slower), one warp of 32 dependent
    // chains (8 experts x 4 tokens) behind a ring of 1-D bulk copies, one row per lane.  They
    // only read x and the router, so they start right away; their result is needed by P3 (and by
    // caller-mask lookups).
    // =====================================================================================
    float* ring = reinterpret_cast<float*>(sm + L.chain);   // [stages][rows][kChRow]
    float* fring = ring;                                    // unaligned operands: [rows][kChRow]
    const int n_cu = n_eb * n_tb;
    const int nsub = ceil_div(D, kChSub);
    const int ch_rows = ch_eb + ch_tb;
    int gsc = 0;  // ring position, continues across units
#pragma unroll 1
    for (int cu = worker ? n_cu : bid - gwn; cu < n_cu; cu += a.n_ch) {
      const int eb = cu % n_eb, tb = cu / n_eb;
      const int e0 = eb * ch_eb, t0 = tb * ch_tb;
      const int n_e = min(ch_eb, E - e0), n_t = min(ch_tb, B - t0);
      const int e_i = lane / ch_tb, t_j = lane % ch_tb;
      const bool valid = (e_i < n_e) && (t_j < n_t);
      const float* wsrc = a.router + static_cast<size_t>(e0) * D;
      const float* xsrc = a.x + static_cast<size_t>(t0) * D;
      float acc = 0.0f;
      DEC_STAMP(kWarpChain * 32, 14);
      if (vec_ok) {
        // the whole warp: sub-chunk sc of this unit into its ring slot, one row per lane
        auto issue = [&](int sc, int gidx) {
          const int slot = gidx % kChStages;
          const int d0 = sc * kChSub;
          const uint32_t bytes = static_cast<uint32_t>(min(kChSub, D - d0)) * 4u;
          if (lane == 0) mbar_arrive_expect_tx(cfull_bar(slot), bytes * static_cast<uint32_t>(n_e + n_t));
          __syncwarp();
          const uint32_t dst = smem_u32(ring + slot * ch_rows * kChRow);
          if (lane < n_e)
            bulk_copy_g2s(dst + lane * kChRow * 4, wsrc + static_cast<size_t>(lane) * D + d0, bytes,
                          cfull_bar(slot));
          else if (lane - n_e < n_t)
            bulk_copy_g2s(dst + (ch_eb + lane - n_e) * kChRow * 4,
                          xsrc + static_cast<size_t>(lane - n_e) * D + d0, bytes, cfull_bar(slot));
        };
        for (int sc = 0; sc < nsub && sc < kChStages; ++sc) issue(sc, gsc + sc);
        __syncwarp();
#pragma unroll 1
        for (int sc = 0; sc < nsub; ++sc) {
          const int gidx = gsc + sc;
          const int slot = gidx % kChStages;
          const float* base = ring + slot * ch_rows * kChRow;
          const int n4 = min(kChSub, D - sc * kChSub) >> 2;
          mbar_wait(cfull_bar(slot), (gidx / kChStages) & 1u);
          const float4* wr = reinterpret_cast<const float4*>(base + min(e_i, n_e - 1) * kChRow);
          const float4* xr = reinterpret_cast<const float4*>(base + (ch_eb + min(t_j, n_t - 1)) * kChRow);
          int q = 0;
#pragma unroll 1
          for (; q + 8 <= n4; q += 8) {
            // every operand of 32 elements in registers first, then the 32 dependent adds
            float4 w[8], xv[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              w[j] = wr[q + j];
              xv[j] = xr[q + j];
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              acc = __fadd_rn(acc, __fmul_rn(w[j].x, xv[j].x));
              acc = __fadd_rn(acc, __fmul_rn(w[j].y, xv[j].y));
              acc = __fadd_rn(acc, __fmul_rn(w[j].z, xv[j].z));
              acc = __fadd_rn(acc, __fmul_rn(w[j].w, xv[j].w));
            }
          }
#pragma unroll 1
          for (; q < n4; ++q) {
            const float4 w = wr[q], xv = xr[q];
            acc = __fadd_rn(acc, __fmul_rn(w.x, xv.x));
            acc = __fadd_rn(acc, __fmul_rn(w.y, xv.y));
            acc = __fadd_rn(acc, __fmul_rn(w.z, xv.z));
            acc = __fadd_rn(acc, __fmul_rn(w.w, xv.w));
          }
          __syncwarp();  // every lane is done with the slot: refill it
          if (sc + kChStages < nsub) issue(sc + kChStages, gidx + kChStages);
        }
        gsc += nsub;
      } else {
        // unaligned operands: the warp stages each sub-chunk itself
        const float* wsrc = a.router + static_cast<size_t>(e0) * D;
#pragma unroll 1
        for (int sc = 0; sc < nsub; ++sc) {
          const int d0 = sc * kChSub;
          const int n = min(kChSub, D - d0);
#pragma unroll 1
          for (int r = 0; r < n_e + n_t; ++r) {
            const float* src = (r < n_e) ? wsrc + static_cast<size_t>(r) * D + d0
                                         : xsrc + static_cast<size_t>(r - n_e) * D + d0;
            float* drow = fring + ((r < n_e) ? r : ch_eb + r - n_e) * kChRow;
#pragma unroll 1
            for (int i = lane; i < n; i += 32) drow[i] = __ldg(src + i);
          }
          __syncwarp();
          const float* wr = fring + min(e_i, n_e - 1) * kChRow;
          const float* xr = fring + (ch_eb + min(t_j, n_t - 1)) * kChRow;
#pragma unroll 4
          for (int i = 0; i < n; ++i) acc = __fadd_rn(acc, __fmul_rn(wr[i], xr[i]));
          __syncwarp();
        }
      }
      DEC_STAMP(kWarpChain * 32, 15);
      if (valid) a.logits[static_cast<size_t>(t0 + t_j) * E + e0 + e_i] = acc;
      __threadfence();
      __syncwarp();
      unsigned prev = 0;
      if (lane == 0) prev = atomicAdd(&a.ctr[kCtrChain + tb], 1u);
      prev = __shfl_sync(0xffffffffu, prev, 0);
      if (prev == static_cast<unsigned>(n_eb - 1)) {
        // last chain of this token block: route() for its tokens
        __threadfence();
        float* scr = reinterpret_cast<float*>(sm + L.rscr);
#pragma unroll 1
        for (int tt = 0; tt < n_t; ++tt) {
          const int t = t0 + tt;
          warp_route_token(a.logits + static_cast<size_t>(t) * E, E, K, a.renorm, scr,
                           a.ids + static_cast<size_t>(t) * K, a.wts + static_cast<size_t>(t) * K);
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(&a.ctr[kCtrRoute], 1u);
        DEC_STAMP(kWarpChain * 32, 10);
      }
    }
  } else {
    // =====================================================================================
    // D role (warps 6..13)
    // =====================================================================================
    const int dtid = tid - kWarpD0 * 32, dwarp = dtid >> 5;
    uint32_t* keys_s = reinterpret_cast<uint32_t*>(sm + L.keys);
    uint16_t* lst = reinterpret_cast<uint16_t*>(sm + L.lst);
    int* hist_s = reinterpret_cast<int*>(sm + L.hist);
    uint32_t* mlist = reinterpret_cast<uint32_t*>(sm + L.mlist);
    int* wc = reinterpret_cast<int*>(sm + L.scr);  // [8] warp counts, [8..16) second set
    float* gred = reinterpret_cast<float*>(sm + L.gred);
    int* p2 = misc + 8;  // 2 b*, 3 below_bins, 4 M, 5 pivot, 6 below, 7 equal, 8 mcount

    // ---- P0: fast logits of (expert, d_model slice) units ----
    const int ND = a.ND, DS = a.DS;
    {
      constexpr int TT = TB < 4 ? TB : 4;  // tokens per pass
      float* red = gred;  // [8 warps][TT tokens][2]
#pragma unroll 1
      for (int unit = bid; unit < E * ND; unit += grid) {
        const int e = unit / ND, j = unit % ND;
        const int d0 = j * DS, d1 = min(D, d0 + DS);
        const float* wr = a.router + static_cast<size_t>(e) * D;
#pragma unroll 1
        for (int t0 = 0; t0 < B; t0 += TT) {
          float pl[TT], pa[TT];
#pragma unroll
          for (int tt = 0; tt < TT; ++tt) pl[tt] = pa[tt] = 0.0f;
          if (vec_ok) {
            const float4* w4 = reinterpret_cast<const float4*>(wr);
#pragma unroll 2
            for (int q = d0 / 4 + dtid; q < d1 / 4; q += kDThreads) {
              const float4 w = __ldg(w4 + q);
#pragma unroll
              for (int tt = 0; tt < TT; ++tt) {
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
            for (int d = d0 + dtid; d < d1; d += kDThreads) {
              const float w = __ldg(wr + d);
#pragma unroll
              for (int tt = 0; tt < TT; ++tt) {
                if (t0 + tt < B) {
                  const float xv = __ldg(a.x + static_cast<size_t>(t0 + tt) * D + d);
                  pl[tt] = fmaf(w, xv, pl[tt]);
                  pa[tt] = fmaf(fabsf(w), fabsf(xv), pa[tt]);
                }
              }
            }
          }
#pragma unroll
          for (int tt = 0; tt < TT; ++tt) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              pl[tt] += __shfl_xor_sync(0xffffffffu, pl[tt], o);
              pa[tt] += __shfl_xor_sync(0xffffffffu, pa[tt], o);
            }
            if (lane == 0) {
              red[(dwarp * TT + tt) * 2 + 0] = pl[tt];
              red[(dwarp * TT + tt) * 2 + 1] = pa[tt];
            }
          }
          d_sync();
          if (dtid < TT && t0 + dtid < B) {
            float s = 0.0f, sa = 0.0f;
#pragma unroll
            for (int w = 0; w < kDThreads / 32; ++w) {
              s += red[(w * TT + dtid) * 2 + 0];
              sa += red[(w * TT + dtid) * 2 + 1];
            }
            uint2* dst = a.p0 + ((static_cast<size_t>(t0 + dtid) * E + e) * ND + j) * 2;
            // published with 64-bit exchanges: performed at L2 at once
            atomicExch(reinterpret_cast<unsigned long long*>(dst),
                       (static_cast<unsigned long long>(epoch) << 32) | __float_as_uint(s));
            atomicExch(reinterpret_cast<unsigned long long*>(dst + 1),
                       (static_cast<unsigned long long>(epoch) << 32) | __float_as_uint(sa));
          }
          d_sync();
        }
      }
    }
    DEC_STAMP(kWarpD0 * 32, 1);

    // ---- candidates (every CTA computes the same tables) ----
    DEC_STAMP(kWarpD0 * 32, 26);
    {
      // every partial of every token: all of this thread's words in flight before the first check
      float2* pf = reinterpret_cast<float2*>(gred);
      const int total = B * E * ND;
#pragma unroll 1
      for (int base = 0; base < total; base += kDThreads * 4) {
        uint2 va[4], vb[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = base + u * kDThreads + dtid;
          if (i < total) {
            va[u] = ld_volatile_u2(a.p0 + 2 * static_cast<size_t>(i));
            vb[u] = ld_volatile_u2(a.p0 + 2 * static_cast<size_t>(i) + 1);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = base + u * kDThreads + dtid;
          if (i < total) {
            DEC_STAMP(kWarpD0 * 32, 27);
            while (va[u].y != epoch) va[u] = ld_volatile_u2(a.p0 + 2 * static_cast<size_t>(i));
            while (vb[u].y != epoch) vb[u] = ld_volatile_u2(a.p0 + 2 * static_cast<size_t>(i) + 1);
            pf[i] = make_float2(__uint_as_float(va[u].x), __uint_as_float(vb[u].x));
          }
        }
      }
      d_sync();
      DEC_STAMP(kWarpD0 * 32, 21);
      // margin = 2 * gamma_D * A, a little inflated for the rounding of A itself
      const float u24 = 5.9604644775390625e-8f;
      const float mfac = 2.02f * (D * u24) / (1.0f - D * u24);
      DEC_STAMP(kWarpD0 * 32, 24);
      if (dwarp < B) {
        const int t = dwarp;
        const float2* pft = pf + static_cast<size_t>(t) * E * ND;
        bool bad;
        if (E <= 64)
          bad = cand_token<2>(pft, ND, E, mfac, K, CM, t, cmask);
        else if (E <= 128)
          bad = cand_token<4>(pft, ND, E, mfac, K, CM, t, cmask);
        else
          bad = cand_token<8>(pft, ND, E, mfac, K, CM, t, cmask);
        if (bad && lane == 0) misc[1] = 1;
      }
      DEC_STAMP(kWarpD0 * 32, 25);
      d_sync();
      if (misc[1] != 0) {
        // rare: the bound could not separate the candidates -- wait for the exact routing
        if (dtid == 0) spin_until(&a.ctr[kCtrRoute], static_cast<unsigned>(n_tb));
        d_sync();
        for (int e = dtid; e < E; e += kDThreads) cmask[e] = 0u;
        d_sync();
        for (int i = dtid; i < B * K; i += kDThreads) atomicOr(&cmask[__ldcg(a.ids + i)], 1u << (i / K));
        d_sync();
      }
      DEC_STAMP(kWarpD0 * 32, 22);
      // tables: warp t walks the experts once for token t -- position in the union of candidate
      // experts (ascending id; every warp forms the same positions, warp 0 records them) and rank
      // among the token's own candidates
      {
        const int t = dwarp;
        const unsigned lt = (1u << lane) - 1u;
        int run_u = 0, run_t = 0;
#pragma unroll 1
        for (int base = 0; base < E; base += 32) {
          const int e = base + lane;
          const uint32_t cm = e < E ? cmask[e] : 0u;
          const unsigned bu = __ballot_sync(0xffffffffu, cm != 0u);
          const int upos = run_u + __popc(bu & lt);
          if (t == 0 && e < E) {
            uidx[e] = cm != 0u ? static_cast<int16_t>(upos) : static_cast<int16_t>(-1);
            if (cm != 0u) ulist[upos] = static_cast<int16_t>(e);
          }
          if (t < B) {
            const bool f = ((cm >> t) & 1u) != 0u;
            const unsigned bt = __ballot_sync(0xffffffffu, f);
            if (f) {
              const int r = run_t + __popc(bt & lt);
              rowtab[upos * 16 + t] = static_cast<int16_t>(t * CM + r);
              cande[t * CM + r] = static_cast<int16_t>(e);
            }
            run_t += __popc(bt);
          }
          run_u += __popc(bu);
        }
        if (lane == 0) {
          if (t == 0) misc[2] = run_u;
          if (t < B) ncand[t] = run_t;
        }
      }
      d_sync();
      tables_arrive();  // the G role may stream the routed experts now
      DEC_STAMP(kWarpD0 * 32, 2);
      // pair list in the order the experts finish: shared expert first, then union order
      if (dwarp == 0) {
        const int n_u = misc[2];
        int run = 0;
        if (a.has_shared) {
          if (lane < B) plist[lane] = static_cast<int16_t>(n_u * 16 + lane);
          run = B;
        }
#pragma unroll 1
        for (int base = 0; base < n_u; base += 32) {
          const int u = base + lane;
          uint32_t cm = u < n_u ? cmask[ulist[u]] : 0u;
          const int cnt = __popc(cm);
          int incl = cnt;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
          }
          int pos = run + incl - cnt;
          while (cm != 0u) {
            const int t = __ffs(cm) - 1;
            cm &= cm - 1u;
            plist[pos++] = static_cast<int16_t>(u * 16 + t);
          }
          run += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) misc[3] = run;
      }
      d_sync();
    }

    // ---- P2: selection + down projection over (pair, neuron-index chunk) units ----
    {
      const int n_u = misc[2];
      const int n_units = misc[3] * CH;
      const int LPR = Dp >> 3;
      const int NT = ceil_div(LPR, 256);
      const int G = NT == 1 ? 256 / LPR : 1;
      const int g = NT == 1 ? dtid / LPR : 0, l = NT == 1 ? dtid % LPR : dtid;
      const bool lane_ok = g < G;
      bool route_ready = false;
      __shared__ SelScratch sel_sc;
      // units are dealt from the CTA after the one that took the last gate/up piece
      const int v_first = worker ? (bid - (n_sh + n_u * PEr) % gwn + gwn) % gwn : n_units;
#pragma unroll 1
      for (int v = v_first; v < n_units; v += gwn) {
        const int pu = plist[v / CH], c = v % CH;
        const int u = pu >> 4, t = pu & 15;
        const bool routed = u < n_u;
        const int row = routed ? rowtab[pu] : kDecTokens * CM + t;
        const int e = routed ? ulist[u] : E;
        const int q = routed ? row - t * CM : CM;
        const int n = routed ? a.N : a.S;
        int mode = a.sel_mode;
        const uint8_t* min_ = nullptr;
        if (mode == kSelectGiven) {
          int slot = t;
          if (routed) {
            // caller masks are indexed by slot: the exact routing is needed here
            if (!route_ready) {
              if (dtid == 0) spin_until(&a.ctr[kCtrRoute], static_cast<unsigned>(n_tb));
              d_sync();
              route_ready = true;
            }
            slot = -1;
            for (int j = 0; j < K; ++j)
              if (__ldcg(a.ids + t * K + j) == e) slot = t * K + j;
            min_ = slot >= 0 ? a.mask_r + static_cast<size_t>(slot) * n : nullptr;
            if (slot < 0) mode = -1;  // a candidate the exact routing rejected: nothing to do
          } else {
            min_ = a.mask_s ? a.mask_s + static_cast<size_t>(slot) * n : nullptr;
            if (min_ == nullptr) mode = kSelectAll;
          }
        }
        if (mode == kSelectThreshold && !routed) mode = kSelectAll;  // the shared expert stays dense
        int n_off = 0;
        if (mode == kSelectTopk) {
          n_off = routed ? a.n_off_r : a.n_off_s;
          if (n_off <= 0) mode = kSelectAll;
        }
        const int n0 = static_cast<int>(static_cast<long long>(c) * n / CH);
        const int n1 = static_cast<int>(static_cast<long long>(c + 1) * n / CH);
        const bool want_pick = mode == kSelectTopk && n_off < n;
        const float* hrow = a.hc + static_cast<size_t>(row) * a.Nh;

        // wait until every gate/up piece of this expert has landed (one polite poller)
        if (dtid == 0) {
          p2[8] = 0;
          spin_until(&a.ctr[kCtrCnt + (routed ? 1 + u : 0)],
                     static_cast<unsigned>(routed ? (thr ? PEr * kStoreWarpsG : PE * kStoreWarps)
                                                  : n_sh * kStoreWarps));
        }
        hist_s[2 * dtid] = 0;
        hist_s[2 * dtid + 1] = 0;
        d_sync();
        DEC_STAMP(kWarpD0 * 32, 8);
        // the row's activations: everything in top-k mode, the chunk otherwise
        {
          const int i_lo = want_pick ? 0 : n0, i_hi = want_pick ? n : n1;
#pragma unroll 4
          for (int i = i_lo + dtid; i < i_hi; i += kDThreads) {
            const uint32_t k = __float_as_uint(__ldcg(hrow + i));
            keys_s[i] = k;
            if (want_pick) atomicAdd(&hist_s[hist_bin(k & 0x7fffffffu)], 1);
          }
        }
        d_sync();

        RowPick pk{0u, 0, true};
        if (want_pick) {
          // ---- pivot bucket from the row's histogram ----
          const uint2 hh = make_uint2(static_cast<unsigned>(hist_s[2 * dtid]),
                                      static_cast<unsigned>(hist_s[2 * dtid + 1]));
          int incl = static_cast<int>(hh.x + hh.y);
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int up = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += up;
          }
          if (lane == 31) wc[dwarp] = incl;
          for (int i = dtid; i < kMemberCap + 4; i += kDThreads) mlist[i] = 0xffffffffu;
          d_sync();
          int base = 0;
#pragma unroll
          for (int w = 0; w < 8; ++w)
            if (w < dwarp) base += wc[w];
          incl += base;
          const int excl = incl - static_cast<int>(hh.x + hh.y);
          if (excl < n_off && n_off <= incl) {
            const bool first = n_off <= excl + static_cast<int>(hh.x);
            p2[2] = 2 * dtid + (first ? 0 : 1);
            p2[3] = first ? excl : excl + static_cast<int>(hh.x);
            p2[4] = first ? static_cast<int>(hh.x) : static_cast<int>(hh.y);
          }
          d_sync();
          const int bstar = p2[2], below_bins = p2[3], M = p2[4];
          if (M <= kMemberCap) {
#pragma unroll 1
            for (int i = dtid; i < n; i += kDThreads) {
              const uint32_t k = keys_s[i] & 0x7fffffffu;
              if (hist_bin(k) == bstar) mlist[atomicAdd(&p2[8], 1)] = k;
            }
            d_sync();
            const int rr = n_off - below_bins;  // 1-based rank inside the bucket
            const int M4 = (M + 3) >> 2;
            // one member per thread (the bucket rarely holds more than a few dozen keys)
#pragma unroll 1
            for (int mi = dtid; mi < M; mi += kDThreads) {
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
            d_sync();
            pk.pivot = static_cast<uint32_t>(p2[5]);
            pk.ties_to_drop = n_off - p2[6];
            pk.drop_all_ties = (pk.ties_to_drop == p2[7]);
          } else {
            // huge bucket (many equal / clamped values): the general search; keys_s is masked in
            // place and restored afterwards
#pragma unroll 1
            for (int i = dtid; i < n; i += kDThreads) keys_s[i] &= 0x7fffffffu;
            d_sync();
            pk = kary_pick_cold(keys_s, n, n_off, sel_sc);
            d_sync();
#pragma unroll 1
            for (int i = dtid; i < n; i += kDThreads) keys_s[i] = __float_as_uint(__ldcg(hrow + i));
            d_sync();
          }
        }
        DEC_STAMP(kWarpD0 * 32, 9);

        // ---- survivors of the chunk [n0, n1), ascending index -> lst[0..m) ----
        int m = 0;
        if (mode >= 0 && !(mode == kSelectTopk && n_off >= n)) {
          // rank of a pivot tie = number of ties at lower indices (ties_to_drop of them go first)
          int tie_base = 0;
          const bool need_ties = want_pick && !pk.drop_all_ties;
          if (need_ties) {
            int cnt = 0;
#pragma unroll 1
            for (int i = dtid; i < n0; i += kDThreads) cnt += ((keys_s[i] & 0x7fffffffu) == pk.pivot) ? 1 : 0;
            cnt = __reduce_add_sync(0xffffffffu, cnt);
            if (lane == 0) wc[8 + dwarp] = cnt;
            d_sync();
#pragma unroll
            for (int w = 0; w < 8; ++w) tie_base += wc[8 + w];
            d_sync();  // wc[8..16) is rewritten by the first block below
          }
          int run = 0;  // survivors before the current 256-index block
#pragma unroll 1
          for (int i0 = n0; i0 < n1; i0 += kDThreads) {
            const int i = i0 + dtid;
            const bool valid = i < n1;
            const uint32_t k = valid ? (keys_s[i] & 0x7fffffffu) : 0u;
            const bool tie = need_ties && valid && k == pk.pivot;
            const unsigned tb = __ballot_sync(0xffffffffu, tie);
            bool f;
            if (mode == kSelectAll) {
              f = valid;
            } else if (mode == kSelectGiven) {
              f = valid && min_[i] != 0;
            } else if (mode == kSelectThreshold) {
              f = valid && __uint_as_float(k) >= a.tau;  // k = bits of |silu(g)| (activation.cpp:62-72)
            } else {
              f = valid && k > pk.pivot;
            }
            if (need_ties) {
              if (lane == 0) wc[8 + dwarp] = __popc(tb);
              d_sync();
              int tb_before = tie_base;
#pragma unroll
              for (int w = 0; w < 8; ++w) {
                const int cw = wc[8 + w];
                if (w < dwarp) tb_before += cw;
                tie_base += cw;
              }
              if (tie) f = tb_before + __popc(tb & ((1u << lane) - 1u)) >= pk.ties_to_drop;
            }
            const unsigned fb = __ballot_sync(0xffffffffu, f);
            if (lane == 0) wc[dwarp] = __popc(fb);
            d_sync();
            int before = run;
#pragma unroll
            for (int w = 0; w < 8; ++w) {
              const int cw = wc[w];
              if (w < dwarp) before += cw;
              run += cw;
            }
            if (f) lst[before + __popc(fb & ((1u << lane) - 1u))] = static_cast<uint16_t>(i);
            d_sync();  // wc is rewritten by the next block
          }
          m = run;
        }
        d_sync();
        DEC_STAMP(kWarpD0 * 32, 12);

        // ---- gather + partial: the unit's rows staged in shared memory by 16-byte cp.async
        // copies (every row of a batch in flight at once, no registers held), then rolled FMA
        // loops: thread l owns the column octets l, l + 256, ... ----
        const __nv_bfloat16* wb = routed ? a.wd + static_cast<size_t>(e) * a.Np * Dp : a.wd_shared;
        float* pout = a.part + (static_cast<size_t>(t * (CM + 1) + q) * CH + c) * Dp;
        {
          float acc[4][8];
#pragma unroll
          for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[nt][i] = 0.0f;
          const uint4* gb = reinterpret_cast<const uint4*>(sm + L.gbuf);
          const uint32_t gb_u32 = sm_u32 + L.gbuf;
          // threshold mode: the buffer holds the W_down rows AND the W_up rows of a batch (a
          // row-major copy of W_up: out of the tiled gate/up image a row is 128-byte segments at
          // a 16 KB stride, measured 3.7 us per batch against 2.5 for contiguous rows)
          const bool thr_unit = mode == kSelectThreshold;
          const int kinds = thr_unit ? 2 : 1;
          // one batch when the unit's rows fit; otherwise two half-buffers, the copies of batch
          // k + 1 in flight while batch k is consumed (cp.async groups complete in order)
          // (threshold mode, once this CTA's gate stream is over -- every consumer warp through
          // with the ring: the W_up rows of the unit go into the idle ring, the W_down rows into
          // the gather buffer, and the whole unit is ONE batch, one round trip instead of ~four)
          bool split = false;
          if (thr_unit && m * kinds > a.gb_rows && m <= a.gb_rows &&
              static_cast<size_t>(m) * LPR * 16 <= static_cast<size_t>(stages) * kStageBytes) {
            if (dtid == 0) wc[16] = *reinterpret_cast<volatile int*>(&misc[4]) == kNumGWarps ? 1 : 0;
            d_sync();
            split = wc[16] != 0;
            d_sync();
          }
          const bool piped = !split && m * kinds > a.gb_rows;
          const int RBS = split ? m : max(1, a.gb_rows / (kinds * (piped ? 2 : 1)));
          const uint32_t up_u32 = split ? sm_u32 + L.ring : 0u;   // W_up rows of the batch
          const uint4* up_ptr = reinterpret_cast<const uint4*>(sm + L.ring);
          float* hval = reinterpret_cast<float*>(mlist);  // [RBS] silu(g) * u of the batch's rows
          if (thr_unit && dtid == 0) atomicAdd(&a.ctr[kCtrKept + row], static_cast<unsigned>(m));
          const int dr = kDThreads / LPR, dc = kDThreads % LPR;
          // rows [k0, k0 + nr) of the survivor list into half `hb`: W_down rows first, then (threshold
          // mode) the same rows of W_up
          auto issue_batch = [&](int k0, int hb) {
            const int nr = min(RBS, m - k0);
            const uint32_t base = gb_u32 + static_cast<uint32_t>(hb * RBS * kinds * LPR) * 16u;
#pragma unroll 1
            for (int kind = 0; kind < kinds; ++kind) {
              const __nv_bfloat16* wsrc =
                  kind == 0 ? wb : a.wu + static_cast<size_t>(e) * a.Np * Dp;
              int r = dtid / LPR, cc = dtid % LPR;
#pragma unroll 1
              while (r < nr) {
                const __nv_bfloat16* src = wsrc + static_cast<size_t>(lst[k0 + r]) * Dp + cc * 8;
                const uint32_t dst =
                    (split && kind == 1) ? up_u32 + static_cast<uint32_t>(r * LPR + cc) * 16u
                                         : base + static_cast<uint32_t>((kind * RBS + r) * LPR + cc) * 16u;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
                cc += dc;
                r += dr;
                if (cc >= LPR) {
                  cc -= LPR;
                  ++r;
                }
              }
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
          };
          if (m > 0) issue_batch(0, 0);
          int hb = 0;
#pragma unroll 1
          for (int k0 = 0; k0 < m; k0 += RBS, hb ^= 1) {
            const int nr = min(RBS, m - k0);
            if (k0 + RBS < m) {
              issue_batch(k0 + RBS, hb ^ 1);
              asm volatile("cp.async.wait_group 1;" ::: "memory");
            } else {
              asm volatile("cp.async.wait_group 0;" ::: "memory");
            }
            d_sync();
            const uint4* gbh = gb + static_cast<size_t>(hb) * RBS * kinds * LPR;
            if (thr_unit) {
              // u = W_up[n] . x_t for the batch's rows, one warp per row; h = silu(g) * u
              const __nv_bfloat16* xt = reinterpret_cast<const __nv_bfloat16*>(sm + L.xs) +
                                        static_cast<size_t>(t) * Dp;
#pragma unroll 1
              for (int r = dwarp; r < nr; r += 8) {
                float sacc = 0.0f;
#pragma unroll 2
                for (int cc = lane; cc < LPR; cc += 32) {
                  float wf[8], xf[8];
                  unpack8(split ? up_ptr[r * LPR + cc] : gbh[(RBS + r) * LPR + cc], wf);
                  unpack8(*reinterpret_cast<const uint4*>(xt + cc * 8), xf);
#pragma unroll
                  for (int i = 0; i < 8; ++i) sacc = fmaf(wf[i], xf[i], sacc);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
                if (lane == 0) hval[r] = __uint_as_float(keys_s[lst[k0 + r]]) * sacc;
              }
              d_sync();
            }
            if (!thr_unit) {
              // the rows' activations side by side (two dependent shared-memory loads per row
              // otherwise sit in front of every FMA group of the loops below)
              for (int r = dtid; r < nr; r += kDThreads) hval[r] = __uint_as_float(keys_s[lst[k0 + r]]);
              d_sync();
            }
            if (NT == 1) {
              // narrow rows: G row groups, group g takes rows g, g + G, ...
              if (lane_ok) {
#pragma unroll 4
                for (int r = g; r < nr; r += G) fma8(gbh[r * LPR + l], hval[r], acc[0]);
              }
            } else {
#pragma unroll 2
              for (int r = 0; r < nr; ++r) {
                const float hk = hval[r];
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) {
                  const int c8 = nt * kDThreads + dtid;
                  if (c8 < LPR) fma8(gbh[r * LPR + c8], hk, acc[nt]);
                }
              }
            }
            d_sync();  // the batch after next overwrites this half (and hval)
          }
          if (NT == 1) {
            if (G > 1) {
              if (lane_ok) {
                float4* d4 = reinterpret_cast<float4*>(gred + static_cast<size_t>(g) * Dp + l * 8);
                d4[0] = make_float4(acc[0][0], acc[0][1], acc[0][2], acc[0][3]);
                d4[1] = make_float4(acc[0][4], acc[0][5], acc[0][6], acc[0][7]);
              }
              d_sync();
              for (int d = dtid; d < Dp; d += kDThreads) {
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
              const int c8 = nt * kDThreads + dtid;
              if (c8 < LPR) {
                float4* d4 = reinterpret_cast<float4*>(pout + c8 * 8);
                d4[0] = make_float4(acc[nt][0], acc[nt][1], acc[nt][2], acc[nt][3]);
                d4[1] = make_float4(acc[nt][4], acc[nt][5], acc[nt][6], acc[nt][7]);
              }
            }
          }
        }
        DEC_STAMP(kWarpD0 * 32, 13);
        d_sync();  // the unit's scratch is reused by the next one
      }
    }
    __threadfence();
    d_sync();
    if (dtid == 0) atomicAdd(&a.ctr[kCtrDone], 1u);
    DEC_STAMP(kWarpD0 * 32, 5);
  }

  // every role of this CTA is through: the ring becomes P3 scratch
  __syncthreads();
  if (warp < kWarpD0) return;

  // =====================================================================================
  // P3 (D role): grid barrier (partials + exact routing), then the ordered combine.  Each CTA owns
  // a contiguous range of (token, 4 columns) outputs: all partials of a batch of 8 outputs are
  // fetched at once into shared memory, summed per slot over the chunks (ascending), then over
  // the slots (ascending, shared expert last with weight 1: router.cpp:109-132,
  // engine.cpp:168-173).
  // =====================================================================================
  {
    const int dtid = tid - kWarpD0 * 32;
    uint8_t* work = sm + L.ring;
    int* srow = reinterpret_cast<int*>(work);            // [B][R] candidate rank of every slot
    float* swt = reinterpret_cast<float*>(work + 2048);  // [B][R] combine weights
    const int R = K + (a.has_shared ? 1 : 0);
    if (dtid == 0) spin_until(&a.ctr[kCtrRoute], static_cast<unsigned>(n_tb));
    d_sync();
    // slot tables (the exact routing is known now); overlaps the wait for the other CTAs
    for (int i = dtid; i < B * R; i += kDThreads) {
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
    DEC_STAMP(kWarpD0 * 32, 19);
    if (dtid == 0) {
      spin_until(&a.ctr[kCtrDone], static_cast<unsigned>(grid));
      if (thr) {
        // survivors per flat slot for the report's tile accounting (engine.cpp:341-348), read
        // before the counters go back to rest
        for (int sl = bid; sl < B * K; sl += grid) {
          const int tt = sl / K;
          const int ee = __ldcg(a.ids + sl);
          a.kcnt[sl] = static_cast<int32_t>(ld_acquire_u32(&a.ctr[kCtrKept + rowtab[uidx[ee] * 16 + tt]]));
          a.inv[sl] = sl;
        }
      }
      // every CTA that gets here has read all the counters for the last time: the last one
      // through puts them back to rest and opens the next epoch
      if (atomicAdd(&a.ctr[kCtrExit], 1u) == static_cast<unsigned>(grid - 1)) {
        const int n_u = misc[2];
        a.ctr[kCtrDone] = 0u;
        a.ctr[kCtrExit] = 0u;
        a.ctr[kCtrRoute] = 0u;
        for (int i = 0; i < 4; ++i) a.ctr[kCtrChain + i] = 0u;
        for (int i = 0; i <= n_u; ++i) a.ctr[kCtrCnt + i] = 0u;
        if (thr)
          for (int i = 0; i < 16 * 20; ++i) a.ctr[kCtrKept + i] = 0u;
        a.ctr[kCtrEpoch] = epoch;
      }
    }
    d_sync();
    DEC_STAMP(kWarpD0 * 32, 6);
    // Every thread takes one (output, slot, group of 8 chunks): one division chain per thread,
    // its 8 partials in flight at once, summed in chunk order; then the groups of a slot in
    // order, then the slots.  (Rolled and short: this code runs once per launch, out of a cold
    // instruction cache.)
    const int CG = (CH + 7) >> 3;
    const int D4 = Dp / 4;
    const int total4 = B * D4;
    constexpr int QB = 8;
    float4* sg = reinterpret_cast<float4*>(work + 4096);  // [QB][R][CG]
    float4* sj = sg + QB * R * CG;                         // [QB][R]
    const bool y_vec = (D % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.y) & 15) == 0);
    const int q0 = static_cast<int>(static_cast<long long>(bid) * total4 / grid);
    const int q1 = static_cast<int>(static_cast<long long>(bid + 1) * total4 / grid);
#pragma unroll 1
    for (int qb = q0; qb < q1; qb += QB) {
      const int nq = min(QB, q1 - qb);
#pragma unroll 1
      for (int idx = dtid; idx < nq * R * CG; idx += kDThreads) {
        const int cg = idx % CG, j = (idx / CG) % R, qi = idx / (CG * R);
        const int qq = qb + qi;
        const int t = qq / D4, d4 = qq - t * D4;
        const int r = srow[t * R + j];
        const float4* pp = reinterpret_cast<const float4*>(
            a.part + (static_cast<size_t>(t * (CM + 1) + r) * CH + cg * 8) * Dp + d4 * 4);
        const int nc = min(8, CH - cg * 8);
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          v[u] = u < nc ? __ldcg(pp + static_cast<size_t>(u) * D4) : make_float4(0.f, 0.f, 0.f, 0.f);
        float4 sacc = v[0];
#pragma unroll
        for (int u = 1; u < 8; ++u) {
          sacc.x = __fadd_rn(sacc.x, v[u].x);
          sacc.y = __fadd_rn(sacc.y, v[u].y);
          sacc.z = __fadd_rn(sacc.z, v[u].z);
          sacc.w = __fadd_rn(sacc.w, v[u].w);
        }
        sg[idx] = sacc;
      }
      d_sync();
      DEC_STAMP(kWarpD0 * 32, 20);
      for (int idx = dtid; idx < nq * R; idx += kDThreads) {
        const float4* pb = sg + static_cast<size_t>(idx) * CG;
        float4 sacc = pb[0];
#pragma unroll 1
        for (int c = 1; c < CG; ++c) {
          const float4 pv = pb[c];
          sacc.x = __fadd_rn(sacc.x, pv.x);
          sacc.y = __fadd_rn(sacc.y, pv.y);
          sacc.z = __fadd_rn(sacc.z, pv.z);
          sacc.w = __fadd_rn(sacc.w, pv.w);
        }
        sj[idx] = sacc;
      }
      d_sync();
      if (dtid < nq) {
        const int qq = qb + dtid;
        const int t = qq / D4, d4 = qq % D4;
        float4 acc = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll 1
        for (int j = 0; j < R; ++j) {
          const float w = swt[t * R + j];
          const float4 sv = sj[dtid * R + j];
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
      d_sync();
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
        const float* src = a.hc + static_cast<size_t>(row) * a.Nh;
        float* dst = a.h_cap + static_cast<size_t>(sl) * a.Nh;
        for (int i = dtid; i < n; i += kDThreads) dst[i] = __ldcg(src + i);
        if (dtid == 0) {
          a.row_expert[sl] = ee;
          if (rt) {
            a.inv[sl] = sl;
            a.perm[sl] = sl;
          }
        }
      }
    }
    DEC_STAMP(kWarpD0 * 32, 7);
  }
}

bool decode_fused_eligible(const Geometry& g, int B) {
  const int nmax = g.N > g.S ? g.N : g.S;
  return B >= 1 && B <= kDecMaxB && g.E <= kDecMaxE && g.K <= 16 && nmax <= kMaxN &&
         g.Dp <= 8192 && (g.Dp % 64) == 0 && g.E + g.K + 8 <= 288 &&
         dec_plan(nmax, dec_tb_for(B), g.Dp).stages >= kMinStages &&
         dec_plan(nmax, dec_tb_for(B), g.Dp).gb_rows >= 2;
}

int decode_counter_words() { return kCtrWords; }
int decode_cand_rows(int K) { return K + 4; }
int decode_p0_words(const Geometry& g) { return 16 * g.E * kMaxND * 2 * 2; }
int decode_chunks(const Geometry& g, int B, int keep_max, int n_sms) {
  // Batch-invariant by design (B is ignored): one token's units fill the grid once.
  (void)B;
  const int R = g.K + (g.has_shared ? 1 : 0);
  int ch = 2 * n_sms / (R + 1);  // two waves of units: 16 rows per unit = one batch of loads
  int cap = keep_max / 8;  // at least ~8 rows per unit
  if (cap < 1) cap = 1;
  if (ch > cap) ch = cap;
  if (ch > 32) ch = 32;
  if (ch < 1) ch = 1;
  return ch;
}


template <int TB>
static void launch_tb(const cudaLaunchConfig_t& cfg, const CUtensorMap* tmap_w3,
                      const CUtensorMap* tmap_w3g, const DecodeArgs& a) {
  // the opt-in is per device: set it on the first launch on each device
  static std::mutex mu;
  static bool attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    if (dev < 0 || dev >= 64 || !attr_set[dev]) {
      cudaFuncSetAttribute(decode_fused_kernel<TB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kSmemBudget + 1024);
      if (dev >= 0 && dev < 64) attr_set[dev] = true;
    }
  }
  cudaLaunchKernelEx(&cfg, decode_fused_kernel<TB>, *tmap_w3, *tmap_w3g, a);
}

int launch_decode_fused(const LaunchCtx& ctx, const CUtensorMap* tmap_w3, const CUtensorMap* tmap_w3g,
                        const DecodeLaunch& d, const Geometry& g, int n_sms) {
  const int nmax = g.N > g.S ? g.N : g.S;
  const int tb = dec_tb_for(d.B);
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
  a.tau = d.tau;
  a.wu = d.wu;
  a.kcnt = d.kcnt;
  a.n_off_r = d.n_off_r;
  a.n_off_s = d.n_off_s;
  a.mask_r = d.mask_r;
  a.mask_s = d.mask_s;
  a.CM = decode_cand_rows(g.K);
  a.CH = d.CH;
  a.capture = d.capture ? 1 : 0;
  const DecPlan plan = dec_plan(nmax, tb, g.Dp);
  a.stages = plan.stages;
  a.gb_rows = plan.gb_rows;
  {
    const int n_cu = ceil_div(g.E, 8) * ceil_div(d.B, 4);
    a.n_ch = n_cu < kMaxChainCtas ? n_cu : kMaxChainCtas;
  }
  {
    // fast-logit units: (expert, d_model slice); as many slices as fill the grid once
    int nd = n_sms / g.E;
    if (nd < 1) nd = 1;
    if (nd > kMaxND) nd = kMaxND;
    const int ds = round_up(ceil_div(g.D, nd), 4);
    a.ND = ceil_div(g.D, ds);
    a.DS = ds;
  }
  a.p0 = reinterpret_cast<uint2*>(d.p0);
  a.logits = d.logits;
  a.ids = d.ids;
  a.wts = d.wts;
  a.hc = d.hc;
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
  cfg.dynamicSmemBytes = dec_smem_layout(a.stages, a.gb_rows, nmax, tb, g.Dp).total + 1024;
  switch (tb) {
    case 1: launch_tb<1>(cfg, tmap_w3, tmap_w3g, a); break;
    case 2: launch_tb<2>(cfg, tmap_w3, tmap_w3g, a); break;
    default: launch_tb<4>(cfg, tmap_w3, tmap_w3g, a); break;
  }
  return 1;
}

}  // namespace skb
