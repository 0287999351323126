// down.cu -- subsystems (3)+(4)+(5): neuron selection, the down projection as a gather over
// the surviving W_down rows, and the router-weighted combine (shared expert included), in ONE
// launch with no global intermediates, no atomics and no fences.  Only rows named by the
// selection are ever addressed, so dropped neurons cost no HBM bytes.
//
// Replaces topk_mask + mask application (proj/src/activation.cpp:31-60, engine.cpp:150-157),
// gathered_matvec_t (proj/src/linalg.cpp:56-81), combine (proj/src/router.cpp:109-132) and the
// shared-expert accumulation (proj/src/engine.cpp:55-84).
//
// One thread-block CLUSTER of 8 CTAs per (token, segment of SEG output columns):
//   phase 1  selection.  The token's R = K (+1 shared) rows are dealt round-robin to the 8
//            CTAs; a CTA ranks |h| of its row (select_device.cuh), walks the survivors in
//            ascending index order and PUSHES entry p of the survivor list into the shared
//            memory of CTA p / C (C = ceil(cnt / 8)) through distributed shared memory.
//            After one cluster barrier every CTA holds its 1/8 slice of every row's list.
//   phase 2  gather.  CTA q streams survivors [qC, qC + C) of every row: warp 0 issues one
//            1-D bulk copy (TMA engine, mbarrier completion) per surviving W_down row piece
//            (SEG * 2 contiguous bytes) into a shared-memory ring -- at decode sizes the whole
//            slice is in flight at once, so HBM sees 128 x ~128 KB of outstanding reads -- and
//            all 8 warps accumulate from the ring in fp32.
//   phase 3  combine.  Fixed tree, identical for every batch size and grid shape:
//              piece order inside a warp: ascending survivor index (fmaf)
//              per row:  acc_total += router_weight * acc_row   (rows ascending = slots
//                        ascending, shared expert last with weight 1, engine.cpp:168-173)
//              8 warps ascending (shared memory), 8 CTAs ascending (distributed shared
//              memory), then y[t] is written once.
#include <cooperative_groups.h>

#include "select_device.cuh"

namespace cg = cooperative_groups;

namespace skb {

namespace {

constexpr int kClusterCtas = 8;
constexpr int kStagePieces = 64;  // survivors per ring stage: 8 per warp
constexpr int kMaxRing = 16;

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// cp.async.wait_group takes an immediate: at most `n` (0..15) groups stay in flight
__device__ __forceinline__ void cp_async_wait_dyn(int n) {
  switch (n) {
#define SKB_W(k) case k: asm volatile("cp.async.wait_group %0;" ::"n"(k) : "memory"); break;
    SKB_W(0) SKB_W(1) SKB_W(2) SKB_W(3) SKB_W(4) SKB_W(5) SKB_W(6) SKB_W(7)
    SKB_W(8) SKB_W(9) SKB_W(10) SKB_W(11) SKB_W(12) SKB_W(13) SKB_W(14)
#undef SKB_W
    default: asm volatile("cp.async.wait_group 15;" ::: "memory"); break;
  }
}

__device__ __forceinline__ void fma_bf16x2(uint32_t u, float hk, float& a0, float& a1) {
  // bf16 -> fp32 is a 16-bit shift
  a0 = fmaf(__uint_as_float(u << 16), hk, a0);
  a1 = fmaf(__uint_as_float(u & 0xffff0000u), hk, a1);
}

struct DownSmemLayout {
  int keys_off, lidx_off, lval_off, meta_off, ring_off, red_off, sum_off, bar_off, total;
};

__host__ __device__ inline DownSmemLayout down_layout(int seg, int R, int cmax, int nmax, int ring) {
  DownSmemLayout l;
  int o = 0;
  l.ring_off = o;  // first: bulk-copy destinations want 128-byte alignment
  o += ring * kStagePieces * seg * 2;
  l.keys_off = o;
  o += round_up(nmax, 4) * 4;
  l.lidx_off = o;
  o += R * cmax * 4;
  l.lval_off = o;
  o += R * cmax * 4;
  l.meta_off = o;
  o += round_up(R, 2) * 32;  // per row: cnt, m, nb, stage0 (ints) + wgt (float) + pad, wbase (8 B)
  l.red_off = o;
  o += kSelWarps * seg * 4;
  l.sum_off = o;
  o += seg * 4;
  l.bar_off = o;
  o += kMaxRing * 8;
  l.total = o;
  return l;
}

struct RowMeta {
  int cnt;      // survivors of the row
  int m;        // survivors in this CTA's slice
  int stage0;   // first ring stage of the row in this CTA
  float wgt;    // router weight (1 for the shared expert)
  const __nv_bfloat16* wbase;  // W_down image of the row's expert
  int C;        // slice length
  int pad;
};
static_assert(sizeof(RowMeta) == 32, "RowMeta is 32 bytes");

}  // namespace

#ifdef SKB_DEBUG_TIMING  // phase timestamps for tools/dbg_rf.py
__device__ long long g_dn_dbg[16];
#define DN_T(i) do { if (tid == 0 && blockIdx.x == 1 && blockIdx.y == 0 && blockIdx.z == 0) g_dn_dbg[i] = clock64(); } while (0)
#else
#define DN_T(i) do { } while (0)
#endif

template <int SEG>
__global__ void __launch_bounds__(256, 1)
down_cluster_kernel(DownArgs a, int E, int Np, int D, int Dp, int R, int cmax, int nmax, int ring) {
  extern __shared__ __align__(128) uint8_t dsm[];
  __shared__ SelScratch sc;
  constexpr int CPL = SEG / 32;  // columns per lane
  const DownSmemLayout L = down_layout(SEG, R, cmax, nmax, ring);
  uint8_t* ring_s = dsm + L.ring_off;
  uint32_t* keys = reinterpret_cast<uint32_t*>(dsm + L.keys_off);
  int32_t* lidx = reinterpret_cast<int32_t*>(dsm + L.lidx_off);
  float* lval = reinterpret_cast<float*>(dsm + L.lval_off);
  RowMeta* meta = reinterpret_cast<RowMeta*>(dsm + L.meta_off);
  float* red = reinterpret_cast<float*>(dsm + L.red_off);
  float* cta_sum = reinterpret_cast<float*>(dsm + L.sum_off);

  cg::cluster_group cluster = cg::this_cluster();
  const int q = static_cast<int>(cluster.block_rank());
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int seg = blockIdx.y, t = blockIdx.z;
  const int col0 = seg * SEG;
  const int piece_cols = min(SEG, Dp - col0);

  DN_T(0);
  pdl_wait();
  pdl_launch_dependents();
  DN_T(1);

  // row j of the token: slots ascending, then the shared expert
  auto row_of = [&](int j) { return j < a.K ? a.inv[t * a.K + j] : a.BK + t; };

  // per-row constants (issued early: these global loads overlap the selection)
  if (tid < R) {
    const int j = tid;
    const int row = row_of(j);
    const int e = a.row_expert[row];
    meta[j].wgt = j < a.K ? a.weights[t * a.K + j] : 1.0f;
    meta[j].wbase = (e < E) ? a.wd + static_cast<size_t>(e) * Np * Dp : a.wd_shared;
  }
  cluster.sync();  // every CTA of the cluster is running: its shared memory may be written
  DN_T(2);

  // ---- phase 1: selection of the rows dealt to this CTA; lists pushed to their consumers ----
  for (int j = q; j < R; j += kClusterCtas) {
    const bool routed = j < a.K;
    const int row = row_of(j);
    const int n = routed ? a.N : a.S;
    const int slot = routed ? t * a.K + j : t;
    const float* hrow = a.h + static_cast<size_t>(row) * a.Nh;
    int mode = a.sel_mode;
    const uint8_t* min_ = nullptr;
    if (mode == kSelectGiven) {
      min_ = routed ? a.mask_in_routed + static_cast<size_t>(slot) * n
                    : (a.mask_in_shared ? a.mask_in_shared + static_cast<size_t>(slot) * n
                                        : nullptr);
      if (min_ == nullptr) mode = kSelectAll;
    }
    int n_off = 0;
    if (mode == kSelectTopk) {
      n_off = routed ? a.n_off_routed : a.n_off_shared;
      if (n_off <= 0) mode = kSelectAll;  // activation.cpp:35
    }
    int cnt;
    RowPick pk{0u, 0, true};
    if (mode == kSelectAll) {
      cnt = n;
    } else if (mode == kSelectTopk) {
      cnt = n_off >= n ? 0 : n - n_off;  // activation.cpp:36-39
      if (cnt > 0) {
        __syncthreads();  // keys of the previous row are no longer read
        for (int i = tid; i < n; i += kSelectThreads)
          keys[i] = __float_as_uint(hrow[i]) & 0x7fffffffu;
        __syncthreads();
        DN_T(3);
        pk = sel_kary_pick(keys, n, n_off, sc);
        DN_T(4);
      }
    } else {
      // caller masks: count first (the slice length depends on it)
      int c = 0;
      for (int i = tid; i < n; i += kSelectThreads) c += (min_[i] != 0) ? 1 : 0;
      int total;
      (void)sel_block_rank(false, sc, 0, total);  // orders the reuse of sc.warp_cnt
      c = __reduce_add_sync(0xffffffffu, c);
      __syncthreads();
      if (lane == 0) sc.kcnt[0][warp] = c;
      __syncthreads();
      cnt = 0;
#pragma unroll
      for (int w = 0; w < kSelWarps; ++w) cnt += sc.kcnt[0][w];
      __syncthreads();
    }
    const int C = ceil_div(cnt, kClusterCtas);
    if (tid < kClusterCtas) {
      RowMeta* rm = cluster.map_shared_rank(meta, tid);
      rm[j].cnt = cnt;
      rm[j].C = C;
    }
    if (cnt > 0) {
      // ordered walk over the row, rounds of 256 consecutive indices
      int kept_base = 0, tie_base = 0, buf = 0;
      const int rounds = ceil_div(n, kSelectThreads);
#pragma unroll 1
      for (int r = 0; r < rounds; ++r) {
        const int i = r * kSelectThreads + tid;
        const bool valid = i < n;
        bool keep;
        if (mode == kSelectAll) {
          keep = valid;
        } else if (mode == kSelectGiven) {
          keep = valid && (min_[i] != 0);
        } else {
          const uint32_t k = valid ? keys[i] : 0u;
          if (pk.drop_all_ties) {
            keep = valid && k > pk.pivot;
          } else {
            const bool tie = valid && k == pk.pivot;
            int tie_total;
            const int tie_rank = tie_base + sel_block_rank(tie, sc, buf, tie_total);
            buf ^= 1;
            tie_base += tie_total;
            keep = valid && (k > pk.pivot || (tie && tie_rank >= pk.ties_to_drop));
          }
        }
        int kept_total;
        const int pos = kept_base + sel_block_rank(keep, sc, buf, kept_total);
        buf ^= 1;
        kept_base += kept_total;
        if (keep) {
          const int c = pos / C;
          const int off = pos - c * C;
          int32_t* ri = cluster.map_shared_rank(lidx, c);
          float* rv = cluster.map_shared_rank(lval, c);
          ri[j * cmax + off] = i;
          rv[j * cmax + off] = hrow[i];
        }
      }
    }
  }
  DN_T(5);
  cluster.sync();  // lists and counts have landed everywhere
  DN_T(6);

  // ---- phase 2: gather ----
  if (tid == 0) {
    int st = 0;
    for (int j = 0; j < R; ++j) {
      const int C = meta[j].C;
      int m = meta[j].cnt - q * C;
      m = m < 0 ? 0 : (m > C ? C : m);
      meta[j].m = m;
      meta[j].stage0 = st;
      st += ceil_div(m, kStagePieces);
    }
    sc.kcnt[1][0] = st;
  }
  __syncthreads();
  const int n_stages = sc.kcnt[1][0];

  // Stage g = up to 64 surviving row pieces.  Every thread copies its 16-byte chunks with
  // cp.async (consecutive lanes = consecutive chunks of one piece: coalesced) and commits one
  // group per stage.  (Per-piece 1-D bulk copies were measured at ~64 cycles of serialised
  // issue each -- 17 us for 512 pieces of 256 B -- so the TMA engine is the wrong tool for
  // sub-KB gathers.)
  constexpr int kChunksPerPiece = SEG / 8;                        // 16-byte chunks
  constexpr int kChunksPerThread = kStagePieces * kChunksPerPiece / 256;
  auto issue = [&](int g) {
    int j = 0;
    while (j + 1 < R && meta[j + 1].stage0 <= g) ++j;
    while (meta[j].m == 0 || g - meta[j].stage0 >= ceil_div(meta[j].m, kStagePieces)) ++j;
    const int b = g - meta[j].stage0;
    const int np = min(kStagePieces, meta[j].m - b * kStagePieces);
    const __nv_bfloat16* wb = meta[j].wbase + col0;
    uint8_t* dst0 = ring_s + static_cast<size_t>(g % ring) * kStagePieces * SEG * 2;
    const int32_t* li = lidx + j * cmax + b * kStagePieces;
#pragma unroll
    for (int i = 0; i < kChunksPerThread; ++i) {
      const int c = tid + 256 * i;
      const int p = c / kChunksPerPiece, sub = c % kChunksPerPiece;
      if (p < np && sub * 8 < piece_cols)
        cp_async16(dst0 + static_cast<size_t>(p) * SEG * 2 + sub * 16,
                   wb + static_cast<size_t>(li[p]) * Dp + sub * 8);
    }
    cp_async_commit();
  };

  {
    const int pre = n_stages < ring ? n_stages : ring;
    for (int g = 0; g < pre; ++g) issue(g);
  }

  DN_T(7);
  float acc_total[CPL], acc_row[CPL];
#pragma unroll
  for (int i = 0; i < CPL; ++i) acc_total[i] = acc_row[i] = 0.0f;

  {
    int g = 0;
    for (int j = 0; j < R; ++j) {
      const int m = meta[j].m;
      const int nb = ceil_div(m, kStagePieces);
      for (int b = 0; b < nb; ++b, ++g) {
        {
          const int rest = n_stages - 1 - g;
          cp_async_wait_dyn(rest < ring - 1 ? rest : ring - 1);
        }
        __syncthreads();
        const uint8_t* st = ring_s + static_cast<size_t>(g % ring) * kStagePieces * SEG * 2;
        const int np = min(kStagePieces, m - b * kStagePieces);
#pragma unroll
        for (int p8 = 0; p8 < kStagePieces / kSelWarps; ++p8) {
          const int p = warp * (kStagePieces / kSelWarps) + p8;
          if (p < np) {
            const float hk = lval[j * cmax + b * kStagePieces + p];
            const uint8_t* piece = st + static_cast<size_t>(p) * SEG * 2;
            if constexpr (CPL == 4) {
              const uint2 u = *reinterpret_cast<const uint2*>(piece + lane * 8);
              if (lane * 4 < piece_cols) {
                fma_bf16x2(u.x, hk, acc_row[0], acc_row[1]);
                fma_bf16x2(u.y, hk, acc_row[2], acc_row[3]);
              }
            } else {
#pragma unroll
              for (int half = 0; half < CPL / 8; ++half) {
                const int c = half * 256 + lane * 8;  // interleaved halves: conflict-free LDS.128
                if (c < piece_cols) {
                  const uint4 u = *reinterpret_cast<const uint4*>(piece + c * 2);
                  fma_bf16x2(u.x, hk, acc_row[8 * half + 0], acc_row[8 * half + 1]);
                  fma_bf16x2(u.y, hk, acc_row[8 * half + 2], acc_row[8 * half + 3]);
                  fma_bf16x2(u.z, hk, acc_row[8 * half + 4], acc_row[8 * half + 5]);
                  fma_bf16x2(u.w, hk, acc_row[8 * half + 6], acc_row[8 * half + 7]);
                }
              }
            }
          }
        }
        if (g + ring < n_stages) {  // ring smaller than the slice: refill the slot just drained
          __syncthreads();
          issue(g + ring);
        }
      }
      const float wgt = meta[j].wgt;
#pragma unroll
      for (int i = 0; i < CPL; ++i) {
        acc_total[i] = __fadd_rn(acc_total[i], __fmul_rn(wgt, acc_row[i]));
        acc_row[i] = 0.0f;
      }
    }
  }

  DN_T(8);
  // ---- phase 3: warps ascending, CTAs ascending ----
#pragma unroll
  for (int i = 0; i < CPL; ++i) {
    const int c = (CPL == 4) ? lane * 4 + i : (i / 8) * 256 + lane * 8 + (i % 8);
    red[warp * SEG + c] = acc_total[i];
  }
  __syncthreads();
  for (int c = tid; c < SEG; c += 256) {
    float s = red[c];
#pragma unroll
    for (int w = 1; w < kSelWarps; ++w) s = __fadd_rn(s, red[w * SEG + c]);
    cta_sum[c] = s;
  }
  cluster.sync();
  constexpr int kFinal = SEG / kClusterCtas;  // columns finalised by each CTA
  if (tid < kFinal) {
    const int c = q * kFinal + tid;
    const int col = col0 + c;
    if (col < D) {
      float s = *(cluster.map_shared_rank(cta_sum, 0) + c);
#pragma unroll
      for (int r = 1; r < kClusterCtas; ++r) s = __fadd_rn(s, *(cluster.map_shared_rank(cta_sum, r) + c));
      a.y[static_cast<size_t>(t) * D + col] = s;
    }
  }
  cluster.sync();  // nobody leaves while its shared memory is still being read
  DN_T(9);
}

#ifdef SKB_DEBUG_TIMING
extern "C" void skb_debug_dn(long long* out) { cudaMemcpyFromSymbol(out, g_dn_dbg, sizeof(g_dn_dbg)); }
#endif

template <int SEG>
static int launch_down_seg(const LaunchCtx& ctx, const DownArgs& a, const Geometry& g, int R,
                           int cmax, int nmax) {
  const int max_stages = R * ceil_div(cmax, kStagePieces);
  const int stage_bytes = kStagePieces * SEG * 2;
  // <= ~64 KB of ring keeps two CTAs per SM, which the 8-CTA clusters need to be co-scheduled
  // in one wave (16 clusters x 8 CTAs at one CTA per SM were measured to take two waves)
  int ring = (64 * 1024) / stage_bytes;
  if (ring > kMaxRing) ring = kMaxRing;
  if (ring > max_stages) ring = max_stages;
  if (ring < 1) ring = 1;
  DownSmemLayout L = down_layout(SEG, R, cmax, nmax, ring);
  while (L.total > 220 * 1024 && ring > 1) {
    --ring;
    L = down_layout(SEG, R, cmax, nmax, ring);
  }
  if (L.total > 220 * 1024) return -1;
  static int smem_set[64] = {};  // per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (L.total > __atomic_load_n(&smem_set[dev & 63], __ATOMIC_ACQUIRE)) {
    cudaFuncSetAttribute(down_cluster_kernel<SEG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         L.total);
    __atomic_store_n(&smem_set[dev & 63], L.total, __ATOMIC_RELEASE);
  }
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kClusterCtas;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = ctx.pdl ? 2 : 1;
  cfg.stream = ctx.stream;
  cfg.gridDim = dim3(kClusterCtas, ceil_div(g.Dp, SEG), a.B);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = L.total;
  cudaLaunchKernelEx(&cfg, down_cluster_kernel<SEG>, a, g.E, g.Np, g.D, g.Dp, R, cmax, nmax, ring);
  return 1;
}

int launch_down(const LaunchCtx& ctx, const DownArgs& a, const Geometry& g) {
  if (a.B <= 0) return 0;
  const int R = a.K + (a.has_shared ? 1 : 0);
  const int nmax = g.N > g.S ? g.N : g.S;
  const int keep = a.max_keep > 0 ? a.max_keep : 1;
  const int cmax = round_up(ceil_div(keep, kClusterCtas), 4);
  // widest segment that still gives the grid >= 256 CTAs (decode batches need the CTA count,
  // large batches prefer long contiguous row pieces)
  int rc;
  if (static_cast<long>(kClusterCtas) * ceil_div(g.Dp, 512) * a.B >= 256)
    rc = launch_down_seg<512>(ctx, a, g, R, cmax, nmax);
  else if (static_cast<long>(kClusterCtas) * ceil_div(g.Dp, 256) * a.B >= 256)
    rc = launch_down_seg<256>(ctx, a, g, R, cmax, nmax);
  else
    rc = launch_down_seg<128>(ctx, a, g, R, cmax, nmax);
  return rc;
}

}  // namespace skb
