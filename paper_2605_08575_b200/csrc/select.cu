// select.cu -- subsystem (3): per-(token, expert) neuron selection.  Ranks post-activation
// magnitudes |h| and drops the n_off smallest with a CTA-wide radix select in shared memory;
// no sort is performed.  Emits the ascending survivor list (indices + values) that the
// down-projection gathers, the survivor count, and optionally the uint8 mask.
//
// Bit-exact restatement of mask_smallest_magnitudes / topk_mask
// (proj/src/activation.cpp:31-60): key = bits(h) & 0x7fffffff is monotone in |h|; among keys
// equal to the pivot the LOWER indices are dropped first (stable_sort, activation.cpp:42-50).
#include "select_device.cuh"

namespace skb {

__global__ void __launch_bounds__(kSelectThreads) select_rows_kernel(SelectArgs a) {
  extern __shared__ __align__(16) uint32_t keys[];  // [max(N,S)]
  __shared__ SelScratch sc;
  __shared__ __align__(16) SelHistScratch hs;

  const int tid = threadIdx.x;
  const int row = blockIdx.x;
  const bool routed = row < a.BK;
  const int n = routed ? a.N : a.S;

  pdl_wait();
  pdl_launch_dependents();

  const int slot = routed ? (a.perm ? a.perm[row] : row) : row - a.BK;
  const float* hrow = a.h + static_cast<size_t>(row) * a.Nh;
  int32_t* kidx = a.kept_idx ? a.kept_idx + static_cast<size_t>(row) * a.Nh : nullptr;
  __nv_bfloat16* hb = a.hb ? a.hb + static_cast<size_t>(row) * a.Nh : nullptr;
  float* kval = a.kept_val ? a.kept_val + static_cast<size_t>(row) * a.Nh : nullptr;
  uint8_t* mout = routed ? (a.mask_out_routed ? a.mask_out_routed + static_cast<size_t>(slot) * n
                                              : nullptr)
                         : (a.mask_out_shared ? a.mask_out_shared + static_cast<size_t>(slot) * n
                                              : nullptr);
  const uint8_t* min_ = nullptr;
  int mode = a.mode;
  if (mode == kSelectGiven) {
    min_ = routed ? a.mask_in_routed + static_cast<size_t>(slot) * n
                  : (a.mask_in_shared ? a.mask_in_shared + static_cast<size_t>(slot) * n : nullptr);
    if (min_ == nullptr) mode = kSelectAll;
  }
  // threshold selection (forward_sparse): |silu(gate)| >= tau on routed rows, the shared expert
  // stays dense (engine.cpp:352)
  const float* sgrow = nullptr;
  if (mode == kSelectThreshold) {
    if (routed) sgrow = a.sg + static_cast<size_t>(row) * a.Nh;
    else mode = kSelectAll;
  }

  int n_off = 0;
  if (mode == kSelectTopk) {
    n_off = a.counts ? a.counts[row]
                     : (routed ? (a.slot_counts ? a.slot_counts[slot % a.K] : a.n_off_routed)
                               : a.n_off_shared);
    if (n_off <= 0) mode = kSelectAll;  // activation.cpp:35
  }

  uint32_t pivot = 0;       // keys < pivot are dropped, keys > pivot survive
  int ties_to_drop = 0;     // how many keys == pivot are dropped (lowest indices first)
  bool drop_all_ties = true;
  bool drop_everything = false;

  if (mode == kSelectTopk) {
    if (n_off >= n) {
      drop_everything = true;  // activation.cpp:36-39
    } else {
      if ((n & 3) == 0 && (a.Nh & 3) == 0) {
        for (int i = 4 * tid; i < n; i += 4 * kSelectThreads) {
          const uint4 q = *reinterpret_cast<const uint4*>(hrow + i);
          *reinterpret_cast<uint4*>(keys + i) =
              make_uint4(q.x & 0x7fffffffu, q.y & 0x7fffffffu, q.z & 0x7fffffffu, q.w & 0x7fffffffu);
        }
      } else {
        for (int i = tid; i < n; i += kSelectThreads)
          keys[i] = __float_as_uint(hrow[i]) & 0x7fffffffu;
      }
      __syncthreads();
      const RowPick pk = sel_hist_pick(keys, n, n_off, hs, sc);
      pivot = pk.pivot;
      ties_to_drop = pk.ties_to_drop;
      drop_all_ties = pk.drop_all_ties;
    }
  }

  // ---- fast path (prefill rows too long for the warp kernel: GPT-OSS shape, 2880 neurons x
  // 16384 rows): no ties at the pivot to order, no lists, no mask export -- four neurons per
  // thread, 128-bit reads of h and the keys, one 64-bit store per bf16 term ----
  if (mode == kSelectTopk && !drop_everything && drop_all_ties && kidx == nullptr &&
      a.kept_cnt == nullptr && mout == nullptr && hb != nullptr && (n & 3) == 0 && (a.Nh & 3) == 0) {
    const int kext4 = routed ? a.kext_routed : a.kext_shared;
    if ((kext4 & 3) == 0 && (a.hb_split_stride & 3) == 0) {
      for (int i = 4 * tid; i < kext4; i += 4 * kSelectThreads) {
        float v[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        if (i < n) {
          const float4 hv4 = *reinterpret_cast<const float4*>(hrow + i);
          const uint4 k4 = *reinterpret_cast<const uint4*>(keys + i);
          v[0] = k4.x > pivot ? hv4.x : 0.0f;
          v[1] = k4.y > pivot ? hv4.y : 0.0f;
          v[2] = k4.z > pivot ? hv4.z : 0.0f;
          v[3] = k4.w > pivot ? hv4.w : 0.0f;
        }
        for (int sp = 0; sp < a.nsplit; ++sp) {
          uint32_t w[2];
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const __nv_bfloat16 lo = __float2bfloat16_rn(v[2 * q]);
            const __nv_bfloat16 hi = __float2bfloat16_rn(v[2 * q + 1]);
            v[2 * q] = __fsub_rn(v[2 * q], __bfloat162float(lo));
            v[2 * q + 1] = __fsub_rn(v[2 * q + 1], __bfloat162float(hi));
            w[q] = static_cast<uint32_t>(__bfloat16_as_ushort(lo)) |
                   (static_cast<uint32_t>(__bfloat16_as_ushort(hi)) << 16);
          }
          *reinterpret_cast<uint2*>(hb + static_cast<size_t>(sp) * a.hb_split_stride + i) =
              make_uint2(w[0], w[1]);
        }
      }
      return;
    }
  }

  // ---- ordered compaction: rounds of 256 consecutive indices ----
  int kept_base = 0, tie_base = 0, buf = 0;
  // positions among the survivors are only needed for the survivor lists and the count: the
  // dense down projection (masked hb) and the mask export do without the block-wide ranks
  const bool need_pos = kidx != nullptr || a.kept_cnt != nullptr;
  // the dense down projection reads the masked row up to the K extent of its expert image
  const int kext = hb ? (routed ? a.kext_routed : a.kext_shared) : n;
  const int rounds = ceil_div(kext, kSelectThreads);
#pragma unroll 1
  for (int r = 0; r < rounds; ++r) {
    const int i = r * kSelectThreads + tid;
    const bool valid = i < n;
    float hv = 0.0f;
    bool keep = false;
    if (mode == kSelectAll) {
      keep = valid;
      if (valid) hv = hrow[i];
    } else if (mode == kSelectGiven) {
      keep = valid && (min_[i] != 0);
      if (valid) hv = hrow[i];
    } else if (mode == kSelectThreshold) {
      keep = valid && fabsf(sgrow[i]) >= a.tau;
      if (valid) hv = hrow[i];
    } else if (!drop_everything) {
      uint32_t k = 0;
      if (valid) {
        hv = hrow[i];
        k = keys[i];
      }
      if (drop_all_ties) {
        keep = valid && k > pivot;
      } else {
        const bool tie = valid && k == pivot;
        int tie_total;
        const int tie_rank = tie_base + sel_block_rank(tie, sc, buf, tie_total);
        buf ^= 1;
        tie_base += tie_total;
        keep = valid && (k > pivot || (tie && tie_rank >= ties_to_drop));
      }
    }
    int pos = 0;
    if (need_pos) {
      int kept_total;
      pos = kept_base + sel_block_rank(keep, sc, buf, kept_total);
      buf ^= 1;
      kept_base += kept_total;
    }
    if (keep && kidx) {
      kidx[pos] = i;
      if (kval) kval[pos] = hv;
    }
    if (mout && valid) mout[i] = keep ? 1 : 0;
    if (hb && i < kext) {
      // masked activation as bf16 terms b0 + b1 + b2 == h exactly (8 + 8 + 8 mantissa bits);
      // nsplit == 1 keeps only the leading term (bf16 mode)
      float v = keep ? hv : 0.0f;
      for (int sp = 0; sp < a.nsplit; ++sp) {
        const __nv_bfloat16 b = __float2bfloat16_rn(v);
        hb[static_cast<size_t>(sp) * a.hb_split_stride + i] = b;
        v = __fsub_rn(v, __bfloat162float(b));
      }
    }
  }
  if (tid == 0 && a.kept_cnt) a.kept_cnt[row] = kept_base;
}

// One warp per row, 8 rows per CTA, keys and values in registers (rows of up to 1024 neurons).
// Lane l owns the NPL consecutive neurons [l * NPL, (l + 1) * NPL): 128-bit loads and stores,
// index order = (lane, j) order, so tie ranks and survivor positions come from one warp scan of
// per-lane counts instead of a ballot per element.  Same outputs as select_rows_kernel, bit for
// bit; no block barriers.
// LEAN: the batch hot case, checked by the launcher -- uniform top-k over full rows (n == 32 *
// NPL == kext, 0 < n_off < n, no shared rows of another length), outputs = masked bf16 terms only.
// Every bounds check, mode branch and optional output folds away (the generic instantiation
// issues ~2200 warp instructions per row, most of them predicated off).
#ifdef SKB_DEBUG_TIMING
// per-warp phase stamps of the lean batch selection (tools/dbg_tc.py): [row][8]
__device__ long long g_sel_dbg[4096 * 8];
#define SEL_STAMP(i)                                                              \
  do {                                                                            \
    if (LEAN && lane == 0 && row < 4096) {                                        \
      if ((i) == 0) {                                                             \
        long long t_;                                                             \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                    \
        g_sel_dbg[row * 8] = t_;                                                  \
        g_sel_dbg[row * 8 + 7] = clock64();                                       \
      } else {                                                                    \
        g_sel_dbg[row * 8 + (i)] = clock64();                                     \
      }                                                                           \
    }                                                                             \
  } while (0)
extern "C" void skb_debug_sel(long long* out) { cudaMemcpyFromSymbol(out, g_sel_dbg, sizeof(g_sel_dbg)); }
#else
#define SEL_STAMP(i) do { } while (0)
#endif

template <int NPL, bool LEAN>
__global__ void __launch_bounds__(kSelectThreads) select_rows_warp_kernel(SelectArgs a) {
  __shared__ uint32_t pick_scratch[kSelWarps][36];
  __shared__ __align__(16) int pick_hist[kSelWarps][256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int row = blockIdx.x * kSelWarps + warp;
  SEL_STAMP(0);
  pdl_wait();
  pdl_launch_dependents();
  if (row >= a.rows) return;
  SEL_STAMP(1);
  const bool routed = LEAN || row < a.BK;
  const int n = LEAN ? 32 * NPL : (routed ? a.N : a.S);
  const int slot = LEAN ? 0 : (routed ? (a.perm ? a.perm[row] : row) : row - a.BK);
  const float* hrow = a.h + static_cast<size_t>(row) * a.Nh;
  int32_t* kidx = (!LEAN && a.kept_idx) ? a.kept_idx + static_cast<size_t>(row) * a.Nh : nullptr;
  float* kval = (!LEAN && a.kept_val) ? a.kept_val + static_cast<size_t>(row) * a.Nh : nullptr;
  __nv_bfloat16* hb = (LEAN || a.hb) ? a.hb + static_cast<size_t>(row) * a.Nh : nullptr;
  uint8_t* mout = LEAN ? nullptr : routed ? (a.mask_out_routed ? a.mask_out_routed + static_cast<size_t>(slot) * n
                                              : nullptr)
                         : (a.mask_out_shared ? a.mask_out_shared + static_cast<size_t>(slot) * n
                                              : nullptr);
  const uint8_t* min_ = nullptr;
  int mode = LEAN ? kSelectTopk : a.mode;
  if (!LEAN && mode == kSelectGiven) {
    min_ = routed ? a.mask_in_routed + static_cast<size_t>(slot) * n
                  : (a.mask_in_shared ? a.mask_in_shared + static_cast<size_t>(slot) * n : nullptr);
    if (min_ == nullptr) mode = kSelectAll;
  }
  // threshold selection (forward_sparse): |silu(gate)| >= tau on routed rows, the shared expert
  // stays dense (engine.cpp:352)
  const float* sgrow = nullptr;
  if (!LEAN && mode == kSelectThreshold) {
    if (routed) sgrow = a.sg + static_cast<size_t>(row) * a.Nh;
    else mode = kSelectAll;
  }
  int n_off = LEAN ? a.n_off_routed : 0;
  if (!LEAN && mode == kSelectTopk) {
    n_off = a.counts ? a.counts[row]
                     : (routed ? (a.slot_counts ? a.slot_counts[slot % a.K] : a.n_off_routed)
                               : a.n_off_shared);
    if (n_off <= 0) mode = kSelectAll;  // activation.cpp:35
  }
  const bool drop_everything = !LEAN && (mode == kSelectTopk) && n_off >= n;  // activation.cpp:36-39

  const int i0 = lane * NPL;
  const bool vec = LEAN || (a.Nh & 3) == 0;  // rows start 16-byte aligned
  auto load_row = [&](const float* src, float (&dst)[NPL]) {
#pragma unroll
    for (int v = 0; v < NPL; v += 4) {
      if (vec && (LEAN || i0 + v + 4 <= n)) {
        const float4 q = *reinterpret_cast<const float4*>(src + i0 + v);
        dst[v] = q.x;
        dst[v + 1] = q.y;
        dst[v + 2] = q.z;
        dst[v + 3] = q.w;
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) dst[v + q] = (i0 + v + q < n) ? src[i0 + v + q] : 0.0f;
      }
    }
  };
  float hv[NPL];
  load_row(hrow, hv);
  constexpr int KW = (NPL + 31) / 32;
  unsigned keepw[KW];  // bit j: neuron i0 + j survives
#pragma unroll
  for (int w = 0; w < KW; ++w) keepw[w] = 0u;
#define KEEP_SET(j, cond) keepw[(j) >> 5] |= (cond) ? (1u << ((j) & 31)) : 0u
#define KEEP_GET(j) ((keepw[(j) >> 5] >> ((j) & 31)) & 1u)
  if (!LEAN && mode == kSelectAll) {
#pragma unroll
    for (int j = 0; j < NPL; ++j) KEEP_SET(j, i0 + j < n);
  } else if (!LEAN && mode == kSelectGiven) {
#pragma unroll
    for (int j = 0; j < NPL; ++j) KEEP_SET(j, i0 + j < n && min_[i0 + j] != 0);
  } else if (!LEAN && mode == kSelectThreshold) {
    float sg[NPL];
    load_row(sgrow, sg);
#pragma unroll
    for (int j = 0; j < NPL; ++j)
      KEEP_SET(j, i0 + j < n && fabsf(sg[j]) >= a.tau);
  } else if (!drop_everything) {
    uint32_t kr[NPL];
#pragma unroll
    for (int j = 0; j < NPL; ++j)
      kr[j] = (LEAN || i0 + j < n) ? (__float_as_uint(hv[j]) & 0x7fffffffu) : 0xffffffffu;
    SEL_STAMP(2);
    const RowPick pk = warp_hist_pick<NPL>(kr, n_off, pick_hist[warp], pick_scratch[warp]);
    SEL_STAMP(3);
    int my_ties = 0;
#pragma unroll
    for (int j = 0; j < NPL; ++j) my_ties += (kr[j] == pk.pivot) ? 1 : 0;
    int tie_rank = warp_excl_scan(my_ties);  // ties at lower indices
#pragma unroll
    for (int j = 0; j < NPL; ++j) {
      const bool tie = kr[j] == pk.pivot;
      const bool above = kr[j] > pk.pivot && (LEAN || kr[j] != 0xffffffffu);
      KEEP_SET(j, above || (tie && tie_rank >= pk.ties_to_drop));
      tie_rank += tie ? 1 : 0;
    }
  }

  int my_kept = 0;
#pragma unroll
  for (int w = 0; w < KW; ++w) my_kept += __popc(keepw[w]);
  if (kidx) {
    int pos = warp_excl_scan(my_kept);
#pragma unroll
    for (int j = 0; j < NPL; ++j) {
      if KEEP_GET(j) {
        kidx[pos] = i0 + j;
        if (kval) kval[pos] = hv[j];
        ++pos;
      }
    }
  }
  if (mout) {
#pragma unroll
    for (int j = 0; j < NPL; ++j)
      if (i0 + j < n) mout[i0 + j] = static_cast<uint8_t>KEEP_GET(j);
  }
  if (hb) {
    const int kext = LEAN ? 32 * NPL : (routed ? a.kext_routed : a.kext_shared);
    const bool vec8 = LEAN || ((a.Nh & 7) == 0 && (kext & 7) == 0);
#pragma unroll
    for (int j = 0; j < NPL; ++j) hv[j] = KEEP_GET(j) ? hv[j] : 0.0f;
    for (int sp = 0; sp < a.nsplit; ++sp) {
      __nv_bfloat16* dst = hb + static_cast<size_t>(sp) * a.hb_split_stride;
#pragma unroll
      for (int v = 0; v < NPL; v += 8) {
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const __nv_bfloat16 lo = __float2bfloat16_rn(hv[v + 2 * q]);
          const __nv_bfloat16 hi = __float2bfloat16_rn(hv[v + 2 * q + 1]);
          hv[v + 2 * q] = __fsub_rn(hv[v + 2 * q], __bfloat162float(lo));
          hv[v + 2 * q + 1] = __fsub_rn(hv[v + 2 * q + 1], __bfloat162float(hi));
          w[q] = static_cast<uint32_t>(__bfloat16_as_ushort(lo)) |
                 (static_cast<uint32_t>(__bfloat16_as_ushort(hi)) << 16);
        }
        if (vec8) {
          if (LEAN || i0 + v < kext) *reinterpret_cast<uint4*>(dst + i0 + v) = make_uint4(w[0], w[1], w[2], w[3]);
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (i0 + v + q < kext)
              dst[i0 + v + q] = __ushort_as_bfloat16(static_cast<unsigned short>(w[q >> 1] >> ((q & 1) * 16)));
        }
      }
    }
  }
  if (a.kept_cnt) {
    const int total = __reduce_add_sync(0xffffffffu, my_kept);
    if (lane == 0) a.kept_cnt[row] = total;
  }
  SEL_STAMP(4);
#undef KEEP_SET
#undef KEEP_GET
}

static bool select_is_lean(const SelectArgs& a) {
  const int nmax = a.N > a.S ? a.N : a.S;
  const int kmax = a.hb ? (a.kext_routed > a.kext_shared ? a.kext_routed : a.kext_shared) : nmax;
  const int span = nmax > kmax ? nmax : kmax;
  if (!(span <= 1024 && a.rows >= 64)) return false;
  const int n = a.N;
  const bool uniform_rows = a.rows == a.BK || (a.S == a.N && a.n_off_shared == a.n_off_routed &&
                                               a.kext_shared == a.kext_routed);
  return a.mode == kSelectTopk && a.counts == nullptr && a.slot_counts == nullptr &&
         a.mask_out_routed == nullptr && a.mask_out_shared == nullptr && a.kept_idx == nullptr &&
         a.hb != nullptr && uniform_rows && a.kext_routed == n && (a.Nh & 7) == 0 &&
         a.n_off_routed > 0 && a.n_off_routed < n && (n == 256 || n == 512 || n == 1024);
}

int launch_select(const LaunchCtx& ctx, const SelectArgs& a) {
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = ctx.pdl ? 1 : 0;
  cfg.stream = ctx.stream;
  cfg.blockDim = dim3(kSelectThreads);
  const int nmax = a.N > a.S ? a.N : a.S;
  const int kmax = a.hb ? (a.kext_routed > a.kext_shared ? a.kext_routed : a.kext_shared) : nmax;
  const int span = nmax > kmax ? nmax : kmax;
  // Many rows: one warp per row (throughput).  Few rows, or rows too long for registers: one
  // CTA per row (latency).
  // (rows of 2880 neurons as 96 keys per lane, one CTA per SM: measured slower than a CTA per
  // row -- GPT-OSS shape prefill, 16384 rows: 0.43 vs 0.35 ms)
  if (span <= 1024 && a.rows >= 64) {
    cfg.gridDim = dim3(ceil_div(a.rows, kSelWarps));
    // the batch hot case gets the instantiation with everything else compiled out
    const int n = a.N;
    if (select_is_lean(a)) {
      if (n == 256) cudaLaunchKernelEx(&cfg, select_rows_warp_kernel<8, true>, a);
      else if (n == 512) cudaLaunchKernelEx(&cfg, select_rows_warp_kernel<16, true>, a);
      else cudaLaunchKernelEx(&cfg, select_rows_warp_kernel<32, true>, a);
      return 1;
    }
    if (span <= 256) cudaLaunchKernelEx(&cfg, select_rows_warp_kernel<8, false>, a);
    else if (span <= 512) cudaLaunchKernelEx(&cfg, select_rows_warp_kernel<16, false>, a);
    else cudaLaunchKernelEx(&cfg, select_rows_warp_kernel<32, false>, a);
    return 1;
  }
  cfg.gridDim = dim3(a.rows);
  cfg.dynamicSmemBytes = static_cast<size_t>(nmax) * sizeof(uint32_t);
  if (cfg.dynamicSmemBytes > 40 * 1024) {
    // rows beyond ~10K keys: above the 48 KB default together with the static scratch
    static int smem_set[64] = {};  // per device
    int dev = 0;
    cudaGetDevice(&dev);
    const int want = static_cast<int>(cfg.dynamicSmemBytes);
    if (want > __atomic_load_n(&smem_set[dev & 63], __ATOMIC_ACQUIRE)) {
      cudaFuncSetAttribute(select_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, want);
      __atomic_store_n(&smem_set[dev & 63], want, __ATOMIC_RELEASE);
    }
  }
  cudaLaunchKernelEx(&cfg, select_rows_kernel, a);
  return 1;
}


// ---------------------------------------------------------------------------------------------
// The threshold variant's index layout (activation.cpp:62-114): keep iff |silu(g)| >= tau, then
// per token the flat list of kept (expert * N + neuron) indices in (slot ascending, neuron
// ascending) order, padded with -1 to `capacity`, clamped where the list is full.
// ---------------------------------------------------------------------------------------------
// silu with the exponential evaluated in double and rounded to float: what glibc's expf returns,
// so that values within an ulp of tau fall on the reference's side (activation.cpp:15)
__device__ __forceinline__ float silu_ref(float x) {
  return __fdiv_rn(x, __fadd_rn(1.0f, static_cast<float>(exp(static_cast<double>(-x)))));
}

__global__ void __launch_bounds__(256) threshold_mask_kernel(const float* __restrict__ g, size_t n,
                                                             float tau, uint8_t* __restrict__ mask) {
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) mask[i] = fabsf(silu_ref(g[i])) >= tau ? 1 : 0;
}

// One CTA per token.  masks [K][N] of the token, ids [K]; flat [capacity], per_slot [K], total [1].
__global__ void __launch_bounds__(kSelectThreads) compact_active_kernel(
    const uint8_t* __restrict__ masks, const int32_t* __restrict__ ids, int K, int N, int capacity,
    int32_t* __restrict__ flat, int32_t* __restrict__ per_slot, int32_t* __restrict__ total) {
  __shared__ SelScratch sc;
  const int t = blockIdx.x, tid = threadIdx.x;
  masks += static_cast<size_t>(t) * K * N;
  ids += static_cast<size_t>(t) * K;
  flat += static_cast<size_t>(t) * capacity;
  per_slot += static_cast<size_t>(t) * K;
  for (int i = tid; i < capacity; i += kSelectThreads) flat[i] = -1;
  __syncthreads();
  int write_base = 0, buf = 0;
  for (int s = 0; s < K; ++s) {
    const uint8_t* m = masks + static_cast<size_t>(s) * N;
    const int base = ids[s] * N;
    int running = 0;  // survivors of this slot before the current block of 256 neurons
    for (int i0 = 0; i0 < N; i0 += kSelectThreads) {
      const int i = i0 + tid;
      const bool keep = i < N && m[i] != 0;
      int blk_total = 0;
      const int rank = sel_block_rank(keep, sc, buf, blk_total);
      buf ^= 1;
      const int wpos = write_base + running + rank;
      if (keep && wpos < capacity) flat[wpos] = base + i;
      running += blk_total;
    }
    const int room = capacity - write_base;
    const int actual = running < room ? running : room;
    if (tid == 0) per_slot[s] = actual;
    write_base += actual;
  }
  if (tid == 0) total[t] = write_base;
}

int launch_threshold_mask(cudaStream_t s, const float* g, size_t n, float tau, uint8_t* mask) {
  if (n == 0) return 0;
  threshold_mask_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(g, n, tau, mask);
  return 1;
}

int launch_compact_active(cudaStream_t s, const uint8_t* masks, const int32_t* ids, int batch, int K,
                          int N, int capacity, int32_t* flat, int32_t* per_slot, int32_t* total) {
  if (batch == 0) return 0;
  compact_active_kernel<<<batch, kSelectThreads, 0, s>>>(masks, ids, K, N, capacity, flat, per_slot,
                                                         total);
  return 1;
}

}  // namespace skb
