// select_device.cuh -- CTA-wide neuron selection shared by select.cu (stand-alone selection:
// masks and survivor lists in global memory) and down.cu (selection fused in front of the
// gather).  256 threads per CTA.
//
// Bit-exact restatement of mask_smallest_magnitudes / topk_mask
// (proj/src/activation.cpp:31-60): key = bits(h) & 0x7fffffff is monotone in |h|; the n_off
// smallest keys are dropped; among keys equal to the pivot the LOWER indices are dropped first
// (stable_sort, activation.cpp:42-50).  No sort: an 8-ary search over the key value finds the
// pivot, a ballot/popc prefix orders the survivors.
#pragma once

#include "skb_internal.cuh"

namespace skb {

constexpr int kSelWarps = kSelectThreads / 32;

struct SelScratch {
  int kcnt[2][kSelWarps];      // per-threshold counts of the k-ary search (double buffered)
  int warp_cnt[2][kSelWarps];  // ballot prefix scratch of sel_block_rank (double buffered)
};

// Who runs a CTA-wide selection: the whole 256-thread CTA (select.cu, down.cu), or the eight
// down-projection warps of the fused decode kernel behind a named barrier (decode.cu).
struct SelWholeCta {
  __device__ static __forceinline__ int tid() { return threadIdx.x; }
  __device__ static __forceinline__ void sync() { __syncthreads(); }
};

// What survives in one row: keys > pivot, plus keys == pivot whose rank among the ties (by
// ascending index) is >= ties_to_drop.
struct RowPick {
  uint32_t pivot;
  int ties_to_drop;
  bool drop_all_ties;
};

// Exclusive prefix of `flag` over the CTA in thread order; `buf` alternates between calls so a
// single __syncthreads per scan suffices.
__device__ __forceinline__ int sel_block_rank(bool flag, SelScratch& sc, int buf, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned b = __ballot_sync(0xffffffffu, flag);
  if (lane == 0) sc.warp_cnt[buf][warp] = __popc(b);
  __syncthreads();
  int base = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < kSelWarps; ++w) {
    const int c = sc.warp_cnt[buf][w];
    if (w < warp) base += c;
    tot += c;
  }
  total = tot;
  return base + __popc(b & ((1u << lane) - 1u));
}

// keys[0..n) in shared memory; 0 < n_off < n.  Every thread returns the same RowPick.
//
// 8-ary search on the key VALUE (31 bits, 3 bits per step, 11 steps): warp w counts the keys
// below threshold lo + (w+1) << shift; the counts are monotone in w, so the digit is the number
// of thresholds whose count is still below the wanted rank.  Pure compare + warp reduce: no
// shared-memory atomics (a 256-bin atomic histogram costs ~2 cycles per key per pass on the
// SM's single shared-memory pipe and made the selection the slowest part of decode).
// For n <= 1024 every warp keeps all keys in registers (32 per lane).
template <class CTX = SelWholeCta>
__device__ __forceinline__ RowPick sel_kary_pick(const uint32_t* keys, int n, int n_off,
                                                 SelScratch& sc) {
  static_assert(kSelWarps == 8, "one threshold per warp, 3 bits per step");
  const int lane = CTX::tid() & 31, warp = CTX::tid() >> 5;
  const bool in_regs = n <= 1024;
  uint32_t kr[32];
  if (in_regs) {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int i = j * 32 + lane;
      kr[j] = (i < n) ? keys[i] : 0xffffffffu;  // padding never falls below a threshold
    }
  }
  uint32_t lo = 0;
  int below = 0, equal = 0, bits = 31, buf = 0;
#pragma unroll 1
  while (bits > 0) {
    const int b = bits >= 3 ? 3 : bits;
    const int shift = bits - b;
    const int n_thr = 1 << b;  // thresholds lo + (q+1) << shift, q < n_thr; the last one is hi
    if (warp < n_thr) {
      const uint32_t T = lo + (static_cast<uint32_t>(warp + 1) << shift);
      int c = 0;
      if (in_regs) {
        // four partial counts: a single accumulator is a 32-deep dependent add chain
        int c0 = 0, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          c0 += (kr[j] < T) ? 1 : 0;
          c1 += (kr[j + 1] < T) ? 1 : 0;
          c2 += (kr[j + 2] < T) ? 1 : 0;
          c3 += (kr[j + 3] < T) ? 1 : 0;
        }
        c = (c0 + c1) + (c2 + c3);
      } else {
#pragma unroll 8
        for (int i = lane; i < n; i += 32) c += (keys[i] < T) ? 1 : 0;
      }
      c = __reduce_add_sync(0xffffffffu, c);
      if (lane == 0) sc.kcnt[buf][warp] = c;
    }
    CTX::sync();
    int d = 0, nb = below;
#pragma unroll
    for (int q = 0; q < 7; ++q) {
      if (q < n_thr - 1) {
        const int cq = sc.kcnt[buf][q];
        if (cq < n_off) {
          d = q + 1;
          nb = cq;
        }
      }
    }
    equal = sc.kcnt[buf][d] - nb;  // keys inside the chosen sub-interval
    lo += static_cast<uint32_t>(d) << shift;
    below = nb;
    bits -= b;
    buf ^= 1;
  }
  RowPick p;
  p.pivot = lo;                  // the n_off-th smallest key
  p.ties_to_drop = n_off - below;  // keys < pivot are all dropped; then the first ties
  p.drop_all_ties = (p.ties_to_drop == equal);
  return p;
}

// Histogram-assisted pick (the selection of the fused decode kernel, as a CTA-wide function):
// a 512-bin histogram over exponent + 3 mantissa bits of the key (shared-memory atomics, one pass)
// locates the bucket of the n_off-th smallest key; only that bucket's keys -- typically a few
// dozen -- are ranked exactly.  Buckets above kSelMemberCap keys (many equal or clamped values)
// fall back to the general search.  Same result as sel_kary_pick, bit for bit; ~5x fewer
// instructions and 4 barriers instead of 11 for rows that do not fit in registers.
constexpr int kSelHistBins = 512;
constexpr int kSelHistBase = (135 << 3) - (kSelHistBins - 1);  // top bin: keys >= 2^8
constexpr int kSelMemberCap = 1024;
struct SelHistScratch {
  int hist[kSelHistBins];
  uint32_t members[kSelMemberCap + 4];
  int wsum[kSelWarps];
  int bstar, below_bins, m, filled, pivot, below, equal;
};
__device__ __forceinline__ int sel_hist_bin(uint32_t key) {
  const int b = static_cast<int>(key >> 20) - kSelHistBase;
  return b < 0 ? 0 : (b > kSelHistBins - 1 ? kSelHistBins - 1 : b);
}
__device__ __forceinline__ RowPick sel_hist_pick(const uint32_t* keys, int n, int n_off,
                                                 SelHistScratch& hs, SelScratch& sc) {
  static_assert(kSelectThreads * 2 == kSelHistBins, "two bins per thread");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  hs.hist[2 * tid] = 0;
  hs.hist[2 * tid + 1] = 0;
  for (int i = tid; i < kSelMemberCap + 4; i += kSelectThreads) hs.members[i] = 0xffffffffu;
  if (tid == 0) hs.filled = 0;
  __syncthreads();
  for (int i = tid; i < n; i += kSelectThreads) atomicAdd(&hs.hist[sel_hist_bin(keys[i])], 1);
  __syncthreads();
  const int h0 = hs.hist[2 * tid], h1 = hs.hist[2 * tid + 1];
  int incl = h0 + h1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int up = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += up;
  }
  if (lane == 31) hs.wsum[warp] = incl;
  __syncthreads();
  int base = 0;
#pragma unroll
  for (int w = 0; w < kSelWarps; ++w)
    if (w < warp) base += hs.wsum[w];
  incl += base;
  const int excl = incl - (h0 + h1);
  if (excl < n_off && n_off <= incl) {  // exactly one thread: the bucket of the n_off-th key
    const bool first = n_off <= excl + h0;
    hs.bstar = 2 * tid + (first ? 0 : 1);
    hs.below_bins = first ? excl : excl + h0;
    hs.m = first ? h0 : h1;
  }
  __syncthreads();
  const int bstar = hs.bstar, below_bins = hs.below_bins, M = hs.m;
  if (M > kSelMemberCap) return sel_kary_pick(keys, n, n_off, sc);
  for (int i = tid; i < n; i += kSelectThreads) {
    const uint32_t k = keys[i];
    if (sel_hist_bin(k) == bstar) hs.members[atomicAdd(&hs.filled, 1)] = k;
  }
  __syncthreads();
  const int rr = n_off - below_bins;  // 1-based rank inside the bucket
  const int M4 = (M + 3) >> 2;
  for (int mi = tid; mi < M; mi += kSelectThreads) {
    const uint32_t k = hs.members[mi];
    int lt = 0, le = 0;
    for (int q4 = 0; q4 < M4; ++q4) {
      const uint4 mm = *reinterpret_cast<const uint4*>(hs.members + 4 * q4);
      lt += (mm.x < k) + (mm.y < k) + (mm.z < k) + (mm.w < k);
      le += (mm.x <= k) + (mm.y <= k) + (mm.z <= k) + (mm.w <= k);
    }
    if (lt < rr && rr <= le) {  // every holder of the pivot value writes the same three words
      hs.pivot = static_cast<int>(k);
      hs.below = below_bins + lt;
      hs.equal = le - lt;
    }
  }
  __syncthreads();
  RowPick p;
  p.pivot = static_cast<uint32_t>(hs.pivot);
  p.ties_to_drop = n_off - hs.below;
  p.drop_all_ties = (p.ties_to_drop == hs.equal);
  __syncthreads();  // the scratch may be reused by the caller's next row
  return p;
}

// One warp, keys in registers (any assignment of elements to lanes; 0xffffffff marks slots past
// the end of the row), 0 < n_off < n.  Finds the n_off-th smallest key:
//   1. the bits all keys share are skipped (warp min / max);
//   2. bit-by-bit counting steps (NPL compares + one warp reduce each) narrow the pivot's value
//      interval until it holds at most 32 keys -- typically ~8 steps for a 512-neuron row;
//   3. those keys are compacted one per lane through `scratch` (33 words of shared memory owned
//      by this warp) and the remaining bits cost one compare + ballot each.
// Every lane returns the same RowPick.  Instruction count is what bounds a batch-sized
// selection (2048 rows: the 31-step version was 4000 warp instructions per row, 49 % issue
// utilisation over 19 us -- profiles/README.md), hence the effort to cut steps.
template <int NPL>
__device__ __forceinline__ RowPick warp_binary_pick(const uint32_t (&kr)[NPL], int n, int n_off,
                                                    uint32_t* scratch) {
  const int lane = threadIdx.x & 31;
  uint32_t mn = 0xffffffffu;
  int mx = -1;  // signed: the 0xffffffff fillers are -1 and never win
#pragma unroll
  for (int j = 0; j < NPL; ++j) {
    mn = min(mn, kr[j]);
    mx = max(mx, static_cast<int>(kr[j]));
  }
  mn = __reduce_min_sync(0xffffffffu, mn);
  mx = __reduce_max_sync(0xffffffffu, mx);
  RowPick pk;
  if (mn == static_cast<uint32_t>(mx)) {  // one value: the lowest n_off indices go
    pk.pivot = mn;
    pk.ties_to_drop = n_off;
    pk.drop_all_ties = false;
    return pk;
  }
  int b = 31 - __clz(mn ^ static_cast<uint32_t>(mx));  // highest bit in which two keys differ
  uint32_t p = mn & ~((2u << b) - 1u);
  int below = 0, upper = n;
  // invariant: the pivot lies in [p, p + 2^(b+1)); below = #keys < p; upper = #keys < p + 2^(b+1)
#pragma unroll 1
  while (b >= 0 && upper - below > 32) {
    const uint32_t T = p | (1u << b);
    int c0 = 0, c1 = 0, c2 = 0, c3 = 0;  // partial counts: no NPL-deep dependent add chain
#pragma unroll
    for (int j = 0; j < NPL; j += 4) {
      c0 += (kr[j] < T) ? 1 : 0;
      c1 += (kr[j + 1] < T) ? 1 : 0;
      c2 += (kr[j + 2] < T) ? 1 : 0;
      c3 += (kr[j + 3] < T) ? 1 : 0;
    }
    const int c = __reduce_add_sync(0xffffffffu, (c0 + c1) + (c2 + c3));
    if (c < n_off) {  // fewer than n_off keys below T: the pivot is >= T
      p = T;
      below = c;
    } else {
      upper = c;
    }
    --b;
  }
  int ties = upper - below;
  if (b >= 0) {
    // at most 32 keys left in the interval: one per lane
    if (lane == 0) scratch[32] = 0u;
    __syncwarp();
    const uint32_t width = 2u << b;
#pragma unroll
    for (int j = 0; j < NPL; ++j)
      if (kr[j] - p < width) scratch[atomicAdd(&scratch[32], 1u)] = kr[j];
    __syncwarp();
    const uint32_t mine = lane < upper - below ? scratch[lane] : 0xffffffffu;
    __syncwarp();
    const int outside = below;  // keys below the interval; `mine` holds everything inside it
#pragma unroll 1
    for (; b >= 0; --b) {
      const uint32_t T = p | (1u << b);
      const int c = outside + __popc(__ballot_sync(0xffffffffu, mine < T));
      if (c < n_off) {
        p = T;
        below = c;
      }
    }
    ties = __popc(__ballot_sync(0xffffffffu, mine == p));
  }
  pk.pivot = p;
  pk.ties_to_drop = n_off - below;
  pk.drop_all_ties = (pk.ties_to_drop == ties);
  return pk;
}

// The same pick by radix histograms (the batch path: keys in registers).
// warp_binary_pick narrows the pivot's interval one bit -- one warp reduce -- at a time: ~30
// dependent steps, measured 3.3 us per 512-neuron row (median, up to 6) with 14 rows per SM in
// flight.  Here a pass drops the keys of the current interval into 256 equal-width bins of the
// warp's own shared-memory histogram (8 bits of the key per pass), a warp scan of the bin counts
// finds the bin that holds the n_off-th smallest key, and as soon as that bin holds at most 32
// keys they are ranked against each other directly (one key per lane, 32 shuffles).  Typically
// two passes + the ranking: ~10 dependent phases.  Every lane returns the same RowPick, bit for
// bit the one warp_binary_pick returns.
//   hist: 256 ints, scratch: 33 words, both private to the warp.
template <int NPL>
__device__ __forceinline__ RowPick warp_hist_pick(const uint32_t (&kr)[NPL], int n_off, int* hist,
                                                  uint32_t* scratch) {
  const int lane = threadIdx.x & 31;
  // slots past the end of a row hold 0xffffffff: as signed values they never win the maximum,
  // and key - p exceeds every interval width below, so no later phase sees them
  uint32_t mn = 0xffffffffu;
  int mxs = -1;
#pragma unroll
  for (int j = 0; j < NPL; ++j) {
    mn = min(mn, kr[j]);
    mxs = max(mxs, static_cast<int>(kr[j]));
  }
  mn = __reduce_min_sync(0xffffffffu, mn);
  const uint32_t mx = static_cast<uint32_t>(__reduce_max_sync(0xffffffffu, mxs));
  RowPick pk;
  if (mn == mx) {  // one value: the lowest n_off indices go
    pk.pivot = mn;
    pk.ties_to_drop = n_off;
    pk.drop_all_ties = false;
    return pk;
  }
  int b = 31 - __clz(mn ^ mx);           // the interval is [p, p + 2^(b+1))
  uint32_t p = mn & ~((2u << b) - 1u);   // (b == 31: 2u << 31 wraps to 0, the mask to 0: p = 0)
  int below = 0;                         // keys < p
  int r = n_off;                         // 1-based rank of the pivot among the keys >= p
  int m_in = 0;                          // keys inside the final interval
  while (true) {
    const int shift = b + 1 > 8 ? b + 1 - 8 : 0;  // bin width 2^shift, at most 256 bins
    const uint32_t span = (2u << b) - 1u;         // interval width - 1
    __syncwarp();
    *reinterpret_cast<int4*>(hist + 8 * lane) = make_int4(0, 0, 0, 0);
    *reinterpret_cast<int4*>(hist + 8 * lane + 4) = make_int4(0, 0, 0, 0);
    __syncwarp();
#pragma unroll
    for (int j = 0; j < NPL; ++j) {
      const uint32_t d = kr[j] - p;
      if (d <= span) atomicAdd(&hist[d >> shift], 1);
    }
    __syncwarp();
    const int4 h0 = *reinterpret_cast<const int4*>(hist + 8 * lane);
    const int4 h1 = *reinterpret_cast<const int4*>(hist + 8 * lane + 4);
    const int hq[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
    const int tot = ((hq[0] + hq[1]) + (hq[2] + hq[3])) + ((hq[4] + hq[5]) + (hq[6] + hq[7]));
    int incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int excl = incl - tot;
    // exactly one lane's eight bins hold rank r
    int bin = 0, under = 0, m = 0;
    if (excl < r && r <= incl) {
      int run = excl;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (run < r && r <= run + hq[q]) {
          bin = 8 * lane + q;
          under = run;
          m = hq[q];
        }
        run += hq[q];
      }
    }
    const int src = __ffs(__ballot_sync(0xffffffffu, excl < r && r <= incl)) - 1;
    bin = __shfl_sync(0xffffffffu, bin, src);
    under = __shfl_sync(0xffffffffu, under, src);
    m = __shfl_sync(0xffffffffu, m, src);
    below += under;
    r -= under;
    p += static_cast<uint32_t>(bin) << shift;
    if (shift == 0) {  // the bin is one key value
      pk.pivot = p;
      pk.ties_to_drop = n_off - below;
      pk.drop_all_ties = (pk.ties_to_drop == m);
      return pk;
    }
    b = shift - 1;
    m_in = m;
    if (m <= 32) break;
  }
  // at most 32 keys left in [p, p + 2^(b+1)): one per lane, ranked against each other
  const uint32_t span = (2u << b) - 1u;
  int cnt = 0;
#pragma unroll
  for (int j = 0; j < NPL; ++j) cnt += (kr[j] - p <= span) ? 1 : 0;
  int pos = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, pos, o);
    if (lane >= o) pos += t;
  }
  pos -= cnt;
  __syncwarp();
#pragma unroll
  for (int j = 0; j < NPL; ++j)
    if (kr[j] - p <= span) scratch[pos++] = kr[j];
  __syncwarp();
  const uint32_t mine = lane < m_in ? scratch[lane] : 0xffffffffu;
  int lt = 0, le = 0;
  for (int i = 0; i < m_in; ++i) {
    const uint32_t v = __shfl_sync(0xffffffffu, mine, i);
    lt += (v < mine) ? 1 : 0;
    le += (v <= mine) ? 1 : 0;
  }
  const bool hit = lane < m_in && lt < r && r <= le;
  const int src = __ffs(__ballot_sync(0xffffffffu, hit)) - 1;
  pk.pivot = __shfl_sync(0xffffffffu, mine, src);
  below += __shfl_sync(0xffffffffu, lt, src);
  const int ties = __shfl_sync(0xffffffffu, le - lt, src);
  pk.ties_to_drop = n_off - below;
  pk.drop_all_ties = (pk.ties_to_drop == ties);
  return pk;
}

// exclusive prefix sum over the lanes of a warp
__device__ __forceinline__ int warp_excl_scan(int v) {
  const int lane = threadIdx.x & 31;
  int s = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, s, o);
    if (lane >= o) s += t;
  }
  return s - v;
}

}  // namespace skb
