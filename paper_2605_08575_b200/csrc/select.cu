// select.cu -- subsystem (3): per-(token, expert) neuron selection.  Ranks post-activation
// magnitudes |h| and drops the n_off smallest with a CTA-wide radix select in shared memory;
// no sort is performed.  Emits the ascending survivor list (indices + values) that the
// down-projection gathers, the survivor count, and optionally the uint8 mask.
//
// Bit-exact restatement of mask_smallest_magnitudes / topk_mask
// (proj/src/activation.cpp:31-60): key = bits(h) & 0x7fffffff is monotone in |h|; among keys
// equal to the pivot the LOWER indices are dropped first (stable_sort, activation.cpp:42-50).
#include "skb_internal.cuh"

namespace skb {

namespace {

constexpr int kWarps = kSelectThreads / 32;

struct ScanScratch {
  int warp_cnt[2][kWarps];
};

// Exclusive prefix of `flag` over the CTA in thread order; `buf` alternates between calls so a
// single __syncthreads per scan suffices.
__device__ __forceinline__ int block_rank(bool flag, ScanScratch& sc, int buf, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned b = __ballot_sync(0xffffffffu, flag);
  if (lane == 0) sc.warp_cnt[buf][warp] = __popc(b);
  __syncthreads();
  int base = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    const int c = sc.warp_cnt[buf][w];
    if (w < warp) base += c;
    tot += c;
  }
  total = tot;
  return base + __popc(b & ((1u << lane) - 1u));
}

}  // namespace

__global__ void __launch_bounds__(kSelectThreads) select_rows_kernel(SelectArgs a) {
  extern __shared__ uint32_t keys[];  // [max(N,S)]
  __shared__ uint32_t hist[kWarps][256];
  __shared__ ScanScratch sc;
  __shared__ int s_bin, s_before, s_equal;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int row = blockIdx.x;
  const bool routed = row < a.BK;
  const int n = routed ? a.N : a.S;

  pdl_wait();
  pdl_launch_dependents();

  const int slot = routed ? (a.perm ? a.perm[row] : row) : row - a.BK;
  const float* hrow = a.h + static_cast<size_t>(row) * a.Nh;
  int32_t* kidx = a.kept_idx + static_cast<size_t>(row) * a.Nh;
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

  int n_off = 0;
  if (mode == kSelectTopk) {
    n_off = a.counts ? a.counts[row] : (routed ? a.n_off_routed : a.n_off_shared);
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
      for (int i = tid; i < n; i += kSelectThreads)
        keys[i] = __float_as_uint(hrow[i]) & 0x7fffffffu;
      // MSB-first radix select of the n_off-th smallest key: digits [30:23] [22:15] [14:7] [6:0]
      uint32_t prefix = 0;
      int remaining = n_off;  // 1-based rank of the target among the current candidates
      int decided_bits = 0;
#pragma unroll 1
      for (int pass = 0; pass < 4; ++pass) {
        const int bits = (pass == 3) ? 7 : 8;
        const int shift = 31 - decided_bits - bits;
        const uint32_t dmask = (1u << bits) - 1u;
        for (int i = tid; i < kWarps * 256; i += kSelectThreads) (&hist[0][0])[i] = 0;
        __syncthreads();
        for (int i = tid; i < n; i += kSelectThreads) {
          const uint32_t k = keys[i];
          const bool cand = (decided_bits == 0) || ((k >> (shift + bits)) == prefix);
          if (cand) atomicAdd(&hist[warp][(k >> shift) & dmask], 1u);
        }
        __syncthreads();
        if (warp == 0) {
          // lane owns bins [8*lane, 8*lane+8)
          uint32_t tot[8];
          uint32_t mine = 0;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            uint32_t t = 0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) t += hist[w][8 * lane + j];
            tot[j] = t;
            mine += t;
          }
          uint32_t incl = mine;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
          }
          uint32_t run = incl - mine;  // keys in lower bins
          int found_bin = -1;
          uint32_t found_before = 0, found_equal = 0;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (found_bin < 0 && run + tot[j] >= static_cast<uint32_t>(remaining)) {
              found_bin = 8 * lane + j;
              found_before = run;
              found_equal = tot[j];
            }
            run += tot[j];
          }
          const unsigned who = __ballot_sync(0xffffffffu, found_bin >= 0);
          if (lane == __ffs(who) - 1) {
            s_bin = found_bin;
            s_before = static_cast<int>(found_before);
            s_equal = static_cast<int>(found_equal);
          }
        }
        __syncthreads();
        prefix = (prefix << bits) | static_cast<uint32_t>(s_bin);
        remaining -= s_before;
        decided_bits += bits;
      }
      pivot = prefix;
      ties_to_drop = remaining;
      drop_all_ties = (ties_to_drop == s_equal);
    }
  }

  // ---- ordered compaction: rounds of 256 consecutive indices ----
  int kept_base = 0, tie_base = 0, buf = 0;
  const int rounds = ceil_div(n, kSelectThreads);
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
        const int tie_rank = tie_base + block_rank(tie, sc, buf, tie_total);
        buf ^= 1;
        tie_base += tie_total;
        keep = valid && (k > pivot || (tie && tie_rank >= ties_to_drop));
      }
    }
    int kept_total;
    const int pos = kept_base + block_rank(keep, sc, buf, kept_total);
    buf ^= 1;
    kept_base += kept_total;
    if (keep) {
      kidx[pos] = i;
      if (kval) kval[pos] = hv;
    }
    if (mout && valid) mout[i] = keep ? 1 : 0;
  }
  if (tid == 0) a.kept_cnt[row] = kept_base;
}

int launch_select(const LaunchCtx& ctx, const SelectArgs& a) {
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = ctx.pdl ? 1 : 0;
  cfg.stream = ctx.stream;
  cfg.gridDim = dim3(a.rows);
  cfg.blockDim = dim3(kSelectThreads);
  const int nmax = a.N > a.S ? a.N : a.S;
  cfg.dynamicSmemBytes = static_cast<size_t>(nmax) * sizeof(uint32_t);
  cudaLaunchKernelEx(&cfg, select_rows_kernel, a);
  return 1;
}

}  // namespace skb
