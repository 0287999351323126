// ep.cu -- device side of the expert-parallel data plane (paper_2605_08575_b200/ep.py): the send /
// receive matrix out of the all-gathered routing, the packed bf16 dispatch rows, and the ordered
// combine at the home rank.  The reference is single-process; the partitioning
// follows proj/src/engine.cpp:132-165 (experts independent given their tokens) and
// proj/src/router.cpp:119-130 (per-token sum over slots, ascending, multiply and add rounded
// separately).
//
// Packed dispatch row: [D bf16 token values][int32 local expert id][pad to 16 bytes].
#include <cstring>

#include "../../include/sparsekit_b200.h"
#include "skb_internal.cuh"

namespace skb {

namespace {

constexpr int kPlanThreads = 1024;
constexpr int kMaxWorld = 16;

__device__ __forceinline__ int owner_of(int e, const int32_t* lo, int W) {
  int r = 0;
#pragma unroll 1
  for (int i = 1; i < W; ++i)
    if (e >= lo[i]) r = i;
  return r;
}

// One CTA.  ids_all [W][Bmax][K] (ids < 0: padding of a short home batch).  Outputs:
//   cnt [W][W]      slots rank src sends to rank dst
//   pos [Bmax * K]  position of this rank's flat slot t*K+s in its send buffer (grouped by
//                   destination rank, ascending flat slot inside a group), -1 for padding
//   loc [Bmax * K]  expert id local to the destination rank
__global__ void __launch_bounds__(kPlanThreads) ep_plan_kernel(const int32_t* __restrict__ ids_all,
                                                               int W, int slots,
                                                               const int32_t* __restrict__ lo, int rank,
                                                               int32_t* __restrict__ cnt,
                                                               int32_t* __restrict__ pos,
                                                               int32_t* __restrict__ loc) {
  __shared__ int s_cnt[kMaxWorld * kMaxWorld];
  __shared__ int s_lo[kMaxWorld + 1];
  __shared__ int s_part[kPlanThreads / 32][kMaxWorld];  // per-warp counts of the own slots
  __shared__ int s_base[kMaxWorld];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < W * W; i += kPlanThreads) s_cnt[i] = 0;
  if (tid <= W) s_lo[tid] = lo[tid];
  __syncthreads();
  // the whole matrix: integer atomics (the result does not depend on their order)
  for (int i = tid; i < W * slots; i += kPlanThreads) {
    const int e = ids_all[i];
    if (e >= 0) atomicAdd(&s_cnt[(i / slots) * W + owner_of(e, s_lo, W)], 1);
  }
  __syncthreads();
  for (int i = tid; i < W * W; i += kPlanThreads) cnt[i] = s_cnt[i];
  if (tid < W) {  // start of every destination group in this rank's send buffer
    int b = 0;
    for (int d = 0; d < tid; ++d) b += s_cnt[rank * W + d];
    s_base[tid] = b;
  }
  // own slots: thread t takes the contiguous range [t * per, (t + 1) * per) -- stable order
  const int32_t* mine = ids_all + static_cast<size_t>(rank) * slots;
  const int per = ceil_div(slots, kPlanThreads);
  const int i0 = tid * per, i1 = min(slots, i0 + per);
  int c[kMaxWorld];
#pragma unroll
  for (int d = 0; d < kMaxWorld; ++d) c[d] = 0;
  for (int i = i0; i < i1; ++i) {
    const int e = mine[i];
    if (e >= 0) {
      const int d = owner_of(e, s_lo, W);
#pragma unroll
      for (int dd = 0; dd < kMaxWorld; ++dd) c[dd] += (dd == d) ? 1 : 0;
    }
  }
  // exclusive prefix over threads, per destination: warp scan, then the warps' totals
  int excl[kMaxWorld];
#pragma unroll
  for (int d = 0; d < kMaxWorld; ++d) {
    int v = c[d];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    excl[d] = v - c[d];
    if (lane == 31 && d < W) s_part[warp][d] = v;
  }
  __syncthreads();
#pragma unroll
  for (int d = 0; d < kMaxWorld; ++d) {
    if (d < W) {
      int b = s_base[d];
      for (int w = 0; w < warp; ++w) b += s_part[w][d];
      excl[d] += b;
    }
  }
  for (int i = i0; i < i1; ++i) {
    const int e = mine[i];
    int p = -1, l = 0;
    if (e >= 0) {
      const int d = owner_of(e, s_lo, W);
#pragma unroll
      for (int dd = 0; dd < kMaxWorld; ++dd)
        if (dd == d) p = excl[dd]++;
      l = e - s_lo[d];
    }
    pos[i] = p;
    loc[i] = l;
  }
}

// one warp per flat slot: token row -> bf16 into its packed send row, local expert id behind it
__global__ void __launch_bounds__(256) ep_pack_kernel(const float* __restrict__ x,
                                                      const int32_t* __restrict__ pos,
                                                      const int32_t* __restrict__ loc, int slots,
                                                      int K, int D, int stride,
                                                      uint8_t* __restrict__ send) {
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= slots) return;
  const int p = pos[i];
  if (p < 0) return;
  const float* src = x + static_cast<size_t>(i / K) * D;
  uint8_t* row = send + static_cast<size_t>(p) * stride;
  __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(row);
  for (int d = lane; d < D; d += 32) dst[d] = __float2bfloat16_rn(__ldg(src + d));
  if (lane == 0) *reinterpret_cast<int32_t*>(row + static_cast<size_t>(D) * 2) = loc[i];
}

// receiver: packed rows -> fp32 token rows + local expert ids (the layer's external-routing inputs)
__global__ void __launch_bounds__(256) ep_unpack_kernel(const uint8_t* __restrict__ recv, int rows,
                                                        int D, int stride, float* __restrict__ x,
                                                        int32_t* __restrict__ ids) {
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const uint8_t* row = recv + static_cast<size_t>(r) * stride;
  const __nv_bfloat16* src = reinterpret_cast<const __nv_bfloat16*>(row);
  float* dst = x + static_cast<size_t>(r) * D;
  for (int d = lane; d < D; d += 32) dst[d] = __bfloat162float(src[d]);
  if (lane == 0) ids[r] = *reinterpret_cast<const int32_t*>(row + static_cast<size_t>(D) * 2);
}

// home rank: y[t] = sum_s w(t, s) * back[pos(t, s)] in ascending slot order, multiply and add
// rounded separately (router.cpp:119-130), then the shared expert's output (engine.cpp:168-173)
__global__ void __launch_bounds__(256) ep_combine_kernel(const float* __restrict__ back,
                                                         const int32_t* __restrict__ pos,
                                                         const float* __restrict__ w,
                                                         const float* __restrict__ shared, int B,
                                                         int K, int D, float* __restrict__ y) {
  const int t = blockIdx.y;
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= B || d >= D) return;
  float acc = 0.0f;
  for (int s = 0; s < K; ++s) {
    const int p = pos[t * K + s];
    acc = __fadd_rn(acc, __fmul_rn(w[t * K + s], back[static_cast<size_t>(p) * D + d]));
  }
  if (shared != nullptr) acc = __fadd_rn(acc, shared[static_cast<size_t>(t) * D + d]);
  y[static_cast<size_t>(t) * D + d] = acc;
}


// ---------------------------------------------------------------------------------------------
// Combine WITHOUT the second collective (combine direction): the expert rank
// writes its un-weighted row outputs straight into the home ranks' `back` buffers over NVLink
// peer mappings, in the position each home rank's plan expects them, and bumps a counter in the
// home rank's memory; the home rank's combine kernel waits on its counters instead of on an
// all-to-all.  Counters are cumulative (never reset): the plan keeps the running totals.
//
// Safe with one buffer per rank: a rank pushes step n+1 only after it has received the home
// rank's step n+1 dispatch rows, which that rank's stream issues after its step n combine.
// ---------------------------------------------------------------------------------------------

// expected cumulative rows per expert rank at this home rank: expect[r] += cnt[rank][r]
__global__ void ep_expect_kernel(const int32_t* __restrict__ cnt, int W, int rank,
                                 unsigned long long* __restrict__ expect) {
  const int r = threadIdx.x;
  if (r < W) expect[r] += static_cast<unsigned long long>(cnt[rank * W + r]);
}

// one warp per received row: rows [roff(s), roff(s) + cnt[s][rank]) came from home rank s and go to
// position base_s + k of its back buffer, base_s = sum_{d < rank} cnt[s][d]
__global__ void __launch_bounds__(256) ep_push_back_kernel(const float* __restrict__ out, int M, int D,
                                                           const int32_t* __restrict__ cnt, int W,
                                                           int rank, float* const* __restrict__ peer_back,
                                                           unsigned long long* const* __restrict__ peer_flag,
                                                           unsigned* __restrict__ done_ctr) {
  __shared__ int s_roff[kMaxWorld + 1], s_base[kMaxWorld];
  if (threadIdx.x == 0) {
    int o = 0;
    for (int s = 0; s < W; ++s) {
      s_roff[s] = o;
      o += cnt[s * W + rank];
      int b = 0;
      for (int d = 0; d < rank; ++d) b += cnt[s * W + d];
      s_base[s] = b;
    }
    s_roff[W] = o;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r < M) {
    int s = 0;
    while (s + 1 < W && r >= s_roff[s + 1]) ++s;
    const float4* src = reinterpret_cast<const float4*>(out + static_cast<size_t>(r) * D);
    float* dst_row = peer_back[s] + static_cast<size_t>(s_base[s] + r - s_roff[s]) * D;
    if ((D & 3) == 0 && (reinterpret_cast<uintptr_t>(dst_row) & 15) == 0) {
      float4* dst = reinterpret_cast<float4*>(dst_row);
      for (int d = lane; d < D / 4; d += 32) dst[d] = src[d];
    } else {
      for (int d = lane; d < D; d += 32) dst_row[d] = out[static_cast<size_t>(r) * D + d];
    }
  }
  // the last CTA through publishes: every row of this launch is in place before any counter moves
  __threadfence_system();
  __syncthreads();
  __shared__ bool s_last;
  if (threadIdx.x == 0) s_last = atomicAdd(done_ctr, 1u) == gridDim.x - 1;
  __syncthreads();
  if (s_last) {
    if (threadIdx.x == 0) *done_ctr = 0u;
    __threadfence_system();
    if (static_cast<int>(threadIdx.x) < W) {
      const int s = threadIdx.x;
      const unsigned long long n = static_cast<unsigned long long>(cnt[s * W + rank]);
      if (n) atomicAdd_system(peer_flag[s] + rank, n);
    }
  }
}

// the home rank: wait until every expert rank has delivered what the plan expects, then combine
__global__ void __launch_bounds__(256) ep_combine_symm_kernel(
    const float* __restrict__ back, const unsigned long long* __restrict__ flag,
    const unsigned long long* __restrict__ expect, int W, const int32_t* __restrict__ pos,
    const float* __restrict__ w, const float* __restrict__ shared, int B, int K, int D,
    float* __restrict__ y) {
  if (threadIdx.x < W) {
    const volatile unsigned long long* f = flag + threadIdx.x;
    const unsigned long long want = expect[threadIdx.x];
    while (*f < want) {
    }
  }
  __threadfence_system();
  __syncthreads();
  const int t = blockIdx.y;
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= B || d >= D) return;
  float acc = 0.0f;
  for (int s = 0; s < K; ++s) {
    const int p = pos[t * K + s];
    acc = __fadd_rn(acc, __fmul_rn(w[t * K + s], __ldcv(back + static_cast<size_t>(p) * D + d)));
  }
  if (shared != nullptr) acc = __fadd_rn(acc, shared[static_cast<size_t>(t) * D + d]);
  y[static_cast<size_t>(t) * D + d] = acc;
}
// ---------------------------------------------------------------------------------------------
// Dispatch WITHOUT the first collective (dispatch direction): the home rank
// packs a token row and writes it straight into the OWNER rank's receive buffer over the peer
// mapping, at the row the owner's own view of the plan gives it -- rows of source rank s start at
// sum_{s' < s} cnt[s'][owner], in s's send order -- and bumps a cumulative counter in the owner's
// memory; the owner's unpack kernel waits on its counters instead of on an all-to-all.
//
// Safe with one receive buffer per rank: a peer pushes step n+1 only after the all-gather of the
// step n+1 ids, a collective this rank's stream joins after its own step n unpack.
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) ep_push_rows_kernel(
    const float* __restrict__ x, const int32_t* __restrict__ pos, const int32_t* __restrict__ loc,
    int slots, int K, int D, int stride, const int32_t* __restrict__ cnt, int W, int rank,
    uint8_t* const* __restrict__ peer_recv, unsigned long long* const* __restrict__ peer_flag,
    unsigned* __restrict__ done_ctr) {
  __shared__ int s_soff[kMaxWorld + 1], s_rbase[kMaxWorld];
  if (threadIdx.x == 0) {
    int o = 0;
    for (int d = 0; d < W; ++d) {
      s_soff[d] = o;  // this rank's send order: destination-major
      o += cnt[rank * W + d];
      int b = 0;
      for (int sr = 0; sr < rank; ++sr) b += cnt[sr * W + d];
      s_rbase[d] = b;  // where this rank's rows start in destination d's receive buffer
    }
    s_soff[W] = o;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i < slots) {
    const int p = pos[i];
    if (p >= 0) {
      int d = 0;
      while (d + 1 < W && p >= s_soff[d + 1]) ++d;
      const float* src = x + static_cast<size_t>(i / K) * D;
      uint8_t* row = peer_recv[d] + static_cast<size_t>(s_rbase[d] + p - s_soff[d]) * stride;
      __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(row);
      for (int c = lane; c < D; c += 32) dst[c] = __float2bfloat16_rn(__ldg(src + c));
      if (lane == 0) *reinterpret_cast<int32_t*>(row + static_cast<size_t>(D) * 2) = loc[i];
    }
  }
  // the last CTA through publishes: every row of this launch is in place before any counter moves
  __threadfence_system();
  __syncthreads();
  __shared__ bool s_last;
  if (threadIdx.x == 0) s_last = atomicAdd(done_ctr, 1u) == gridDim.x - 1;
  __syncthreads();
  if (s_last) {
    if (threadIdx.x == 0) *done_ctr = 0u;
    __threadfence_system();
    if (static_cast<int>(threadIdx.x) < W) {
      const int d = threadIdx.x;
      const unsigned long long n = static_cast<unsigned long long>(cnt[rank * W + d]);
      if (n) atomicAdd_system(peer_flag[d] + rank, n);
    }
  }
}

// where received row r's OUTPUT goes: its home rank's back buffer, the row that rank's plan
// expects (the arithmetic of ep_push_back_kernel, as pointers for the expert layer's last kernel)
__global__ void __launch_bounds__(256) ep_back_ptrs_kernel(const int32_t* __restrict__ cnt, int W,
                                                           int rank, int M, int D,
                                                           float* const* __restrict__ peer_back,
                                                           float** __restrict__ ptrs) {
  __shared__ int s_roff[kMaxWorld + 1], s_base[kMaxWorld];
  if (threadIdx.x == 0) {
    int o = 0;
    for (int s = 0; s < W; ++s) {
      s_roff[s] = o;
      o += cnt[s * W + rank];
      int b = 0;
      for (int d = 0; d < rank; ++d) b += cnt[s * W + d];
      s_base[s] = b;
    }
    s_roff[W] = o;
  }
  __syncthreads();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= M) return;
  int s = 0;
  while (s + 1 < W && r >= s_roff[s + 1]) ++s;
  ptrs[r] = peer_back[s] + static_cast<size_t>(s_base[s] + r - s_roff[s]) * D;
}

// after the expert layer (stream order: its stores are complete): system fence, then the home
// ranks' counters
__global__ void ep_signal_back_kernel(const int32_t* __restrict__ cnt, int W, int rank,
                                      unsigned long long* const* __restrict__ peer_flag) {
  __threadfence_system();
  const int s = threadIdx.x;
  if (s < W) {
    const unsigned long long n = static_cast<unsigned long long>(cnt[s * W + rank]);
    if (n) atomicAdd_system(peer_flag[s] + rank, n);
  }
}

// expected cumulative rows per SOURCE rank at this owner rank: expect[s] += cnt[s][rank]
__global__ void ep_expect_in_kernel(const int32_t* __restrict__ cnt, int W, int rank,
                                    unsigned long long* __restrict__ expect) {
  const int s = threadIdx.x;
  if (s < W) expect[s] += static_cast<unsigned long long>(cnt[s * W + rank]);
}

// the owner rank: wait until every source rank has delivered what the plan expects, then unpack
__global__ void __launch_bounds__(256) ep_unpack_symm_kernel(
    const uint8_t* __restrict__ recv, const unsigned long long* __restrict__ flag,
    const unsigned long long* __restrict__ expect, int W, int rows, int D, int stride,
    float* __restrict__ x, int32_t* __restrict__ ids) {
  if (threadIdx.x < W) {
    const volatile unsigned long long* f = flag + threadIdx.x;
    const unsigned long long want = expect[threadIdx.x];
    while (*f < want) {
    }
  }
  __threadfence_system();
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const uint8_t* row = recv + static_cast<size_t>(r) * stride;
  const unsigned short* src = reinterpret_cast<const unsigned short*>(row);
  float* dst = x + static_cast<size_t>(r) * D;
  for (int d = lane; d < D; d += 32) dst[d] = __bfloat162float(__ushort_as_bfloat16(__ldcv(src + d)));
  if (lane == 0) ids[r] = __ldcv(reinterpret_cast<const int32_t*>(row + static_cast<size_t>(D) * 2));
}
}  // namespace
}  // namespace skb

using namespace skb;

extern "C" {

int skb_ep_row_stride(int d_model) { return round_up(d_model * 2 + 4, 16); }

int skb_ep_plan(const int32_t* ids_all, int world, int slots_per_rank, const int32_t* expert_lo,
                int rank, int32_t* counts, int32_t* pos, int32_t* local_ids, void* stream) {
  if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world || slots_per_rank < 0) return SKB_ECONFIG;
  if (slots_per_rank == 0) return SKB_OK;
  ep_plan_kernel<<<1, kPlanThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      ids_all, world, slots_per_rank, expert_lo, rank, counts, pos, local_ids);
  return cudaGetLastError() == cudaSuccess ? SKB_OK : SKB_ECUDA;
}

int skb_ep_pack(const float* x, const int32_t* pos, const int32_t* local_ids, int slots, int top_k,
                int d_model, uint8_t* send, void* stream) {
  if (slots <= 0) return SKB_OK;
  ep_pack_kernel<<<ceil_div(slots, 8), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      x, pos, local_ids, slots, top_k, d_model, skb_ep_row_stride(d_model), send);
  return cudaGetLastError() == cudaSuccess ? SKB_OK : SKB_ECUDA;
}

int skb_ep_unpack(const uint8_t* recv, int rows, int d_model, float* x, int32_t* ids, void* stream) {
  if (rows <= 0) return SKB_OK;
  ep_unpack_kernel<<<ceil_div(rows, 8), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      recv, rows, d_model, skb_ep_row_stride(d_model), x, ids);
  return cudaGetLastError() == cudaSuccess ? SKB_OK : SKB_ECUDA;
}

int skb_ep_combine(const float* back, const int32_t* pos, const float* weights, const float* shared,
                   int batch, int top_k, int d_model, float* y, void* stream) {
  if (batch <= 0) return SKB_OK;
  ep_combine_kernel<<<dim3(ceil_div(d_model, 256), batch), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      back, pos, weights, shared, batch, top_k, d_model, y);
  return cudaGetLastError() == cudaSuccess ? SKB_OK : SKB_ECUDA;
}

/* ---- peer-memory combine (no second collective) ---- */
int skb_ep_symm_alloc(uint64_t bytes, void** ptr) {
  if (ptr == nullptr) return SKB_EINTERNAL;
  if (cudaMalloc(ptr, bytes ? bytes : 16) != cudaSuccess) return SKB_ECUDA;
  return cudaMemset(*ptr, 0, bytes ? bytes : 16) == cudaSuccess ? SKB_OK : SKB_ECUDA;
}
int skb_ep_symm_free(void* ptr) { return cudaFree(ptr) == cudaSuccess ? SKB_OK : SKB_ECUDA; }
int skb_ep_ipc_export(void* ptr, uint8_t* handle64) {
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, ptr) != cudaSuccess) return SKB_ECUDA;
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(handle64, &h, 64);
  return SKB_OK;
}
int skb_ep_ipc_import(const uint8_t* handle64, void** peer_ptr) {
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, 64);
  return cudaIpcOpenMemHandle(peer_ptr, h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess ? SKB_OK
                                                                                          : SKB_ECUDA;
}
int skb_ep_ipc_close(void* peer_ptr) {
  return cudaIpcCloseMemHandle(peer_ptr) == cudaSuccess ? SKB_OK : SKB_ECUDA;
}

int skb_ep_push_back(const float* out_rows, int rows, int d_model, const int32_t* counts, int world,
                     int rank, float* const* peer_back, unsigned long long* const* peer_flag,
                     unsigned long long* expect, uint32_t* done_ctr, void* stream) {
  if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world) return SKB_ECONFIG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ep_expect_kernel<<<1, 32, 0, s>>>(counts, world, rank, expect);
  const int grid = rows > 0 ? ceil_div(rows, 8) : 1;
  ep_push_back_kernel<<<grid, 256, 0, s>>>(out_rows, rows, d_model, counts, world, rank, peer_back,
                                           peer_flag, done_ctr);
  return cudaGetLastError() == cudaSuccess ? SKB_OK : SKB_ECUDA;
}

int skb_ep_push_rows(const float* x, const int32_t* pos, const int32_t* local_ids, int slots, int top_k,
                     int d_model, const int32_t* counts, int world, int rank, uint8_t* const* peer_recv,
                     unsigned long long* const* peer_flag, uint32_t* done_ctr, void* stream) {
  if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world || slots < 0) return SKB_ECONFIG;
  const int grid = slots > 0 ? ceil_div(slots, 8) : 1;
  ep_push_rows_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      x, pos, local_ids, slots, top_k, d_model, skb_ep_row_stride(d_model), counts, world, rank,
      peer_recv, peer_flag, done_ctr);
  return cudaGetLastError() == cudaSuccess ? SKB_OK : SKB_ECUDA;
}

int skb_ep_unpack_symm(const uint8_t* recv, const unsigned long long* flag, unsigned long long* expect,
                       const int32_t* counts, int world, int rank, int rows, int d_model, float* x,
                       int32_t* ids, void* stream) {
  if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world || rows < 0) return SKB_ECONFIG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ep_expect_in_kernel<<<1, 32, 0, s>>>(counts, world, rank, expect);
  const int grid = rows > 0 ? ceil_div(rows, 8) : 1;
  ep_unpack_symm_kernel<<<grid, 256, 0, s>>>(recv, flag, expect, world, rows, d_model,
                                             skb_ep_row_stride(d_model), x, ids);
  return cudaGetLastError() == cudaSuccess ? SKB_OK : SKB_ECUDA;
}

int skb_ep_back_ptrs(const int32_t* counts, int world, int rank, int rows, int d_model,
                     float* const* peer_back, float** ptrs, void* stream) {
  if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world || rows < 0) return SKB_ECONFIG;
  if (rows == 0) return SKB_OK;
  ep_back_ptrs_kernel<<<ceil_div(rows, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      counts, world, rank, rows, d_model, peer_back, ptrs);
  return cudaGetLastError() == cudaSuccess ? SKB_OK : SKB_ECUDA;
}

int skb_ep_signal_back(const int32_t* counts, int world, int rank,
                       unsigned long long* const* peer_flag, unsigned long long* expect, void* stream) {
  if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world) return SKB_ECONFIG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ep_expect_kernel<<<1, 32, 0, s>>>(counts, world, rank, expect);
  ep_signal_back_kernel<<<1, 32, 0, s>>>(counts, world, rank, peer_flag);
  return cudaGetLastError() == cudaSuccess ? SKB_OK : SKB_ECUDA;
}

int skb_ep_combine_symm(const float* back, const unsigned long long* flag,
                        const unsigned long long* expect, int world, const int32_t* pos,
                        const float* weights, const float* shared, int batch, int top_k, int d_model,
                        float* y, void* stream) {
  if (batch <= 0) return SKB_OK;
  if (world < 1 || world > kMaxWorld) return SKB_ECONFIG;
  ep_combine_symm_kernel<<<dim3(ceil_div(d_model, 256), batch), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      back, flag, expect, world, pos, weights, shared, batch, top_k, d_model, y);
  return cudaGetLastError() == cudaSuccess ? SKB_OK : SKB_ECUDA;
}

}  // extern "C"
