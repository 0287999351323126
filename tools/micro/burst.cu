// micro-benchmark (round 2): what does ONE launch that must move ~67 MB out of cold HBM cost,
// by access method and CTA->address mapping, timed inside the kernel (%globaltimer, first CTA
// start -> last CTA end) and outside (events)?  Plus: null-launch cost (plain / cooperative),
// grid-barrier cost, scattered 4 KB row gathers with everything in flight.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o burst burst.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(c)); }
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint32_t bar) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@p bra D;\nbra W;\nD:\n}\n" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(dst), "l"(src), "r"(bytes), "r"(bar), "l"(pol) : "memory");
}
__device__ __forceinline__ void bulk_g2s_nohint(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap* m, int c0, int c1, uint32_t bar, uint64_t pol) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst), "l"((uint64_t)m), "r"(bar), "r"(c0), "r"(c1), "l"(pol) : "memory");
}
__device__ __forceinline__ long long gtime() { long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
constexpr uint64_t kEvictFirst = 0x12F0000000000000ull;

struct Stamp { long long t0, t1; };

__global__ void k_null(Stamp* st) { if (threadIdx.x == 0) { st[blockIdx.x].t0 = gtime(); st[blockIdx.x].t1 = gtime(); } }

// ---- LDG stream.  MAP 0: grid-interleaved (thread i of the whole grid reads 16-byte word i, i + stride ...);
// MAP 1: each CTA owns a contiguous slice. ----
template <int U, int MAP>
__global__ void __launch_bounds__(1024) k_ldg(const uint4* __restrict__ src, size_t n16, unsigned* sink, Stamp* st) {
  if (threadIdx.x == 0) st[blockIdx.x].t0 = gtime();
  unsigned acc = 0;
  size_t i, end, stride;
  if (MAP == 0) { i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; stride = (size_t)gridDim.x * blockDim.x; end = n16; }
  else { const size_t per = n16 / gridDim.x; i = (size_t)blockIdx.x * per + threadIdx.x; stride = blockDim.x; end = (size_t)(blockIdx.x + 1) * per; }
  for (; i + (U - 1) * stride < end; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(src + i + u * stride));
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) *sink = acc;
  __syncthreads();
  if (threadIdx.x == 0) st[blockIdx.x].t1 = gtime();
}

// ---- LDG GEMV-like: rows of 4 KB (2048 bf16); a warp owns row pairs, lane reads 16 B pieces, FMAs with x in
// registers (one token), warp-reduces per row.  Contiguous slice per CTA, rows dealt to warps round-robin. ----
template <int U, int THR>
__global__ void __launch_bounds__(THR) k_gemv(const uint4* __restrict__ src, size_t n_rows, const float* __restrict__ x, float* out, Stamp* st) {
  if (threadIdx.x == 0) st[blockIdx.x].t0 = gtime();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // x for this lane: pieces lane, lane + 32, ... (8 pieces of 8 values each for D = 2048)
  float xr[8][8];
#pragma unroll
  for (int p = 0; p < 8; ++p)
#pragma unroll
    for (int j = 0; j < 8; ++j) xr[p][j] = x[(p * 32 + lane) * 8 + j];
  const size_t per = n_rows / gridDim.x;
  const size_t r0 = (size_t)blockIdx.x * per;
  for (size_t r = r0 + warp * U; r + U <= r0 + per; r += (size_t)nw * U) {
    uint4 v[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int p = 0; p < 8; ++p)
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u][p].x), "=r"(v[u][p].y), "=r"(v[u][p].z), "=r"(v[u][p].w) : "l"(src + (r + u) * 256 + p * 32 + lane));
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float a = 0.f;
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const uint4 w = v[u][p];
        a = fmaf(__uint_as_float(w.x << 16), xr[p][0], a); a = fmaf(__uint_as_float(w.x & 0xffff0000u), xr[p][1], a);
        a = fmaf(__uint_as_float(w.y << 16), xr[p][2], a); a = fmaf(__uint_as_float(w.y & 0xffff0000u), xr[p][3], a);
        a = fmaf(__uint_as_float(w.z << 16), xr[p][4], a); a = fmaf(__uint_as_float(w.z & 0xffff0000u), xr[p][5], a);
        a = fmaf(__uint_as_float(w.w << 16), xr[p][6], a); a = fmaf(__uint_as_float(w.w & 0xffff0000u), xr[p][7], a);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      if (lane == 0) out[r + u] = a;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) st[blockIdx.x].t1 = gtime();
}

// ---- TMA / bulk ring: thread 0 produces, thread 32 consumes.  MAP 0: chunk c of the whole stream goes to CTA c % grid;
// MAP 1: contiguous slice per CTA. ----
template <int MODE, int MAP>
__global__ void __launch_bounds__(64) k_ring(const uint8_t* __restrict__ src, const __grid_constant__ CUtensorMap tm,
                                             size_t total, int chunk, int stages, size_t base_off, Stamp* st, uint64_t pol = kEvictFirst) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  const uint32_t bars = smem_u32(base + (size_t)stages * chunk);
  if (threadIdx.x == 0) {
    st[blockIdx.x].t0 = gtime();
    for (int s = 0; s < stages; ++s) { mbar_init(bars + 8 * s, 1); mbar_init(bars + 8 * (stages + s), 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t n_chunks = total / chunk;
  size_t c0, cstep, n;
  if (MAP == 0) { c0 = blockIdx.x; cstep = gridDim.x; n = (n_chunks - blockIdx.x + gridDim.x - 1) / gridDim.x; }
  else { const size_t per = n_chunks / gridDim.x; c0 = blockIdx.x * per; cstep = 1; n = per; }
  if (threadIdx.x == 0) {
    for (size_t i = 0; i < n; ++i) {
      const int s = (int)(i % stages);
      mbar_wait(bars + 8 * (stages + s), ((i / stages) & 1) ^ 1);
      mbar_expect(bars + 8 * s, chunk);
      const uint32_t dst = smem_u32(base + (size_t)s * chunk);
      const size_t off = (c0 + i * cstep) * chunk;
      if (MODE == 0) { if (pol) bulk_g2s(dst, src + off, chunk, bars + 8 * s, pol); else bulk_g2s_nohint(dst, src + off, chunk, bars + 8 * s); }
      else tma2d(dst, &tm, 0, (int)((base_off + off) / 128), bars + 8 * s, kEvictFirst);
    }
  } else if (threadIdx.x == 32) {
    for (size_t i = 0; i < n; ++i) {
      const int s = (int)(i % stages);
      mbar_wait(bars + 8 * s, (i / stages) & 1);
      mbar_arrive(bars + 8 * (stages + s));
    }
    st[blockIdx.x].t1 = gtime();
  }
}

__device__ __forceinline__ void tma3d(uint32_t dst, const CUtensorMap* m, int c0, int c1, int c2, uint32_t bar, uint64_t pol) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(dst), "l"((uint64_t)m), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "l"(pol) : "memory");
}
// ---- quarter pieces: the stream is a sequence of 16 KB tiles (128 rows x 64 bf16); piece p = rows [32q, 32q+32) of the
// 32 consecutive tiles of row block rb (p = rb * 4 + q): 128 KB in 4 KB segments at a 16 KB stride.  One TMA 3-D box
// {64, 32, KBOX} per stage.  Piece p goes to CTA p % grid (expert-major progressive order). ----
__global__ void __launch_bounds__(64) k_quarter(const __grid_constant__ CUtensorMap tm, int n_pieces, int kbox, int stages, int tile0, Stamp* st) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  const int chunk = kbox * 4096;
  const uint32_t bars = smem_u32(base + (size_t)stages * chunk);
  if (threadIdx.x == 0) {
    st[blockIdx.x].t0 = gtime();
    for (int s = 0; s < stages; ++s) { mbar_init(bars + 8 * s, 1); mbar_init(bars + 8 * (stages + s), 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int per_piece = 32 / kbox;
  if (threadIdx.x == 0) {
    int i = 0;
    for (int p = blockIdx.x; p < n_pieces; p += gridDim.x)
      for (int j = 0; j < per_piece; ++j, ++i) {
        const int s = i % stages;
        mbar_wait(bars + 8 * (stages + s), ((i / stages) & 1) ^ 1);
        mbar_expect(bars + 8 * s, chunk);
        tma3d(smem_u32(base + (size_t)s * chunk), &tm, 0, (p & 3) * 32, tile0 + (p >> 2) * 32 + j * kbox, bars + 8 * s, kEvictFirst);
      }
  } else if (threadIdx.x == 32) {
    int i = 0;
    for (int p = blockIdx.x; p < n_pieces; p += gridDim.x)
      for (int j = 0; j < per_piece; ++j, ++i) {
        const int s = i % stages;
        mbar_wait(bars + 8 * s, (i / stages) & 1);
        mbar_arrive(bars + 8 * (stages + s));
      }
    st[blockIdx.x].t1 = gtime();
  }
}

// ---- grid barriers: R rounds of (atomicAdd, spin) by thread 0, monotonic counter ----
__global__ void k_barrier(unsigned* ctr, int rounds, Stamp* st, long long* per_round) {
  if (threadIdx.x == 0) st[blockIdx.x].t0 = gtime();
  for (int r = 0; r < rounds; ++r) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(ctr, 1u);
      const unsigned target = (unsigned)(r + 1) * gridDim.x;
      unsigned v;
      do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory"); } while (v < target);
      if (blockIdx.x == 0) per_round[r] = gtime();
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) st[blockIdx.x].t1 = gtime();
}

// ---- gather: R rows of 4 KB per CTA, all in flight as direct loads, 256 threads ----
template <int R>
__global__ void __launch_bounds__(256) k_gather(const uint8_t* __restrict__ base, const int* __restrict__ rows, float* out, Stamp* st) {
  if (threadIdx.x == 0) st[blockIdx.x].t0 = gtime();
  const int* my = rows + blockIdx.x * R;
  uint4 v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const uint8_t* p = base + (size_t)my[r] * 4096 + threadIdx.x * 16;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[r].x), "=r"(v[r].y), "=r"(v[r].z), "=r"(v[r].w) : "l"(p));
  }
  unsigned acc = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) acc ^= v[r].x ^ v[r].y ^ v[r].z ^ v[r].w;
  if (acc == 0x1234567u) out[0] = 1.0f;
  __syncthreads();
  if (threadIdx.x == 0) st[blockIdx.x].t1 = gtime();
}


// ---- touch: one 16-byte word every `step` bytes of a region (TLB / DRAM page warm-up experiment) ----
__global__ void k_touch(const uint8_t* __restrict__ base, size_t bytes, size_t step, unsigned* sink) {
  unsigned acc = 0;
  for (size_t o = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * step; o < bytes; o += (size_t)gridDim.x * blockDim.x * step) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(base + o));
    acc ^= v.x;
  }
  if (acc == 0x12345678u) *sink = acc;
}


// ---- latency: one warp per CTA, `hops` dependent 16-byte loads at a 1 MB + 4 KB stride (cold lines, cold pages) ----
__global__ void k_chase(const uint8_t* __restrict__ base, size_t span, int hops, unsigned* sink, Stamp* st, long long* per) {
  if (threadIdx.x == 0) {
    st[blockIdx.x].t0 = gtime();
    size_t off = ((size_t)blockIdx.x * 7919 * 4096) % span;
    unsigned acc = 0;
    long long t_prev = gtime();
    for (int h = 0; h < hops; ++h) {
      uint4 v;
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(base + off));
      acc += v.x;
      off = (off + (1u << 20) + 4096 + (acc & 0)) % span;
      const long long t = gtime();
      if (blockIdx.x == 0 && h < 16) per[h] = t - t_prev;
      t_prev = t;
    }
    if (acc == 0x12345678u) *sink = acc;
    st[blockIdx.x].t1 = gtime();
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const size_t total = 6ull << 30;
  uint8_t* buf; CK(cudaMalloc(&buf, total)); CK(cudaMemset(buf, 1, total));
  uint8_t* flush; CK(cudaMalloc(&flush, 512ull << 20));
  unsigned* sink; CK(cudaMalloc(&sink, 64)); CK(cudaMemset(sink, 0, 64));
  Stamp* st; CK(cudaMalloc(&st, sizeof(Stamp) * 1024));
  float* xd; CK(cudaMalloc(&xd, 2048 * 4)); CK(cudaMemset(xd, 0, 2048 * 4));
  float* outd; CK(cudaMalloc(&outd, 4 << 20));
  long long* pr; CK(cudaMalloc(&pr, 8 * 64));
  int nsm = 0; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  void* fn = nullptr; cudaDriverEntryPointQueryResult qr;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr));
  CUtensorMap tm;
  {
    cuuint64_t dims[2] = {64, total / 128}; cuuint64_t strides[1] = {128}; cuuint32_t box[2] = {64, 128}; cuuint32_t es[2] = {1, 1};
    CUresult r = ((EncodeFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  }
  CK(cudaFuncSetAttribute(k_ring<0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  CK(cudaFuncSetAttribute(k_ring<0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  CK(cudaFuncSetAttribute(k_ring<1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  CK(cudaFuncSetAttribute(k_ring<1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  size_t cursor = 0;
  auto region = [&](size_t bytes) { if (cursor + bytes > total) cursor = 0; uint8_t* p = buf + cursor; cursor += (bytes + (2u << 20) - 1) / (2u << 20) * (2u << 20); return p; };
  std::vector<Stamp> hs(1024);
  auto finish = [&](const char* name, int grid, size_t bytes) {
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    CK(cudaMemcpy(hs.data(), st, sizeof(Stamp) * grid, cudaMemcpyDeviceToHost));
    long long a = hs[0].t0, b = hs[0].t1, amax = hs[0].t0;
    for (int i = 1; i < grid; ++i) { a = std::min(a, hs[i].t0); amax = std::max(amax, hs[i].t0); b = std::max(b, hs[i].t1); }
    const double in_us = (b - a) * 1e-3;
    printf("%-44s grid %4d %6.1f MB  event %7.2f us  in-kernel %7.2f us (start spread %5.2f)  %7.1f GB/s in-kernel  %7.1f GB/s event\n", name, grid, bytes / 1048576.0, ms * 1e3, in_us, (amax - a) * 1e-3,
           bytes / in_us / 1e3, bytes / (ms * 1e3) / 1e3);
  };
  auto pre = [&]() { CK(cudaMemsetAsync(flush, 0, 512ull << 20)); CK(cudaMemsetAsync(st, 0, sizeof(Stamp) * 1024)); };
  char name[160];



  if (getenv("BURST6")) {
    // cold-DRAM load latency seen by one thread, after an L2 flush by memset (dirty lines) and by a read sweep (clean)
    uint8_t* other; CK(cudaMalloc(&other, 512ull << 20)); CK(cudaMemset(other, 2, 512ull << 20));
    for (int rep = 0; rep < 3; ++rep)
      for (int mode = 0; mode < 2; ++mode)
        for (int grid : {1, 148}) {
          CK(cudaMemsetAsync(st, 0, sizeof(Stamp) * 1024));
          if (mode == 0) CK(cudaMemsetAsync(flush, 0, 512ull << 20));
          else k_ldg<16, 0><<<296, 512>>>((const uint4*)other, (512ull << 20) / 16, sink, st + 512);
          cudaEventRecord(e0); k_chase<<<grid, 32>>>(buf, (size_t)4 << 30, 8, sink, st, pr); cudaEventRecord(e1);
          CK(cudaEventSynchronize(e1));
          long long h[8]; CK(cudaMemcpy(h, pr, sizeof(h), cudaMemcpyDeviceToHost));
          printf("chase %s grid %3d: hops (ns)", mode == 0 ? "after memset    " : "after read sweep", grid);
          for (int i = 0; i < 8; ++i) printf(" %lld", h[i]);
          printf("\n");
        }
    return 0;
  }
  if (getenv("BURST5")) {
    // is the ~3 us ramp of a cold burst address translation?  Same 64 MB ring stream, preceded (in its own launch,
    // after the L2 flush) by a touch of one word per 2 MB / 64 KB / 4 KB of the region
    const size_t bytes = 64ull << 20; const int grid = 148, chunk = 16384, stages = 9; const size_t smem = (size_t)stages * chunk + 16 * stages + 1024;
    for (int rep = 0; rep < 3; ++rep) {
      for (size_t step : {(size_t)0, (size_t)2 << 20, (size_t)65536, (size_t)4096}) {
        uint8_t* p = region(bytes); pre();
        if (step) k_touch<<<148, 256>>>(p, bytes, step, sink);
        cudaEventRecord(e0); k_ring<0, 0><<<grid, 64, smem>>>(p, tm, bytes, chunk, stages, 0, st, kEvictFirst); cudaEventRecord(e1);
        snprintf(name, sizeof name, "ring 64 MB after touch step=%zu", step); finish(name, grid, bytes);
      }
      // the touch covers the whole 6 GB buffer at 2 MB steps (what a kernel could do before it knows its experts)
      { uint8_t* p = region(bytes); pre(); k_touch<<<148, 256>>>(buf, total, (size_t)2 << 20, sink);
        cudaEventRecord(e0); k_ring<0, 0><<<grid, 64, smem>>>(p, tm, bytes, chunk, stages, 0, st, kEvictFirst); cudaEventRecord(e1);
        finish("ring 64 MB after touch of 6 GB at 2 MB steps", grid, bytes); }
      // back-to-back null + stream launches: what a launch costs when it queues behind another kernel
      { uint8_t* p = region(4 * bytes); pre(); cudaEventRecord(e0);
        for (int j = 0; j < 4; ++j) k_ring<0, 0><<<grid, 64, smem>>>(p + j * bytes, tm, bytes, chunk, stages, 0, st, kEvictFirst);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("4 back-to-back ring launches of 64 MB: %.2f us per launch\n", ms * 1e3 / 4); }
      { pre(); cudaEventRecord(e0); for (int j = 0; j < 16; ++j) k_null<<<nsm, 256>>>(st); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("16 back-to-back null launches: %.2f us per launch\n", ms * 1e3 / 16); }
    }
    return 0;
  }
  if (getenv("BURST4")) {
    // does the state the L2 flush leaves behind matter?  dirty lines (memset) vs clean lines (read sweep of another region)
    uint8_t* other; CK(cudaMalloc(&other, 512ull << 20)); CK(cudaMemset(other, 2, 512ull << 20));
    const size_t bytes = 64ull << 20; const int grid = 148, chunk = 16384, stages = 9; const size_t smem = (size_t)stages * chunk + 16 * stages + 1024;
    for (int rep = 0; rep < 3; ++rep) {
      for (int mode = 0; mode < 3; ++mode) {
        uint8_t* p = region(bytes);
        CK(cudaMemsetAsync(st, 0, sizeof(Stamp) * 1024));
        if (mode == 0) CK(cudaMemsetAsync(flush, 0, 512ull << 20));
        if (mode == 1) { CK(cudaMemsetAsync(flush, 0, 512ull << 20)); k_ldg<16, 0><<<grid * 2, 512>>>((const uint4*)other, (512ull << 20) / 16, sink, st + 512); }
        if (mode == 2) { k_ldg<16, 0><<<grid * 2, 512>>>((const uint4*)other, (512ull << 20) / 16, sink, st + 512); }
        cudaEventRecord(e0); k_ring<0, 0><<<grid, 64, smem>>>(p, tm, bytes, chunk, stages, 0, st, kEvictFirst); cudaEventRecord(e1);
        finish(mode == 0 ? "ring 64 MB after memset (dirty L2)" : mode == 1 ? "ring 64 MB after memset + read sweep (clean L2)" : "ring 64 MB after read sweep only", grid, bytes);
      }
      for (int mode = 0; mode < 2; ++mode) {
        // back-to-back: 4 launches over distinct cold 64 MB regions, one event pair (launch overhead hidden)
        uint8_t* p = region(4 * bytes);
        if (mode == 0) CK(cudaMemsetAsync(flush, 0, 512ull << 20)); else k_ldg<16, 0><<<grid * 2, 512>>>((const uint4*)other, (512ull << 20) / 16, sink, st + 512);
        cudaEventRecord(e0);
        for (int j = 0; j < 4; ++j) k_ring<0, 0><<<grid, 64, smem>>>(p + j * bytes, tm, bytes, chunk, stages, 0, st, kEvictFirst);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("4 back-to-back ring launches of 64 MB after %s: %.2f us per launch\n", mode == 0 ? "memset" : "read sweep", ms * 1e3 / 4);
      }
    }
    return 0;
  }
  if (getenv("BURST3")) {
    CUtensorMap tm3;
    cuuint64_t dims[3] = {64, 128, total / 16384}; cuuint64_t strides[2] = {128, 16384}; cuuint32_t es[3] = {1, 1, 1};
    CK(cudaFuncSetAttribute(k_quarter, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    for (int rep = 0; rep < 2; ++rep)
      for (int kbox : {2, 4, 8}) {
        cuuint32_t box[3] = {64, 32, (cuuint32_t)kbox};
        CUresult r = ((EncodeFn)fn)(&tm3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode3 failed %d\n", (int)r); return 1; }
        for (int grid : {128, 148}) for (int kb_in_flight : {96, 144, 192}) {
          const int stages = kb_in_flight * 1024 / (kbox * 4096); const size_t smem = (size_t)stages * kbox * 4096 + 16 * stages + 1024;
          const size_t bytes = 512ull * 131072; uint8_t* p = region(bytes); pre(); cudaEventRecord(e0);
          k_quarter<<<grid, 64, smem>>>(tm3, 512, kbox, stages, (int)((p - buf) / 16384), st); cudaEventRecord(e1);
          snprintf(name, sizeof name, "tma3d quarter pieces kbox=%d stages=%d (%d KB)", kbox, stages, kb_in_flight); finish(name, grid, bytes);
        }
      }
    return 0;
  }
  if (getenv("BURST2")) {
    for (int rep = 0; rep < 2; ++rep) {
      for (size_t mb : {16, 32, 64, 128, 256, 512}) {
        const size_t bytes = mb << 20; const int grid = 148; const int chunk = 16384; const int stages = 9; const size_t smem = (size_t)stages * chunk + 16 * stages + 1024;
        { uint8_t* p = region(bytes); pre(); cudaEventRecord(e0); k_ring<0, 0><<<grid, 64, smem>>>(p, tm, bytes, chunk, stages, 0, st, kEvictFirst); cudaEventRecord(e1); finish("bulk1d 16K interleaved s=9 evict_first", grid, bytes); }
        { uint8_t* p = region(bytes); pre(); cudaEventRecord(e0); k_ring<0, 0><<<grid, 64, smem>>>(p, tm, bytes, chunk, stages, 0, st, 0); cudaEventRecord(e1); finish("bulk1d 16K interleaved s=9 no hint", grid, bytes); }
        { uint8_t* p = region(bytes); pre(); cudaEventRecord(e0); k_ring<0, 0><<<grid, 64, smem>>>(p, tm, bytes, chunk, stages, 0, st, 0x14F0000000000000ull); cudaEventRecord(e1); finish("bulk1d 16K interleaved s=9 evict_last", grid, bytes); }
        { uint8_t* p = region(bytes); pre(); cudaEventRecord(e0); k_ring<0, 1><<<grid, 64, smem>>>(p, tm, bytes, chunk, stages, 0, st, 0); cudaEventRecord(e1); finish("bulk1d 16K contiguous s=9 no hint", grid, bytes / chunk / grid * grid * chunk); }
        { uint8_t* p = region(bytes); pre(); cudaEventRecord(e0); k_ldg<16, 0><<<grid, 1024>>>((const uint4*)p, bytes / 16, sink, st); cudaEventRecord(e1); finish("ldg U=16 interleaved thr=1024", grid, bytes); }
        { uint8_t* p = region(bytes); pre(); cudaEventRecord(e0); k_ldg<16, 0><<<grid * 2, 512>>>((const uint4*)p, bytes / 16, sink, st); cudaEventRecord(e1); finish("ldg U=16 interleaved thr=512 x2", grid * 2, bytes); }
        { uint8_t* p = region(bytes); pre(); cudaEventRecord(e0); k_ldg<8, 0><<<grid, 512>>>((const uint4*)p, bytes / 16, sink, st); cudaEventRecord(e1); finish("ldg U=8 interleaved thr=512", grid, bytes); }
      }
      printf("\n");
    }
    return 0;
  }
  // 0. null launches
  for (int rep = 0; rep < 3; ++rep) {
    pre(); cudaEventRecord(e0); k_null<<<nsm, 256>>>(st); cudaEventRecord(e1); finish("null plain", nsm, 0);
    pre(); cudaEventRecord(e0);
    { void* args[] = {&st}; CK(cudaLaunchCooperativeKernel((void*)k_null, dim3(nsm), dim3(256), args, 0, 0)); }
    cudaEventRecord(e1); finish("null cooperative", nsm, 0);
  }
  {
    cudaStream_t s; cudaStreamCreate(&s); cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    { void* args[] = {&st}; CK(cudaLaunchCooperativeKernel((void*)k_null, dim3(nsm), dim3(256), args, 0, s)); }
    cudaStreamEndCapture(s, &g); CK(cudaGraphInstantiate(&ge, g, 0));
    for (int rep = 0; rep < 3; ++rep) {
      CK(cudaMemsetAsync(flush, 0, 512ull << 20, s));
      cudaEventRecord(e0, s); cudaGraphLaunch(ge, s); cudaEventRecord(e1, s); finish("null cooperative in graph", nsm, 0);
    }
  }
  // 1. grid barrier
  for (int rep = 0; rep < 2; ++rep) {
    pre(); CK(cudaMemset(sink, 0, 64));
    cudaEventRecord(e0);
    { int rounds = 16; unsigned* c = sink; void* args[] = {&c, &rounds, &st, &pr}; CK(cudaLaunchCooperativeKernel((void*)k_barrier, dim3(nsm), dim3(256), args, 0, 0)); }
    cudaEventRecord(e1); finish("16 grid barriers", nsm, 0);
    long long h[16]; CK(cudaMemcpy(h, pr, sizeof(h), cudaMemcpyDeviceToHost));
    printf("   per barrier (ns):"); for (int i = 1; i < 16; ++i) printf(" %lld", h[i] - h[i - 1]); printf("\n");
  }
  // 2. streams
  const size_t bytes = 128ull * 512 * 1024;  // 67.1 MB = OLMoE B=1 gate/up
  for (int rep = 0; rep < 2; ++rep) {
    for (int grid : {128, 148}) {
      for (int stages : {9, 13}) {
        const int chunk = 16384; const size_t smem = (size_t)stages * chunk + 16 * stages + 1024;
        { uint8_t* p = region(bytes); pre(); cudaEventRecord(e0); k_ring<1, 1><<<grid, 64, smem>>>(buf, tm, bytes, chunk, stages, (size_t)(p - buf), st); cudaEventRecord(e1);
          snprintf(name, sizeof name, "tma2d 16K contiguous-per-CTA stages=%d", stages); finish(name, grid, bytes / chunk / grid * grid * chunk); }
        { uint8_t* p = region(bytes); pre(); cudaEventRecord(e0); k_ring<1, 0><<<grid, 64, smem>>>(buf, tm, bytes, chunk, stages, (size_t)(p - buf), st); cudaEventRecord(e1);
          snprintf(name, sizeof name, "tma2d 16K interleaved stages=%d", stages); finish(name, grid, bytes); }
        { uint8_t* p = region(bytes); pre(); cudaEventRecord(e0); k_ring<0, 1><<<grid, 64, smem>>>(p, tm, bytes, chunk, stages, 0, st); cudaEventRecord(e1);
          snprintf(name, sizeof name, "bulk1d 16K contiguous-per-CTA stages=%d", stages); finish(name, grid, bytes / chunk / grid * grid * chunk); }
        { uint8_t* p = region(bytes); pre(); cudaEventRecord(e0); k_ring<0, 0><<<grid, 64, smem>>>(p, tm, bytes, chunk, stages, 0, st); cudaEventRecord(e1);
          snprintf(name, sizeof name, "bulk1d 16K interleaved stages=%d", stages); finish(name, grid, bytes); }
      }
      // two and four ring CTAs per SM
      for (int per_sm : {2, 4}) {
        const int chunk = 16384; const int stages = 12 / per_sm; const size_t smem = (size_t)stages * chunk + 16 * stages + 1024;
        uint8_t* p = region(bytes); pre(); cudaEventRecord(e0); k_ring<0, 0><<<grid * per_sm, 64, smem>>>(p, tm, bytes, chunk, stages, 0, st); cudaEventRecord(e1);
        snprintf(name, sizeof name, "bulk1d 16K interleaved %d CTA/SM stages=%d", per_sm, stages); finish(name, grid * per_sm, bytes);
      }
      for (int chunk : {4096, 8192, 32768}) {
        const int stages = 196608 / chunk > 24 ? 24 : 196608 / chunk; const size_t smem = (size_t)stages * chunk + 16 * stages + 1024;
        uint8_t* p = region(bytes); pre(); cudaEventRecord(e0); k_ring<0, 0><<<grid, 64, smem>>>(p, tm, bytes, chunk, stages, 0, st); cudaEventRecord(e1);
        snprintf(name, sizeof name, "bulk1d %dK interleaved stages=%d", chunk / 1024, stages); finish(name, grid, bytes);
      }
    }
    for (int grid : {148, 296, 592}) {
      for (int thr : {256, 512, 1024}) {
        if ((long)grid * thr > 148L * 2048) continue;
        { uint8_t* p = region(bytes); pre(); cudaEventRecord(e0); k_ldg<8, 0><<<grid, thr>>>((const uint4*)p, bytes / 16, sink, st); cudaEventRecord(e1);
          snprintf(name, sizeof name, "ldg U=8 interleaved thr=%d", thr); finish(name, grid, bytes); }
        { uint8_t* p = region(bytes); pre(); cudaEventRecord(e0); k_ldg<16, 0><<<grid, thr>>>((const uint4*)p, bytes / 16, sink, st); cudaEventRecord(e1);
          snprintf(name, sizeof name, "ldg U=16 interleaved thr=%d", thr); finish(name, grid, bytes); }
        { uint8_t* p = region(bytes); pre(); cudaEventRecord(e0); k_ldg<16, 1><<<grid, thr>>>((const uint4*)p, bytes / 16, sink, st); cudaEventRecord(e1);
          snprintf(name, sizeof name, "ldg U=16 contiguous-per-CTA thr=%d", thr); finish(name, grid, bytes); }
      }
    }
    { uint8_t* p = region(bytes); pre(); cudaEventRecord(e0); k_gemv<2, 512><<<nsm, 512>>>((const uint4*)p, bytes / 4096, xd, outd, st); cudaEventRecord(e1);
      finish("gemv U=2 rows (16 ld/lane) thr=512", nsm, bytes); }
    { uint8_t* p = region(bytes); pre(); cudaEventRecord(e0); k_gemv<2, 256><<<nsm, 256>>>((const uint4*)p, bytes / 4096, xd, outd, st); cudaEventRecord(e1);
      finish("gemv U=2 rows (16 ld/lane) thr=256", nsm, bytes); }
    { uint8_t* p = region(bytes); pre(); cudaEventRecord(e0); k_gemv<4, 256><<<nsm, 256>>>((const uint4*)p, bytes / 4096, xd, outd, st); cudaEventRecord(e1);
      finish("gemv U=4 rows (32 ld/lane) thr=256", nsm, bytes); }
    { uint8_t* p = region(bytes); pre(); cudaEventRecord(e0); k_gemv<2, 256><<<nsm * 2, 256>>>((const uint4*)p, bytes / 4096, xd, outd, st); cudaEventRecord(e1);
      finish("gemv U=2 rows thr=256 2 CTA/SM", nsm * 2, bytes); }
    { uint8_t* p = region(bytes); pre(); cudaEventRecord(e0); k_gemv<2, 512><<<nsm * 2, 512>>>((const uint4*)p, bytes / 4096, xd, outd, st); cudaEventRecord(e1);
      finish("gemv U=2 rows thr=512 2 CTA/SM", nsm * 2, bytes); }
    printf("\n");
  }
  // 3. gathers: 4096 rows of 4 KB (16.8 MB) scattered over 1 GB
  {
    int* drows; CK(cudaMalloc(&drows, 1024 * 64 * 4));
    for (int rep = 0; rep < 3; ++rep) {
      std::vector<int> rows(1024 * 64);
      uint64_t s = 88172645463325252ull + rep;
      const size_t base_row = (size_t)rep * (1ull << 30) / 4096;
      for (auto& r : rows) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; r = (int)(base_row + s % ((1ull << 30) / 4096)); }
      CK(cudaMemcpy(drows, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice));
      pre(); cudaEventRecord(e0); k_gather<28><<<nsm, 256>>>(buf, drows, outd, st); cudaEventRecord(e1); finish("gather 28 rows x 4 KB per CTA, all in flight", nsm, (size_t)nsm * 28 * 4096);
      pre(); cudaEventRecord(e0); k_gather<14><<<nsm * 2, 256>>>(buf, drows, outd, st); cudaEventRecord(e1); finish("gather 14 rows x 4 KB, 2 CTA/SM", nsm * 2, (size_t)nsm * 28 * 4096);
      pre(); cudaEventRecord(e0); k_gather<7><<<nsm * 4, 256>>>(buf, drows, outd, st); cudaEventRecord(e1); finish("gather 7 rows x 4 KB, 4 CTA/SM", nsm * 4, (size_t)nsm * 28 * 4096);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
