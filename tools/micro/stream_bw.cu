// micro-benchmark: how fast can one launch stream N MB out of HBM on sm_100a, per method?
//   ldg     : LDG.128, U loads in flight per thread
//   bulk    : 1-D cp.async.bulk of CHUNK bytes into an S-stage shared-memory ring (one CTA per SM)
//   tma2d   : 2-D tensor-map box 128 rows x 64 bf16 (swizzle 128B), same ring
// Every repetition reads a fresh region of a 4 GB buffer (cold L2).  Prints GB/s.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
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
__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap* m, int c0, int c1, uint32_t bar, uint64_t pol) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst), "l"((uint64_t)m), "r"(bar), "r"(c0), "r"(c1), "l"(pol) : "memory");
}
constexpr uint64_t kEvictFirst = 0x12F0000000000000ull;

// ---- LDG ----
template <int U>
__global__ void __launch_bounds__(1024) k_ldg(const uint4* __restrict__ src, size_t n16, unsigned* sink) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  unsigned acc = 0;
  for (; i + (U - 1) * stride < n16; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(src + i + u * stride));
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) *sink = acc;
}

// ---- ring of bulk copies: warp 0 lane 0 produces, warp 1 lane 0 "consumes" ----
// each CTA streams a contiguous slice [bid * per_cta, +per_cta) in CHUNK-byte pieces
template <int MODE>  // 0: 1-D bulk, 1: 2-D tensor map (chunk = 16 KB box)
__global__ void __launch_bounds__(64) k_ring(const uint8_t* __restrict__ src, const __grid_constant__ CUtensorMap tm,
                                             size_t per_cta, int chunk, int stages, int split, size_t base_off) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  const uint32_t bars = smem_u32(base + (size_t)stages * chunk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(bars + 8 * s, 1); mbar_init(bars + 8 * (stages + s), 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int n = (int)(per_cta / chunk);
  const uint8_t* my = src + (size_t)blockIdx.x * per_cta;
  if (threadIdx.x == 0) {
    for (int i = 0; i < n; ++i) {
      const int s = i % stages;
      mbar_wait(bars + 8 * (stages + s), ((i / stages) & 1) ^ 1);
      mbar_expect(bars + 8 * s, chunk);
      const uint32_t dst = smem_u32(base + (size_t)s * chunk);
      if (MODE == 0) {
        const int piece = chunk / split;
        for (int p = 0; p < split; ++p) bulk_g2s(dst + p * piece, my + (size_t)i * chunk + p * piece, piece, bars + 8 * s, kEvictFirst);
      } else {
        // tensor map over the whole buffer viewed as [rows][64 bf16]; one box = 128 rows = 16 KB
        const size_t row = (base_off + (size_t)blockIdx.x * per_cta + (size_t)i * chunk) / 128;
        tma2d(dst, &tm, 0, (int)row, bars + 8 * s, kEvictFirst);
      }
    }
  } else if (threadIdx.x == 32) {
    for (int i = 0; i < n; ++i) {
      const int s = i % stages;
      mbar_wait(bars + 8 * s, (i / stages) & 1);
      mbar_arrive(bars + 8 * (stages + s));
    }
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const size_t total = 4ull << 30;
  uint8_t* buf;
  CK(cudaMalloc(&buf, total));
  CK(cudaMemset(buf, 1, total));
  unsigned* sink;
  CK(cudaMalloc(&sink, 4));
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr));
  CUtensorMap tm;
  {
    cuuint64_t dims[2] = {64, total / 128};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t es[2] = {1, 1};
    CUresult r = ((EncodeFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  }
  CK(cudaFuncSetAttribute(k_ring<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  CK(cudaFuncSetAttribute(k_ring<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));

  size_t cursor = 0;
  auto region = [&](size_t bytes) { if (cursor + bytes > total) cursor = 0; uint8_t* p = buf + cursor; cursor += bytes; return p; };
  auto report = [&](const char* name, size_t bytes, float ms, int grid) { printf("%-40s grid %3d %4zu MB  %8.1f us  %7.1f GB/s  %6.1f GB/s/SM\n", name, grid, bytes >> 20, ms * 1e3, bytes / (ms * 1e-3) / 1e9, bytes / (ms * 1e-3) / 1e9 / grid); };
  // per-SM ceilings: few CTAs (one per SM) on a long stream
  for (int rep = 0; rep < 2; ++rep) {
    for (int grid : {16, 32, 64, 128, 148}) {
      const size_t bytes = (size_t)grid * (2ull << 20);  // 2 MB per CTA
      char name[128];
      for (int mode = 0; mode < 2; ++mode) {
        for (int stages : {8, 12}) {
          const int chunk = 16384;
          const size_t per_cta = bytes / grid / chunk * chunk;
          uint8_t* p = region(bytes);
          const size_t smem = (size_t)stages * chunk + 16 * stages + 1024;
          cudaEventRecord(e0);
          if (mode == 0) k_ring<0><<<grid, 64, smem>>>(p, tm, per_cta, chunk, stages, 4, 0);
          else k_ring<1><<<grid, 64, smem>>>(buf, tm, per_cta, chunk, stages, 1, (size_t)(p - buf));
          cudaEventRecord(e1);
          CK(cudaEventSynchronize(e1));
          float ms; cudaEventElapsedTime(&ms, e0, e1);
          snprintf(name, sizeof name, "%s 16KB stages=%d", mode ? "tma2d" : "bulk1d/4", stages);
          report(name, per_cta * grid, ms, grid);
        }
      }
      {
        uint8_t* p = region(bytes);
        cudaEventRecord(e0);
        k_ldg<16><<<grid, 1024>>>((const uint4*)p, bytes / 16, sink);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        report("ldg U=16 1024 thr", bytes, ms, grid);
      }
    }
    printf("\n");
  }
  {
    // L2-resident: the same 48 MB region over and over (after a warm pass it is all hits)
    const size_t bytes = 48ull << 20;
    const int chunk = 16384, stages = 8;
    for (int grid : {32, 64, 148}) {
      const size_t per_cta = bytes / grid / chunk * chunk;
      const size_t smem = (size_t)stages * chunk + 16 * stages + 1024;
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        k_ring<1><<<grid, 64, smem>>>(buf, tm, per_cta, chunk, stages, 1, 0);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep >= 2) report("tma2d L2-resident 48 MB", per_cta * grid, ms, grid);
      }
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        k_ldg<16><<<grid * 4, 1024>>>((const uint4*)buf, bytes / 16, sink);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep >= 2) report("ldg L2-resident 48 MB (4 CTAs/SM-slot)", bytes, ms, grid);
      }
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
