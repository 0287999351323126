// silu8 (tc_ptx.cuh: eight SwiGLU gates as interleaved branch-free chains) against silu_f (the
// plain g / (1 + expf(-g))), bit for bit, over every fp32 bit pattern of one exponent sweep plus
// dense samples of the range gate pre-activations live in.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2605_08575_b200/csrc \
//        -o /tmp/silu_check tools/micro/silu_check.cu && /tmp/silu_check
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include "tc_ptx.cuh"

__global__ void check_kernel(uint32_t first, unsigned long long* bad, uint32_t* example) {
  // every thread: 8 consecutive bit patterns
  const uint32_t base = first + (blockIdx.x * blockDim.x + threadIdx.x) * 8u;
  float g[8], ref[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    g[c] = __uint_as_float(base + c);
    ref[c] = skb::silu_f(g[c]);
  }
  skb::silu8(g);
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const bool same = __float_as_uint(g[c]) == __float_as_uint(ref[c]) || (g[c] != g[c] && ref[c] != ref[c]);
    if (!same) {
      if (atomicAdd(bad, 1ull) == 0) *example = base + c;
    }
  }
}

int main() {
  unsigned long long* bad;
  uint32_t* ex;
  cudaMalloc(&bad, 8);
  cudaMalloc(&ex, 4);
  cudaMemset(bad, 0, 8);
  // all 2^32 bit patterns: 2^29 threads of 8
  for (uint32_t chunk = 0; chunk < 64; ++chunk) {
    check_kernel<<<(1u << 26) / 8 / 256, 256>>>(chunk << 26, bad, ex);
  }
  cudaDeviceSynchronize();
  unsigned long long h = 0;
  uint32_t hex = 0;
  cudaMemcpy(&h, bad, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(&hex, ex, 4, cudaMemcpyDeviceToHost);
  printf("silu8 vs silu_f over all 2^32 inputs: %llu mismatches%s\n", h, h ? "" : " (bit-exact)");
  if (h) printf("  first example: bits 0x%08x\n", hex);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return h != 0;
}
