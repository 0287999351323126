// image.cu -- builds the device weight image.
//
//   router   fp32 [E][D]                         (kept in fp32: routing must match the reference)
//   gateup   bf16 [E*2*Np + 2*Sp][Dp]            per 64-neuron block, 128 rows interleaved as
//                                                gateup_row() describes; K-major for TMA/UMMA,
//                                                stored tiled (tiled_index(): 16 KB tiles)
//   down^T   bf16 [E][Dp128][Np] (+ [Dp128][Sp])  A operand of the dense down projection, tiled
//   down     bf16 [E][Np][Dp] (+ shared [Sp][Dp]) one contiguous Dp*2-byte row per neuron,
//                                                i.e. MoELayerWeights::down_t as stored by the
//                                                reference (proj/include/sparsekit/model.hpp:34-43)
//
// The synthetic generators evaluate generate_synthetic (proj/src/model.cpp:129-166) element by
// element with SplitMix64 jump-ahead (proj/include/sparsekit/rng.hpp:16-40): draw q of the
// stream has state seed + (q+1)*0x9E3779B97F4A7C15.
#include "skb_internal.cuh"

namespace skb {

namespace {

__device__ __forceinline__ float splitmix_symmetric(uint64_t seed, uint64_t q, float scale) {
  uint64_t z = seed + (q + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z = z ^ (z >> 31);
  const float u = __fmul_rn(static_cast<float>(z >> 40), 0x1.0p-24f);
  return __fmul_rn(__fsub_rn(__fmul_rn(2.0f, u), 1.0f), scale);
}

__global__ void pack_gateup_kernel(const float* __restrict__ gate, const float* __restrict__ up,
                                   int n_rows, int D, int Dp, __nv_bfloat16* __restrict__ dst) {
  const int n = blockIdx.x;
  const int which = blockIdx.y;
  const float* src = (which ? up : gate) + static_cast<size_t>(n) * D;
  const size_t img_row = static_cast<size_t>(n / kNeuronBlock) * 128 +
                         gateup_row(n % kNeuronBlock, which);
  for (int d = threadIdx.x; d < D; d += blockDim.x)
    dst[tiled_index(img_row, d, Dp)] = __float2bfloat16_rn(src[d]);
}

__global__ void pack_rows_kernel(const float* __restrict__ src, int D, int Dp,
                                 __nv_bfloat16* __restrict__ dst) {
  const int n = blockIdx.x;
  for (int d = threadIdx.x; d < D; d += blockDim.x)
    dst[static_cast<size_t>(n) * Dp + d] = __float2bfloat16_rn(src[static_cast<size_t>(n) * D + d]);
}

__global__ void synth_gateup_kernel(uint64_t seed, float scale, uint64_t off_gate, uint64_t off_up,
                                    int D, int Dp, __nv_bfloat16* __restrict__ dst) {
  const int n = blockIdx.x;
  const int which = blockIdx.y;
  const uint64_t off = (which ? off_up : off_gate) + static_cast<uint64_t>(n) * D;
  const size_t img_row = static_cast<size_t>(n / kNeuronBlock) * 128 +
                         gateup_row(n % kNeuronBlock, which);
  for (int d = threadIdx.x; d < D; d += blockDim.x)
    dst[tiled_index(img_row, d, Dp)] = __float2bfloat16_rn(splitmix_symmetric(seed, off + d, scale));
}

__global__ void synth_rows_kernel(uint64_t seed, float scale, uint64_t off, int D, int Dp,
                                  __nv_bfloat16* __restrict__ dst) {
  const int n = blockIdx.x;
  for (int d = threadIdx.x; d < D; d += blockDim.x)
    dst[static_cast<size_t>(n) * Dp + d] =
        __float2bfloat16_rn(splitmix_symmetric(seed, off + static_cast<uint64_t>(n) * D + d, scale));
}

// W_down^T image for the dense down projection: dst[d][n] = bf16(down_t[n][d]), [Dp128][Kp]
// (rows d >= D and columns n >= n_rows stay zero from the memset).
__global__ void pack_down_t_kernel(const float* __restrict__ src, int n_rows, int D, int Kp,
                                   __nv_bfloat16* __restrict__ dst) {
  __shared__ float tile[32][33];
  const int n0 = blockIdx.x * 32, d0 = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int n = n0 + j, d = d0 + threadIdx.x;
    tile[j][threadIdx.x] = (n < n_rows && d < D) ? src[static_cast<size_t>(n) * D + d] : 0.0f;
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int d = d0 + j, n = n0 + threadIdx.x;
    if (d < D && n < n_rows) dst[tiled_index(d, n, Kp)] = __float2bfloat16_rn(tile[threadIdx.x][j]);
  }
}

__global__ void synth_down_t_kernel(uint64_t seed, float scale, uint64_t off, int n_rows, int D,
                                    int Kp, __nv_bfloat16* __restrict__ dst) {
  const int d = blockIdx.x;
  for (int n = threadIdx.x; n < n_rows; n += blockDim.x)
    dst[tiled_index(d, n, Kp)] =
        __float2bfloat16_rn(splitmix_symmetric(seed, off + static_cast<uint64_t>(n) * D + d, scale));
}

__global__ void synth_f32_kernel(uint64_t seed, float scale, uint64_t off, uint64_t count,
                                 float* __restrict__ dst) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < count) dst[i] = splitmix_symmetric(seed, off + i, scale);
}

}  // namespace

int launch_pack_gateup(cudaStream_t s, const float* gate, const float* up, int n_rows, int D,
                       int Dp, __nv_bfloat16* dst_block_base) {
  pack_gateup_kernel<<<dim3(n_rows, 2), 256, 0, s>>>(gate, up, n_rows, D, Dp, dst_block_base);
  return 1;
}
int launch_pack_rows(cudaStream_t s, const float* src, int n_rows, int D, int Dp,
                     __nv_bfloat16* dst) {
  pack_rows_kernel<<<n_rows, 256, 0, s>>>(src, D, Dp, dst);
  return 1;
}
int launch_synth_gateup(cudaStream_t s, uint64_t seed, float scale, uint64_t off_gate,
                        uint64_t off_up, int n_rows, int /*n_rows_padded*/, int D, int Dp,
                        __nv_bfloat16* dst) {
  synth_gateup_kernel<<<dim3(n_rows, 2), 256, 0, s>>>(seed, scale, off_gate, off_up, D, Dp, dst);
  return 1;
}
int launch_synth_rows_bf16(cudaStream_t s, uint64_t seed, float scale, uint64_t off, int n_rows,
                           int /*n_rows_padded*/, int D, int Dp, __nv_bfloat16* dst) {
  synth_rows_kernel<<<n_rows, 256, 0, s>>>(seed, scale, off, D, Dp, dst);
  return 1;
}
int launch_pack_down_t(cudaStream_t s, const float* down_t, int n_rows, int D, int Kp,
                       __nv_bfloat16* dst) {
  pack_down_t_kernel<<<dim3(ceil_div(n_rows, 32), ceil_div(D, 32)), dim3(32, 8), 0, s>>>(
      down_t, n_rows, D, Kp, dst);
  return 1;
}
int launch_synth_down_t(cudaStream_t s, uint64_t seed, float scale, uint64_t off, int n_rows, int D,
                        int Kp, __nv_bfloat16* dst) {
  synth_down_t_kernel<<<D, 256, 0, s>>>(seed, scale, off, n_rows, D, Kp, dst);
  return 1;
}
__global__ void fill_f32_kernel(float* __restrict__ dst, float value, size_t count) {
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < count) dst[i] = value;
}
int launch_fill_f32(cudaStream_t s, float* dst, float value, size_t count) {
  if (count == 0) return 0;
  fill_f32_kernel<<<static_cast<unsigned>((count + 255) / 256), 256, 0, s>>>(dst, value, count);
  return 1;
}
int launch_synth_f32(cudaStream_t s, uint64_t seed, float scale, uint64_t off, uint64_t count,
                     float* dst) {
  synth_f32_kernel<<<static_cast<unsigned>((count + 255) / 256), 256, 0, s>>>(seed, scale, off,
                                                                             count, dst);
  return 1;
}

}  // namespace skb
