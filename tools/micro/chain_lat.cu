// micro-benchmark: dependent-issue latency of FADD / FFMA / FMUL->FADD chains on sm_100a
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(const float* __restrict__ in, float* out, long long* cyc, int n) {
  __shared__ float w[4096], x[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) { w[i] = in[i]; x[i] = in[4096 + i]; }
  __syncthreads();
  float acc = 0.f;
  long long t0 = clock64();
#pragma unroll 8
  for (int q = 0; q < n / 4; ++q) {
    float4 a = *reinterpret_cast<const float4*>(&w[(4 * q) & 4095]);
    float4 b = *reinterpret_cast<const float4*>(&x[(4 * q) & 4095]);
    if (MODE == 0) {  // fmul + fadd
      acc = __fadd_rn(acc, __fmul_rn(a.x, b.x)); acc = __fadd_rn(acc, __fmul_rn(a.y, b.y));
      acc = __fadd_rn(acc, __fmul_rn(a.z, b.z)); acc = __fadd_rn(acc, __fmul_rn(a.w, b.w));
    } else if (MODE == 1) {  // fmul + ffma(p,1,acc)
      acc = __fmaf_rn(__fmul_rn(a.x, b.x), 1.0f, acc); acc = __fmaf_rn(__fmul_rn(a.y, b.y), 1.0f, acc);
      acc = __fmaf_rn(__fmul_rn(a.z, b.z), 1.0f, acc); acc = __fmaf_rn(__fmul_rn(a.w, b.w), 1.0f, acc);
    } else if (MODE == 2) {  // fused fma (not order-faithful; for reference)
      acc = __fmaf_rn(a.x, b.x, acc); acc = __fmaf_rn(a.y, b.y, acc);
      acc = __fmaf_rn(a.z, b.z, acc); acc = __fmaf_rn(a.w, b.w, acc);
    } else {  // pure fadd chain on preloaded values
      acc = __fadd_rn(acc, a.x); acc = __fadd_rn(acc, a.y); acc = __fadd_rn(acc, b.x); acc = __fadd_rn(acc, b.y);
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { *out = acc; *cyc = t1 - t0; }
}
// software-pipelined: products of group q+1 are issued between the dependent adds of group q
__global__ void kpipe(const float* __restrict__ in, float* out, long long* cyc, int n) {
  __shared__ float w[4096], x[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) { w[i] = in[i]; x[i] = in[4096 + i]; }
  __syncthreads();
  float acc = 0.f;
  long long t0 = clock64();
  float4 a = *reinterpret_cast<const float4*>(&w[0]);
  float4 b = *reinterpret_cast<const float4*>(&x[0]);
  float p0 = __fmul_rn(a.x, b.x), p1 = __fmul_rn(a.y, b.y), p2 = __fmul_rn(a.z, b.z), p3 = __fmul_rn(a.w, b.w);
#pragma unroll 8
  for (int q = 1; q < n / 4; ++q) {
    a = *reinterpret_cast<const float4*>(&w[(4 * q) & 4095]);
    b = *reinterpret_cast<const float4*>(&x[(4 * q) & 4095]);
    acc = __fadd_rn(acc, p0); p0 = __fmul_rn(a.x, b.x);
    acc = __fadd_rn(acc, p1); p1 = __fmul_rn(a.y, b.y);
    acc = __fadd_rn(acc, p2); p2 = __fmul_rn(a.z, b.z);
    acc = __fadd_rn(acc, p3); p3 = __fmul_rn(a.w, b.w);
  }
  acc = __fadd_rn(acc, p0); acc = __fadd_rn(acc, p1); acc = __fadd_rn(acc, p2); acc = __fadd_rn(acc, p3);
  long long t1 = clock64();
  if (threadIdx.x == 0) { *out = acc; *cyc = t1 - t0; }
}
// explicit order in PTX: mul for element i+4 placed between the dependent adds
__global__ void kasm(const float* __restrict__ in, float* out, long long* cyc, int n) {
  __shared__ float w[4096], x[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) { w[i] = in[i]; x[i] = in[4096 + i]; }
  __syncthreads();
  float acc = 0.f;
  long long t0 = clock64();
  float4 a = *reinterpret_cast<const float4*>(&w[0]);
  float4 b = *reinterpret_cast<const float4*>(&x[0]);
  float p0 = __fmul_rn(a.x, b.x), p1 = __fmul_rn(a.y, b.y), p2 = __fmul_rn(a.z, b.z), p3 = __fmul_rn(a.w, b.w);
#pragma unroll 4
  for (int q = 1; q < n / 4; ++q) {
    a = *reinterpret_cast<const float4*>(&w[(4 * q) & 4095]);
    b = *reinterpret_cast<const float4*>(&x[(4 * q) & 4095]);
    asm volatile(
        "add.rn.f32 %0, %0, %1;\n\t"
        "mul.rn.f32 %1, %5, %9;\n\t"
        "add.rn.f32 %0, %0, %2;\n\t"
        "mul.rn.f32 %2, %6, %10;\n\t"
        "add.rn.f32 %0, %0, %3;\n\t"
        "mul.rn.f32 %3, %7, %11;\n\t"
        "add.rn.f32 %0, %0, %4;\n\t"
        "mul.rn.f32 %4, %8, %12;\n\t"
        : "+f"(acc), "+f"(p0), "+f"(p1), "+f"(p2), "+f"(p3)
        : "f"(a.x), "f"(a.y), "f"(a.z), "f"(a.w), "f"(b.x), "f"(b.y), "f"(b.z), "f"(b.w));
  }
  acc = __fadd_rn(acc, p0); acc = __fadd_rn(acc, p1); acc = __fadd_rn(acc, p2); acc = __fadd_rn(acc, p3);
  long long t1 = clock64();
  if (threadIdx.x == 0) { *out = acc; *cyc = t1 - t0; }
}
// two independent chains per lane (two tokens or two experts per lane): hides the add latency
__global__ void k2chain(const float* __restrict__ in, float* out, long long* cyc, int n) {
  __shared__ float w[4096], x[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) { w[i] = in[i]; x[i] = in[4096 + i]; }
  __syncthreads();
  float acc = 0.f, acc2 = 0.f;
  long long t0 = clock64();
#pragma unroll 8
  for (int q = 0; q < n / 4; ++q) {
    float4 a = *reinterpret_cast<const float4*>(&w[(4 * q) & 4095]);
    float4 b = *reinterpret_cast<const float4*>(&x[(4 * q) & 4095]);
    acc = __fadd_rn(acc, __fmul_rn(a.x, b.x)); acc2 = __fadd_rn(acc2, __fmul_rn(a.x, b.y));
    acc = __fadd_rn(acc, __fmul_rn(a.y, b.y)); acc2 = __fadd_rn(acc2, __fmul_rn(a.y, b.z));
    acc = __fadd_rn(acc, __fmul_rn(a.z, b.z)); acc2 = __fadd_rn(acc2, __fmul_rn(a.z, b.w));
    acc = __fadd_rn(acc, __fmul_rn(a.w, b.w)); acc2 = __fadd_rn(acc2, __fmul_rn(a.w, b.x));
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { *out = acc + acc2; *cyc = t1 - t0; }
}
int main() {
  float *in, *out; long long* cyc;
  cudaMalloc(&in, 8192 * 4); cudaMalloc(&out, 4); cudaMalloc(&cyc, 8);
  float h[8192]; for (int i = 0; i < 8192; ++i) h[i] = 0.001f * (i % 97) - 0.04f;
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  const int n = 8192;
  for (int rep = 0; rep < 2; ++rep) {
    long long c;
    k<0><<<1, 32>>>(in, out, cyc, n); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost); printf("fmul+fadd   %.2f cyc/elem\n", (double)c / n);
    k<1><<<1, 32>>>(in, out, cyc, n); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost); printf("fmul+ffma1  %.2f cyc/elem\n", (double)c / n);
    k<2><<<1, 32>>>(in, out, cyc, n); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost); printf("ffma        %.2f cyc/elem\n", (double)c / n);
    k<3><<<1, 32>>>(in, out, cyc, n); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost); printf("fadd only   %.2f cyc/elem\n", (double)c / n);
    kasm<<<1, 32>>>(in, out, cyc, n); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost); printf("asm order   %.2f cyc/elem\n", (double)c / n);
    k2chain<<<1, 32>>>(in, out, cyc, n); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost); printf("2 chains    %.2f cyc/elem (per chain element)\n", (double)c / n);
    kpipe<<<1, 32>>>(in, out, cyc, n); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost); printf("pipelined   %.2f cyc/elem\n", (double)c / n);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
