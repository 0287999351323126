// route_device.cuh -- route() for one token by one warp, shared by router.cu and decode.cu.
#pragma once

#include "skb_internal.cuh"

namespace skb {

// E <= 32 * VPL (VPL experts per lane, in registers): the same arithmetic as below with the
// latency taken out -- independent double exps interleaved, the two serial float sums fed by
// 128-bit shared-memory broadcasts, ranks by direct counting four probabilities per load.
// `sc` holds round_up(E, 4) + K floats.
template <int VPL>
__device__ __forceinline__ void warp_route_token_small(const float* __restrict__ row, int E, int K,
                                                       int renorm, float* sc, int32_t* out_ids,
                                                       float* out_w) {
  const int lane = threadIdx.x & 31;
  const int E4 = (E + 3) & ~3;
  float l[VPL], p[VPL];
  float mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int e = i * 32 + lane;
    l[i] = e < E ? __ldcg(row + e) : -INFINITY;
    mx = fmaxf(mx, l[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int e = i * 32 + lane;
    p[i] = e < E ? static_cast<float>(exp(static_cast<double>(__fsub_rn(l[i], mx)))) : 0.0f;
    if (e < E4) sc[e] = p[i];  // pad entries are zeros: x + 0 == x
  }
  __syncwarp();
  float denom = 0.0f;  // ascending float sum (router.cpp:41-46), computed by every lane
#pragma unroll 4
  for (int e = 0; e < E4; e += 4) {
    const float4 v = *reinterpret_cast<const float4*>(sc + e);
    denom = __fadd_rn(denom, v.x);
    denom = __fadd_rn(denom, v.y);
    denom = __fadd_rn(denom, v.z);
    denom = __fadd_rn(denom, v.w);
  }
  __syncwarp();
  int rank[VPL];
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int e = i * 32 + lane;
    p[i] = e < E ? __fdiv_rn(p[i], denom) : -1.0f;
    if (e < E4) sc[e] = e < E ? p[i] : -1.0f;
    rank[i] = 0;
  }
  __syncwarp();
  // rank under the reference's total order: probability descending, expert id ascending
#pragma unroll 2
  for (int e = 0; e < E4; e += 4) {
    const float4 v = *reinterpret_cast<const float4*>(sc + e);
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int me = i * 32 + lane;
      rank[i] += (v.x > p[i] || (v.x == p[i] && e + 0 < me)) ? 1 : 0;
      rank[i] += (v.y > p[i] || (v.y == p[i] && e + 1 < me)) ? 1 : 0;
      rank[i] += (v.z > p[i] || (v.z == p[i] && e + 2 < me)) ? 1 : 0;
      rank[i] += (v.w > p[i] || (v.w == p[i] && e + 3 < me)) ? 1 : 0;
    }
  }
  float* sel = sc + E4;  // the K selected probabilities in slot order
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int me = i * 32 + lane;
    if (me < E && rank[i] < K) {
      out_ids[rank[i]] = me;
      sel[rank[i]] = p[i];
    }
  }
  __syncwarp();
  float selected_sum = 0.0f;  // router.cpp:56-60, slot order
  for (int s = 0; s < K; ++s) selected_sum = __fadd_rn(selected_sum, sel[s]);
  for (int s = lane; s < K; s += 32) out_w[s] = renorm ? __fdiv_rn(sel[s], selected_sum) : sel[s];
  __syncwarp();
}

// route() for one token by one warp (proj/src/router.cpp:13-68): softmax with max
// subtraction, exp evaluated in double and rounded to float (what glibc's expf returns),
// ascending float sum for the denominator, IEEE division, then K rounds of warp arg-max under
// the reference's total order (probability descending, expert id ascending on ties).
// `sc` is round_up(E, 4) + K floats of shared scratch private to the warp.
__device__ inline void warp_route_token_any(const float* __restrict__ row, int E, int K, int renorm,
                                            float* sc, int32_t* out_ids, float* out_w);
__device__ inline void warp_route_token(const float* __restrict__ row, int E, int K, int renorm,
                                 float* sc, int32_t* out_ids, float* out_w) {
  if (E <= 32) return warp_route_token_small<1>(row, E, K, renorm, sc, out_ids, out_w);
  if (E <= 64) return warp_route_token_small<2>(row, E, K, renorm, sc, out_ids, out_w);
  if (E <= 128) return warp_route_token_small<4>(row, E, K, renorm, sc, out_ids, out_w);
  warp_route_token_any(row, E, K, renorm, sc, out_ids, out_w);
}
// One variant only (kernels that are instantiated per expert-count class keep their code short:
// code that runs once per CTA costs its instruction fetch).  V = 1, 2, 4: E <= 32 * V; 0: any E.
template <int V>
__device__ __forceinline__ void warp_route_token_v(const float* __restrict__ row, int E, int K,
                                                   int renorm, float* sc, int32_t* out_ids,
                                                   float* out_w) {
  if (V == 0) warp_route_token_any(row, E, K, renorm, sc, out_ids, out_w);
  else warp_route_token_small<(V == 0 ? 1 : V)>(row, E, K, renorm, sc, out_ids, out_w);
}
__device__ inline void warp_route_token_any(const float* __restrict__ row, int E, int K, int renorm,
                                            float* sc, int32_t* out_ids, float* out_w) {
  const int lane = threadIdx.x & 31;
  float mx = -INFINITY;
  for (int e = lane; e < E; e += 32) {
    const float l = __ldcg(row + e);
    sc[e] = l;
    mx = fmaxf(mx, l);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  for (int e = lane; e < E; e += 32)
    sc[e] = static_cast<float>(exp(static_cast<double>(__fsub_rn(sc[e], mx))));
  __syncwarp();
  float denom = 0.0f;
  if (lane == 0)
    for (int e = 0; e < E; ++e) denom = __fadd_rn(denom, sc[e]);
  denom = __shfl_sync(0xffffffffu, denom, 0);
  for (int e = lane; e < E; e += 32) sc[e] = __fdiv_rn(sc[e], denom);
  __syncwarp();
  float selected_sum = 0.0f;
  {
  for (int s = 0; s < K; ++s) {
    float bp = -3.0f;
    int be = 0x7fffffff;
    for (int e = lane; e < E; e += 32) {  // e ascending => lowest id kept on equal probability
      const float v = sc[e];
      if (v > bp) {
        bp = v;
        be = e;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float op = __shfl_xor_sync(0xffffffffu, bp, o);
      const int oe = __shfl_xor_sync(0xffffffffu, be, o);
      if (op > bp || (op == bp && oe < be)) {
        bp = op;
        be = oe;
      }
    }
    if (lane == 0) {
      sc[be] = -1.0f;  // selected: never wins again (probabilities are >= 0)
      out_ids[s] = be;
      out_w[s] = bp;
    }
    selected_sum = __fadd_rn(selected_sum, bp);
    __syncwarp();
  }
  }
  if (renorm)
    for (int s = lane; s < K; s += 32) out_w[s] = __fdiv_rn(out_w[s], selected_sum);
  __syncwarp();
}

}  // namespace skb
