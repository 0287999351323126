// route_device.cuh -- route() for one token by one warp, shared by router.cu and decode.cu.
#pragma once

#include "skb_internal.cuh"

namespace skb {

// route() for one token by one warp (proj/src/router.cpp:13-68): softmax with max
// subtraction, exp evaluated in double and rounded to float (what glibc's expf returns),
// ascending float sum for the denominator, IEEE division, then K rounds of warp arg-max under
// the reference's total order (probability descending, expert id ascending on ties).
// `sc` is E floats of shared scratch private to the warp.
__device__ inline void warp_route_token(const float* __restrict__ row, int E, int K, int renorm,
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
  if (E <= 128) {
    // rank of every probability under the reference's total order (probability descending,
    // expert id ascending on ties) by direct counting: no serial arg-max rounds.  Each lane
    // owns experts lane, lane+32, ...; the E probabilities are read as shared-memory broadcasts.
    float mine[4];
    int rank[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      mine[j] = (j * 32 + lane < E) ? sc[j * 32 + lane] : -1.0f;
      rank[j] = 0;
    }
    for (int e = 0; e < E; ++e) {
      const float v = sc[e];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int me = j * 32 + lane;
        rank[j] += (v > mine[j] || (v == mine[j] && e < me)) ? 1 : 0;
      }
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int me = j * 32 + lane;
      if (me < E && rank[j] < K) {
        out_ids[rank[j]] = me;
        out_w[rank[j]] = mine[j];
        sc[E + rank[j]] = mine[j];  // scratch holds E + K floats
      }
    }
    __syncwarp();
    if (lane == 0)
      for (int s = 0; s < K; ++s) selected_sum = __fadd_rn(selected_sum, sc[E + s]);
    selected_sum = __shfl_sync(0xffffffffu, selected_sum, 0);
  } else {
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
