// gateup.cu -- subsystem (2): the gate/up projection as a grouped bf16 GEMM on tcgen05 with
// TMEM accumulators, fed by TMA, SwiGLU fused into the epilogue.
//
// Replaces the per-slot matvec pair + swiglu_rows of the reference
// (proj/src/engine.cpp:147-149, proj/src/linalg.cpp:22-40, proj/src/activation.cpp:15-29).
//
// Shape of the contraction ("swap-AB"): for one expert e and one tile of TN token rows,
//     D[128, TN] = A[128, Dp] * B[TN, Dp]^T
//   A = 128 rows of the interleaved gate/up image of e (64 neurons: per TMEM lane quarter,
//       16 gate rows then 16 up rows), K-major, streamed once from HBM by TMA;
//   B = TN rows of the expert-sorted bf16 token matrix xs, K-major (L2 resident);
//   D = fp32 accumulator in TMEM: lane = image row, column = token.
// Neurons sit on the UMMA M axis so that a decode batch (1..256 tokens per expert) uses
// UMMA N = 16..256 without padding the weight stream; the kernel is HBM-bound at decode sizes
// and the design goal is bytes in flight per SM (8 stages x 18-24 KB), not tensor occupancy.
//
// Warp roles (192 threads): warp 0 TMA producer, warp 1 TMEM allocator + MMA issuer,
// warps 2-5 epilogue (TMEM lane quarter = warp_idx % 4).
//
// The same kernel, MODE 1, is the dense down projection used when a batch routes enough tokens
// to every expert that gathering rows per token would re-read W_down from L2 many times over:
//     D[128, TN] = A[128, Np] * B[TN, Np]^T
//   A = 128 output columns of the expert's W_down^T image ([Dp128][Np], K-major);
//   B = TN rows of the MASKED activations (dropped neurons are zeros) as bf16.  To keep the
//       fp32-accumulation parity mode (1e-5), h is split into bf16 terms b0 + b1 (+ b2): two
//       terms carry 16 mantissa bits (residual <= 2^-18 |h| per element, i.e. ~1e-6 of the
//       output after the sum), three are exact; the products accumulate into the same TMEM tile.
//       nsplit = 1 is the bf16 mode (1e-2).
//   D is stored un-weighted per row (slot); combine_rows_kernel applies the router weights.
#include "skb_internal.cuh"
#include "tc_ptx.cuh"

namespace skb {

namespace {

constexpr int kGateupThreads = 192;
constexpr int kATileBytes = 128 * kBlockK * 2;  // 16 KB: 128 rows x 128 B

constexpr int kMaxSplit = 3;
constexpr uint32_t kPartBoxBytes = 32 * kBlockK * 2;  // a 32-row box of the token operand (4 KB)
__host__ __device__ constexpr int b_tile_bytes(int tn) { return tn * kBlockK * 2; }
// MB = 128-row A blocks per CTA.  MB = 2 ("paired blocks"): two weight blocks of the same expert
// share every token tile a CTA fetches, so the bytes an SM ingests per unit of work drop by 25 %
// (gate/up) to 37 % (down, three h terms per tile).  Measured bound of these kernels is per-SM
// ingest (~45 GB/s per SM when all SMs pull, tools/micro/stream_bw.cu), not HBM.
__host__ __device__ constexpr int stage_bytes(int tn, int mode, int mb = 1) {
  return mb * kATileBytes + (mode == 0 ? 1 : kMaxSplit) * b_tile_bytes(tn);
}
__host__ __device__ constexpr int num_stages(int tn, int mode, int mb = 1) {
  // MODE 0, 128-token tiles: two stages of 48 KB so that two CTAs share an SM (prefill grids)
  if (mb == 2) return mode == 0 ? (tn <= 64 ? 5 : 2) : (tn <= 64 ? 3 : 2);
  // MODE 0: <= ~110 KB per CTA so that two CTAs share an SM (grids larger than the SM count then
  // run in one wave and one CTA's prologue/epilogue overlaps the other's stream); ~100 KB in
  // flight per CTA is still several times the latency-bandwidth product per SM.
  // MODE 1, small token tiles: many short tiles (8 K blocks at d_ffn 512), so two CTAs per SM --
  // one tile's ramp and epilogue under the other's stream -- beat one CTA with a deep ring
  return mode == 0 ? (tn <= 16 ? 4 : (tn <= 32 ? 5 : (tn <= 64 ? 4 : (tn <= 128 ? 3 : 2))))
                   : (tn <= 16 ? 2 : (tn <= 32 ? 3 : (tn <= 64 ? 5 : 3)));
}
__host__ __device__ constexpr int tmem_cols(int tn) { return tn < 32 ? 32 : tn; }
__host__ __device__ constexpr int gateup_smem_bytes(int tn, int mode, int mb = 1) {
  return num_stages(tn, mode, mb) * stage_bytes(tn, mode, mb) + 1024 /*alignment slack*/ +
         256 /*barriers*/;
}

}  // namespace

#ifdef SKB_DEBUG_TIMING
// per-CTA phase stamps of grouped_tc_kernel (tools/dbg_tc.py): [MODE][cta][8]
__device__ long long g_tc_dbg[2 * 1024 * 8];
#define TC_STAMP(thr, i)                                                                         \
  do {                                                                                           \
    const int cta_ = blockIdx.y * gridDim.x + blockIdx.x;                                        \
    if (threadIdx.x == (thr) && cta_ < 1024) {                                                   \
      long long* p_ = g_tc_dbg + (MODE * 1024 + cta_) * 8;                                       \
      if ((i) == 0) {                                                                            \
        long long t_;                                                                            \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                   \
        p_[0] = t_;                                                                              \
        p_[7] = clock64();                                                                       \
      } else {                                                                                   \
        p_[i] = clock64();                                                                       \
      }                                                                                          \
    }                                                                                            \
  } while (0)
extern "C" void skb_debug_tc(long long* out) { cudaMemcpyFromSymbol(out, g_tc_dbg, sizeof(g_tc_dbg)); }
extern "C" void skb_debug_tc_clear() {
  static long long z[2 * 1024 * 8];
  cudaMemcpyToSymbol(g_tc_dbg, z, sizeof(z));
}
#else
#define TC_STAMP(thr, i) do { } while (0)
#endif

struct TcArgs {
  const int32_t* tile_expert;
  const int32_t* tile_row0;
  const int32_t* tile_nrows;
  const int32_t* n_tiles;
  const int32_t* tile_colrow;  // token-indexed tiles (MODE 0, TN 16): [tile][16] h row or -1
  const void* a_base;         // the A image behind tmap_a (L2 prefetch), or nullptr
  const void* a_shared_base;  // ... behind tmap_a_shared
  float* out;       // MODE 0: h [rows][out_stride];  MODE 1: slot outputs [rows][out_stride]
  float* sg_out;    // MODE 0, optional: silu(gate) [rows][out_stride] (threshold selection)
  int out_stride;
  int n_experts;
  int mblocks_routed, mblocks_shared;  // 128-row A blocks per routed expert / of the shared expert
  int m_routed, m_shared;              // valid outputs: MODE 0 neurons (N, S); MODE 1 columns (D, D)
  int kblocks_routed, kblocks_shared;  // 64-element K blocks
  int rows_per_expert;                 // A-image rows per routed expert
  int nsplit;                          // MODE 1: B operands accumulated per K block (1 or 3)
  const int* tiles_flag;  // MODE 0: non-zero once the tile list is written (implies early_tiles)
  // MODE 1, optional: output row r (expert-sorted) goes to out_rows[out_perm[r]] instead of `out`
  // -- expert parallelism with one expert per row and weight 1: the slot output IS the layer's
  // output, stored straight into the home rank's peer-mapped buffer from the TMEM epilogue
  float* const* out_rows;
  const int32_t* out_perm;
  int early_tiles;  // the tile list was written at least two kernels upstream: readable -- and the
                    // weight stream startable -- before the programmatic-launch wait
};

// MODE 0 epilogue of 16 accumulator columns held by one warp: lanes 0-15 hold gate(n) for the
// columns, lanes 16-31 hold up(n).  One exchange per column pair -- gate lanes finish column c,
// up lanes finish column c + 1 -- then the eight SwiGLUs of a lane as interleaved straight-line
// chains (silu8), then the stores.
template <int TN>
__device__ __forceinline__ void swiglu_store16(const uint32_t (&v)[16], int lane, int c0, int nrows,
                                               int n, int m_valid, int row0, int tile,
                                               const TcArgs& a) {
  const bool is_gate_lane = lane < 16;
  float gv[8], uv[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const float mine0 = __uint_as_float(v[2 * c]);
    const float mine1 = __uint_as_float(v[2 * c + 1]);
    const float recv = __shfl_xor_sync(0xffffffffu, is_gate_lane ? mine1 : mine0, 16);
    gv[c] = is_gate_lane ? mine0 : recv;
    uv[c] = is_gate_lane ? recv : mine1;
  }
  silu8(gv);
  const int colb = c0 + (is_gate_lane ? 0 : 1);
  if (TN == 16 && a.tile_colrow != nullptr) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int col = colb + 2 * c;
      const int r = (col < nrows && n < m_valid) ? a.tile_colrow[tile * 16 + col] : -1;
      if (r >= 0) {
        a.out[static_cast<size_t>(r) * a.out_stride + n] = gv[c] * uv[c];
        if (a.sg_out != nullptr) a.sg_out[static_cast<size_t>(r) * a.out_stride + n] = gv[c];
      }
    }
  } else {
    float* orow = a.out + static_cast<size_t>(row0 + colb) * a.out_stride + n;
    float* srow = a.sg_out ? a.sg_out + static_cast<size_t>(row0 + colb) * a.out_stride + n : nullptr;
    const size_t step = 2 * static_cast<size_t>(a.out_stride);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (colb + 2 * c < nrows && n < m_valid) {
        orow[c * step] = gv[c] * uv[c];
        if (srow != nullptr) srow[c * step] = gv[c];
      }
    }
  }
}

template <int TN, int MODE, int MB>
__global__ void __launch_bounds__(kGateupThreads, (MB == 2) ? ((MODE == 0 && TN == 128) ? 2 : 1) : ((MODE == 1 && TN <= 16) ? 4 : ((MODE == 0 && TN <= 16) ? 3 : ((MODE == 0 || TN <= 32) ? 2 : 1))))
grouped_tc_kernel(const __grid_constant__ CUtensorMap tmap_a,
                  const __grid_constant__ CUtensorMap tmap_a_shared,
                  const __grid_constant__ CUtensorMap tmap_b0,
                  const __grid_constant__ CUtensorMap tmap_b1,
                  const __grid_constant__ CUtensorMap tmap_b2,
                  const __grid_constant__ CUtensorMap tmap_s0,
                  const __grid_constant__ CUtensorMap tmap_s1,
                  const __grid_constant__ CUtensorMap tmap_s2, const TcArgs a) {
  constexpr int kStages = num_stages(TN, MODE, MB);
  constexpr int kStageBytes = stage_bytes(TN, MODE, MB);
  constexpr int kBTile = b_tile_bytes(TN);
  constexpr int kAll = MB * kATileBytes;  // A tiles of one stage; the B tiles follow
  constexpr uint32_t kTmemCols = tmem_cols(TN) * MB;

  extern __shared__ uint8_t smem_raw[];
  const uint32_t smem_base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t bar_base = smem_base + kStages * kStageBytes;
  // barriers: full[kStages], empty[kStages], tmem_full; then the TMEM base address word
  auto full_bar = [&](int s) { return bar_base + 8u * s; };
  auto empty_bar = [&](int s) { return bar_base + 8u * (kStages + s); };
  const uint32_t tmem_full_bar = bar_base + 8u * (2 * kStages);
  const uint32_t tmem_ptr_addr = bar_base + 8u * (2 * kStages + 1);
  volatile uint32_t* tmem_ptr_generic = reinterpret_cast<volatile uint32_t*>(
      smem_raw + (tmem_ptr_addr - smem_u32(smem_raw)));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  TC_STAMP(0, 0);
  // ---- prologue: nothing here reads memory written by the previous kernel ----
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b0);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    mbar_init(tmem_full_bar, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_ptr_addr, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_ptr_generic;

  // Programmatic dependent launch: this kernel's CTAs start while the previous kernel (token
  // permute / selection) is still running and wait for it below.  The tile list is older than
  // that (dispatch, at least two kernels upstream, complete before the previous kernel released
  // its own wait), and the weights are constants: so the ring's first stages of the A operand are
  // requested -- and the rest of this CTA's weight blocks prefetched into the L2 -- BEFORE the
  // wait; only the token operand waits.  Hides the tile-list reads and the first HBM latency
  // (~2.5 us per GEMM) under the previous kernel's tail.
  // (When the kernel directly upstream writes the tile list -- route_dispatch_kernel -- it raises
  // a flag as soon as the list is out, before it copies the tokens: the CTAs here poll that flag
  // instead, and the early start survives.  router_fused_kernel lowers the flag again.)
  if (a.tiles_flag != nullptr) {
    if (threadIdx.x == 0) {
      int seen;
      do {
        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(seen) : "l"(a.tiles_flag) : "memory");
      } while (seen == 0);
    }
    __syncthreads();
  } else if (!a.early_tiles) {
    pdl_wait();
    pdl_launch_dependents();
  }
  TC_STAMP(0, 1);

  const int tile = blockIdx.y;
  bool active = tile < __ldcg(a.n_tiles);
  int e = 0, row0 = 0, nrows = 0;
  bool shared_expert = false;
  if (active) {
    e = __ldcg(a.tile_expert + tile);
    row0 = __ldcg(a.tile_row0 + tile);
    nrows = __ldcg(a.tile_nrows + tile);
    shared_expert = e >= a.n_experts;
    active = static_cast<int>(blockIdx.x) * MB < (shared_expert ? a.mblocks_shared : a.mblocks_routed);
  }
  const int num_k_blocks = shared_expert ? a.kblocks_shared : a.kblocks_routed;
  const int nsplit = (MODE == 0) ? 1 : a.nsplit;
  // A tile with fewer token rows than TN (the usual case: tiles are cut per expert) fetches only
  // the 32-row boxes that hold rows and multiplies only round_up(nrows, 16) columns.
  const int n32 = (nrows + 31) >> 5;
  const bool part = TN >= 64 && n32 * 32 < TN;
  const uint32_t b_bytes = part ? static_cast<uint32_t>(n32) * kPartBoxBytes : kBTile;
  const uint32_t idesc = make_idesc_bf16(128, part ? ((nrows + 15) & ~15) : TN);
  // first A-image row of this (expert, block).  MODE 0: the shared expert's rows follow the
  // routed experts in one image; MODE 1: the shared expert has its own tensor map (its K
  // extent differs).
  const bool own_map = (MODE == 1) && shared_expert;
  const CUtensorMap* map_a = own_map ? &tmap_a_shared : &tmap_a;
  const int a_row = (own_map ? 0 : (shared_expert ? a.n_experts : e) * a.rows_per_expert) +
                    static_cast<int>(blockIdx.x) * MB * 128;
  // A blocks this CTA really has (an odd block count leaves the last CTA with one)
  const int n_mb = min(MB, (shared_expert ? a.mblocks_shared : a.mblocks_routed) -
                               static_cast<int>(blockIdx.x) * MB);

  int preloaded = 0;  // stages whose A tiles are already in flight (producer thread only)
  if (a.early_tiles) {
    if (active && warp == 0 && lane == 0) {
      preloaded = min(kStages, num_k_blocks);
      // tiled image: tile (a_row / 128, kb) is 128 consecutive rows of the 64-column view
      for (int kb = 0; kb < preloaded; ++kb) {
        mbar_arrive_expect_tx(full_bar(kb), n_mb * kATileBytes + nsplit * b_bytes);
#pragma unroll
        for (int m = 0; m < MB; ++m)
          if (m < n_mb)
            tma_load_2d(smem_base + kb * kStageBytes + m * kATileBytes, map_a, 0,
                        (((a_row >> 7) + m) * num_k_blocks + kb) * 128, full_bar(kb),
                        kPolicyEvictFirst);
      }
      // the blocks' remaining K tiles: 16 KB each, contiguous per block in the tiled image
      const char* img = reinterpret_cast<const char*>(own_map ? a.a_shared_base : a.a_base);
      if (img != nullptr)
        for (int m = 0; m < n_mb; ++m)
          for (int kb = preloaded; kb < num_k_blocks; ++kb)
            l2_prefetch(img + (static_cast<size_t>((a_row >> 7) + m) * num_k_blocks + kb) * kATileBytes,
                        kATileBytes);
    }
    pdl_wait();
    pdl_launch_dependents();
  }

  if (active) {
    if (warp == 0) {
      if (lane == 0) {
        for (int kb = 0; kb < num_k_blocks; ++kb) {
          const int s = kb % kStages;
          const uint32_t ph = (kb / kStages) & 1u;
          const uint32_t a_smem = smem_base + s * kStageBytes;
          if (kb >= preloaded) {
            mbar_wait(empty_bar(s), ph ^ 1u);
            mbar_arrive_expect_tx(full_bar(s), n_mb * kATileBytes + nsplit * b_bytes);
#pragma unroll
            for (int m = 0; m < MB; ++m)
              if (m < n_mb)
                tma_load_2d(a_smem + m * kATileBytes, map_a, 0,
                            (((a_row >> 7) + m) * num_k_blocks + kb) * 128, full_bar(s),
                            kPolicyEvictFirst);
          }
          if (kb == num_k_blocks - 1) TC_STAMP(0, 2);
          if (part) {
            for (int j = 0; j < n32; ++j) {
              const uint32_t dst = a_smem + kAll + j * kPartBoxBytes;
              tma_load_2d(dst, &tmap_s0, kb * kBlockK, row0 + 32 * j, full_bar(s), kPolicyEvictLast);
              if (MODE == 1 && nsplit > 1)
                tma_load_2d(dst + kBTile, &tmap_s1, kb * kBlockK, row0 + 32 * j, full_bar(s),
                            kPolicyEvictLast);
              if (MODE == 1 && nsplit > 2)
                tma_load_2d(dst + 2 * kBTile, &tmap_s2, kb * kBlockK, row0 + 32 * j, full_bar(s),
                            kPolicyEvictLast);
            }
            continue;
          }
          tma_load_2d(a_smem + kAll, &tmap_b0, kb * kBlockK, row0, full_bar(s), kPolicyEvictLast);
          if (MODE == 1 && nsplit > 1)
            tma_load_2d(a_smem + kAll + kBTile, &tmap_b1, kb * kBlockK, row0, full_bar(s),
                        kPolicyEvictLast);
          if (MODE == 1 && nsplit > 2)
            tma_load_2d(a_smem + kAll + 2 * kBTile, &tmap_b2, kb * kBlockK, row0, full_bar(s),
                        kPolicyEvictLast);
        }
      }
    } else if (warp == 1) {
      if (lane == 0) {
        for (int kb = 0; kb < num_k_blocks; ++kb) {
          const int s = kb % kStages;
          const uint32_t ph = (kb / kStages) & 1u;
          mbar_wait(full_bar(s), ph);
          tc_fence_after();
          if (kb == 0) TC_STAMP(32, 3);
          if (kb == num_k_blocks - 1) TC_STAMP(32, 4);
          const uint32_t a_smem = smem_base + s * kStageBytes;
#pragma unroll
          for (int m = 0; m < MB; ++m) {
            if (m < n_mb) {
              const uint64_t a_desc = make_smem_desc_sw128(a_smem + m * kATileBytes);
#pragma unroll
              for (int sp = 0; sp < (MODE == 0 ? 1 : kMaxSplit); ++sp) {
                if (sp < nsplit) {
                  const uint64_t b_desc = make_smem_desc_sw128(a_smem + kAll + sp * kBTile);
#pragma unroll
                  for (int k = 0; k < kBlockK / 16; ++k) {
                    // +32 bytes per UMMA K step (16 bf16) inside the 128-byte swizzle row
                    umma_bf16(tmem_base + static_cast<uint32_t>(m * TN), a_desc + 2u * k,
                              b_desc + 2u * k, idesc, (kb | k | sp) != 0 ? 1u : 0u);
                  }
                }
              }
            }
          }
          umma_commit(empty_bar(s));
        }
        umma_commit(tmem_full_bar);
      }
    } else {
      // ---- epilogue: TMEM -> registers -> (SwiGLU) -> global ----
      const int q = warp & 3;  // TMEM lane quarter this warp may read
      const int m_valid = shared_expert ? a.m_shared : a.m_routed;
      mbar_wait(tmem_full_bar, 0);
      tc_fence_after();
      TC_STAMP(64, 5);
#pragma unroll 1
      for (int m = 0; m < n_mb; ++m) {
      const uint32_t tmem_blk = tmem_base + static_cast<uint32_t>(m * TN);
      if (MODE == 0) {
        const int n = (static_cast<int>(blockIdx.x) * MB + m) * kNeuronBlock + 16 * q + (lane & 15);
#pragma unroll 1
        for (int c0 = 0; c0 < TN; c0 += 16) {
          if (c0 >= nrows) break;
          uint32_t v[16];
          tmem_ld_32x32b_x16(tmem_blk + (static_cast<uint32_t>(32 * q) << 16) + c0, v);
          tmem_ld_wait();
          swiglu_store16<TN>(v, lane, c0, nrows, n, m_valid, row0, tile, a);
        }
      } else {
        const int d = (static_cast<int>(blockIdx.x) * MB + m) * 128 + 32 * q + lane;
        // 32 columns per TMEM round trip
#pragma unroll 1
        for (int c0 = 0; c0 < TN; c0 += 32) {
          if (c0 >= nrows) break;
          uint32_t v0[16], v1[16];
          const uint32_t taddr = tmem_blk + (static_cast<uint32_t>(32 * q) << 16) + c0;
          tmem_ld_32x32b_x16(taddr, v0);
          if (TN >= 32) tmem_ld_32x32b_x16(taddr + 16, v1);
          tmem_ld_wait();
          if (a.out_rows != nullptr) {
            // lane c fetches the destination of column c0 + c once; the stores get it by shuffle
            const int col = c0 + lane;
            const unsigned long long mine =
                (col < nrows && (TN >= 32 || lane < 16))
                    ? reinterpret_cast<unsigned long long>(a.out_rows[a.out_perm[row0 + col]])
                    : 0ull;
#pragma unroll
            for (int c = 0; c < 16; ++c) {
              float* dst = reinterpret_cast<float*>(__shfl_sync(0xffffffffu, mine, c));
              if (c0 + c < nrows && d < m_valid) dst[d] = __uint_as_float(v0[c]);
            }
            if (TN >= 32) {
#pragma unroll
              for (int c = 0; c < 16; ++c) {
                float* dst = reinterpret_cast<float*>(__shfl_sync(0xffffffffu, mine, 16 + c));
                if (c0 + 16 + c < nrows && d < m_valid) dst[d] = __uint_as_float(v1[c]);
              }
            }
            continue;
          }
          float* orow = a.out + static_cast<size_t>(row0 + c0) * a.out_stride + d;
#pragma unroll
          for (int c = 0; c < 16; ++c)
            if (c0 + c < nrows && d < m_valid)
              orow[static_cast<size_t>(c) * a.out_stride] = __uint_as_float(v0[c]);
          if (TN >= 32) {
#pragma unroll
            for (int c = 0; c < 16; ++c)
              if (c0 + 16 + c < nrows && d < m_valid)
                orow[static_cast<size_t>(16 + c) * a.out_stride] = __uint_as_float(v1[c]);
          }
        }
      }
      }  // A blocks
      tc_fence_before();
      TC_STAMP(64, 6);
    }
  }

  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
}

// ---------------------------------------------------------------------------------------------
// The same GEMM with CHUNKED accumulation, for the fp32-accumulation parity mode (1e-5) on long
// contractions.  The tensor core adds every 16-element step into the fp32 accumulator with
// truncation: measured on B200 the result drifts by ~3.7e-8 of its magnitude per step, always
// the same way, i.e. 1.2e-5 after the 320 steps of d_model = 5120 (tools/h_err_probe.py).  Here
// the MMAs of at most kChunkSteps steps accumulate from zero into one of two TMEM chunk buffers;
// the epilogue warps fold each finished chunk into a MASTER accumulator (a third TMEM region)
// with round-to-nearest adds -- tcgen05.ld chunk + master, add, tcgen05.st master, 16 columns at
// a time -- while the MMAs of the next chunk run into the other buffer.  The last chunk is added
// in registers on its way to the epilogue proper.  One A block per CTA, token tiles <= 128.
// ---------------------------------------------------------------------------------------------
namespace {
constexpr int kChunkSteps = 32;  // MMA steps (16 elements each) per chunk
__host__ __device__ constexpr int pow2_cols(int c) { return c <= 32 ? 32 : (c <= 64 ? 64 : (c <= 128 ? 128 : (c <= 256 ? 256 : 512))); }
__host__ __device__ constexpr int chunked_tmem_cols(int tn) { return pow2_cols(3 * tmem_cols(tn)); }
__host__ __device__ constexpr int chunked_ctas_per_sm(int tn) { return 512 / chunked_tmem_cols(tn) > 4 ? 4 : 512 / chunked_tmem_cols(tn); }
__host__ __device__ constexpr int chunked_stages(int tn, int mode) {
  // the shared memory of an SM split over the CTAs its TMEM allows
  const int budget = (220 * 1024) / chunked_ctas_per_sm(tn) - 2048;
  const int s = budget / stage_bytes(tn, mode, 1);
  return s > 8 ? 8 : (s < 2 ? 2 : s);
}
__host__ __device__ constexpr int chunked_smem_bytes(int tn, int mode) {
  return chunked_stages(tn, mode) * stage_bytes(tn, mode, 1) + 1024 + 256;
}
}  // namespace

template <int TN, int MODE>
__global__ void __launch_bounds__(kGateupThreads, chunked_ctas_per_sm(TN))
grouped_tc_chunked_kernel(const __grid_constant__ CUtensorMap tmap_a,
                          const __grid_constant__ CUtensorMap tmap_a_shared,
                          const __grid_constant__ CUtensorMap tmap_b0,
                          const __grid_constant__ CUtensorMap tmap_b1,
                          const __grid_constant__ CUtensorMap tmap_b2,
                          const __grid_constant__ CUtensorMap tmap_s0,
                          const __grid_constant__ CUtensorMap tmap_s1,
                          const __grid_constant__ CUtensorMap tmap_s2, const TcArgs a) {
  constexpr int kStages = chunked_stages(TN, MODE);
  constexpr int kStageBytes = stage_bytes(TN, MODE, 1);
  constexpr int kBTile = b_tile_bytes(TN);
  constexpr uint32_t kCols = tmem_cols(TN);            // columns of one accumulator
  constexpr uint32_t kTmemCols = chunked_tmem_cols(TN);  // master + two chunk buffers

  extern __shared__ uint8_t smem_raw[];
  const uint32_t smem_base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t bar_base = smem_base + kStages * kStageBytes;
  auto full_bar = [&](int s) { return bar_base + 8u * s; };
  auto empty_bar = [&](int s) { return bar_base + 8u * (kStages + s); };
  auto cfull_bar = [&](int b) { return bar_base + 8u * (2 * kStages + b); };
  auto cempty_bar = [&](int b) { return bar_base + 8u * (2 * kStages + 2 + b); };
  const uint32_t tmem_ptr_addr = bar_base + 8u * (2 * kStages + 4);
  volatile uint32_t* tmem_ptr_generic = reinterpret_cast<volatile uint32_t*>(
      smem_raw + (tmem_ptr_addr - smem_u32(smem_raw)));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b0);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(cfull_bar(b), 1);
      mbar_init(cempty_bar(b), 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_ptr_addr, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_ptr_generic;

  pdl_wait();
  pdl_launch_dependents();

  const int tile = blockIdx.y;
  bool active = tile < *a.n_tiles;
  int e = 0, row0 = 0, nrows = 0;
  bool shared_expert = false;
  if (active) {
    e = a.tile_expert[tile];
    row0 = a.tile_row0[tile];
    nrows = a.tile_nrows[tile];
    shared_expert = e >= a.n_experts;
    active = static_cast<int>(blockIdx.x) < (shared_expert ? a.mblocks_shared : a.mblocks_routed);
  }

  if (active) {
    const int num_k_blocks = shared_expert ? a.kblocks_shared : a.kblocks_routed;
    const int nsplit = (MODE == 0) ? 1 : a.nsplit;
    // partial token tiles: only the 32-row boxes that hold rows (see grouped_tc_kernel)
    const int n32 = (nrows + 31) >> 5;
    const bool part = TN >= 64 && n32 * 32 < TN;
    const uint32_t b_bytes = part ? static_cast<uint32_t>(n32) * kPartBoxBytes : kBTile;
    const uint32_t idesc = make_idesc_bf16(128, part ? ((nrows + 15) & ~15) : TN);
    const int kc = max(1, kChunkSteps / (4 * nsplit));  // K blocks per chunk
    const int n_chunks = ceil_div(num_k_blocks, kc);
    const bool own_map = (MODE == 1) && shared_expert;
    const CUtensorMap* map_a = own_map ? &tmap_a_shared : &tmap_a;
    const int a_row = (own_map ? 0 : (shared_expert ? a.n_experts : e) * a.rows_per_expert) +
                      static_cast<int>(blockIdx.x) * 128;

    if (warp == 0) {
      if (lane == 0) {
        for (int kb = 0; kb < num_k_blocks; ++kb) {
          const int s = kb % kStages;
          const uint32_t ph = (kb / kStages) & 1u;
          mbar_wait(empty_bar(s), ph ^ 1u);
          mbar_arrive_expect_tx(full_bar(s), kATileBytes + nsplit * b_bytes);
          const uint32_t a_smem = smem_base + s * kStageBytes;
          tma_load_2d(a_smem, map_a, 0, ((a_row >> 7) * num_k_blocks + kb) * 128, full_bar(s),
                      kPolicyEvictFirst);
          if (part) {
            for (int j = 0; j < n32; ++j) {
              const uint32_t dst = a_smem + kATileBytes + j * kPartBoxBytes;
              tma_load_2d(dst, &tmap_s0, kb * kBlockK, row0 + 32 * j, full_bar(s), kPolicyEvictLast);
              if (MODE == 1 && nsplit > 1)
                tma_load_2d(dst + kBTile, &tmap_s1, kb * kBlockK, row0 + 32 * j, full_bar(s),
                            kPolicyEvictLast);
              if (MODE == 1 && nsplit > 2)
                tma_load_2d(dst + 2 * kBTile, &tmap_s2, kb * kBlockK, row0 + 32 * j, full_bar(s),
                            kPolicyEvictLast);
            }
            continue;
          }
          tma_load_2d(a_smem + kATileBytes, &tmap_b0, kb * kBlockK, row0, full_bar(s), kPolicyEvictLast);
          if (MODE == 1 && nsplit > 1)
            tma_load_2d(a_smem + kATileBytes + kBTile, &tmap_b1, kb * kBlockK, row0, full_bar(s),
                        kPolicyEvictLast);
          if (MODE == 1 && nsplit > 2)
            tma_load_2d(a_smem + kATileBytes + 2 * kBTile, &tmap_b2, kb * kBlockK, row0, full_bar(s),
                        kPolicyEvictLast);
        }
      }
    } else if (warp == 1) {
      if (lane == 0) {
        int kb = 0;
        for (int c = 0; c < n_chunks; ++c) {
          const int b = c & 1;
          if (c >= 2) {  // the epilogue warps have folded chunk c - 2 out of this buffer
            mbar_wait(cempty_bar(b), ((c >> 1) - 1) & 1u);
            tc_fence_after();
          }
          const uint32_t acc = tmem_base + (1u + b) * kCols;
          const int kb_end = min(num_k_blocks, kb + kc);
          bool first = true;
          for (; kb < kb_end; ++kb) {
            const int s = kb % kStages;
            const uint32_t ph = (kb / kStages) & 1u;
            mbar_wait(full_bar(s), ph);
            tc_fence_after();
            const uint32_t a_smem = smem_base + s * kStageBytes;
            const uint64_t a_desc = make_smem_desc_sw128(a_smem);
#pragma unroll
            for (int sp = 0; sp < (MODE == 0 ? 1 : kMaxSplit); ++sp) {
              if (sp < nsplit) {
                const uint64_t b_desc = make_smem_desc_sw128(a_smem + kATileBytes + sp * kBTile);
#pragma unroll
                for (int k = 0; k < kBlockK / 16; ++k) {
                  umma_bf16(acc, a_desc + 2u * k, b_desc + 2u * k, idesc, first ? 0u : 1u);
                  first = false;
                }
              }
            }
            umma_commit(empty_bar(s));
          }
          umma_commit(cfull_bar(b));
        }
      }
    } else {
      // ---- epilogue warps: fold chunks into the master accumulator, then the epilogue proper ----
      const int q = warp & 3;  // TMEM lane quarter this warp may read
      const int m_valid = shared_expert ? a.m_shared : a.m_routed;
      const uint32_t lane_off = static_cast<uint32_t>(32 * q) << 16;
      const uint32_t master = tmem_base + lane_off;
#pragma unroll 1
      for (int c = 0; c < n_chunks; ++c) {
        const int b = c & 1;
        mbar_wait(cfull_bar(b), (c >> 1) & 1u);
        tc_fence_after();
        const uint32_t chunk = tmem_base + lane_off + (1u + b) * kCols;
        const bool last = c == n_chunks - 1;
        const int n = (MODE == 0) ? static_cast<int>(blockIdx.x) * kNeuronBlock + 16 * q + (lane & 15)
                                  : static_cast<int>(blockIdx.x) * 128 + 32 * q + lane;
#pragma unroll 1
        for (int c0 = 0; c0 < TN; c0 += 16) {
          if (c0 >= nrows) break;
          uint32_t v[16], mm[16];
          tmem_ld_32x32b_x16(chunk + c0, v);
          if (c > 0) tmem_ld_32x32b_x16(master + c0, mm);
          tmem_ld_wait();
          if (c > 0) {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              v[i] = __float_as_uint(__fadd_rn(__uint_as_float(mm[i]), __uint_as_float(v[i])));
          }
          if (!last) {
            tmem_st_32x32b_x16(master + c0, v);
            continue;
          }
          if (MODE == 0) {
            swiglu_store16<TN>(v, lane, c0, nrows, n, m_valid, row0, tile, a);
          } else {
#pragma unroll
            if (a.out_rows != nullptr) {
              const int col = c0 + lane;
              const unsigned long long mine =
                  (lane < 16 && col < nrows)
                      ? reinterpret_cast<unsigned long long>(a.out_rows[a.out_perm[row0 + col]])
                      : 0ull;
#pragma unroll
              for (int cc = 0; cc < 16; ++cc) {
                float* dst = reinterpret_cast<float*>(__shfl_sync(0xffffffffu, mine, cc));
                if (c0 + cc < nrows && n < m_valid) dst[n] = __uint_as_float(v[cc]);
              }
            } else {
#pragma unroll
              for (int cc = 0; cc < 16; ++cc)
                if (c0 + cc < nrows && n < m_valid)
                  a.out[static_cast<size_t>(row0 + c0 + cc) * a.out_stride + n] = __uint_as_float(v[cc]);
            }
          }
        }
        if (!last) {
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(cempty_bar(b));
        }
      }
      tc_fence_before();
    }
  }

  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
}

// the dynamic shared memory opt-in is per device: one flag per (kernel, device)
template <class K>
static void ensure_smem_attr(K kernel, int smem, unsigned long long* mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(__atomic_load_n(mask, __ATOMIC_ACQUIRE) & bit)) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    __atomic_fetch_or(mask, bit, __ATOMIC_RELEASE);
  }
}

template <int TN, int MODE>
static void launch_tc_chunked(const LaunchCtx& ctx, const CUtensorMap* ta, const CUtensorMap* ta_sh,
                              const CUtensorMap* tb0, const CUtensorMap* tb1, const CUtensorMap* tb2,
                              const CUtensorMap* ts /*[3]: 32-row boxes*/, const TcArgs& a, int grid_x,
                              int max_tiles) {
  static unsigned long long mask = 0;
  constexpr int smem = chunked_smem_bytes(TN, MODE);
  ensure_smem_attr(grouped_tc_chunked_kernel<TN, MODE>, smem, &mask);
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = ctx.pdl ? 1 : 0;
  cfg.stream = ctx.stream;
  cfg.gridDim = dim3(grid_x, max_tiles);
  cfg.blockDim = dim3(kGateupThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchKernelEx(&cfg, grouped_tc_chunked_kernel<TN, MODE>, *ta, *ta_sh, *tb0, *tb1, *tb2, ts[0],
                     ts[MODE == 1 ? 1 : 0], ts[MODE == 1 ? 2 : 0], a);
}

// Chunked accumulation pays when one accumulator would take more than ~96 truncating steps
// (drift above ~3.5e-6 of the result); shorter contractions keep the single accumulator.
static bool wants_chunks(bool precise, int k_blocks, int nsplit) {
  return precise && k_blocks * 4 * nsplit > 96;
}

static int pick_tile_case(int tile_tokens) {
  if (tile_tokens <= 16) return 16;
  if (tile_tokens <= 32) return 32;
  if (tile_tokens <= 64) return 64;
  if (tile_tokens <= 128) return 128;
  return 256;
}

template <int TN, int MODE, int MB = 1>
static void launch_tc_case(const LaunchCtx& ctx, const CUtensorMap* ta, const CUtensorMap* ta_sh,
                           const CUtensorMap* tb0, const CUtensorMap* tb1, const CUtensorMap* tb2,
                           const CUtensorMap* ts /*[3]: 32-row boxes*/, const TcArgs& a, int grid_x,
                           int max_tiles) {
  static unsigned long long mask = 0;
  constexpr int smem = gateup_smem_bytes(TN, MODE, MB);
  ensure_smem_attr(grouped_tc_kernel<TN, MODE, MB>, smem, &mask);
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = ctx.pdl ? 1 : 0;
  cfg.stream = ctx.stream;
  cfg.gridDim = dim3(ceil_div(grid_x, MB), max_tiles);
  cfg.blockDim = dim3(kGateupThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchKernelEx(&cfg, grouped_tc_kernel<TN, MODE, MB>, *ta, *ta_sh, *tb0, *tb1, *tb2, ts[0],
                     ts[MODE == 1 ? 1 : 0], ts[MODE == 1 ? 2 : 0], a);
}

int launch_gateup_tc(const LaunchCtx& ctx, const CUtensorMap* tmap_w, const CUtensorMap* tmap_x,
                     const CUtensorMap* tmap_x32, int tile_tokens, const DispatchBuffers& d, int max_tiles, const Geometry& g,
                     float* h, bool token_tiles, float* sg, bool pair_blocks, bool precise,
                     bool early_tiles, const void* w_image, const int* tiles_flag) {
  TcArgs a{};
  a.tiles_flag = tiles_flag;
  a.early_tiles = (early_tiles || tiles_flag != nullptr) ? 1 : 0;
  a.a_base = a.a_shared_base = w_image;
  a.sg_out = sg;
  a.tile_colrow = token_tiles ? d.tile_colrow : nullptr;
  a.tile_expert = d.tile_expert;
  a.tile_row0 = d.tile_row0;
  a.tile_nrows = d.tile_nrows;
  a.n_tiles = d.n_tiles;
  a.out = h;
  a.out_stride = g.Nh;
  a.n_experts = g.E;
  a.mblocks_routed = g.Np / kNeuronBlock;
  a.mblocks_shared = g.Sp / kNeuronBlock;
  a.m_routed = g.N;
  a.m_shared = g.S;
  a.kblocks_routed = a.kblocks_shared = g.Dp / kBlockK;
  a.rows_per_expert = 2 * g.Np;
  a.nsplit = 1;
  const int gx = a.mblocks_routed > a.mblocks_shared ? a.mblocks_routed : a.mblocks_shared;
  if (wants_chunks(precise, a.kblocks_routed, 1)) {
    switch (pick_tile_case(tile_tokens)) {
      case 16: launch_tc_chunked<16, 0>(ctx, tmap_w, tmap_w, tmap_x, tmap_x, tmap_x, tmap_x32, a, gx, max_tiles); break;
      case 32: launch_tc_chunked<32, 0>(ctx, tmap_w, tmap_w, tmap_x, tmap_x, tmap_x, tmap_x32, a, gx, max_tiles); break;
      case 64: launch_tc_chunked<64, 0>(ctx, tmap_w, tmap_w, tmap_x, tmap_x, tmap_x, tmap_x32, a, gx, max_tiles); break;
      default: launch_tc_chunked<128, 0>(ctx, tmap_w, tmap_w, tmap_x, tmap_x, tmap_x, tmap_x32, a, gx, max_tiles); break;
    }
    return 1;
  }
  if (pair_blocks && pick_tile_case(tile_tokens) == 64) {
    launch_tc_case<64, 0, 2>(ctx, tmap_w, tmap_w, tmap_x, tmap_x, tmap_x, tmap_x32, a, gx, max_tiles);
    return 1;
  }
  if (pair_blocks && pick_tile_case(tile_tokens) == 128) {
    launch_tc_case<128, 0, 2>(ctx, tmap_w, tmap_w, tmap_x, tmap_x, tmap_x, tmap_x32, a, gx, max_tiles);
    return 1;
  }
  switch (pick_tile_case(tile_tokens)) {
    case 16: launch_tc_case<16, 0>(ctx, tmap_w, tmap_w, tmap_x, tmap_x, tmap_x, tmap_x32, a, gx, max_tiles); break;
    case 32: launch_tc_case<32, 0>(ctx, tmap_w, tmap_w, tmap_x, tmap_x, tmap_x, tmap_x32, a, gx, max_tiles); break;
    case 64: launch_tc_case<64, 0>(ctx, tmap_w, tmap_w, tmap_x, tmap_x, tmap_x, tmap_x32, a, gx, max_tiles); break;
    case 128: launch_tc_case<128, 0>(ctx, tmap_w, tmap_w, tmap_x, tmap_x, tmap_x, tmap_x32, a, gx, max_tiles); break;
    default: launch_tc_case<256, 0>(ctx, tmap_w, tmap_w, tmap_x, tmap_x, tmap_x, tmap_x32, a, gx, max_tiles); break;
  }
  return 1;
}

int launch_down_tc(const LaunchCtx& ctx, const CUtensorMap* tmap_wdt,
                   const CUtensorMap* tmap_wdt_shared, const CUtensorMap* tmap_hb /*[3]*/,
                   const CUtensorMap* tmap_hb32 /*[3]*/, int nsplit, int tile_tokens, const DispatchBuffers& d, int max_tiles,
                   const Geometry& g, float* slot_out, bool pair_blocks, bool precise,
                   bool early_tiles, const void* wdt_image, const void* wdt_shared_image,
                   float* const* out_rows, const int32_t* out_perm) {
  TcArgs a{};
  a.out_rows = out_rows;
  a.out_perm = out_perm;
  a.early_tiles = early_tiles ? 1 : 0;
  a.a_base = wdt_image;
  a.a_shared_base = wdt_shared_image;
  a.tile_expert = d.tile_expert;
  a.tile_row0 = d.tile_row0;
  a.tile_nrows = d.tile_nrows;
  a.n_tiles = d.n_tiles;
  a.out = slot_out;
  a.out_stride = g.Dp;
  a.n_experts = g.E;
  a.mblocks_routed = a.mblocks_shared = g.Dp128 / 128;
  a.m_routed = a.m_shared = g.D;
  a.kblocks_routed = g.Np / kBlockK;
  a.kblocks_shared = g.Sp / kBlockK;
  a.rows_per_expert = g.Dp128;
  a.nsplit = nsplit;
  const CUtensorMap* sh = tmap_wdt_shared ? tmap_wdt_shared : tmap_wdt;
  const int gx = a.mblocks_routed;
  {
    const int kmax = a.kblocks_routed > a.kblocks_shared ? a.kblocks_routed : a.kblocks_shared;
    if (wants_chunks(precise, kmax, nsplit)) {
      switch (pick_tile_case(tile_tokens)) {
        case 16: launch_tc_chunked<16, 1>(ctx, tmap_wdt, sh, tmap_hb, tmap_hb + 1, tmap_hb + 2, tmap_hb32, a, gx, max_tiles); break;
        case 32: launch_tc_chunked<32, 1>(ctx, tmap_wdt, sh, tmap_hb, tmap_hb + 1, tmap_hb + 2, tmap_hb32, a, gx, max_tiles); break;
        case 64: launch_tc_chunked<64, 1>(ctx, tmap_wdt, sh, tmap_hb, tmap_hb + 1, tmap_hb + 2, tmap_hb32, a, gx, max_tiles); break;
        default: launch_tc_chunked<128, 1>(ctx, tmap_wdt, sh, tmap_hb, tmap_hb + 1, tmap_hb + 2, tmap_hb32, a, gx, max_tiles); break;
      }
      return 1;
    }
  }
  if (pair_blocks && pick_tile_case(tile_tokens) == 64) {
    launch_tc_case<64, 1, 2>(ctx, tmap_wdt, sh, tmap_hb, tmap_hb + 1, tmap_hb + 2, tmap_hb32, a, gx, max_tiles);
    return 1;
  }
  if (pair_blocks && pick_tile_case(tile_tokens) >= 128) {
    launch_tc_case<128, 1, 2>(ctx, tmap_wdt, sh, tmap_hb, tmap_hb + 1, tmap_hb + 2, tmap_hb32, a, gx, max_tiles);
    return 1;
  }
  switch (pick_tile_case(tile_tokens)) {
    case 16: launch_tc_case<16, 1>(ctx, tmap_wdt, sh, tmap_hb, tmap_hb + 1, tmap_hb + 2, tmap_hb32, a, gx, max_tiles); break;
    case 32: launch_tc_case<32, 1>(ctx, tmap_wdt, sh, tmap_hb, tmap_hb + 1, tmap_hb + 2, tmap_hb32, a, gx, max_tiles); break;
    case 64: launch_tc_case<64, 1>(ctx, tmap_wdt, sh, tmap_hb, tmap_hb + 1, tmap_hb + 2, tmap_hb32, a, gx, max_tiles); break;
    default: launch_tc_case<128, 1>(ctx, tmap_wdt, sh, tmap_hb, tmap_hb + 1, tmap_hb + 2, tmap_hb32, a, gx, max_tiles); break;
  }
  return 1;
}

// ---------------------------------------------------------------------------------------------
// Verification-only CUDA-core gate/up (SKB_FLAG_SIMT_GATEUP): one warp per (row, neuron), same
// bf16 operands and fp32 accumulation.  Never selected implicitly; exists so that the tcgen05
// path can be cross-checked on the device, operand for operand.
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) gateup_simt_kernel(const __nv_bfloat16* __restrict__ wgu,
                                                          const __nv_bfloat16* __restrict__ xs,
                                                          const int32_t* __restrict__ row_expert,
                                                          int rows, Geometry g,
                                                          float* __restrict__ h) {
  pdl_wait();
  pdl_launch_dependents();
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.y;
  const int n = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int e = row_expert[row];
  const int Ne = (e < g.E) ? g.N : g.S;
  if (n >= Ne) return;
  const size_t img_row0 =
      (e < g.E) ? static_cast<size_t>(e) * 2 * g.Np : static_cast<size_t>(g.E) * 2 * g.Np;
  const size_t blk = img_row0 + static_cast<size_t>(n / kNeuronBlock) * 128;
  const size_t rg = blk + gateup_row(n % kNeuronBlock, 0), ru = blk + gateup_row(n % kNeuronBlock, 1);
  const __nv_bfloat16* xr = xs + static_cast<size_t>(row) * g.Dp;
  float ag = 0.0f, au = 0.0f;
  for (int d = lane; d < g.Dp; d += 32) {
    const float xv = __bfloat162float(xr[d]);
    ag = fmaf(__bfloat162float(wgu[tiled_index(rg, d, g.Dp)]), xv, ag);
    au = fmaf(__bfloat162float(wgu[tiled_index(ru, d, g.Dp)]), xv, au);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ag += __shfl_xor_sync(0xffffffffu, ag, o);
    au += __shfl_xor_sync(0xffffffffu, au, o);
  }
  if (lane == 0) h[static_cast<size_t>(row) * g.Nh + n] = silu_f(ag) * au;
}

int launch_gateup_simt(const LaunchCtx& ctx, const __nv_bfloat16* wgu, const __nv_bfloat16* xs,
                       const int32_t* row_expert, int rows, const Geometry& g, float* h) {
  const int nmax = g.N > g.S ? g.N : g.S;
  gateup_simt_kernel<<<dim3(ceil_div(nmax, 8), rows), 256, 0, ctx.stream>>>(wgu, xs, row_expert,
                                                                           rows, g, h);
  return 1;
}

}  // namespace skb
