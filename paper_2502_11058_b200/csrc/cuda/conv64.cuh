// conv64.cuh — the 64-channel 3x3 convolutions of the ResNet stem stage
// (forward and dgrad; 64 input and 64 output channels, stride 1, 32x32 or
// 16x16 images) as one specialised implicit GEMM.
//
// The general implicit conv (nn_gemm.cuh, kConvFwd / kConvDgrad) stages,
// per 64-wide k-block, a 16 KB activation box and an 8 KB weight box; with
// N = 64 its MMAs finish long before the next 24 KB arrive from L2.  Here:
//   * the weights stay resident in shared memory (9 taps x 64 x 64 bf16 =
//     72 KB, reloaded only when the tile's worker changes);
//   * the activations are staged once per horizontal tap: one box covers the
//     tile's R = 128/W output rows plus a halo row above and below, and the
//     three vertical taps are views into it at whole-row offsets (W x 128 B:
//     4 KB / 2 KB, multiples of the 1 KB swizzle atom).
// So a 128-pixel tile moves 3 x (R+2) x W x 128 B (72 KB at W = 32) instead
// of 9 x 24 KB, all nine taps' MMAs run from three stages.  Warp roles,
// double-buffered TMEM accumulator and the TMA-store epilogue are those of
// gemm_tc_kernel, with 8 epilogue warps (two per TMEM lane quarter, one
// 32-column chunk each): with 9 k-blocks per tile the epilogue's operand
// loads (ReLU' mask, residual) bound the dgrad otherwise (489 -> 643 TFLOP/s).
#pragma once

#include "nn_gemm.cuh"

namespace dsx_nn {

struct Conv64Cfg {
  static constexpr int kABytesMax = (128 + 2 * 32) * 128;  // W = 32: 6 rows x 32 px x 128 B
  static constexpr int kStages = 5;
  static constexpr int kBBytes = 9 * 64 * 64 * 2;          // resident weights, 9 taps
  static constexpr int kEpiWarps = 8;                      // two per TMEM lane quarter
  static constexpr int kEpiBytes = kEpiWarps * 32 * 33 * 4;
  static constexpr int kSmem = kStages * kABytesMax + kBBytes + kEpiBytes + 1024 + 256;
  static constexpr int kTmemCols = 128;                    // 2 x 64-column accumulators
};

// MODE: kConvFwd (B = W[o][tap][c] K-major) or kConvDgrad (B(n=c, k=o) =
// W[o][tap][c], MN-major).  g.conv_w in {16, 32}, g.M = B*H*W pixels.
template <int MODE>
__global__ void __launch_bounds__(64 + 32 * Conv64Cfg::kEpiWarps, 1)
conv64_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, GemmArgs g,
              const __grid_constant__ CUtensorMap tcm) {
  using Cfg = Conv64Cfg;
  constexpr bool B_MN = MODE == kConvDgrad;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* bres = smem + Cfg::kStages * Cfg::kABytesMax;
  float* epi_smem = reinterpret_cast<float*>(bres + Cfg::kBBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(bres + Cfg::kBBytes + Cfg::kEpiBytes);
  uint64_t* empty = full + Cfg::kStages;
  uint64_t* tfull = empty + Cfg::kStages;  // [2]
  uint64_t* tempty = tfull + 2;            // [2]
  uint64_t* bfull = tempty + 2;            // resident weights landed
  uint64_t* bfree = bfull + 1;             // MMAs on the previous worker's weights done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfree + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int W = g.conv_w, R = kBM / W;
  const int abytes = (R + 2) * W * 128;
  const int mt = (g.M + kBM - 1) / kBM;
  const int tiles = mt * g.batch;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&ta) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tb) : "memory");
    for (int s = 0; s < Cfg::kStages; ++s) {
      nn_mbar_init(&full[s], 1);
      nn_mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      nn_mbar_init(&tfull[a], 1);
      nn_mbar_init(&tempty[a], Cfg::kEpiWarps);
    }
    nn_mbar_init(bfull, 1);
    nn_mbar_init(bfree, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(Cfg::kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_enter();

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      int it = 0, cur_b = -1;
      unsigned bfree_ph = 0;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const int b = tile / mt, m0 = (tile - b * mt) * kBM;
        if (b != cur_b) {
          if (cur_b >= 0) {
            nn_mbar_wait(bfree, bfree_ph);
            bfree_ph ^= 1u;
          }
          nn_mbar_expect_tx(bfull, Cfg::kBBytes);
#pragma unroll 1
          for (int tap = 0; tap < 9; ++tap) {
            if constexpr (MODE == kConvFwd) tma_load_3d(bres + tap * 8192, &tb, bfull, tap * 64, 0, b);
            else tma_load_4d(bres + tap * 8192, &tb, bfull, 0, tap, 0, b);
          }
          cur_b = b;
        }
        int img, h0;
        conv_pix(g, m0, &img, &h0);
#pragma unroll 1
        for (int kw = 0; kw < 3; ++kw, ++it) {
          const int s = it % Cfg::kStages;
          nn_mbar_wait(&empty[s], ((unsigned)(it / Cfg::kStages) & 1u) ^ 1u);
          nn_mbar_expect_tx(&full[s], (unsigned)abytes);
          // rows h0-1 .. h0+R (halo), columns shifted by the horizontal tap
          tma_load_5d(smem + s * Cfg::kABytesMax, &ta, &full[s], 0, MODE == kConvFwd ? kw - 1 : 1 - kw, h0 - 1, img,
                      b);
        }
      }
    }
  } else if (warp == 1) {
    {  // MMA issuer: converged warp, elected lane (tc_mma_kblock / tc_commit_elect)
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((B_MN ? 1u : 0u) << 16) |
                             ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(kBM >> 4) << 24);
      int it = 0, tc = 0, cur_b = -1;
      unsigned bfull_ph = 0;
      const unsigned bsm = su32(bres);
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++tc) {
        const int b = tile / mt;
        if (b != cur_b) {
          if (cur_b >= 0) tc_commit_elect(bfree);  // the previous worker's MMAs release the weights
          nn_mbar_wait(bfull, bfull_ph);
          bfull_ph ^= 1u;
          tc_fence_after();
          cur_b = b;
        }
        const int acc = tc & 1;
        nn_mbar_wait(&tempty[acc], ((unsigned)(tc >> 1) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(acc * 64);
#pragma unroll 1
        for (int kw = 0; kw < 3; ++kw, ++it) {
          const int s = it % Cfg::kStages;
          nn_mbar_wait(&full[s], (unsigned)(it / Cfg::kStages) & 1u);
          tc_fence_after();
          const unsigned sa = su32(smem + s * Cfg::kABytesMax);
#pragma unroll
          for (int kh = 0; kh < 3; ++kh) {
            // forward: input row h + kh - 1 = halo row kh; dgrad: dy row h + 1 - kh = halo row 2 - kh
            const unsigned a0 = sa + (unsigned)((MODE == kConvFwd ? kh : 2 - kh) * W * 128);
            const unsigned b0 = bsm + (unsigned)((kh * 3 + kw) * 8192);
            tc_mma_kblock<false, B_MN>(d, smem_desc(a0, 16, 1024),
                                       B_MN ? smem_desc(b0, kBK * 128, 1024) : smem_desc(b0, 16, 1024), idesc,
                                       (kw | kh) != 0 ? 1u : 0u);
          }
          tc_commit_elect(&empty[s]);
        }
        tc_commit_elect(&tfull[acc]);
      }
    }
  } else {  // epilogue warps (TMA-store, bf16): lane quarter warp % 4, 64 / (kEpiWarps / 4) columns each
    constexpr int kCols = 64 / (Cfg::kEpiWarps / 4);
    const int q = warp & 3, cbeg = ((warp - 2) >> 2) * kCols;
    uint8_t* stg = reinterpret_cast<uint8_t*>(epi_smem + (warp - 2) * 32 * 33);
    int tc = 0, chunk_ctr = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++tc) {
      const int b = tile / mt, m0 = (tile - b * mt) * kBM + 32 * q;
      const int acc = tc & 1;
      nn_mbar_wait(&tfull[acc], (unsigned)(tc >> 1) & 1u);
      tc_fence_after();
#pragma unroll 1
      for (int c = cbeg; c < cbeg + kCols; c += 32)
        epi_chunk_tma(g, &tcm, tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(acc * 64 + c),
                      stg + (chunk_ctr++ & 1) * 2048, lane, b, m0, c);
      tc_fence_before();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&tempty[acc])) : "memory");
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(Cfg::kTmemCols) : "memory");
  }
}

}  // namespace dsx_nn
