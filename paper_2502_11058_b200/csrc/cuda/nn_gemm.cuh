// nn_gemm.cuh — the dense-layer GEMMs of the NN local step (north_star (1)):
//
//   gemm_tc_kernel   bf16 x bf16 -> fp32 on the 5th-gen tensor cores:
//                    TMA (cp.async.bulk.tensor, 128-B swizzle) stages A/B
//                    tiles through a multi-stage mbarrier ring, one elected
//                    thread issues tcgen05.mma (kind::f16, M=128, N=BN, K=16)
//                    into a TMEM accumulator, four epilogue warps drain it
//                    with tcgen05.ld and apply the layer epilogue.
//   gemm_f32_kernel  fp32 SIMT FFMA GEMM for the 1e-5 parity runs (TF32 or
//                    bf16 tensor cores cannot meet 1e-5; SURVEY §7 "fp32
//                    GEMM parity").
//
// One GEMM, C[m][n] = sum_k A(m,k) B(n,k), batched over local workers
// (blockIdx.z), covers the three GEMMs of a Linear layer y = x W^T with
// row-major tensors x[B][in], W[out][in], y[B][out]:
//   forward  y  = x  W^T : A = x  (K-major),  B = W  (K-major)
//   dgrad    dx = dy W   : A = dy (K-major),  B = W  (N-major: W[k=out][n=in])
//   wgrad    dW = dy^T x : A = dy (M-major),  B = x  (N-major)
// MN-major operands are read by TMA in 64-element-wide boxes and described
// to the MMA as MN-major canonical layouts, so no transposed copies exist.
#pragma once
#include <cstdlib>
#include <utility>

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "dsx.h"

namespace dsx_nn {

// epilogue kinds
enum : int {
  kEpiF32 = 0,       // C fp32 = acc (+ C if accumulate)
  kEpiBiasAct = 1,   // C = act(acc + bias[n])   (act: none / relu), T out
  kEpiDRelu = 2,     // C = acc * (mask(m,n) > 0), T out (dgrad through relu)
  kEpiAdd = 3,       // C = acc + mask(m,n), T out (dgrad into a residual sum)
  // the residual block's elementwise ops fused into its GEMMs (TMA-store /
  // SIMT epilogues only):
  kEpiBiasAddAct = 4,  // C = act(acc + bias[n] + mask(m,n)): block output relu(conv + shortcut)
  kEpiAddDRelu = 5,    // C = (acc + mask(m,n)) * (mask2(m,n) > 0): input grad of a block,
                       //     times the previous block's ReLU'
};

// Implicit-GEMM convolution (3x3, stride 1, pad 1, NHWC, channel counts
// multiples of 64): the operand tiles are read straight from the activation
// tensors by 5-D TMA boxes shifted by the filter tap, the padding coming from
// TMA's out-of-bounds zero fill — no im2col / col2im buffers.
//   kConvFwd    A(m=pixel, k=(tap,c)) = x[pixel + tap - 1][c]     (5-D map on x)
//   kConvWgrad  B(n=(tap,c), k=pixel) = x[pixel + tap - 1][c]     (5-D map on x, MN-major)
//   kConvDgrad  A(m=pixel, k=(tap,o)) = dy[pixel - tap + 1][o]    (5-D map on dy)
//               B(n=c, k=(tap,o))     = W[o][tap][c]              (4-D map on W, MN-major)
// A 128-pixel M tile / 64-pixel K block covers whole image rows (W | 64).
//   kConvWgradT A(m=(tap,c), k=pixel) = x[pixel + tap - 1][c]    (5-D map on x, MN-major)
//               B(n=o, k=pixel)       = dy[pixel][o]              (dW^T: narrow Cout fills M-tiles)
enum : int { kConvNone = 0, kConvFwd = 1, kConvWgrad = 2, kConvDgrad = 3, kConvWgradT = 4 };

struct GemmArgs {
  int M, N, K, batch;
  int epi, relu, accumulate;
  void* C;
  long long ldc, strideC;        // elements
  const float* bias;             // [batch][...] fp32, indexed bias[b*strideBias + n]
  long long strideBias;
  const void* mask;              // relu' source, same element type as C
  long long ldmask, strideMask;
  // split-K (tensor-core path, kEpiF32 without accumulate): K is cut into
  // ksplit ranges of whole k-blocks; split s writes its partial product to
  // C + s * strideSplit, the caller sums the partials in a fixed order.
  // 0 / 1: off.
  int ksplit;
  long long strideSplit;
  // implicit conv geometry (CONV != kConvNone): image H x W, 64-channel
  // chunks of the reduction operand per tap (Cin/64 fwd, Cout/64 dgrad),
  // input channels (wgrad: the tap of output column n is n / cin)
  int conv_h, conv_w, conv_cpb, conv_cin;
  // stride-2 convs (3x3 pad 1, or 1x1 pad 0: the projection shortcuts),
  // forward and wgrad only: conv_h / conv_w are the OUTPUT grid, the 5-D
  // input boxes traverse every second row / column (TMA element strides)
  int conv_stride, conv_k;
  const void* mask2;  // kEpiAddDRelu: the ReLU' source (same layout as mask)
  long long ldmask2, strideMask2;
};

// pixel index p (multiple of the tile's row span) -> (image, row)
__device__ __forceinline__ void conv_pix(const GemmArgs& g, int p, int* img, int* h) {
  const int hw = g.conv_h * g.conv_w;
  *img = p / hw;
  *h = (p % hw) / g.conv_w;
}

// One GEMM call: operands (element pointers, leading dims, per-batch
// strides), majors, tile width (0: auto) and the epilogue.  gemm() (gemm.cu)
// launches the tcgen05 kernel for bf16 and the SIMT kernel for fp32.
struct GemmCall {
  bool bf16;
  bool a_mn, b_mn;
  const void* A;
  long long lda, sA;
  const void* B;
  long long ldb, sB;
  bool out_bf16;
  int bn;
  GemmArgs g;
};
dsx_status gemm(const GemmCall& c, cudaStream_t s, int nsm);
// Implicit-GEMM 3x3 / stride 1 / pad 1 convolution on the tensor cores
// (see kConv*): B images of H x W, NHWC bf16 activations.  GemmCall carries
// the operand pointers and per-worker strides (A = x or dy, B = W or x) and
// the epilogue; M / N / K are derived from the geometry.
struct ConvGeom {
  int mode, H, W, B, cin, cout;  // H, W: the input grid
  int stride = 1, k = 3;         // stride 2 (3x3 or 1x1): forward / wgrad only
};
dsx_status conv_gemm(const GemmCall& c, const ConvGeom& q, cudaStream_t s, int nsm);

constexpr int kBM = 128, kBK = 64, kUmmaK = 16;

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void nn_mbar_init(uint64_t* b, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void nn_mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void nn_mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n NN_WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra NN_WAIT_%=;\n}\n" ::"r"(
          su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          su32(dst)),
      "l"(map), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];" ::"r"(su32(dst)),
      "l"(map), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, "
      "%7}], [%2];" ::"r"(su32(dst)),
      "l"(map), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// Programmatic dependent launch: once this CTA's prologue (barriers, TMEM,
// tensor-map prefetch) is done, let the next PDL-launched grid start its own
// prologue on free SMs, then wait for every prerequisite grid to finish and
// flush before touching global memory.  Both are no-ops for a normal launch.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Launches a kernel that starts with pdl_enter() with programmatic stream
// serialization (PDL): it may start while the previous kernel on the stream
// drains and waits in pdl_enter() (griddepcontrol.wait) before its first
// global access.  DSX_PDL=0: plain launches.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  static const bool on = [] {
    const char* e = std::getenv("DSX_PDL");
    return !(e && e[0] == '0');
  }();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = on ? at : nullptr;
  cfg.numAttrs = on ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(
          tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

// The four K=16 MMAs of one 64-wide k-block in ONE asm statement: the MMA
// thread runs inside a lane-0 branch, where the compiler wraps every
// uniform-datapath UTCHMMA in its own elect / branch loop (~17 instructions,
// longer than a 128 x 64 x 16 MMA takes); one statement pays that once.
// Descriptor k advances: K-major +32 B (2 in 16-B units), MN-major +2 KB.
// Called by the whole (converged) MMA warp: elect.sync picks the issuing
// lane inside the statement, so no per-instruction elect loop is generated.
template <bool A_MN, bool B_MN>
__device__ __forceinline__ void tc_mma_kblock(uint32_t tmem, uint64_t ad, uint64_t bd, uint32_t idesc,
                                              uint32_t acc) {
  constexpr uint64_t da = A_MN ? (16 * 128) >> 4 : 2, db = B_MN ? (16 * 128) >> 4 : 2;
  asm volatile(
      "{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %5, %6, %3, 1;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %7, %8, %3, 1;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %9, %10, %3, 1;\n}\n" ::"r"(tmem),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc), "l"(ad + da), "l"(bd + db), "l"(ad + 2 * da), "l"(bd + 2 * db),
      "l"(ad + 3 * da), "l"(bd + 3 * db)
      : "memory");
}
// tcgen05.commit from one elected lane of a converged warp
__device__ __forceinline__ void tc_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(su32(bar))
      : "memory");
}

// Shared-memory matrix descriptor (sm_100 UMMA): start address, leading /
// stride byte offsets (16-B units), version 1, 128-B swizzle.
__device__ __forceinline__ uint64_t smem_desc(unsigned addr, unsigned lbo_bytes, unsigned sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (Blackwell)
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// Epilogue of one output element (m, n) of batch b.
template <typename TOut>
__device__ __forceinline__ void epi_store(const GemmArgs& g, int b, int m, int n, float acc) {
  if (g.epi == kEpiF32) {
    float* c = static_cast<float*>(g.C) + (long long)b * g.strideC + (long long)m * g.ldc + n;
    *c = g.accumulate ? *c + acc : acc;
    return;
  }
  TOut* c = static_cast<TOut*>(g.C) + (long long)b * g.strideC + (long long)m * g.ldc + n;
  if (g.epi == kEpiBiasAct) {
    float v = acc + (g.bias ? g.bias[(long long)b * g.strideBias + n] : 0.f);
    if (g.relu) v = fmaxf(v, 0.f);
    *c = from_f<TOut>(v);
  } else {  // kEpiDRelu / kEpiAdd / kEpiBiasAddAct / kEpiAddDRelu
    const float mk =
        to_f<TOut>(static_cast<const TOut*>(g.mask)[(long long)b * g.strideMask + (long long)m * g.ldmask + n]);
    float v;
    if (g.epi == kEpiAdd) {
      v = acc + mk;
    } else if (g.epi == kEpiBiasAddAct) {
      v = acc + (g.bias ? g.bias[(long long)b * g.strideBias + n] : 0.f) + mk;
      if (g.relu) v = fmaxf(v, 0.f);
    } else if (g.epi == kEpiAddDRelu) {
      const float m2 = to_f<TOut>(
          static_cast<const TOut*>(g.mask2)[(long long)b * g.strideMask2 + (long long)m * g.ldmask2 + n]);
      v = m2 > 0.f ? acc + mk : 0.f;
    } else {
      v = mk > 0.f ? acc : 0.f;
    }
    *c = from_f<TOut>(v);
  }
}

// ---------------------------------------------------------------------------
// tcgen05 GEMM, persistent: one CTA per SM walks the 128 x BN output tiles
// (tile = blockIdx.x + i * gridDim.x).  Warp 0 = TMA producer (smem ring of
// kStages stages, mbarrier full/empty), warp 1 = TMEM owner + MMA issuer,
// warps 2..5 = epilogue.  The accumulator is double-buffered in TMEM
// (2 x BN columns), so tile i's epilogue overlaps tile i+1's MMAs.  The
// epilogue drains TMEM with tcgen05.ld (each warp owns TMEM lanes
// 32*(warp%4) .. +31 = 32 tile rows), transposes 32x32 chunks through a
// padded shared-memory buffer and stores full rows: coalesced 128-B (fp32)
// or 64-B (bf16) row segments per warp instruction, with bias / ReLU / ReLU'
// applied on the coalesced side.
// ---------------------------------------------------------------------------
template <int BN, int EW = 4>
struct TcCfg {
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStage = kABytes + kBBytes;
  static constexpr int kStages = BN >= 256 ? 4 : (BN >= 128 ? 6 : 8);
  static constexpr int kEpiWarps = EW;
  static constexpr int kThreads = 64 + 32 * EW;
  static constexpr int kEpiBytes = EW * 32 * 33 * 4;  // per epilogue warp: 32 x 33 fp32
  static constexpr int kSmem = kStages * kStage + kEpiBytes + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int kTmemCols = 2 * BN < 32 ? 32 : 2 * BN;  // two accumulator buffers
};

template <typename TOut>
__device__ __forceinline__ float epi_value(const GemmArgs& g, int b, int m, int n, float acc) {
  if (g.epi == kEpiBiasAct) {
    float v = acc + (g.bias ? g.bias[(long long)b * g.strideBias + n] : 0.f);
    return g.relu ? fmaxf(v, 0.f) : v;
  }
  if (g.epi == kEpiDRelu || g.epi == kEpiAdd) {
    const TOut mk = static_cast<const TOut*>(g.mask)[(long long)b * g.strideMask + (long long)m * g.ldmask + n];
    return g.epi == kEpiAdd ? acc + to_f<TOut>(mk) : (to_f<TOut>(mk) > 0.f ? acc : 0.f);
  }
  return acc;
}

// Tile order: within a batch entry, groups of 8 M-tiles walk the N-tiles
// column by column, so the CTAs running at once share B panels through L2
// (the 32000-class head read its 131 MB weight 16x from DRAM in row order).
__device__ __forceinline__ void tile_coords(int tile, int mt, int ntl, int* b, int* mb, int* nb) {
  constexpr int G = 8;
  const int per = mt * ntl;
  *b = tile / per;
  const int t = tile % per;
  const int group = t / (G * ntl), first = group * G;
  const int gsz = min(G, mt - first);
  const int r = t % (G * ntl);
  *mb = first + r % gsz;
  *nb = r / gsz;
}

// ReLU' mask words of one 32x32 bf16 chunk, the layout epi_chunk's bf16 path
// uses (lane: rows 2*i2 + lane/16, columns n, n+1), one 4-B load per row.
template <typename TOut>
__device__ __forceinline__ void load_mask_words(const GemmArgs& g, int b, int m0, int n, int lane, uint32_t w[16]) {
  const bool ok = n + 1 < g.N;
  const TOut* mp = static_cast<const TOut*>(g.mask) + (long long)b * g.strideMask + n;
#pragma unroll
  for (int i2 = 0; i2 < 16; ++i2) {
    const int m = m0 + 2 * i2 + (lane >> 4);
    w[i2] = (ok && m < g.M) ? *reinterpret_cast<const uint32_t*>(mp + (long long)m * g.ldmask) : 0u;
  }
}

// Epilogue of one 32-row x 32-column accumulator chunk: tcgen05.ld (this
// warp's TMEM lanes), transpose through padded smem, coalesced row stores
// with the epilogue op applied on the coalesced side.  m0 / n0: the chunk's
// first row / column in C.
template <typename TOut>
__device__ __forceinline__ void epi_chunk(const GemmArgs& g, uint32_t taddr, float* st, int lane, int b, int m0,
                                          int n0, bool ob, const uint32_t* mwords) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
      "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
        "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
        "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  // row-per-lane -> padded smem (conflict-free: bank = (lane + j) % 32)
#pragma unroll
  for (int j = 0; j < 32; ++j) st[lane * 33 + j] = __uint_as_float(r[j]);
  __syncwarp();
  // Epilogue operands are fetched before any store, all loads of the chunk in
  // flight at once (stores to C could alias them, so the compiler would
  // otherwise serialise one global-latency round trip per row): bias once
  // per column, the ReLU' mask of every row of the chunk.
  if (ob) {
    // bf16: two rows per instruction, 16 lanes x 2 columns each
    const int cc = 2 * (lane & 15), n = n0 + cc;
    const bool n_ok = n < g.N, n1_ok = n + 1 < g.N;
    float b0 = 0.f, b1 = 0.f;
    if (g.epi == kEpiBiasAct && g.bias) {
      const float* bp = g.bias + (long long)b * g.strideBias + n;
      if (n_ok) b0 = bp[0];
      if (n1_ok) b1 = bp[1];
    }
    float mk0[16], mk1[16];
    if (g.epi == kEpiDRelu || g.epi == kEpiAdd) {
      if (mwords && n1_ok) {  // prefetched by the caller one chunk ahead
#pragma unroll
        for (int i2 = 0; i2 < 16; ++i2) {
          mk0[i2] = __uint_as_float(mwords[i2] << 16);
          mk1[i2] = __uint_as_float(mwords[i2] & 0xFFFF0000u);
        }
      } else {
        const TOut* mp = static_cast<const TOut*>(g.mask) + (long long)b * g.strideMask + n;
#pragma unroll
        for (int i2 = 0; i2 < 16; ++i2) {
          const int m = m0 + 2 * i2 + (lane >> 4);
          mk0[i2] = (m < g.M && n_ok) ? to_f<TOut>(mp[(long long)m * g.ldmask]) : 0.f;
          mk1[i2] = (m < g.M && n1_ok) ? to_f<TOut>(mp[(long long)m * g.ldmask + 1]) : 0.f;
        }
      }
    }
#pragma unroll
    for (int i2 = 0; i2 < 16; ++i2) {
      const int row = 2 * i2 + (lane >> 4);
      const int m = m0 + row;
      if (m < g.M && n_ok) {
        TOut* dst = static_cast<TOut*>(g.C) + (long long)b * g.strideC + (long long)m * g.ldc + n;
        float v0 = st[row * 33 + cc], v1 = st[row * 33 + cc + 1];
        if (g.epi == kEpiBiasAct) {
          v0 += b0;
          v1 += b1;
          if (g.relu) {
            v0 = fmaxf(v0, 0.f);
            v1 = fmaxf(v1, 0.f);
          }
        } else if (g.epi == kEpiDRelu) {
          v0 = mk0[i2] > 0.f ? v0 : 0.f;
          v1 = mk1[i2] > 0.f ? v1 : 0.f;
        } else if (g.epi == kEpiAdd) {
          v0 += mk0[i2];
          v1 += mk1[i2];
        }
        if (n1_ok) *reinterpret_cast<__nv_bfloat162*>(dst) = __floats2bfloat162_rn(v0, v1);
        else *dst = from_f<TOut>(v0);
      }
    }
  } else {
    // fp32 (or scalar bf16): one row per instruction, one column per lane
    const int n = n0 + lane;
    const bool n_ok = n < g.N;
    const float bv = (g.epi == kEpiBiasAct && g.bias && n_ok) ? g.bias[(long long)b * g.strideBias + n] : 0.f;
#pragma unroll
    for (int r0 = 0; r0 < 32; r0 += 8) {
      float mk[8];
      if (g.epi == kEpiDRelu || g.epi == kEpiAdd) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int m = m0 + r0 + u;
          mk[u] = (m < g.M && n_ok)
                      ? to_f<TOut>(static_cast<const TOut*>(g.mask)[(long long)b * g.strideMask +
                                                                   (long long)m * g.ldmask + n])
                      : 0.f;
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int row = r0 + u, m = m0 + row;
        if (m < g.M && n_ok) {
          const float v = st[row * 33 + lane];
          if (g.epi == kEpiF32) {
            float* dst = static_cast<float*>(g.C) + (long long)b * g.strideC + (long long)m * g.ldc + n;
            *dst = g.accumulate ? *dst + v : v;
          } else {
            float o = v;
            if (g.epi == kEpiBiasAct) {
              o += bv;
              if (g.relu) o = fmaxf(o, 0.f);
            } else if (g.epi == kEpiDRelu) {
              o = mk[u] > 0.f ? o : 0.f;
            } else if (g.epi == kEpiAdd) {
              o += mk[u];
            }
            TOut* dst = static_cast<TOut*>(g.C) + (long long)b * g.strideC + (long long)m * g.ldc + n;
            *dst = from_f<TOut>(o);
          }
        }
      }
    }
  }
  __syncwarp();
}

// fp32 TMA-store epilogue (kEpiF32: the wgrad outputs / split-K partials):
// the lane's accumulator row goes to this warp's staging buffers as two
// 16-column halves (64-B rows, the same 2 x 2 KB double buffer as bf16) and
// leaves by two 4-D tensor stores (n, m, batch entry, split).
__device__ __forceinline__ void epi_chunk_tma_f32(const CUtensorMap* tcm, uint32_t taddr, uint8_t* stg, int* ctr,
                                                  int lane, int b, int m0, int n0, int split) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
      "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
        "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
        "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    uint8_t* stage = stg + ((*ctr)++ & 1) * 2048;
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncwarp();
    uint4* dst = reinterpret_cast<uint4*>(stage + lane * 64);
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4)
      dst[q4] = make_uint4(r[16 * h + 4 * q4], r[16 * h + 4 * q4 + 1], r[16 * h + 4 * q4 + 2], r[16 * h + 4 * q4 + 3]);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      asm volatile(
          "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(tcm),
          "r"(su32(stage)), "r"(n0 + 16 * h), "r"(m0), "r"(b), "r"(split)
          : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
}

// TMA-store epilogue of one 32-row x 32-column bf16 chunk (the CST kernels):
// the accumulator row each lane holds after tcgen05.ld gets bias (one
// coalesced load + shuffles) / ReLU / ReLU' or the residual addend (the
// lane's 64-B row segment, vector loads), is packed to bf16 into this warp's
// staging buffer (64-B rows, double-buffered) and written by one
// cp.async.bulk.tensor store; TMA clips rows / columns outside C.
__device__ __forceinline__ void epi_chunk_tma(const GemmArgs& g, const CUtensorMap* tcm, uint32_t taddr,
                                              uint8_t* stage, int lane, int b, int m0, int n0) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
      "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
        "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
        "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  const int m = m0 + lane;
  // operands fetched while the TMEM load is in flight
  float bl = 0.f;
  const bool has_bias = g.epi == kEpiBiasAct || g.epi == kEpiBiasAddAct;
  if (has_bias && g.bias && n0 + lane < g.N) bl = g.bias[(long long)b * g.strideBias + n0 + lane];
  // the lane's 32-element row segment of an elementwise operand
  auto row_seg = [&](const void* base, long long ld, long long sb, uint4 out[4]) {
    const __nv_bfloat16* mp = static_cast<const __nv_bfloat16*>(base) + (long long)b * sb + (long long)m * ld + n0;
    if (n0 + 32 <= g.N) {
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) out[q4] = reinterpret_cast<const uint4*>(mp)[q4];
    } else {
      __nv_bfloat16* mb = reinterpret_cast<__nv_bfloat16*>(out);
      for (int j = 0; j < 32 && n0 + j < g.N; ++j) mb[j] = mp[j];
    }
  };
  uint4 mw[4] = {}, mw2[4] = {};
  if (g.epi >= kEpiDRelu && m < g.M) row_seg(g.mask, g.ldmask, g.strideMask, mw);
  if (g.epi == kEpiAddDRelu && m < g.M) row_seg(g.mask2, g.ldmask2, g.strideMask2, mw2);
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
  if (has_bias) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] += __shfl_sync(0xffffffffu, bl, j);
  }
  if (g.epi >= kEpiDRelu) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(mw);
    const uint32_t* w2 = reinterpret_cast<const uint32_t*>(mw2);
#pragma unroll
    for (int j2 = 0; j2 < 16; ++j2) {
      const float lo = __uint_as_float(w[j2] << 16), hi = __uint_as_float(w[j2] & 0xFFFF0000u);
      if (g.epi == kEpiDRelu) {
        v[2 * j2] = lo > 0.f ? v[2 * j2] : 0.f;
        v[2 * j2 + 1] = hi > 0.f ? v[2 * j2 + 1] : 0.f;
      } else if (g.epi == kEpiAddDRelu) {
        const float lo2 = __uint_as_float(w2[j2] << 16), hi2 = __uint_as_float(w2[j2] & 0xFFFF0000u);
        v[2 * j2] = lo2 > 0.f ? v[2 * j2] + lo : 0.f;
        v[2 * j2 + 1] = hi2 > 0.f ? v[2 * j2 + 1] + hi : 0.f;
      } else {  // kEpiAdd, kEpiBiasAddAct
        v[2 * j2] += lo;
        v[2 * j2 + 1] += hi;
      }
    }
  }
  if ((g.epi == kEpiBiasAct || g.epi == kEpiBiasAddAct) && g.relu) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.f);
  }
  // the store issued from this buffer two chunks ago must have read it
  if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
  __syncwarp();
  uint4* dst = reinterpret_cast<uint4*>(stage + lane * 64);
#pragma unroll
  for (int q4 = 0; q4 < 4; ++q4) {
    uint4 o;
    __nv_bfloat162 p0 = __floats2bfloat162_rn(v[8 * q4 + 0], v[8 * q4 + 1]);
    __nv_bfloat162 p1 = __floats2bfloat162_rn(v[8 * q4 + 2], v[8 * q4 + 3]);
    __nv_bfloat162 p2 = __floats2bfloat162_rn(v[8 * q4 + 4], v[8 * q4 + 5]);
    __nv_bfloat162 p3 = __floats2bfloat162_rn(v[8 * q4 + 6], v[8 * q4 + 7]);
    o.x = *reinterpret_cast<uint32_t*>(&p0);
    o.y = *reinterpret_cast<uint32_t*>(&p1);
    o.z = *reinterpret_cast<uint32_t*>(&p2);
    o.w = *reinterpret_cast<uint32_t*>(&p3);
    dst[q4] = o;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) {
    asm volatile(
        "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(tcm),
        "r"(su32(stage)), "r"(n0), "r"(m0), "r"(b)
        : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
}

// CST (TMA-store epilogue) kernels run 8 epilogue warps, two per TMEM lane
// quarter splitting the tile's columns: the epilogue's operand loads
// otherwise bound short-K tiles (conv64.cuh measured 489 -> 643 TFLOP/s)
template <int BN, bool A_MN, bool B_MN, typename TOut, int CONV = kConvNone, bool CST = false>
__global__ void __launch_bounds__(TcCfg<BN, CST ? 8 : 4>::kThreads, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, GemmArgs g,
               const __grid_constant__ CUtensorMap tcm) {
  using Cfg = TcCfg<BN, CST ? 8 : 4>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* epi_smem = reinterpret_cast<float*>(smem + Cfg::kStages * Cfg::kStage);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::kStages * Cfg::kStage + Cfg::kEpiBytes);
  uint64_t* empty = full + Cfg::kStages;
  uint64_t* tfull = empty + Cfg::kStages;  // [2]
  uint64_t* tempty = tfull + 2;            // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk_all = (g.K + kBK - 1) / kBK;
  const int ks = g.ksplit > 1 ? g.ksplit : 1;
  const int kper = (nk_all + ks - 1) / ks;  // k-blocks per split (the host keeps every split non-empty)
  const int mt = (g.M + kBM - 1) / kBM, ntl = (g.N + BN - 1) / BN;
  const int per_split = mt * ntl * g.batch;
  const int tiles = per_split * ks;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&ta) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tb) : "memory");
    for (int s = 0; s < Cfg::kStages; ++s) {
      nn_mbar_init(&full[s], 1);
      nn_mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      nn_mbar_init(&tfull[a], 1);
      nn_mbar_init(&tempty[a], Cfg::kEpiWarps);  // one arrive per epilogue warp
    }
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
      // conv modes: box coordinates advance incrementally along k (no
      // divisions in the loop — the single producer thread issues 2-6 TMA
      // ops per k-block)
      const int rstep = CONV != kConvNone ? kBK / g.conv_w : 0;             // image rows per 64-pixel block
      const int istep = CONV != kConvNone && rstep >= g.conv_h ? rstep / g.conv_h : 0;  // or whole images
      const int cs = g.conv_stride > 1 ? g.conv_stride : 1;  // input rows per output row
      const bool k3 = g.conv_k != 1;                          // 3x3 taps (else 1x1, pad 0)
      int it = 0;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        int b, mb, nb;
        tile_coords(tile % per_split, mt, ntl, &b, &mb, &nb);
        const int m0 = mb * kBM, n0 = nb * BN;
        const int kb0 = (tile / per_split) * kper, kb1 = min(nk_all, kb0 + kper);
        int ctap = 0, ccb = 0, fimg = 0, fh = 0, pimg = 0, prow = 0;
        int xtap[4] = {0, 0, 0, 0}, xc0[4] = {0, 0, 0, 0};  // implicit-patch chunks: tap, channel
        if constexpr (CONV == kConvFwd || CONV == kConvDgrad) {
          ctap = kb0 / g.conv_cpb;
          ccb = kb0 - ctap * g.conv_cpb;
          conv_pix(g, m0, &fimg, &fh);
        }
        if constexpr (CONV == kConvWgrad || CONV == kConvWgradT) conv_pix(g, kb0 * kBK, &pimg, &prow);
        if constexpr (CONV == kConvWgrad) {
#pragma unroll
          for (int i = 0; i < BN / 64; ++i) {
            const int n = min(n0 + 64 * i, g.N - 64);  // columns past N: any in-bounds data
            xtap[i] = n / g.conv_cin;
            xc0[i] = n - xtap[i] * g.conv_cin;
          }
        }
        if constexpr (CONV == kConvWgradT) {
#pragma unroll
          for (int i = 0; i < kBM / 64; ++i) {
            const int mm = min(m0 + 64 * i, g.M - 64);  // rows past M: any in-bounds data
            xtap[i] = mm / g.conv_cin;
            xc0[i] = mm - xtap[i] * g.conv_cin;
          }
        }
        for (int k = kb0; k < kb1; ++k, ++it) {
          const int s = it % Cfg::kStages;
          const unsigned ph = (unsigned)(it / Cfg::kStages) & 1u;
          nn_mbar_wait(&empty[s], ph ^ 1u);
          uint8_t* sa = smem + s * Cfg::kStage;
          uint8_t* sb = sa + Cfg::kABytes;
          nn_mbar_expect_tx(&full[s], Cfg::kStage);
          if constexpr (CONV == kConvFwd || CONV == kConvDgrad) {
            // k-block = (tap, 64-channel chunk); the box is shifted by the tap
            const int dh = k3 ? ctap / 3 - 1 : 0, dw = k3 ? ctap % 3 - 1 : 0;
            if constexpr (CONV == kConvFwd) tma_load_5d(sa, &ta, &full[s], ccb * kBK, dw, cs * fh + dh, fimg, b);
            else tma_load_5d(sa, &ta, &full[s], ccb * kBK, -dw, fh - dh, fimg, b);
          } else if constexpr (CONV == kConvWgradT) {
#pragma unroll
            for (int i = 0; i < kBM / 64; ++i)
              tma_load_5d(sa + i * 64 * kBK * 2, &ta, &full[s], xc0[i], k3 ? xtap[i] % 3 - 1 : 0,
                          cs * prow + (k3 ? xtap[i] / 3 - 1 : 0), pimg, b);
          } else if constexpr (!A_MN) {
            tma_load_3d(sa, &ta, &full[s], k * kBK, m0, b);
          } else {
#pragma unroll
            for (int i = 0; i < kBM / 64; ++i)
              tma_load_3d(sa + i * 64 * kBK * 2, &ta, &full[s], m0 + 64 * i, k * kBK, b);
          }
          if constexpr (CONV == kConvWgrad) {
            // 64 pixels of the reduction x 64 columns (one tap, 64 channels) per box
#pragma unroll
            for (int i = 0; i < BN / 64; ++i)
              tma_load_5d(sb + i * 64 * kBK * 2, &tb, &full[s], xc0[i], k3 ? xtap[i] % 3 - 1 : 0,
                          cs * prow + (k3 ? xtap[i] / 3 - 1 : 0), pimg, b);
          } else if constexpr (CONV == kConvDgrad) {
#pragma unroll
            for (int i = 0; i < BN / 64; ++i)
              tma_load_4d(sb + i * 64 * kBK * 2, &tb, &full[s], n0 + 64 * i, ctap, ccb * kBK, b);
          } else if constexpr (!B_MN) {
            tma_load_3d(sb, &tb, &full[s], k * kBK, n0, b);
          } else {
#pragma unroll
            for (int i = 0; i < BN / 64; ++i)
              tma_load_3d(sb + i * 64 * kBK * 2, &tb, &full[s], n0 + 64 * i, k * kBK, b);
          }
          if constexpr (CONV == kConvFwd || CONV == kConvDgrad) {
            if (++ccb == g.conv_cpb) {
              ccb = 0;
              ++ctap;
            }
          }
          if constexpr (CONV == kConvWgrad || CONV == kConvWgradT) {
            if (istep) {
              pimg += istep;
            } else if ((prow += rstep) >= g.conv_h) {
              prow -= g.conv_h;
              ++pimg;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    {  // MMA issuer: the converged warp, one elected lane issues (tc_mma_kblock)
      // instruction descriptor: D f32, A/B bf16, majors, N>>3, M>>4
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((A_MN ? 1u : 0u) << 15) |
                             ((B_MN ? 1u : 0u) << 16) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(kBM >> 4) << 24);
      int it = 0, tc = 0;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++tc) {
        const int acc = tc & 1;
        const unsigned aph = (unsigned)(tc >> 1) & 1u;
        nn_mbar_wait(&tempty[acc], aph ^ 1u);  // the epilogue drained this buffer
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(acc * BN);
        const int nk = min(nk_all, (tile / per_split + 1) * kper) - (tile / per_split) * kper;
        for (int k = 0; k < nk; ++k, ++it) {
          const int s = it % Cfg::kStages;
          const unsigned ph = (unsigned)(it / Cfg::kStages) & 1u;
          nn_mbar_wait(&full[s], ph);
          tc_fence_after();
          const unsigned sa = su32(smem + s * Cfg::kStage);
          const unsigned sb = sa + Cfg::kABytes;
          // K-major: the 16-element K slice is 32 B into each 128-B swizzled
          // row (8-row atoms 1024 B apart); MN-major: 16 K rows of 128 B
          // further, 64-element MN chunks kBK*128 B apart.
          const uint64_t ad = A_MN ? smem_desc(sa, kBK * 128, 1024) : smem_desc(sa, 16, 1024);
          const uint64_t bd = B_MN ? smem_desc(sb, kBK * 128, 1024) : smem_desc(sb, 16, 1024);
          tc_mma_kblock<A_MN, B_MN>(d, ad, bd, idesc, k != 0 ? 1u : 0u);
          tc_commit_elect(&empty[s]);  // frees the stage once these MMAs have read it
        }
        tc_commit_elect(&tfull[acc]);  // accumulator ready for the epilogue
      }
    }
  } else {  // epilogue warps 2..5
    const int q = warp & 3;  // TMEM lane quarter this warp may access = tile rows 32q..32q+31
    float* st = epi_smem + (warp - 2) * 32 * 33;
    const bool ob = sizeof(TOut) == 2 && g.epi != kEpiF32 && (g.ldc & 1) == 0;
    int tc = 0;
    int chunk_ctr = 0;  // CST: alternates the two staging buffers
    GemmArgs gs = g;  // split s writes its partial at C + s * strideSplit
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++tc) {
      int b, mb, nb;
      tile_coords(tile % per_split, mt, ntl, &b, &mb, &nb);
      const int m0 = mb * kBM + 32 * q, n0 = nb * BN;
      const int acc = tc & 1;
      if (ks > 1) gs.C = static_cast<float*>(g.C) + (long long)(tile / per_split) * g.strideSplit;
      nn_mbar_wait(&tfull[acc], (unsigned)(tc >> 1) & 1u);
      tc_fence_after();
      // bf16 dgrad: the ReLU' mask words of chunk c+1 load while chunk c drains
      const bool pre = ob && (g.epi == kEpiDRelu || g.epi == kEpiAdd) && (g.ldmask & 1) == 0;
      uint32_t mw_cur[16], mw_nxt[16];
      if constexpr (CST) {
        uint8_t* stg = reinterpret_cast<uint8_t*>(st);  // 2 x 2 KB staging buffers of this warp
        constexpr int kCols = BN / (Cfg::kEpiWarps / 4);  // this warp's share of the tile's columns
        const int cbeg = ((warp - 2) >> 2) * kCols;
#pragma unroll 1
        for (int c = cbeg; c < cbeg + kCols; c += 32) {
          if (n0 + c >= g.N) break;
          if constexpr (std::is_same_v<TOut, float>)
            epi_chunk_tma_f32(&tcm, tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(acc * BN + c), stg, &chunk_ctr,
                              lane, b, m0, n0 + c, tile / per_split);
          else
            epi_chunk_tma(g, &tcm, tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(acc * BN + c),
                          stg + (chunk_ctr++ & 1) * 2048, lane, b, m0, n0 + c);
        }
        tc_fence_before();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&tempty[acc])) : "memory");
        continue;
      }
      if (pre) load_mask_words<TOut>(g, b, m0, n0 + 2 * (lane & 15), lane, mw_cur);
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        if (n0 + c >= g.N) break;
        const bool more = pre && c + 32 < BN && n0 + c + 32 < g.N;
        if (more) load_mask_words<TOut>(g, b, m0, n0 + c + 32 + 2 * (lane & 15), lane, mw_nxt);
        epi_chunk<TOut>(gs, tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(acc * BN + c), st, lane, b, m0, n0 + c, ob,
                        pre ? mw_cur : nullptr);
        if (more)
#pragma unroll
          for (int i = 0; i < 16; ++i) mw_cur[i] = mw_nxt[i];
        __syncwarp();
      }
      // this warp's TMEM reads of buffer `acc` are complete (wait::ld above)
      tc_fence_before();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&tempty[acc])) : "memory");
    }
    if constexpr (CST) {
      if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(Cfg::kTmemCols) : "memory");
  }
}

// ---------------------------------------------------------------------------
// tcgen05 GEMM on CTA pairs (cta_group::2): a cluster of 2 CTAs on paired
// SMs computes a 256 x BN tile with M=256 MMAs issued by the leader CTA.
// Each CTA stages its own 128 rows of A and BN/2 rows of B (TMA
// .cta_group::2: both CTAs' bytes complete on the leader's full barrier), so
// per SM the B traffic and smem footprint halve; each CTA's TMEM holds its
// 128 rows x BN accumulator (double-buffered) and its 4 epilogue warps drain
// it.  MMA completion is multicast to both CTAs' barriers; the peer's
// epilogue releases the leader's tempty barrier remotely (mapa).
// ---------------------------------------------------------------------------
template <int BN>
struct Tc2Cfg {
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = (BN / 2) * kBK * 2;
  static constexpr int kStage = kABytes + kBBytes;
  static constexpr int kStages = BN >= 256 ? 6 : 8;
  static constexpr int kEpiBytes = 4 * 32 * 33 * 4;
  static constexpr int kSmem = kStages * kStage + kEpiBytes + 1024 + 256;
  static constexpr int kTmemCols = 2 * BN;
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// both CTAs' transaction bytes land on the leader's barrier (peer bit cleared)
__device__ __forceinline__ void tma_load_3d_2sm(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                                int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          su32(dst)),
      "l"(map), "r"(su32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d_2sm(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                                int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5, %6}], [%2];" ::"r"(su32(dst)),
      "l"(map), "r"(su32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma_load_5d_2sm(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                                int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5, %6, %7}], [%2];" ::"r"(su32(dst)),
      "l"(map), "r"(su32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
__device__ __forceinline__ void tc2_mma(uint32_t tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(
          tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tc2_commit_both(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          su32(bar)),
      "h"((unsigned short)3)
      : "memory");
}
// bounded wait (a protocol error traps instead of hanging the GPU)
__device__ __forceinline__ void nn_mbar_wait_bounded(uint64_t* b, unsigned parity) {
  unsigned ok = 0;
  unsigned long long t0 = 0;
  for (int it = 0;; ++it) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(su32(b)), "r"(parity)
        : "memory");
    if (ok) return;
    if (it == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    if ((it & 1023) == 1023) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 10000000000ull) __trap();  // 10 s
    }
  }
}

template <int BN, bool A_MN, bool B_MN, typename TOut, int CONV = kConvNone>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
gemm_tc2_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, GemmArgs g) {
  using Cfg = Tc2Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* epi_smem = reinterpret_cast<float*>(smem + Cfg::kStages * Cfg::kStage);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::kStages * Cfg::kStage + Cfg::kEpiBytes);
  uint64_t* empty = full + Cfg::kStages;
  uint64_t* tfull = empty + Cfg::kStages;  // [2]
  uint64_t* tempty = tfull + 2;            // [2] (the leader's counts both CTAs' epilogues)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int nk = (g.K + kBK - 1) / kBK;
  const int mt = (g.M + 2 * kBM - 1) / (2 * kBM), ntl = (g.N + BN - 1) / BN;
  const int tiles = mt * ntl * g.batch;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&ta) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tb) : "memory");
    for (int s = 0; s < Cfg::kStages; ++s) {
      nn_mbar_init(&full[s], 1);
      nn_mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      nn_mbar_init(&tfull[a], 1);
      nn_mbar_init(&tempty[a], 8);  // 4 epilogue warps x 2 CTAs
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(Cfg::kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_enter();

  if (warp == 0) {
    if (lane == 0) {  // TMA producer (both CTAs: each stages its half)
      int it = 0;
      for (int tile = cid; tile < tiles; tile += ncl) {
        int b, mb, nb;
        tile_coords(tile, mt, ntl, &b, &mb, &nb);
        const int m0 = mb * 2 * kBM + (int)rank * kBM, n0 = nb * BN + (int)rank * (BN / 2);
        for (int k = 0; k < nk; ++k, ++it) {
          const int s = it % Cfg::kStages;
          const unsigned ph = (unsigned)(it / Cfg::kStages) & 1u;
          nn_mbar_wait_bounded(&empty[s], ph ^ 1u);
          uint8_t* sa = smem + s * Cfg::kStage;
          uint8_t* sb = sa + Cfg::kABytes;
          if (leader) nn_mbar_expect_tx(&full[s], 2 * Cfg::kStage);
          if constexpr (CONV == kConvFwd || CONV == kConvDgrad) {
            const int tap = k / g.conv_cpb, cb = k - tap * g.conv_cpb;
            const int dh = tap / 3 - 1, dw = tap % 3 - 1;
            int img, h;
            conv_pix(g, m0, &img, &h);
            if constexpr (CONV == kConvFwd) tma_load_5d_2sm(sa, &ta, &full[s], cb * kBK, dw, h + dh, img, b);
            else tma_load_5d_2sm(sa, &ta, &full[s], cb * kBK, -dw, h - dh, img, b);
          } else if constexpr (!A_MN) {
            tma_load_3d_2sm(sa, &ta, &full[s], k * kBK, m0, b);
          } else {
#pragma unroll
            for (int i = 0; i < kBM / 64; ++i)
              tma_load_3d_2sm(sa + i * 64 * kBK * 2, &ta, &full[s], m0 + 64 * i, k * kBK, b);
          }
          if constexpr (CONV == kConvWgrad) {
            int img, h;
            conv_pix(g, k * kBK, &img, &h);
#pragma unroll
            for (int i = 0; i < BN / 2 / 64; ++i) {
              const int n = min(n0 + 64 * i, g.N - 64);
              const int tap = n / g.conv_cin, c0 = n - tap * g.conv_cin;
              tma_load_5d_2sm(sb + i * 64 * kBK * 2, &tb, &full[s], c0, tap % 3 - 1, h + tap / 3 - 1, img, b);
            }
          } else if constexpr (CONV == kConvDgrad) {
            const int tap = k / g.conv_cpb, cb = k - tap * g.conv_cpb;
#pragma unroll
            for (int i = 0; i < BN / 2 / 64; ++i)
              tma_load_4d_2sm(sb + i * 64 * kBK * 2, &tb, &full[s], n0 + 64 * i, tap, cb * kBK, b);
          } else if constexpr (!B_MN) {
            tma_load_3d_2sm(sb, &tb, &full[s], k * kBK, n0, b);
          } else {
#pragma unroll
            for (int i = 0; i < BN / 2 / 64; ++i)
              tma_load_3d_2sm(sb + i * 64 * kBK * 2, &tb, &full[s], n0 + 64 * i, k * kBK, b);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // MMA issuer: the leader CTA only
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((A_MN ? 1u : 0u) << 15) |
                             ((B_MN ? 1u : 0u) << 16) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)((2 * kBM) >> 4) << 24);
      int it = 0, tc = 0;
      for (int tile = cid; tile < tiles; tile += ncl, ++tc) {
        const int acc = tc & 1;
        nn_mbar_wait_bounded(&tempty[acc], ((unsigned)(tc >> 1) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(acc * BN);
        for (int k = 0; k < nk; ++k, ++it) {
          const int s = it % Cfg::kStages;
          nn_mbar_wait_bounded(&full[s], (unsigned)(it / Cfg::kStages) & 1u);
          tc_fence_after();
          const unsigned sa = su32(smem + s * Cfg::kStage);
          const unsigned sb = sa + Cfg::kABytes;
#pragma unroll
          for (int kk = 0; kk < kBK / kUmmaK; ++kk) {
            const uint64_t ad = A_MN ? smem_desc(sa + kk * kUmmaK * 128, kBK * 128, 1024)
                                     : smem_desc(sa + kk * kUmmaK * 2, 16, 1024);
            const uint64_t bd = B_MN ? smem_desc(sb + kk * kUmmaK * 128, kBK * 128, 1024)
                                     : smem_desc(sb + kk * kUmmaK * 2, 16, 1024);
            tc2_mma(d, ad, bd, idesc, (k | kk) != 0 ? 1u : 0u);
          }
          tc2_commit_both(&empty[s]);  // frees the stage in both CTAs
        }
        tc2_commit_both(&tfull[acc]);  // both CTAs' accumulator halves ready
      }
    }
  } else {  // epilogue warps 2..5 of both CTAs
    const int q = warp & 3;
    float* st = epi_smem + (warp - 2) * 32 * 33;
    const bool ob = sizeof(TOut) == 2 && g.epi != kEpiF32 && (g.ldc & 1) == 0;
    uint32_t tempty_leader[2];
    for (int a = 0; a < 2; ++a)
      asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(tempty_leader[a]) : "r"(su32(&tempty[a])));
    int tc = 0;
    for (int tile = cid; tile < tiles; tile += ncl, ++tc) {
      int b, mb, nb;
      tile_coords(tile, mt, ntl, &b, &mb, &nb);
      const int m0 = mb * 2 * kBM + (int)rank * kBM + 32 * q, n0 = nb * BN;
      const int acc = tc & 1;
      nn_mbar_wait_bounded(&tfull[acc], (unsigned)(tc >> 1) & 1u);
      tc_fence_after();
      // bf16 dgrad: the ReLU' mask words of chunk c+1 load while chunk c drains
      const bool pre = ob && (g.epi == kEpiDRelu || g.epi == kEpiAdd) && (g.ldmask & 1) == 0;
      uint32_t mw_cur[16], mw_nxt[16];
      if (pre) load_mask_words<TOut>(g, b, m0, n0 + 2 * (lane & 15), lane, mw_cur);
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        if (n0 + c >= g.N) break;
        const bool more = pre && c + 32 < BN && n0 + c + 32 < g.N;
        if (more) load_mask_words<TOut>(g, b, m0, n0 + c + 32 + 2 * (lane & 15), lane, mw_nxt);
        epi_chunk<TOut>(g, tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(acc * BN + c), st, lane, b, m0, n0 + c, ob,
                        pre ? mw_cur : nullptr);
        if (more)
#pragma unroll
          for (int i = 0; i < 16; ++i) mw_cur[i] = mw_nxt[i];
      }
      tc_fence_before();
      if (lane == 0)
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(tempty_leader[acc])
                     : "memory");
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(Cfg::kTmemCols) : "memory");
  }
}

// ---------------------------------------------------------------------------
// fp32 SIMT GEMM (parity path): 64x64 tile, 256 threads, 4x4 per thread,
// K staged 16 at a time through shared memory; same operand majors and
// epilogues as the tensor-core kernel.
// ---------------------------------------------------------------------------
template <bool A_MN, bool B_MN>
__global__ void __launch_bounds__(256) gemm_f32_kernel(const float* __restrict__ A, long long lda, long long sA,
                                                       const float* __restrict__ B, long long ldb, long long sB,
                                                       GemmArgs g) {
  constexpr int T = 64, TK = 16;
  __shared__ float as[TK][T + 4];
  __shared__ float bs[TK][T + 4];
  const int b = blockIdx.z;
  const int m0 = blockIdx.y * T, n0 = blockIdx.x * T;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const float* Ab = A + (long long)b * sA;
  const float* Bb = B + (long long)b * sB;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < g.K; k0 += TK) {
    // 64x16 elements of each operand, 4 per thread
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = threadIdx.x + 256 * i;
      int mm, kk;
      if (A_MN) { kk = e >> 6; mm = e & 63; } else { mm = e >> 4; kk = e & 15; }
      const int gm = m0 + mm, gk = k0 + kk;
      float v = 0.f;
      if (gm < g.M && gk < g.K) v = A_MN ? Ab[(long long)gk * lda + gm] : Ab[(long long)gm * lda + gk];
      as[kk][mm] = v;
      int nn;
      if (B_MN) { kk = e >> 6; nn = e & 63; } else { nn = e >> 4; kk = e & 15; }
      const int gn = n0 + nn, gk2 = k0 + kk;
      float w = 0.f;
      if (gn < g.N && gk2 < g.K) w = B_MN ? Bb[(long long)gk2 * ldb + gn] : Bb[(long long)gn * ldb + gk2];
      bs[kk][nn] = w;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        av[i] = as[kk][ty + 16 * i];
        bv[i] = bs[kk][tx + 16 * i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int m = m0 + ty + 16 * i, n = n0 + tx + 16 * j;
      if (m < g.M && n < g.N) epi_store<float>(g, b, m, n, acc[i][j]);
    }
}

}  // namespace dsx_nn
