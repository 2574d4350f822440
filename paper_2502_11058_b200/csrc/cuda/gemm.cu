// gemm.cu — launcher of the dense-layer GEMMs (nn_gemm.cuh): TMA tensor
// maps + tcgen05 kernel for bf16, SIMT kernel for fp32; dsx_gemm test hook.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "device_once.cuh"
#include "dsx.h"
#include "dsx_nn.h"
#include "nn_gemm.cuh"
#include "conv64.cuh"

namespace dsx {
extern thread_local std::string g_last_error;
}

namespace dsx_nn {


namespace {

dsx_status nfail(dsx_status code, const std::string& msg) {
  dsx::g_last_error = msg;
  return code;
}

#define NN_CUDA(expr)                                                                           \
  do {                                                                                          \
    cudaError_t e_ = (expr);                                                                    \
    if (e_ != cudaSuccess) return nfail(DSX_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)
#define NN_TRY(expr)              \
  do {                            \
    dsx_status s_ = (expr);       \
    if (s_ != DSX_OK) return s_;  \
  } while (0)

// ---------------------------------------------------------------------------
// TMA descriptors and GEMM launch
// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

dsx_status get_encoder() {
  if (g_encode) return DSX_OK;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  NN_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (q != cudaDriverEntryPointSuccess || !fn) return nfail(DSX_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return DSX_OK;
}

// 3-D bf16 view [batch][outer][inner] (inner contiguous), box {64, box_outer, 1}, 128-B swizzle
dsx_status make_map(CUtensorMap* map, const void* base, long long inner, long long outer, long long batch,
                    long long pitch, long long bstride, int box_outer) {
  NN_TRY(get_encoder());
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (pitch * 2) % 16 || (bstride * 2) % 16)
    return nfail(DSX_ERR_ARGUMENT, "gemm: bf16 operands need 16-B aligned base and strides");
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)outer, (cuuint64_t)batch};
  cuuint64_t strides[2] = {(cuuint64_t)(pitch * 2), (cuuint64_t)(std::max<long long>(bstride, pitch * outer) * 2)};
  if (bstride > 0) strides[1] = (cuuint64_t)(bstride * 2);
  cuuint32_t box[3] = {64, (cuuint32_t)box_outer, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return nfail(DSX_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return DSX_OK;
}

// bf16 C written by TMA stores (the CST epilogue): C, its strides and the
// ReLU' / residual operand must be 16-B aligned.  DSX_GEMM_TMA_STORE=0: off.
bool tma_store_ok(const GemmArgs& g) {
  static const bool on = [] {
    const char* e = std::getenv("DSX_GEMM_TMA_STORE");
    return !(e && e[0] == '0');
  }();
  if (!on || g.epi == kEpiF32 || (reinterpret_cast<uintptr_t>(g.C) & 15) || g.ldc % 8 || g.strideC % 8) return false;
  const auto aligned = [](const void* p, long long ld, long long sb) {
    return p && !(reinterpret_cast<uintptr_t>(p) & 15) && ld % 8 == 0 && sb % 8 == 0;
  };
  if (g.epi >= kEpiDRelu && !aligned(g.mask, g.ldmask, g.strideMask)) return false;
  if (g.epi == kEpiAddDRelu && !aligned(g.mask2, g.ldmask2, g.strideMask2)) return false;
  return true;
}

dsx_status make_c_map(CUtensorMap* map, const GemmArgs& g) {
  NN_TRY(get_encoder());
  cuuint64_t dims[3] = {(cuuint64_t)g.N, (cuuint64_t)g.M, (cuuint64_t)g.batch};
  cuuint64_t strides[2] = {(cuuint64_t)g.ldc * 2,
                           (cuuint64_t)std::max<long long>(g.strideC, g.ldc * (long long)g.M) * 2};
  cuuint32_t box[3] = {32, 32, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, g.C, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return nfail(DSX_ERR_CUDA, "cuTensorMapEncodeTiled(C) failed (" + std::to_string((int)r) + ")");
  return DSX_OK;
}

// fp32 C (kEpiF32, no accumulate) through TMA stores: 4-D map (n, m, batch
// entry, split), 16 x 32 boxes
bool tma_store_f32_ok(const GemmArgs& g) {
  static const bool on = [] {
    const char* e = std::getenv("DSX_GEMM_TMA_STORE");
    return !(e && e[0] == '0');
  }();
  const int ks = std::max(1, g.ksplit);
  return on && g.epi == kEpiF32 && !g.accumulate && !(reinterpret_cast<uintptr_t>(g.C) & 15) && g.ldc % 4 == 0 &&
         g.strideC % 4 == 0 && (ks == 1 || g.strideSplit % 4 == 0);
}

dsx_status make_c_map_f32(CUtensorMap* map, const GemmArgs& g) {
  NN_TRY(get_encoder());
  const int ks = std::max(1, g.ksplit);
  const long long sc = std::max<long long>(g.strideC, g.ldc * (long long)g.M);
  cuuint64_t dims[4] = {(cuuint64_t)g.N, (cuuint64_t)g.M, (cuuint64_t)g.batch, (cuuint64_t)ks};
  cuuint64_t strides[3] = {(cuuint64_t)g.ldc * 4, (cuuint64_t)sc * 4,
                           (cuuint64_t)std::max<long long>(g.strideSplit, sc * g.batch) * 4};
  cuuint32_t box[4] = {16, 32, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, g.C, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return nfail(DSX_ERR_CUDA, "cuTensorMapEncodeTiled(C fp32) failed (" + std::to_string((int)r) + ")");
  return DSX_OK;
}

template <int BN, bool AM, bool BM_, typename TOut, int CONV = kConvNone>
dsx_status launch_tc_t(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& g, cudaStream_t s) {
  if constexpr (std::is_same_v<TOut, float>) {
    if (tma_store_f32_ok(g)) {
      static std::atomic<unsigned long long> attr_c{0};
      auto kc = gemm_tc_kernel<BN, AM, BM_, TOut, CONV, true>;
      dsx::once_per_device(attr_c, [&] {
        cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, TcCfg<BN, 8>::kSmem);
      });
      CUtensorMap tcm;
      NN_TRY(make_c_map_f32(&tcm, g));
      int dev = 0, nsm = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      const long long tiles =
          (long long)((g.N + BN - 1) / BN) * ((g.M + kBM - 1) / kBM) * g.batch * std::max(1, g.ksplit);
      NN_CUDA(launch_pdl(kc, (int)std::min<long long>(tiles, nsm), TcCfg<BN, 8>::kThreads, TcCfg<BN, 8>::kSmem, s, ta, tb, g, tcm));
      NN_CUDA(cudaGetLastError());
      return DSX_OK;
    }
  }
  if constexpr (std::is_same_v<TOut, __nv_bfloat16>) {
    if (tma_store_ok(g)) {
      static std::atomic<unsigned long long> attr_c{0};
      auto kc = gemm_tc_kernel<BN, AM, BM_, TOut, CONV, true>;
      dsx::once_per_device(attr_c, [&] {
        cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, TcCfg<BN, 8>::kSmem);
      });
      CUtensorMap tcm;
      NN_TRY(make_c_map(&tcm, g));
      int dev = 0, nsm = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      const long long tiles =
          (long long)((g.N + BN - 1) / BN) * ((g.M + kBM - 1) / kBM) * g.batch * std::max(1, g.ksplit);
      NN_CUDA(launch_pdl(kc, (int)std::min<long long>(tiles, nsm), TcCfg<BN, 8>::kThreads, TcCfg<BN, 8>::kSmem, s, ta, tb, g, tcm));
      NN_CUDA(cudaGetLastError());
      return DSX_OK;
    }
  }
  if (g.epi >= kEpiBiasAddAct)
    return nfail(DSX_ERR_ARGUMENT, "gemm: fused residual epilogues need a bf16, 16-B aligned C and operands");
  static std::atomic<unsigned long long> attr{0};
  auto kern = gemm_tc_kernel<BN, AM, BM_, TOut, CONV>;
  dsx::once_per_device(attr, [&] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, TcCfg<BN>::kSmem);
  });
  // persistent: at most one CTA per SM (the smem ring holds the SM)
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const long long tiles =
      (long long)((g.N + BN - 1) / BN) * ((g.M + kBM - 1) / kBM) * g.batch * std::max(1, g.ksplit);
  const int grid = (int)std::min<long long>(tiles, nsm);
  CUtensorMap unused{};
  NN_CUDA(launch_pdl(kern, grid, 192, TcCfg<BN>::kSmem, s, ta, tb, g, unused));
  NN_CUDA(cudaGetLastError());
  return DSX_OK;
}

// CTA-pair kernel: grid = 2 x clusters (compile-time cluster dims 2x1x1)
template <int BN, bool AM, bool BM_, typename TOut, int CONV = kConvNone>
dsx_status launch_tc2_t(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& g, cudaStream_t s) {
  static std::atomic<unsigned long long> attr{0};
  auto kern = gemm_tc2_kernel<BN, AM, BM_, TOut, CONV>;
  dsx::once_per_device(attr, [&] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Tc2Cfg<BN>::kSmem);
  });
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const long long tiles = (long long)((g.N + BN - 1) / BN) * ((g.M + 2 * kBM - 1) / (2 * kBM)) * g.batch;
  const int clusters = (int)std::min<long long>(tiles, nsm / 2);
  NN_CUDA(launch_pdl(kern, 2 * clusters, 192, Tc2Cfg<BN>::kSmem, s, ta, tb, g));
  NN_CUDA(cudaGetLastError());
  return DSX_OK;
}

template <int BN>
dsx_status launch_tc2_bn(bool am, bool bm, bool ob, const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& g,
                         cudaStream_t s) {
  if (!am && !bm) return ob ? launch_tc2_t<BN, false, false, __nv_bfloat16>(ta, tb, g, s)
                            : launch_tc2_t<BN, false, false, float>(ta, tb, g, s);
  if (!am && bm) return ob ? launch_tc2_t<BN, false, true, __nv_bfloat16>(ta, tb, g, s)
                           : launch_tc2_t<BN, false, true, float>(ta, tb, g, s);
  if (am && bm && !ob) return launch_tc2_t<BN, true, true, float>(ta, tb, g, s);
  return nfail(DSX_ERR_ARGUMENT, "gemm: unsupported operand-major / output combination for the tensor-core path");
}

// the operand-major / output-type combinations the Linear layers use:
// forward (K,K) -> bf16 activations or fp32 logits, dgrad (K,N) -> bf16,
// wgrad (M,N) -> fp32 dW
template <int BN>
dsx_status launch_tc_bn(bool am, bool bm, bool ob, const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& g,
                        cudaStream_t s) {
  if (!am && !bm) return ob ? launch_tc_t<BN, false, false, __nv_bfloat16>(ta, tb, g, s)
                            : launch_tc_t<BN, false, false, float>(ta, tb, g, s);
  if (!am && bm) return ob ? launch_tc_t<BN, false, true, __nv_bfloat16>(ta, tb, g, s)
                           : launch_tc_t<BN, false, true, float>(ta, tb, g, s);
  if (am && bm && !ob) return launch_tc_t<BN, true, true, float>(ta, tb, g, s);
  return nfail(DSX_ERR_ARGUMENT, "gemm: unsupported operand-major / output combination for the tensor-core path");
}

int pick_bn(const GemmArgs& g, int nsm) {
  // widest tile that still gives about one wave of CTAs
  const long long mt = (g.M + kBM - 1) / kBM;
  // widest tile that still fills every SM; small GEMMs take the narrowest
  // (most CTAs in flight)
  for (int bn : {256, 128}) {
    const long long ctas = mt * ((g.N + bn - 1) / bn) * g.batch;
    if (g.N >= bn && ctas >= nsm) return bn;
  }
  return 64;
}

// 5-D activation view (c, w, h, image, worker) of an NHWC tensor whose
// workers sit `wstride` elements apart; a box covers `pix` consecutive
// pixels = whole rows of one image, or whole images
dsx_status make_act_map(CUtensorMap* map, const void* base, int C, int W, int H, int B, int batch, long long wstride,
                        int pix, int stride = 1) {
  NN_TRY(get_encoder());
  if ((reinterpret_cast<uintptr_t>(base) & 15) || C % 64 || (wstride * 2) % 16)
    return nfail(DSX_ERR_ARGUMENT, "conv: activations need 16-B aligned base/stride and 64-channel multiples");
  // the box covers `pix` OUTPUT pixels; with stride 2 it traverses every
  // second input row / column (element strides), i.e. 2x the extent
  const int Wo = W / stride, Ho = H / stride;
  int rows = Ho, imgs = 1;
  if (Ho * Wo >= pix) {
    if (pix % Wo) return nfail(DSX_ERR_ARGUMENT, "conv: tile pixels must cover whole image rows");
    rows = pix / Wo;
  } else {
    if (pix % (Ho * Wo)) return nfail(DSX_ERR_ARGUMENT, "conv: tile pixels must cover whole images");
    imgs = pix / (Ho * Wo);
  }
  cuuint64_t dims[5] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)B, (cuuint64_t)batch};
  cuuint64_t strides[4] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2,
                           (cuuint64_t)wstride * 2};
  cuuint32_t box[5] = {64, (cuuint32_t)(Wo * stride), (cuuint32_t)(rows * stride), (cuuint32_t)imgs, 1};
  cuuint32_t es[5] = {1, (cuuint32_t)stride, (cuuint32_t)stride, 1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    std::string d = "cuTensorMapEncodeTiled(5-D) failed (" + std::to_string((int)r) + "): dims";
    for (auto v : dims) d += " " + std::to_string((unsigned long long)v);
    d += " strides";
    for (auto v : strides) d += " " + std::to_string((unsigned long long)v);
    d += " box";
    for (auto v : box) d += " " + std::to_string(v);
    d += " base " + std::to_string(reinterpret_cast<uintptr_t>(base));
    return nfail(DSX_ERR_CUDA, d);
  }
  return DSX_OK;
}

// 4-D view (c, tap, o, worker) of 3x3 weights W[o][tap][c], workers `wstride` apart
dsx_status make_tap_map(CUtensorMap* map, const void* base, int cin, int cout, int batch, long long wstride) {
  NN_TRY(get_encoder());
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (wstride * 2) % 16 || cin % 64)
    return nfail(DSX_ERR_ARGUMENT, "conv: weights need 16-B aligned base/stride and 64-channel multiples");
  cuuint64_t dims[4] = {(cuuint64_t)cin, 9, (cuuint64_t)cout, (cuuint64_t)batch};
  cuuint64_t strides[3] = {(cuuint64_t)cin * 2, (cuuint64_t)9 * cin * 2, (cuuint64_t)wstride * 2};
  cuuint32_t box[4] = {64, 1, 64, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return nfail(DSX_ERR_CUDA, "cuTensorMapEncodeTiled(4-D) failed (" + std::to_string((int)r) + ")");
  return DSX_OK;
}

template <int MODE>
dsx_status launch_conv_bn(int bn, bool two_sm, const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& g,
                          cudaStream_t s) {
  if constexpr (MODE == kConvWgradT) {
    if (bn != 64) return nfail(DSX_ERR_ARGUMENT, "conv_gemm: the transposed wgrad runs 64-wide tiles");
    return launch_tc_t<64, true, true, float, kConvWgradT>(ta, tb, g, s);
  }
  constexpr bool AM = MODE == kConvWgrad, BM_ = MODE != kConvFwd;
  using T = std::conditional_t<MODE == kConvWgrad, float, __nv_bfloat16>;
  if (two_sm) return bn == 128 ? launch_tc2_t<128, AM, BM_, T, MODE>(ta, tb, g, s)
                               : launch_tc2_t<256, AM, BM_, T, MODE>(ta, tb, g, s);
  switch (bn) {
    case 64: return launch_tc_t<64, AM, BM_, T, MODE>(ta, tb, g, s);
    case 128: return launch_tc_t<128, AM, BM_, T, MODE>(ta, tb, g, s);
    default: return launch_tc_t<256, AM, BM_, T, MODE>(ta, tb, g, s);
  }
}

}  // namespace

dsx_status conv_gemm(const GemmCall& c, const ConvGeom& q, cudaStream_t s, int nsm) {
  GemmArgs g = c.g;
  if (!c.bf16) return nfail(DSX_ERR_ARGUMENT, "conv_gemm: tensor-core (bf16) path only");
  const int st = q.stride > 1 ? q.stride : 1, kk = q.k == 1 ? 1 : 3;
  const int Ho = q.H / st, Wo = q.W / st;
  if (Wo > 64 || 64 % Wo || q.cin % 64 || q.cout % 64 || (st != 1 && st != 2) || q.H % st || q.W % st)
    return nfail(DSX_ERR_ARGUMENT, "conv_gemm: needs W_out | 64, 64-channel multiples, stride 1 or 2");
  if ((st != 1 || kk != 3) && (q.mode == kConvDgrad || (kk == 1 && st == 1)))
    return nfail(DSX_ERR_ARGUMENT, "conv_gemm: strided / 1x1 convs: forward and wgrad only (stride 2)");
  g.conv_h = Ho;
  g.conv_w = Wo;
  g.conv_cin = q.cin;
  g.conv_stride = st;
  g.conv_k = kk;
  const int pixels = q.B * Ho * Wo;
  CUtensorMap ta, tb;
  if (q.mode == kConvFwd) {
    g.M = pixels, g.N = q.cout, g.K = kk * kk * q.cin, g.conv_cpb = q.cin / 64;
    NN_TRY(make_act_map(&ta, c.A, q.cin, q.W, q.H, q.B, g.batch, c.sA, kBM, st));
  } else if (q.mode == kConvWgrad) {
    g.M = q.cout, g.N = kk * kk * q.cin, g.K = pixels;
    NN_TRY(make_map(&ta, c.A, g.M, g.K, g.batch, c.lda, c.sA, kBK));
    NN_TRY(make_act_map(&tb, c.B, q.cin, q.W, q.H, q.B, g.batch, c.sB, kBK, st));
  } else if (q.mode == kConvWgradT) {
    // dW^T[(tap,c)][o]: A = x (implicit, MN-major), B = dy (MN-major)
    g.M = kk * kk * q.cin, g.N = q.cout, g.K = pixels;
    NN_TRY(make_act_map(&ta, c.A, q.cin, q.W, q.H, q.B, g.batch, c.sA, kBK, st));
    NN_TRY(make_map(&tb, c.B, g.N, g.K, g.batch, c.ldb, c.sB, kBK));
  } else if (q.mode == kConvDgrad) {
    g.M = pixels, g.N = q.cin, g.K = 9 * q.cout, g.conv_cpb = q.cout / 64;
    NN_TRY(make_act_map(&ta, c.A, q.cout, q.W, q.H, q.B, g.batch, c.sA, kBM));
    NN_TRY(make_tap_map(&tb, c.B, q.cin, q.cout, g.batch, c.sB));
  } else {
    return nfail(DSX_ERR_ARGUMENT, "conv_gemm: bad mode");
  }
  if (g.ksplit > 1) {
    if ((q.mode != kConvWgrad && q.mode != kConvWgradT) || g.epi != kEpiF32 || g.accumulate)
      return nfail(DSX_ERR_ARGUMENT, "conv_gemm: split-K only for the fp32 wgrad");
    const int nk = (g.K + kBK - 1) / kBK;
    const int kper = (nk + g.ksplit - 1) / g.ksplit;
    g.ksplit = (nk + kper - 1) / kper;
  }
  // 64-in / 64-out 3x3 stride-1 convs on 32x32 / 16x16 images: the resident-
  // weight, halo-staged kernel (conv64.cuh).  DSX_CONV64=0: general path.
  static const bool c64_ok = [] {
    const char* e = std::getenv("DSX_CONV64");
    return !(e && e[0] == '0');
  }();
  if (c64_ok && (q.mode == kConvFwd || q.mode == kConvDgrad) && st == 1 && kk == 3 && q.cin == 64 && q.cout == 64 &&
      (q.W == 32 || q.W == 16) && q.H >= kBM / q.W + 2 && tma_store_ok(g) && c.bn == 0) {
    CUtensorMap tcm;
    NN_TRY(make_act_map(&ta, c.A, 64, q.W, q.H, q.B, g.batch, c.sA, (kBM / q.W + 2) * q.W));
    if (q.mode == kConvFwd) NN_TRY(make_map(&tb, c.B, g.K, g.N, g.batch, c.ldb, c.sB, 64));
    NN_TRY(make_c_map(&tcm, g));
    static std::atomic<unsigned long long> attr{0};
    auto kf = conv64_kernel<kConvFwd>;
    auto kd = conv64_kernel<kConvDgrad>;
    dsx::once_per_device(attr, [&] {
      cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, Conv64Cfg::kSmem);
      cudaFuncSetAttribute(kd, cudaFuncAttributeMaxDynamicSharedMemorySize, Conv64Cfg::kSmem);
    });
    const long long tiles = (long long)((g.M + kBM - 1) / kBM) * g.batch;
    const int grid = (int)std::min<long long>(tiles, nsm);
    constexpr int threads = 64 + 32 * Conv64Cfg::kEpiWarps;
    if (q.mode == kConvFwd) NN_CUDA(launch_pdl(kf, grid, threads, Conv64Cfg::kSmem, s, ta, tb, g, tcm));
    else NN_CUDA(launch_pdl(kd, grid, threads, Conv64Cfg::kSmem, s, ta, tb, g, tcm));
    NN_CUDA(cudaGetLastError());
    return DSX_OK;
  }
  const int bn = c.bn ? c.bn : pick_bn(g, nsm);
  if (bn != 64 && bn != 128 && bn != 256) return nfail(DSX_ERR_ARGUMENT, "conv_gemm: bn must be 64, 128 or 256");
  // CTA pairs (M = 256 MMAs; each SM loads half of B): DSX_CONV_2SM=1.
  // Off by default: measured 12.73 vs 12.61 ms per ResNet-18 step (pairs
  // halve the weight traffic, but these short-K tiles are not B-bound).
  static const bool pairs_ok = [] {
    const char* e = std::getenv("DSX_CONV_2SM");
    return e && e[0] == '1';
  }();
  const long long tiles2 = (long long)((g.N + bn - 1) / bn) * ((g.M + 2 * kBM - 1) / (2 * kBM)) * g.batch;
  const bool two_sm = pairs_ok && bn >= 128 && g.ksplit <= 1 && g.M >= 2 * kBM && tiles2 >= nsm / 2 &&
                      g.epi < kEpiBiasAddAct;
  if (q.mode == kConvFwd) {
    NN_TRY(make_map(&tb, c.B, g.K, g.N, g.batch, c.ldb, c.sB, two_sm ? bn / 2 : bn));
    return launch_conv_bn<kConvFwd>(bn, two_sm, ta, tb, g, s);
  }
  if (q.mode == kConvWgrad) return launch_conv_bn<kConvWgrad>(bn, two_sm, ta, tb, g, s);
  if (q.mode == kConvWgradT) return launch_conv_bn<kConvWgradT>(64, false, ta, tb, g, s);
  return launch_conv_bn<kConvDgrad>(bn, two_sm, ta, tb, g, s);
}

dsx_status gemm(const GemmCall& c, cudaStream_t s, int nsm) {
  GemmArgs g = c.g;
  if (g.M <= 0 || g.N <= 0 || g.K <= 0 || g.batch <= 0) return DSX_OK;
  if (g.ksplit > 1) {
    if (!c.bf16 || g.epi != kEpiF32 || g.accumulate)
      return nfail(DSX_ERR_ARGUMENT, "gemm: split-K needs the tensor-core path, fp32 output, no accumulate");
    const int nk = (g.K + kBK - 1) / kBK;
    const int kper = (nk + g.ksplit - 1) / g.ksplit;
    g.ksplit = (nk + kper - 1) / kper;  // every split non-empty
  }
  if (!c.bf16) {
    dim3 grid((g.N + 63) / 64, (g.M + 63) / 64, g.batch);
    const float* A = static_cast<const float*>(c.A);
    const float* B = static_cast<const float*>(c.B);
    if (!c.a_mn && !c.b_mn) gemm_f32_kernel<false, false><<<grid, 256, 0, s>>>(A, c.lda, c.sA, B, c.ldb, c.sB, g);
    else if (!c.a_mn && c.b_mn) gemm_f32_kernel<false, true><<<grid, 256, 0, s>>>(A, c.lda, c.sA, B, c.ldb, c.sB, g);
    else if (c.a_mn && !c.b_mn) gemm_f32_kernel<true, false><<<grid, 256, 0, s>>>(A, c.lda, c.sA, B, c.ldb, c.sB, g);
    else gemm_f32_kernel<true, true><<<grid, 256, 0, s>>>(A, c.lda, c.sA, B, c.ldb, c.sB, g);
    NN_CUDA(cudaGetLastError());
    return DSX_OK;
  }
  const int bn = c.bn ? c.bn : pick_bn(g, nsm);
  if (bn != 64 && bn != 128 && bn != 256) return nfail(DSX_ERR_ARGUMENT, "gemm: bn must be 64, 128 or 256");
  const bool ob2 = c.out_bf16 && g.epi != kEpiF32;
  // CTA pairs (M=256 MMAs, half the B traffic per SM) once there are enough
  // 256-row tiles to give every SM pair one; DSX_GEMM_2SM=0 turns them off,
  // =1 forces them (tests)
  static const int two_sm_env = [] {
    const char* e = std::getenv("DSX_GEMM_2SM");
    return e ? std::atoi(e) : -1;
  }();
  const long long tiles2 = (long long)((g.N + bn - 1) / bn) * ((g.M + 2 * kBM - 1) / (2 * kBM)) * g.batch;
  // (measured: 256-wide pairs 1290 -> 1431 TFLOP/s at 8192^3 with fp32 C;
  // 128-wide pairs lose to single-CTA 128 tiles; bf16 C goes through the
  // single-CTA TMA-store epilogue, which beats the pairs: wide MLP 126.5 ->
  // 129.8 it/s, ResNet-18 step 10.06 -> 9.26 ms — so auto mode pairs only
  // 256-wide fp32-output tiles)
  // fp32 C with MN-major operands (the wgrads) likewise takes the
  // single-CTA TMA-store kernel (wide wgrad 704 -> 1283 TFLOP/s); K-major
  // fp32-output GEMMs keep the pairs (8192^3: 1420 vs 1229)
  const bool cst = c.out_bf16 ? tma_store_ok(g) : (tma_store_f32_ok(g) && (c.a_mn || c.b_mn));
  const bool two_sm = bn >= 128 && two_sm_env != 0 && g.ksplit <= 1 && g.epi < kEpiBiasAddAct &&
                      (two_sm_env == 1 || (bn == 256 && !cst && tiles2 >= nsm / 2));
  CUtensorMap ta, tb;
  if (two_sm) {
    if (!c.a_mn) NN_TRY(make_map(&ta, c.A, g.K, g.M, g.batch, c.lda, c.sA, kBM));
    else NN_TRY(make_map(&ta, c.A, g.M, g.K, g.batch, c.lda, c.sA, kBK));
    if (!c.b_mn) NN_TRY(make_map(&tb, c.B, g.K, g.N, g.batch, c.ldb, c.sB, bn / 2));
    else NN_TRY(make_map(&tb, c.B, g.N, g.K, g.batch, c.ldb, c.sB, kBK));
    return bn == 128 ? launch_tc2_bn<128>(c.a_mn, c.b_mn, ob2, ta, tb, g, s)
                     : launch_tc2_bn<256>(c.a_mn, c.b_mn, ob2, ta, tb, g, s);
  }
  if (!c.a_mn) NN_TRY(make_map(&ta, c.A, g.K, g.M, g.batch, c.lda, c.sA, kBM));
  else NN_TRY(make_map(&ta, c.A, g.M, g.K, g.batch, c.lda, c.sA, kBK));
  if (!c.b_mn) NN_TRY(make_map(&tb, c.B, g.K, g.N, g.batch, c.ldb, c.sB, bn));
  else NN_TRY(make_map(&tb, c.B, g.N, g.K, g.batch, c.ldb, c.sB, kBK));
  const bool ob = c.out_bf16 && g.epi != kEpiF32;
  switch (bn) {
    case 64: return launch_tc_bn<64>(c.a_mn, c.b_mn, ob, ta, tb, g, s);
    case 128: return launch_tc_bn<128>(c.a_mn, c.b_mn, ob, ta, tb, g, s);
    default: return launch_tc_bn<256>(c.a_mn, c.b_mn, ob, ta, tb, g, s);
  }
}


}  // namespace dsx_nn

using namespace dsx_nn;

extern "C" {

dsx_status dsx_gemm(const dsx_gemm_desc* d) {
  if (!d) return nfail(DSX_ERR_ARGUMENT, "null gemm desc");
  if (d->dtype != DSX_BF16 && d->dtype != DSX_F32) return nfail(DSX_ERR_ARGUMENT, "gemm dtype");
  // run on the device that owns C (not whatever device an earlier call on
  // this thread left current: a launch there would reach C over peer
  // access, unordered with the owner's default stream)
  int prev = 0, dev = 0, nsm = 148;
  cudaGetDevice(&prev);
  dev = prev;
  cudaPointerAttributes pa{};
  if (d->C && cudaPointerGetAttributes(&pa, d->C) == cudaSuccess && pa.type == cudaMemoryTypeDevice) dev = pa.device;
  cudaGetLastError();
  if (dev != prev) NN_CUDA(cudaSetDevice(dev));
  struct Restore {
    int prev, dev;
    ~Restore() {
      if (dev != prev) cudaSetDevice(prev);
    }
  } restore{prev, dev};
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  GemmCall c{};
  c.bf16 = d->dtype == DSX_BF16;
  c.a_mn = d->a_mn != 0;
  c.b_mn = d->b_mn != 0;
  c.A = d->A;
  c.lda = d->lda;
  c.sA = d->strideA;
  c.B = d->B;
  c.ldb = d->ldb;
  c.sB = d->strideB;
  c.out_bf16 = d->out_dtype == DSX_BF16;
  c.bn = d->bn;
  c.g.ksplit = d->ksplit;
  c.g.strideSplit = d->strideSplit;
  c.g.mask2 = d->mask2;
  c.g.ldmask2 = d->ldmask2;
  c.g.strideMask2 = d->strideMask2;
  c.g.M = d->M;
  c.g.N = d->N;
  c.g.K = d->K;
  c.g.batch = d->batch;
  c.g.epi = d->epi;
  c.g.relu = d->relu;
  c.g.accumulate = d->accumulate;
  c.g.C = d->C;
  c.g.ldc = d->ldc;
  c.g.strideC = d->strideC;
  c.g.bias = d->bias;
  c.g.strideBias = d->strideBias;
  c.g.mask = d->mask;
  c.g.ldmask = d->ldmask;
  c.g.strideMask = d->strideMask;
  if (!c.bf16 && c.out_bf16) return nfail(DSX_ERR_ARGUMENT, "fp32 gemm writes fp32");
  if (d->conv) {
    ConvGeom q{d->conv, d->conv_h, d->conv_w, d->conv_images, d->conv_cin, d->conv_cout};
    q.stride = d->conv_stride > 1 ? d->conv_stride : 1;
    q.k = d->conv_k == 1 ? 1 : 3;
    return conv_gemm(c, q, static_cast<cudaStream_t>(d->stream), nsm);
  }
  return gemm(c, static_cast<cudaStream_t>(d->stream), nsm);
}

}  // extern "C"
