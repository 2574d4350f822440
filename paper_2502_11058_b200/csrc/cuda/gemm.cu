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

#include "device_once.cuh"
#include "dsx.h"
#include "dsx_nn.h"
#include "nn_gemm.cuh"

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

template <int BN, bool AM, bool BM_, typename TOut>
dsx_status launch_tc_t(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& g, cudaStream_t s) {
  static std::atomic<unsigned long long> attr{0};
  auto kern = gemm_tc_kernel<BN, AM, BM_, TOut>;
  dsx::once_per_device(attr, [&] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, TcCfg<BN>::kSmem);
  });
  // persistent: at most one CTA per SM (the smem ring holds the SM)
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const long long tiles = (long long)((g.N + BN - 1) / BN) * ((g.M + kBM - 1) / kBM) * g.batch;
  const int grid = (int)std::min<long long>(tiles, nsm);
  kern<<<grid, 192, TcCfg<BN>::kSmem, s>>>(ta, tb, g);
  NN_CUDA(cudaGetLastError());
  return DSX_OK;
}

// CTA-pair kernel: grid = 2 x clusters (compile-time cluster dims 2x1x1)
template <int BN, bool AM, bool BM_, typename TOut>
dsx_status launch_tc2_t(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& g, cudaStream_t s) {
  static std::atomic<unsigned long long> attr{0};
  auto kern = gemm_tc2_kernel<BN, AM, BM_, TOut>;
  dsx::once_per_device(attr, [&] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Tc2Cfg<BN>::kSmem);
  });
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const long long tiles = (long long)((g.N + BN - 1) / BN) * ((g.M + 2 * kBM - 1) / (2 * kBM)) * g.batch;
  const int clusters = (int)std::min<long long>(tiles, nsm / 2);
  kern<<<2 * clusters, 192, Tc2Cfg<BN>::kSmem, s>>>(ta, tb, g);
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

}  // namespace

dsx_status gemm(const GemmCall& c, cudaStream_t s, int nsm) {
  const GemmArgs& g = c.g;
  if (g.M <= 0 || g.N <= 0 || g.K <= 0 || g.batch <= 0) return DSX_OK;
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
  // (measured: 256-wide pairs 1290 -> 1431 TFLOP/s at 8192^3; 128-wide pairs
  // lose to single-CTA 128 tiles, so auto mode pairs only 256-wide tiles)
  const bool two_sm = bn >= 128 && two_sm_env != 0 &&
                      (two_sm_env == 1 || (bn == 256 && tiles2 >= nsm / 2));
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
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
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
  return gemm(c, static_cast<cudaStream_t>(d->stream), nsm);
}

}  // extern "C"
