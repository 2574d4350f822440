// cnn.cu — BASELINE configs[1] as a real network: a K-worker ResNet-18-shaped
// conv stack (CIFAR geometry: 32x32 inputs, 3x3 stem, four stages of two
// basic blocks, widths w0..8w0, stride-2 1x1 projection shortcuts, global
// average pool, linear head; no normalisation layers) trained with DreamDDP's
// scheduled partial synchronisation (include/dsx_nn.h, dsx_cnn_*).
//
// Every convolution is an implicit-GEMM pass over the layer GEMMs of
// nn_gemm.cuh (tcgen05/TMA bf16 or fp32 SIMT):
//   forward  col = im2col(x) [B*Ho*Wo][k*k*Cin];  y = act(col W^T + b)
//   wgrad    dW = dy^T col          (A = dy M-major, B = col N-major)
//   dgrad    dcol = dy W            (B = W N-major)  ->  dx = col2im(dcol)
// with the ReLU' masks and the residual sums fused into the col2im gather.
// Registered layers (1-based, input side first, forward order) are the 20
// convolutions and the head; BP visits them in descending order (a block's
// shortcut, second conv, first conv), each layer's optimizer runs right after
// its gradients and a scheduled layer's average starts on the side stream.
//
// Layout (one rank, kl local workers), activations NHWC in T (bf16 / fp32):
//   params/grads/mom/var fp32 [kl][P], pbf bf16 [kl][P]: layer l = W_l
//   [Cout][k*k*Cin] ((kh, kw, c) order) then b_l [Cout], 64-element aligned
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "dsx.h"
#include "dsx_nn.h"
#include "nn_gemm.cuh"
#include "nn_kernels.cuh"

namespace dsx {
extern thread_local std::string g_last_error;
}

namespace dsx_nn {
namespace {

dsx_status cfail(dsx_status code, const std::string& msg) {
  dsx::g_last_error = msg;
  return code;
}

#define CN_CUDA(expr)                                                                            \
  do {                                                                                           \
    cudaError_t e_ = (expr);                                                                     \
    if (e_ != cudaSuccess) return cfail(DSX_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)
#define CN_NCCL(expr)                                                                            \
  do {                                                                                           \
    ncclResult_t r_ = (expr);                                                                    \
    if (r_ != ncclSuccess) return cfail(DSX_ERR_NCCL, std::string(#expr) + ": " + ncclGetErrorString(r_)); \
  } while (0)
#define CN_TRY(expr)              \
  do {                            \
    dsx_status s_ = (expr);       \
    if (s_ != DSX_OK) return s_;  \
  } while (0)

// 8 consecutive elements (16 B in bf16, 32 B in fp32)
template <typename T>
struct Vec8 {
  uint4 u[sizeof(T) * 8 / 16];
};
template <typename T>
__device__ __forceinline__ Vec8<T> ld8(const T* p) {
  Vec8<T> v;
#pragma unroll
  for (int i = 0; i < (int)(sizeof(T) * 8 / 16); ++i) v.u[i] = reinterpret_cast<const uint4*>(p)[i];
  return v;
}
template <typename T>
__device__ __forceinline__ void st8(T* p, const Vec8<T>& v) {
#pragma unroll
  for (int i = 0; i < (int)(sizeof(T) * 8 / 16); ++i) reinterpret_cast<uint4*>(p)[i] = v.u[i];
}
template <typename T>
__device__ __forceinline__ float el(const Vec8<T>& v, int j) {
  return to_f<T>(reinterpret_cast<const T*>(&v)[j]);
}
template <typename T>
__device__ __forceinline__ void set_el(Vec8<T>& v, int j, float x) {
  reinterpret_cast<T*>(&v)[j] = from_f<T>(x);
}

// im2col, 8 channels per thread: col[(b,ho,wo)][(kh,kw,c)] = x[b][hi][wi][c]
// (0 outside the image); blockIdx.y = local worker
template <typename T>
__global__ void im2col_kernel(const T* __restrict__ x, T* __restrict__ col, int B, int H, int W, int C, int Ho, int Wo,
                              int k, int stride, int pad, long long sx, long long scol) {
  pdl_enter();
  const int cv = C / 8;
  const long long Kc = (long long)k * k * C;
  const int total = B * Ho * Wo * k * k * cv;  // < 2^31 (host-checked): 32-bit index math
  const T* xw = x + blockIdx.y * sx;
  T* cw = col + blockIdx.y * scol;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    int t = idx;
    const int c8 = t % cv;
    t /= cv;
    const int kw = t % k;
    t /= k;
    const int kh = t % k;
    t /= k;
    const int wo = t % Wo;
    t /= Wo;
    const int ho = t % Ho;
    const int b = t / Ho;
    const int hi = ho * stride - pad + kh, wi = wo * stride - pad + kw;
    T* dst = cw + ((long long)(b * Ho + ho) * Wo + wo) * Kc + (long long)(kh * k + kw) * C + c8 * 8;
    Vec8<T> v;
    if (hi >= 0 && hi < H && wi >= 0 && wi < W) {
      v = ld8(xw + (((long long)b * H + hi) * W + wi) * C + c8 * 8);
    } else {
#pragma unroll
      for (int i = 0; i < (int)(sizeof(T) * 8 / 16); ++i) v.u[i] = make_uint4(0, 0, 0, 0);
    }
    st8(dst, v);
  }
}

// col2im as a gather (no atomics, fixed order): dx[b][hi][wi][c] = sum over
// the taps (kh, kw) whose output pixel exists of dcol[(b,ho,wo)][(kh,kw,c)];
// then + add[...] (the other branch of a residual sum) and * (mask > 0)
// (ReLU' of the tensor this gradient belongs to), both optional.
template <typename T>
__global__ void col2im_kernel(const T* __restrict__ dcol, T* __restrict__ dx, int B, int H, int W, int C, int Ho,
                              int Wo, int k, int stride, int pad, const T* __restrict__ add,
                              const T* __restrict__ mask, long long sdcol, long long sx,
                              const T* __restrict__ sub2) {
  pdl_enter();
  // 32-bit index math (the host keeps B*H*W*C/8 < 2^31): 64-bit divisions
  // had made this gather 7x slower than its bytes
  const int cv = C / 8;
  const long long Kc = (long long)k * k * C;
  const int total = B * H * W * cv;
  const T* dcw = dcol + blockIdx.y * sdcol;
  T* dxw = dx + blockIdx.y * sx;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    int t = idx;
    const int c8 = t % cv;
    t /= cv;
    const int wi = t % W;
    t /= W;
    const int hi = t % H;
    const int b = t / H;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int kh = 0; kh < k; ++kh) {
      const int hs = hi + pad - kh;
      if (hs < 0 || hs % stride) continue;
      const int ho = hs / stride;
      if (ho >= Ho) continue;
      for (int kw = 0; kw < k; ++kw) {
        const int ws = wi + pad - kw;
        if (ws < 0 || ws % stride) continue;
        const int wo = ws / stride;
        if (wo >= Wo) continue;
        const Vec8<T> v = ld8(dcw + ((long long)(b * Ho + ho) * Wo + wo) * Kc + (long long)(kh * k + kw) * C + c8 * 8);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += el(v, j);
      }
    }
    const long long o = (((long long)b * H + hi) * W + wi) * C + c8 * 8;
    if (sub2 && !(hi & 1) && !(wi & 1)) {  // a 1x1 stride-2 projection's dgrad [B][H/2][W/2][C]
      const Vec8<T> a = ld8(sub2 + blockIdx.y * sx + (((long long)b * (H >> 1) + (hi >> 1)) * (W >> 1) + (wi >> 1)) * C +
                            c8 * 8);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += el(a, j);
    }
    if (add) {
      const Vec8<T> a = ld8(add + blockIdx.y * sx + o);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += el(a, j);
    }
    if (mask) {
      const Vec8<T> mk = ld8(mask + blockIdx.y * sx + o);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = el(mk, j) > 0.f ? acc[j] : 0.f;
    }
    Vec8<T> out;
#pragma unroll
    for (int j = 0; j < 8; ++j) set_el(out, j, acc[j]);
    st8(dxw + o, out);
  }
}

// Column sums of rows [chunk*chunk_rows, +chunk_rows) of dz[b] (C columns,
// C % 8 == 0, C <= 2048): part[(chunk * kl + b) * C + c].  Each thread sums
// 8 columns of every rows_par-th row; the row groups combine in a fixed order.
template <typename T>
__global__ void __launch_bounds__(256) colsum_part_kernel(const T* __restrict__ dz, long long ld, long long s_dz,
                                                          int rows, int C, int chunk_rows, float* __restrict__ part) {
  pdl_enter();
  __shared__ float sh[2048];
  const int b = blockIdx.y;
  const int tpr = C / 8, rows_par = max(1, 256 / tpr);
  const int r_off = threadIdx.x / tpr, cv = threadIdx.x % tpr;
  const int r0 = blockIdx.x * chunk_rows, r1 = min(rows, r0 + chunk_rows);
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  const bool active = r_off < rows_par && tpr <= 256;
  if (active) {
    const T* p = dz + b * s_dz + cv * 8;
    int r = r0 + r_off;
    for (; r + 3 * rows_par < r1; r += 4 * rows_par) {  // 4 rows in flight, summed in row order
      Vec8<T> v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = ld8(p + (long long)(r + u * rows_par) * ld);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += el(v[u], j);
    }
    for (; r < r1; r += rows_par) {
      const Vec8<T> v = ld8(p + (long long)r * ld);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += el(v, j);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) sh[r_off * C + cv * 8 + j] = acc[j];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float t = 0.f;
    for (int rr = 0; rr < rows_par; ++rr) t += sh[rr * C + c];
    part[((long long)blockIdx.x * gridDim.y + b) * C + c] = t;
  }
}

// split-K partials of dW^T [rows = k*k*Cin][Cout] -> dW [Cout][rows]:
// out[b*s_out + o*rows + r] = sum_s part[s*s_split + (b*rows + r)*cout + o]
// (split order fixed; reads coalesced over o)
__global__ void splitk_reduce_t_kernel(const float* __restrict__ part, int ks, long long s_split, int rows, int cout,
                                       float* __restrict__ out, long long s_out) {
  pdl_enter();
  const long long b = blockIdx.y, n = (long long)rows * cout;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / cout), o = (int)(i % cout);
    float acc = 0.f;
    int s = 0;
    for (; s + 8 <= ks; s += 8) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = part[(s + u) * s_split + b * n + i];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += v[u];
    }
    for (; s < ks; ++s) acc += part[s * s_split + b * n + i];
    out[b * s_out + (long long)o * rows + r] = acc;
  }
}

// global average pool: p[w][b][c] = mean over HW of y[w][b][hw][c]
template <typename T>
__global__ void pool_fwd_kernel(const T* __restrict__ y, T* __restrict__ p, int B, int HW, int C, long long sy,
                                long long sp) {
  pdl_enter();
  const int b = blockIdx.x, w = blockIdx.y;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float s = 0.f;
    for (int i = 0; i < HW; ++i) s += to_f<T>(y[w * sy + ((long long)b * HW + i) * C + c]);
    p[w * sp + (long long)b * C + c] = from_f<T>(s / (float)HW);
  }
}

// its gradient through the last block's ReLU: g[w][b][hw][c] = dp[w][b][c] / HW
// where y[w][b][hw][c] > 0
template <typename T>
__global__ void pool_bwd_kernel(const T* __restrict__ dp, const T* __restrict__ y, T* __restrict__ gy, int B, int HW,
                                int C, long long sdp, long long sy) {
  pdl_enter();
  const long long n = (long long)B * HW * C;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    const int b = (int)(i / ((long long)HW * C));
    const float v = to_f<T>(dp[blockIdx.y * sdp + (long long)b * C + c]) / (float)HW;
    gy[blockIdx.y * sy + i] = from_f<T>(to_f<T>(y[blockIdx.y * sy + i]) > 0.f ? v : 0.f);
  }
}

// NHWC fp32 input with Cin channels -> T with Cp (>= Cin, zero-padded)
// channels; worker blockIdx.y (pixels per worker, activation stride sx)
template <typename T>
__global__ void load_image_kernel(const StepDev* __restrict__ sp, T* __restrict__ x0, long long pixels, int cin,
                                  int cp, long long sx) {
  pdl_enter();
  const float* __restrict__ x = sp->x + blockIdx.y * pixels * cin;
  T* __restrict__ xw = x0 + blockIdx.y * sx;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < pixels * cp;
       i += (long long)gridDim.x * blockDim.x) {
    const long long px = i / cp;
    const int c = (int)(i % cp);
    xw[i] = from_f<T>(c < cin ? x[px * cin + c] : 0.f);
  }
}

struct Conv {
  int cin, cout, k, stride, pad, H, W, Ho, Wo;
  bool relu;          // epilogue ReLU (stem, first conv of a block)
  bool implicit = false;     // forward + wgrad as tensor-core implicit GEMMs (no im2col buffer)
  bool implicit_dg = false;  // dgrad too (3x3 stride 1; stride-2 convs keep gcol + col2im)
  int layer;          // registered layer (0-based)
  void* in = nullptr;   // input activation (not owned)
  void* col = nullptr;  // im2col buffer (owned), worker stride col_stride
  long long col_stride = 0;
  void* out = nullptr;  // output activation (owned)
  void* dst = nullptr;        // where the forward writes (out, or the block output when fused)
  const void* res = nullptr;  // residual addend fused into the epilogue: dst = relu(conv + res)
  long long rows() const { return (long long)Ho * Wo; }
  long long kc() const { return (long long)k * k * cin; }
};

struct Block {
  int a, b, sc;       // conv indices (sc = -1: identity shortcut)
  void* x = nullptr;  // block input (not owned)
  void* y = nullptr;  // block output relu(b + shortcut) (owned)
};

}  // namespace
}  // namespace dsx_nn

using namespace dsx_nn;

struct dsx_cnn {
  int device = 0;
  bool bf16 = false;
  int K = 1, kbegin = 0, kl = 1;
  int batch = 0, image = 32, cin = 3, cp = 8, w0 = 64, classes = 10;
  int opt = DSX_OPT_SGD;
  float mu = 0.9f, b1 = 0.9f, b2 = 0.999f, eps = 1e-8f, wd = 0.f;
  int nsm = 148;
  int L = 0;                      // registered layers: convs + head
  std::vector<Conv> convs;
  std::vector<Block> blocks;
  std::vector<long long> off, boff, packed;  // per registered layer
  std::vector<int> fan_in, fan_out;
  long long P = 0;
  float *params = nullptr, *grads = nullptr, *mom = nullptr, *var = nullptr;
  __nv_bfloat16* pbf = nullptr;
  void* x0 = nullptr;            // padded input [kl][B][32][32][cp]
  void* pool = nullptr;          // [kl][B][C]
  float* logits = nullptr;       // [kl][B][classes]
  void* dlog = nullptr;          // [kl][B][ldc] T
  void* dpool = nullptr;         // [kl][B][C]
  void *g0 = nullptr, *g1 = nullptr, *gh = nullptr, *gcol = nullptr, *gsc = nullptr;
  float* wpart = nullptr;  // split-K wgrad partials
  float* cpart = nullptr;  // bias-gradient column-sum partials [4*nsm][C]
  long long act_max = 0, col_max = 0;  // elements per worker
  float *loss_part = nullptr, *loss = nullptr;
  float* xin = nullptr;
  int* labels = nullptr;
  const float* x_dev = nullptr;
  const int* labels_dev = nullptr;
  StepDev* sp = nullptr;
  StepDev* ring = nullptr;
  std::vector<cudaEvent_t> ring_ev;
  unsigned long long ring_i = 0;
  cudaStream_t stream = nullptr, side = nullptr;
  std::vector<cudaEvent_t> ev_upd, ev_sync;
  std::vector<unsigned char> synced_prev;
  cudaEvent_t ev[8] = {};
  cudaEvent_t iev[4] = {};
  std::vector<cudaEvent_t> pf, pb;  // dsx_cnn_profile: after each layer's FP / BP
  bool prof = false;
  bool instrument = false, any_synced = false;
  double link_bw = 0.0, link_lat = 0.0;  // throttled sync link (bw <= 0: off)
  bool overlap = true;                   // false: averages after the whole local step
  uint64_t launches = 0;
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  std::vector<void*> owned;
};

namespace dsx_nn {
namespace {

size_t esz(const dsx_cnn* m) { return m->bf16 ? 2 : 4; }

GemmCall cbase(const dsx_cnn* m) {
  GemmCall c{};
  c.bf16 = m->bf16;
  c.out_bf16 = m->bf16;
  c.g.batch = m->kl;
  return c;
}

const void* wptr(const dsx_cnn* m, int l) {
  return m->bf16 ? static_cast<const void*>(m->pbf + m->off[l]) : static_cast<const void*>(m->params + m->off[l]);
}

ConvGeom geom(const dsx_cnn* m, const Conv& cv, int mode) {
  ConvGeom q{mode, cv.H, cv.W, m->batch, cv.cin, cv.cout};
  q.stride = cv.stride;
  q.k = cv.k;
  return q;
}

// forward epilogue: bias (+ ReLU); a block's last conv also adds the
// residual and applies the block ReLU (dst = the block output)
void fwd_epilogue(const dsx_cnn* m, const Conv& cv, GemmArgs* g) {
  g->epi = cv.res ? kEpiBiasAddAct : kEpiBiasAct;
  g->relu = cv.relu ? 1 : 0;
  g->bias = m->params + m->boff[cv.layer];
  g->strideBias = m->P;
  g->mask = cv.res;
  g->ldmask = cv.cout;
  g->strideMask = m->act_max;
  g->C = cv.dst;
  g->ldc = cv.cout;
  g->strideC = m->act_max;
}

dsx_status conv_forward(dsx_cnn* m, const Conv& cv) {
  const long long M = (long long)m->batch * cv.rows(), Kc = cv.kc();
  if (cv.implicit) {
    GemmCall c = cbase(m);
    c.A = cv.in;
    c.sA = m->act_max;
    c.B = wptr(m, cv.layer);
    c.ldb = Kc;
    c.sB = m->P;
    fwd_epilogue(m, cv, &c.g);
    ++m->launches;
    return conv_gemm(c, geom(m, cv, kConvFwd), m->stream, m->nsm);
  }
  const int grid = blocks_for(M * cv.k * cv.k * (cv.cin / 8), m->nsm) / std::max(1, m->kl) + 1;
  if (m->bf16)
    CN_CUDA(launch_pdl(im2col_kernel<__nv_bfloat16>, dim3(grid, m->kl), 256, 0, m->stream, 
        static_cast<const __nv_bfloat16*>(cv.in), static_cast<__nv_bfloat16*>(cv.col), m->batch, cv.H, cv.W, cv.cin,
        cv.Ho, cv.Wo, cv.k, cv.stride, cv.pad, m->act_max, cv.col_stride));
  else
    CN_CUDA(launch_pdl(im2col_kernel<float>, dim3(grid, m->kl), 256, 0, m->stream, 
        static_cast<const float*>(cv.in), static_cast<float*>(cv.col), m->batch, cv.H, cv.W, cv.cin, cv.Ho, cv.Wo,
        cv.k, cv.stride, cv.pad, m->act_max, cv.col_stride));
  ++m->launches;
  GemmCall c = cbase(m);
  c.A = cv.col;
  c.lda = Kc;
  c.sA = cv.col_stride;
  c.B = wptr(m, cv.layer);
  c.ldb = Kc;
  c.sB = m->P;
  c.g.M = (int)M;
  c.g.N = cv.cout;
  c.g.K = (int)Kc;
  fwd_epilogue(m, cv, &c.g);
  ++m->launches;
  return gemm(c, m->stream, m->nsm);
}

// wgrad tiling: the widest tile, and split-K over the B*Ho*Wo reduction when
// the (Cout x k*k*Cin) output has fewer than two waves of tiles (the 64-wide
// stage-0 convs: 8 workers x 3 tiles for a 131072-long K)
// implicit convs with 64 output channels compute dW^T = x-patches^T dy
// (M = 9*Cin fills the 128-row tiles that Cout = 64 would leave half empty,
// and the per-k-block traffic halves); the split-K reduce transposes back
bool wgrad_transposed(const Conv& cv) {
  static const bool on = [] {
    const char* e = std::getenv("DSX_CONV_WGRAD_T");
    return !(e && e[0] == '0');
  }();
  return on && cv.implicit && cv.cout == 64;
}

void wgrad_plan(const dsx_cnn* m, const Conv& cv, int* bn, int* ks) {
  const long long Kc = cv.kc(), Kg = (long long)m->batch * cv.rows();
  const bool tr = wgrad_transposed(cv);
  *bn = tr ? 64 : Kc >= 256 ? 256 : Kc >= 128 ? 128 : 64;
  const long long units = tr ? ((Kc + kBM - 1) / kBM) * m->kl
                             : ((cv.cout + kBM - 1) / kBM) * ((Kc + *bn - 1) / *bn) * m->kl;
  const long long nk = (Kg + kBK - 1) / kBK;
  *ks = 1;
  if (m->bf16 && units < 2LL * m->nsm)
    *ks = (int)std::max<long long>(1, std::min<long long>((2LL * m->nsm + units - 1) / units, nk / 8));
}

dsx_status col2im(dsx_cnn* m, const Conv& cv, void* dx, const void* add, const void* mask,
                  const void* sub2 = nullptr);

// wgrad + bias grad + (dx != null) the input gradient dx = dgrad (+ add)
// (* (mask > 0)), then the layer's optimizer step; g = dL/d(conv output)
// [B*Ho*Wo][Cout].  Implicit convs produce dx in the dgrad GEMM's epilogue;
// the others through gcol + col2im.
// raw (1x1 convs on the explicit path): dx = the dgrad GEMM's [B*Ho*Wo][Cin]
// output itself, for the caller's col2im to scatter (sub2); sub2: such a
// projection gradient folded into this conv's col2im
dsx_status conv_backward(dsx_cnn* m, const Conv& cv, const void* g, void* dx, const void* add, const void* mask,
                         const OptArgs& o, const StepDev* sp, const float* db_from = nullptr, bool raw = false,
                         const void* sub2 = nullptr) {
  const long long M = (long long)m->batch * cv.rows(), Kc = cv.kc();
  const bool dgrad = dx != nullptr;
  if (wgrad_transposed(cv)) {
    GemmCall c = cbase(m);
    c.A = cv.in;
    c.sA = m->act_max;
    c.B = g;
    c.ldb = cv.cout;
    c.sB = m->act_max;
    c.g.epi = kEpiF32;
    int ks = 1;
    wgrad_plan(m, cv, &c.bn, &ks);
    c.g.C = m->wpart;
    c.g.ldc = cv.cout;
    c.g.strideC = (long long)cv.cout * Kc;
    c.g.ksplit = ks;
    c.g.strideSplit = (long long)m->kl * cv.cout * Kc;
    ++m->launches;
    CN_TRY(conv_gemm(c, geom(m, cv, kConvWgradT), m->stream, m->nsm));
    const long long nk = (M + kBK - 1) / kBK, kper = (nk + ks - 1) / ks;
    const long long n = (long long)cv.cout * Kc;
    CN_CUDA(launch_pdl(splitk_reduce_t_kernel, dim3(blocks_for(n, m->nsm) / m->kl + 1, m->kl), 256, 0, m->stream, 
        m->wpart, (int)((nk + kper - 1) / kper), c.g.strideSplit, (int)Kc, cv.cout, m->grads + m->off[cv.layer],
        m->P));
    ++m->launches;
  } else if (cv.implicit) {
    GemmCall c = cbase(m);
    c.A = g;
    c.lda = cv.cout;
    c.sA = m->act_max;
    c.B = cv.in;
    c.sB = m->act_max;
    c.g.epi = kEpiF32;
    int ks = 1;
    wgrad_plan(m, cv, &c.bn, &ks);
    c.g.ldc = Kc;
    if (ks > 1) {
      c.g.C = m->wpart;
      c.g.strideC = (long long)cv.cout * Kc;
      c.g.ksplit = ks;
      c.g.strideSplit = (long long)m->kl * cv.cout * Kc;
    } else {
      c.g.C = m->grads + m->off[cv.layer];
      c.g.strideC = m->P;
    }
    ++m->launches;
    CN_TRY(conv_gemm(c, geom(m, cv, kConvWgrad), m->stream, m->nsm));
    if (ks > 1) {
      const long long nk = (M + kBK - 1) / kBK, kper = (nk + ks - 1) / ks;
      const long long n = (long long)cv.cout * Kc;
      CN_CUDA(launch_pdl(splitk_reduce_kernel, dim3(blocks_for(n, m->nsm) / m->kl + 1, m->kl), 256, 0, m->stream, 
          m->wpart, (int)((nk + kper - 1) / kper), c.g.strideSplit, n, m->grads + m->off[cv.layer], m->P));
      ++m->launches;
    }
  } else {
    GemmCall c = cbase(m);
    c.a_mn = true;
    c.b_mn = true;
    c.A = g;
    c.lda = cv.cout;
    c.sA = m->act_max;
    c.B = cv.col;
    c.ldb = Kc;
    c.sB = cv.col_stride;
    c.g.M = cv.cout;
    c.g.N = (int)Kc;
    c.g.K = (int)M;
    c.g.epi = kEpiF32;
    int ks = 1;
    wgrad_plan(m, cv, &c.bn, &ks);
    c.g.ldc = Kc;
    if (ks > 1) {
      c.g.C = m->wpart;
      c.g.strideC = (long long)cv.cout * Kc;
      c.g.ksplit = ks;
      c.g.strideSplit = (long long)m->kl * cv.cout * Kc;
    } else {
      c.g.C = m->grads + m->off[cv.layer];
      c.g.strideC = m->P;
    }
    ++m->launches;
    CN_TRY(gemm(c, m->stream, m->nsm));
    if (ks > 1) {
      // gemm() may have lowered ks to keep every split non-empty: the unused
      // partial slots are never read (same rounding as in gemm())
      const long long nk = ((long long)M + kBK - 1) / kBK, kper = (nk + ks - 1) / ks;
      const int ks_eff = (int)((nk + kper - 1) / kper);
      const long long n = (long long)cv.cout * Kc;
      CN_CUDA(launch_pdl(splitk_reduce_kernel, dim3(blocks_for(n, m->nsm) / m->kl + 1, m->kl), 256, 0, m->stream, 
          m->wpart, ks_eff, c.g.strideSplit, n, m->grads + m->off[cv.layer], m->P));
      ++m->launches;
    }
  }
  {
    // bias gradient: two-pass column sum over the B*Ho*Wo rows (row chunks
    // -> per-chunk partials -> fixed-order sum), ~4 blocks per SM; a
    // projection block's conv b reuses its shortcut's (same gradient)
    const int tpr = cv.cout / 8, rows_par = std::max(1, 256 / tpr);
    const int nchunks = (int)std::max<long long>(
        1, std::min<long long>(4LL * m->nsm / m->kl, M / (4LL * rows_par)));
    const int chunk_rows = (int)((M + nchunks - 1) / nchunks);
    dim3 grid(nchunks, m->kl);
    if (db_from) {
      CN_CUDA(cudaMemcpy2DAsync(m->grads + m->boff[cv.layer], 4ull * m->P, db_from, 4ull * m->P, 4ull * cv.cout,
                                m->kl, cudaMemcpyDeviceToDevice, m->stream));
    } else if (m->bf16)
      CN_CUDA(launch_pdl(colsum_part_kernel<__nv_bfloat16>, grid, 256, 0, m->stream, static_cast<const __nv_bfloat16*>(g), cv.cout,
                                                                     m->act_max, (int)M, cv.cout, chunk_rows, m->cpart));
    else
      CN_CUDA(launch_pdl(colsum_part_kernel<float>, grid, 256, 0, m->stream, static_cast<const float*>(g), cv.cout, m->act_max,
                                                             (int)M, cv.cout, chunk_rows, m->cpart));
    if (!db_from) {
      CN_CUDA(launch_pdl(splitk_reduce_kernel, dim3((cv.cout + 63) / 64, m->kl), 64, 0, m->stream, 
          m->cpart, nchunks, (long long)m->kl * cv.cout, cv.cout, m->grads + m->boff[cv.layer], m->P));
      m->launches += 2;
    }
  }
  if (dgrad && cv.implicit_dg) {
    GemmCall c = cbase(m);
    c.A = g;
    c.sA = m->act_max;
    c.B = wptr(m, cv.layer);
    c.sB = m->P;
    c.g.epi = add && mask ? kEpiAddDRelu : add ? kEpiAdd : (mask ? kEpiDRelu : kEpiBiasAct);
    c.g.relu = 0;
    c.g.bias = nullptr;
    c.g.mask = add ? add : mask;
    c.g.ldmask = cv.cin;
    c.g.strideMask = m->act_max;
    c.g.mask2 = add ? mask : nullptr;
    c.g.ldmask2 = cv.cin;
    c.g.strideMask2 = m->act_max;
    c.g.C = dx;
    c.g.ldc = cv.cin;
    c.g.strideC = m->act_max;
    ++m->launches;
    CN_TRY(conv_gemm(c, geom(m, cv, kConvDgrad), m->stream, m->nsm));
  } else if (dgrad) {
    GemmCall c = cbase(m);
    c.a_mn = false;
    c.b_mn = true;
    c.A = g;
    c.lda = cv.cout;
    c.sA = m->act_max;
    c.B = wptr(m, cv.layer);
    c.ldb = Kc;
    c.sB = m->P;
    c.g.M = (int)M;
    c.g.N = (int)Kc;
    c.g.K = cv.cout;
    c.g.epi = kEpiBiasAct;  // plain copy-out (no bias, no ReLU)
    c.g.relu = 0;
    c.g.bias = nullptr;
    c.g.C = raw ? dx : m->gcol;
    c.g.ldc = Kc;
    c.g.strideC = raw ? m->act_max : m->col_max;
    ++m->launches;
    CN_TRY(gemm(c, m->stream, m->nsm));
  }
  const long long lo = m->off[cv.layer], n = m->boff[cv.layer] + cv.cout - lo;
  const long long want = (n / 8 + 255) / 256;
  dim3 grid((unsigned)std::max<long long>(1, std::min<long long>(want, (long long)m->nsm * 8 / m->kl)), m->kl);
  CN_CUDA(launch_pdl(optimizer_kernel, grid, 256, 0, m->stream, m->params, m->grads, m->mom, m->var, m->bf16 ? m->pbf : nullptr, m->P,
                                                lo, n, o, sp));
  ++m->launches;
  CN_CUDA(cudaGetLastError());
  if (dgrad && !cv.implicit_dg && !raw) return col2im(m, cv, dx, add, mask, sub2);
  return DSX_OK;
}

// dx = col2im(gcol) (+ add) (* (mask > 0)) for conv cv's input geometry
dsx_status col2im(dsx_cnn* m, const Conv& cv, void* dx, const void* add, const void* mask, const void* sub2) {
  const long long total = (long long)m->batch * cv.H * cv.W * (cv.cin / 8);
  const int grid = blocks_for(total, m->nsm) / std::max(1, m->kl) + 1;
  if (m->bf16)
    CN_CUDA(launch_pdl(col2im_kernel<__nv_bfloat16>, dim3(grid, m->kl), 256, 0, m->stream, 
        static_cast<const __nv_bfloat16*>(m->gcol), static_cast<__nv_bfloat16*>(dx), m->batch, cv.H, cv.W, cv.cin,
        cv.Ho, cv.Wo, cv.k, cv.stride, cv.pad, static_cast<const __nv_bfloat16*>(add),
        static_cast<const __nv_bfloat16*>(mask), m->col_max, m->act_max, static_cast<const __nv_bfloat16*>(sub2)));
  else
    CN_CUDA(launch_pdl(col2im_kernel<float>, dim3(grid, m->kl), 256, 0, m->stream, 
        static_cast<const float*>(m->gcol), static_cast<float*>(dx), m->batch, cv.H, cv.W, cv.cin, cv.Ho, cv.Wo, cv.k,
        cv.stride, cv.pad, static_cast<const float*>(add), static_cast<const float*>(mask), m->col_max, m->act_max,
        static_cast<const float*>(sub2)));
  ++m->launches;
  CN_CUDA(cudaGetLastError());
  return DSX_OK;
}


dsx_status average_layer(dsx_cnn* m, int l, cudaStream_t s) {
  std::string err;
  const long long n = m->packed[l + 1] - m->packed[l];
  const dsx_status st = average_range(m->params, m->bf16 ? m->pbf : nullptr, m->P, m->kl, m->K, m->nranks, m->comm,
                                      m->off[l], n, m->nsm, s, &m->launches, &err);
  if (st != DSX_OK) return cfail(st, err);
  return DSX_OK;
}

dsx_status write_step(dsx_cnn* m, double lr, long long t) {
  if (!m->x_dev || !m->labels_dev) return cfail(DSX_ERR_STATE, "dsx_cnn_step: no batch set (dsx_cnn_set_batch)");
  const int slot = (int)(m->ring_i++ % m->ring_ev.size());
  CN_CUDA(cudaEventSynchronize(m->ring_ev[slot]));
  StepDev& h = m->ring[slot];
  h.lr = (float)lr;
  h.bc1 = (float)(1.0 - std::pow((double)m->b1, (double)(t + 1)));
  h.bc2 = (float)(1.0 - std::pow((double)m->b2, (double)(t + 1)));
  h.pad = 0.f;
  h.x = m->x_dev;
  h.labels = m->labels_dev;
  CN_CUDA(cudaMemcpyAsync(m->sp, &h, sizeof(StepDev), cudaMemcpyHostToDevice, m->stream));
  CN_CUDA(cudaEventRecord(m->ring_ev[slot], m->stream));
  return DSX_OK;
}

// forward pass up to the logits (the layer waits handle last step's averages)
dsx_status forward(dsx_cnn* m, bool wait_syncs) {
  const long long pixels = (long long)m->batch * m->image * m->image;
  const dim3 lgrid(blocks_for(pixels * m->cp, m->nsm) / m->kl + 1, m->kl);
  if (m->bf16)
    CN_CUDA(launch_pdl(load_image_kernel<__nv_bfloat16>, lgrid, 256, 0, m->stream, m->sp, static_cast<__nv_bfloat16*>(m->x0),
                                                                   pixels, m->cin, m->cp, m->act_max));
  else
    CN_CUDA(launch_pdl(load_image_kernel<float>, lgrid, 256, 0, m->stream, m->sp, static_cast<float*>(m->x0), pixels, m->cin,
                                                           m->cp, m->act_max));
  ++m->launches;
  auto wait_layer = [&](int l) -> dsx_status {
    if (wait_syncs && m->synced_prev[l]) CN_CUDA(cudaStreamWaitEvent(m->stream, m->ev_sync[l], 0));
    return DSX_OK;
  };
  auto mark = [&](int l) -> dsx_status {
    if (m->prof) CN_CUDA(cudaEventRecord(m->pf[l], m->stream));
    return DSX_OK;
  };
  CN_TRY(mark(0));
  CN_TRY(wait_layer(m->convs[0].layer));
  CN_TRY(conv_forward(m, m->convs[0]));
  CN_TRY(mark(1));
  for (const Block& bk : m->blocks) {
    const Conv& a = m->convs[bk.a];
    const Conv& b = m->convs[bk.b];
    CN_TRY(wait_layer(a.layer));
    CN_TRY(conv_forward(m, a));
    CN_TRY(mark(a.layer + 1));
    CN_TRY(wait_layer(b.layer));
    CN_TRY(conv_forward(m, b));
    CN_TRY(mark(b.layer + 1));
    // the block output relu(b + shortcut) comes out of the last conv's
    // epilogue (conv b with an identity shortcut, else the 1x1 projection)
    if (bk.sc >= 0) {
      CN_TRY(wait_layer(m->convs[bk.sc].layer));
      CN_TRY(conv_forward(m, m->convs[bk.sc]));
      CN_TRY(mark(bk.sc + 1));
    }
  }
  // global average pool + head
  const Block& last = m->blocks.back();
  const Conv& lc = m->convs[last.b];
  const int C = lc.cout, HW = lc.Ho * lc.Wo;
  if (m->bf16)
    CN_CUDA(launch_pdl(pool_fwd_kernel<__nv_bfloat16>, dim3(m->batch, m->kl), 256, 0, m->stream, 
        static_cast<const __nv_bfloat16*>(last.y), static_cast<__nv_bfloat16*>(m->pool), m->batch, HW, C, m->act_max,
        (long long)m->batch * C));
  else
    CN_CUDA(launch_pdl(pool_fwd_kernel<float>, dim3(m->batch, m->kl), 256, 0, m->stream, 
        static_cast<const float*>(last.y), static_cast<float*>(m->pool), m->batch, HW, C, m->act_max,
        (long long)m->batch * C));
  ++m->launches;
  const int hl = m->L - 1;
  CN_TRY(wait_layer(hl));
  GemmCall c = cbase(m);
  c.A = m->pool;
  c.lda = C;
  c.sA = (long long)m->batch * C;
  c.B = wptr(m, hl);
  c.ldb = C;
  c.sB = m->P;
  c.g.M = m->batch;
  c.g.N = m->classes;
  c.g.K = C;
  c.g.epi = kEpiBiasAct;
  c.g.bias = m->params + m->boff[hl];
  c.g.strideBias = m->P;
  c.out_bf16 = false;
  c.g.C = m->logits;
  c.g.ldc = m->classes;
  c.g.strideC = (long long)m->batch * m->classes;
  ++m->launches;
  CN_TRY(gemm(c, m->stream, m->nsm));
  return mark(hl + 1);
}

long long ld_classes(const dsx_cnn* m) { return m->bf16 ? (m->classes + 7) / 8 * 8 : m->classes; }

dsx_status step_impl(dsx_cnn* m, double lr, long long t, const unsigned char* mask) {
  OptArgs o{};
  o.kind = m->opt;
  o.lr = (float)lr;
  o.mu = m->mu;
  o.b1 = m->b1;
  o.b2 = m->b2;
  o.eps = m->eps;
  o.wd = m->wd;
  o.bc1 = o.bc2 = 1.f;
  if (m->instrument) CN_CUDA(cudaEventRecord(m->iev[0], m->stream));
  CN_TRY(forward(m, true));
  // loss + dlogits
  const int C = m->classes;
  {
    dim3 grid((m->batch * 32 + 255) / 256, m->kl);
    if (m->bf16)
      CN_CUDA(launch_pdl(softmax_xent_kernel<__nv_bfloat16>, grid, 256, 0, m->stream, 
          m->logits, C, (long long)m->batch * C, nullptr, m->batch, C, static_cast<__nv_bfloat16*>(m->dlog),
          ld_classes(m), (long long)m->batch * ld_classes(m), m->loss_part, m->sp));
    else
      CN_CUDA(launch_pdl(softmax_xent_kernel<float>, grid, 256, 0, m->stream, m->logits, C, (long long)m->batch * C, nullptr, m->batch,
                                                              C, static_cast<float*>(m->dlog), ld_classes(m),
                                                              (long long)m->batch * ld_classes(m), m->loss_part, m->sp));
    CN_CUDA(launch_pdl(loss_mean_kernel, m->kl, 256, 0, m->stream, m->loss_part, m->batch, m->loss));
    m->launches += 2;
  }
  if (m->prof) CN_CUDA(cudaEventRecord(m->pb[m->L], m->stream));
  bool any = false;
  // one layer's sync on the side stream (+ the throttled link's busy time)
  auto sync_layer = [&](int l) -> dsx_status {
    if (m->instrument && !any) CN_CUDA(cudaEventRecord(m->ev[7], m->side));
    CN_TRY(average_layer(m, l, m->side));
    if (m->link_bw > 0.0) {
      const double bytes = 4.0 * (double)(m->packed[l + 1] - m->packed[l]);
      nn_link_spin_kernel<<<1, 1, 0, m->side>>>((unsigned long long)((m->link_lat + bytes / m->link_bw) * 1e9));
      ++m->launches;
    }
    CN_CUDA(cudaEventRecord(m->ev_sync[l], m->side));
    any = true;
    return DSX_OK;
  };
  auto done_layer = [&](int l) -> dsx_status {
    if (m->prof) CN_CUDA(cudaEventRecord(m->pb[l], m->stream));
    const bool sync_l = mask[l + 1] != 0 && m->K > 1;
    m->synced_prev[l] = sync_l ? 1 : 0;
    if (!sync_l || !m->overlap) return DSX_OK;
    CN_CUDA(cudaEventRecord(m->ev_upd[l], m->stream));
    CN_CUDA(cudaStreamWaitEvent(m->side, m->ev_upd[l], 0));
    return sync_layer(l);
  };
  // head: dW = dlog^T pool, db, dpool = dlog W  ->  pool backward into g0
  const int hl = m->L - 1;
  const Block& last = m->blocks.back();
  const int Cl = m->convs[last.b].cout, HW = m->convs[last.b].Ho * m->convs[last.b].Wo;
  {
    GemmCall c = cbase(m);
    c.a_mn = true;
    c.b_mn = true;
    c.A = m->dlog;
    c.lda = ld_classes(m);
    c.sA = (long long)m->batch * ld_classes(m);
    c.B = m->pool;
    c.ldb = Cl;
    c.sB = (long long)m->batch * Cl;
    c.g.M = C;
    c.g.N = Cl;
    c.g.K = m->batch;
    c.g.epi = kEpiF32;
    c.g.C = m->grads + m->off[hl];
    c.g.ldc = Cl;
    c.g.strideC = m->P;
    ++m->launches;
    CN_TRY(gemm(c, m->stream, m->nsm));
    dim3 grid((C + 31) / 32, m->kl);
    if (m->bf16)
      CN_CUDA(launch_pdl(colsum_kernel<__nv_bfloat16>, grid, 256, 0, m->stream, static_cast<const __nv_bfloat16*>(m->dlog),
                                                                ld_classes(m), (long long)m->batch * ld_classes(m),
                                                                m->batch, C, m->grads + m->boff[hl], m->P));
    else
      CN_CUDA(launch_pdl(colsum_kernel<float>, grid, 256, 0, m->stream, static_cast<const float*>(m->dlog), ld_classes(m),
                                                        (long long)m->batch * ld_classes(m), m->batch, C,
                                                        m->grads + m->boff[hl], m->P));
    ++m->launches;
    GemmCall d = cbase(m);
    d.a_mn = false;
    d.b_mn = true;
    d.A = m->dlog;
    d.lda = ld_classes(m);
    d.sA = (long long)m->batch * ld_classes(m);
    d.B = wptr(m, hl);
    d.ldb = Cl;
    d.sB = m->P;
    d.g.M = m->batch;
    d.g.N = Cl;
    d.g.K = C;
    d.g.epi = kEpiBiasAct;
    d.g.relu = 0;
    d.g.bias = nullptr;
    d.g.C = m->dpool;
    d.g.ldc = Cl;
    d.g.strideC = (long long)m->batch * Cl;
    ++m->launches;
    CN_TRY(gemm(d, m->stream, m->nsm));
    const long long lo = m->off[hl], n = m->packed[hl + 1] - m->packed[hl];
    CN_CUDA(launch_pdl(optimizer_kernel, dim3((unsigned)std::max<long long>(1, (n / 8 + 255) / 256), m->kl), 256, 0, m->stream, 
        m->params, m->grads, m->mom, m->var, m->bf16 ? m->pbf : nullptr, m->P, lo, n, o, m->sp));
    ++m->launches;
    CN_TRY(done_layer(hl));
    if (m->bf16)
      CN_CUDA(launch_pdl(pool_bwd_kernel<__nv_bfloat16>, dim3(blocks_for((long long)m->batch * HW * Cl, m->nsm), m->kl), 256, 0,
                                       m->stream, static_cast<const __nv_bfloat16*>(m->dpool),
                                                    static_cast<const __nv_bfloat16*>(last.y),
                                                    static_cast<__nv_bfloat16*>(m->g0), m->batch, HW, Cl,
                                                    (long long)m->batch * Cl, m->act_max));
    else
      CN_CUDA(launch_pdl(pool_bwd_kernel<float>, dim3(blocks_for((long long)m->batch * HW * Cl, m->nsm), m->kl), 256, 0, m->stream, 
          static_cast<const float*>(m->dpool), static_cast<const float*>(last.y), static_cast<float*>(m->g0),
          m->batch, HW, Cl, (long long)m->batch * Cl, m->act_max));
    ++m->launches;
  }
  // blocks, last to first.  ga = dL/d(block output) * (block output > 0) —
  // the gradient of the block's last convs — lives in g0/g1: the pool
  // backward produces the top block's, each block's first-conv dgrad the one
  // below (epilogue: (dgrad + shortcut gradient) * (block input > 0))
  void* ga = m->g0;
  void* gnext = m->g1;
  for (int bi = (int)m->blocks.size() - 1; bi >= 0; --bi) {
    const Block& bk = m->blocks[bi];
    const Conv& a = m->convs[bk.a];
    const Conv& b = m->convs[bk.b];
    const void* sc_grad = ga;  // identity shortcut: dx gets ga
    const void* sc_raw = nullptr;
    if (bk.sc >= 0) {
      const Conv& s = m->convs[bk.sc];
      // a 1x1 stride-2 projection's dgrad stays [B][H/2][W/2][C]; conv a's
      // col2im adds it at the even pixels
      const bool fold = s.k == 1 && s.stride == 2 && !a.implicit_dg;
      CN_TRY(conv_backward(m, s, ga, m->gsc, nullptr, nullptr, o, m->sp, nullptr, fold));
      if (fold) sc_raw = m->gsc;
      sc_grad = fold ? nullptr : m->gsc;
      CN_TRY(done_layer(s.layer));
    }
    // second conv; its input h = relu(first conv): gh = dgrad * (h > 0)
    CN_TRY(conv_backward(m, b, ga, m->gh, nullptr, b.in, o, m->sp,
                         bk.sc >= 0 ? m->grads + m->boff[m->convs[bk.sc].layer] : nullptr));
    CN_TRY(done_layer(b.layer));
    // first conv; (dgrad + shortcut grad) * (x > 0), x = the block input =
    // the previous block's output (or the stem's): that block's ga
    CN_TRY(conv_backward(m, a, m->gh, gnext, sc_grad, bk.x, o, m->sp, nullptr, false, sc_raw));
    CN_TRY(done_layer(a.layer));
    std::swap(ga, gnext);
  }
  // stem: wgrad only, its output gradient already through its ReLU'
  {
    const Conv& st = m->convs[0];
    CN_TRY(conv_backward(m, st, ga, nullptr, nullptr, nullptr, o, m->sp));
    CN_TRY(done_layer(st.layer));
  }
  if (!m->overlap) {
    // ssgd / flsgd: the transfers start after the whole local step
    CN_CUDA(cudaEventRecord(m->ev_upd[0], m->stream));
    CN_CUDA(cudaStreamWaitEvent(m->side, m->ev_upd[0], 0));
    for (int l = m->L - 1; l >= 0; --l)
      if (m->synced_prev[l]) CN_TRY(sync_layer(l));
  }
  m->any_synced = any;
  if (m->instrument) {
    CN_CUDA(cudaEventRecord(m->iev[1], m->stream));
    CN_CUDA(cudaEventRecord(m->iev[2], m->side));
  }
  CN_CUDA(cudaGetLastError());
  return DSX_OK;
}

dsx_status ccheck(dsx_cnn* m) {
  if (!m) return cfail(DSX_ERR_ARGUMENT, "null cnn");
  CN_CUDA(cudaSetDevice(m->device));
  return DSX_OK;
}

}  // namespace
}  // namespace dsx_nn

extern "C" {

dsx_status dsx_cnn_create(const dsx_cnn_desc* d, dsx_cnn** out) {
  if (!d || !out) return cfail(DSX_ERR_ARGUMENT, "null argument");
  *out = nullptr;
  if (d->dtype != DSX_F32 && d->dtype != DSX_BF16) return cfail(DSX_ERR_ARGUMENT, "dtype must be DSX_F32 or DSX_BF16");
  if (d->workers_total < 1 || d->workers_local < 1 || d->worker_begin < 0 ||
      d->worker_begin + d->workers_local > d->workers_total)
    return cfail(DSX_ERR_ARGUMENT, "bad worker range");
  if (d->workers_local != 1 && d->workers_local != 2 && d->workers_local != 4 && d->workers_local != 8)
    return cfail(DSX_ERR_ARGUMENT, "workers_local must be 1, 2, 4 or 8");
  if (d->width < 8 || d->width % 8 || d->image < 8 || d->image % 8 || d->in_channels < 1 || d->in_channels > 8 ||
      d->classes < 2 || d->batch < 1)
    return cfail(DSX_ERR_ARGUMENT, "width and image must be multiples of 8, in_channels <= 8, classes >= 2");
  if (d->optimizer < DSX_OPT_SGD || d->optimizer > DSX_OPT_ADAM) return cfail(DSX_ERR_ARGUMENT, "bad optimizer");
  int ndev = 0;
  CN_CUDA(cudaGetDeviceCount(&ndev));
  if (d->device < 0 || d->device >= ndev) return cfail(DSX_ERR_CUDA, "no such CUDA device");
  CN_CUDA(cudaSetDevice(d->device));
  auto* m = new dsx_cnn();
  auto cleanup = [&](dsx_status s) {
    dsx_cnn_destroy(m);
    return s;
  };
  m->device = d->device;
  m->bf16 = d->dtype == DSX_BF16;
  m->K = d->workers_total;
  m->kbegin = d->worker_begin;
  m->kl = d->workers_local;
  m->batch = d->batch;
  m->image = d->image;
  m->cin = d->in_channels;
  m->cp = 8;
  m->w0 = d->width;
  m->classes = d->classes;
  m->opt = d->optimizer;
  m->mu = (float)d->momentum;
  m->b1 = (float)d->beta1;
  m->b2 = (float)d->beta2;
  m->eps = (float)d->eps;
  m->wd = (float)d->weight_decay;
  cudaDeviceGetAttribute(&m->nsm, cudaDevAttrMultiProcessorCount, d->device);
  // topology: stem, 4 stages x 2 basic blocks, head
  auto add_conv = [&](int cin, int cout, int k, int stride, int H, bool relu) {
    Conv c;
    c.cin = cin;
    c.cout = cout;
    c.k = k;
    c.stride = stride;
    c.pad = k == 3 ? 1 : 0;
    c.H = c.W = H;
    c.Ho = c.Wo = (H + 2 * c.pad - k) / stride + 1;
    c.relu = relu;
    // DSX_CONV_IMPLICIT=0: every conv through im2col / col2im (A/B measurements)
    static const bool implicit_ok = [] {
      const char* e = std::getenv("DSX_CONV_IMPLICIT");
      return !(e && e[0] == '0');
    }();
    const int Wo = c.Wo;
    c.implicit = implicit_ok && m->bf16 && cin % 64 == 0 && cout % 64 == 0 && Wo <= 64 && 64 % Wo == 0 &&
                 ((k == 3 && (stride == 1 || stride == 2)) || (k == 1 && stride == 2));
    c.implicit_dg = c.implicit && k == 3 && stride == 1;
    c.layer = (int)m->convs.size();
    m->convs.push_back(c);
    return (int)m->convs.size() - 1;
  };
  int H = m->image;
  add_conv(m->cp, m->w0, 3, 1, H, true);
  int cin = m->w0;
  for (int s = 0; s < 4; ++s) {
    const int w = m->w0 << s;
    for (int blk = 0; blk < 2; ++blk) {
      const int stride = (s > 0 && blk == 0) ? 2 : 1;
      Block b;
      b.a = add_conv(cin, w, 3, stride, H, true);
      const int Ho = m->convs[b.a].Ho;
      b.b = add_conv(w, w, 3, 1, Ho, false);
      b.sc = (stride != 1 || cin != w) ? add_conv(cin, w, 1, stride, H, false) : -1;
      m->blocks.push_back(b);
      cin = w;
      H = Ho;
    }
  }
  m->L = (int)m->convs.size() + 1;
  long long o = 0, po = 0;
  m->packed.push_back(0);
  for (int l = 0; l < m->L; ++l) {
    long long wsz, bsz;
    if (l < (int)m->convs.size()) {
      wsz = (long long)m->convs[l].cout * m->convs[l].kc();
      bsz = m->convs[l].cout;
      m->fan_in.push_back((int)m->convs[l].kc());
    } else {
      wsz = (long long)m->classes * cin;
      bsz = m->classes;
      m->fan_in.push_back(cin);
    }
    m->off.push_back(o);
    m->boff.push_back(o + wsz);
    o = (o + wsz + bsz + 63) / 64 * 64;
    po += wsz + bsz;
    m->packed.push_back(po);
  }
  m->P = o;
  // buffer sizes (elements per worker)
  long long act = (long long)m->batch * m->image * m->image * m->cp, col = 0;
  for (const Conv& c : m->convs) {
    act = std::max(act, (long long)m->batch * c.Ho * c.Wo * c.cout);
    act = std::max(act, (long long)m->batch * c.H * c.W * c.cin);
    if (!c.implicit_dg) col = std::max(col, (long long)m->batch * c.rows() * c.kc());
  }
  // im2col / col2im index one worker's 8-channel vectors with 32-bit ints
  if (std::max(col, act) / 8 >= (1LL << 31))
    return cleanup(cfail(DSX_ERR_ARGUMENT, "batch too large: one worker's im2col exceeds 2^34 elements"));
  m->act_max = (act + 63) / 64 * 64;
  long long wpart = 0;
  for (const Conv& c : m->convs) {
    int bn = 0, ks = 1;
    wgrad_plan(m, c, &bn, &ks);
    if (ks > 1 || wgrad_transposed(c)) wpart = std::max(wpart, (long long)ks * m->kl * c.cout * c.kc());
  }
  m->col_max = (col + 63) / 64 * 64;
  const size_t es = m->bf16 ? 2 : 4;
  auto alloc = [&](void** p, size_t bytes) -> bool {
    if (cudaMalloc(p, bytes) != cudaSuccess) return false;
    cudaMemset(*p, 0, bytes);
    m->owned.push_back(*p);
    return true;
  };
  const size_t arena = 4ull * m->P * m->kl;
  const size_t actb = es * m->act_max * m->kl, colb = es * m->col_max * m->kl;
  bool ok = alloc((void**)&m->params, arena) && alloc((void**)&m->grads, arena) &&
            (m->opt == DSX_OPT_SGD || alloc((void**)&m->mom, arena)) &&
            (m->opt != DSX_OPT_ADAM || alloc((void**)&m->var, arena)) &&
            (!m->bf16 || alloc((void**)&m->pbf, 2ull * m->P * m->kl)) && alloc(&m->x0, actb);
  for (size_t i = 0; ok && i < m->convs.size(); ++i) {
    Conv& c = m->convs[i];
    if (c.implicit) {
      ok = alloc(&c.out, actb);
      continue;
    }
    c.col_stride = ((long long)m->batch * c.rows() * c.kc() + 63) / 64 * 64;
    ok = alloc(&c.col, es * c.col_stride * m->kl) && alloc(&c.out, actb);
  }
  for (size_t i = 0; ok && i < m->blocks.size(); ++i) ok = alloc(&m->blocks[i].y, actb);
  ok = ok && alloc(&m->g0, actb) && alloc(&m->g1, actb) && alloc(&m->gh, actb) &&
       alloc(&m->gsc, actb) && alloc(&m->gcol, colb) && (wpart == 0 || alloc((void**)&m->wpart, 4ull * wpart)) &&
       alloc((void**)&m->cpart, 4ull * 4 * m->nsm * (m->w0 << 3)) &&
       alloc(&m->pool, es * m->kl * m->batch * cin) && alloc(&m->dpool, es * m->kl * m->batch * cin) &&
       alloc((void**)&m->logits, 4ull * m->kl * m->batch * m->classes) &&
       alloc(&m->dlog, es * m->kl * m->batch * ((m->classes + 7) / 8 * 8)) &&
       alloc((void**)&m->loss_part, 4ull * m->kl * m->batch) && alloc((void**)&m->loss, 4ull * m->kl) &&
       alloc((void**)&m->xin, 4ull * m->kl * m->batch * m->image * m->image * m->cin) &&
       alloc((void**)&m->labels, 4ull * m->kl * m->batch) && alloc((void**)&m->sp, sizeof(StepDev));
  if (!ok) return cleanup(cfail(DSX_ERR_CUDA, "cudaMalloc(conv-stack buffers) failed"));
  // wire the activations: stem reads x0; block a/sc read the block input;
  // b reads a's output
  m->convs[0].in = m->x0;
  for (Conv& c : m->convs) c.dst = c.out;
  void* x = m->convs[0].out;
  for (Block& b : m->blocks) {
    b.x = x;
    m->convs[b.a].in = x;
    m->convs[b.b].in = m->convs[b.a].out;
    if (b.sc >= 0) m->convs[b.sc].in = x;
    // the block's last conv writes relu(conv + residual) = the block output
    Conv& last = m->convs[b.sc >= 0 ? b.sc : b.b];
    last.res = b.sc >= 0 ? m->convs[b.b].out : x;
    last.dst = b.y;
    last.relu = true;
    x = b.y;
  }
  if (cudaHostAlloc(&m->ring, sizeof(StepDev) * 64, cudaHostAllocDefault) != cudaSuccess)
    return cleanup(cfail(DSX_ERR_CUDA, "pinned step-parameter ring"));
  m->ring_ev.assign(64, nullptr);
  for (auto& e : m->ring_ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  if (cudaStreamCreateWithPriority(&m->stream, cudaStreamNonBlocking, lo) != cudaSuccess ||
      cudaStreamCreateWithPriority(&m->side, cudaStreamNonBlocking, hi) != cudaSuccess)
    return cleanup(cfail(DSX_ERR_CUDA, "stream creation failed"));
  m->ev_upd.assign(m->L, nullptr);
  m->ev_sync.assign(m->L, nullptr);
  for (int l = 0; l < m->L; ++l) {
    cudaEventCreateWithFlags(&m->ev_upd[l], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&m->ev_sync[l], cudaEventDisableTiming);
  }
  for (auto& e : m->ev) cudaEventCreate(&e);
  for (auto& e : m->iev) cudaEventCreate(&e);
  m->synced_prev.assign(m->L, 0);
  const cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cleanup(cfail(DSX_ERR_CUDA, std::string("cnn init: ") + cudaGetErrorString(e)));
  *out = m;
  return DSX_OK;
}

dsx_status dsx_cnn_destroy(dsx_cnn* m) {
  if (!m) return DSX_OK;
  cudaSetDevice(m->device);
  if (m->stream) cudaStreamSynchronize(m->stream);
  if (m->side) cudaStreamSynchronize(m->side);
  if (m->comm) ncclCommDestroy(m->comm);
  for (void* p : m->owned) cudaFree(p);
  if (m->ring) cudaFreeHost(m->ring);
  for (auto e : m->ring_ev)
    if (e) cudaEventDestroy(e);
  for (auto e : m->ev_upd)
    if (e) cudaEventDestroy(e);
  for (auto e : m->ev_sync)
    if (e) cudaEventDestroy(e);
  for (auto e : m->ev)
    if (e) cudaEventDestroy(e);
  for (auto e : m->iev)
    if (e) cudaEventDestroy(e);
  if (m->stream) cudaStreamDestroy(m->stream);
  if (m->side) cudaStreamDestroy(m->side);
  delete m;
  return DSX_OK;
}

dsx_status dsx_cnn_param_layout(dsx_cnn* m, int* layers, uint64_t* total, uint64_t* offsets, int* fan_in) {
  if (!m) return cfail(DSX_ERR_ARGUMENT, "null cnn");
  if (layers) *layers = m->L;
  if (total) *total = (uint64_t)m->packed.back();
  if (offsets)
    for (int l = 0; l <= m->L; ++l) offsets[l] = (uint64_t)m->packed[l];
  if (fan_in)
    for (int l = 0; l < m->L; ++l) fan_in[l] = m->fan_in[l];
  return DSX_OK;
}

namespace {
dsx_status ccopy(dsx_cnn* m, float* dev, int local, float* host, bool to_dev) {
  for (int l = 0; l < m->L; ++l) {
    const long long n = m->packed[l + 1] - m->packed[l];
    float* d = dev + (long long)local * m->P + m->off[l];
    float* h = host + m->packed[l];
    CN_CUDA(cudaMemcpy(to_dev ? (void*)d : (void*)h, to_dev ? (void*)h : (void*)d, 4ull * n,
                       to_dev ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost));
  }
  return DSX_OK;
}
}  // namespace

dsx_status dsx_cnn_set_params(dsx_cnn* m, int local, const float* packed) {
  CN_TRY(ccheck(m));
  if (local < 0 || local >= m->kl || !packed) return cfail(DSX_ERR_ARGUMENT, "bad local worker / null params");
  CN_CUDA(cudaStreamSynchronize(m->side));
  CN_CUDA(cudaStreamSynchronize(m->stream));
  CN_TRY(ccopy(m, m->params, local, const_cast<float*>(packed), true));
  if (m->bf16) {
    cast_bf16_kernel<<<blocks_for(m->P, m->nsm), 256, 0, m->stream>>>(m->params + (long long)local * m->P,
                                                                     m->pbf + (long long)local * m->P, 0, 1, 0, m->P);
    CN_CUDA(cudaStreamSynchronize(m->stream));
  }
  return DSX_OK;
}

dsx_status dsx_cnn_get_params(dsx_cnn* m, int local, float* packed) {
  CN_TRY(ccheck(m));
  if (local < 0 || local >= m->kl || !packed) return cfail(DSX_ERR_ARGUMENT, "bad local worker / null params");
  CN_CUDA(cudaStreamSynchronize(m->side));
  CN_CUDA(cudaStreamSynchronize(m->stream));
  return ccopy(m, m->params, local, packed, false);
}

dsx_status dsx_cnn_set_batch(dsx_cnn* m, const float* x, const int32_t* labels, int on_device) {
  CN_TRY(ccheck(m));
  if (!x || !labels) return cfail(DSX_ERR_ARGUMENT, "null batch");
  if (on_device) {
    m->x_dev = x;
    m->labels_dev = labels;
    return DSX_OK;
  }
  const size_t nx = 4ull * m->kl * m->batch * m->image * m->image * m->cin, nl = 4ull * m->kl * m->batch;
  CN_CUDA(cudaMemcpyAsync(m->xin, x, nx, cudaMemcpyHostToDevice, m->stream));
  CN_CUDA(cudaMemcpyAsync(m->labels, labels, nl, cudaMemcpyHostToDevice, m->stream));
  m->x_dev = m->xin;
  m->labels_dev = m->labels;
  return DSX_OK;
}

dsx_status dsx_cnn_step(dsx_cnn* m, double lr, long long step_index, const unsigned char* mask) {
  CN_TRY(ccheck(m));
  if (!mask) return cfail(DSX_ERR_ARGUMENT, "null mask");
  CN_TRY(write_step(m, lr, step_index));
  return step_impl(m, lr, step_index, mask);
}

dsx_status dsx_cnn_last_loss(dsx_cnn* m, float* loss) {
  CN_TRY(ccheck(m));
  if (!loss) return cfail(DSX_ERR_ARGUMENT, "null out");
  CN_CUDA(cudaStreamSynchronize(m->stream));
  CN_CUDA(cudaMemcpy(loss, m->loss, 4ull * m->kl, cudaMemcpyDeviceToHost));
  return DSX_OK;
}

dsx_status dsx_cnn_sync(dsx_cnn* m) {
  CN_TRY(ccheck(m));
  CN_CUDA(cudaStreamSynchronize(m->side));
  CN_CUDA(cudaStreamSynchronize(m->stream));
  CN_CUDA(cudaGetLastError());
  return DSX_OK;
}

dsx_status dsx_cnn_comm_init(dsx_cnn* m, const unsigned char id[128], int nranks, int rank) {
  CN_TRY(ccheck(m));
  if (!id || nranks < 1 || rank < 0 || rank >= nranks) return cfail(DSX_ERR_ARGUMENT, "bad comm args");
  if (m->comm) return cfail(DSX_ERR_STATE, "comm already initialised");
  if (m->K != m->kl * nranks || m->kbegin != rank * m->kl)
    return cfail(DSX_ERR_ARGUMENT, "ranks must hold equal contiguous worker ranges");
  ncclUniqueId u;
  std::memcpy(u.internal, id, 128);
  CN_NCCL(ncclCommInitRank(&m->comm, nranks, u, rank));
  m->nranks = nranks;
  m->rank = rank;
  return DSX_OK;
}

dsx_status dsx_cnn_set_instrument(dsx_cnn* m, int enabled) {
  CN_TRY(ccheck(m));
  m->instrument = enabled != 0;
  return DSX_OK;
}

dsx_status dsx_cnn_last_step_times(dsx_cnn* m, float* out4) {
  CN_TRY(ccheck(m));
  if (!out4) return cfail(DSX_ERR_ARGUMENT, "null out");
  if (!m->instrument) return cfail(DSX_ERR_STATE, "instrumentation is off");
  CN_CUDA(cudaStreamWaitEvent(m->stream, m->iev[2], 0));
  CN_CUDA(cudaEventRecord(m->iev[3], m->stream));
  CN_CUDA(cudaEventSynchronize(m->iev[3]));
  float total = 0, comp = 0, span = 0, done = 0;
  CN_CUDA(cudaEventElapsedTime(&total, m->iev[0], m->iev[3]));
  CN_CUDA(cudaEventElapsedTime(&comp, m->iev[0], m->iev[1]));
  if (m->any_synced) {
    CN_CUDA(cudaEventElapsedTime(&span, m->ev[7], m->iev[2]));
    CN_CUDA(cudaEventElapsedTime(&done, m->iev[0], m->iev[2]));
  }
  out4[0] = total;
  out4[1] = comp;
  out4[2] = m->any_synced ? span : 0.f;
  out4[3] = m->any_synced ? std::max(0.f, done - comp) : 0.f;
  return DSX_OK;
}

dsx_status dsx_cnn_event_record(dsx_cnn* m, int slot) {
  CN_TRY(ccheck(m));
  if (slot < 0 || slot >= 7) return cfail(DSX_ERR_ARGUMENT, "slot must be in [0, 7)");
  CN_CUDA(cudaEventRecord(m->iev[2], m->side));
  CN_CUDA(cudaStreamWaitEvent(m->stream, m->iev[2], 0));
  CN_CUDA(cudaEventRecord(m->ev[slot], m->stream));
  return DSX_OK;
}

dsx_status dsx_cnn_event_elapsed(dsx_cnn* m, int a, int b, float* ms) {
  CN_TRY(ccheck(m));
  if (!ms || a < 0 || a >= 7 || b < 0 || b >= 7) return cfail(DSX_ERR_ARGUMENT, "bad slots");
  CN_CUDA(cudaEventSynchronize(m->ev[b]));
  CN_CUDA(cudaEventElapsedTime(ms, m->ev[a], m->ev[b]));
  return DSX_OK;
}

dsx_status dsx_cnn_profile(dsx_cnn* m, int reps, double* t_fp, double* t_bp, double* t_comm) {
  CN_TRY(ccheck(m));
  if (!t_fp || !t_bp || !t_comm) return cfail(DSX_ERR_ARGUMENT, "null out");
  reps = std::max(1, reps);
  CN_CUDA(cudaStreamSynchronize(m->side));
  CN_CUDA(cudaStreamSynchronize(m->stream));
  // the profile must not change the state: snapshot params / states, steps at lr 0
  const size_t arena = 4ull * m->P * m->kl;
  std::vector<std::pair<float*, void*>> keep;
  for (float* p : {m->params, m->mom, m->var}) {
    if (!p) continue;
    void* c = nullptr;
    CN_CUDA(cudaMalloc(&c, arena));
    keep.emplace_back(p, c);
    CN_CUDA(cudaMemcpy(c, p, arena, cudaMemcpyDeviceToDevice));
  }
  m->pf.assign(m->L + 1, nullptr);
  m->pb.assign(m->L + 1, nullptr);
  for (auto& e : m->pf) CN_CUDA(cudaEventCreate(&e));
  for (auto& e : m->pb) CN_CUDA(cudaEventCreate(&e));
  std::vector<std::vector<float>> fp(m->L), bp(m->L), cm(m->L);
  std::vector<unsigned char> none(m->L + 1, 0);
  const std::vector<unsigned char> prev = m->synced_prev;
  std::fill(m->synced_prev.begin(), m->synced_prev.end(), 0);
  dsx_status st = DSX_OK;
  m->prof = true;
  for (int r = 0; r < reps + 1 && st == DSX_OK; ++r) {
    st = write_step(m, 0.0, 0);
    if (st == DSX_OK) st = step_impl(m, 0.0, 0, none.data());
    if (st != DSX_OK) break;
    CN_CUDA(cudaStreamSynchronize(m->stream));
    if (r == 0) continue;
    for (int l = 0; l < m->L; ++l) {
      float t = 0;
      CN_CUDA(cudaEventElapsedTime(&t, m->pf[l], m->pf[l + 1]));
      fp[l].push_back(t);
      CN_CUDA(cudaEventElapsedTime(&t, m->pb[l + 1 < m->L ? l + 1 : m->L], m->pb[l]));
      bp[l].push_back(t);
    }
  }
  m->prof = false;
  cudaEvent_t e0 = m->pf[0], e1 = m->pf[1];
  for (int r = 0; r < reps + 1 && m->K > 1 && st == DSX_OK; ++r) {
    for (int l = 0; l < m->L; ++l) {
      CN_CUDA(cudaEventRecord(e0, m->side));
      st = average_layer(m, l, m->side);
      if (st != DSX_OK) break;
      CN_CUDA(cudaEventRecord(e1, m->side));
      CN_CUDA(cudaEventSynchronize(e1));
      float t = 0;
      CN_CUDA(cudaEventElapsedTime(&t, e0, e1));
      if (r > 0) cm[l].push_back(t);
    }
  }
  CN_CUDA(cudaStreamSynchronize(m->side));
  CN_CUDA(cudaStreamSynchronize(m->stream));
  for (auto& [p, c] : keep) {
    CN_CUDA(cudaMemcpy(p, c, arena, cudaMemcpyDeviceToDevice));
    cudaFree(c);
  }
  if (m->bf16)
    cast_bf16_kernel<<<blocks_for(m->P * m->kl, m->nsm), 256, 0, m->stream>>>(m->params, m->pbf, m->P, m->kl, 0,
                                                                             m->P);
  CN_CUDA(cudaStreamSynchronize(m->stream));
  for (auto e : m->pf) cudaEventDestroy(e);
  for (auto e : m->pb) cudaEventDestroy(e);
  m->pf.clear();
  m->pb.clear();
  m->synced_prev = prev;
  if (st != DSX_OK) return st;
  auto med = [](std::vector<float> v) {
    if (v.empty()) return 0.0;
    std::sort(v.begin(), v.end());
    return (double)v[v.size() / 2] * 1e-3;
  };
  for (int l = 0; l < m->L; ++l) {
    t_fp[l] = med(fp[l]);
    t_bp[l] = med(bp[l]);
    t_comm[l] = med(cm[l]);
  }
  return DSX_OK;
}

dsx_status dsx_cnn_set_link(dsx_cnn* m, double bandwidth, double latency) {
  CN_TRY(ccheck(m));
  if (!(latency >= 0.0)) return cfail(DSX_ERR_ARGUMENT, "latency must be >= 0");
  m->link_bw = bandwidth > 0.0 ? bandwidth : 0.0;
  m->link_lat = latency;
  return DSX_OK;
}

dsx_status dsx_cnn_set_overlap(dsx_cnn* m, int enabled) {
  CN_TRY(ccheck(m));
  m->overlap = enabled != 0;
  return DSX_OK;
}

dsx_status dsx_cnn_launch_count(dsx_cnn* m, uint64_t* out) {
  if (!m || !out) return cfail(DSX_ERR_ARGUMENT, "null argument");
  *out = m->launches;
  return DSX_OK;
}

}  // extern "C"
