// nn_kernels.cuh — the element-wise / reduction kernels the NN local steps
// share (MLP: nn.cu, conv stack: cnn.cu): softmax cross-entropy, bias
// column sums, the fused per-layer optimizer, the cross-worker averages of a
// parameter range, the throttled-link spin, and the per-step device scalars
// a replayed CUDA graph reads.  Internal linkage: each including TU owns its
// copy.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdint>
#include <string>

#include "dsx.h"
#include "dsx_nn.h"
#include "nn_gemm.cuh"

namespace dsx_nn {
namespace {

// Per-step scalars and data pointers, read by the kernels from device memory
// so that one captured CUDA graph per sync mask replays every step.
struct StepDev {
  float lr, bc1, bc2, pad;
  const float* x;
  const int* labels;
};

// ---------------------------------------------------------------------------
// MLP kernels
// ---------------------------------------------------------------------------

// Softmax cross-entropy over C classes per sample (one warp per sample):
// loss partials, and dlogits = (softmax - onehot) / batch written in T.
template <typename T>
__global__ void softmax_xent_kernel(const float* __restrict__ logits, long long ld_logit, long long s_logit,
                                    const int* __restrict__ labels_arg, int batch, int C, T* __restrict__ dz,
                                    long long ld_dz, long long s_dz, float* __restrict__ loss_part,
                                    const StepDev* __restrict__ sp) {
  pdl_enter();
  const int* __restrict__ labels = sp ? sp->labels : labels_arg;
  const int b = blockIdx.y;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= batch) return;
  const float* z = logits + b * s_logit + (long long)warp * ld_logit;
  float mx = -INFINITY;
  for (int c = lane; c < C; c += 32) mx = fmaxf(mx, z[c]);
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float se = 0.f;
  for (int c = lane; c < C; c += 32) se += expf(z[c] - mx);
  for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
  const int y = labels[(long long)b * batch + warp];
  const float lse = mx + logf(se);
  T* d = dz + b * s_dz + (long long)warp * ld_dz;
  const float inv = 1.f / (float)batch;
  for (int c = lane; c < C; c += 32) {
    const float p = expf(z[c] - lse);
    d[c] = from_f<T>((p - (c == y ? 1.f : 0.f)) * inv);
  }
  if (lane == 0) loss_part[(long long)b * batch + warp] = lse - z[y];
}

// loss[b] = mean over the batch of loss_part (fixed order)
__global__ void loss_mean_kernel(const float* __restrict__ part, int batch, float* __restrict__ loss) {
  pdl_enter();
  const int b = blockIdx.x;
  __shared__ float sh[256];
  float s = 0.f;
  for (int i = threadIdx.x; i < batch; i += blockDim.x) s += part[(long long)b * batch + i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) loss[b] = sh[0] / (float)batch;
}

// db[b][n] = sum over rows of dz[b][row][n] (bias gradient).  256 threads
// = 32 columns x 8 row groups; each thread sums every 8th row (8 loads in
// flight), the 8 partial sums are added in a fixed order: deterministic.
template <typename T>
__global__ void __launch_bounds__(256) colsum_kernel(const T* __restrict__ dz, long long ld, long long s_dz, int rows,
                                                     int n_out, float* __restrict__ db, long long s_db) {
  pdl_enter();
  __shared__ float part[8][33];
  const int b = blockIdx.y;
  const int cx = threadIdx.x & 31, rg = threadIdx.x >> 5;
  const int n = blockIdx.x * 32 + cx;
  float s = 0.f;
  if (n < n_out) {
    const T* p = dz + b * s_dz + n;
    int r = rg;
    for (; r + 56 < rows; r += 64) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = to_f<T>(p[(long long)(r + 8 * u) * ld]);
#pragma unroll
      for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; r < rows; r += 8) s += to_f<T>(p[(long long)r * ld]);
  }
  part[rg][cx] = s;
  __syncthreads();
  if (rg == 0 && n < n_out) {
    float t = part[0][cx];
#pragma unroll
    for (int g = 1; g < 8; ++g) t += part[g][cx];
    db[b * s_db + n] = t;
  }
}

struct OptArgs {
  int kind;
  float lr, mu, b1, b2, eps, wd, bc1, bc2;  // bc = 1 - beta^t
};

__device__ __forceinline__ float opt_one(const OptArgs& o, float w, float g, float* m, float* v) {
  if (o.kind == DSX_OPT_SGD) {
    if (o.wd != 0.f) g += o.wd * w;
    return w - o.lr * g;
  }
  if (o.kind == DSX_OPT_MOMENTUM) {
    if (o.wd != 0.f) g += o.wd * w;
    *m = o.mu * *m + g;
    return w - o.lr * *m;
  }
  // Adam(W)
  *m = o.b1 * *m + (1.f - o.b1) * g;
  *v = o.b2 * *v + (1.f - o.b2) * g * g;
  const float mh = *m / o.bc1, vh = *v / o.bc2;
  return w - o.lr * (mh / (sqrtf(vh) + o.eps) + o.wd * w);
}

// Fused optimizer over one layer range [lo, lo+n) of every local worker
// (blockIdx.y): reads w, g (+ states), writes w, states and the bf16 GEMM
// copy.  HBM-bound: 16-B vector loads/stores (lo is 64-element aligned),
// two vectors per thread in flight, scalar tail.
__global__ void __launch_bounds__(256) optimizer_kernel(float* __restrict__ w, const float* __restrict__ g,
                                                        float* __restrict__ m, float* __restrict__ v,
                                                        __nv_bfloat16* __restrict__ wb, long long ld, long long lo,
                                                        long long n, OptArgs o, const StepDev* __restrict__ sp) {
  pdl_enter();
  if (sp) {
    o.lr = sp->lr;
    o.bc1 = sp->bc1;
    o.bc2 = sp->bc2;
  }
  const long long base = (long long)blockIdx.y * ld + lo;
  const long long nv4 = n / 4;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const bool mom = o.kind != DSX_OPT_SGD, adam = o.kind == DSX_OPT_ADAM;
  auto vec = [&](long long q) {
    const long long j = base + 4 * q;
    float4 wv = *reinterpret_cast<const float4*>(w + j);
    const float4 gv = *reinterpret_cast<const float4*>(g + j);
    float4 mv = mom ? *reinterpret_cast<const float4*>(m + j) : make_float4(0.f, 0.f, 0.f, 0.f);
    float4 vv = adam ? *reinterpret_cast<const float4*>(v + j) : make_float4(0.f, 0.f, 0.f, 0.f);
    wv.x = opt_one(o, wv.x, gv.x, &mv.x, &vv.x);
    wv.y = opt_one(o, wv.y, gv.y, &mv.y, &vv.y);
    wv.z = opt_one(o, wv.z, gv.z, &mv.z, &vv.z);
    wv.w = opt_one(o, wv.w, gv.w, &mv.w, &vv.w);
    *reinterpret_cast<float4*>(w + j) = wv;
    if (mom) *reinterpret_cast<float4*>(m + j) = mv;
    if (adam) *reinterpret_cast<float4*>(v + j) = vv;
    if (wb) {
      __nv_bfloat162* d = reinterpret_cast<__nv_bfloat162*>(wb + j);
      d[0] = __floats2bfloat162_rn(wv.x, wv.y);
      d[1] = __floats2bfloat162_rn(wv.z, wv.w);
    }
  };
  long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; q + stride < nv4; q += 2 * stride) {
    vec(q);
    vec(q + stride);
  }
  if (q < nv4) vec(q);
  for (long long i = 4 * nv4 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    const long long j = base + i;
    float mj = mom ? m[j] : 0.f, vj = adam ? v[j] : 0.f;
    const float wj = opt_one(o, w[j], g[j], &mj, &vj);
    w[j] = wj;
    if (mom) m[j] = mj;
    if (adam) v[j] = vj;
    if (wb) wb[j] = __float2bfloat16_rn(wj);
  }
}

// pairwise_coord_sum's tree (trainer.cpp:31-38) over KL local rows
template <int LO, int HI>
__device__ __forceinline__ float ptree(const float* v) {
  if constexpr (HI - LO == 1) return v[LO];
  else if constexpr (HI - LO == 2) return v[LO] + v[LO + 1];
  else return ptree<LO, LO + (HI - LO) / 2>(v) + ptree<LO + (HI - LO) / 2, HI>(v);
}

// Average of a layer range across the KL local workers (one rank): every
// worker's copy (and its bf16 twin) becomes the pairwise mean / K.
template <int KL>
__global__ void local_average_kernel(float* __restrict__ w, __nv_bfloat16* __restrict__ wb, long long ld, long long lo,
                                     long long n, float inv_k) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float v[KL];
#pragma unroll
    for (int k = 0; k < KL; ++k) v[k] = w[(long long)k * ld + lo + i];
    const float mean = ptree<0, KL>(v) * inv_k;
#pragma unroll
    for (int k = 0; k < KL; ++k) {
      w[(long long)k * ld + lo + i] = mean;
      if (wb) wb[(long long)k * ld + lo + i] = __float2bfloat16_rn(mean);
    }
  }
}

// multi-rank with several local rows: row 0 <- local pairwise sum (then the
// NCCL sum over ranks), afterwards every row <- sum / K
template <int KL>
__global__ void local_sum_kernel(float* __restrict__ w, long long ld, long long lo, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float v[KL];
#pragma unroll
    for (int k = 0; k < KL; ++k) v[k] = w[(long long)k * ld + lo + i];
    w[lo + i] = ptree<0, KL>(v);
  }
}
__global__ void scale_broadcast_kernel(float* __restrict__ w, __nv_bfloat16* __restrict__ wb, long long ld, int kl,
                                       long long lo, long long n, float inv_k) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float mean = w[lo + i] * inv_k;
    for (int k = 0; k < kl; ++k) {
      w[(long long)k * ld + lo + i] = mean;
      if (wb) wb[(long long)k * ld + lo + i] = __float2bfloat16_rn(mean);
    }
  }
}
__global__ void cast_bf16_kernel(const float* __restrict__ w, __nv_bfloat16* __restrict__ wb, long long ld, int kl,
                                 long long lo, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    for (int k = 0; k < kl; ++k) wb[(long long)k * ld + lo + i] = __float2bfloat16_rn(w[(long long)k * ld + lo + i]);
}
// Throttled link (the paper's low-bandwidth regime): the sync stream is a
// FIFO link; after a layer's average it stays busy latency + bytes/bandwidth
// (comm_time, profile.cpp:103-110).
__global__ void nn_link_spin_kernel(unsigned long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(500);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

// the step's input batch -> act[0] (bf16 for the tensor-core path)
template <typename T>
__global__ void load_x_kernel(const StepDev* __restrict__ sp, T* __restrict__ y, long long n) {
  pdl_enter();
  const float* __restrict__ x = sp->x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = from_f<T>(x[i]);
}


// split-K partials -> out: out[b*s_out + i] = sum_s part[s*s_split + b*n + i]
// in split order (deterministic); n elements per batch entry (blockIdx.y)
__global__ void splitk_reduce_kernel(const float* __restrict__ part, int ks, long long s_split, long long n,
                                     float* __restrict__ out, long long s_out) {
  pdl_enter();
  const long long b = blockIdx.y;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    // 8 loads in flight, summed in split order
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
    out[b * s_out + i] = acc;
  }
}

inline int blocks_for(long long n, int nsm) {
  return (int)std::max<long long>(1, std::min<long long>((n + 255) / 256, nsm * 8LL));
}

// Average of one parameter range [lo, lo+n) of every worker (K in total, kl
// here, arena stride P) on stream s, fp32 masters + bf16 twin (wb may be
// null): local pairwise kernel on one rank; ncclAvg in place across ranks
// with one local worker; local pairwise sum + ncclSum + 1/K otherwise.
// Returns the launches issued through *launches.
inline dsx_status average_range(float* w, __nv_bfloat16* wb, long long P, int kl, int K, int nranks, ncclComm_t comm,
                                long long lo, long long n, int nsm, cudaStream_t s, uint64_t* launches,
                                std::string* err) {
  const float inv = 1.f / (float)K;
  const int nb = blocks_for(n, nsm);
  auto nccl = [&](ncclResult_t r) {
    if (r != ncclSuccess) *err = std::string("NCCL: ") + ncclGetErrorString(r);
    return r == ncclSuccess;
  };
  if (nranks == 1) {
    if (kl == 1) return DSX_OK;
    switch (kl) {
      case 2: local_average_kernel<2><<<nb, 256, 0, s>>>(w, wb, P, lo, n, inv); break;
      case 4: local_average_kernel<4><<<nb, 256, 0, s>>>(w, wb, P, lo, n, inv); break;
      case 8: local_average_kernel<8><<<nb, 256, 0, s>>>(w, wb, P, lo, n, inv); break;
      default: *err = "local workers must be 1, 2, 4 or 8"; return DSX_ERR_ARGUMENT;
    }
    ++*launches;
    return DSX_OK;
  }
  if (kl == 1) {
    if (!nccl(ncclAllReduce(w + lo, w + lo, (size_t)n, ncclFloat, ncclAvg, comm, s))) return DSX_ERR_NCCL;
    if (wb) {
      cast_bf16_kernel<<<nb, 256, 0, s>>>(w, wb, P, 1, lo, n);
      ++*launches;
    }
    return DSX_OK;
  }
  switch (kl) {
    case 2: local_sum_kernel<2><<<nb, 256, 0, s>>>(w, P, lo, n); break;
    case 4: local_sum_kernel<4><<<nb, 256, 0, s>>>(w, P, lo, n); break;
    case 8: local_sum_kernel<8><<<nb, 256, 0, s>>>(w, P, lo, n); break;
    default: *err = "local workers must be 1, 2, 4 or 8"; return DSX_ERR_ARGUMENT;
  }
  if (!nccl(ncclAllReduce(w + lo, w + lo, (size_t)n, ncclFloat, ncclSum, comm, s))) return DSX_ERR_NCCL;
  scale_broadcast_kernel<<<nb, 256, 0, s>>>(w, wb, P, kl, lo, n, inv);
  *launches += 2;
  return DSX_OK;
}

}  // namespace
}  // namespace dsx_nn
