// lab.cu — the B200 partial-synchronization local-SGD engine behind dsx.h.
//
// HBM layout (one device, one rank):
//   w      [workers_local][ld]  parameter arena, T = double|float, ld = dim
//                               rounded up to 64 elements (256 B rows); each
//                               registered layer is a contiguous coordinate
//                               range, so a sync set is a byte range.
//   noise  [workers_local][ld]  fp64 per-coordinate noise (sigma > 0 only)
//   mt     [workers_local][313] std::mt19937_64 state (x[312], cursor)
//   curv/opt [dim] fp64         only when the problem is not make_quadratic-
//                               shaped (otherwise lambda_i is recomputed
//                               in-kernel with the reference's exact formula)
//
// One plsgd_step (reference trainer.cpp:187-235) on a single rank is
//   [noise engine]  ->  lab_update (fused: gradient, ||g||^2 partials,
//   SGD update AND, for masked blocks, the pairwise cross-worker mean written
//   back to every row)  ->  norm finalize.
// The update+average kernel touches each parameter exactly once (read K
// rows, write K rows): the reference's separate averaging pass costs no
// extra HBM traffic here.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <random>
#include <sstream>
#include <string>
#include <type_traits>
#include <vector>

#include "device_once.cuh"
#include "dsx.h"
#include "mt_engine.cuh"
#include "noise_engine.cuh"

namespace dsx {

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
thread_local std::string g_last_error;

static dsx_status fail(dsx_status code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define DSX_CUDA(expr)                                                                 \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return ::dsx::fail(DSX_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define DSX_NCCL(expr)                                                                 \
  do {                                                                                 \
    ncclResult_t r_ = (expr);                                                          \
    if (r_ != ncclSuccess)                                                             \
      return ::dsx::fail(DSX_ERR_NCCL, std::string(#expr) + ": " + ncclGetErrorString(r_)); \
  } while (0)

#define DSX_TRY(expr)                      \
  do {                                     \
    dsx_status s_ = (expr);                \
    if (s_ != DSX_OK) return s_;           \
  } while (0)

// ---------------------------------------------------------------------------
// kernel parameter blocks
// ---------------------------------------------------------------------------
constexpr int kTile = 8192;       // default coordinates per CTA (never crosses a block; DSX_TILE)
constexpr int kThreads = 256;
constexpr int kMaxMaskWords = 128;  // 4096 layers
constexpr int kMaxProg = 64;        // generic pairwise program (K <= 64)
constexpr int kMaxChunks = 8;
constexpr int kNoiseBatch = 8;   // steps per noise-engine run when pipelining (DSX_NOISE_BATCH)

struct Tile {
  long long start;
  int len;
  int block;  // 0-based layer index
};

struct MaskBits {
  uint32_t w[kMaxMaskWords];
};

__host__ __device__ __forceinline__ bool mask_has(const MaskBits& m, int block) {
  return (m.w[block >> 5] >> (block & 31)) & 1u;
}

// Postorder program of the reference's pairwise_coord_sum tree
// (trainer.cpp:31-38) for a runtime worker count: step j computes
// v[dst] = v[a] + v[b].
struct PairProg {
  int n;
  unsigned char dst[kMaxProg], a[kMaxProg], b[kMaxProg];
};

struct QuadParams {
  bool analytic;
  double mu, beta_minus_mu, dim_minus_1, opt_value;
  const double* curv;
  const double* opt;
};

// ranks whose scratch buffer (the NVLink probe's) is mapped into every peer
constexpr int kMaxFuse = 8;

template <typename T>
struct UpdateArgs {
  T* w;
  long long ld;
  int kl;             // rows held here
  int k_total;        // K (divisor of the mean)
  const Tile* tiles;
  int ntiles;
  int tile_base;      // first tile of this launch (split launches for overlap)
  const double* noise;  // [kl][ld] flat noise (NM == 1)
  NoiseView nv;         // segmented engine output (NM == 2)
  double eta;
  QuadParams q;
  MaskBits mask;
  bool average;       // average masked blocks in-kernel (single rank)
  double* norm_part;  // [kl][ntiles]
  T* partial_out;     // multi-rank: subtree sums of synced tiles (else null)
  const T* mean_in;   // multi-rank: cross-rank means of the layers in `stale`
  MaskBits stale;     // layers whose rows are stale: every row equals mean_in
};

// lambda_i and w*_i.  The analytic form is make_quadratic's
// mu + (beta - mu) * i / (dim - 1) (trainer.cpp:117-120), evaluated with the
// same rounding sequence.
__device__ __forceinline__ void quad_coeffs(const QuadParams& q, long long i, double* lam,
                                            double* opt) {
  if (q.analytic) {
    *lam = q.dim_minus_1 == 0.0
               ? q.mu
               : __dadd_rn(q.mu, __ddiv_rn(__dmul_rn(q.beta_minus_mu, (double)i), q.dim_minus_1));
    *opt = q.opt_value;
  } else {
    *lam = q.curv[i];
    *opt = q.opt[i];
  }
}

// pairwise_coord_sum over v[LO..HI) with the reference's split at n/2.
template <int LO, int HI, typename T>
__device__ __forceinline__ T psum(const T* v) {
  constexpr int N = HI - LO;
  if constexpr (N == 1) {
    return v[LO];
  } else if constexpr (N == 2) {
    return v[LO] + v[LO + 1];
  } else {
    constexpr int MID = LO + N / 2;
    return psum<LO, MID, T>(v) + psum<MID, HI, T>(v);
  }
}

// Pairwise sum over the R ranks' values (split at R/2, like the in-process tree)
template <typename T>
__device__ __forceinline__ T rank_psum(const T* v, int R) {
  switch (R) {
    case 2: return psum<0, 2, T>(v);
    case 4: return psum<0, 4, T>(v);
    case 8: return psum<0, 8, T>(v);
    case 3: return psum<0, 3, T>(v);
    case 5: return psum<0, 5, T>(v);
    case 6: return psum<0, 6, T>(v);
    case 7: return psum<0, 7, T>(v);
    default: return v[0];
  }
}

template <typename T>
__device__ __forceinline__ T run_prog(const PairProg& p, T* v) {
  for (int j = 0; j < p.n; ++j) v[p.dst[j]] = v[p.a[j]] + v[p.b[j]];
  return v[0];
}

__device__ __forceinline__ double block_sum(double x, double* red) {
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = x;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
  }
  return s;  // valid in thread 0
}

__device__ __forceinline__ double to_d(double x) { return x; }
__device__ __forceinline__ double to_d(float x) { return (double)x; }

// g = lambda*(w - w*) (+ xi);  w' = w - eta*g   — in T arithmetic.
__device__ __forceinline__ double grad_step(double w, double lam, double opt, double xi,
                                            double eta, bool noise, double* wout) {
  double g = __dmul_rn(lam, __dsub_rn(w, opt));
  if (noise) g = __dadd_rn(g, xi);
  *wout = __dsub_rn(w, __dmul_rn(eta, g));
  return g;
}
__device__ __forceinline__ float grad_step(float w, double lam, double opt, double xi, double eta,
                                           bool noise, float* wout) {
  float g = __fmul_rn((float)lam, __fsub_rn(w, (float)opt));
  if (noise) g = __fadd_rn(g, (float)xi);
  *wout = __fsub_rn(w, __fmul_rn((float)eta, g));
  return g;
}

// ---------------------------------------------------------------------------
// fused local step (+ in-place averaging of masked blocks on a single rank)
// KL > 0: compile-time local worker count; KL == 0: runtime count via prog.
// ---------------------------------------------------------------------------
template <typename T>
struct Vec2;
template <>
struct Vec2<double> {
  using type = double2;
};
template <>
struct Vec2<float> {
  using type = float2;
};

// Segmented engine lookup: normal i of worker k (in the run's step t, whose
// first pair is base = t*ceil(dim/2)) is pair m = base + i/2; it lives in
// segment s with pfx[s] <= m < pfx[s+1], at slot offset 2*(m - pfx[s]) + (i&1).
__device__ __forceinline__ int seg_search(const unsigned long long* pf, int P, unsigned long long m) {
  int lo = 0, hi = P;  // answer in [0, P]
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pf[mid] <= m) lo = mid; else hi = mid - 1;
  }
  return lo;
}

template <bool RAW>
__device__ __forceinline__ double seg_noise(const NoiseView& nv, int k, int seg, long long i) {
  const unsigned long long* pf = nv.pfx + (long long)k * (nv.P + 2);
  const unsigned long long m = nv.base + ((unsigned long long)i >> 1);
  const double* at = nv.slots + ((long long)k * (nv.P + 1) + seg) * nv.cap + 2 * (long long)(m - pf[seg]);
  if constexpr (RAW) {  // the accepted attempt (x, y) of pair m -> its two normals
    const double2 n = mt_polar_normals(at[0], at[1], nv.stddev);
    return (i & 1) ? n.y : n.x;
  }
  return at[i & 1];
}

// NM: 0 no noise, 1 flat noise buffer, 2 segmented engine output.
template <typename T, int KL, int NM>
__global__ void __launch_bounds__(kThreads, 2)
lab_update_kernel(UpdateArgs<T> a, PairProg prog) {
  constexpr int KMAX = KL > 0 ? KL : kMaxProg;
  constexpr bool NOISE = NM != 0;
  constexpr bool SEG = NM >= 2;   // engine segments: 2 finished normals, 3 raw attempts
  const int tile_id = a.tile_base + blockIdx.x;
  const Tile t = a.tiles[tile_id];
  const int kl = KL > 0 ? KL : a.kl;
  const bool avg = a.average && mask_has(a.mask, t.block);
  const bool part = KL > 1 && a.partial_out != nullptr && mask_has(a.mask, t.block);
  T* const part_dst = a.partial_out;
  // lazy broadcast: after a cross-rank average the mean lives once in the
  // exchange buffer; all kl rows are logically equal to it, so it is read
  // once instead of kl times (and the rows are never written back while the
  // layer keeps being synced)
  const bool stale = KL > 1 && a.mean_in != nullptr && mask_has(a.stale, t.block);
  double nsq[KMAX];
#pragma unroll
  for (int k = 0; k < KMAX; ++k) nsq[k] = 0.0;
  // Engine noise of coordinate i lives at slot_seg[i - 2*pfx[seg]]: per tile
  // and worker the tile spans at most two segments (segments hold >= 7.8k
  // pairs, a tile 1024), so one boundary + two rebased base pointers suffice.
  __shared__ const double* s_base[KL > 0 ? KL : 1][2];
  __shared__ unsigned long long s_bound[KL > 0 ? KL : 1];
  __shared__ int s_simple;
  if constexpr (SEG && KL > 0) {
    if (threadIdx.x == 0) s_simple = 1;
    __syncthreads();
    if (threadIdx.x < KL) {
      const int k = threadIdx.x;
      const unsigned long long* pf = a.nv.pfx + (long long)k * (a.nv.P + 2);
      const unsigned long long m0 = a.nv.base + ((unsigned long long)t.start >> 1);
      const unsigned long long m1 = a.nv.base + ((unsigned long long)(t.start + t.len - 1) >> 1);
      const int s0 = seg_search(pf, a.nv.P, m0);
      const int s1 = s0 < a.nv.P ? s0 + 1 : s0;
      const double* slot0 = a.nv.slots + ((long long)k * (a.nv.P + 1) + s0) * a.nv.cap;
      const double* slot1 = a.nv.slots + ((long long)k * (a.nv.P + 1) + s1) * a.nv.cap;
      // rebased so that s_base[k][.] + i addresses coordinate i's normal
      s_base[k][0] = slot0 - 2 * (long long)pf[s0] + 2 * (long long)a.nv.base;
      s_base[k][1] = slot1 - 2 * (long long)pf[s1] + 2 * (long long)a.nv.base;
      s_bound[k] = s0 < a.nv.P ? pf[s0 + 1] - a.nv.base : ~0ull;
      if (s1 < a.nv.P && m1 >= pf[s1 + 1]) s_simple = 0;  // spans 3+ segments
    }
    __syncthreads();
  }

  if constexpr (KL > 0) {
    // Coordinate pairs (i, i+1), i even: 16-byte (fp64) / 8-byte (fp32)
    // vector loads/stores of every row and of the engine noise (its
    // segments start at even coordinates, so a pair never straddles one).
    // An odd tile start / end is handled as a scalar head / tail.
    using V2 = typename Vec2<T>::type;
    const long long first = t.start + (t.start & 1);
    const long long end = t.start + t.len;
    const int npairs = (int)((end - first) >> 1);
    auto noise_at = [&](int k, long long i) -> double {
      if constexpr (NM == 1) return a.noise[k * a.ld + i];
      if constexpr (SEG) {
        if (s_simple) {
          const double* at = s_base[k][((unsigned long long)i >> 1) >= s_bound[k]];
          if constexpr (NM == 2) {
            return at[i];
          } else {
            const double2 n = mt_polar_normals(at[i & ~1LL], at[(i & ~1LL) + 1], a.nv.stddev);
            return (i & 1) ? n.y : n.x;
          }
        }
        const int sg = seg_search(a.nv.pfx + (long long)k * (a.nv.P + 2), a.nv.P,
                                  a.nv.base + ((unsigned long long)i >> 1));
        return seg_noise<NM == 3>(a.nv, k, sg, i);
      }
      return 0.0;
    };
    auto scalar = [&](long long i) {
      double lam, opt;
      quad_coeffs(a.q, i, &lam, &opt);
      T wn[KL];
#pragma unroll
      for (int k = 0; k < KL; ++k) {
        const auto g = grad_step(stale ? a.mean_in[i] : a.w[k * a.ld + i], lam, opt, noise_at(k, i),
                                 a.eta, NOISE, &wn[k]);
        nsq[k] += to_d(g) * to_d(g);
      }
      if (part) {
        part_dst[i] = psum<0, KL, T>(wn);
        return;
      }
      const T m = avg ? psum<0, KL, T>(wn) / (T)a.k_total : T(0);
#pragma unroll
      for (int k = 0; k < KL; ++k) a.w[k * a.ld + i] = avg ? m : wn[k];
    };
    if (threadIdx.x == 0 && first != t.start) scalar(t.start);
    if (threadIdx.x == 1 && first + 2 * (long long)npairs < end) scalar(end - 1);
    // Main loop, specialised per tile on (stale rows, simple noise
    // addressing) so that every row load and every noise load of an
    // iteration is independent and issued back to back: the noise base of
    // worker k is one of two rebased pointers (a select, no dependent chain),
    // and noise — read exactly once — is streamed with evict-first loads.
    auto pairs = [&](auto stale_c, auto simple_c) {
      constexpr bool STALE = decltype(stale_c)::value;
      constexpr bool SIMPLE = decltype(simple_c)::value;
      // U pairs per thread per iteration, all their loads issued before any
      // compute: with 1-2 local rows a single pair keeps too few bytes in
      // flight to cover HBM latency (ncu, 2 rows: long_scoreboard 59 %,
      // 0.53 of DRAM peak)
      constexpr int U = KL >= 4 ? 1 : (KL == 2 ? 2 : 4);
      for (int pr0 = threadIdx.x; pr0 < npairs; pr0 += kThreads * U) {
        V2 wv[U][KL];
        double2 xv[U][KL];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int pr = pr0 + u * kThreads;
          if (pr >= npairs) break;
          const long long i = first + 2 * (long long)pr;
          if constexpr (STALE) {
            const V2 m = *reinterpret_cast<const V2*>(a.mean_in + i);
#pragma unroll
            for (int k = 0; k < KL; ++k) wv[u][k] = m;
          } else {
#pragma unroll
            for (int k = 0; k < KL; ++k) wv[u][k] = *reinterpret_cast<const V2*>(a.w + k * a.ld + i);
          }
          if constexpr (NM == 1) {
#pragma unroll
            for (int k = 0; k < KL; ++k)
              xv[u][k] = __ldcs(reinterpret_cast<const double2*>(a.noise + k * a.ld + i));
          }
          if constexpr (SEG) {
            if constexpr (SIMPLE) {
              const unsigned long long m = (unsigned long long)i >> 1;
              const double* np[KL];
#pragma unroll
              for (int k = 0; k < KL; ++k) np[k] = s_base[k][m >= s_bound[k] ? 1 : 0];
#pragma unroll
              for (int k = 0; k < KL; ++k) xv[u][k] = __ldcs(reinterpret_cast<const double2*>(np[k] + i));
            } else {
#pragma unroll
              for (int k = 0; k < KL; ++k) xv[u][k] = make_double2(noise_at(k, i), noise_at(k, i + 1));
            }
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int pr = pr0 + u * kThreads;
          if (pr >= npairs) break;
          const long long i = first + 2 * (long long)pr;
          double lam0, opt0, lam1, opt1;
          quad_coeffs(a.q, i, &lam0, &opt0);
          quad_coeffs(a.q, i + 1, &lam1, &opt1);
          if constexpr (NM == 3 && SIMPLE) {
            // the polar transform of the engine's raw attempts, here where
            // the issue slots idle on HBM latency anyway
#pragma unroll
            for (int k = 0; k < KL; ++k) xv[u][k] = mt_polar_normals(xv[u][k].x, xv[u][k].y, a.nv.stddev);
          }
          T w0[KL], w1[KL];
#pragma unroll
          for (int k = 0; k < KL; ++k) {
            const double x0 = NOISE ? xv[u][k].x : 0.0, x1 = NOISE ? xv[u][k].y : 0.0;
            const auto g0 = grad_step(wv[u][k].x, lam0, opt0, x0, a.eta, NOISE, &w0[k]);
            const auto g1 = grad_step(wv[u][k].y, lam1, opt1, x1, a.eta, NOISE, &w1[k]);
            nsq[k] += to_d(g0) * to_d(g0) + to_d(g1) * to_d(g1);
          }
          if (avg) {
            V2 m;
            m.x = psum<0, KL, T>(w0) / (T)a.k_total;
            m.y = psum<0, KL, T>(w1) / (T)a.k_total;
#pragma unroll
            for (int k = 0; k < KL; ++k) *reinterpret_cast<V2*>(a.w + k * a.ld + i) = m;
          } else if (part) {
            // multi-rank synced tile: only this rank's subtree sum leaves the
            // kernel; the rows are rewritten by the cross-rank average
            V2 m;
            m.x = psum<0, KL, T>(w0);
            m.y = psum<0, KL, T>(w1);
            *reinterpret_cast<V2*>(part_dst + i) = m;
          } else {
#pragma unroll
            for (int k = 0; k < KL; ++k) {
              V2 o;
              o.x = w0[k];
              o.y = w1[k];
              *reinterpret_cast<V2*>(a.w + k * a.ld + i) = o;
            }
          }
        }
      }
    };
    using Yes = std::true_type;
    using No = std::false_type;
    const bool simple = !SEG || s_simple;
    if (stale) {
      if (simple) pairs(Yes{}, Yes{}); else pairs(Yes{}, No{});
    } else {
      if (simple) pairs(No{}, Yes{}); else pairs(No{}, No{});
    }
  } else {
    // generic worker count: row pass, then the pairwise program for
    // averaged coordinates.
    T v[KMAX];
    for (int off = threadIdx.x; off < t.len; off += kThreads) {
      const long long i = t.start + off;
      double lam, opt;
      quad_coeffs(a.q, i, &lam, &opt);
      for (int k = 0; k < kl; ++k) {
        const T w = a.w[k * a.ld + i];
        double xi = 0.0;
        if constexpr (NM == 1) xi = a.noise[k * a.ld + i];
        if constexpr (SEG) {
          const int s = seg_search(a.nv.pfx + (long long)k * (a.nv.P + 2), a.nv.P,
                                   a.nv.base + ((unsigned long long)i >> 1));
          xi = seg_noise<NM == 3>(a.nv, k, s, i);
        }
        T wn;
        const auto g = grad_step(w, lam, opt, xi, a.eta, NOISE, &wn);
        v[k] = wn;
        if (!avg) a.w[k * a.ld + i] = wn;
        nsq[k] += to_d(g) * to_d(g);
      }
      if (avg) {
        const T m = run_prog(prog, v) / (T)a.k_total;
        for (int k = 0; k < kl; ++k) a.w[k * a.ld + i] = m;
      }
    }
  }

  {
    __shared__ double red[kThreads / 32];
    for (int k = 0; k < kl; ++k) {
      const double s = block_sum(nsq[k], red);
      if (threadIdx.x == 0) a.norm_part[(long long)k * a.ntiles + tile_id] = s;
    }
  }
}

// ---------------------------------------------------------------------------
// Bulk-copy (TMA 1-D) update kernel, single GPU, fp64 (default with engine noise).
// Persistent CTAs, each walking whole tiles in 512-coordinate chunks: one
// producer lane moves a chunk's 8 row slices and 8 noise slices into shared
// memory with cp.async.bulk (completion counted on an mbarrier), 8 consumer
// warps update and average it in place, and the rows go back with bulk
// stores — the memory pipeline costs no registers, so fewer SMs can carry
// the full HBM stream and the rest stay free for the noise engine.
// ---------------------------------------------------------------------------
constexpr int kBChunk = 512;                 // coordinates per chunk with 8 local rows
// chunk length by local row count: every stage moves the same 64 KB (rows +
// noise), so 1-4 rows carry as many bytes per mbarrier round trip as 8
template <int KL>
__host__ __device__ constexpr int bulk_chunk() { return kBChunk * 8 / KL; }
constexpr int kBStages = 3;
constexpr int kBConsumers = 256;             // one pair per consumer thread
constexpr int kBThreads = kBConsumers + 32;  // + producer warp

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}

struct BulkChunk {  // producer -> consumers, per stage
  int tile;
  long long a0, a1;  // coordinate window [a0, a1), even-aligned
  int simple;        // noise staged (else consumers look it up)
  int last;          // last chunk of its tile
};

template <int KL, int NM>
__global__ void __launch_bounds__(kBThreads, 1)
lab_update_bulk_kernel(UpdateArgs<double> a, int count) {
  constexpr bool NOISE = NM != 0;
  constexpr int CH = bulk_chunk<KL>();
  extern __shared__ __align__(128) double bsm[];  // [stage][2: w, x][KL][CH]
  __shared__ __align__(8) uint64_t full[kBStages], empty[kBStages];
  __shared__ BulkChunk info[kBStages];
  __shared__ double red[kBConsumers / 32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  auto wbuf = [&](int st, int k) { return bsm + ((long long)(st * 2 + 0) * KL + k) * CH; };
  auto xbuf = [&](int st, int k) { return bsm + ((long long)(st * 2 + 1) * KL + k) * CH; };
  if (tid == 0) {
    for (int st = 0; st < kBStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == kBConsumers / 32) {
    // ------------------------------- producer -------------------------------
    int j = 0;  // chunk counter (ring position)
    for (int ti = blockIdx.x; ti < count; ti += gridDim.x) {
      const int tile_id = a.tile_base + ti;
      const Tile t = a.tiles[tile_id];
      // per-worker noise split of this tile (lane k)
      const double* nb0 = nullptr;
      const double* nb1 = nullptr;
      long long ibound = 0;
      int simple = 1;
      if constexpr (NM >= 2) {
        if (lane < KL) {
          const int k = lane;
          const unsigned long long* pf = a.nv.pfx + (long long)k * (a.nv.P + 2);
          const unsigned long long m0 = a.nv.base + ((unsigned long long)t.start >> 1);
          const unsigned long long m1 = a.nv.base + ((unsigned long long)(t.start + t.len - 1) >> 1);
          const int s0 = seg_search(pf, a.nv.P, m0);
          const int s1 = s0 < a.nv.P ? s0 + 1 : s0;
          nb0 = a.nv.slots + ((long long)k * (a.nv.P + 1) + s0) * a.nv.cap - 2 * (long long)pf[s0] + 2 * (long long)a.nv.base;
          nb1 = a.nv.slots + ((long long)k * (a.nv.P + 1) + s1) * a.nv.cap - 2 * (long long)pf[s1] + 2 * (long long)a.nv.base;
          ibound = s0 < a.nv.P ? 2 * (long long)(pf[s0 + 1] - a.nv.base) : (1LL << 62);
          if (s1 < a.nv.P && m1 >= pf[s1 + 1]) simple = 0;
        }
        simple = __all_sync(0xffffffffu, simple);
      }
      // lazy multi-rank rows: a layer averaged last step is read once (its mean)
      const bool stale = a.mean_in != nullptr && mask_has(a.stale, t.block);
      const long long lo = t.start & ~1LL, hi = (t.start + t.len + 1) & ~1LL;
      for (long long a0 = lo; a0 < hi; a0 += CH, ++j) {
        const long long a1 = a0 + CH < hi ? a0 + CH : hi;
        const int st = j % kBStages, u = j / kBStages;
        if (u > 0) mbar_wait(&empty[st], (u - 1) & 1);
        if (lane == 0) {
          info[st] = BulkChunk{tile_id, a0, a1, simple, a1 >= hi ? 1 : 0};
          const unsigned row = 8u * (unsigned)(a1 - a0);
          const unsigned bytes = row * ((stale ? 1u : (unsigned)KL) + ((NM >= 2 && simple) ? (unsigned)KL : 0u));
          mbar_expect_tx(&full[st], bytes);
          if (stale) bulk_g2s(wbuf(st, 0), a.mean_in + a0, row, &full[st]);
          else
            for (int k = 0; k < KL; ++k) bulk_g2s(wbuf(st, k), a.w + k * a.ld + a0, row, &full[st]);
        }
        if constexpr (NM >= 2) {
          if (simple && lane < KL) {
            const int k = lane;
            const long long cut = min(max(ibound, (long long)a0), (long long)a1);
            if (cut > a0) bulk_g2s(xbuf(st, k), nb0 + a0, 8u * (unsigned)(cut - a0), &full[st]);
            if (a1 > cut) bulk_g2s(xbuf(st, k) + (cut - a0), nb1 + cut, 8u * (unsigned)(a1 - cut), &full[st]);
          }
        }
        __syncwarp();
      }
    }
    return;
  }
  // -------------------------------- consumers --------------------------------
  double nsq[KL];
#pragma unroll
  for (int k = 0; k < KL; ++k) nsq[k] = 0.0;
  int j = 0;
  for (int ti = blockIdx.x; ti < count; ti += gridDim.x) {
    const int tile_id = a.tile_base + ti;
    const Tile t = a.tiles[tile_id];
    const bool avg = a.average && mask_has(a.mask, t.block);
    const bool part = a.partial_out != nullptr && mask_has(a.mask, t.block);
    const bool stale = a.mean_in != nullptr && mask_has(a.stale, t.block);
    const long long lo = t.start & ~1LL, hi = (t.start + t.len + 1) & ~1LL;
    for (long long a0 = lo; a0 < hi; a0 += CH, ++j) {
      const int st = j % kBStages, u = j / kBStages;
      mbar_wait(&full[st], u & 1);
      const BulkChunk ci = info[st];
      const long long a1 = ci.a1;
#pragma unroll
      for (int p = tid; p < CH / 2; p += kBConsumers) {  // pairs of the chunk
      const long long i = a0 + 2 * (long long)p;
      const bool in0 = i < a1 && i >= t.start && i < t.start + t.len;
      const bool in1 = i + 1 < a1 && i + 1 >= t.start && i + 1 < t.start + t.len;
      if (in0 || in1) {
        double lam0, opt0, lam1, opt1;
        quad_coeffs(a.q, i, &lam0, &opt0);
        quad_coeffs(a.q, i + 1, &lam1, &opt1);
        double w0[KL], w1[KL];
#pragma unroll
        for (int k = 0; k < KL; ++k) {
          const double2 wv = *reinterpret_cast<const double2*>(wbuf(st, stale ? 0 : k) + 2 * p);
          double2 xv = make_double2(0.0, 0.0);
          if constexpr (NM >= 2) {
            if (ci.simple) {
              xv = *reinterpret_cast<const double2*>(xbuf(st, k) + 2 * p);
            } else {
              const unsigned long long* pf = a.nv.pfx + (long long)k * (a.nv.P + 2);
              const int sg = seg_search(pf, a.nv.P, a.nv.base + ((unsigned long long)i >> 1));
              xv = *reinterpret_cast<const double2*>(a.nv.slots + ((long long)k * (a.nv.P + 1) + sg) * a.nv.cap +
                                                     2 * (long long)(a.nv.base + ((unsigned long long)i >> 1) - pf[sg]));
            }
          }
          // raw attempts (DSX_NOISE_RAW): the polar transform here, in the
          // issue slots the HBM-bound update leaves idle
          if constexpr (NM == 3) xv = mt_polar_normals(xv.x, xv.y, a.nv.stddev);
          const double g0 = grad_step(wv.x, lam0, opt0, xv.x, a.eta, NOISE, &w0[k]);
          const double g1 = grad_step(wv.y, lam1, opt1, xv.y, a.eta, NOISE, &w1[k]);
          if (in0) nsq[k] += g0 * g0;
          if (in1) nsq[k] += g1 * g1;
        }
        if (avg) {
          const double m0 = psum<0, KL, double>(w0) / (double)a.k_total;
          const double m1 = psum<0, KL, double>(w1) / (double)a.k_total;
#pragma unroll
          for (int k = 0; k < KL; ++k) {
            w0[k] = m0;
            w1[k] = m1;
          }
        }
        const bool full_pair = in0 && in1;
        if (part) {
          // multi-rank synced tile: only this rank's subtree sum leaves
          const double m0 = psum<0, KL, double>(w0), m1 = psum<0, KL, double>(w1);
          if (full_pair) {
            *reinterpret_cast<double2*>(a.partial_out + i) = make_double2(m0, m1);
          } else {
            if (in0) a.partial_out[i] = m0;
            if (in1) a.partial_out[i + 1] = m1;
          }
        } else
#pragma unroll
        for (int k = 0; k < KL; ++k) {
          if (full_pair) {
            *reinterpret_cast<double2*>(wbuf(st, k) + 2 * p) = make_double2(w0[k], w1[k]);
          } else {  // a tile edge: write the in-tile coordinate directly
            if (in0) a.w[k * a.ld + i] = w0[k];
            if (in1) a.w[k * a.ld + i + 1] = w1[k];
          }
        }
      }
      }  // pairs of the chunk
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync 1, %0;" ::"n"(kBConsumers) : "memory");
      if (tid == 0) {
        // rows back with bulk stores, full pairs inside the tile only
        const long long e0 = (t.start + 1) & ~1LL, e1 = (t.start + t.len) & ~1LL;
        const long long s0 = a0 > e0 ? a0 : e0, s1 = a1 < e1 ? a1 : e1;
        if (s1 > s0 && !part)
          for (int k = 0; k < KL; ++k)
            bulk_s2g(a.w + k * a.ld + s0, wbuf(st, k) + (s0 - a0), 8u * (unsigned)(s1 - s0));
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        mbar_arrive(&empty[st]);
      }
      if (ci.last) {
        // the tile's gradient-norm partials (fixed order within the CTA)
#pragma unroll
        for (int k = 0; k < KL; ++k) {
          double x = nsq[k];
          for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
          asm volatile("bar.sync 1, %0;" ::"n"(kBConsumers) : "memory");
          if (lane == 0) red[warp] = x;
          asm volatile("bar.sync 1, %0;" ::"n"(kBConsumers) : "memory");
          if (tid == 0) {
            double sk = 0.0;
            for (int q = 0; q < kBConsumers / 32; ++q) sk += red[q];
            a.norm_part[(long long)k * a.ntiles + tile_id] = sk;
          }
          nsq[k] = 0.0;
        }
      }
    }
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ||g_k||^2 = fixed-order sum of the tile partials (one CTA per worker row),
// then the max over rows (atomicMax on the bit pattern: non-negative doubles
// order like their uint64 images, so the result is order-independent).
__global__ void __launch_bounds__(1024)
norm_finalize_kernel(const double* part, int ntiles, double* norm, unsigned long long* maxnorm) {
  __shared__ double red[32];
  const int k = blockIdx.x;
  double s = 0.0;
  for (int i = threadIdx.x; i < ntiles; i += blockDim.x) s += part[(long long)k * ntiles + i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) {
    norm[k] = s;
    atomicMax(maxnorm, (unsigned long long)__double_as_longlong(s));
  }
}

// Bandwidth-throttled link emulation: occupies the sync stream for `ns`
// nanoseconds (globaltimer), the modelled transfer time of the layers just
// synced on a link of the profile's alpha-beta kind (profile.cpp:103-110).
__global__ void link_spin_kernel(unsigned long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(500);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

__global__ void zero_kernel(double* p, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = 0.0;
}

// ---------------------------------------------------------------------------
// noise engine, single chain per worker: one CTA walks the worker's stream
// generation by generation exactly like libstdc++ (twist, temper, canonical,
// polar accept), a CTA-wide scan orders the accepted pairs, and normals are
// written to noise[k][0..dim).  Consumption stops right after the attempt
// that yields normal dim-1 (the cached second value of an odd tail is
// dropped, as the reference's per-call distribution object does).
// ---------------------------------------------------------------------------
constexpr int kMtThreads = 320;

__global__ void __launch_bounds__(kMtThreads)
mt_noise_chain_kernel(uint64_t* state, double* noise, long long ld, unsigned long long dim,
                      double stddev) {
  __shared__ uint64_t x[kMtN];
  __shared__ double v[kMtN + 2];
  __shared__ int warp_cnt[kMtThreads / 32];
  __shared__ int s_last;  // attempt index where the run ends, or -1
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  uint64_t* st = state + (long long)blockIdx.x * (kMtN + 1);
  double* out = noise + (long long)blockIdx.x * ld;
  if (tid < kMtN) x[tid] = st[tid];
  int p = (int)st[kMtN];
  const unsigned long long pairs_needed = (dim + 1) / 2;
  unsigned long long pairs_done = 0;
  int have_half = 0;
  double half = 0.0;
  __syncthreads();
  if (dim == 0) return;

  for (;;) {
    if (p >= kMtN) {  // _M_gen_rand
      uint64_t a0 = 0, a1 = 0, a2 = 0;
      if (tid < kMtM) {
        a0 = x[tid];
        a1 = x[tid + 1];
        a2 = x[tid + kMtM];
      }
      __syncthreads();
      if (tid < kMtM) x[tid] = mt_next_word(a0, a1, a2);
      __syncthreads();
      if (tid < kMtM) {
        const int k = kMtM + tid;
        a0 = x[k];
        a1 = (k + 1 < kMtN) ? x[k + 1] : x[0];
        a2 = x[k - kMtM];
      }
      __syncthreads();
      if (tid < kMtM) x[kMtM + tid] = mt_next_word(a0, a1, a2);
      __syncthreads();
      p = 0;
    }
    // values of this generation, prefixed by a carried half pair
    if (tid >= p && tid < kMtN) v[have_half + tid - p] = mt_polar_coord(mt_temper(x[tid]));
    if (tid == 0 && have_half) v[0] = half;
    if (tid == 0) s_last = -1;
    __syncthreads();
    const int nvals = have_half + kMtN - p;
    const int npairs = nvals >> 1;
    double px = 0.0, py = 0.0, r2 = 0.0;
    bool acc = false;
    if (tid < npairs) {
      px = v[2 * tid];
      py = v[2 * tid + 1];
      acc = mt_polar_accept(px, py, &r2);
    }
    const unsigned bal = __ballot_sync(0xffffffffu, acc);
    if (lane == 0) warp_cnt[warp] = __popc(bal);
    __syncthreads();
    int before = __popc(bal & ((1u << lane) - 1u));
    int total = 0;
    for (int w = 0; w < kMtThreads / 32; ++w) {
      if (w < warp) before += warp_cnt[w];
      total += warp_cnt[w];
    }
    const unsigned long long remaining = pairs_needed - pairs_done;
    const bool finishing = (unsigned long long)total >= remaining;
    if (acc) {
      const unsigned long long m = pairs_done + (unsigned long long)before;
      if (m < pairs_needed) {
        const double mult = mt_polar_mult(r2);
        out[2 * m] = mt_scale(py, mult, stddev);
        if (2 * m + 1 < dim) out[2 * m + 1] = mt_scale(px, mult, stddev);
        if (m == pairs_needed - 1) s_last = tid;
      }
    }
    __syncthreads();
    if (finishing) {
      const int last = s_last;
      const int consumed = 2 * (last + 1) - have_half;  // outputs of this generation
      if (tid < kMtN) st[tid] = x[tid];
      if (tid == 0) st[kMtN] = (uint64_t)(p + consumed);
      return;
    }
    pairs_done += (unsigned long long)total;
    if (nvals & 1) {
      half = v[nvals - 1];
      have_half = 1;
    } else {
      have_half = 0;
    }
    p = kMtN;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// run_training helpers
// ---------------------------------------------------------------------------
// worker_mean (trainer.cpp:40-50) of coordinate i: pairwise over the local
// rows, or (multi-rank) the cross-rank mean already reduced into gm.
template <typename T, int KL>
__device__ __forceinline__ double row_mean(const T* w, long long ld, long long i, int kl, int k_total,
                                           const PairProg& prog, const T* gm) {
  if (gm) return to_d(gm[i]);
  if constexpr (KL > 0) {
    T v[KL];
#pragma unroll
    for (int k = 0; k < KL; ++k) v[k] = w[k * ld + i];
    return to_d(psum<0, KL, T>(v) / (T)k_total);
  } else {
    T v[kMaxProg];
    for (int k = 0; k < kl; ++k) v[k] = w[k * ld + i];
    return to_d(run_prog(prog, v) / (T)k_total);
  }
}

template <typename T, int KL>
__global__ void mean_accumulate_kernel(const T* w, long long ld, int kl, int k_total,
                                       unsigned long long dim, double weight, double* what,
                                       PairProg prog, const T* gm) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)dim;
       i += (long long)gridDim.x * blockDim.x) {
    const double m = row_mean<T, KL>(w, ld, i, kl, k_total, prog, gm);
    what[i] = __dadd_rn(what[i], __dmul_rn(weight, m));
  }
}

// Per tile: sum_k sum_i (mean_i - w_ki)^2, f(w_hat) and f(mean) partials.
template <typename T, int KL>
__global__ void __launch_bounds__(kThreads)
log_kernel(const T* w, long long ld, int kl, int k_total, const Tile* tiles, int ntiles,
           QuadParams q, const double* what, double weight_total, double* part /*[3][ntiles]*/,
           PairProg prog, const T* gm) {
  const Tile t = tiles[blockIdx.x];
  double gsum = 0.0, fhat = 0.0, fmean = 0.0;
  for (int off = threadIdx.x; off < t.len; off += kThreads) {
    const long long i = t.start + off;
    const double m = row_mean<T, KL>(w, ld, i, kl, k_total, prog, gm);
    for (int k = 0; k < kl; ++k) {
      const double d = m - to_d(w[k * ld + i]);
      gsum += d * d;
    }
    double lam, opt;
    quad_coeffs(q, i, &lam, &opt);
    const double dm = m - opt;
    fmean += 0.5 * lam * dm * dm;
    const double wh = weight_total > 0.0 ? what[i] / weight_total : m;
    const double dh = wh - opt;
    fhat += 0.5 * lam * dh * dh;
  }
  __shared__ double red[kThreads / 32];
  gsum = block_sum(gsum, red);
  fhat = block_sum(fhat, red);
  fmean = block_sum(fmean, red);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = gsum;
    part[ntiles + blockIdx.x] = fhat;
    part[2 * ntiles + blockIdx.x] = fmean;
  }
}

// g = lambda*(w - w*) + xi for one row (stochastic_gradient).
template <typename T>
__global__ void gradient_kernel(const T* w, unsigned long long dim, QuadParams q, int nm,
                                const double* flat, NoiseView nv, int k, double* g) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)dim;
       i += (long long)gridDim.x * blockDim.x) {
    double lam, opt;
    quad_coeffs(q, i, &lam, &opt);
    double gi = __dmul_rn(lam, __dsub_rn(to_d(w[i]), opt));
    if (nm == 1) gi = __dadd_rn(gi, flat[i]);
    if (nm == 2) {
      const int s = seg_search(nv.pfx + (long long)k * (nv.P + 2), nv.P, nv.base + ((unsigned long long)i >> 1));
      gi = __dadd_rn(gi, nv.raw ? seg_noise<true>(nv, k, s, i) : seg_noise<false>(nv, k, s, i));
    }
    g[i] = gi;
  }
}

// ---------------------------------------------------------------------------
// multi-rank averaging helpers
// ---------------------------------------------------------------------------
// staging[i] = pairwise over local rows of w[.][lo + i] (local subtree sum).
template <typename T, int KL>
__global__ void local_partial_kernel(const T* w, long long ld, int kl, long long lo, long long n,
                                     T* staging, PairProg prog) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n;
       j += (long long)gridDim.x * blockDim.x) {
    const long long i = lo + j;
    if constexpr (KL > 0) {
      T v[KL];
#pragma unroll
      for (int k = 0; k < KL; ++k) v[k] = w[k * ld + i];
      staging[j] = psum<0, KL, T>(v);
    } else {
      T v[kMaxProg];
      for (int k = 0; k < kl; ++k) v[k] = w[k * ld + i];
      staging[j] = run_prog(prog, v);
    }
  }
}

// recv holds `nr` rank partials of one slice ([nr][count]); reduce them in
// the reference's pairwise order over ranks, divide by K, write to out.
template <typename T>
__global__ void rank_reduce_kernel(const T* recv, long long count, int nr, int k_total,
                                   T* out, PairProg prog) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < count;
       j += (long long)gridDim.x * blockDim.x) {
    T v[kMaxProg];
    for (int r = 0; r < nr; ++r) v[r] = recv[(long long)r * count + j];
    out[j] = run_prog(prog, v) / (T)k_total;
  }
}

// w[k][lo + i] = src[i] * scale  for every local row (scale 1 => copy).
template <typename T>
__global__ void broadcast_rows_kernel(T* w, long long ld, int kl, long long lo, long long n,
                                      const T* src, T divisor) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n;
       j += (long long)gridDim.x * blockDim.x) {
    const T m = divisor == (T)1 ? src[j] : src[j] / divisor;
    for (int k = 0; k < kl; ++k) w[k * ld + lo + j] = m;
  }
}

// Cross-rank in-place average over NVLink peer memory: x[q] is rank q's
// exchange buffer (its subtree sums, or its only worker row), mapped into
// this process with CUDA IPC.  This rank owns slice [a, b) of the chunk: it
// loads every rank's value (P2P reads), sums them in the reference's
// pairwise rank order, divides by K and stores the mean into every rank's
// buffer (P2P writes).  One kernel = reduce-scatter + all-gather, exact.
struct PeerPtrs {
  void* p[kMaxProg];
};

// Cross-rank flags in peer memory (replacing 4-byte NCCL all-reduces as
// barriers).  Every rank owns kFlagWords u64 words, mapped into all peers:
// [0, kMaxProg) ready epochs by source rank, [kMaxProg, 2 kMaxProg) counts
// of completed averaging launches by source rank.  Values only grow, so no
// reset is needed; writers fence at system scope before publishing.
constexpr int kFlagWords = 2 * kMaxProg;
struct FlagPtrs {
  unsigned long long* p[kMaxProg];
};
struct Signal {
  FlagPtrs f;
  int rank, R;
  unsigned long long value;  // count published by this launch's last block
  unsigned int* counter;     // local finished-block counter (nullptr: no signal)
};

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Thread q < R: optionally publishes `value` into rank q's slot[rank], then
// waits until this rank's slot[q] reached `value` (every peer published).
// A peer that never arrives traps after `timeout_ns` (DSX_FLAG_TIMEOUT_S,
// default 600 s: a slow host thread on a peer is not a failure) instead of
// hanging the GPU forever; the trap message names the rank and epoch.
__global__ void flag_wait_kernel(FlagPtrs f, int rank, int R, int slot, unsigned long long value, int publish,
                                 unsigned long long timeout_ns) {
  const int q = threadIdx.x;
  if (q >= R) return;
  if (publish) {
    __threadfence_system();
    st_release_sys(f.p[q] + slot + rank, value);
  }
  const unsigned long long* mine = f.p[rank] + slot + q;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (ld_acquire_sys(mine) < value) {
    __nanosleep(64);
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) {
      printf("dsx: rank %d timed out waiting for rank %d (flag slot %d, epoch %llu)\n", rank, q, slot, value);
      __trap();
    }
  }
}

template <typename T, int W>
__global__ void __launch_bounds__(256)
p2p_average_kernel(PeerPtrs peers, long long a, long long b, int k_total, PairProg prog, Signal sig) {
  using V2 = typename Vec2<T>::type;
  // vector body on even coordinates, scalar head/tail
  const long long first = a + (a & 1);
  const long long npairs = (b - first) >> 1;
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long j0 = tid;
  if constexpr (W > 0) {
    // two pairs per thread per iteration: all 2W peer loads in flight at once
    for (; j0 + stride < npairs; j0 += 2 * stride) {
      const long long i0 = first + 2 * j0, i1 = first + 2 * (j0 + stride);
      V2 v0[W], v1[W];
#pragma unroll
      for (int q = 0; q < W; ++q) {
        v0[q] = *reinterpret_cast<const V2*>(static_cast<const T*>(peers.p[q]) + i0);
        v1[q] = *reinterpret_cast<const V2*>(static_cast<const T*>(peers.p[q]) + i1);
      }
      T ax[W], ay[W], bx[W], by[W];
#pragma unroll
      for (int q = 0; q < W; ++q) {
        ax[q] = v0[q].x;
        ay[q] = v0[q].y;
        bx[q] = v1[q].x;
        by[q] = v1[q].y;
      }
      V2 m0, m1;
      m0.x = psum<0, W, T>(ax) / (T)k_total;
      m0.y = psum<0, W, T>(ay) / (T)k_total;
      m1.x = psum<0, W, T>(bx) / (T)k_total;
      m1.y = psum<0, W, T>(by) / (T)k_total;
#pragma unroll
      for (int q = 0; q < W; ++q) {
        *reinterpret_cast<V2*>(static_cast<T*>(peers.p[q]) + i0) = m0;
        *reinterpret_cast<V2*>(static_cast<T*>(peers.p[q]) + i1) = m1;
      }
    }
  }
  for (long long j = j0; j < npairs; j += stride) {
    const long long i = first + 2 * j;
    T vx[W > 0 ? W : kMaxProg], vy[W > 0 ? W : kMaxProg];
    const int nr = W > 0 ? W : prog.n + 1;
#pragma unroll
    for (int q = 0; q < (W > 0 ? W : kMaxProg); ++q) {
      if (q >= nr) break;
      const V2 v = *reinterpret_cast<const V2*>(static_cast<const T*>(peers.p[q]) + i);
      vx[q] = v.x;
      vy[q] = v.y;
    }
    V2 m;
    if constexpr (W > 0) {
      m.x = psum<0, W, T>(vx) / (T)k_total;
      m.y = psum<0, W, T>(vy) / (T)k_total;
    } else {
      m.x = run_prog(prog, vx) / (T)k_total;
      m.y = run_prog(prog, vy) / (T)k_total;
    }
#pragma unroll
    for (int q = 0; q < (W > 0 ? W : kMaxProg); ++q) {
      if (q >= nr) break;
      *reinterpret_cast<V2*>(static_cast<T*>(peers.p[q]) + i) = m;
    }
  }
  if (tid < 2) {  // odd head (a) / tail (b-1)
    const long long i = tid == 0 ? a : b - 1;
    const bool take = tid == 0 ? (first != a && a < b) : (first + 2 * npairs < b && b - 1 >= first);
    if (take) {
      T v[W > 0 ? W : kMaxProg];
      const int nr = W > 0 ? W : prog.n + 1;
      for (int q = 0; q < nr; ++q) v[q] = static_cast<const T*>(peers.p[q])[i];
      T m;
      if constexpr (W > 0) m = psum<0, W, T>(v) / (T)k_total;
      else m = run_prog(prog, v) / (T)k_total;
      for (int q = 0; q < nr; ++q) static_cast<T*>(peers.p[q])[i] = m;
    }
  }
  __threadfence_system();
  if (sig.counter) {  // the last block to finish publishes this launch's count to every rank
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(sig.counter, 1u) == gridDim.x - 1) {
      *sig.counter = 0;
      __threadfence_system();
      for (int q = 0; q < sig.R; ++q) st_release_sys(sig.f.p[q] + kMaxProg + sig.rank, sig.value);
    }
  }
}

// NVLink roofline probe: the averaging kernel's exact access pattern (this
// rank's slice read from every rank's buffer, written back to every rank's
// buffer: 2(W-1)/W x S bytes over NVLink per rank) as a plain copy — 16-B
// vectors, four slices in flight per thread, no reduction.  What p2p_average
// achieves is reported against this, measured in the same run.
template <int W>
__global__ void __launch_bounds__(256) p2p_probe_kernel(PeerPtrs peers, long long a, long long b) {
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = a + tid;
  for (; i + 3 * stride < b; i += 4 * stride) {
    double2 v[4][W];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int q = 0; q < W; ++q) v[u][q] = static_cast<const double2*>(peers.p[q])[i + u * stride];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int q = 0; q < W; ++q) static_cast<double2*>(peers.p[(q + 1) % W])[i + u * stride] = v[u][q];
  }
  for (; i < b; i += stride) {
    double2 v[W];
#pragma unroll
    for (int q = 0; q < W; ++q) v[q] = static_cast<const double2*>(peers.p[q])[i];
#pragma unroll
    for (int q = 0; q < W; ++q) static_cast<double2*>(peers.p[(q + 1) % W])[i] = v[q];
  }
}

// ---------------------------------------------------------------------------
// host helpers
// ---------------------------------------------------------------------------
static void build_prog(int n, PairProg* p) {
  // Recursively mirrors pairwise_coord_sum: range [lo, hi) result lands in v[lo].
  p->n = 0;
  struct Rec {
    static void go(PairProg* p, int lo, int hi) {
      const int cnt = hi - lo;
      if (cnt == 1) return;
      if (cnt == 2) {
        p->dst[p->n] = (unsigned char)lo;
        p->a[p->n] = (unsigned char)lo;
        p->b[p->n] = (unsigned char)(lo + 1);
        ++p->n;
        return;
      }
      const int mid = lo + cnt / 2;
      go(p, lo, mid);
      go(p, mid, hi);
      p->dst[p->n] = (unsigned char)lo;
      p->a[p->n] = (unsigned char)lo;
      p->b[p->n] = (unsigned char)mid;
      ++p->n;
    }
  };
  if (n >= 1) Rec::go(p, 0, n);
}

// The global pairwise tree restricted to [begin, begin+count) is a subtree
// iff recursing from [0, K) reaches exactly that range.
static bool is_subtree(int K, int begin, int count) {
  int lo = 0, hi = K;
  for (;;) {
    if (lo == begin && hi == begin + count) return true;
    const int n = hi - lo;
    if (n <= 1) return false;
    const int mid = lo + n / 2;
    if (begin + count <= mid) {
      hi = mid;
    } else if (begin >= mid) {
      lo = mid;
    } else {
      return false;
    }
  }
}

}  // namespace dsx

using namespace dsx;

struct dsx_lab {
  int device = 0;
  int dtype = DSX_F64;
  int K = 1, kbegin = 0, kl = 1;
  unsigned long long dim = 0;
  long long ld = 0;
  int L = 0;
  std::vector<unsigned long long> offs;  // L+1
  QuadParams q{};
  double sigma = 0.0, stddev = 0.0;

  void* w = nullptr;
  double* stage64 = nullptr;  // fp32 labs: dense fp64 rows for host transfers (lazy)
  double* curv = nullptr;
  double* opt = nullptr;
  double* noise = nullptr;
  uint64_t* mt = nullptr;
  double* what = nullptr;
  double* grad_buf = nullptr;  // dsx_lab_gradient output staging
  Tile* tiles = nullptr;
  int ntiles = 0;
  std::vector<Tile> h_tiles;
  double* norm_part = nullptr;
  double* norm = nullptr;
  double* maxnorm = nullptr;
  double* log_part = nullptr;
  PairProg prog_local{};

  cudaStream_t stream = nullptr;  // compute
  cudaStream_t side = nullptr;    // sync (high priority)
  cudaEvent_t ev[32] = {};
  cudaEvent_t ev_split = nullptr, ev_synced = nullptr;
  // instrumentation: 0 step start, 1 sync may start, 2 sync done (side),
  // 3 local step done, 4 step end, 5 noise done / update start
  cudaEvent_t iev[6] = {};
  bool instrument = false;
  dsx::NoiseEngine* engine = nullptr;  // parallel exact noise (sigma > 0)
  bool use_chain = false;
  // noise pipelining: the engine runs on nstream one step ahead, into the
  // buffer set the update is not reading; two rng-state buffers keep the
  // committed state (visible through get_rng) apart from a prefetched one.
  cudaStream_t nstream = nullptr;
  cudaEvent_t ev_noise[2] = {}, ev_upd[2] = {};
  // rng-state slots [1 + 2*tmax][kl][313]: slot 0 = host-written, then per
  // buffer set the state after each step of that set's engine run
  int mt_commit = 0;                       // slot of the committed states
  int tmax = 1;                            // steps per engine run (pipelined)
  int cur_set = 0, cur_t = 0;              // noise the current step reads
  int batch_set = -1, batch_t = 0, batch_n = 0;  // current run: set, next step, steps
  int pf_set = -1, pf_n = 0;               // run prefetched into the other set
  bool pipeline = true;
  long long horizon = -1;                  // steps the engine may generate ahead (-1: unbounded)
  bool has_ranges = false, synced_last = false;
  bool overlap = true;
  uint64_t launches = 0;

  // multi-rank
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  int sync_algo = DSX_SYNC_PAIRWISE;
  double link_bw = 0.0, link_lat = 0.0;  // throttled link (bw <= 0: off)
  std::vector<cudaEvent_t> layer_ev;     // per-layer "BP done" events (throttled mode)
  std::vector<cudaEvent_t> tl_ev;        // [4L] timeline: BP start/end, COMM start/end
  std::vector<unsigned char> tl_mask;    // mask of the step the timeline belongs to
  bool p2p = false;            // NVLink peer-memory average available
  PeerPtrs peers{};            // every rank's exchange buffer, mapped here
  std::vector<void*> opened;   // IPC mappings to close
  int* bar = nullptr;          // 4-byte barrier all-reduce scratch
  // peer-memory flag barriers (DSX_FLAG_BARRIER=0: NCCL all-reduce barriers)
  bool flag_bar = false;
  unsigned long long* flags = nullptr;   // this rank's flag block [kFlagWords]
  FlagPtrs fpeers{};                     // every rank's flag block, mapped here
  unsigned int* sig_counter = nullptr;   // finished-block counter of the averaging kernel
  unsigned long long epoch = 0, sig_count = 0;
  unsigned long long flag_timeout_ns = 600ull * 1000000000ull;  // DSX_FLAG_TIMEOUT_S
  // scratch [2][ld] of every rank, mapped into every peer: the NVLink
  // roofline probe's buffer (dsx_lab_link_probe)
  void* xsum = nullptr;
  void* xpeer[kMaxFuse] = {};
  int chunks = 4;              // overlap groups per step (at most)
  int wave = 296;              // update CTAs resident at once (blocks/SM x SMs)
  bool lazy = true;            // lazy broadcast of cross-rank means (DSX_LAZY=0: off)
  MaskBits stale_bits{};       // layers whose rows are stale (mean in staging)
  bool stale_any = false;
  cudaEvent_t ev_chunk[8] = {};
  bool local_subtree = true;
  PairProg prog_ranks{};
  void* staging = nullptr;  // partial sums of synced range
  void* recv = nullptr;     // [nranks][slice]
  void* gmean = nullptr;    // run_training logging: [nranks][dim] subtree sums -> mean in row 0
  // host-state step (dsx_lab_step_host): copy-engine streams + per-chunk events
  cudaStream_t h2d = nullptr, d2h = nullptr;
  std::vector<cudaEvent_t> ev_in, ev_out;
  int host_chunks = 24;
  // the rng states the last host-state step returned: a caller passing them
  // back unchanged finds that step's successor noise already generated
  std::vector<uint64_t> host_rng;
  bool host_rng_valid = false;
  size_t staging_elems = 0;
  int nsm = 148;
};

namespace {

size_t elem_size(const dsx_lab* lab) { return lab->dtype == DSX_F64 ? 8 : 4; }

bool detect_analytic(const dsx_lab_desc* d, QuadParams* q) {
  const unsigned long long n = d->dim;
  const double mu = d->curvature[0];
  const double beta = d->curvature[n - 1];
  const double opt = d->optimum[0];
  for (unsigned long long i = 0; i < n; ++i) {
    const double lam =
        n == 1 ? mu : mu + (beta - mu) * static_cast<double>(i) / static_cast<double>(n - 1);
    if (lam != d->curvature[i] || d->optimum[i] != opt) return false;
  }
  q->analytic = true;
  q->mu = mu;
  q->beta_minus_mu = beta - mu;
  q->dim_minus_1 = n == 1 ? 0.0 : static_cast<double>(n - 1);
  q->opt_value = opt;
  return true;
}

dsx_status check_lab(dsx_lab* lab) {
  if (!lab) return fail(DSX_ERR_ARGUMENT, "null lab");
  DSX_CUDA(cudaSetDevice(lab->device));
  return DSX_OK;
}

dsx_status check_row(dsx_lab* lab, int local) {
  DSX_TRY(check_lab(lab));
  if (local < 0 || local >= lab->kl) return fail(DSX_ERR_ARGUMENT, "worker row out of range");
  return DSX_OK;
}

template <typename T, int KL>
void launch_update_t(dsx_lab* lab, cudaStream_t s, int tile_base, int count, int nm, bool average,
                     const MaskBits& mask, double eta, T* partial_out) {
  UpdateArgs<T> a{};
  a.w = static_cast<T*>(lab->w);
  a.ld = lab->ld;
  a.kl = lab->kl;
  a.k_total = lab->K;
  a.tiles = lab->tiles;
  a.ntiles = lab->ntiles;
  a.tile_base = tile_base;
  a.noise = lab->noise;
  a.eta = eta;
  a.q = lab->q;
  a.mask = mask;
  a.average = average;
  a.norm_part = lab->norm_part;
  a.partial_out = partial_out;
  a.mean_in = lab->stale_any ? static_cast<const T*>(lab->staging) : nullptr;
  a.stale = lab->stale_bits;
  if (lab->engine) a.nv = lab->engine->view(lab->cur_set, lab->cur_t);
  if constexpr (std::is_same_v<T, double> && (KL == 1 || KL == 2 || KL == 4 || KL == 8)) {
    // bulk-copy kernel: the default with engine noise (0.91 vs 0.84 of HBM at
    // sigma=1); the register-staged kernel stays faster without noise (0.83
    // vs 0.80).  DSX_UPD_BULK=0 off, =1 on (one CTA per SM), =n n CTAs.
    static const int bulk_env = [] {
      const char* e = std::getenv("DSX_UPD_BULK");
      return e ? std::atoi(e) : -1;
    }();
    // (with 2-4 local rows a 512-coordinate chunk carries too little per
    // mbarrier round trip: 4 GPUs 0.29 vs 0.17 ms, so 8 rows only by default)
    const int bulk_ctas = bulk_env >= 0 ? bulk_env : (nm == 2 && KL == 8 ? 1 : 0);
    if (bulk_ctas > 0 && (nm == 0 || nm == 2)) {
      const bool raw = nm == 2 && a.nv.raw;
      constexpr size_t smem = sizeof(double) * kBStages * 2 * KL * bulk_chunk<KL>();
      static std::atomic<unsigned long long> attr{0};
      dsx::once_per_device(attr, [] {
        cudaFuncSetAttribute(lab_update_bulk_kernel<KL, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(lab_update_bulk_kernel<KL, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(lab_update_bulk_kernel<KL, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      });
      const int grid = std::min(count, bulk_ctas == 1 ? lab->nsm : bulk_ctas);
      if (raw) lab_update_bulk_kernel<KL, 3><<<grid, kBThreads, smem, s>>>(a, count);
      else if (nm == 2) lab_update_bulk_kernel<KL, 2><<<grid, kBThreads, smem, s>>>(a, count);
      else lab_update_bulk_kernel<KL, 0><<<grid, kBThreads, smem, s>>>(a, count);
      ++lab->launches;
      return;
    }
  }
  if (nm == 2 && a.nv.raw) {
    lab_update_kernel<T, KL, 3><<<count, kThreads, 0, s>>>(a, lab->prog_local);
  } else if (nm == 2) {
    lab_update_kernel<T, KL, 2><<<count, kThreads, 0, s>>>(a, lab->prog_local);
  } else if (nm == 1) {
    lab_update_kernel<T, KL, 1><<<count, kThreads, 0, s>>>(a, lab->prog_local);
  } else {
    lab_update_kernel<T, KL, 0><<<count, kThreads, 0, s>>>(a, lab->prog_local);
  }
  ++lab->launches;
}

template <typename T>
void launch_update(dsx_lab* lab, cudaStream_t s, int tile_base, int count, int noise, bool average,
                   const MaskBits& mask, double eta, T* partial_out = nullptr) {
  switch (lab->kl) {
    case 1: return launch_update_t<T, 1>(lab, s, tile_base, count, noise, average, mask, eta, partial_out);
    case 2: return launch_update_t<T, 2>(lab, s, tile_base, count, noise, average, mask, eta, partial_out);
    case 3: return launch_update_t<T, 3>(lab, s, tile_base, count, noise, average, mask, eta, partial_out);
    case 4: return launch_update_t<T, 4>(lab, s, tile_base, count, noise, average, mask, eta, partial_out);
    case 5: return launch_update_t<T, 5>(lab, s, tile_base, count, noise, average, mask, eta, partial_out);
    case 6: return launch_update_t<T, 6>(lab, s, tile_base, count, noise, average, mask, eta, partial_out);
    case 7: return launch_update_t<T, 7>(lab, s, tile_base, count, noise, average, mask, eta, partial_out);
    case 8: return launch_update_t<T, 8>(lab, s, tile_base, count, noise, average, mask, eta, partial_out);
    default: return launch_update_t<T, 0>(lab, s, tile_base, count, noise, average, mask, eta, partial_out);
  }
}

// Resident update CTAs per SM for this lab's kernel variant (a "wave" is
// that times the SM count).
template <typename T, int KL>
int update_blocks_per_sm_t(int nm) {
  int n = 0;
  if (nm == 2) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, lab_update_kernel<T, KL, 2>, kThreads, 0);
  else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, lab_update_kernel<T, KL, 0>, kThreads, 0);
  return std::max(1, n);
}

template <typename T>
int update_blocks_per_sm(int kl, int nm) {
  switch (kl) {
    case 1: return update_blocks_per_sm_t<T, 1>(nm);
    case 2: return update_blocks_per_sm_t<T, 2>(nm);
    case 4: return update_blocks_per_sm_t<T, 4>(nm);
    case 8: return update_blocks_per_sm_t<T, 8>(nm);
    default: return 2;
  }
}

// Overlap groups of the multi-rank step, from the top layer down: cuts[0] =
// ntiles > cuts[1] > ... > cuts[G] = 0.  When the step has at least G waves
// of update CTAs, every group but the last holds whole waves, so its launch
// ends on a full wave instead of leaving SMs idle in a partial one.
std::vector<int> overlap_groups(const dsx_lab* lab, int want) {
  const int wave = std::max(1, lab->wave);
  const int G = std::max(1, std::min(want, lab->ntiles));
  std::vector<int> cuts{lab->ntiles};
  if (lab->ntiles >= G * wave) {  // whole waves per group
    const int per = (lab->ntiles / G / wave) * wave;
    for (int g = 1; g < G; ++g) cuts.push_back(lab->ntiles - g * per);
  } else {  // fewer tiles than G waves: equal groups (measured better than fewer groups)
    for (int g = 1; g < G; ++g) cuts.push_back(lab->ntiles - (int)((long long)lab->ntiles * g / G));
  }
  cuts.push_back(0);
  return cuts;
}

template <typename T, int KL>
void launch_rowwise_t(dsx_lab* lab, int what, double weight, double weight_total, const T* gm) {
  const T* w = static_cast<const T*>(lab->w);
  if (what == 0) {
    mean_accumulate_kernel<T, KL><<<lab->nsm * 8, 256, 0, lab->stream>>>(
        w, lab->ld, lab->kl, lab->K, lab->dim, weight, lab->what, lab->prog_local, gm);
  } else {
    log_kernel<T, KL><<<lab->ntiles, kThreads, 0, lab->stream>>>(
        w, lab->ld, lab->kl, lab->K, lab->tiles, lab->ntiles, lab->q, lab->what, weight_total,
        lab->log_part, lab->prog_local, gm);
  }
  ++lab->launches;
}

template <typename T>
void launch_rowwise(dsx_lab* lab, int what, double weight, double weight_total, const T* gm) {
  switch (lab->kl) {
    case 1: return launch_rowwise_t<T, 1>(lab, what, weight, weight_total, gm);
    case 2: return launch_rowwise_t<T, 2>(lab, what, weight, weight_total, gm);
    case 4: return launch_rowwise_t<T, 4>(lab, what, weight, weight_total, gm);
    case 8: return launch_rowwise_t<T, 8>(lab, what, weight, weight_total, gm);
    default: return launch_rowwise_t<T, 0>(lab, what, weight, weight_total, gm);
  }
}

template <typename T, int KL>
void launch_partial_t(dsx_lab* lab, cudaStream_t s, long long lo, long long n, T* dst) {
  local_partial_kernel<T, KL><<<lab->nsm * 4, 256, 0, s>>>(static_cast<const T*>(lab->w), lab->ld,
                                                           lab->kl, lo, n, dst, lab->prog_local);
  ++lab->launches;
}

template <typename T>
void launch_partial(dsx_lab* lab, cudaStream_t s, long long lo, long long n, T* dst) {
  switch (lab->kl) {
    case 2: return launch_partial_t<T, 2>(lab, s, lo, n, dst);
    case 4: return launch_partial_t<T, 4>(lab, s, lo, n, dst);
    case 8: return launch_partial_t<T, 8>(lab, s, lo, n, dst);
    default: return launch_partial_t<T, 0>(lab, s, lo, n, dst);
  }
}

ncclDataType_t nccl_type(const dsx_lab* lab) { return lab->dtype == DSX_F64 ? ncclFloat64 : ncclFloat32; }

// Cross-rank average of coordinates [lo, lo+n) on stream s (all local rows
// end up holding the global mean).  Requires comm.
template <typename T>
dsx_status sync_range(dsx_lab* lab, cudaStream_t s, long long lo, long long n) {
  T* w = static_cast<T*>(lab->w);
  const int R = lab->nranks;
  // 1. this rank's subtree sum of the range
  T* part = nullptr;
  if (lab->kl == 1) {
    part = w + lo;  // in place: row 0 is its own partial
  } else {
    part = static_cast<T*>(lab->staging);
    launch_partial<T>(lab, s, lo, n, part);
  }
  if (lab->sync_algo == DSX_SYNC_NCCL_AVG) {
    DSX_NCCL(ncclAllReduce(part, part, (size_t)n, nccl_type(lab), ncclSum, lab->comm, s));
    broadcast_rows_kernel<T><<<lab->nsm * 4, 256, 0, s>>>(w, lab->ld, lab->kl, lo, n, part,
                                                          (T)lab->K);
    ++lab->launches;
    return DSX_OK;
  }
  // 2. reduce-scatter in the reference's pairwise rank order: rank r owns
  //    slice r; all-to-all of partial slices, local fixed-order reduction.
  const long long base = n / R, extra = n % R;
  auto slice_lo = [&](int r) { return r * base + std::min<long long>(r, extra); };
  auto slice_n = [&](int r) { return base + (r < extra ? 1 : 0); };
  const long long my_n = slice_n(lab->rank);
  T* recv = static_cast<T*>(lab->recv);
  DSX_NCCL(ncclGroupStart());
  for (int r = 0; r < R; ++r) {
    if (slice_n(r) > 0) DSX_NCCL(ncclSend(part + slice_lo(r), (size_t)slice_n(r), nccl_type(lab), r, lab->comm, s));
    if (my_n > 0) DSX_NCCL(ncclRecv(recv + (long long)r * my_n, (size_t)my_n, nccl_type(lab), r, lab->comm, s));
  }
  DSX_NCCL(ncclGroupEnd());
  if (my_n > 0) {
    rank_reduce_kernel<T><<<lab->nsm * 4, 256, 0, s>>>(recv, my_n, R, lab->K, part + slice_lo(lab->rank),
                                                        lab->prog_ranks);
    ++lab->launches;
  }
  // 3. all-gather the reduced slices in place (one broadcast per owner).
  DSX_NCCL(ncclGroupStart());
  for (int r = 0; r < R; ++r) {
    if (slice_n(r) > 0)
      DSX_NCCL(ncclBroadcast(part + slice_lo(r), part + slice_lo(r), (size_t)slice_n(r), nccl_type(lab), r,
                             lab->comm, s));
  }
  DSX_NCCL(ncclGroupEnd());
  if (lab->kl > 1) {
    broadcast_rows_kernel<T><<<lab->nsm * 4, 256, 0, s>>>(w, lab->ld, lab->kl, lo, n, part, (T)1);
    ++lab->launches;
  }
  return DSX_OK;
}

// Masked blocks -> maximal contiguous coordinate ranges.
std::vector<std::pair<long long, long long>> masked_ranges(const dsx_lab* lab, const unsigned char* mask) {
  std::vector<std::pair<long long, long long>> out;
  for (int b = 0; b < lab->L; ++b) {
    if (!mask[b + 1]) continue;
    const long long lo = (long long)lab->offs[b], hi = (long long)lab->offs[b + 1];
    if (!out.empty() && out.back().first + out.back().second == lo) {
      out.back().second += hi - lo;
    } else {
      out.push_back({lo, hi - lo});
    }
  }
  return out;
}

// Modelled link time of the synced layers overlapping [lo, lo+n): per layer
// latency + bytes/bandwidth, like comm_time() (profile.cpp:103-110).
unsigned long long link_ns(const dsx_lab* lab, const unsigned char* mask, long long lo, long long n) {
  double sec = 0.0;
  const size_t es = lab->dtype == DSX_F64 ? 8 : 4;
  for (int b = 0; b < lab->L; ++b) {
    if (!mask[b + 1]) continue;
    const long long a = std::max<long long>(lo, (long long)lab->offs[b]);
    const long long e = std::min<long long>(lo + n, (long long)lab->offs[b + 1]);
    if (a >= e) continue;
    sec += lab->link_lat + (double)((e - a) * (long long)es) / lab->link_bw;
  }
  return (unsigned long long)(sec * 1e9);
}

// Single GPU with a throttled link: the local step runs layer by layer in
// backward order (L..1) on the compute stream and each synced layer's
// modelled transfer occupies the FIFO sync stream from the moment its
// update is done — the discrete-event model of simulator.cpp:145-157
// executed for real.  The averaging itself stays fused in the update kernel.
template <typename T>
dsx_status step_single_throttled(dsx_lab* lab, double eta, const unsigned char* mask,
                                 const MaskBits& bits, int noise) {
  if ((int)lab->layer_ev.size() < lab->L) {
    const size_t old = lab->layer_ev.size();
    lab->layer_ev.resize(lab->L);
    for (size_t i = old; i < lab->layer_ev.size(); ++i)
      DSX_CUDA(cudaEventCreateWithFlags(&lab->layer_ev[i], cudaEventDisableTiming));
  }
  // measured timeline (dsx_lab_last_timeline): timing events around every
  // layer's local step and modelled transfer
  const bool tl = lab->instrument;
  if (tl && (int)lab->tl_ev.size() < 4 * lab->L) {
    const size_t old = lab->tl_ev.size();
    lab->tl_ev.resize(4 * lab->L);
    for (size_t i = old; i < lab->tl_ev.size(); ++i) DSX_CUDA(cudaEventCreate(&lab->tl_ev[i]));
  }
  if (tl) lab->tl_mask.assign(mask, mask + lab->L + 1);
  // tile range of each layer
  int te = lab->ntiles;
  bool any = false;
  std::vector<int> deferred;  // no-overlap (ssgd): transfers start after the whole local step
  auto transfer = [&](int b) -> dsx_status {
    if (tl) DSX_CUDA(cudaEventRecord(lab->tl_ev[4 * b + 2], lab->side));
    const unsigned long long ns =
        link_ns(lab, mask, (long long)lab->offs[b], (long long)(lab->offs[b + 1] - lab->offs[b]));
    link_spin_kernel<<<1, 1, 0, lab->side>>>(ns);
    ++lab->launches;
    if (tl) DSX_CUDA(cudaEventRecord(lab->tl_ev[4 * b + 3], lab->side));
    return DSX_OK;
  };
  for (int b = lab->L - 1; b >= 0; --b) {
    int tb = te;
    while (tb > 0 && lab->h_tiles[tb - 1].block == b) --tb;
    if (tl) DSX_CUDA(cudaEventRecord(lab->tl_ev[4 * b + 0], lab->stream));
    if (te > tb) launch_update<T>(lab, lab->stream, tb, te - tb, noise, lab->K > 1, bits, eta);
    if (tl) DSX_CUDA(cudaEventRecord(lab->tl_ev[4 * b + 1], lab->stream));
    te = tb;
    if (!mask[b + 1]) continue;
    if (!any && lab->instrument) DSX_CUDA(cudaEventRecord(lab->iev[1], lab->stream));
    any = true;
    if (!lab->overlap) {
      deferred.push_back(b);
      continue;
    }
    DSX_CUDA(cudaEventRecord(lab->layer_ev[b], lab->stream));
    DSX_CUDA(cudaStreamWaitEvent(lab->side, lab->layer_ev[b], 0));
    DSX_TRY(transfer(b));
  }
  if (!deferred.empty()) {
    DSX_CUDA(cudaEventRecord(lab->ev_split, lab->stream));
    DSX_CUDA(cudaStreamWaitEvent(lab->side, lab->ev_split, 0));
    for (int b : deferred) DSX_TRY(transfer(b));
  }
  lab->has_ranges = any;
  if (lab->instrument) DSX_CUDA(cudaEventRecord(lab->iev[3], lab->stream));
  if (any) {
    DSX_CUDA(cudaEventRecord(lab->ev_synced, lab->side));
    if (lab->instrument) DSX_CUDA(cudaEventRecord(lab->iev[2], lab->side));
    DSX_CUDA(cudaStreamWaitEvent(lab->stream, lab->ev_synced, 0));
  }
  return DSX_OK;
}

// Multi-rank step with the NVLink peer-memory average: the local step runs
// in `chunks` tile groups from the top layer down (backward order); as soon
// as a group is updated the side stream averages its synced coordinates
// across ranks (one p2p_average_kernel per range), overlapping the update
// of the groups below.  Cross-rank ordering uses 4-byte NCCL all-reduces as
// barriers: before a group's average (every rank's subtree sums are final)
// and after it (every rank's peer writes landed).
template <typename T>
dsx_status step_multi_p2p(dsx_lab* lab, double eta, const unsigned char* mask, const MaskBits& bits,
                          int noise) {
  const auto ranges = masked_ranges(lab, mask);
  lab->has_ranges = !ranges.empty();
  // (one group per layer on the throttled link was measured: the per-layer
  // cross-rank barriers cost far more than the finer overlap gains)
  const std::vector<int> cuts = overlap_groups(lab, lab->overlap ? lab->chunks : 1);
  const int G = (int)cuts.size() - 1;
  T* part = lab->kl > 1 ? static_cast<T*>(lab->staging) : nullptr;
  const bool fused_partial = lab->kl > 1 && lab->kl <= 8;
  // lazy broadcast (fused path): the synced layers' rows stay stale, their
  // mean lives in the exchange buffer and the next update reads it there
  const bool lazy = fused_partial && lab->lazy;
  const int R = lab->nranks;
  const bool fb = lab->flag_bar;
  auto barrier = [&]() -> dsx_status {
    DSX_NCCL(ncclAllReduce(lab->bar, lab->bar, 1, ncclInt32, ncclSum, lab->comm, lab->side));
    return DSX_OK;
  };
  // "every rank's subtree sums of this group are final"
  auto ready = [&]() -> dsx_status {
    if (!fb) return barrier();
    flag_wait_kernel<<<1, 64, 0, lab->side>>>(lab->fpeers, lab->rank, R, 0, ++lab->epoch, 1, lab->flag_timeout_ns);
    ++lab->launches;
    return DSX_OK;
  };
  // "every rank's averaging writes so far have landed"
  auto landed = [&]() -> dsx_status {
    if (!fb) return barrier();
    flag_wait_kernel<<<1, 64, 0, lab->side>>>(lab->fpeers, lab->rank, R, kMaxProg, lab->sig_count, 0, lab->flag_timeout_ns);
    ++lab->launches;
    return DSX_OK;
  };
  bool any = false, started = false;
  std::vector<std::pair<long long, long long>> pending;  // ranges awaiting the row broadcast
  for (int g = 0; g < G; ++g) {
    // group g = tiles [tb, te), counted from the top
    const int te = cuts[g], tb = cuts[g + 1];
    if (te <= tb) continue;
    launch_update<T>(lab, lab->stream, tb, te - tb, noise, false, bits, eta, fused_partial ? part : nullptr);
    if (g == 0 && lab->instrument) DSX_CUDA(cudaEventRecord(lab->iev[1], lab->stream));
    const long long lo = lab->h_tiles[tb].start;
    const long long hi = lab->h_tiles[te - 1].start + lab->h_tiles[te - 1].len;
    std::vector<std::pair<long long, long long>> sub;
    for (const auto& r : ranges) {
      const long long a = std::max(lo, r.first), b = std::min(hi, r.first + r.second);
      if (a < b) sub.push_back({a, b - a});
    }
    if (sub.empty()) continue;
    DSX_CUDA(cudaEventRecord(lab->ev_chunk[g % kMaxChunks], lab->stream));
    DSX_CUDA(cudaStreamWaitEvent(lab->side, lab->ev_chunk[g % kMaxChunks], 0));
    if (lab->kl > 1 && !fused_partial)
      for (const auto& r : sub) launch_partial<T>(lab, lab->side, r.first, r.second, part + r.first);
    DSX_TRY(ready());  // this group's subtree sums final on every rank
    started = true;
    if (!pending.empty() && !lazy) {  // previous group's averages must have landed
      if (fb) DSX_TRY(landed());
      for (const auto& r : pending) {
        broadcast_rows_kernel<T><<<lab->nsm * 2, 256, 0, lab->side>>>(static_cast<T*>(lab->w), lab->ld,
                                                                       lab->kl, r.first, r.second,
                                                                       part + r.first, (T)1);
        ++lab->launches;
      }
      pending.clear();
    }
    for (const auto& r : sub) {
      const long long base = r.second / R, extra = r.second % R;
      const long long a = r.first + lab->rank * base + std::min<long long>(lab->rank, extra);
      const long long n = base + (lab->rank < extra ? 1 : 0);
      // with flag barriers every rank launches (possibly empty) so the
      // published launch counts stay in lockstep
      if (n <= 0 && !fb) continue;
      const int blocks = (int)std::min<long long>(lab->nsm * 4, (std::max(n, 0LL) / 2 + 255) / 256 + 1);
      Signal sig{};
      if (fb) sig = Signal{lab->fpeers, lab->rank, R, ++lab->sig_count, lab->sig_counter};
      const long long e = a + std::max(n, 0LL);
      switch (R) {
        case 2: p2p_average_kernel<T, 2><<<blocks, 256, 0, lab->side>>>(lab->peers, a, e, lab->K, lab->prog_ranks, sig); break;
        case 4: p2p_average_kernel<T, 4><<<blocks, 256, 0, lab->side>>>(lab->peers, a, e, lab->K, lab->prog_ranks, sig); break;
        case 8: p2p_average_kernel<T, 8><<<blocks, 256, 0, lab->side>>>(lab->peers, a, e, lab->K, lab->prog_ranks, sig); break;
        default: p2p_average_kernel<T, 0><<<blocks, 256, 0, lab->side>>>(lab->peers, a, e, lab->K, lab->prog_ranks, sig);
      }
      ++lab->launches;
    }
    if (lab->link_bw > 0.0) {
      unsigned long long ns = 0;
      for (const auto& r : sub) ns += link_ns(lab, mask, r.first, r.second);
      link_spin_kernel<<<1, 1, 0, lab->side>>>(ns);
      ++lab->launches;
    }
    if (lab->kl > 1) pending.insert(pending.end(), sub.begin(), sub.end());
    any = true;
  }
  if (lab->instrument) DSX_CUDA(cudaEventRecord(lab->iev[3], lab->stream));
  if (any) {
    DSX_TRY(landed());  // every group's peer writes landed everywhere
    if (!lazy) {
      for (const auto& r : pending) {
        broadcast_rows_kernel<T><<<lab->nsm * 2, 256, 0, lab->side>>>(static_cast<T*>(lab->w), lab->ld,
                                                                       lab->kl, r.first, r.second,
                                                                       part + r.first, (T)1);
        ++lab->launches;
      }
    }
    DSX_CUDA(cudaEventRecord(lab->ev_synced, lab->side));
    if (lab->instrument) DSX_CUDA(cudaEventRecord(lab->iev[2], lab->side));
    DSX_CUDA(cudaStreamWaitEvent(lab->stream, lab->ev_synced, 0));
  }
  (void)started;
  if (lazy) {
    // this step's synced layers are stale now (the previous stale set was
    // consumed: unsynced tiles rewrote their rows, synced ones are stale again)
    lab->stale_bits = bits;
    lab->stale_any = any;
  }
  return DSX_OK;
}

template <typename T>
dsx_status step_impl(dsx_lab* lab, double eta, const unsigned char* mask, int noise) {
  MaskBits bits{};
  for (int b = 0; b < lab->L; ++b)
    if (mask[b + 1]) bits.w[b >> 5] |= 1u << (b & 31);
  const bool single = lab->nranks == 1;
  if (lab->kl == 0 || lab->ntiles == 0) return DSX_OK;
  if (single && lab->link_bw > 0.0) {
    DSX_TRY(step_single_throttled<T>(lab, eta, mask, bits, noise));
  } else if (single) {
    launch_update<T>(lab, lab->stream, 0, lab->ntiles, noise, lab->K > 1, bits, eta);
  } else if (lab->p2p && lab->sync_algo == DSX_SYNC_PAIRWISE) {
    DSX_TRY(step_multi_p2p<T>(lab, eta, mask, bits, noise));
  } else {
    const auto ranges = masked_ranges(lab, mask);
    lab->has_ranges = !ranges.empty();
    // Split point: the local step runs backward-order (high layers first) so
    // the synced ranges become final early; tiles are ordered by coordinate,
    // so the first synced coordinate decides which tiles must finish before
    // the sync may start.
    int split = 0;
    if (!ranges.empty() && lab->overlap) {
      const long long first = ranges.front().first;
      split = 0;
      while (split < lab->ntiles && lab->h_tiles[split].start < first) ++split;
    }
    if (split < lab->ntiles) {
      launch_update<T>(lab, lab->stream, split, lab->ntiles - split, noise, false, bits, eta);
    }
    DSX_CUDA(cudaEventRecord(lab->ev_split, lab->stream));
    if (lab->instrument) DSX_CUDA(cudaEventRecord(lab->iev[1], lab->stream));
    if (!ranges.empty()) {
      DSX_CUDA(cudaStreamWaitEvent(lab->side, lab->ev_split, 0));
      for (const auto& r : ranges) DSX_TRY(sync_range<T>(lab, lab->side, r.first, r.second));
      DSX_CUDA(cudaEventRecord(lab->ev_synced, lab->side));
      if (lab->instrument) DSX_CUDA(cudaEventRecord(lab->iev[2], lab->side));
    }
    if (split > 0) launch_update<T>(lab, lab->stream, 0, split, noise, false, bits, eta);
    if (lab->instrument) DSX_CUDA(cudaEventRecord(lab->iev[3], lab->stream));
    if (!ranges.empty()) DSX_CUDA(cudaStreamWaitEvent(lab->stream, lab->ev_synced, 0));
  }
  DSX_CUDA(cudaMemsetAsync(lab->maxnorm, 0, 8, lab->stream));
  norm_finalize_kernel<<<lab->kl, 1024, 0, lab->stream>>>(
      lab->norm_part, lab->ntiles, lab->norm, reinterpret_cast<unsigned long long*>(lab->maxnorm));
  ++lab->launches;
  if (lab->instrument) DSX_CUDA(cudaEventRecord(lab->iev[4], lab->stream));
  lab->synced_last = (!single || lab->link_bw > 0.0) && lab->has_ranges;
  DSX_CUDA(cudaGetLastError());
  return DSX_OK;
}

uint64_t* mt_state(dsx_lab* lab, int idx) { return lab->mt + (long long)idx * lab->kl * (kMtN + 1); }

// Writes the lazily kept cross-rank means back into every local row (before
// anything reads or partially overwrites the rows).
template <typename T>
dsx_status materialize_t(dsx_lab* lab) {
  DSX_CUDA(cudaStreamWaitEvent(lab->stream, lab->ev_synced, 0));
  for (int b = 0; b < lab->L; ++b) {
    if (!mask_has(lab->stale_bits, b)) continue;
    const long long lo = (long long)lab->offs[b], n = (long long)(lab->offs[b + 1] - lab->offs[b]);
    broadcast_rows_kernel<T><<<lab->nsm * 2, 256, 0, lab->stream>>>(
        static_cast<T*>(lab->w), lab->ld, lab->kl, lo, n, static_cast<const T*>(lab->staging) + lo, (T)1);
    ++lab->launches;
  }
  lab->stale_bits = MaskBits{};
  lab->stale_any = false;
  DSX_CUDA(cudaGetLastError());
  return DSX_OK;
}

dsx_status materialize(dsx_lab* lab) {
  if (!lab->stale_any) return DSX_OK;
  return lab->dtype == DSX_F64 ? materialize_t<double>(lab) : materialize_t<float>(lab);
}

// run_training logging on several ranks: worker_mean over ALL K workers,
// exact — each rank's local subtree sum is all-gathered and reduced in the
// reference's pairwise rank order (the same tree the step's average uses).
// Returns the [dim] mean (row 0 of the gather buffer), on lab->stream.
template <typename T>
dsx_status global_mean(dsx_lab* lab, const T** out) {
  DSX_TRY(materialize(lab));
  const long long D = (long long)lab->dim;
  if (!lab->gmean) DSX_CUDA(cudaMalloc(&lab->gmean, sizeof(T) * D * lab->nranks));
  T* all = static_cast<T*>(lab->gmean);
  launch_partial<T>(lab, lab->stream, 0, D, all + lab->rank * D);
  DSX_NCCL(ncclAllGather(all + lab->rank * D, all, (size_t)D, nccl_type(lab), lab->comm, lab->stream));
  // in place: element j of row 0 is written after its thread read column j
  rank_reduce_kernel<T><<<lab->nsm * 4, 256, 0, lab->stream>>>(all, D, lab->nranks, lab->K, all,
                                                               lab->prog_ranks);
  ++lab->launches;
  DSX_CUDA(cudaGetLastError());
  *out = all;
  return DSX_OK;
}

// mean_accumulate (what = 0) / log (what = 1) over the (global) worker mean
template <typename T>
dsx_status rowwise(dsx_lab* lab, int what, double weight, double weight_total) {
  const T* gm = nullptr;
  if (lab->nranks > 1) DSX_TRY(global_mean<T>(lab, &gm));
  else DSX_TRY(materialize(lab));
  launch_rowwise<T>(lab, what, weight, weight_total, gm);
  DSX_CUDA(cudaGetLastError());
  return DSX_OK;
}

void drop_stale(dsx_lab* lab) {  // every row is about to be overwritten
  lab->stale_bits = MaskBits{};
  lab->stale_any = false;
}

int boundary_slot(const dsx_lab* lab, int set, int t) { return 1 + set * lab->tmax + t; }

// Launches an engine run of `steps` steps on the noise stream: states in
// slot src -> the set's boundary slots, normals into `set`, after the last
// update that read `set` finished.
dsx_status launch_engine(dsx_lab* lab, int set, int steps, int src) {
  std::string err;
  DSX_CUDA(cudaStreamWaitEvent(lab->nstream, lab->ev_upd[set], 0));
  const uint64_t before = lab->engine->launches();
  if (!lab->engine->run(mt_state(lab, src), mt_state(lab, boundary_slot(lab, set, 0)), set, steps,
                        lab->stddev, lab->nstream, &err))
    return fail(DSX_ERR_CUDA, err);
  lab->launches += lab->engine->launches() - before;
  DSX_CUDA(cudaEventRecord(lab->ev_noise[set], lab->nstream));
  return DSX_OK;
}

// Drops generated-but-unconsumed noise (the rest of the current run and a
// prefetched run): the committed rng state is about to change.
dsx_status invalidate_prefetch(dsx_lab* lab) {
  lab->host_rng_valid = false;
  if (lab->nstream) DSX_CUDA(cudaStreamSynchronize(lab->nstream));
  lab->pf_set = -1;
  lab->batch_set = -1;
  lab->batch_t = lab->batch_n = 0;
  return DSX_OK;
}

// Makes this step's noise available to the compute stream; returns the
// update kernels' noise mode and selects (cur_set, cur_t).  One engine run
// covers tmax consecutive steps when pipelining (the jump-ahead is paid once
// per run); the committed state advances to the state after this step.
dsx_status run_noise(dsx_lab* lab, int* mode) {
  *mode = 0;
  if (lab->sigma <= 0.0) return DSX_OK;
  if (lab->use_chain) {  // DSX_NOISE_CHAIN=1: the single-chain reference engine
    mt_noise_chain_kernel<<<lab->kl, kMtThreads, 0, lab->stream>>>(mt_state(lab, lab->mt_commit),
                                                                   lab->noise, lab->ld, lab->dim,
                                                                   lab->stddev);
    ++lab->launches;
    *mode = 1;
    return DSX_OK;
  }
  if (lab->batch_set < 0 || lab->batch_t >= lab->batch_n) {
    if (lab->pf_set >= 0) {  // generated during the previous run's steps
      lab->batch_set = lab->pf_set;
      lab->batch_n = lab->pf_n;
      lab->pf_set = -1;
    } else {
      const int commit_set = lab->mt_commit == 0 ? -1 : (lab->mt_commit - 1) / lab->tmax;
      const int set = commit_set == 0 ? 1 : 0;
      const int steps = (lab->pipeline && (lab->horizon < 0 || lab->horizon >= lab->tmax)) ? lab->tmax : 1;
      DSX_TRY(launch_engine(lab, set, steps, lab->mt_commit));
      lab->batch_set = set;
      lab->batch_n = steps;
    }
    lab->batch_t = 0;
  }
  lab->cur_set = lab->batch_set;
  lab->cur_t = lab->batch_t;
  lab->mt_commit = boundary_slot(lab, lab->batch_set, lab->batch_t);
  ++lab->batch_t;
  DSX_CUDA(cudaStreamWaitEvent(lab->stream, lab->ev_noise[lab->cur_set], 0));
  *mode = 2;
  return DSX_OK;
}

// After the update of this step was enqueued: start the next run on the
// noise stream (from the current run's last state) so it overlaps this
// run's (HBM-bound) updates.
dsx_status after_update(dsx_lab* lab, int mode) {
  if (mode != 2) return DSX_OK;
  DSX_CUDA(cudaEventRecord(lab->ev_upd[lab->cur_set], lab->stream));
  if (!lab->pipeline || lab->pf_set >= 0 || lab->batch_set < 0) return DSX_OK;
  // a bounded horizon: never generate noise for steps beyond it (the whole
  // next run must be consumed within the horizon)
  if (lab->horizon >= 0 && lab->horizon - (lab->batch_n - lab->batch_t) < lab->tmax) return DSX_OK;
  const int set = 1 - lab->batch_set;
  DSX_TRY(launch_engine(lab, set, lab->tmax, boundary_slot(lab, lab->batch_set, lab->batch_n - 1)));
  lab->pf_set = set;
  lab->pf_n = lab->tmax;
  return DSX_OK;
}

// fp32 labs: narrowing / widening between fp64 staging and fp32 rows
// (round-to-nearest, the same rounding as a host double->float conversion).
// staged element e of a chunk starting at flat index off <-> row (off+e)/dim
__global__ void narrow_rows_kernel(const double* __restrict__ src, float* __restrict__ dst, long long ld,
                                   long long dim, long long off, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long f = off + i;
    dst[(f / dim) * ld + f % dim] = __double2float_rn(src[i]);
  }
}

__global__ void widen_rows_kernel(const float* __restrict__ src, double* __restrict__ dst, long long ld,
                                  long long dim, long long off, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long f = off + i;
    dst[i] = (double)src[(f / dim) * ld + f % dim];
  }
}

// fp32 labs keep the fp64 host interface: whole-state transfers go through a
// bounded fp64 staging chunk (at most 256 MB, allocated on first use), one
// chunk at a time on the lab stream.  Both directions return with the copies
// complete (the caller may reuse / read its buffer immediately).
constexpr long long kStageElems = 32ll << 20;

dsx_status ensure_stage64(dsx_lab* lab) {
  if (lab->stage64) return DSX_OK;
  const long long n = std::min<long long>(kStageElems, (long long)lab->dim * lab->kl);
  DSX_CUDA(cudaMalloc(&lab->stage64, 8 * (size_t)n));
  return DSX_OK;
}

// host fp64 [kl][dim] -> fp32 rows
dsx_status set_all_f32(dsx_lab* lab, const double* w) {
  DSX_TRY(ensure_stage64(lab));
  const long long n = (long long)lab->dim * lab->kl;
  for (long long off = 0; off < n; off += kStageElems) {
    const long long len = std::min(kStageElems, n - off);
    DSX_CUDA(cudaMemcpyAsync(lab->stage64, w + off, 8 * (size_t)len, cudaMemcpyHostToDevice, lab->stream));
    narrow_rows_kernel<<<4 * lab->nsm, 256, 0, lab->stream>>>(lab->stage64, static_cast<float*>(lab->w), lab->ld,
                                                             lab->dim, off, len);
    DSX_CUDA(cudaGetLastError());
    ++lab->launches;
  }
  DSX_CUDA(cudaStreamSynchronize(lab->stream));
  return DSX_OK;
}

// fp32 rows -> host fp64 [kl][dim]
dsx_status get_all_f32(dsx_lab* lab, double* w) {
  DSX_TRY(ensure_stage64(lab));
  const long long n = (long long)lab->dim * lab->kl;
  for (long long off = 0; off < n; off += kStageElems) {
    const long long len = std::min(kStageElems, n - off);
    widen_rows_kernel<<<4 * lab->nsm, 256, 0, lab->stream>>>(static_cast<const float*>(lab->w), lab->stage64, lab->ld,
                                                            lab->dim, off, len);
    DSX_CUDA(cudaGetLastError());
    ++lab->launches;
    DSX_CUDA(cudaMemcpyAsync(w + off, lab->stage64, 8 * (size_t)len, cudaMemcpyDeviceToHost, lab->stream));
  }
  DSX_CUDA(cudaStreamSynchronize(lab->stream));
  return DSX_OK;
}

}  // namespace

extern "C" {

const char* dsx_last_error(void) { return g_last_error.c_str(); }

dsx_status dsx_warmup(void) {
  const char* env = std::getenv("DREAMSCHED_DEVICE");
  const int dev = env ? std::atoi(env) : 0;
  (void)dsx::mt_char_poly();
  DSX_CUDA(cudaSetDevice(dev));
  DSX_CUDA(cudaFree(nullptr));
  return DSX_OK;
}

dsx_status dsx_device_count(int* count) {
  if (!count) return fail(DSX_ERR_ARGUMENT, "null count");
  DSX_CUDA(cudaGetDeviceCount(count));
  return DSX_OK;
}

dsx_status dsx_lab_create(const dsx_lab_desc* d, dsx_lab** out) {
  if (!d || !out) return fail(DSX_ERR_ARGUMENT, "null argument");
  *out = nullptr;
  if (d->dim < 1) return fail(DSX_ERR_ARGUMENT, "dim must be >= 1");
  if (d->layers < 1 || d->layers > kMaxMaskWords * 32)
    return fail(DSX_ERR_ARGUMENT, "layers must be in [1, 4096]");
  if (d->workers_total < 1 || d->workers_total > kMaxProg)
    return fail(DSX_ERR_ARGUMENT, "workers_total must be in [1, 64]");
  if (d->workers_local < 1 || d->worker_begin < 0 ||
      d->worker_begin + d->workers_local > d->workers_total)
    return fail(DSX_ERR_ARGUMENT, "bad local worker range");
  if (d->dtype != DSX_F64 && d->dtype != DSX_F32) return fail(DSX_ERR_ARGUMENT, "bad dtype");
  if (!d->block_sizes || !d->curvature || !d->optimum) return fail(DSX_ERR_ARGUMENT, "null arrays");
  unsigned long long covered = 0;
  for (int b = 0; b < d->layers; ++b) {
    if (d->block_sizes[b] == 0) return fail(DSX_ERR_ARGUMENT, "zero-sized layer block");
    covered += d->block_sizes[b];
  }
  if (covered != d->dim) return fail(DSX_ERR_ARGUMENT, "block sizes do not sum to dim");
  if (!(d->noise_sigma >= 0.0)) return fail(DSX_ERR_ARGUMENT, "sigma must be non-negative");
  int ndev = 0;
  DSX_CUDA(cudaGetDeviceCount(&ndev));
  if (d->device < 0 || d->device >= ndev) return fail(DSX_ERR_CUDA, "no such CUDA device");
  DSX_CUDA(cudaSetDevice(d->device));

  auto* lab = new dsx_lab();
  lab->device = d->device;
  lab->dtype = d->dtype;
  lab->K = d->workers_total;
  lab->kbegin = d->worker_begin;
  lab->kl = d->workers_local;
  lab->dim = d->dim;
  lab->ld = (long long)((d->dim + 63) / 64 * 64);
  lab->L = d->layers;
  lab->sigma = d->noise_sigma;
  lab->stddev = d->noise_sigma / std::sqrt(static_cast<double>(d->dim));  // trainer.cpp:180-181
  lab->offs.assign(d->layers + 1, 0);
  for (int b = 0; b < d->layers; ++b) lab->offs[b + 1] = lab->offs[b] + d->block_sizes[b];
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d->device);
  lab->nsm = sms;
  build_prog(lab->kl, &lab->prog_local);

  auto cleanup = [&](dsx_status s) {
    dsx_lab_destroy(lab);
    return s;
  };
  const size_t es = elem_size(lab);
  cudaError_t e = cudaMalloc(&lab->w, es * (size_t)lab->ld * lab->kl);
  if (e != cudaSuccess) return cleanup(fail(DSX_ERR_CUDA, std::string("cudaMalloc(w): ") + cudaGetErrorString(e)));
  cudaMemset(lab->w, 0, es * (size_t)lab->ld * lab->kl);
  if (!detect_analytic(d, &lab->q)) {
    lab->q.analytic = false;
    if (cudaMalloc(&lab->curv, 8 * d->dim) != cudaSuccess || cudaMalloc(&lab->opt, 8 * d->dim) != cudaSuccess)
      return cleanup(fail(DSX_ERR_CUDA, "cudaMalloc(curvature/optimum) failed"));
    cudaMemcpy(lab->curv, d->curvature, 8 * d->dim, cudaMemcpyHostToDevice);
    cudaMemcpy(lab->opt, d->optimum, 8 * d->dim, cudaMemcpyHostToDevice);
    lab->q.curv = lab->curv;
    lab->q.opt = lab->opt;
  }
  if (lab->sigma > 0.0) {
    // steps per engine run: the jump-ahead count per run is ~P*kl (P capped
    // so the segment CTAs fill the GPU), so fewer local workers need longer
    // runs to amortise it: 8 steps at 4-8 workers (8 vs 4 at 8 workers: +3 % it/s), 16 at 1-2
    const char* nb = std::getenv("DSX_NOISE_BATCH");
    const int def = std::max(kNoiseBatch, std::min(16, 32 / std::max(1, lab->kl)));
    lab->tmax = std::max(1, std::min(16, nb ? std::atoi(nb) : def));
    // The engine's normals buffers hold two runs (double-buffered) of tmax
    // steps: ~2 x 8 B x kl x 2.55 x dim x tmax / 2 plus checkpoints.  At
    // GPT-2 size (dim 124M, 8 workers) 8-step runs would need ~170 GB, so
    // the run length is cut until the engine fits the free HBM (keeping a
    // reserve for the caller).
    size_t freeb = 0, totb = 0;
    if (cudaMemGetInfo(&freeb, &totb) == cudaSuccess) {
      const double reserve = 3.0 * (1ull << 30);
      const double avail = 0.9 * ((double)freeb - reserve);
      auto engine_bytes = [&](int T) {
        const double E = 2.0 * ((double)((lab->dim + 1) / 2) * T / 0.78539816339744831) + 4096.0;
        return 8.0 * lab->kl * E * 2.10 + 256.0 * (1 << 20);
      };
      while (lab->tmax > 1 && engine_bytes(lab->tmax) > avail) --lab->tmax;
      if (engine_bytes(lab->tmax) > avail)
        return cleanup(fail(DSX_ERR_CUDA, "noise engine does not fit in free HBM (" +
                                              std::to_string((long long)(engine_bytes(1) / 1e9)) +
                                              " GB needed for one-step runs); use fewer workers per GPU"));
    }
  }
  if (cudaMalloc(&lab->mt, (1 + 2 * (size_t)lab->tmax) * 8 * (size_t)(kMtN + 1) * lab->kl) != cudaSuccess)
    return cleanup(fail(DSX_ERR_CUDA, "cudaMalloc(mt) failed"));
  if (lab->sigma > 0.0) {
    const char* chain = std::getenv("DSX_NOISE_CHAIN");
    lab->use_chain = chain && chain[0] == '1';
    if (lab->use_chain) {
      if (cudaMalloc(&lab->noise, 8 * (size_t)lab->ld * lab->kl) != cudaSuccess)
        return cleanup(fail(DSX_ERR_CUDA, "cudaMalloc(noise) failed"));
    } else {
      lab->engine = new dsx::NoiseEngine();
      std::string err;
      // DSX_ENGINE_SMS: SMs the engine sizes its segment wave for (default
      // all); fewer leaves SMs that the update and the average never have
      // to wait for while a long engine run is resident
      int esms = lab->nsm;
      if (const char* e = std::getenv("DSX_ENGINE_SMS")) esms = std::max(1, std::min(lab->nsm, std::atoi(e)));
      if (!lab->engine->init(lab->dim, lab->kl, esms, lab->tmax, &err)) return cleanup(fail(DSX_ERR_CUDA, err));
    }
  }
  // tiles: per block, `tile` coordinates each (never crossing a block)
  long long tile = kTile;
  if (const char* e = std::getenv("DSX_TILE")) tile = std::max(256LL, std::atoll(e) / 2 * 2);
  for (int b = 0; b < lab->L; ++b) {
    for (unsigned long long s = lab->offs[b]; s < lab->offs[b + 1]; s += tile) {
      lab->h_tiles.push_back({(long long)s, (int)std::min<unsigned long long>(tile, lab->offs[b + 1] - s), b});
    }
  }
  lab->ntiles = (int)lab->h_tiles.size();
  if (cudaMalloc(&lab->tiles, sizeof(Tile) * lab->ntiles) != cudaSuccess ||
      cudaMalloc(&lab->norm_part, 8 * (size_t)lab->ntiles * lab->kl) != cudaSuccess ||
      cudaMalloc(&lab->norm, 8 * (size_t)lab->kl) != cudaSuccess ||
      cudaMalloc(&lab->maxnorm, 8) != cudaSuccess ||
      cudaMalloc(&lab->log_part, 8 * 3 * (size_t)lab->ntiles) != cudaSuccess)
    return cleanup(fail(DSX_ERR_CUDA, "cudaMalloc(tiles/partials) failed"));
  cudaMemcpy(lab->tiles, lab->h_tiles.data(), sizeof(Tile) * lab->ntiles, cudaMemcpyHostToDevice);
  cudaMemset(lab->maxnorm, 0, 8);
  int lo_prio = 0, hi_prio = 0;
  cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
  if (cudaStreamCreateWithPriority(&lab->stream, cudaStreamNonBlocking, lo_prio) != cudaSuccess ||
      cudaStreamCreateWithPriority(&lab->side, cudaStreamNonBlocking, hi_prio) != cudaSuccess)
    return cleanup(fail(DSX_ERR_CUDA, "stream creation failed"));
  for (auto& ev : lab->ev) cudaEventCreate(&ev);
  for (auto& ev : lab->iev) cudaEventCreate(&ev);
  cudaEventCreateWithFlags(&lab->ev_split, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&lab->ev_synced, cudaEventDisableTiming);
  if (lab->engine) {
    // DSX_NOISE_PRIO=0: the engine stream at the compute stream's priority
    // (batched runs have several steps of slack), else high priority
    const char* np = std::getenv("DSX_NOISE_PRIO");
    const int nprio = (np && np[0] == '0') ? lo_prio : hi_prio;
    if (cudaStreamCreateWithPriority(&lab->nstream, cudaStreamNonBlocking, nprio) != cudaSuccess)
      return cleanup(fail(DSX_ERR_CUDA, "noise stream creation failed"));
    for (int b = 0; b < 2; ++b) {
      cudaEventCreateWithFlags(&lab->ev_noise[b], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&lab->ev_upd[b], cudaEventDisableTiming);
    }
    const char* pl = std::getenv("DSX_NOISE_PIPELINE");
    lab->pipeline = !(pl && pl[0] == '0');
  }
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cleanup(fail(DSX_ERR_CUDA, std::string("lab init: ") + cudaGetErrorString(e)));
  // default rng: worker_rng(0, k)
  if (dsx_lab_seed_rng(lab, 0) != DSX_OK) return cleanup(DSX_ERR_CUDA);
  *out = lab;
  return DSX_OK;
}

dsx_status dsx_lab_destroy(dsx_lab* lab) {
  if (!lab) return DSX_OK;
  cudaSetDevice(lab->device);
  if (lab->stream) cudaStreamSynchronize(lab->stream);
  if (lab->side) cudaStreamSynchronize(lab->side);
  if (lab->nstream) cudaStreamSynchronize(lab->nstream);
  if (lab->comm) ncclCommDestroy(lab->comm);
  delete lab->engine;
  for (void* p : lab->opened) cudaIpcCloseMemHandle(p);
  for (auto& ev : lab->layer_ev)
    if (ev) cudaEventDestroy(ev);
  for (auto& ev : lab->tl_ev)
    if (ev) cudaEventDestroy(ev);
  if (lab->stage64) cudaFree(lab->stage64);
  if (lab->bar) cudaFree(lab->bar);
  if (lab->flags) cudaFree(lab->flags);
  if (lab->xsum) cudaFree(lab->xsum);
  if (lab->sig_counter) cudaFree(lab->sig_counter);
  for (auto& ev : lab->ev_chunk)
    if (ev) cudaEventDestroy(ev);
  for (void* p : {lab->w, (void*)lab->curv, (void*)lab->opt, (void*)lab->noise, (void*)lab->mt, (void*)lab->grad_buf,
                  (void*)lab->what, (void*)lab->tiles, (void*)lab->norm_part, (void*)lab->norm,
                  (void*)lab->maxnorm, (void*)lab->log_part, lab->staging, lab->recv, lab->gmean})
    if (p) cudaFree(p);
  for (auto& ev : lab->ev)
    if (ev) cudaEventDestroy(ev);
  for (auto& ev : lab->iev)
    if (ev) cudaEventDestroy(ev);
  for (auto* v : {&lab->ev_in, &lab->ev_out})
    for (auto& ev : *v)
      if (ev) cudaEventDestroy(ev);
  if (lab->h2d) cudaStreamDestroy(lab->h2d);
  if (lab->d2h) cudaStreamDestroy(lab->d2h);
  if (lab->ev_split) cudaEventDestroy(lab->ev_split);
  if (lab->ev_synced) cudaEventDestroy(lab->ev_synced);
  if (lab->stream) cudaStreamDestroy(lab->stream);
  if (lab->side) cudaStreamDestroy(lab->side);
  if (lab->nstream) cudaStreamDestroy(lab->nstream);
  for (int b = 0; b < 2; ++b) {
    if (lab->ev_noise[b]) cudaEventDestroy(lab->ev_noise[b]);
    if (lab->ev_upd[b]) cudaEventDestroy(lab->ev_upd[b]);
  }
  delete lab;
  return DSX_OK;
}

dsx_status dsx_lab_set_params(dsx_lab* lab, int local, const double* w) {
  DSX_TRY(check_row(lab, local));
  if (!w) return fail(DSX_ERR_ARGUMENT, "null params");
  DSX_TRY(materialize(lab));  // the other rows keep their (lazy) values
  DSX_CUDA(cudaStreamSynchronize(lab->stream));
  if (lab->dtype == DSX_F64) {
    DSX_CUDA(cudaMemcpy(static_cast<double*>(lab->w) + (long long)local * lab->ld, w, 8 * lab->dim,
                        cudaMemcpyHostToDevice));
  } else {
    std::vector<float> tmp(w, w + lab->dim);
    DSX_CUDA(cudaMemcpy(static_cast<float*>(lab->w) + (long long)local * lab->ld, tmp.data(), 4 * lab->dim,
                        cudaMemcpyHostToDevice));
  }
  return DSX_OK;
}

dsx_status dsx_lab_get_params(dsx_lab* lab, int local, double* w) {
  DSX_TRY(check_row(lab, local));
  if (!w) return fail(DSX_ERR_ARGUMENT, "null params");
  DSX_TRY(materialize(lab));
  DSX_CUDA(cudaStreamSynchronize(lab->stream));
  DSX_CUDA(cudaStreamSynchronize(lab->side));
  if (lab->dtype == DSX_F64) {
    DSX_CUDA(cudaMemcpy(w, static_cast<double*>(lab->w) + (long long)local * lab->ld, 8 * lab->dim,
                        cudaMemcpyDeviceToHost));
  } else {
    std::vector<float> tmp(lab->dim);
    DSX_CUDA(cudaMemcpy(tmp.data(), static_cast<float*>(lab->w) + (long long)local * lab->ld, 4 * lab->dim,
                        cudaMemcpyDeviceToHost));
    std::copy(tmp.begin(), tmp.end(), w);
  }
  return DSX_OK;
}

dsx_status dsx_lab_set_all_params(dsx_lab* lab, const double* w) {
  DSX_TRY(check_lab(lab));
  if (!w) return fail(DSX_ERR_ARGUMENT, "null params");
  DSX_CUDA(cudaStreamSynchronize(lab->side));
  drop_stale(lab);
  if (lab->dtype == DSX_F64) {
    DSX_CUDA(cudaMemcpy2DAsync(lab->w, 8 * lab->ld, w, 8 * lab->dim, 8 * lab->dim, lab->kl,
                               cudaMemcpyHostToDevice, lab->stream));
    return DSX_OK;
  }
  return set_all_f32(lab, w);
}

dsx_status dsx_lab_set_state(dsx_lab* lab, const double* w, const uint64_t* rng) {
  DSX_TRY(check_lab(lab));
  DSX_CUDA(cudaStreamSynchronize(lab->stream));
  DSX_CUDA(cudaStreamSynchronize(lab->side));
  if (w) drop_stale(lab);
  if (rng) DSX_TRY(invalidate_prefetch(lab));
  if (w) {
    if (lab->dtype == DSX_F64) {
      DSX_CUDA(cudaMemcpy2DAsync(lab->w, 8 * lab->ld, w, 8 * lab->dim, 8 * lab->dim, lab->kl,
                                 cudaMemcpyHostToDevice, lab->stream));
    } else {
      DSX_TRY(set_all_f32(lab, w));
    }
  }
  if (rng) {
    for (int k = 0; k < lab->kl; ++k)
      if (rng[(long long)k * (kMtN + 1) + kMtN] > kMtN) return fail(DSX_ERR_ARGUMENT, "bad rng cursor");
    DSX_CUDA(cudaMemcpyAsync(mt_state(lab, lab->mt_commit), rng, 8ull * (kMtN + 1) * lab->kl,
                             cudaMemcpyHostToDevice, lab->stream));
  }
  DSX_CUDA(cudaStreamSynchronize(lab->stream));
  return DSX_OK;
}

dsx_status dsx_lab_get_state(dsx_lab* lab, double* w, uint64_t* rng) {
  DSX_TRY(check_lab(lab));
  if (w) DSX_TRY(materialize(lab));
  DSX_CUDA(cudaStreamSynchronize(lab->side));
  if (lab->nstream) DSX_CUDA(cudaStreamSynchronize(lab->nstream));
  if (w) {
    if (lab->dtype == DSX_F64) {
      DSX_CUDA(cudaMemcpy2DAsync(w, 8 * lab->dim, lab->w, 8 * lab->ld, 8 * lab->dim, lab->kl,
                                 cudaMemcpyDeviceToHost, lab->stream));
    } else {
      DSX_TRY(get_all_f32(lab, w));
    }
  }
  if (rng) {
    DSX_CUDA(cudaMemcpyAsync(rng, mt_state(lab, lab->mt_commit), 8ull * (kMtN + 1) * lab->kl,
                             cudaMemcpyDeviceToHost, lab->stream));
  }
  DSX_CUDA(cudaStreamSynchronize(lab->stream));
  return DSX_OK;
}

dsx_status dsx_lab_step_host(dsx_lab* lab, double eta, const unsigned char* mask, double* const* rows,
                             uint64_t* rng) {
  DSX_TRY(check_lab(lab));
  if (!mask || !rows || !rng) return fail(DSX_ERR_ARGUMENT, "null step_host argument");
  for (int k = 0; k < lab->kl; ++k) {
    if (!rows[k]) return fail(DSX_ERR_ARGUMENT, "null worker row");
    if (rng[(long long)k * (kMtN + 1) + kMtN] > kMtN) return fail(DSX_ERR_ARGUMENT, "bad rng cursor");
  }
  DSX_CUDA(cudaStreamSynchronize(lab->stream));
  DSX_CUDA(cudaStreamSynchronize(lab->side));
  drop_stale(lab);
  const size_t rng_words = (size_t)(kMtN + 1) * lab->kl;
  // the caller handing back the states this lab returned last time (a
  // training loop) keeps the noise generated ahead for them; any other
  // state drops it
  const bool rng_hit = lab->host_rng_valid && lab->engine && lab->host_rng.size() == rng_words &&
                       std::memcmp(lab->host_rng.data(), rng, 8 * rng_words) == 0;
  if (!rng_hit) DSX_TRY(invalidate_prefetch(lab));
  lab->host_rng_valid = false;
  // fresh engine runs here are one step; runs generated ahead use the batch
  struct PipelineOff {
    dsx_lab* l;
    bool on;
    ~PipelineOff() { l->pipeline = on; }
  } guard{lab, lab->pipeline};
  lab->pipeline = false;
  const long long D = (long long)lab->dim;
  bool contiguous = true;  // rows packed as one [kl][dim] buffer
  for (int k = 1; k < lab->kl; ++k)
    if (rows[k] != rows[0] + (long long)k * D) contiguous = false;
  if (lab->dtype != DSX_F64 || lab->nranks != 1 || lab->link_bw > 0.0 || lab->use_chain) {
    // the staged path: whole rows in (one async copy, overlapping the noise
    // engine), one step, whole rows out
    DSX_CUDA(cudaMemcpy(mt_state(lab, lab->mt_commit), rng, 8ull * (kMtN + 1) * lab->kl, cudaMemcpyHostToDevice));
    if (contiguous) DSX_TRY(dsx_lab_set_all_params(lab, rows[0]));
    else
      for (int k = 0; k < lab->kl; ++k) DSX_TRY(dsx_lab_set_params(lab, k, rows[k]));
    DSX_TRY(dsx_lab_step(lab, eta, mask));
    if (contiguous) DSX_TRY(dsx_lab_get_all_params(lab, rows[0]));
    else
      for (int k = 0; k < lab->kl; ++k) DSX_TRY(dsx_lab_get_params(lab, k, rows[k]));
    return dsx_lab_get_state(lab, nullptr, rng);
  }
  if (!lab->h2d) {
    DSX_CUDA(cudaStreamCreateWithFlags(&lab->h2d, cudaStreamNonBlocking));
    DSX_CUDA(cudaStreamCreateWithFlags(&lab->d2h, cudaStreamNonBlocking));
  }
  if (const char* c = std::getenv("DSX_HOST_CHUNKS")) lab->host_chunks = std::max(1, std::atoi(c));
  const int C = std::max(1, std::min(lab->host_chunks, lab->ntiles));
  while ((int)lab->ev_in.size() < C) {
    cudaEvent_t a, b;
    DSX_CUDA(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
    DSX_CUDA(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
    lab->ev_in.push_back(a);
    lab->ev_out.push_back(b);
  }
  // engine states first (small), then the noise engine overlaps the first
  // parameter chunks' transfer (or its output is already there: rng_hit)
  if (!rng_hit)
    DSX_CUDA(cudaMemcpy(mt_state(lab, lab->mt_commit), rng, 8ull * (kMtN + 1) * lab->kl, cudaMemcpyHostToDevice));
  if (lab->instrument) DSX_CUDA(cudaEventRecord(lab->iev[0], lab->stream));
  int noise = 0;
  DSX_TRY(run_noise(lab, &noise));
  if (lab->instrument) DSX_CUDA(cudaEventRecord(lab->iev[5], lab->stream));
  MaskBits bits{};
  for (int b = 0; b < lab->L; ++b)
    if (mask[b + 1]) bits.w[b >> 5] |= 1u << (b & 31);
  double* w = static_cast<double*>(lab->w);
  // rows at a constant host pitch (one [kl][pitch] buffer) move as one 2D
  // copy per chunk and direction
  long long pitch = lab->kl > 1 ? (long long)(rows[1] - rows[0]) : (long long)D;
  for (int k = 1; k < lab->kl && pitch >= D; ++k)
    if (rows[k] - rows[k - 1] != pitch) pitch = 0;
  const bool strided = pitch >= D;
  // (every stream touching the rows was drained above)
  for (int c = 0; c < C; ++c) {
    const int tb = (int)((long long)lab->ntiles * c / C), te = (int)((long long)lab->ntiles * (c + 1) / C);
    if (te <= tb) continue;
    const long long lo = lab->h_tiles[tb].start;
    const long long hi = te < lab->ntiles ? lab->h_tiles[te].start : D;
    if (strided) {
      DSX_CUDA(cudaMemcpy2DAsync(w + lo, 8 * lab->ld, rows[0] + lo, 8 * pitch, 8ull * (hi - lo), lab->kl,
                                 cudaMemcpyHostToDevice, lab->h2d));
    } else {
      for (int k = 0; k < lab->kl; ++k)
        DSX_CUDA(cudaMemcpyAsync(w + (long long)k * lab->ld + lo, rows[k] + lo, 8ull * (hi - lo),
                                 cudaMemcpyHostToDevice, lab->h2d));
    }
    DSX_CUDA(cudaEventRecord(lab->ev_in[c], lab->h2d));
    DSX_CUDA(cudaStreamWaitEvent(lab->stream, lab->ev_in[c], 0));
    launch_update<double>(lab, lab->stream, tb, te - tb, noise, lab->K > 1, bits, eta);
    DSX_CUDA(cudaEventRecord(lab->ev_out[c], lab->stream));
    DSX_CUDA(cudaStreamWaitEvent(lab->d2h, lab->ev_out[c], 0));
    if (strided) {
      DSX_CUDA(cudaMemcpy2DAsync(rows[0] + lo, 8 * pitch, w + lo, 8 * lab->ld, 8ull * (hi - lo), lab->kl,
                                 cudaMemcpyDeviceToHost, lab->d2h));
    } else {
      for (int k = 0; k < lab->kl; ++k)
        DSX_CUDA(cudaMemcpyAsync(rows[k] + lo, w + (long long)k * lab->ld + lo, 8ull * (hi - lo),
                                 cudaMemcpyDeviceToHost, lab->d2h));
    }
  }
  lab->has_ranges = false;
  lab->synced_last = false;
  if (lab->instrument) DSX_CUDA(cudaEventRecord(lab->iev[3], lab->stream));
  DSX_CUDA(cudaMemsetAsync(lab->maxnorm, 0, 8, lab->stream));
  norm_finalize_kernel<<<lab->kl, 1024, 0, lab->stream>>>(
      lab->norm_part, lab->ntiles, lab->norm, reinterpret_cast<unsigned long long*>(lab->maxnorm));
  ++lab->launches;
  if (lab->instrument) DSX_CUDA(cudaEventRecord(lab->iev[4], lab->stream));
  DSX_TRY(after_update(lab, noise));
  // generate the next engine run now, from the state this call returns,
  // while the parameters stream back (and the caller does its host work)
  if (noise == 2 && lab->pf_set < 0 && lab->batch_set >= 0 && lab->batch_t >= lab->batch_n) {
    const int set = 1 - lab->batch_set;
    DSX_TRY(launch_engine(lab, set, lab->tmax, boundary_slot(lab, lab->batch_set, lab->batch_n - 1)));
    lab->pf_set = set;
    lab->pf_n = lab->tmax;
  }
  DSX_CUDA(cudaMemcpyAsync(rng, mt_state(lab, lab->mt_commit), 8ull * (kMtN + 1) * lab->kl,
                           cudaMemcpyDeviceToHost, lab->stream));
  DSX_CUDA(cudaStreamSynchronize(lab->d2h));
  DSX_CUDA(cudaStreamSynchronize(lab->stream));
  DSX_CUDA(cudaGetLastError());
  if (noise == 2) {
    lab->host_rng.assign(rng, rng + rng_words);
    lab->host_rng_valid = true;
  }
  return DSX_OK;
}

dsx_status dsx_host_alloc(size_t bytes, void** out) {
  if (!out) return fail(DSX_ERR_ARGUMENT, "null out");
  *out = nullptr;
  DSX_CUDA(cudaHostAlloc(out, bytes, cudaHostAllocPortable));
  return DSX_OK;
}

dsx_status dsx_host_free(void* p) {
  if (p) DSX_CUDA(cudaFreeHost(p));
  return DSX_OK;
}

dsx_status dsx_lab_get_all_params(dsx_lab* lab, double* w) {
  DSX_TRY(check_lab(lab));
  if (!w) return fail(DSX_ERR_ARGUMENT, "null params");
  DSX_TRY(materialize(lab));
  if (lab->dtype == DSX_F64) {
    DSX_CUDA(cudaStreamSynchronize(lab->side));
    DSX_CUDA(cudaMemcpy2DAsync(w, 8 * lab->dim, lab->w, 8 * lab->ld, 8 * lab->dim, lab->kl,
                               cudaMemcpyDeviceToHost, lab->stream));
    DSX_CUDA(cudaStreamSynchronize(lab->stream));
    return DSX_OK;
  }
  DSX_CUDA(cudaStreamSynchronize(lab->side));
  DSX_TRY(get_all_f32(lab, w));
  DSX_CUDA(cudaStreamSynchronize(lab->stream));
  return DSX_OK;
}

dsx_status dsx_lab_fill_params(dsx_lab* lab, double value) {
  DSX_TRY(check_lab(lab));
  std::vector<double> row(lab->dim, value);
  for (int k = 0; k < lab->kl; ++k) DSX_TRY(dsx_lab_set_params(lab, k, row.data()));
  return DSX_OK;
}

dsx_status dsx_lab_set_rng(dsx_lab* lab, int local, const uint64_t* x312, uint64_t p) {
  DSX_TRY(check_row(lab, local));
  if (!x312 || p > kMtN) return fail(DSX_ERR_ARGUMENT, "bad rng state");
  uint64_t buf[kMtN + 1];
  std::memcpy(buf, x312, 8 * kMtN);
  buf[kMtN] = p;
  DSX_CUDA(cudaStreamSynchronize(lab->stream));
  DSX_TRY(invalidate_prefetch(lab));
  DSX_CUDA(cudaMemcpy(mt_state(lab, lab->mt_commit) + (long long)local * (kMtN + 1), buf, sizeof buf,
                      cudaMemcpyHostToDevice));
  return DSX_OK;
}

dsx_status dsx_lab_get_rng(dsx_lab* lab, int local, uint64_t* x312, uint64_t* p) {
  DSX_TRY(check_row(lab, local));
  if (!x312 || !p) return fail(DSX_ERR_ARGUMENT, "null rng out");
  uint64_t buf[kMtN + 1];
  DSX_CUDA(cudaStreamSynchronize(lab->stream));
  if (lab->nstream) DSX_CUDA(cudaStreamSynchronize(lab->nstream));
  // the committed state (after the last step's noise), not a prefetched one
  DSX_CUDA(cudaMemcpy(buf, mt_state(lab, lab->mt_commit) + (long long)local * (kMtN + 1), sizeof buf,
                      cudaMemcpyDeviceToHost));
  std::memcpy(x312, buf, 8 * kMtN);
  *p = buf[kMtN];
  return DSX_OK;
}

// worker_rng(seed, k) (trainer.cpp:169-173) for every local row, seeded on
// the host with libstdc++'s own seed_seq and read back through operator<<.
dsx_status dsx_lab_seed_rng(dsx_lab* lab, uint64_t seed) {
  DSX_TRY(check_lab(lab));
  for (int k = 0; k < lab->kl; ++k) {
    const int global = lab->kbegin + k;
    std::seed_seq seq{static_cast<std::uint32_t>(seed), static_cast<std::uint32_t>(seed >> 32),
                      static_cast<std::uint32_t>(global), 0x5eedu};
    std::mt19937_64 eng(seq);
    std::stringstream ss;
    ss << eng;
    uint64_t x[kMtN], p = 0;
    for (int i = 0; i < kMtN; ++i) ss >> x[i];
    ss >> p;
    DSX_TRY(dsx_lab_set_rng(lab, k, x, p));
  }
  return DSX_OK;
}

dsx_status dsx_lab_step(dsx_lab* lab, double eta, const unsigned char* mask) {
  DSX_TRY(check_lab(lab));
  if (!mask) return fail(DSX_ERR_ARGUMENT, "null mask");
  if (lab->instrument) DSX_CUDA(cudaEventRecord(lab->iev[0], lab->stream));
  int noise = 0;
  DSX_TRY(run_noise(lab, &noise));
  if (lab->horizon > 0) --lab->horizon;
  if (lab->instrument) DSX_CUDA(cudaEventRecord(lab->iev[5], lab->stream));
  DSX_TRY(lab->dtype == DSX_F64 ? step_impl<double>(lab, eta, mask, noise)
                                : step_impl<float>(lab, eta, mask, noise));
  return after_update(lab, noise);
}

dsx_status dsx_lab_step_with_noise(dsx_lab* lab, double eta, const unsigned char* mask,
                                   const double* xi) {
  DSX_TRY(check_lab(lab));
  if (!mask || !xi) return fail(DSX_ERR_ARGUMENT, "null mask/noise");
  if (!lab->noise) {
    DSX_CUDA(cudaMalloc(&lab->noise, 8 * (size_t)lab->ld * lab->kl));
  }
  DSX_CUDA(cudaMemcpy2DAsync(lab->noise, 8 * lab->ld, xi, 8 * lab->dim, 8 * lab->dim, lab->kl,
                             cudaMemcpyHostToDevice, lab->stream));
  if (lab->instrument) {
    DSX_CUDA(cudaEventRecord(lab->iev[0], lab->stream));
    DSX_CUDA(cudaEventRecord(lab->iev[5], lab->stream));
  }
  return lab->dtype == DSX_F64 ? step_impl<double>(lab, eta, mask, 1)
                               : step_impl<float>(lab, eta, mask, 1);
}

dsx_status dsx_lab_last_max_grad_norm_sq(dsx_lab* lab, double* out) {
  DSX_TRY(check_lab(lab));
  if (!out) return fail(DSX_ERR_ARGUMENT, "null out");
  if (lab->nranks > 1 && lab->comm) {
    // the reference's max runs over all K workers (trainer.cpp:190-200):
    // every rank holds a max over its own rows, so reduce across ranks
    // (a collective: every rank calls this after the same step)
    DSX_NCCL(ncclAllReduce(lab->maxnorm, lab->maxnorm, 1, ncclDouble, ncclMax, lab->comm, lab->stream));
  }
  DSX_CUDA(cudaStreamSynchronize(lab->stream));
  DSX_CUDA(cudaMemcpy(out, lab->maxnorm, 8, cudaMemcpyDeviceToHost));
  return DSX_OK;
}

dsx_status dsx_lab_sync(dsx_lab* lab) {
  DSX_TRY(check_lab(lab));
  DSX_CUDA(cudaStreamSynchronize(lab->side));
  DSX_CUDA(cudaStreamSynchronize(lab->stream));
  DSX_CUDA(cudaGetLastError());
  return DSX_OK;
}

dsx_status dsx_lab_gradient(dsx_lab* lab, int local, double* g_out) {
  DSX_TRY(check_row(lab, local));
  if (!g_out) return fail(DSX_ERR_ARGUMENT, "null gradient out");
  int nm = 0;
  DSX_TRY(materialize(lab));
  DSX_TRY(invalidate_prefetch(lab));
  DSX_TRY(run_noise(lab, &nm));  // advances every local row's stream
  double* g = nullptr;
  if (!lab->grad_buf) DSX_CUDA(cudaMalloc(&lab->grad_buf, 8 * lab->dim));
  g = lab->grad_buf;
  const double* xi = nm == 1 ? lab->noise + (long long)local * lab->ld : nullptr;
  const NoiseView nv = lab->engine ? lab->engine->view(lab->cur_set, lab->cur_t) : NoiseView{};
  if (lab->dtype == DSX_F64) {
    gradient_kernel<double><<<lab->nsm * 4, 256, 0, lab->stream>>>(
        static_cast<const double*>(lab->w) + (long long)local * lab->ld, lab->dim, lab->q, nm, xi, nv,
        local, g);
  } else {
    gradient_kernel<float><<<lab->nsm * 4, 256, 0, lab->stream>>>(
        static_cast<const float*>(lab->w) + (long long)local * lab->ld, lab->dim, lab->q, nm, xi, nv,
        local, g);
  }
  ++lab->launches;
  DSX_CUDA(cudaMemcpyAsync(g_out, g, 8 * lab->dim, cudaMemcpyDeviceToHost, lab->stream));
  DSX_CUDA(cudaStreamSynchronize(lab->stream));
  return DSX_OK;
}

// Multi-rank: every rank keeps the same w_hat (it accumulates the global
// mean); the per-layer Gamma partials of the local rows are summed over
// ranks, the objectives are identical on every rank.
dsx_status dsx_lab_mean_accumulate(dsx_lab* lab, double weight) {
  DSX_TRY(check_lab(lab));
  if (!lab->what) {
    DSX_CUDA(cudaMalloc(&lab->what, 8 * lab->dim));
    DSX_CUDA(cudaMemsetAsync(lab->what, 0, 8 * lab->dim, lab->stream));
  }
  return lab->dtype == DSX_F64 ? rowwise<double>(lab, 0, weight, 0.0) : rowwise<float>(lab, 0, weight, 0.0);
}

dsx_status dsx_lab_log(dsx_lab* lab, double weight_total, double* gamma_per_layer, double* out2) {
  DSX_TRY(check_lab(lab));
  if (!gamma_per_layer || !out2) return fail(DSX_ERR_ARGUMENT, "null log outputs");
  if (!lab->what) {
    DSX_CUDA(cudaMalloc(&lab->what, 8 * lab->dim));
    DSX_CUDA(cudaMemsetAsync(lab->what, 0, 8 * lab->dim, lab->stream));
  }
  DSX_TRY(lab->dtype == DSX_F64 ? rowwise<double>(lab, 1, 0.0, weight_total)
                                : rowwise<float>(lab, 1, 0.0, weight_total));
  if (lab->nranks > 1)
    DSX_NCCL(ncclAllReduce(lab->log_part, lab->log_part, (size_t)lab->ntiles, ncclFloat64, ncclSum, lab->comm,
                           lab->stream));
  std::vector<double> part(3 * (size_t)lab->ntiles);
  DSX_CUDA(cudaMemcpyAsync(part.data(), lab->log_part, 8 * part.size(), cudaMemcpyDeviceToHost, lab->stream));
  DSX_CUDA(cudaStreamSynchronize(lab->stream));
  for (int b = 0; b < lab->L; ++b) gamma_per_layer[b] = 0.0;
  double fh = 0.0, fm = 0.0;
  for (int t = 0; t < lab->ntiles; ++t) {
    gamma_per_layer[lab->h_tiles[t].block] += part[t];
    fh += part[lab->ntiles + t];
    fm += part[2 * lab->ntiles + t];
  }
  for (int b = 0; b < lab->L; ++b) gamma_per_layer[b] /= static_cast<double>(lab->K);
  out2[0] = fh;
  out2[1] = fm;
  return DSX_OK;
}

dsx_status dsx_nccl_unique_id(unsigned char id[128]) {
  if (!id) return fail(DSX_ERR_ARGUMENT, "null id");
  ncclUniqueId u;
  DSX_NCCL(ncclGetUniqueId(&u));
  std::memcpy(id, u.internal, 128);
  return DSX_OK;
}

namespace {

// Communicator-independent part of joining a multi-rank run: rank layout,
// exactness check, exchange buffers, overlap groups.
dsx_status comm_prepare(dsx_lab* lab, int nranks, int rank, int sync_algo) {
  lab->nranks = nranks;
  lab->rank = rank;
  lab->sync_algo = sync_algo;
  // Exactness needs every rank's rows to be a subtree of the pairwise tree.
  lab->local_subtree = is_subtree(lab->K, lab->kbegin, lab->kl);
  for (int r = 0; r < nranks && lab->local_subtree; ++r)
    lab->local_subtree = is_subtree(lab->K, r * lab->kl, lab->kl);
  if (sync_algo == DSX_SYNC_PAIRWISE && !lab->local_subtree)
    return fail(DSX_ERR_ARGUMENT, "pairwise sync needs rank worker ranges aligned to the pairwise tree");
  build_prog(nranks, &lab->prog_ranks);
  const size_t es = elem_size(lab);
  lab->staging_elems = lab->dim;
  if (lab->kl > 1) DSX_CUDA(cudaMalloc(&lab->staging, es * lab->dim));
  DSX_CUDA(cudaMalloc(&lab->recv, es * (lab->dim / nranks + 1) * nranks));
  DSX_CUDA(cudaMalloc(&lab->bar, 4));
  DSX_CUDA(cudaMemset(lab->bar, 0, 4));
  for (auto& ev : lab->ev_chunk) DSX_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  // Overlap groups: the local step runs in backward-order tile groups and
  // each group's average starts while the next group updates.  Round 2, exact-window timing, 2 GPUs x 4 rows: 1 group 1607 it/s with
  // 99 % of the sync exposed; 2 / 3 / 6 groups 1628 / 1620 / 1614 it/s with
  // 54 / 43 / 33 % exposed -> 6 groups everywhere
  lab->chunks = 6;
  if (const char* c = std::getenv("DSX_SYNC_CHUNKS")) lab->chunks = std::max(1, std::min(kMaxChunks, std::atoi(c)));
  {
    const int nm = lab->sigma > 0.0 ? 2 : 0;
    lab->wave = lab->nsm * (lab->dtype == DSX_F64 ? update_blocks_per_sm<double>(lab->kl, nm)
                                                  : update_blocks_per_sm<float>(lab->kl, nm));
  }
  if (const char* z = std::getenv("DSX_LAZY")) lab->lazy = z[0] != '0';

  DSX_CUDA(cudaMalloc(&lab->flags, 8 * kFlagWords));
  DSX_CUDA(cudaMemset(lab->flags, 0, 8 * kFlagWords));
  DSX_CUDA(cudaMalloc(&lab->sig_counter, 4));
  DSX_CUDA(cudaMemset(lab->sig_counter, 0, 4));
  DSX_CUDA(cudaMalloc(&lab->xsum, es * 2 * lab->ld));  // [2][ld]: 16-B aligned halves
  return DSX_OK;
}

// The exchange buffers of one rank, in the order the peers map them:
// averaging exchange row, flag block, probe scratch.
constexpr int kNB = 3;
void exchange_buffers(dsx_lab* lab, void* out[kNB]) {
  out[0] = lab->kl == 1 ? lab->w : lab->staging;
  out[1] = lab->flags;
  out[2] = lab->xsum;
}

void set_peer(dsx_lab* lab, int q, void* const got[kNB]) {
  lab->peers.p[q] = got[0];
  lab->fpeers.p[q] = static_cast<unsigned long long*>(got[1]);
  if (q < kMaxFuse) lab->xpeer[q] = got[2];
}

// After the peers are mapped (or not): barrier flavour, engine SM budget.
dsx_status comm_finish(dsx_lab* lab, int ok, int nranks) {
  lab->p2p = ok != 0;
  if (const char* t = std::getenv("DSX_FLAG_TIMEOUT_S"))
    lab->flag_timeout_ns = (unsigned long long)std::max(1.0, std::atof(t)) * 1000000000ull;
  const char* fb = std::getenv("DSX_FLAG_BARRIER");
  lab->flag_bar = lab->p2p && !(fb && fb[0] == '0');
  // Several ranks: size the noise engine's segment wave for two thirds of the
  // SMs.  A resident engine run then never blocks the update and the average
  // (2 GPUs: 1510 -> 1710 it/s, 4 GPUs: 2260 -> 2590); one GPU keeps every
  // SM for its engine-bound step.  DSX_ENGINE_SMS overrides.
  if (lab->engine && nranks > 1 && !std::getenv("DSX_ENGINE_SMS")) {
    DSX_TRY(invalidate_prefetch(lab));
    DSX_CUDA(cudaStreamSynchronize(lab->stream));
    auto* e = new dsx::NoiseEngine();
    std::string err;
    if (!e->init(lab->dim, lab->kl, std::max(1, lab->nsm * 2 / 3), lab->tmax, &err)) {
      delete e;
      return fail(DSX_ERR_CUDA, err);
    }
    delete lab->engine;
    lab->engine = e;
  }
  return DSX_OK;
}

}  // namespace

dsx_status dsx_lab_comm_init(dsx_lab* lab, const unsigned char id[128], int nranks, int rank,
                             int sync_algo) {
  DSX_TRY(check_lab(lab));
  if (!id || nranks < 1 || rank < 0 || rank >= nranks) return fail(DSX_ERR_ARGUMENT, "bad comm args");
  if (sync_algo != DSX_SYNC_PAIRWISE && sync_algo != DSX_SYNC_NCCL_AVG)
    return fail(DSX_ERR_ARGUMENT, "bad sync algorithm");
  if (lab->comm) return fail(DSX_ERR_STATE, "comm already initialised");
  if (lab->K % nranks != 0 || lab->kl != lab->K / nranks || lab->kbegin != rank * lab->kl)
    return fail(DSX_ERR_ARGUMENT, "ranks must hold equal contiguous worker ranges");
  ncclUniqueId u;
  std::memcpy(u.internal, id, 128);
  DSX_NCCL(ncclCommInitRank(&lab->comm, nranks, u, rank));
  DSX_TRY(comm_prepare(lab, nranks, rank, sync_algo));
  // NVLink peer-memory exchange: map every rank's exchange buffer (its only
  // worker row, or its subtree-sum staging) through CUDA IPC.  All ranks must
  // agree on using it, so the per-rank outcome is min-reduced.
  const char* p2p_env = std::getenv("DSX_P2P");
  int ok = (p2p_env && p2p_env[0] == '0') || nranks > kMaxProg ? 0 : 1;
  // three handles per rank: exchange buffer, flag block, probe scratch
  constexpr size_t kH = sizeof(cudaIpcMemHandle_t);
  void* bufs[kNB];
  exchange_buffers(lab, bufs);
  cudaIpcMemHandle_t mine[kNB]{};
  for (int b = 0; b < kNB && ok; ++b)
    if (cudaIpcGetMemHandle(&mine[b], bufs[b]) != cudaSuccess) ok = 0;
  char* d_handles = nullptr;
  int* d_ok = nullptr;
  DSX_CUDA(cudaMalloc(&d_handles, kNB * kH * nranks));
  DSX_CUDA(cudaMalloc(&d_ok, 4));
  DSX_CUDA(cudaMemcpy(d_handles + kNB * kH * rank, mine, kNB * kH, cudaMemcpyHostToDevice));
  DSX_CUDA(cudaMemcpy(d_ok, &ok, 4, cudaMemcpyHostToDevice));
  DSX_NCCL(ncclAllGather(d_handles + kNB * kH * rank, d_handles, kNB * kH, ncclChar, lab->comm, lab->side));
  DSX_NCCL(ncclAllReduce(d_ok, d_ok, 1, ncclInt32, ncclMin, lab->comm, lab->side));
  DSX_CUDA(cudaStreamSynchronize(lab->side));
  std::vector<cudaIpcMemHandle_t> handles(kNB * (size_t)nranks);
  DSX_CUDA(cudaMemcpy(handles.data(), d_handles, kNB * kH * nranks, cudaMemcpyDeviceToHost));
  DSX_CUDA(cudaMemcpy(&ok, d_ok, 4, cudaMemcpyDeviceToHost));
  int local_ok = ok;
  if (ok) {
    for (int q = 0; q < nranks && local_ok; ++q) {
      void* got[kNB];
      for (int b = 0; b < kNB; ++b) {
        if (q == rank) {
          got[b] = bufs[b];
          continue;
        }
        void* ptr = nullptr;
        if (cudaIpcOpenMemHandle(&ptr, handles[kNB * q + b], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
          cudaGetLastError();
          local_ok = 0;
          break;
        }
        lab->opened.push_back(ptr);
        got[b] = ptr;
      }
      if (!local_ok) break;
      set_peer(lab, q, got);
    }
  }
  DSX_CUDA(cudaMemcpy(d_ok, &local_ok, 4, cudaMemcpyHostToDevice));
  DSX_NCCL(ncclAllReduce(d_ok, d_ok, 1, ncclInt32, ncclMin, lab->comm, lab->side));
  DSX_CUDA(cudaStreamSynchronize(lab->side));
  DSX_CUDA(cudaMemcpy(&ok, d_ok, 4, cudaMemcpyDeviceToHost));
  cudaFree(d_handles);
  cudaFree(d_ok);
  return comm_finish(lab, ok, nranks);
}

// Restores the calling thread's current device when a multi-device entry
// point returns (callers such as torch keep using the device they had).
struct CurrentDeviceGuard {
  int dev = 0;
  CurrentDeviceGuard() { cudaGetDevice(&dev); }
  ~CurrentDeviceGuard() { cudaSetDevice(dev); }
};

dsx_status dsx_lab_comm_init_local(dsx_lab* const* labs, int n, int sync_algo) {
  const CurrentDeviceGuard keep_device;
  if (!labs || n < 1 || n > kMaxProg) return fail(DSX_ERR_ARGUMENT, "bad lab group");
  if (sync_algo != DSX_SYNC_PAIRWISE && sync_algo != DSX_SYNC_NCCL_AVG)
    return fail(DSX_ERR_ARGUMENT, "bad sync algorithm");
  std::vector<int> devs(n);
  for (int r = 0; r < n; ++r) {
    DSX_TRY(check_lab(labs[r]));
    if (labs[r]->comm) return fail(DSX_ERR_STATE, "comm already initialised");
    if (labs[r]->K % n != 0 || labs[r]->kl != labs[r]->K / n || labs[r]->kbegin != r * labs[r]->kl)
      return fail(DSX_ERR_ARGUMENT, "labs must hold equal contiguous worker ranges in rank order");
    devs[r] = labs[r]->device;
    for (int q = 0; q < r; ++q)
      if (devs[q] == devs[r]) return fail(DSX_ERR_ARGUMENT, "one lab per device");
  }
  // one process, one communicator per device (NCCL's single-thread init)
  std::vector<ncclComm_t> comms(n);
  DSX_NCCL(ncclCommInitAll(comms.data(), n, devs.data()));
  for (int r = 0; r < n; ++r) {
    DSX_CUDA(cudaSetDevice(devs[r]));
    labs[r]->comm = comms[r];
    DSX_TRY(comm_prepare(labs[r], n, r, sync_algo));
  }
  // peer buffers are plain device pointers here (unified addressing + peer
  // access), not IPC mappings
  const char* p2p_env = std::getenv("DSX_P2P");
  int ok = (p2p_env && p2p_env[0] == '0') ? 0 : 1;
  for (int r = 0; r < n && ok; ++r) {
    DSX_CUDA(cudaSetDevice(devs[r]));
    for (int q = 0; q < n && ok; ++q) {
      if (q == r) continue;
      int can = 0;
      DSX_CUDA(cudaDeviceCanAccessPeer(&can, devs[r], devs[q]));
      if (!can) {
        ok = 0;
        break;
      }
      const cudaError_t e = cudaDeviceEnablePeerAccess(devs[q], 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) ok = 0;
      cudaGetLastError();
    }
  }
  if (ok) {
    for (int r = 0; r < n; ++r) {
      for (int q = 0; q < n; ++q) {
        void* got[kNB];
        exchange_buffers(labs[q], got);
        set_peer(labs[r], q, got);
      }
    }
  }
  for (int r = 0; r < n; ++r) {
    DSX_CUDA(cudaSetDevice(devs[r]));
    DSX_TRY(comm_finish(labs[r], ok, n));
  }
  return DSX_OK;
}

dsx_status dsx_p2p_average_selftest(int nranks, long long n, double* max_abs_err) {
  const CurrentDeviceGuard keep_device;
  if (!max_abs_err || nranks < 1 || nranks > kMaxProg || n < 1) return fail(DSX_ERR_ARGUMENT, "bad selftest args");
  *max_abs_err = -1.0;
  int ndev = 0;
  DSX_CUDA(cudaGetDeviceCount(&ndev));
  if (ndev < 1) return fail(DSX_ERR_CUDA, "no CUDA device");
  std::vector<int> dev(nranks);
  for (int r = 0; r < nranks; ++r) dev[r] = r % ndev;
  for (int a = 0; a < std::min(ndev, nranks); ++a) {
    DSX_CUDA(cudaSetDevice(a));
    for (int b = 0; b < std::min(ndev, nranks); ++b) {
      if (a == b) continue;
      int can = 0;
      DSX_CUDA(cudaDeviceCanAccessPeer(&can, a, b));
      if (!can) return fail(DSX_ERR_CUDA, "no peer access between the devices");
      const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return fail(DSX_ERR_CUDA, "peer access");
      cudaGetLastError();
    }
  }
  // rank r's row: distinct, non-representable-sum values (rounding matters)
  std::vector<std::vector<double>> host(nranks, std::vector<double>(n));
  for (int r = 0; r < nranks; ++r)
    for (long long i = 0; i < n; ++i) host[r][i] = std::sin(0.37 * (double)i + 1.7 * r) * (1.0 + 0.1 * r) + 1e-3 * r;
  PeerPtrs peers{};
  for (int r = 0; r < nranks; ++r) {
    DSX_CUDA(cudaSetDevice(dev[r]));
    DSX_CUDA(cudaMalloc(&peers.p[r], 8 * n));
    DSX_CUDA(cudaMemcpy(peers.p[r], host[r].data(), 8 * n, cudaMemcpyHostToDevice));
  }
  PairProg prog{};
  build_prog(nranks, &prog);
  // every rank averages its slice, like the step's averaging kernel
  for (int r = 0; r < nranks; ++r) {
    DSX_CUDA(cudaSetDevice(dev[r]));
    const long long base = n / nranks, extra = n % nranks;
    const long long a = r * base + std::min<long long>(r, extra);
    const long long e = a + base + (r < extra ? 1 : 0);
    const int blocks = (int)std::min<long long>(592, ((e - a) / 2 + 255) / 256 + 1);
    switch (nranks) {
      case 2: p2p_average_kernel<double, 2><<<blocks, 256>>>(peers, a, e, nranks, prog, Signal{}); break;
      case 4: p2p_average_kernel<double, 4><<<blocks, 256>>>(peers, a, e, nranks, prog, Signal{}); break;
      case 8: p2p_average_kernel<double, 8><<<blocks, 256>>>(peers, a, e, nranks, prog, Signal{}); break;
      default: p2p_average_kernel<double, 0><<<blocks, 256>>>(peers, a, e, nranks, prog, Signal{});
    }
    DSX_CUDA(cudaGetLastError());
  }
  for (int d = 0; d < std::min(ndev, nranks); ++d) {
    DSX_CUDA(cudaSetDevice(d));
    DSX_CUDA(cudaDeviceSynchronize());
  }
  // expected: pairwise_coord_sum over the ranks / K (trainer.cpp:31-38)
  std::vector<double> col(nranks);
  std::function<double(int, int)> pw = [&](int lo, int cnt) -> double {
    if (cnt == 1) return col[lo];
    if (cnt == 2) return col[lo] + col[lo + 1];
    return pw(lo, cnt / 2) + pw(lo + cnt / 2, cnt - cnt / 2);
  };
  double worst = 0.0;
  std::vector<double> got(n);
  std::vector<double> want(n);
  for (long long i = 0; i < n; ++i) {
    for (int r = 0; r < nranks; ++r) col[r] = host[r][i];
    want[i] = pw(0, nranks) / (double)nranks;
  }
  for (int r = 0; r < nranks; ++r) {
    DSX_CUDA(cudaSetDevice(dev[r]));
    DSX_CUDA(cudaMemcpy(got.data(), peers.p[r], 8 * n, cudaMemcpyDeviceToHost));
    for (long long i = 0; i < n; ++i) worst = std::max(worst, std::fabs(got[i] - want[i]));
    cudaFree(peers.p[r]);
  }
  *max_abs_err = worst;
  return DSX_OK;
}

dsx_status dsx_lab_link_probe(dsx_lab* lab, int reps, double* gbs) {
  DSX_TRY(check_lab(lab));
  if (!gbs) return fail(DSX_ERR_ARGUMENT, "null out");
  *gbs = 0.0;
  if (lab->nranks < 2) return DSX_OK;
  if (!lab->p2p) return fail(DSX_ERR_STATE, "link probe needs the NVLink peer-memory exchange");
  const int W = lab->nranks;
  // scratch: every rank's probe buffer [2][ld] (mapped into all
  // peers at comm init, idle between steps) as 16-B units
  const long long units = (long long)(elem_size(lab) * 2 * lab->ld / 16);
  const long long per = units / W;
  const long long a = per * lab->rank, b = a + per;
  PeerPtrs pp{};
  for (int q = 0; q < W; ++q) pp.p[q] = lab->xpeer[q];
  DSX_CUDA(cudaStreamSynchronize(lab->stream));
  DSX_CUDA(cudaStreamSynchronize(lab->side));
  auto barrier = [&]() -> dsx_status {
    DSX_NCCL(ncclAllReduce(lab->bar, lab->bar, 1, ncclInt32, ncclSum, lab->comm, lab->side));
    DSX_CUDA(cudaStreamSynchronize(lab->side));
    return DSX_OK;
  };
  auto launch = [&]() {
    const int grid = lab->nsm * 4;
    switch (W) {
      case 2: p2p_probe_kernel<2><<<grid, 256, 0, lab->side>>>(pp, a, b); break;
      case 4: p2p_probe_kernel<4><<<grid, 256, 0, lab->side>>>(pp, a, b); break;
      case 8: p2p_probe_kernel<8><<<grid, 256, 0, lab->side>>>(pp, a, b); break;
      default: break;
    }
  };
  if (W != 2 && W != 4 && W != 8) return fail(DSX_ERR_STATE, "link probe: 2, 4 or 8 ranks");
  std::vector<float> ms;
  cudaEvent_t e0, e1;
  DSX_CUDA(cudaEventCreate(&e0));
  DSX_CUDA(cudaEventCreate(&e1));
  for (int r = 0; r < std::max(1, reps) + 1; ++r) {  // first launch warms up
    DSX_TRY(barrier());
    DSX_CUDA(cudaEventRecord(e0, lab->side));
    launch();
    DSX_CUDA(cudaEventRecord(e1, lab->side));
    DSX_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    DSX_CUDA(cudaEventElapsedTime(&t, e0, e1));
    if (r > 0) ms.push_back(t);
  }
  DSX_TRY(barrier());
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  std::sort(ms.begin(), ms.end());
  const double med = ms[ms.size() / 2];
  // ring convention: 2(W-1)/W x S per rank, S = W x slice bytes
  const double bus = 2.0 * (W - 1) * (double)per * 16.0;
  *gbs = bus / (med * 1e-3) / 1e9;
  return DSX_OK;
}

dsx_status dsx_lab_set_link(dsx_lab* lab, double bandwidth, double latency) {
  DSX_TRY(check_lab(lab));
  if (!(latency >= 0.0)) return fail(DSX_ERR_ARGUMENT, "latency must be >= 0");
  lab->link_bw = bandwidth > 0.0 ? bandwidth : 0.0;
  lab->link_lat = latency;
  return DSX_OK;
}

// CUDA-event layer profiler: per registered layer, the
// device time of its local step (gradient + update over the layer's tiles,
// eta = 0 and no noise so the state is untouched) and, on multiple ranks,
// of its cross-rank average (on a saved-and-restored arena).  Median of
// `reps` repetitions, seconds.  t_comm[l] < 0 means "not measured" (single
// rank without a throttled link: use the link model).
dsx_status dsx_lab_profile(dsx_lab* lab, int reps, double* t_bp, double* t_comm) {
  DSX_TRY(check_lab(lab));
  if (!t_bp || reps < 1) return fail(DSX_ERR_ARGUMENT, "bad profile args");
  DSX_TRY(materialize(lab));
  DSX_CUDA(cudaStreamSynchronize(lab->stream));
  DSX_CUDA(cudaStreamSynchronize(lab->side));
  if (lab->nstream) DSX_CUDA(cudaStreamSynchronize(lab->nstream));
  MaskBits none{};
  cudaEvent_t e0, e1;
  DSX_CUDA(cudaEventCreate(&e0));
  DSX_CUDA(cudaEventCreate(&e1));
  std::vector<float> ts(reps);
  // with an engine run available, the local step reads its noise like the
  // real step does (reading leaves every state untouched)
  const int pnoise = (lab->engine && lab->batch_set >= 0) ? 2 : 0;
  int tb = 0;
  for (int b = 0; b < lab->L; ++b) {
    int te = tb;
    while (te < lab->ntiles && lab->h_tiles[te].block == b) ++te;
    for (int r = 0; r < reps; ++r) {
      DSX_CUDA(cudaEventRecord(e0, lab->stream));
      if (lab->dtype == DSX_F64) launch_update<double>(lab, lab->stream, tb, te - tb, pnoise, false, none, 0.0);
      else launch_update<float>(lab, lab->stream, tb, te - tb, pnoise, false, none, 0.0);
      DSX_CUDA(cudaEventRecord(e1, lab->stream));
      DSX_CUDA(cudaEventSynchronize(e1));
      DSX_CUDA(cudaEventElapsedTime(&ts[r], e0, e1));
    }
    std::sort(ts.begin(), ts.end());
    t_bp[b] = ts[reps / 2] * 1e-3;
    tb = te;
  }
  // Layers alone carry one launch each; the real step updates every layer in
  // one fused pass (except the single-GPU throttled mode, which launches per
  // layer).  Rescale so the layers sum to the fused pass's time (relative
  // costs kept), i.e. the profile describes the step as it runs.
  if (!(lab->nranks == 1 && lab->link_bw > 0.0)) {
    for (int r = 0; r < reps; ++r) {
      DSX_CUDA(cudaEventRecord(e0, lab->stream));
      if (lab->dtype == DSX_F64) launch_update<double>(lab, lab->stream, 0, lab->ntiles, pnoise, false, none, 0.0);
      else launch_update<float>(lab, lab->stream, 0, lab->ntiles, pnoise, false, none, 0.0);
      DSX_CUDA(cudaEventRecord(e1, lab->stream));
      DSX_CUDA(cudaEventSynchronize(e1));
      DSX_CUDA(cudaEventElapsedTime(&ts[r], e0, e1));
    }
    std::sort(ts.begin(), ts.end());
    double alone = 0.0;
    for (int b = 0; b < lab->L; ++b) alone += t_bp[b];
    if (alone > 0.0) {
      const double scale = ts[reps / 2] * 1e-3 / alone;
      for (int b = 0; b < lab->L; ++b) t_bp[b] *= scale;
    }
  }
  if (t_comm) {
    std::vector<unsigned char> one(lab->L + 1, 0);
    for (int b = 0; b < lab->L; ++b) {
      t_comm[b] = -1.0;
      if (lab->link_bw > 0.0) {
        std::fill(one.begin(), one.end(), 0);
        one[b + 1] = 1;
        t_comm[b] = (double)link_ns(lab, one.data(), (long long)lab->offs[b],
                                    (long long)(lab->offs[b + 1] - lab->offs[b])) * 1e-9;
      }
    }
    if (lab->nranks > 1 && lab->p2p && lab->link_bw <= 0.0) {
      // measure the real NVLink average per layer on a backup of the arena
      const size_t es = elem_size(lab);
      void* backup = nullptr;
      const size_t bytes = es * (size_t)lab->ld * lab->kl;
      DSX_CUDA(cudaMalloc(&backup, bytes));
      DSX_CUDA(cudaMemcpyAsync(backup, lab->w, bytes, cudaMemcpyDeviceToDevice, lab->side));
      // the step's own barriers: peer-memory flags (or NCCL all-reduces)
      const bool fb = lab->flag_bar;
      auto bar_ready = [&]() -> dsx_status {
        if (fb) {
          flag_wait_kernel<<<1, 64, 0, lab->side>>>(lab->fpeers, lab->rank, lab->nranks, 0, ++lab->epoch, 1, lab->flag_timeout_ns);
        } else {
          DSX_NCCL(ncclAllReduce(lab->bar, lab->bar, 1, ncclInt32, ncclSum, lab->comm, lab->side));
        }
        return DSX_OK;
      };
      auto bar_landed = [&]() -> dsx_status {
        if (fb) {
          flag_wait_kernel<<<1, 64, 0, lab->side>>>(lab->fpeers, lab->rank, lab->nranks, kMaxProg, lab->sig_count, 0, lab->flag_timeout_ns);
        } else {
          DSX_NCCL(ncclAllReduce(lab->bar, lab->bar, 1, ncclInt32, ncclSum, lab->comm, lab->side));
        }
        return DSX_OK;
      };
      auto sig = [&]() { return fb ? Signal{lab->fpeers, lab->rank, lab->nranks, ++lab->sig_count, lab->sig_counter} : Signal{}; };
      for (int b = 0; b < lab->L; ++b) {
        const long long lo = (long long)lab->offs[b], n = (long long)(lab->offs[b + 1] - lab->offs[b]);
        for (int r = 0; r < reps; ++r) {
          DSX_TRY(bar_landed());
          DSX_CUDA(cudaEventRecord(e0, lab->side));
          DSX_TRY(bar_ready());
          const int R = lab->nranks;
          const long long base = n / R, extra = n % R;
          const long long a = lo + lab->rank * base + std::min<long long>(lab->rank, extra);
          const long long m = base + (lab->rank < extra ? 1 : 0);
          {
            const int blocks = (int)std::min<long long>(lab->nsm * 4, (std::max(m, 0LL) / 2 + 255) / 256 + 1);
            const long long e = a + std::max(m, 0LL);
            if (lab->dtype == DSX_F64)
              p2p_average_kernel<double, 0><<<blocks, 256, 0, lab->side>>>(lab->peers, a, e, lab->K, lab->prog_ranks, sig());
            else
              p2p_average_kernel<float, 0><<<blocks, 256, 0, lab->side>>>(lab->peers, a, e, lab->K, lab->prog_ranks, sig());
          }
          DSX_TRY(bar_landed());
          DSX_CUDA(cudaEventRecord(e1, lab->side));
          DSX_CUDA(cudaEventSynchronize(e1));
          DSX_CUDA(cudaEventElapsedTime(&ts[r], e0, e1));
        }
        std::sort(ts.begin(), ts.end());
        t_comm[b] = ts[reps / 2] * 1e-3;
      }
      // the step averages in `chunks` groups (two barriers each), not per
      // layer, and while the local step runs: rescale to the grouped
      // whole-model average timed under a concurrent fused update
      const std::vector<int> cuts = overlap_groups(lab, lab->overlap ? lab->chunks : 1);
      const int G = (int)cuts.size() - 1;
      for (int r = 0; r < reps; ++r) {
        DSX_TRY(bar_landed());
        DSX_CUDA(cudaStreamSynchronize(lab->side));
        if (lab->overlap) {
          if (lab->dtype == DSX_F64) launch_update<double>(lab, lab->stream, 0, lab->ntiles, pnoise, false, none, 0.0);
          else launch_update<float>(lab, lab->stream, 0, lab->ntiles, pnoise, false, none, 0.0);
        }
        DSX_CUDA(cudaEventRecord(e0, lab->side));
        for (int g = 0; g < G; ++g) {
          const int te = cuts[g], tb = cuts[g + 1];
          if (te <= tb) continue;
          const long long lo = lab->h_tiles[tb].start;
          const long long n = lab->h_tiles[te - 1].start + lab->h_tiles[te - 1].len - lo;
          const int R = lab->nranks;
          const long long base = n / R, extra = n % R;
          const long long a = lo + lab->rank * base + std::min<long long>(lab->rank, extra);
          const long long m = base + (lab->rank < extra ? 1 : 0);
          DSX_TRY(bar_ready());
          {
            const int blocks = (int)std::min<long long>(lab->nsm * 4, (std::max(m, 0LL) / 2 + 255) / 256 + 1);
            const long long e = a + std::max(m, 0LL);
            if (lab->dtype == DSX_F64)
              p2p_average_kernel<double, 0><<<blocks, 256, 0, lab->side>>>(lab->peers, a, e, lab->K, lab->prog_ranks, sig());
            else
              p2p_average_kernel<float, 0><<<blocks, 256, 0, lab->side>>>(lab->peers, a, e, lab->K, lab->prog_ranks, sig());
          }
        }
        DSX_TRY(bar_landed());
        DSX_CUDA(cudaEventRecord(e1, lab->side));
        DSX_CUDA(cudaEventSynchronize(e1));
        DSX_CUDA(cudaEventElapsedTime(&ts[r], e0, e1));
      }
      std::sort(ts.begin(), ts.end());
      double alone = 0.0;
      for (int b = 0; b < lab->L; ++b) alone += t_comm[b];
      if (alone > 0.0) {
        const double scale = ts[reps / 2] * 1e-3 / alone;
        for (int b = 0; b < lab->L; ++b) t_comm[b] *= scale;
      }
      DSX_CUDA(cudaStreamSynchronize(lab->stream));
      DSX_CUDA(cudaMemcpyAsync(lab->w, backup, bytes, cudaMemcpyDeviceToDevice, lab->side));
      DSX_CUDA(cudaStreamSynchronize(lab->side));
      cudaFree(backup);
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return DSX_OK;
}

dsx_status dsx_lab_set_pipeline(dsx_lab* lab, int enabled) {
  DSX_TRY(check_lab(lab));
  if (!enabled) DSX_TRY(invalidate_prefetch(lab));
  lab->pipeline = enabled != 0;
  return DSX_OK;
}

dsx_status dsx_lab_set_noise_horizon(dsx_lab* lab, long long steps) {
  DSX_TRY(check_lab(lab));
  if (steps >= 0) {
    DSX_CUDA(cudaStreamSynchronize(lab->stream));
    DSX_TRY(invalidate_prefetch(lab));
  }
  lab->horizon = steps < 0 ? -1 : steps;
  return DSX_OK;
}

dsx_status dsx_lab_set_overlap(dsx_lab* lab, int enabled) {
  DSX_TRY(check_lab(lab));
  lab->overlap = enabled != 0;
  return DSX_OK;
}

dsx_status dsx_lab_event_record(dsx_lab* lab, int slot) {
  DSX_TRY(check_lab(lab));
  if (slot < 0 || slot >= 32) return fail(DSX_ERR_ARGUMENT, "event slot out of range");
  DSX_CUDA(cudaEventRecord(lab->ev[slot], lab->stream));
  return DSX_OK;
}

dsx_status dsx_lab_event_elapsed(dsx_lab* lab, int a, int b, float* ms) {
  DSX_TRY(check_lab(lab));
  if (a < 0 || a >= 32 || b < 0 || b >= 32 || !ms) return fail(DSX_ERR_ARGUMENT, "bad event args");
  DSX_CUDA(cudaEventSynchronize(lab->ev[b]));
  DSX_CUDA(cudaEventElapsedTime(ms, lab->ev[a], lab->ev[b]));
  return DSX_OK;
}

dsx_status dsx_lab_set_instrument(dsx_lab* lab, int enabled) {
  DSX_TRY(check_lab(lab));
  lab->instrument = enabled != 0;
  return DSX_OK;
}

// Measured timeline of the last instrumented single-GPU throttled step: per
// layer l (0-based), bp[2l..2l+1] = start/end ms of its local step on the
// compute lane, comm[2l..2l+1] = start/end ms of its transfer on the link
// lane (-1 when not synced), relative to the step start.  The same events
// as simulate_run's timeline (simulator.cpp:145-157), measured.
dsx_status dsx_lab_last_timeline(dsx_lab* lab, float* bp, float* comm) {
  DSX_TRY(check_lab(lab));
  if (!bp || !comm) return fail(DSX_ERR_ARGUMENT, "null timeline out");
  if (!lab->instrument || (int)lab->tl_ev.size() < 4 * lab->L || (int)lab->tl_mask.size() != lab->L + 1)
    return fail(DSX_ERR_STATE, "no instrumented throttled step recorded");
  DSX_CUDA(cudaEventSynchronize(lab->iev[4]));
  for (int b = 0; b < lab->L; ++b) {
    DSX_CUDA(cudaEventElapsedTime(&bp[2 * b], lab->iev[0], lab->tl_ev[4 * b]));
    DSX_CUDA(cudaEventElapsedTime(&bp[2 * b + 1], lab->iev[0], lab->tl_ev[4 * b + 1]));
    comm[2 * b] = comm[2 * b + 1] = -1.0f;
    if (lab->tl_mask[b + 1]) {
      DSX_CUDA(cudaEventElapsedTime(&comm[2 * b], lab->iev[0], lab->tl_ev[4 * b + 2]));
      DSX_CUDA(cudaEventElapsedTime(&comm[2 * b + 1], lab->iev[0], lab->tl_ev[4 * b + 3]));
    }
  }
  return DSX_OK;
}

dsx_status dsx_lab_engine_time(dsx_lab* lab, int steps, int reps, float* ms, int* batch_out) {
  DSX_TRY(check_lab(lab));
  if (!ms || reps < 1) return fail(DSX_ERR_ARGUMENT, "bad engine_time args");
  if (batch_out) *batch_out = lab->tmax;
  *ms = 0.0f;
  if (!lab->engine) return DSX_OK;
  if (steps != 1 && steps != lab->tmax) return fail(DSX_ERR_ARGUMENT, "steps must be 1 or the batch length");
  DSX_CUDA(cudaStreamSynchronize(lab->stream));
  DSX_TRY(invalidate_prefetch(lab));
  // run into the set that does not hold the committed state; it is dropped
  const int commit_set = lab->mt_commit == 0 ? -1 : (lab->mt_commit - 1) / lab->tmax;
  const int set = commit_set == 0 ? 1 : 0;
  cudaEvent_t e0, e1;
  DSX_CUDA(cudaEventCreate(&e0));
  DSX_CUDA(cudaEventCreate(&e1));
  std::vector<float> ts(reps);
  for (int r = 0; r < reps; ++r) {
    DSX_CUDA(cudaEventRecord(e0, lab->nstream));
    DSX_TRY(launch_engine(lab, set, steps, lab->mt_commit));
    DSX_CUDA(cudaEventRecord(e1, lab->nstream));
    DSX_CUDA(cudaEventSynchronize(e1));
    DSX_CUDA(cudaEventElapsedTime(&ts[r], e0, e1));
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  std::sort(ts.begin(), ts.end());
  *ms = ts[reps / 2];
  return invalidate_prefetch(lab);
}

dsx_status dsx_lab_last_step_times(dsx_lab* lab, float* out3) {
  DSX_TRY(check_lab(lab));
  if (!out3) return fail(DSX_ERR_ARGUMENT, "null out");
  if (!lab->instrument) return fail(DSX_ERR_STATE, "instrumentation disabled");
  DSX_CUDA(cudaEventSynchronize(lab->iev[4]));
  DSX_CUDA(cudaEventElapsedTime(&out3[0], lab->iev[0], lab->iev[4]));
  DSX_CUDA(cudaEventElapsedTime(&out3[3], lab->iev[0], lab->iev[5]));
  // update span: from update start to the local step's end (single rank:
  // the fused update kernel + norm finalize)
  DSX_CUDA(cudaEventElapsedTime(&out3[4], lab->iev[5], lab->synced_last ? lab->iev[3] : lab->iev[4]));
  out3[1] = out3[2] = 0.0f;
  if (lab->synced_last) {
    // sync = side-stream span; exposed = how long the synced blocks finished
    // after the local step did (cost_model.cpp:39: term - bp_total).
    float sync_start = 0.0f, sync_end = 0.0f, local_end = 0.0f;
    DSX_CUDA(cudaEventElapsedTime(&sync_start, lab->iev[0], lab->iev[1]));
    DSX_CUDA(cudaEventElapsedTime(&sync_end, lab->iev[0], lab->iev[2]));
    DSX_CUDA(cudaEventElapsedTime(&local_end, lab->iev[0], lab->iev[3]));
    out3[1] = sync_end - sync_start;
    out3[2] = std::max(0.0f, sync_end - local_end);
  }
  return DSX_OK;
}

// Host-only: can `nranks` equal contiguous worker ranges reproduce the
// reference's pairwise summation order (each range a subtree)?
dsx_status dsx_sync_plan(int workers_total, int nranks, int* pairwise_exact) {
  if (!pairwise_exact || workers_total < 1 || nranks < 1) return fail(DSX_ERR_ARGUMENT, "bad plan args");
  if (workers_total % nranks) {
    *pairwise_exact = 0;
    return DSX_OK;
  }
  const int kl = workers_total / nranks;
  int ok = 1;
  for (int r = 0; r < nranks; ++r) ok &= is_subtree(workers_total, r * kl, kl) ? 1 : 0;
  *pairwise_exact = ok;
  return DSX_OK;
}

// Host-only check of the MT19937-64 jump-ahead: the window at stream
// offset 1+J computed by the characteristic-polynomial jump equals the one
// produced by running the recurrence.  Needs no GPU.
dsx_status dsx_mt_jump_selftest(unsigned long long jump, int* ok) {
  if (!ok) return fail(DSX_ERR_ARGUMENT, "null ok");
  if (jump > 50'000'000ull) return fail(DSX_ERR_ARGUMENT, "jump too large for the direct check");
  std::mt19937_64 eng(12345u);
  for (int i = 0; i < 1000; ++i) eng();
  std::stringstream ss;
  ss << eng;
  uint64_t x[kMtN];
  for (int i = 0; i < kMtN; ++i) ss >> x[i];
  if (dsx::mt_char_poly().empty()) return fail(DSX_ERR_STATE, "characteristic polynomial unavailable");
  const std::vector<uint64_t> jumped = dsx::mt_jump_host(x, dsx::mt_jump_poly(jump));
  std::vector<uint64_t> y(x, x + kMtN);
  y.reserve(jump + 2 * kMtN + 2);
  while (y.size() < jump + 1 + kMtN) {
    const size_t k = y.size() - kMtN;
    y.push_back(mt_next_word(y[k], y[k + 1], y[k + kMtM]));
  }
  *ok = 1;
  for (int j = 0; j < kMtN; ++j) *ok &= jumped[j] == y[1 + jump + j];
  return DSX_OK;
}

dsx_status dsx_lab_launch_count(dsx_lab* lab, uint64_t* out) {
  if (!lab || !out) return fail(DSX_ERR_ARGUMENT, "null argument");
  *out = lab->launches;
  return DSX_OK;
}

}  // extern "C"
