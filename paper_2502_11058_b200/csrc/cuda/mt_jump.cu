// mt_jump.cu — the parallel, stream-exact noise engine (see noise_engine.cuh).
//
// Host: the MT19937-64 characteristic polynomial (Berlekamp-Massey over
// GF(2)) and jump polynomials c_s = x^(s*S - 1) mod phi.
// Device: prefix -> jump -> segment -> finish kernels, one CUDA stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <random>
#include <sstream>

#include "device_once.cuh"
#include "mt_engine.cuh"
#include "noise_engine.cuh"

#if defined(__x86_64__)
#include <wmmintrin.h>
#endif

namespace dsx {

namespace {

constexpr int kDeg = 19937;               // deg phi
constexpr int kPolyWords = 312;            // ceil(19938 / 64)
constexpr int kPrefixWords = 66 * kMtN;    // Y[0 .. 20592): >= 1 + 19968 + 311 + 16 (jump2 reads)
constexpr int kJumpBits = 19952;           // c padded to a multiple of 16
constexpr int kCkWords = kMtN + 4;         // x[312], carry flag, carry bits, local count, pad
constexpr int kThreads = 320;

using Poly = std::vector<uint64_t>;

// ---- host GF(2) polynomial arithmetic -----------------------------------

void xor_shifted(uint64_t* dst, size_t dst_words, const uint64_t* src, size_t src_words, size_t shift) {
  const size_t ws = shift / 64, bs = shift % 64;
  for (size_t i = 0; i < src_words; ++i) {
    const uint64_t v = src[i];
    if (!v) continue;
    if (i + ws < dst_words) dst[i + ws] ^= v << bs;
    if (bs && i + ws + 1 < dst_words) dst[i + ws + 1] ^= v >> (64 - bs);
  }
}

bool get_bit(const uint64_t* p, size_t i) { return (p[i / 64] >> (i % 64)) & 1u; }

// reduce r (any length, degree < 64*len) modulo phi in place; result in the
// low kPolyWords words.
void reduce(Poly& r, const Poly& phi) {
  // byte table of v(x) * phi(x), v in [0, 256)
  static std::vector<Poly> table;
  static std::once_flag once;
  std::call_once(once, [&] {
    table.assign(256, Poly(kPolyWords + 1, 0));
    for (int v = 1; v < 256; ++v)
      for (int b = 0; b < 8; ++b)
        if ((v >> b) & 1) xor_shifted(table[v].data(), kPolyWords + 1, phi.data(), kPolyWords, b);
  });
  const long top = (long)r.size() * 64 - 1;
  long t = top;
  for (; t - 7 >= kDeg; t -= 8) {
    // byte of r at bits [t-7, t]
    const size_t lo = (size_t)(t - 7);
    uint64_t v = r[lo / 64] >> (lo % 64);
    if (lo % 64 > 56 && lo / 64 + 1 < r.size()) v |= r[lo / 64 + 1] << (64 - lo % 64);
    v &= 0xff;
    if (v) xor_shifted(r.data(), r.size(), table[v].data(), kPolyWords + 1, lo - kDeg);
  }
  for (; t >= kDeg; --t)
    if (get_bit(r.data(), (size_t)t)) xor_shifted(r.data(), r.size(), phi.data(), kPolyWords, (size_t)t - kDeg);
  r.resize(kPolyWords);
}

#if defined(__x86_64__)
__attribute__((target("pclmul,sse2"))) void clmul_words(const uint64_t* a, const uint64_t* b, uint64_t* out,
                                                        size_t n) {
  for (size_t i = 0; i < n; ++i) {
    if (!a[i]) continue;
    const __m128i av = _mm_set_epi64x(0, (long long)a[i]);
    for (size_t j = 0; j < n; ++j) {
      const __m128i bv = _mm_set_epi64x(0, (long long)b[j]);
      const __m128i p = _mm_clmulepi64_si128(av, bv, 0x00);
      out[i + j] ^= (uint64_t)_mm_cvtsi128_si64(p);
      out[i + j + 1] ^= (uint64_t)_mm_cvtsi128_si64(_mm_unpackhi_epi64(p, p));
    }
  }
}
#endif

void clmul_portable(const uint64_t* a, const uint64_t* b, uint64_t* out, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    for (int bit = 0; bit < 64; ++bit) {
      if (!((a[i] >> bit) & 1)) continue;
      xor_shifted(out + i, 2 * n - i, b, n, (size_t)bit);
    }
  }
}

Poly mulmod(const Poly& a, const Poly& b, const Poly& phi) {
  Poly prod(2 * kPolyWords + 1, 0);
#if defined(__x86_64__)
  if (__builtin_cpu_supports("pclmul")) {
    clmul_words(a.data(), b.data(), prod.data(), kPolyWords);
  } else {
    clmul_portable(a.data(), b.data(), prod.data(), kPolyWords);
  }
#else
  clmul_portable(a.data(), b.data(), prod.data(), kPolyWords);
#endif
  reduce(prod, phi);
  return prod;
}

Poly sqrmod(const Poly& a, const Poly& phi) {
  Poly sq(2 * kPolyWords + 1, 0);
  for (size_t i = 0; i < kPolyWords; ++i) {
    uint64_t v = a[i];
    uint64_t lo = 0, hi = 0;
    for (int b = 0; b < 32; ++b) {
      lo |= ((v >> b) & 1ull) << (2 * b);
      hi |= ((v >> (b + 32)) & 1ull) << (2 * b);
    }
    sq[2 * i] = lo;
    sq[2 * i + 1] = hi;
  }
  reduce(sq, phi);
  return sq;
}

Poly x_pow(unsigned long long J, const Poly& phi) {
  Poly r(kPolyWords, 0);
  r[0] = 1;
  for (int bit = 63; bit >= 0; --bit) {
    r = sqrmod(r, phi);
    if ((J >> bit) & 1ull) {  // r *= x
      Poly t(kPolyWords + 1, 0);
      xor_shifted(t.data(), t.size(), r.data(), kPolyWords, 1);
      reduce(t, phi);
      r = t;
    }
  }
  return r;
}

// Y[0..n) from a generation-aligned 312-word array.
void host_sequence(const uint64_t* x, size_t n, std::vector<uint64_t>& y) {
  y.assign(x, x + kMtN);
  y.reserve(n);
  while (y.size() < n) {
    const size_t k = y.size() - kMtN;
    y.push_back(mt_next_word(y[k], y[k + 1], y[k + kMtM]));
  }
}

Poly compute_char_poly() {
  // Bit 0 of Y[1..] of an arbitrary stream; its minimal polynomial is phi.
  std::mt19937_64 eng(5489u);
  std::stringstream ss;
  ss << eng;
  uint64_t x[kMtN];
  for (int i = 0; i < kMtN; ++i) ss >> x[i];
  const size_t N = 2 * kDeg + 256;
  std::vector<uint64_t> y;
  host_sequence(x, N + 2, y);
  // reversed bit sequence: rev[k] = s_{N-1-k}, s_n = Y[1+n] & 1
  const size_t RW = (N + 63) / 64 + 2;
  std::vector<uint64_t> rev(RW, 0);
  for (size_t n = 0; n < N; ++n)
    if (y[1 + n] & 1) {
      const size_t k = N - 1 - n;
      rev[k / 64] |= 1ull << (k % 64);
    }
  const size_t CW = (N + 63) / 64 + 2;
  std::vector<uint64_t> C(CW, 0), B(CW, 0), T;
  C[0] = B[0] = 1;
  size_t L = 0, m = 1;
  for (size_t n = 0; n < N; ++n) {
    // d = sum_{i=0..L} C_i s_{n-i} = sum_i C_i rev[N-1-n+i]
    const size_t off = N - 1 - n;
    uint64_t acc = 0;
    const size_t words = L / 64 + 1;
    for (size_t w = 0; w < words; ++w) {
      const size_t bit = off + 64 * w;
      uint64_t r = rev[bit / 64] >> (bit % 64);
      if (bit % 64 && bit / 64 + 1 < RW) r |= rev[bit / 64 + 1] << (64 - bit % 64);
      uint64_t c = C[w];
      if (w == words - 1 && (L % 64) != 63) c &= (2ull << (L % 64)) - 1;
      acc ^= c & r;
    }
    const bool d = __builtin_popcountll(acc) & 1;
    if (!d) {
      ++m;
    } else if (2 * L <= n) {
      T = C;
      xor_shifted(C.data(), CW, B.data(), CW, m);
      L = n + 1 - L;
      B = T;
      m = 1;
    } else {
      xor_shifted(C.data(), CW, B.data(), CW, m);
      ++m;
    }
  }
  Poly phi(kPolyWords, 0);
  if (L != (size_t)kDeg) return Poly();  // signals failure
  // phi_k = C_{L-k}
  for (size_t k = 0; k <= L; ++k)
    if (get_bit(C.data(), L - k)) phi[k / 64] |= 1ull << (k % 64);
  return phi;
}

}  // namespace

const std::vector<uint64_t>& mt_char_poly() {
  static Poly phi;
  static std::once_flag once;
  std::call_once(once, [] { phi = compute_char_poly(); });
  return phi;
}

std::vector<uint64_t> mt_jump_poly(unsigned long long J) { return x_pow(J, mt_char_poly()); }

std::vector<uint64_t> mt_jump_host(const uint64_t* x312, const std::vector<uint64_t>& c) {
  std::vector<uint64_t> y;
  host_sequence(x312, kPrefixWords, y);
  std::vector<uint64_t> out(kMtN, 0);
  for (int i = 0; i < kDeg; ++i)
    if (get_bit(c.data(), (size_t)i))
      for (int j = 0; j < kMtN; ++j) out[j] ^= y[1 + i + j];
  return out;
}

// ---- device ----------------------------------------------------------------

namespace {

struct Smem {
  uint64_t x[kMtN];
  double v[kMtN + 2];
  int wcnt[kThreads / 32];
  int misc[4];
};

__device__ __forceinline__ void block_twist(uint64_t* x) {
  const int tid = threadIdx.x;
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
}

// One generation's outputs [lo, hi) with a carried half pair: fills v,
// evaluates this thread's attempt (tid < npairs), returns the CTA total and
// the thread's rank among accepted attempts.  Updates the carry.
struct PairEval {
  bool acc;
  int rank;
  int total;
  int npairs;
  double px, py, r2;
};

__device__ __forceinline__ PairEval eval_generation(Smem& sm, int lo, int hi, int& have_half,
                                                    double& half) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid >= lo && tid < hi) sm.v[have_half + tid - lo] = mt_polar_coord(mt_temper(sm.x[tid]));
  if (tid == 0 && have_half) sm.v[0] = half;
  __syncthreads();
  const int nvals = have_half + (hi - lo);
  PairEval e;
  e.npairs = nvals >> 1;
  e.acc = false;
  e.px = e.py = e.r2 = 0.0;
  if (tid < e.npairs) {
    e.px = sm.v[2 * tid];
    e.py = sm.v[2 * tid + 1];
    e.acc = mt_polar_accept(e.px, e.py, &e.r2);
  }
  const unsigned bal = __ballot_sync(0xffffffffu, e.acc);
  if (lane == 0) sm.wcnt[warp] = __popc(bal);
  __syncthreads();
  int before = __popc(bal & ((1u << lane) - 1u));
  int total = 0;
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w) {
    if (w < warp) before += sm.wcnt[w];
    total += sm.wcnt[w];
  }
  e.rank = before;
  e.total = total;
  if (nvals & 1) {
    half = sm.v[nvals - 1];
    have_half = 1;
  } else {
    have_half = 0;
  }
  __syncthreads();  // v / wcnt reusable
  return e;
}

// dst = the generation after src (separate buffers, 2 barriers).  Phase A
// (k < 156) reads only src; phase B (k >= 156) also reads the new dst[k-156]
// and, for k = 311, dst[0] — exactly _M_gen_rand's in-place order.
__device__ __forceinline__ void twist_into(const uint64_t* src, uint64_t* dst) {
  const int tid = threadIdx.x;
  if (tid < kMtM) dst[tid] = mt_next_word(src[tid], src[tid + 1], src[tid + kMtM]);
  __syncthreads();
  if (tid < kMtM) {
    const int k = kMtM + tid;
    dst[k] = mt_next_word(src[k], (k + 1 < kMtN) ? src[k + 1] : dst[0], dst[tid]);
  }
  __syncthreads();
}

constexpr int kRound = 4;  // generations per segment-kernel round

// Normalizes the cursor (p == 312 -> twist) and writes Y[0..kPrefixWords).
__global__ void __launch_bounds__(kThreads)
mt_prefix_kernel(const uint64_t* mt, uint64_t* ybuf, uint64_t* win, int P, int* pnorm) {
  __shared__ uint64_t x[kMtN];
  const int w = blockIdx.x, tid = threadIdx.x;
  const uint64_t* st = mt + (long long)w * (kMtN + 1);
  if (tid < kMtN) x[tid] = st[tid];
  int p = (int)st[kMtN];
  __syncthreads();
  if (p >= kMtN) {
    block_twist(x);
    p = 0;
  }
  uint64_t* y = ybuf + (long long)w * kPrefixWords;
  for (int g = 0; g < kPrefixWords / kMtN; ++g) {
    if (g) block_twist(x);
    if (tid < kMtN) {
      y[g * kMtN + tid] = x[tid];
      if (g == 0) win[(long long)w * P * kMtN + tid] = x[tid];
    }
  }
  if (tid == 0) pnorm[w] = p;
}

// Jump kernel v2 (the default).  The polynomial c_s is split into kJ2Parts
// bit ranges, one warp each; a warp covers all 312 window words (lane l owns
// words 11l .. 11l+10, an odd stride so the 64-bit shared loads are
// conflict-free), so each set bit costs 11 XOR64 per lane against one
// shared load per bit for the sliding window — 2.4x fewer instructions per
// jump than one warp per quarter window.  The parts' partial windows are
// XOR-reduced through shared memory.  kJ2PerCta jumps of one worker share
// the CTA's copy of the stream prefix.
constexpr int kJ2PerCta = 2;
constexpr int kJ2A = 11;                              // words per lane
constexpr int kJ2Q = 16;                              // ring (= kJ2A + 5 prefetch)
constexpr int kJ2Lanes = (kMtN + kJ2A - 1) / kJ2A;    // 29
constexpr int kJ2Span = 19968;                        // bits over all parts (c padded)
static_assert(kJ2Span >= kDeg && kJ2Span <= 32 * (kJumpBits / 32 + 1), "parts");
static_assert(1 + kJ2Span + kJ2Lanes * kJ2A + kJ2Q <= kPrefixWords + kJ2A, "prefix");

template <int kJ2Parts>
__global__ void __launch_bounds__(kJ2PerCta * kJ2Parts * 32)
mt_jump2_kernel(const uint64_t* ybuf, const uint32_t* cbits, uint64_t* win, int P) {
  constexpr int kJ2Bits = kJ2Span / kJ2Parts;  // bits per part, a multiple of 16
  static_assert(kJ2Bits % 32 == 0 || kJ2Bits % 16 == 0, "16-bit words");
  extern __shared__ uint64_t ys[];                    // [kPrefixWords] then partials
  uint64_t* part = ys + kPrefixWords;                 // [kJ2PerCta][kJ2Parts][kMtN]
  const int w = blockIdx.y;
  const uint64_t* y = ybuf + (long long)w * kPrefixWords;
  for (int i = threadIdx.x; i < kPrefixWords; i += blockDim.x) ys[i] = y[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int jl = warp / kJ2Parts, pt = warp % kJ2Parts;
  const int s = 1 + blockIdx.x * kJ2PerCta + jl;
  constexpr int kCW = kJumpBits / 32 + 1;
  uint64_t acc[kJ2A];
#pragma unroll
  for (int q = 0; q < kJ2A; ++q) acc[q] = 0;
  if (s < P) {
    const uint32_t* c = cbits + (long long)(s - 1) * kCW;
    const int i_begin = pt * kJ2Bits;
    const int j0 = lane < kJ2Lanes ? kJ2A * lane : 0;
    // lanes past the window read (harmless) words near the start; their
    // accumulators are never stored.  Reads stay inside the prefix: the
    // last part's bits beyond deg(phi) are zero but the ring still loads.
    const uint64_t* yb = ys + 1 + j0 + i_begin;
    uint64_t ring[kJ2Q];
#pragma unroll
    for (int q = 0; q < kJ2Q; ++q) ring[q] = yb[q];
    for (int i0 = 0; i0 < kJ2Bits; i0 += kJ2Q) {
      const uint32_t cw = c[(i_begin + i0) >> 5] >> ((i_begin + i0) & 31);  // 16 bits
#pragma unroll
      for (int u = 0; u < kJ2Q; ++u) {
        if ((cw >> u) & 1u) {
#pragma unroll
          for (int q = 0; q < kJ2A; ++q) acc[q] ^= ring[(u + q) % kJ2Q];
        }
        const int nxt = i0 + u + kJ2Q;
        ring[u] = nxt < kJ2Bits + kJ2Q ? yb[nxt] : 0;
      }
    }
  }
  uint64_t* mine = part + ((long long)jl * kJ2Parts + pt) * kMtN;
  if (lane < kJ2Lanes) {
#pragma unroll
    for (int q = 0; q < kJ2A; ++q)
      if (kJ2A * lane + q < kMtN) mine[kJ2A * lane + q] = acc[q];
  }
  __syncthreads();
  // XOR the parts: the CTA's threads cover both jumps' 312 words
  for (int t = threadIdx.x; t < kJ2PerCta * kMtN; t += blockDim.x) {
    const int j = t / kMtN, m = t % kMtN;
    const int sj = 1 + blockIdx.x * kJ2PerCta + j;
    if (sj >= P) continue;
    uint64_t v = 0;
#pragma unroll
    for (int q = 0; q < kJ2Parts; ++q) v ^= part[((long long)j * kJ2Parts + q) * kMtN + m];
    win[((long long)w * P + sj) * kMtN + m] = v;
  }
}

__device__ __forceinline__ void store_ck(uint64_t* ck, const uint64_t* x, int have_half, double half,
                                         unsigned long long local) {
  const int tid = threadIdx.x;
  if (tid < kMtN) ck[tid] = x[tid];
  if (tid == 0) {
    ck[kMtN] = (uint64_t)have_half;
    ck[kMtN + 1] = (uint64_t)__double_as_longlong(half);
    ck[kMtN + 2] = local;
  }
}

// Warp-specialized segment kernel helpers.  Warp 0 is the twister: it
// produces the generation arrays into a double-buffered ring (R arrays per
// half) with warp-level sync only, one round ahead; warps 1..10 consume a
// round at a time (temper, polar accept, scan, compaction, fp64 transform)
// and never wait on twist barriers.  Producer/consumer hand-off uses named
// barriers: FULL_h (producer arrives once half h is written), EMPTY_h
// (consumers arrive once they stopped reading half h).  Consumer-only sync
// uses named barrier kBarCons over the 320 consumer threads.
constexpr int kWsR = 4;                       // generations per round
constexpr int kWsThreads = 32 + kThreads;     // producer warp + 320 consumers
constexpr int kBarFull = 1, kBarEmpty = 3, kBarCons = 5;

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// dst = next generation of src, by one warp (phase A then phase B).
__device__ __forceinline__ void warp_twist(const uint64_t* src, uint64_t* dst, int lane) {
  for (int k = lane; k < kMtM; k += 32) dst[k] = mt_next_word(src[k], src[k + 1], src[k + kMtM]);
  __syncwarp();
  for (int k = kMtM + lane; k < kMtN; k += 32)
    dst[k] = mt_next_word(src[k], (k + 1 < kMtN) ? src[k + 1] : dst[0], dst[k - kMtM]);
  __syncwarp();
}

// Segment kernel v5 (the default; earlier single-twister and block-synchronous
// versions were measured slower and removed), rebalanced after ncu showed
// consumers stalled on the single twister warp
// (~12 % of samples) and on the uneven per-round transform split (~8 %):
//  * kProdWarps twister warps split every generation's two phases (a 64-
//    thread named barrier between phases) — half the producer latency;
//  * interior rounds read the pair coordinates straight from the ring (the
//    ring half is R*312 contiguous words, so output n of the round is word
//    n), no staging array and no barrier between temper and accept;
//  * every consumer warp scans the 20 per-warp accepted counts itself (one
//    barrier instead of scan + two barriers);
//  * accepted pairs go to a shared FIFO and are transformed in full chunks
//    of 320 (or 640 with 2-way ILP), the remainder carried to the next round,
//    so no warp idles at the end of a round with a half-empty transform.
constexpr int kProdWarps = 4;
constexpr int kProdThreads = 32 * kProdWarps;
constexpr int kWs2Threads = kProdThreads + kThreads;
constexpr int kBarProd = 6;
constexpr int kQCap = 1024;  // FIFO capacity: < 320 carried + 624 new per round

// RAW (opt-in): the accepted attempts (x, y) are stored as they are and
// the consumer applies the polar transform (mt_polar_normals) — the update
// kernel has idle issue slots while it waits on HBM, the engine does not.
// Shared memory of the v5 segment kernel with R generations per round.
template <int R>
struct Ws2Smem {
  static constexpr int kQ = (kThreads + R * kMtN / 2) <= 1024 ? 1024 : 2048;  // FIFO entries
  static constexpr size_t kRing = sizeof(uint64_t) * 2 * R * kMtN;
  static constexpr size_t kV = sizeof(double) * (R * kMtN + 2);
  static constexpr size_t kBytes = kRing + kV + sizeof(double2) * kQ;
};

template <bool RAW, int R>
__global__ void __launch_bounds__(kWs2Threads, 2)
mt_segment_ws2_kernel(const uint64_t* win_state, const uint64_t* win, const int* pnorm_in,
                      int* pnorm_out, int P, int gens, int ck_every, int nck, double stddev,
                      double* slots, long long cap, unsigned long long* cnt, uint64_t* ck,
                      uint64_t* tail) {
  constexpr int kPairSlots = (R * kMtN / 2 + kThreads - 1) / kThreads;  // pairs per consumer per round
  constexpr int kCounts = kPairSlots * (kThreads / 32);
  constexpr int kQCap = Ws2Smem<R>::kQ;
  static_assert(kCounts <= 32, "scan fits one warp");
  static_assert(kThreads + R * kMtN / 2 <= kQCap, "FIFO holds the carry plus one round");
  extern __shared__ __align__(16) unsigned char ws2_dsm[];
  // ring[2][R*312] | v[R*312+2] (boundary rounds + boot) | fifo[kQCap]
  auto ring_half = [&](int h) { return reinterpret_cast<uint64_t*>(ws2_dsm) + (long long)h * R * kMtN; };
  double* v = reinterpret_cast<double*>(ws2_dsm + Ws2Smem<R>::kRing);
  double2* fifo = reinterpret_cast<double2*>(ws2_dsm + Ws2Smem<R>::kRing + Ws2Smem<R>::kV);
  __shared__ int wcnt[2][kCounts];
  __shared__ double s_half[2];
  __shared__ int s_p;
  const int s = blockIdx.x, w = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* boot = reinterpret_cast<uint64_t*>(v);

  if (warp < kProdWarps) {
    // ---------------- producers: generations into the ring ----------------
    const int pt = threadIdx.x;
    int p;
    if (s == 0) {
      const uint64_t* st = win_state + (long long)w * (kMtN + 1);
      for (int k = pt; k < kMtN; k += kProdThreads) boot[k] = st[k];
      p = (int)st[kMtN];
      named_sync(kBarProd, kProdThreads);
      if (p >= kMtN) {
        for (int k = pt; k < kMtM; k += kProdThreads) ring_half(0)[k] = mt_next_word(boot[k], boot[k + 1], boot[k + kMtM]);
        named_sync(kBarProd, kProdThreads);
        for (int k = kMtM + pt; k < kMtN; k += kProdThreads)
          ring_half(0)[k] = mt_next_word(boot[k], (k + 1 < kMtN) ? boot[k + 1] : ring_half(0)[0], ring_half(0)[k - kMtM]);
        p = 0;
      } else {
        for (int k = pt; k < kMtN; k += kProdThreads) ring_half(0)[k] = boot[k];
      }
      if (pt == 0) pnorm_out[w] = p;
    } else {
      for (int k = pt; k < kMtN; k += kProdThreads) ring_half(0)[k] = win[((long long)w * P + s) * kMtN + k];
      p = pnorm_in[w];
    }
    if (pt == 0) s_p = p;
    named_sync(kBarProd, kProdThreads);
    const int ngen = gens + (p > 0 ? 1 : 0);
    const int rounds = (ngen + R - 1) / R;
    for (int k = 0; k < rounds; ++k) {
      const int h = k & 1;
      if (k >= 2) named_sync(kBarEmpty + h, kWs2Threads);  // consumers done with round k-2
      const int rg = min(R, ngen - k * R);
      for (int g = 0; g < rg; ++g) {
        if (k == 0 && g == 0) continue;  // gen 0 already in place
        const uint64_t* src = g ? ring_half(h) + (g - 1) * kMtN : ring_half(1 - h) + (R - 1) * kMtN;
        uint64_t* dst = ring_half(h) + g * kMtN;
        for (int i = pt; i < kMtM; i += kProdThreads) dst[i] = mt_next_word(src[i], src[i + 1], src[i + kMtM]);
        named_sync(kBarProd, kProdThreads);
        for (int i = kMtM + pt; i < kMtN; i += kProdThreads)
          dst[i] = mt_next_word(src[i], (i + 1 < kMtN) ? src[i + 1] : dst[0], dst[i - kMtM]);
        named_sync(kBarProd, kProdThreads);
      }
      __threadfence_block();
      named_arrive(kBarFull + h, kWs2Threads);
    }
    return;
  }

  // ---------------- consumers (320 threads) ----------------
  const int tid = threadIdx.x - kProdThreads, cw = tid >> 5;
  if (tid == 0) s_half[0] = 0.0;
  named_sync(kBarFull + 0, kWs2Threads);  // round 0 ready (also publishes s_p)
  const int p = s_p;
  const int ngen = gens + (p > 0 ? 1 : 0);
  const int rounds = (ngen + R - 1) / R;
  double* out = slots + ((long long)w * (P + 1) + s) * cap;
  uint64_t* ckw = ck + ((long long)w * P + s) * (long long)nck * kCkWords;
  int hh = 0;                      // a carried half pair enters this round
  unsigned long long local = 0;    // accepted pairs pushed to the FIFO
  unsigned long long head = 0;     // accepted pairs transformed and stored
  int ck_next = 0, ck_idx = 0;     // next checkpoint generation / its index
  auto transform = [&](unsigned long long g) {
    const double2 xy = fifo[g % kQCap];
    double r2;
    mt_polar_accept(xy.x, xy.y, &r2);
    const double m = mt_polar_mult(r2);
    double2 o;
    o.x = mt_scale(xy.y, m, stddev);
    o.y = mt_scale(xy.x, m, stddev);
    *reinterpret_cast<double2*>(out + 2 * g) = o;
  };
  for (int k = 0; k < rounds; ++k) {
    const int h = k & 1;
    const int q = k * R;
    if (k) named_sync(kBarFull + h, kWs2Threads);
    const int rg = min(R, ngen - q);
    const double half_in = s_half[h];
    if (q == ck_next) {  // every ck_every generations (no integer division)
      uint64_t* c = ckw + (long long)ck_idx * kCkWords;
      ck_next += ck_every;
      ++ck_idx;
      if (tid < kMtN) c[tid] = ring_half(h)[tid];
      if (tid == 0) {
        c[kMtN] = (uint64_t)hh;
        c[kMtN + 1] = (uint64_t)__double_as_longlong(half_in);
        c[kMtN + 2] = local;
      }
    }
    if (k == rounds - 1) {  // end state for an overflow continuation
      uint64_t* c = tail + ((long long)w * P + s) * kCkWords;
      if (tid < kMtN) c[tid] = ring_half(h)[(rg - 1) * kMtN + tid];
    }
    bool acc[kPairSlots];
    double px[kPairSlots], py[kPairSlots];
    int npairs, hh_next;
    if (q > 0 && q + R <= gens) {
      // interior: R complete generations; round output n is ring word n
      const uint64_t* rw = ring_half(h);
      npairs = (hh + R * kMtN) >> 1;
      hh_next = (hh + R * kMtN) & 1;
#pragma unroll
      for (int u = 0; u < kPairSlots; ++u) {
        const int a = tid + u * kThreads;
        acc[u] = false;
        px[u] = py[u] = 0.0;
        if (a < npairs) {
          const int n0 = 2 * a - hh;
          px[u] = n0 < 0 ? half_in : mt_polar_coord(mt_temper(rw[n0]));
          py[u] = mt_polar_coord(mt_temper(rw[n0 + 1]));
          double r2;
          acc[u] = mt_polar_accept(px[u], py[u], &r2);
        }
      }
      if (hh_next && tid == kThreads - 1) s_half[1 - h] = mt_polar_coord(mt_temper(rw[R * kMtN - 1]));
      named_arrive(kBarEmpty + h, kWs2Threads);  // done reading ring half h
    } else {
      // boundary round (the segment's first / last): partial generations
      int nvals = hh;
#pragma unroll
      for (int g = 0; g < R; ++g) {
        if (g < rg) {
          const int gen = q + g;
          const int lo = gen == 0 ? p : 0;
          const int hi = (gen == gens) ? p : kMtN;
          if (tid >= lo && tid < hi) v[nvals + tid - lo] = mt_polar_coord(mt_temper(ring_half(h)[g * kMtN + tid]));
          nvals += hi - lo;
        }
      }
      if (tid == 0 && hh) v[0] = half_in;
      named_arrive(kBarEmpty + h, kWs2Threads);
      named_sync(kBarCons, kThreads);  // v complete
      npairs = nvals >> 1;
      hh_next = nvals & 1;
#pragma unroll
      for (int u = 0; u < kPairSlots; ++u) {
        const int a = tid + u * kThreads;
        acc[u] = false;
        px[u] = py[u] = 0.0;
        if (a < npairs) {
          px[u] = v[2 * a];
          py[u] = v[2 * a + 1];
          double r2;
          acc[u] = mt_polar_accept(px[u], py[u], &r2);
        }
      }
      if (hh_next && tid == 0) s_half[1 - h] = v[nvals - 1];
    }
    // accepted counts per (slot, warp), slot-major = pair order
    int before[kPairSlots];
#pragma unroll
    for (int u = 0; u < kPairSlots; ++u) {
      const unsigned bal = __ballot_sync(0xffffffffu, acc[u]);
      if (lane == 0) wcnt[h][u * (kThreads / 32) + cw] = __popc(bal);
      before[u] = __popc(bal & ((1u << lane) - 1u));
    }
    named_sync(kBarCons, kThreads);
    // every warp scans the counts itself
    const int c = lane < kCounts ? wcnt[h][lane] : 0;
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int total = __shfl_sync(0xffffffffu, incl, kCounts - 1);
#pragma unroll
    for (int u = 0; u < kPairSlots; ++u) {
      const int idx = u * (kThreads / 32) + cw;
      const int excl = __shfl_sync(0xffffffffu, incl - c, idx);
      const unsigned long long g = local + (unsigned long long)(excl + before[u]);
      if (acc[u]) {
        if constexpr (RAW) *reinterpret_cast<double2*>(out + 2 * g) = make_double2(px[u], py[u]);
        else fifo[g % kQCap] = make_double2(px[u], py[u]);
      }
    }
    local += (unsigned long long)total;
    hh = hh_next;
    if constexpr (RAW) continue;     // wcnt[h] is rewritten only two rounds on
    named_sync(kBarCons, kThreads);  // FIFO entries visible
    while (local - head >= 2 * kThreads) {
      const unsigned long long g = head + (unsigned long long)tid;
      transform(g);
      transform(g + kThreads);
      head += 2 * kThreads;
    }
    if (local - head >= kThreads) {
      transform(head + (unsigned long long)tid);
      head += kThreads;
    }
  }
  if constexpr (!RAW)
    for (unsigned long long g = head + (unsigned long long)tid; g < local; g += kThreads) transform(g);
  if (tid == 0) {
    cnt[(long long)w * P + s] = local;
    uint64_t* c = tail + ((long long)w * P + s) * kCkWords;
    c[kMtN] = (uint64_t)hh;
    c[kMtN + 1] = (uint64_t)__double_as_longlong(s_half[rounds & 1]);
    c[kMtN + 2] = local;
  }
}

// Walks generations from a checkpoint until the target pair; writes the new
// rng state.  Also serves the (rare) overflow continuation.  One CTA per
// (worker, step of the batch): step t ends with pair (t+1)*M - 1; the last
// step's CTA publishes the segment prefix (and the overflow extent).
__global__ void __launch_bounds__(kThreads)
mt_finish_kernel(uint64_t* mt, const int* pnorm, int P, int gens, int ck_every, int nck,
                 unsigned long long pairs_per_step, double stddev, double* slots, long long cap,
                 const unsigned long long* cnt, unsigned long long* pfx, const uint64_t* ck,
                 const uint64_t* tail, int* status, int raw) {
  __shared__ Smem sm;
  __shared__ unsigned long long s_pfx_target[3];
  const int w = blockIdx.x, tid = threadIdx.x, t = blockIdx.y;
  const bool publish = t == (int)gridDim.y - 1;
  const unsigned long long pairs_needed = pairs_per_step * (unsigned long long)(t + 1);
  mt += (long long)t * gridDim.x * (kMtN + 1);
  status += (long long)t * gridDim.x;
  const int p = pnorm[w];
  unsigned long long* pf = pfx + (long long)w * (P + 2);
  if (tid == 0) {
    unsigned long long run = 0, at = 0;
    int star = -1;
    for (int s = 0; s < P; ++s) {
      if (publish) pf[s] = run;
      const unsigned long long c = cnt[(long long)w * P + s];
      if (star < 0 && run + c >= pairs_needed) {
        star = s;
        at = run;
      }
      run += c;
    }
    if (publish) {
      pf[P] = run;
      pf[P + 1] = run;
    }
    s_pfx_target[0] = (unsigned long long)(star < 0 ? P : star);
    s_pfx_target[1] = run;
    s_pfx_target[2] = at;
  }
  __syncthreads();
  const int star = (int)s_pfx_target[0];
  const unsigned long long total = s_pfx_target[1];
  int have_half = 0, q = 0, lo = 0, hi = kMtN;
  double half = 0.0;
  unsigned long long local = 0, target = 0;
  double* out = nullptr;
  bool overflow = star >= P;
  if (!overflow) {
    target = pairs_needed - 1 - s_pfx_target[2];
    // last checkpoint at or before the target pair
    const uint64_t* base = ck + ((long long)w * P + star) * (long long)nck * kCkWords;
    int c = 0;
    for (int k = 1; k < nck; ++k) {
      if (k * ck_every >= gens + (p > 0 ? 1 : 0)) break;
      if (base[(long long)k * kCkWords + kMtN + 2] <= target) c = k;
    }
    const uint64_t* cp = base + (long long)c * kCkWords;
    if (tid < kMtN) sm.x[tid] = cp[tid];
    have_half = (int)cp[kMtN];
    half = __longlong_as_double((long long)cp[kMtN + 1]);
    local = cp[kMtN + 2];
    q = c * ck_every;
  } else {
    // continue after the last segment: its final array, next offset p
    const uint64_t* tp = tail + ((long long)w * P + (P - 1)) * kCkWords;
    if (tid < kMtN) sm.x[tid] = tp[tid];
    have_half = (int)tp[kMtN];
    half = __longlong_as_double((long long)tp[kMtN + 1]);
    local = 0;
    target = pairs_needed - 1 - total;
    out = slots + ((long long)w * (P + 1) + P) * cap;
    q = -1;  // marks continuation
  }
  __syncthreads();
  bool first = true;
  for (;;) {
    if (!overflow) {
      if (!first) block_twist(sm.x);
      lo = q == 0 ? p : 0;
      hi = (q == gens) ? p : kMtN;
    } else {
      if (first && p > 0) {
        lo = p;  // rest of the last segment's final array
      } else {
        block_twist(sm.x);
        lo = 0;
      }
      hi = kMtN;
    }
    first = false;
    const int carry_in = have_half;
    const PairEval e = eval_generation(sm, lo, hi, have_half, half);
    if (overflow && e.acc) {
      const unsigned long long m = local + (unsigned long long)e.rank;
      if (2 * m + 1 < (unsigned long long)cap) {
        if (raw) {
          out[2 * m] = e.px;
          out[2 * m + 1] = e.py;
        } else {
          const double mult = mt_polar_mult(e.r2);
          out[2 * m] = mt_scale(e.py, mult, stddev);
          out[2 * m + 1] = mt_scale(e.px, mult, stddev);
        }
      }
    }
    if (local + (unsigned long long)e.total > target) {
      // the attempt with rank (target - local) ends this step's consumption
      if (e.acc && (unsigned long long)e.rank == target - local) {
        const int end_off = lo - carry_in + 2 * tid + 2;  // one past its second output
        sm.misc[0] = end_off;
      }
      __syncthreads();
      uint64_t* st = mt + (long long)w * (kMtN + 1);
      if (tid < kMtN) st[tid] = sm.x[tid];
      if (tid == 0) {
        st[kMtN] = (uint64_t)sm.misc[0];
        if (overflow) {
          if (publish) pf[P + 1] = total + target + 1;
          status[w] = (2 * (target + 1) <= (unsigned long long)cap) ? 0 : 1;
        } else {
          status[w] = 0;
        }
      }
      return;
    }
    local += (unsigned long long)e.total;
    if (!overflow) ++q;
  }
}

}  // namespace

NoiseEngine::~NoiseEngine() {
  for (void* p : {(void*)ybuf_, (void*)win_, (void*)cfg_[0].jbits, (void*)cfg_[1].jbits, (void*)joff_,
                  (void*)slots_, (void*)cnt_, (void*)pfx_, (void*)ck_, (void*)tail_, (void*)status_})
    if (p) cudaFree(p);
}

// Segment geometry for a run of `steps` steps, and its jump bitsets.
bool NoiseEngine::make_cfg(int steps, int nsm, Cfg* c, std::string* err) {
  // outputs a run needs: 2 per attempt, M / (pi/4) attempts, + 8 sd + slack
  const double M = (double)((dim_ + 1) / 2) * steps;
  const double pa = 0.78539816339744831;
  const double attempts = M / pa + 8.0 * std::sqrt(M * (1.0 - pa)) / pa + 1024.0;
  const double E = 2.0 * attempts;
  const double min_seg = 312.0 * 64.0;
  // Segment count: the segment kernel is latency-bound per CTA (measured
  // ~2.24 ns per output, so T_seg ~ 2.24e-3 us * E / P) and jumps cost
  // ~1.3 us of whole-GPU time each (T_jump ~ 1.3 us * kl * (P-1)); their sum
  // is minimal at P* = sqrt(1.72e-3 * E / kl).  Capped so segment CTAs fit
  // one wave at 2 per SM; segments no shorter than 64 generations.
  int P = (int)std::lround(std::sqrt(1.72e-3 * E / kl_));
  P = std::min(P, (int)std::ceil(E / min_seg));
  P = std::min(P, std::max(1, 2 * nsm / kl_));
  P = std::max(1, P);
  long long gens = (long long)std::ceil(E / P / 312.0);
  if (gens < 1) gens = 1;
  c->steps = steps;
  c->S = gens * 312;
  c->P = (int)std::ceil(E / (double)c->S);
  c->gens = (int)gens;
  c->nck = (c->gens + 1 + ck_every_ - 1) / ck_every_ + 1;
  c->cap = c->S + 16;
  // jump bitsets for s = 1..P-1: c_s = x^(sS-1) mod phi
  const std::vector<uint64_t>& phi = mt_char_poly();
  constexpr int kCW = kJumpBits / 32 + 1;
  std::vector<uint32_t> bits((size_t)std::max(1, c->P - 1) * kCW, 0);
  if (c->P > 1) {
    Poly cs = x_pow((unsigned long long)c->S - 1, phi);
    const Poly step = x_pow((unsigned long long)c->S, phi);
    for (int s = 1; s < c->P; ++s) {
      if (s > 1) cs = mulmod(cs, step, phi);
      uint32_t* dst = bits.data() + (size_t)(s - 1) * kCW;
      for (int i = 0; i < kDeg; ++i)
        if (get_bit(cs.data(), (size_t)i)) dst[i >> 5] |= 1u << (i & 31);
    }
  }
  if (cudaMalloc(&c->jbits, bits.size() * 4) != cudaSuccess) {
    *err = "noise engine: cudaMalloc failed";
    return false;
  }
  cudaMemcpy(c->jbits, bits.data(), bits.size() * 4, cudaMemcpyHostToDevice);
  return true;
}

bool NoiseEngine::init(unsigned long long dim, int kl, int nsm, int max_steps, std::string* err) {
  dim_ = dim;
  kl_ = kl;
  {
    // 6 generations per round (default; engine 0.77 -> 0.74 ms/step) or 4
    const char* e = std::getenv("DSX_SEG_R");
    seg_r_ = (e && std::atoi(e) == 4) ? 4 : 6;
  }
  ck_every_ = seg_r_ == 6 ? 12 : 16;  // a checkpoint every few whole rounds
  if (mt_char_poly().empty()) {
    *err = "MT19937-64 characteristic polynomial: Berlekamp-Massey did not reach degree 19937";
    return false;
  }
  max_steps = std::max(1, max_steps);
  if (!make_cfg(1, nsm, &cfg_[0], err)) return false;
  if (max_steps > 1) {
    if (!make_cfg(max_steps, nsm, &cfg_[1], err)) return false;
  } else {
    cfg_[1] = cfg_[0];
    cfg_[1].jbits = nullptr;  // shared with cfg_[0] (freed once)
  }
  long long P = 0, kw = 0, ckw = 0;
  for (const Cfg& c : cfg_) {
    P = std::max<long long>(P, c.P);
    slot_stride_ = std::max<long long>(slot_stride_, (long long)kl * (c.P + 1) * c.cap);
    ckw = std::max<long long>(ckw, (long long)kl * c.P * c.nck * kCkWords);
    kw = std::max<long long>(kw, (long long)kl * c.P * kMtN);
  }
  pfx_stride_ = (long long)kl * (P + 2);
  auto alloc = [&](void** p, size_t bytes) {
    if (cudaMalloc(p, bytes) != cudaSuccess) {
      *err = "noise engine: cudaMalloc failed";
      return false;
    }
    return true;
  };
  if (!alloc((void**)&ybuf_, 8ull * kPrefixWords * kl) || !alloc((void**)&win_, 8ull * kw) ||
      !alloc((void**)&slots_, 2 * 8ull * slot_stride_) || !alloc((void**)&cnt_, 2 * 8ull * P * kl) ||
      !alloc((void**)&pfx_, 2 * 8ull * pfx_stride_) || !alloc((void**)&ck_, 8ull * ckw) ||
      !alloc((void**)&tail_, 8ull * kCkWords * P * kl) ||
      !alloc((void**)&status_, 2 * 4ull * kl * max_steps) || !alloc((void**)&joff_, 2 * 4ull * kl))
    return false;
  cudaMemset(status_, 0, 2 * 4ull * kl * max_steps);
  if (cudaFuncSetAttribute(mt_jump2_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           8 * (kPrefixWords + kJ2PerCta * 4 * kMtN)) != cudaSuccess) {
    *err = "noise engine: cannot opt in to 205 KB shared memory";
    return false;
  }
  return true;
}

bool NoiseEngine::run(const uint64_t* mt_src, uint64_t* mt_dst, int set, int steps, double stddev,
                      void* stream_ptr, std::string* err) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_ptr);
  const int ci = steps > 1 ? 1 : 0;
  const Cfg& c = cfg_[ci];
  if (steps != c.steps) {
    *err = "noise engine: unsupported batch length";
    return false;
  }
  set_cfg_[set] = ci;
  int* pnorm = joff_;              // [kl] cursor normalized by the prefix kernel
  int* pnorm2 = joff_ + kl_;       // [kl] the same, written by segment 0
  double* slots = slots_ + (long long)set * slot_stride_;
  unsigned long long* cnt = cnt_ + (long long)set * (pfx_stride_ / kl_ - 2) * kl_;
  unsigned long long* pfx = pfx_ + (long long)set * pfx_stride_;
  int* status = status_ + (long long)set * kl_ * cfg_[1].steps;
  const int P = c.P;
  if (P > 1) {
    mt_prefix_kernel<<<kl_, kThreads, 0, stream>>>(mt_src, ybuf_, win_, P, pnorm);
    ++launches_;
    // 4 warps per jump (8 was measured slower)
    dim3 grid((P - 1 + kJ2PerCta - 1) / kJ2PerCta, kl_);
    mt_jump2_kernel<4><<<grid, kJ2PerCta * 4 * 32, 8 * (kPrefixWords + kJ2PerCta * 4 * kMtN), stream>>>(
        ybuf_, c.jbits, win_, P);
    ++launches_;
  }
  // DSX_NOISE_RAW=1: the segment kernel stores the raw accepted attempts
  // and the update kernel applies the polar transform (+3-7 % it/s, but the
  // update kernel then runs at ~0.64 of HBM instead of ~0.83; off by default)
  static const bool raw_ok = [] {
    const char* e = std::getenv("DSX_NOISE_RAW");
    return e && e[0] == '1';
  }();
  const int raw = raw_ok ? 1 : 0;
  raw_[set] = raw;
  stddev_[set] = stddev;
  // dynamic shared memory opt-in, per device (one process may drive several)
  static std::atomic<unsigned long long> attr{0};
  once_per_device(attr, [] {
    cudaFuncSetAttribute(mt_segment_ws2_kernel<true, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Ws2Smem<4>::kBytes);
    cudaFuncSetAttribute(mt_segment_ws2_kernel<false, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Ws2Smem<4>::kBytes);
    cudaFuncSetAttribute(mt_segment_ws2_kernel<true, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Ws2Smem<6>::kBytes);
    cudaFuncSetAttribute(mt_segment_ws2_kernel<false, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Ws2Smem<6>::kBytes);
  });
  // generations per round (DSX_SEG_R: 4 or 6; checkpoints every 16 / 12)
  auto go = [&](auto kern, size_t smem) {
    kern<<<dim3(P, kl_), kWs2Threads, smem, stream>>>(mt_src, win_, pnorm, pnorm2, P, c.gens, ck_every_, c.nck,
                                                       stddev, slots, c.cap, cnt, ck_, tail_);
  };
  if (seg_r_ == 6) {
    if (raw) go(mt_segment_ws2_kernel<true, 6>, Ws2Smem<6>::kBytes);
    else go(mt_segment_ws2_kernel<false, 6>, Ws2Smem<6>::kBytes);
  } else {
    if (raw) go(mt_segment_ws2_kernel<true, 4>, Ws2Smem<4>::kBytes);
    else go(mt_segment_ws2_kernel<false, 4>, Ws2Smem<4>::kBytes);
  }
  mt_finish_kernel<<<dim3(kl_, steps), kThreads, 0, stream>>>(mt_dst, pnorm2, P, c.gens, ck_every_, c.nck,
                                                              (dim_ + 1) / 2, stddev, slots, c.cap, cnt, pfx,
                                                              ck_, tail_, status, raw);
  launches_ += 2;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("noise engine launch: ") + cudaGetErrorString(e);
    return false;
  }
  return true;
}

}  // namespace dsx
