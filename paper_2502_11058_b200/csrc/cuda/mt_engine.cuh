// mt_engine.cuh — the reference's worker noise stream, reproduced on the GPU.
//
// The reference draws per-coordinate gradient noise with
//   std::normal_distribution<double>(0, sigma/sqrt(d)) over std::mt19937_64
// (trainer.cpp:179-183), i.e. libstdc++'s Marsaglia polar method
// (random.tcc:1812-1844) fed by generate_canonical<double,53>
// (random.tcc:3349-3381) of the 64-bit Mersenne twister (random.tcc:399-425).
// These helpers restate that arithmetic with explicit IEEE round-to-nearest
// intrinsics (no FMA contraction), so every accept/reject decision and every
// stream position is bit-identical to the host library; the only possible
// difference is the last ulp of log() in the polar transform (CUDA's log is
// within 1 ulp; glibc's is nearly correctly rounded).
#pragma once

#include <cstdint>

namespace dsx {

constexpr int kMtN = 312;
constexpr int kMtM = 156;
constexpr uint64_t kMtUpper = 0xFFFFFFFF80000000ull;
constexpr uint64_t kMtLower = 0x000000007FFFFFFFull;
constexpr uint64_t kMtA = 0xB5026F5AA96619E9ull;

// x[k+312] = x[k+156] ^ twist(x[k], x[k+1])
__host__ __device__ __forceinline__ uint64_t mt_next_word(uint64_t xk, uint64_t xk1, uint64_t xkm) {
  const uint64_t y = (xk & kMtUpper) | (xk1 & kMtLower);
  return xkm ^ (y >> 1) ^ ((y & 1ull) ? kMtA : 0ull);
}

__host__ __device__ __forceinline__ uint64_t mt_temper(uint64_t z) {
  z ^= (z >> 29) & 0x5555555555555555ull;
  z ^= (z << 17) & 0x71D67FFFEDA60000ull;
  z ^= (z << 37) & 0xFFF7EEE000000000ull;
  z ^= z >> 43;
  return z;
}

// 2 * generate_canonical<double,53>(z) - 1.  (double)z rounds to nearest,
// the 2^-64 scale is exact, and the >= 1 clamp mirrors random.tcc:3371.
// Computed as t = 2u directly ((double)z * 2^-63, exact power-of-two
// scaling, so t == 2 * u bit for bit; the clamp u -> 1 - 2^-53 is t -> 2 - 2^-52).
__device__ __forceinline__ double mt_polar_coord(uint64_t tempered) {
  double t = __dmul_rn(__ull2double_rn(tempered), 0x1p-63);
  if (t >= 2.0) t = 0x1.fffffffffffffp0;
  return __dsub_rn(t, 1.0);
}

// Polar acceptance: !(r2 > 1 || r2 == 0) with r2 = x*x + y*y (no FMA).
__device__ __forceinline__ bool mt_polar_accept(double x, double y, double* r2_out) {
  const double r2 = __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y));
  *r2_out = r2;
  return !(r2 > 1.0 || r2 == 0.0);
}

// sqrt(-2 * log(r2) / r2)
__device__ __forceinline__ double mt_polar_mult(double r2) {
  return __dsqrt_rn(__ddiv_rn(__dmul_rn(-2.0, log(r2)), r2));
}

// ret * stddev + mean(0.0)
__device__ __forceinline__ double mt_scale(double v, double mult, double stddev) {
  return __dadd_rn(__dmul_rn(__dmul_rn(v, mult), stddev), 0.0);
}

// An accepted attempt (x, y) -> its two normals in the order
// normal_distribution hands them out: (y * mult, x * mult), scaled
// (random.tcc:1836-1840).  The same arithmetic wherever it runs, so the
// engine may store raw attempts and let the consumer transform them.
__device__ __forceinline__ double2 mt_polar_normals(double x, double y, double stddev) {
  double r2;
  mt_polar_accept(x, y, &r2);
  const double m = mt_polar_mult(r2);
  return make_double2(mt_scale(y, m, stddev), mt_scale(x, m, stddev));
}

}  // namespace dsx
