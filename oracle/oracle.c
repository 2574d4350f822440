/*
 * oracle.c — CPU restatement of the reference's partial-sync local-SGD hot
 * path.  TEST INFRASTRUCTURE ONLY (see oracle.h): tests/, smoke() and the
 * bench's CPU legs use it as the checker; the product never links it.
 *
 * Build: -O2 -ffp-contract=off, no -march flags, so the double arithmetic
 * rounds exactly like the reference compiled by g++ 13 for baseline x86-64
 * (no FMA contraction is possible there).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- libstdc++ <random> restatements ---------------------------------- */

/* std::mt19937_64 parameters ([rand.predef]). */
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ull /* (~0) << 31 */
#define MT_LOWER 0x000000007FFFFFFFull
#define MT_A 0xB5026F5AA96619E9ull

/* seed_seq::generate (random.tcc:3257) over `count` input words producing
 * out[0..n). */
static void seed_seq_generate(const uint32_t* v, size_t s, uint32_t* out, size_t n) {
  for (size_t i = 0; i < n; ++i) out[i] = 0x8b8b8b8bu;
  const size_t t = n >= 623 ? 11 : n >= 68 ? 7 : n >= 39 ? 5 : n >= 7 ? 3 : (n - 1) / 2;
  const size_t p = (n - t) / 2;
  const size_t q = p + t;
  const size_t m = (s + 1 > n) ? s + 1 : n;
  for (size_t k = 0; k < m; ++k) {
    const size_t kn = k % n, kp = (k + p) % n, kq = (k + q) % n, km = (k + n - 1) % n;
    uint32_t arg = out[kn] ^ out[kp] ^ out[km];
    uint32_t r1 = 1664525u * (arg ^ (arg >> 27));
    uint32_t r2 = r1 + (k == 0 ? (uint32_t)s : (uint32_t)kn + (k <= s ? v[k - 1] : 0u));
    out[kp] += r1;
    out[kq] += r2;
    out[kn] = r2;
  }
  for (size_t k = m; k < m + n; ++k) {
    const size_t kn = k % n, kp = (k + p) % n, kq = (k + q) % n, km = (k + n - 1) % n;
    uint32_t arg = out[kn] + out[kp] + out[km];
    uint32_t r3 = 1566083941u * (arg ^ (arg >> 27));
    uint32_t r4 = r3 - (uint32_t)kn;
    out[kp] ^= r3;
    out[kq] ^= r4;
    out[kn] = r4;
  }
}

/* mersenne_twister_engine::seed(seed_seq&) (random.tcc:354-389). */
void orc_mt_seed_seq(orc_mt* mt, const uint32_t* words, size_t count) {
  uint32_t arr[2 * ORC_MT_N];
  seed_seq_generate(words, count, arr, 2 * ORC_MT_N);
  int zero = 1;
  for (int i = 0; i < ORC_MT_N; ++i) {
    mt->x[i] = (uint64_t)arr[2 * i] | ((uint64_t)arr[2 * i + 1] << 32);
    if (zero) {
      if (i == 0) {
        if ((mt->x[0] & MT_UPPER) != 0) zero = 0;
      } else if (mt->x[i] != 0) {
        zero = 0;
      }
    }
  }
  if (zero) mt->x[0] = 1ull << 63;
  mt->p = ORC_MT_N;
}

/* trainer.cpp:169-173 */
void orc_worker_rng(orc_mt* mt, uint64_t seed, int worker) {
  const uint32_t words[4] = {(uint32_t)seed, (uint32_t)(seed >> 32), (uint32_t)worker, 0x5eedu};
  orc_mt_seed_seq(mt, words, 4);
}

/* _M_gen_rand (random.tcc:399-425): the in-place twist of all 312 words. */
static void mt_twist(orc_mt* mt) {
  uint64_t* x = mt->x;
  for (int k = 0; k < ORC_MT_N; ++k) {
    const uint64_t y = (x[k] & MT_UPPER) | (x[(k + 1) % ORC_MT_N] & MT_LOWER);
    x[k] = x[(k + MT_M) % ORC_MT_N] ^ (y >> 1) ^ ((y & 1) ? MT_A : 0);
  }
  mt->p = 0;
}

uint64_t orc_mt_next(orc_mt* mt) {
  if (mt->p >= ORC_MT_N) mt_twist(mt);
  uint64_t z = mt->x[mt->p++];
  z ^= (z >> 29) & 0x5555555555555555ull;
  z ^= (z << 17) & 0x71D67FFFEDA60000ull;
  z ^= (z << 37) & 0xFFF7EEE000000000ull;
  z ^= z >> 43;
  return z;
}

/* generate_canonical<double,53> (random.tcc:3349-3381): one 64-bit draw,
 * converted to double (round to nearest) and scaled by 2^-64, clamped
 * below 1. */
double orc_canonical(orc_mt* mt) {
  const double sum = (double)orc_mt_next(mt);
  double ret = sum / 18446744073709551616.0;
  if (ret >= 1.0) ret = nextafter(1.0, 0.0);
  return ret;
}

/* normal_distribution<double>::operator() (random.tcc:1812-1844) for one
 * distribution object living across n calls. */
void orc_normal_fill(orc_mt* mt, double stddev, double* out, size_t n) {
  int saved_available = 0;
  double saved = 0.0;
  for (size_t i = 0; i < n; ++i) {
    double ret;
    if (saved_available) {
      saved_available = 0;
      ret = saved;
    } else {
      double x, y, r2;
      do {
        x = 2.0 * orc_canonical(mt) - 1.0;
        y = 2.0 * orc_canonical(mt) - 1.0;
        r2 = x * x + y * y;
      } while (r2 > 1.0 || r2 == 0.0);
      const double mult = sqrt(-2 * log(r2) / r2);
      saved = x * mult;
      saved_available = 1;
      ret = y * mult;
    }
    out[i] = ret * stddev + 0.0;
  }
}

/* ---- quadratic lab ------------------------------------------------------ */

/* trainer.cpp:100-124 */
int orc_make_quadratic(size_t dim, int blocks, double mu, double beta, double* curvature,
                       uint64_t* block_sizes) {
  if (blocks < 1 || (size_t)blocks > dim) return -1;
  if (!(mu > 0.0) || !(beta >= mu)) return -1;
  const size_t base = dim / (size_t)blocks, extra = dim % (size_t)blocks;
  for (int b = 0; b < blocks; ++b) block_sizes[b] = base + ((size_t)b < extra ? 1 : 0);
  for (size_t i = 0; i < dim; ++i) {
    curvature[i] = dim == 1 ? mu : mu + (beta - mu) * (double)i / (double)(dim - 1);
  }
  return 0;
}

/* trainer.cpp:126-130 */
double orc_shift(double mu, double beta, int period, double shift_a) {
  if (shift_a > 0.0) return shift_a;
  const double kappa = beta / mu;
  const double a = 16.0 * kappa, b = (double)period;
  return (a < b ? b : a) + 1.0;
}

/* trainer.cpp:132-135 */
double orc_learning_rate(long long r, double mu, double beta, int period, double shift_a,
                         int constant, double eta) {
  if (constant) return eta;
  return 4.0 / (mu * (orc_shift(mu, beta, period, shift_a) + (double)r));
}

/* trainer.cpp:73-77 + 175-185 */
void orc_stochastic_gradient(size_t dim, const double* curvature, const double* optimum,
                             double sigma, const double* w, orc_mt* rng, double* g) {
  for (size_t i = 0; i < dim; ++i) g[i] = curvature[i] * (w[i] - optimum[i]);
  if (sigma > 0.0) {
    double* xi = (double*)malloc(dim * sizeof(double));
    orc_normal_fill(rng, sigma / sqrt((double)dim), xi, dim);
    for (size_t i = 0; i < dim; ++i) g[i] += xi[i];
    free(xi);
  }
}

/* trainer.cpp:31-38 */
double orc_pairwise_sum(const double* w, size_t stride, size_t i, size_t lo, size_t hi) {
  const size_t n = hi - lo;
  if (n == 1) return w[lo * stride + i];
  if (n == 2) return w[lo * stride + i] + w[(lo + 1) * stride + i];
  const size_t mid = lo + n / 2;
  return orc_pairwise_sum(w, stride, i, lo, mid) + orc_pairwise_sum(w, stride, i, mid, hi);
}

/* trainer.cpp:202-224 */
void orc_sync_mask(int mode, int period, long long r, int layer_count, const int* set_ptr,
                   const int* set_idx, const int* fill_ptr, const int* fill_idx,
                   unsigned char* mask) {
  memset(mask, 0, (size_t)layer_count + 1);
  const long long phase = (r + 1) % period;
  if (mode == 2 || (mode == 1 && phase == 0)) {
    memset(mask, 1, (size_t)layer_count + 1);
    return;
  }
  if (mode != 0) return;
  const int h = phase == 0 ? period : (int)phase;
  for (int j = set_ptr[h - 1]; j < set_ptr[h]; ++j) mask[set_idx[j]] = 1;
  if (fill_ptr) {
    for (int j = fill_ptr[h - 1]; j < fill_ptr[h]; ++j) mask[fill_idx[j]] = 1;
  }
}

/* trainer.cpp:187-235 */
void orc_plsgd_step(double* w, orc_mt* rngs, int workers, size_t dim, const double* curvature,
                    const double* optimum, double sigma, const uint64_t* block_sizes,
                    int layer_count, double eta, const unsigned char* mask,
                    double* max_norm_sq) {
  double max_sq = 0.0;
  double* g = (double*)malloc(dim * sizeof(double));
  for (int k = 0; k < workers; ++k) {
    double* wk = w + (size_t)k * dim;
    orc_stochastic_gradient(dim, curvature, optimum, sigma, wk, &rngs[k], g);
    double norm_sq = 0.0;
    for (size_t i = 0; i < dim; ++i) {
      norm_sq += g[i] * g[i];
      wk[i] -= eta * g[i];
    }
    if (norm_sq > max_sq) max_sq = norm_sq;
  }
  free(g);
  if (max_norm_sq) *max_norm_sq = max_sq;

  size_t lo = 0;
  for (int b = 0; b < layer_count; ++b) {
    const size_t hi = lo + block_sizes[b];
    if (mask[b + 1]) {
      for (size_t i = lo; i < hi; ++i) {
        const double mean = orc_pairwise_sum(w, dim, i, 0, (size_t)workers) / (double)workers;
        for (int k = 0; k < workers; ++k) w[(size_t)k * dim + i] = mean;
      }
    }
    lo = hi;
  }
}

static double objective(size_t dim, const double* curvature, const double* optimum,
                        const double* w) {
  double value = 0.0;
  for (size_t i = 0; i < dim; ++i) {
    const double d = w[i] - optimum[i];
    value += 0.5 * curvature[i] * d * d;
  }
  return value;
}

/* trainer.cpp:237-307 */
long long orc_run_training(int workers, int period, long long iterations, int mode,
                           int constant_lr, double eta, double shift_a, uint64_t seed,
                           long long log_stride, size_t dim, const double* curvature,
                           const double* optimum, double sigma, const uint64_t* block_sizes,
                           int layer_count, const int* set_ptr, const int* set_idx,
                           const int* fill_ptr, const int* fill_idx, long long max_rows,
                           long long* iteration, double* gamma, double* gamma_per_layer,
                           double* lemma, double* subopt, double* iterate_subopt,
                           double* eta_out, double* out_scalars, double* w_out) {
  double mu = curvature[0], beta = curvature[0];
  for (size_t i = 1; i < dim; ++i) {
    if (curvature[i] < mu) mu = curvature[i];
    if (curvature[i] > beta) beta = curvature[i];
  }
  const size_t K = (size_t)workers;
  double* w = (double*)calloc(K * dim, sizeof(double));
  orc_mt* rngs = (orc_mt*)malloc(K * sizeof(orc_mt));
  for (int k = 0; k < workers; ++k) orc_worker_rng(&rngs[k], seed, k);
  double* weighted = (double*)calloc(dim, sizeof(double));
  double* w_hat = (double*)calloc(dim, sizeof(double));
  double* mean = (double*)malloc(dim * sizeof(double));
  unsigned char* mask = (unsigned char*)malloc((size_t)layer_count + 1);
  double weight_total = 0.0, g_meas = 0.0;
  const double shift = orc_shift(mu, beta, period, shift_a);
  long long rows = 0;

  for (long long r = -1; r < iterations; ++r) {
    if (r >= 0) {
      for (size_t i = 0; i < dim; ++i) mean[i] = orc_pairwise_sum(w, dim, i, 0, K) / (double)K;
      const double p_r = constant_lr ? 1.0 : (shift + (double)r) * (shift + (double)r);
      for (size_t i = 0; i < dim; ++i) weighted[i] += p_r * mean[i];
      weight_total += p_r;
      const double eta_r = orc_learning_rate(r, mu, beta, period, shift_a, constant_lr, eta);
      orc_sync_mask(mode, period, r, layer_count, set_ptr, set_idx, fill_ptr, fill_idx, mask);
      double max_sq = 0.0;
      orc_plsgd_step(w, rngs, workers, dim, curvature, optimum, sigma, block_sizes,
                     layer_count, eta_r, mask, &max_sq);
      const double gn = sqrt(max_sq);
      if (gn > g_meas) g_meas = gn;
    }
    const long long n = r + 1;
    if (!(n == 0 || n % log_stride == 0 || n == iterations)) continue;
    if (rows >= max_rows) break;
    /* log_row (trainer.cpp:254-284) */
    for (size_t i = 0; i < dim; ++i) mean[i] = orc_pairwise_sum(w, dim, i, 0, K) / (double)K;
    double gsum = 0.0;
    size_t lo = 0;
    for (int b = 0; b < layer_count; ++b) {
      const size_t hi = lo + block_sizes[b];
      double acc = 0.0;
      for (size_t k = 0; k < K; ++k) {
        for (size_t i = lo; i < hi; ++i) {
          const double d = mean[i] - w[k * dim + i];
          acc += d * d;
        }
      }
      const double pl = acc / (double)workers;
      gamma_per_layer[rows * layer_count + b] = pl;
      lo = hi;
    }
    for (int b = 0; b < layer_count; ++b) gsum += gamma_per_layer[rows * layer_count + b];
    const double eta_n = orc_learning_rate(n, mu, beta, period, shift_a, constant_lr, eta);
    const double h = (double)period;
    iteration[rows] = n;
    gamma[rows] = gsum;
    lemma[rows] = 4.0 * h * h * eta_n * eta_n * g_meas * g_meas;
    if (weight_total > 0.0) {
      for (size_t i = 0; i < dim; ++i) w_hat[i] = weighted[i] / weight_total;
      subopt[rows] = objective(dim, curvature, optimum, w_hat);
    } else {
      subopt[rows] = objective(dim, curvature, optimum, mean);
    }
    iterate_subopt[rows] = objective(dim, curvature, optimum, mean);
    eta_out[rows] = eta_n;
    ++rows;
  }
  out_scalars[0] = g_meas;
  out_scalars[1] = rows ? subopt[rows - 1] : 0.0;
  out_scalars[2] = rows ? iterate_subopt[rows - 1] : 0.0;
  if (w_out) memcpy(w_out, w, K * dim * sizeof(double));
  free(w);
  free(rngs);
  free(weighted);
  free(w_hat);
  free(mean);
  free(mask);
  return rows;
}
