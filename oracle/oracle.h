/*
 * oracle.h — CPU restatement of the reference's partial-sync local-SGD path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2502_11058_b200/)
 * may link, load or call this code; only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs use it, and only as the
 * checker.  Parity is pinned against the compiled reference (oracle/_ref, see
 * oracle/Makefile) and the golden fixtures under tests/golden/.
 *
 * Every function cites the reference source it restates
 * (/root/reference/proj/core/src/trainer.cpp unless noted) and the libstdc++
 * (GCC 13.3, /usr/include/c++/13/bits/random.tcc) algorithms the reference
 * inherits through <random>: mt19937_64, seed_seq, generate_canonical and the
 * Marsaglia-polar normal_distribution.
 */
#ifndef DREAMDDP_ORACLE_H_
#define DREAMDDP_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MT_N 312

/* std::mt19937_64 state: x[] and the read cursor p (libstdc++ _M_x/_M_p). */
typedef struct {
  uint64_t x[ORC_MT_N];
  uint64_t p;
} orc_mt;

/* trainer.cpp:169-173 worker_rng: seed_seq{lo32, hi32, worker, 0x5eed}. */
void orc_worker_rng(orc_mt* mt, uint64_t seed, int worker);
/* seed_seq over an arbitrary list of 32-bit words (profile.cpp:188 uses it too). */
void orc_mt_seed_seq(orc_mt* mt, const uint32_t* words, size_t count);
uint64_t orc_mt_next(orc_mt* mt);
/* generate_canonical<double, 53>(mt) */
double orc_canonical(orc_mt* mt);

/* Fills out[0..n) with one normal_distribution<double>(0, stddev) object's
 * draws (polar method, second value cached inside the object and dropped when
 * the object dies) — trainer.cpp:179-183. */
void orc_normal_fill(orc_mt* mt, double stddev, double* out, size_t n);

/* trainer.cpp:100-124 make_quadratic: curvature and block sizes. */
int orc_make_quadratic(size_t dim, int blocks, double mu, double beta,
                       double* curvature /*dim*/, uint64_t* block_sizes /*blocks*/);

/* trainer.cpp:126-135 learning rate (decaying when constant_eta <= 0). */
double orc_shift(double mu, double beta, int period, double shift_a);
double orc_learning_rate(long long r, double mu, double beta, int period,
                         double shift_a, int constant, double eta);

/* trainer.cpp:175-185 stochastic_gradient (g must hold dim doubles). */
void orc_stochastic_gradient(size_t dim, const double* curvature, const double* optimum,
                             double sigma, const double* w, orc_mt* rng, double* g);

/* trainer.cpp:31-38 pairwise_coord_sum over w[lo..hi)[i] with row stride. */
double orc_pairwise_sum(const double* w, size_t stride, size_t i, size_t lo, size_t hi);

/* trainer.cpp:202-224 sync mask.  mode: 0 partial, 1 full, 2 ssgd.
 * sets/fills: flat CSR over H iterations (ptr has H+1 entries).  mask has
 * L+1 entries, 1-based like the reference's vector<bool>. */
void orc_sync_mask(int mode, int period, long long r, int layer_count,
                   const int* set_ptr, const int* set_idx,
                   const int* fill_ptr, const int* fill_idx, unsigned char* mask);

/* trainer.cpp:187-235 plsgd_step on K workers stored row-major w[K][dim]. */
void orc_plsgd_step(double* w, orc_mt* rngs, int workers, size_t dim,
                    const double* curvature, const double* optimum, double sigma,
                    const uint64_t* block_sizes, int layer_count, double eta,
                    const unsigned char* mask, double* max_norm_sq);

/* trainer.cpp:237-307 run_training.  Returns the number of logged rows.
 * Outputs (sized by the caller for max_rows rows): iteration, gamma,
 * gamma_per_layer[row*L+b], lemma, subopt, iterate_subopt, eta; scalars via
 * out_scalars = {g_meas, final_subopt, final_iterate_subopt}.  w_out (K*dim)
 * receives the final worker parameters when non-NULL. */
long long orc_run_training(int workers, int period, long long iterations, int mode,
                           int constant_lr, double eta, double shift_a, uint64_t seed,
                           long long log_stride, size_t dim, const double* curvature,
                           const double* optimum, double sigma, const uint64_t* block_sizes,
                           int layer_count, const int* set_ptr, const int* set_idx,
                           const int* fill_ptr, const int* fill_idx, long long max_rows,
                           long long* iteration, double* gamma, double* gamma_per_layer,
                           double* lemma, double* subopt, double* iterate_subopt,
                           double* eta_out, double* out_scalars, double* w_out);

#ifdef __cplusplus
}
#endif

#endif /* DREAMDDP_ORACLE_H_ */
