/*
 * dsx.h — C ABI of the B200 partial-synchronization local-SGD engine.
 *
 * This is the thin layer between the C++ host API (include/dreamsched/ headers,
 * the drop-in surface of the reference's dreamsched::core) and the sm_100a
 * kernels.  Plain pointers and sizes only; no C++ or torch types; no
 * exception ever crosses it: every entry point returns a dsx_status and
 * dsx_last_error() holds the message (thread-local).
 *
 * Reference interface each entry point replaces (reference paths relative to
 * /root/reference/proj/core):
 *   dsx_lab_create          — the per-run state of run_training (trainer.cpp:237-252):
 *                             K worker parameter vectors + Problem arrays, here a
 *                             device-resident arena [workers_local][ld] in HBM.
 *   dsx_lab_set/get_params  — WorkerState::w (trainer.hpp:76-79) in / out.
 *   dsx_lab_set/get_rng     — WorkerState::rng, the std::mt19937_64 state
 *                             (x[312], cursor) as libstdc++ stores it.
 *   dsx_lab_seed_rng        — worker_rng(seed, k) (trainer.cpp:169-173).
 *   dsx_lab_step            — plsgd_step (trainer.cpp:187-235): local step of every
 *                             worker (stochastic_gradient 175-185, update 191-199)
 *                             then in-place averaging of the masked blocks
 *                             (226-234), mask from trainer.cpp:202-224.
 *   dsx_lab_gradient        — stochastic_gradient (trainer.cpp:175-185).
 *   dsx_lab_mean_accumulate — the w_hat weighted average of run_training (290-295).
 *   dsx_lab_log             — log_row's divergence / objective terms (254-284).
 *   dsx_lab_comm_init       — (no reference counterpart: the reference averages
 *                             in-process) one rank per GPU over NCCL/NVLink.
 */
#ifndef DREAMDDP_DSX_H_
#define DREAMDDP_DSX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int dsx_status;
enum {
  DSX_OK = 0,
  DSX_ERR_ARGUMENT = 1, /* maps to dreamsched::ArgumentError */
  DSX_ERR_STATE = 2,    /* call out of order / unsupported configuration */
  DSX_ERR_CUDA = 3,     /* CUDA runtime failure (incl. no device) */
  DSX_ERR_NCCL = 4      /* NCCL failure */
};

/* arithmetic type of the parameter arena */
enum { DSX_F64 = 0, DSX_F32 = 1 };

/* cross-rank averaging algorithm (only used when nranks > 1) */
enum {
  DSX_SYNC_PAIRWISE = 0, /* reduce-scatter/all-gather with the reference's fixed
                            pairwise summation order: bit-identical to K
                            in-process workers */
  DSX_SYNC_NCCL_AVG = 1  /* one in-place ncclAllReduce per masked range (sum),
                            1/K fused into the local broadcast */
};

typedef struct dsx_lab dsx_lab;

typedef struct dsx_lab_desc {
  int device;                  /* CUDA ordinal */
  int dtype;                   /* DSX_F64 | DSX_F32 */
  int workers_total;           /* K (all ranks) */
  int worker_begin;            /* global id of the first worker held here */
  int workers_local;           /* rows held on this device */
  uint64_t dim;                /* parameters per worker */
  int layers;                  /* L registered layers (blocks) */
  const uint64_t* block_sizes; /* [layers], sums to dim; layer 1 first */
  const double* curvature;     /* [dim] host */
  const double* optimum;       /* [dim] host */
  double noise_sigma;          /* sigma; per-coordinate stddev sigma/sqrt(dim) */
} dsx_lab_desc;

const char* dsx_last_error(void);
dsx_status dsx_device_count(int* count);
/* Creates the CUDA context on DREAMSCHED_DEVICE (default 0) and the noise
 * engine's host tables; optional (everything is created lazily otherwise). */
dsx_status dsx_warmup(void);

dsx_status dsx_lab_create(const dsx_lab_desc* desc, dsx_lab** out);
dsx_status dsx_lab_destroy(dsx_lab* lab);

/* Worker rows.  `local` indexes the rows held here (0..workers_local-1). */
dsx_status dsx_lab_set_params(dsx_lab* lab, int local, const double* w);
dsx_status dsx_lab_get_params(dsx_lab* lab, int local, double* w);
dsx_status dsx_lab_fill_params(dsx_lab* lab, double value);
/* Whole arena in one copy each way: w is [workers_local][dim] row-major. */
dsx_status dsx_lab_set_all_params(dsx_lab* lab, const double* w);
dsx_status dsx_lab_get_all_params(dsx_lab* lab, double* w);

/* Every local worker's parameters w[workers_local][dim] and/or rng states
 * rng[workers_local][313] (x[312] then the cursor) in one transfer each —
 * plsgd_step's host WorkerState round trip.  Either pointer may be NULL.
 * Both calls return with the copies complete. */
dsx_status dsx_lab_set_state(dsx_lab* lab, const double* w, const uint64_t* rng);
dsx_status dsx_lab_get_state(dsx_lab* lab, double* w, uint64_t* rng);

/* One plsgd_step (trainer.cpp:187-235) on HOST-resident worker state:
 * rows[k] is worker k's dim parameters (read, then overwritten with the
 * result), rng[workers_local][313] the engine states in/out.  Replaces
 * set_state + step + get_state: the parameter transfers are split into
 * coordinate chunks and pipelined — chunk c+1 host->device, chunk c's fused
 * update and chunk c-1 device->host run concurrently (two copy engines), so
 * the call costs about one direction's PCIe time instead of both.  Rows in
 * pinned memory (cudaHostAlloc / dsx_host_alloc) get the overlap; pageable
 * rows are still correct.  Single rank, fp64; other labs take the
 * set_state/step/get_state path inside the call.  Returns with every copy
 * complete. */
dsx_status dsx_lab_step_host(dsx_lab* lab, double eta, const unsigned char* mask, double* const* rows,
                             uint64_t* rng);
/* Pinned host memory for rows / rng buffers (cudaHostAlloc, portable). */
dsx_status dsx_host_alloc(size_t bytes, void** out);
dsx_status dsx_host_free(void* p);

/* std::mt19937_64 state: 312 words and the cursor p (libstdc++ _M_x/_M_p). */
dsx_status dsx_lab_set_rng(dsx_lab* lab, int local, const uint64_t* x312, uint64_t p);
dsx_status dsx_lab_get_rng(dsx_lab* lab, int local, uint64_t* x312, uint64_t* p);
dsx_status dsx_lab_seed_rng(dsx_lab* lab, uint64_t seed);

/* One iteration (asynchronous on the lab's stream).  mask has layers+1
 * entries, 1-based like the reference's vector<bool>; mask[l] != 0 averages
 * layer l's block across all workers_total workers. */
dsx_status dsx_lab_step(dsx_lab* lab, double eta, const unsigned char* mask);
/* Same, but the per-coordinate noise xi[workers_local][dim] (already scaled)
 * is supplied by the caller instead of the device generator.  Test hook that
 * isolates the update/averaging kernels from the noise engine. */
dsx_status dsx_lab_step_with_noise(dsx_lab* lab, double eta, const unsigned char* mask,
                                   const double* xi);
/* max_k ||g_k||^2 of the last step (synchronizes). */
dsx_status dsx_lab_last_max_grad_norm_sq(dsx_lab* lab, double* out);
dsx_status dsx_lab_sync(dsx_lab* lab);

/* g = curvature*(w-optimum) + noise for row `local` at its current params,
 * advancing its rng (no update). g_out has dim entries. */
dsx_status dsx_lab_gradient(dsx_lab* lab, int local, double* g_out);

/* run_training helpers (single rank): w_hat_sum += weight * mean_k(w_k). */
dsx_status dsx_lab_mean_accumulate(dsx_lab* lab, double weight);
/* gamma_per_layer[layers] = (1/K) sum_k ||mean - w_k||^2 over each block;
 * out2[0] = f(w_hat_sum / weight_total) (or f(mean) when weight_total == 0);
 * out2[1] = f(mean).  Synchronizes. */
dsx_status dsx_lab_log(dsx_lab* lab, double weight_total, double* gamma_per_layer, double* out2);

/* Multi-GPU: one rank per GPU.  id is ncclUniqueId (128 bytes) from rank 0. */
dsx_status dsx_nccl_unique_id(unsigned char id[128]);
dsx_status dsx_lab_comm_init(dsx_lab* lab, const unsigned char id[128], int nranks, int rank,
                             int sync_algo);

/* Multi-GPU inside ONE process (the drop-in C++ API's DREAMSCHED_GPUS):
 * labs[r] is rank r's lab (distinct devices, equal contiguous worker
 * ranges in rank order).  Creates the communicators with ncclCommInitAll and
 * maps the peers' exchange buffers directly (peer access, no IPC).  After
 * this, every multi-rank call must be issued for all labs concurrently, one
 * host thread per lab (the calls contain cross-GPU barriers). */
dsx_status dsx_lab_comm_init_local(dsx_lab* const* labs, int n, int sync_algo);

/* Overlapped sync: when enabled (default), the local step runs in two
 * launches — layers above the lowest synced layer first — and the cross-rank
 * averaging of the synced blocks starts on a high-priority side stream as soon
 * as the first launch is done, overlapping the rest of the local step. */
dsx_status dsx_lab_set_overlap(dsx_lab* lab, int enabled);

/* Noise pipelining (default on): the exact noise engine generates step r+1's
 * noise on its own high-priority stream while step r's update runs; the rng
 * state visible through dsx_lab_get_rng stays the committed one.  Disabling
 * serializes noise and update (used to time each alone). */
dsx_status dsx_lab_set_pipeline(dsx_lab* lab, int enabled);

/* Bounded noise look-ahead (timing windows): drains the noise stream, drops
 * noise generated ahead of the committed rng state, and lets the engine
 * generate noise only for the next `steps` dsx_lab_step calls (runs are cut
 * to one step when a whole batch would reach past the horizon).  A window of
 * exactly `steps` steps then contains exactly its own engine work.  steps < 0
 * restores unbounded pipelining.  Results are unchanged either way. */
dsx_status dsx_lab_set_noise_horizon(dsx_lab* lab, long long steps);

/* NVLink roofline for the averaging kernel, measured now (collective: every
 * rank calls it between steps): a copy kernel with the averaging kernel's
 * access pattern over every rank's peer-mapped scratch buffer; *gbs = bus
 * bytes 2(W-1)/W x S per rank / median time.  0 on a single rank. */
dsx_status dsx_lab_link_probe(dsx_lab* lab, int reps, double* gbs);

/* Bandwidth-throttled sync (the paper's low-bandwidth regime): every synced
 * layer additionally occupies the FIFO sync stream for latency +
 * layer_bytes/bandwidth seconds (comm_time, profile.cpp:103-110), issued
 * when the layer's local step is done.  bandwidth <= 0 switches it off. */
dsx_status dsx_lab_set_link(dsx_lab* lab, double bandwidth, double latency);

/* CUDA-event layer profiler: t_bp[l] = device seconds of layer l's local
 * step (state untouched), t_comm[l] = seconds of its cross-rank average
 * (multi-rank), or the throttled link's model, or -1 (not measured).
 * Median of `reps`.  Each layer is timed alone, then the set is rescaled to
 * the step as it runs (one fused update pass; the grouped whole-model
 * average), keeping the layers' relative costs.  Feeds dsc_write_profile ->
 * schedule_dfs. */
dsx_status dsx_lab_profile(dsx_lab* lab, int reps, double* t_bp, double* t_comm);

/* Timing on the lab's compute stream: CUDA events in slots 0..31. */
dsx_status dsx_lab_event_record(dsx_lab* lab, int slot);
dsx_status dsx_lab_event_elapsed(dsx_lab* lab, int from_slot, int to_slot, float* ms);
/* Per-step instrumentation of the last dsx_lab_step: out5 = milliseconds of
 * [whole step, sync span, exposed sync, noise engine, local update] measured
 * with CUDA events on the lab's streams (sync/exposed are 0 on a single
 * rank, where averaging is fused into the update kernel).  Exposed sync is
 * max(0, sync done - local step done), the measured counterpart of
 * iteration_cost(...).term - bp_total (cost_model.cpp:26-41).
 * Enabled by dsx_lab_set_instrument(lab, 1). */
dsx_status dsx_lab_set_instrument(dsx_lab* lab, int enabled);
dsx_status dsx_lab_last_step_times(dsx_lab* lab, float* out5);
/* Noise engine alone: device milliseconds of one run generating `steps`
 * steps (1 or the lab's batch length, *batch_out), median of `reps`, from the
 * committed rng state; the generated noise is discarded (state untouched). */
dsx_status dsx_lab_engine_time(dsx_lab* lab, int steps, int reps, float* ms, int* batch_out);

/* Host-only: *pairwise_exact = 1 when splitting workers_total workers into
 * nranks equal contiguous ranges keeps each range a subtree of the
 * reference's pairwise summation tree (trainer.cpp:31-38), i.e. when
 * DSX_SYNC_PAIRWISE reproduces the in-process result bit-for-bit. */
dsx_status dsx_sync_plan(int workers_total, int nranks, int* pairwise_exact);

/* Host-only self-test of the MT19937-64 jump-ahead used by the parallel
 * noise engine: *ok = 1 when jumping J outputs by polynomial equals running
 * the recurrence (no GPU needed). */
dsx_status dsx_mt_jump_selftest(unsigned long long jump, int* ok);

/* Measured timeline of the last instrumented single-GPU step with a
 * throttled link: bp[2l], bp[2l+1] = start/end ms of layer l's local step,
 * comm[2l], comm[2l+1] = start/end ms of its transfer on the FIFO link (-1
 * if not synced), relative to the step start — simulate_run's events,
 * measured (simulator.cpp:145-157).  With overlap disabled
 * (dsx_lab_set_overlap(lab, 0)) transfers start after the whole local step
 * (the ssgd mode). */
dsx_status dsx_lab_last_timeline(dsx_lab* lab, float* bp, float* comm);

/* Self-test of the cross-rank averaging kernel for `nranks` ranks spread
 * round-robin over the visible GPUs in this process (peer access): every
 * rank's slice averaged from every rank's buffer over NVLink, compared
 * with the reference's pairwise tree / K on the host.  *max_abs_err is 0
 * when bit-exact.  Exercises the 8-rank kernel on a 2- or 4-GPU box. */
dsx_status dsx_p2p_average_selftest(int nranks, long long n, double* max_abs_err);

/* Number of kernel launches issued by this lab since creation. */
dsx_status dsx_lab_launch_count(dsx_lab* lab, uint64_t* out);

#ifdef __cplusplus
}
#endif

#endif /* DREAMDDP_DSX_H_ */
