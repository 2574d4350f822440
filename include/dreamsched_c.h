/*
 * dreamsched_c.h — C entry points into the drop-in dreamsched:: C++ API
 * (libdreamsched.so) for non-C++ callers (the Python harness, ctypes).
 * Scheduling and profile I/O only: the training path is reached through the
 * C++ API itself or directly through dsx.h.
 *
 *   dsc_schedule_profile — load_profile (profile.cpp:154) -> schedule_dfs
 *                          (scheduler.cpp:171) -> bubble_fill (253) ->
 *                          write_schedule (schedule.cpp:209) text.
 *   dsc_profile_layers   — per-layer param_bytes / t_fp / t_bp of a profile.
 *   dsc_write_profile    — write_profile (profile.cpp:160) from measured
 *                          per-layer times (the CUDA-event profiler's output).
 *   dsc_compare_modes / dsc_simulate_trace — the simulator's predictions,
 *                          set beside the measured GPU timeline.
 *   dsc_synth_profile    — synth_profile (profile.cpp:188-228) saved as a
 *                          profile v1 file (the schedule sweep's inputs).
 */
#ifndef DREAMDDP_DREAMSCHED_C_H_
#define DREAMDDP_DREAMSCHED_C_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* dsc_last_error(void);
/* Returns 0, or 1 (dreamsched::Error) / 2 (other) with dsc_last_error set.
 * out receives the NUL-terminated schedule file text; *objective the period
 * objective of the filled schedule; *explored the DFS |Omega|. */
int dsc_schedule_profile(const char* profile_path, int period, int fill, char* out, size_t cap,
                         double* objective, uint64_t* explored);
/* Fills up to cap entries; *count receives the layer count. */
int dsc_profile_layers(const char* profile_path, uint64_t* param_bytes, double* t_fp,
                       double* t_bp, int cap, int* count);
int dsc_write_profile(const char* path, int layers, const char* const* names,
                      const uint64_t* param_bytes, const double* t_fp, const double* t_bp,
                      const double* t_comm /* nullable: link model */, double bandwidth,
                      double latency);

/* compare_modes (simulator.cpp:212-229): the four-mode report text. */
int dsc_compare_modes(const char* profile_path, int period, long long iters, char* out, size_t cap);
/* simulate_run (simulator.cpp:76-184) of one mode (plsgd: the DFS + fill
 * schedule) -> trace-event JSON text and the makespan. */
int dsc_simulate_trace(const char* profile_path, const char* mode, int period, long long iters,
                       char* out, size_t cap, double* makespan);
/* synth_profile(layers, seed, regime "balanced" | "comm-heavy" |
 * "compute-heavy") -> save_profile(path). */
int dsc_synth_profile(const char* path, int layers, uint64_t seed, const char* regime);

#ifdef __cplusplus
}
#endif

#endif /* DREAMDDP_DREAMSCHED_C_H_ */
