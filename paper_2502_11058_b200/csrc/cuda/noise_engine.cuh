// noise_engine.cuh — parallel, stream-exact reproduction of the reference's
// per-worker gradient noise (std::mt19937_64 + std::normal_distribution,
// trainer.cpp:179-183) on sm_100a.
//
// A worker's step consumes a contiguous run of its Mersenne-twister stream;
// how long the run is depends on the polar method's rejections, i.e. on the
// stream itself (never on the parameters).  The engine cuts the run into P
// segments of S outputs (S a multiple of 312), reaches each segment's start
// state with an MT19937-64 jump-ahead — W_{1+J} = sum_i c_i W_{1+i} over
// GF(2) with c = x^J mod phi, phi the characteristic polynomial of the
// twister (computed once by Berlekamp-Massey on the host) — and lets one CTA
// per segment generate, accept/reject and transform its attempts.  A
// finisher scans the per-segment accepted-pair counts, pins the exact attempt
// that produces normal dim-1, and writes back the worker's new
// (x[312], cursor) state.  The update kernel maps coordinate i -> (segment,
// slot) through the scanned counts.  Every accept/reject and every stream
// position is bit-identical to libstdc++; see mt_engine.cuh for the per-draw
// arithmetic.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace dsx {

struct NoiseView {
  const double* slots;              // [kl][P+1][cap]
  const unsigned long long* pfx;    // [kl][P+2] exclusive pair prefix per segment
  long long cap;                    // slot capacity (doubles)
  int P;                            // segments (slot P = overflow)
  unsigned long long base;          // first pair of this step in the run's stream
  int raw;                          // slots hold accepted attempts (x, y), not normals
  double stddev;                    // for the consumer-side transform (raw)
};

class NoiseEngine {
 public:
  // dim: normals per worker per step; kl: local workers; nsm: SM count;
  // max_steps: the longest batch one run generates (1 or a larger T).
  NoiseEngine() = default;
  ~NoiseEngine();
  bool init(unsigned long long dim, int kl, int nsm, int max_steps, std::string* err);
  // Generates `steps` (1 or max_steps) consecutive steps' noise for all local
  // workers from the states mt_src[kl][313] into buffer set `set` (0/1,
  // double-buffered so the next batch is produced while updates read the
  // other set) and writes the state after each step t to
  // mt_dst[t][kl][313].  One run pays the jump-ahead once for all its steps.
  bool run(const uint64_t* mt_src, uint64_t* mt_dst, int set, int steps, double stddev, void* stream,
           std::string* err);
  // Noise of step t (< steps of the set's last run).
  NoiseView view(int set, int t) const {
    const Cfg& c = cfg_[set_cfg_[set]];
    return {slots_ + (long long)set * slot_stride_, pfx_ + (long long)set * pfx_stride_, c.cap, c.P,
            (unsigned long long)t * ((dim_ + 1) / 2), raw_[set], stddev_[set]};
  }
  int max_steps() const { return cfg_[1].steps; }
  int segments(int steps = 1) const { return cfg_[steps > 1 ? 1 : 0].P; }
  long long segment_outputs(int steps = 1) const { return cfg_[steps > 1 ? 1 : 0].S; }
  uint64_t launches() const { return launches_; }

 private:
  struct Cfg {
    int steps = 1, P = 1, gens = 1, nck = 1;
    long long S = 0, cap = 0;
    uint32_t* jbits = nullptr;     // [P-1][kJumpBits/32+1] bitsets of c_s = x^(sS-1) mod phi
  };
  bool make_cfg(int steps, int nsm, Cfg* c, std::string* err);
  unsigned long long dim_ = 0;
  int kl_ = 0, ck_every_ = 16, seg_r_ = 4;
  Cfg cfg_[2];                     // [0]: one step per run, [1]: max_steps per run
  int set_cfg_[2] = {0, 0};
  int raw_[2] = {0, 0};            // per set: the last run stored raw attempts
  double stddev_[2] = {0.0, 0.0};
  long long slot_stride_ = 0, pfx_stride_ = 0;
  uint64_t* ybuf_ = nullptr;       // [kl][kPrefixWords]
  uint64_t* win_ = nullptr;        // [kl][P][312]
  int* joff_ = nullptr;            // [2][kl] normalized cursors
  double* slots_ = nullptr;        // [2][kl][P+1][cap]
  unsigned long long* cnt_ = nullptr;  // [2][kl][P]
  unsigned long long* pfx_ = nullptr;  // [2][kl][P+2]
  uint64_t* ck_ = nullptr;         // [kl][P][nck][kCkWords]
  uint64_t* tail_ = nullptr;       // [kl][P][kCkWords] segment end states
  int* status_ = nullptr;          // [2][steps][kl] 0 ok, else overflow failure
  uint64_t launches_ = 0;
};

// Host-side MT19937-64 jump machinery (exposed for the CPU self-test).
// Characteristic polynomial phi (degree 19937) as 312 little-endian words.
const std::vector<uint64_t>& mt_char_poly();
// c = x^J mod phi.
std::vector<uint64_t> mt_jump_poly(unsigned long long J);
// Applies c to the window starting at Y[1] of a sequence whose first 312
// words are x (generation-aligned state): returns Y[1+J .. 1+J+311].
std::vector<uint64_t> mt_jump_host(const uint64_t* x312, const std::vector<uint64_t>& c);

}  // namespace dsx
