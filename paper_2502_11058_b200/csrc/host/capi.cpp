// C entry points of libdreamsched.so (include/dreamsched_c.h).
#include "dreamsched_c.h"

#include <cstring>
#include <optional>
#include <sstream>
#include <string>

#include "dreamsched/cost_model.hpp"
#include "dreamsched/errors.hpp"
#include "dreamsched/profile.hpp"
#include "dreamsched/schedule.hpp"
#include "dreamsched/scheduler.hpp"
#include "dreamsched/simulator.hpp"

namespace {
thread_local std::string g_error;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const dreamsched::Error& e) {
    g_error = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_error = e.what();
    return 2;
  }
}
}  // namespace

extern "C" {

const char* dsc_last_error(void) { return g_error.c_str(); }

int dsc_schedule_profile(const char* profile_path, int period, int fill, char* out, size_t cap,
                         double* objective, uint64_t* explored) {
  return guarded([&] {
    const dreamsched::ModelProfile profile = dreamsched::load_profile(profile_path);
    const dreamsched::SearchReport rep = dreamsched::schedule_dfs(profile, period);
    const dreamsched::Schedule s = fill ? dreamsched::bubble_fill(rep.best, profile) : rep.best;
    std::ostringstream text;
    dreamsched::write_schedule(s, text);
    const std::string t = text.str();
    if (t.size() + 1 > cap) throw dreamsched::ArgumentError("schedule text buffer too small");
    std::memcpy(out, t.c_str(), t.size() + 1);
    if (objective) *objective = dreamsched::period_objective(s, profile).objective;
    if (explored) *explored = rep.solutions_explored;
  });
}

int dsc_profile_layers(const char* profile_path, uint64_t* param_bytes, double* t_fp, double* t_bp,
                       int cap, int* count) {
  return guarded([&] {
    const dreamsched::ModelProfile p = dreamsched::load_profile(profile_path);
    *count = p.layer_count();
    for (int i = 0; i < p.layer_count() && i < cap; ++i) {
      const auto& l = p.layers[static_cast<std::size_t>(i)];
      if (param_bytes) param_bytes[i] = l.param_bytes.value_or(0);
      if (t_fp) t_fp[i] = l.t_fp;
      if (t_bp) t_bp[i] = l.t_bp;
    }
  });
}

int dsc_write_profile(const char* path, int layers, const char* const* names,
                      const uint64_t* param_bytes, const double* t_fp, const double* t_bp,
                      const double* t_comm, double bandwidth, double latency) {
  return guarded([&] {
    dreamsched::ModelProfile p;
    p.label = path;
    for (int i = 0; i < layers; ++i) {
      dreamsched::LayerProfile l;
      l.index = i + 1;
      l.name = names ? names[i] : "layer" + std::to_string(i + 1);
      l.param_bytes = param_bytes[i];
      l.t_fp = t_fp[i];
      l.t_bp = t_bp[i];
      if (t_comm) l.t_comm_override = t_comm[i];
      p.layers.push_back(l);
    }
    p.link = {bandwidth, latency};
    p.validate();
    dreamsched::save_profile(p, path);
  });
}

int dsc_synth_profile(const char* path, int layers, uint64_t seed, const char* regime) {
  return guarded([&] {
    const dreamsched::ModelProfile p =
        dreamsched::synth_profile(layers, seed, dreamsched::parse_regime(regime ? regime : "balanced"));
    dreamsched::save_profile(p, path);
  });
}

namespace {
void copy_out(const std::string& t, char* out, size_t cap) {
  if (t.size() + 1 > cap) throw dreamsched::ArgumentError("output buffer too small");
  std::memcpy(out, t.c_str(), t.size() + 1);
}
}  // namespace

int dsc_compare_modes(const char* profile_path, int period, long long iters, char* out, size_t cap) {
  return guarded([&] {
    const dreamsched::ModelProfile profile = dreamsched::load_profile(profile_path);
    std::ostringstream text;
    dreamsched::write_mode_report(dreamsched::compare_modes(profile, period, iters), text);
    copy_out(text.str(), out, cap);
  });
}

int dsc_simulate_trace(const char* profile_path, const char* mode, int period, long long iters,
                       char* out, size_t cap, double* makespan) {
  return guarded([&] {
    const dreamsched::ModelProfile profile = dreamsched::load_profile(profile_path);
    const dreamsched::Mode m = dreamsched::parse_mode(mode);
    std::optional<dreamsched::Schedule> sched;
    if (m == dreamsched::Mode::kPlsgd)
      sched = dreamsched::bubble_fill(dreamsched::schedule_dfs(profile, period).best, profile);
    const dreamsched::Timeline tl = dreamsched::simulate_run(profile, m, sched, iters, period);
    std::ostringstream text;
    dreamsched::write_trace(tl, text);
    copy_out(text.str(), out, cap);
    if (makespan) *makespan = tl.makespan;
  });
}

}  // extern "C"
