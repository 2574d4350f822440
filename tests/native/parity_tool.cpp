// parity_tool — one driver source compiled twice: against the reference
// library (oracle/_ref/parity_tool_ref, via oracle/Makefile) and against this
// framework's drop-in library (build/parity_tool).  It uses only the public
// dreamsched:: API (reference headers core/include/dreamsched/*.hpp), so the
// fact that it compiles against both is itself the API-compatibility check,
// and byte-identical stdout between the two builds is the parity check.
//
// Test infrastructure: not part of the product.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "dreamsched/cost_model.hpp"
#include "dreamsched/errors.hpp"
#include "dreamsched/profile.hpp"
#include "dreamsched/schedule.hpp"
#include "dreamsched/scheduler.hpp"
#include "dreamsched/simulator.hpp"
#include "dreamsched/text_format.hpp"
#include "dreamsched/trainer.hpp"

using namespace dreamsched;

namespace {

std::uint64_t fnv(const std::string& s) {
  std::uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

const char* rule_char(AssignRule r) {
  switch (r) {
    case AssignRule::kAtLeastOne: return "A";
    case AssignRule::kOptimalHiding: return "H";
    case AssignRule::kDelayedCo: return "D";
    case AssignRule::kDfsBranch: return "B";
  }
  return "?";
}

// Same contiguous random partition generator as the reference's
// tests/support/instance_gen.hpp (restated so this file needs no test headers).
Schedule random_partition(int layer_count, int period, std::mt19937_64& rng) {
  Schedule s;
  s.period = period;
  s.sets.assign(static_cast<std::size_t>(period), {});
  s.supplemental.assign(static_cast<std::size_t>(period), {});
  const int used = 1 + static_cast<int>(rng() % static_cast<std::uint64_t>(std::min(period, layer_count)));
  std::vector<int> cuts;
  while (static_cast<int>(cuts.size()) < used - 1) {
    const int c = 1 + static_cast<int>(rng() % static_cast<std::uint64_t>(layer_count - 1));
    bool dup = false;
    for (int x : cuts) dup |= x == c;
    if (!dup) cuts.push_back(c);
  }
  std::sort(cuts.begin(), cuts.end());
  int layer = layer_count;
  for (int j = 0; j < used; ++j) {
    const int low = (j + 1 < used) ? cuts[static_cast<std::size_t>(used - 2 - j)] : 0;
    while (layer > low) s.sets[static_cast<std::size_t>(j)].push_back(layer--);
  }
  return s;
}

void report_schedule_case(const ModelProfile& profile, int period, bool brute) {
  const SearchReport dfs = schedule_dfs(profile, period);
  std::string rules;
  for (const auto& d : dfs.classification_log) {
    rules += rule_char(d.rule);
    rules += std::to_string(d.layer) + "/" + std::to_string(d.iteration) + " ";
  }
  std::cout << "dfs_cost=" << format_real(dfs.best_cost) << " explored=" << dfs.solutions_explored
            << " log=" << dfs.classification_log.size() << " loghash=" << fnv(rules) << "\n";
  const Schedule filled = bubble_fill(dfs.best, profile);
  write_schedule(filled, std::cout);
  write_cost_report(period_objective(filled, profile), std::cout);
  if (brute && brute_force_candidate_count(profile.layer_count(), period) <= 200000) {
    const SearchReport bf = schedule_brute_force(profile, period);
    std::cout << "bf_cost=" << format_real(bf.best_cost) << " candidates=" << bf.solutions_explored
              << "\n";
    write_schedule(bf.best, std::cout);
  }
  const long long iters = 2 * period + 1;
  for (Mode m : {Mode::kSsgd, Mode::kWfbp, Mode::kFlsgd, Mode::kPlsgd}) {
    const auto tl = simulate_run(profile, m, m == Mode::kPlsgd ? std::optional<Schedule>(filled)
                                                               : std::nullopt,
                                 iters, period);
    std::cout << mode_name(m) << "_makespan=" << format_real(tl.makespan)
              << " events=" << tl.events.size() << "\n";
  }
  std::cout << "t_ssgd=" << format_real(t_ssgd_total(profile, 1000))
            << " t_lsgd=" << format_real(t_lsgd_total(profile, 1000, period))
            << " saved=" << format_real(saved_ratio(profile, period)) << "\n";
}

int cmd_sched_fuzz(std::uint64_t seed, int count, int max_layers) {
  std::mt19937_64 rng(seed);
  for (int i = 0; i < count; ++i) {
    const int layers = 1 + static_cast<int>(rng() % static_cast<std::uint64_t>(max_layers));
    const int period = 1 + static_cast<int>(rng() % static_cast<std::uint64_t>(std::min(layers, 8)));
    const auto regime = static_cast<Regime>(rng() % 3);
    const std::uint64_t pseed = rng();
    const ModelProfile profile = synth_profile(layers, pseed, regime);
    std::ostringstream ptxt;
    write_profile(profile, ptxt);
    std::cout << "# case " << i << " L=" << layers << " H=" << period << " "
              << profile.label << " profile_hash=" << fnv(ptxt.str()) << "\n";
    report_schedule_case(profile, period, true);
    // random partitions + fills through the closed form, the simulator and bubble fill
    Schedule rp = random_partition(layers, period, rng);
    const Schedule rpf = bubble_fill(rp, profile);
    write_schedule(rpf, std::cout);
    const auto pc = period_objective(rpf, profile);
    const auto tl = simulate_run(profile, Mode::kPlsgd, rpf, period);
    std::cout << "rp_objective=" << format_real(pc.objective)
              << " rp_total=" << format_real(pc.total_with_fp)
              << " rp_sim=" << format_real(tl.makespan) << "\n";
  }
  return 0;
}

int cmd_profile(const std::string& path, int period) {
  const ModelProfile profile = load_profile(path);
  write_profile(profile, std::cout);
  report_schedule_case(profile, period, false);
  return 0;
}

int cmd_trace(const std::string& path, const std::string& mode, int period, long long iters) {
  const ModelProfile profile = load_profile(path);
  const Mode m = parse_mode(mode);
  std::optional<Schedule> sched;
  if (m == Mode::kPlsgd) sched = bubble_fill(schedule_dfs(profile, period).best, profile);
  const Timeline tl = simulate_run(profile, m, sched, iters, period);
  write_trace(tl, std::cout);
  write_mode_report(compare_modes(profile, period, iters), std::cout);
  return 0;
}

// synth_profile (profile.cpp:188-228) for every regime, then its DFS + fill
// schedule: the schedule sweep's inputs.
int cmd_synth(int l_count, unsigned long long seed) {
  for (const char* regime : {"balanced", "comm-heavy", "compute-heavy"}) {
    const ModelProfile p = synth_profile(l_count, seed, parse_regime(regime));
    write_profile(p, std::cout);
    for (int h : {2, 4, 8}) {
      if (h > l_count) continue;
      const Schedule s = bubble_fill(schedule_dfs(p, h).best, p);
      write_schedule(s, std::cout);
    }
  }
  return 0;
}

// Builds the lab problem: either make_quadratic(dim, blocks, ...) or, when
// `profile` is non-empty, one block per profile layer sized param_bytes/4
// (min 1) with make_quadratic's evenly spread curvature.
Problem lab_problem(std::size_t dim, int blocks, double sigma, const std::string& profile) {
  if (profile.empty()) return make_quadratic(dim, blocks, 1.0, 2.0, sigma);
  const ModelProfile p = load_profile(profile);
  std::vector<std::size_t> sizes;
  std::size_t total = 0;
  for (const auto& l : p.layers) {
    const std::size_t n = std::max<std::size_t>(1, l.param_bytes.value_or(0) / 4);
    sizes.push_back(n);
    total += n;
  }
  Problem q = make_quadratic(total, static_cast<int>(sizes.size()), 1.0, 2.0, sigma);
  q.block_sizes = sizes;
  q.validate();
  return q;
}

TrainerConfig lab_config(const Problem& problem, int workers, int period, std::uint64_t seed,
                         const std::string& mode, const std::string& schedule,
                         const std::string& profile) {
  TrainerConfig c;
  c.workers = workers;
  c.period = period;
  c.seed = seed;
  c.mode = mode == "full" ? SyncMode::kFull : mode == "ssgd" ? SyncMode::kSsgdEvery
                                                               : SyncMode::kPartial;
  if (schedule == "enp") {
    c.schedule = Schedule::equal_number_partition(problem.layer_count(), period);
  } else if (schedule == "dfs") {
    const ModelProfile p = load_profile(profile);
    c.schedule = bubble_fill(schedule_dfs(p, period).best, p);
  } else if (schedule == "single") {
    c.schedule = Schedule::single_set(problem.layer_count());
  } else {
    c.schedule = load_schedule(schedule);
  }
  return c;
}

// Runs R plsgd_step calls from zeros and prints every worker parameter,
// the rng states and the per-step max ||g||^2.
int cmd_steps(int argc, char** argv) {
  // steps dim blocks K H sigma seed R mode schedule [profile]
  if (argc < 11) return 2;
  const std::size_t dim = std::strtoull(argv[2], nullptr, 10);
  const int blocks = std::atoi(argv[3]);
  const int K = std::atoi(argv[4]);
  const int H = std::atoi(argv[5]);
  const double sigma = std::atof(argv[6]);
  const std::uint64_t seed = std::strtoull(argv[7], nullptr, 10);
  const long long R = std::atoll(argv[8]);
  const std::string mode = argv[9], schedule = argv[10];
  const std::string profile = argc > 11 ? argv[11] : "";
  const Problem problem = lab_problem(dim, blocks, sigma, profile);
  TrainerConfig config = lab_config(problem, K, H, seed, mode, schedule, profile);
  config.iterations = R;
  config.validate(problem);
  std::vector<WorkerState> workers(static_cast<std::size_t>(K));
  for (int k = 0; k < K; ++k) {
    workers[static_cast<std::size_t>(k)].w.assign(problem.dim, 0.0);
    workers[static_cast<std::size_t>(k)].rng = worker_rng(seed, k);
  }
  for (long long r = 0; r < R; ++r) {
    StepStats stats;
    plsgd_step(workers, r, config, problem, &stats);
    std::cout << "r=" << r << " eta=" << format_real(config.learning_rate(r, problem))
              << " max_g2=" << format_real(stats.max_grad_norm_sq) << "\n";
  }
  for (int k = 0; k < K; ++k) {
    std::cout << "w" << k;
    for (double v : workers[static_cast<std::size_t>(k)].w) std::cout << ' ' << format_real(v);
    std::cout << "\nrng" << k << ' ' << workers[static_cast<std::size_t>(k)].rng << "\n";
  }
  return 0;
}

// Parses the reference CLI's flat key=value train file (dreamsched_main.cpp
// semantics) and prints run_training's summary + divergence CSV.
int cmd_train(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw IoError("cannot open " + path);
  std::map<std::string, std::string> kv;
  std::string line;
  while (std::getline(in, line)) {
    const auto hash = line.find('#');
    if (hash != std::string::npos) line.resize(hash);
    const auto text = trim(line);
    if (text.empty()) continue;
    const auto eq = text.find('=');
    kv[std::string(trim(text.substr(0, eq)))] = std::string(trim(text.substr(eq + 1)));
  }
  auto get = [&](const char* k, const char* dflt) {
    auto it = kv.find(k);
    return it == kv.end() ? std::string(dflt) : it->second;
  };
  const std::size_t dim = parse_u64_field(get("dim", "0"), "dim");
  const int period = static_cast<int>(parse_u64_field(get("period", "1"), "period"));
  const int blocks = static_cast<int>(parse_u64_field(get("blocks", std::to_string(period).c_str()), "blocks"));
  const std::string opt = get("optimum", "ones");
  const double optimum = opt == "ones" ? 1.0 : opt == "zeros" ? 0.0 : parse_real_field(opt, "optimum");
  const Problem problem = make_quadratic(dim, blocks, parse_real_field(get("lambda_min", "1.0"), "l"),
                                         parse_real_field(get("lambda_max", "2.0"), "l"),
                                         parse_real_field(get("sigma", "0.0"), "s"), optimum);
  TrainerConfig c;
  c.workers = static_cast<int>(parse_u64_field(get("workers", "1"), "workers"));
  c.period = period;
  c.iterations = static_cast<long long>(parse_u64_field(get("iters", "0"), "iters"));
  c.lr = get("lr", "decaying") == "constant" ? LrSchedule::kConstant : LrSchedule::kDecaying;
  c.eta = parse_real_field(get("eta", "0.0"), "eta");
  c.shift_a = parse_real_field(get("shift_a", "0.0"), "shift_a");
  c.seed = parse_u64_field(get("seed", "0"), "seed");
  c.log_stride = static_cast<long long>(parse_u64_field(get("log_stride", "1"), "log_stride"));
  const std::string mode = get("mode", "partial");
  c.mode = mode == "full" ? SyncMode::kFull : mode == "ssgd" ? SyncMode::kSsgdEvery : SyncMode::kPartial;
  const std::string sk = get("schedule", "enp");
  c.schedule = sk == "enp" ? Schedule::equal_number_partition(blocks, period)
               : sk == "single" ? Schedule::single_set(blocks) : load_schedule(sk);
  const DivergenceTrace trace = run_training(c, problem);
  write_run_summary(trace, std::cout);
  write_divergence_csv(trace, std::cout);
  return 0;
}

// Per-call latency of the host-state API on a tiny problem (the shape of
// the reference acceptance criterion 6): microseconds per call.
int cmd_apibench() {
  const Problem problem = make_quadratic(64, 4, 1.0, 2.0, 1.0);
  TrainerConfig config;
  config.workers = 4;
  config.period = 1;
  config.schedule = Schedule::single_set(4);
  config.seed = 7;
  std::vector<WorkerState> workers(4);
  for (int k = 0; k < 4; ++k) {
    workers[static_cast<std::size_t>(k)].w.assign(64, 0.0);
    workers[static_cast<std::size_t>(k)].rng = worker_rng(7, k);
  }
  std::vector<double> ref(64, 0.0);
  std::mt19937_64 stream = worker_rng(7, 0);
  plsgd_step(workers, 0, config, problem);  // warm (creates the device state)
  (void)stochastic_gradient(problem, ref, stream);
  auto t0 = std::chrono::steady_clock::now();
  for (long long r = 1; r <= 100; ++r) plsgd_step(workers, r, config, problem);
  auto t1 = std::chrono::steady_clock::now();
  for (int i = 0; i < 100; ++i) (void)stochastic_gradient(problem, ref, stream);
  auto t2 = std::chrono::steady_clock::now();
  std::printf("{\"plsgd_step_us\": %.1f, \"stochastic_gradient_us\": %.1f}\n",
              std::chrono::duration<double, std::micro>(t1 - t0).count() / 100.0,
              std::chrono::duration<double, std::micro>(t2 - t1).count() / 100.0);
  return 0;
}

// CPU timing of plsgd_step: one JSON line.
int cmd_bench(int argc, char** argv) {
  // bench dim blocks K H sigma seed steps warmup mode schedule [profile]
  if (argc < 12) return 2;
  const std::size_t dim = std::strtoull(argv[2], nullptr, 10);
  const int blocks = std::atoi(argv[3]);
  const int K = std::atoi(argv[4]);
  const int H = std::atoi(argv[5]);
  const double sigma = std::atof(argv[6]);
  const std::uint64_t seed = std::strtoull(argv[7], nullptr, 10);
  const int steps = std::atoi(argv[8]);
  const int warmup = std::atoi(argv[9]);
  const std::string mode = argv[10], schedule = argv[11];
  const std::string profile = argc > 12 ? argv[12] : "";
  const Problem problem = lab_problem(dim, blocks, sigma, profile);
  TrainerConfig config = lab_config(problem, K, H, seed, mode, schedule, profile);
  config.iterations = steps + warmup;
  config.validate(problem);
  std::vector<WorkerState> workers(static_cast<std::size_t>(K));
  for (int k = 0; k < K; ++k) {
    workers[static_cast<std::size_t>(k)].w.assign(problem.dim, 0.0);
    workers[static_cast<std::size_t>(k)].rng = worker_rng(seed, k);
  }
  long long r = 0;
  for (; r < warmup; ++r) plsgd_step(workers, r, config, problem);
  const auto t0 = std::chrono::steady_clock::now();
  for (int s = 0; s < steps; ++s, ++r) plsgd_step(workers, r, config, problem);
  const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  double checksum = 0.0;
  for (const auto& w : workers) for (double v : w.w) checksum += v;
  // Parity digest of the state after warmup + steps iterations, per worker:
  // sequential sum and sum of squares of w, 64 strided samples of w, and the
  // FNV-1a 64 hash of the rng state's text form (operator<<: 312 words + p).
  std::string digest = "[";
  for (int k = 0; k < K; ++k) {
    const auto& w = workers[static_cast<std::size_t>(k)].w;
    double s1 = 0.0, s2 = 0.0;
    for (double v : w) {
      s1 += v;
      s2 += v * v;
    }
    std::ostringstream ss;
    ss << workers[static_cast<std::size_t>(k)].rng;
    const std::string text = ss.str();
    std::uint64_t h = 1469598103934665603ull;
    for (unsigned char ch : text) {
      h ^= ch;
      h *= 1099511628211ull;
    }
    char buf[128];
    digest += (k ? ", " : "");
    std::snprintf(buf, sizeof buf, "{\"sum\": %.17g, \"sumsq\": %.17g, \"rng_fnv\": \"%016llx\", \"samples\": [",
                  s1, s2, static_cast<unsigned long long>(h));
    digest += buf;
    for (int j = 0; j < 64; ++j) {
      const std::size_t i = static_cast<std::size_t>(j) * (w.size() - 1) / 63;
      std::snprintf(buf, sizeof buf, "%s%.17g", j ? ", " : "", w[i]);
      digest += buf;
    }
    digest += "]}";
  }
  digest += "]";
  std::printf("{\"steps\": %d, \"seconds\": %.6f, \"it_per_s\": %.6f, \"dim\": %zu, \"workers\": %d, "
              "\"blocks\": %d, \"period\": %d, \"sigma\": %g, \"checksum\": %.17g, \"total_steps\": %lld, "
              "\"digest\": %s}\n",
              steps, sec, steps / sec, problem.dim, K, problem.layer_count(), H, sigma, checksum, r,
              digest.c_str());
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "usage: parity_tool sched-fuzz|profile|trace|steps|train|bench ...\n";
    return 2;
  }
  const std::string cmd = argv[1];
  try {
    if (cmd == "sched-fuzz" && argc >= 5)
      return cmd_sched_fuzz(std::strtoull(argv[2], nullptr, 10), std::atoi(argv[3]), std::atoi(argv[4]));
    if (cmd == "profile" && argc >= 4) return cmd_profile(argv[2], std::atoi(argv[3]));
    if (cmd == "trace" && argc >= 6) return cmd_trace(argv[2], argv[3], std::atoi(argv[4]), std::atoll(argv[5]));
    if (cmd == "steps") return cmd_steps(argc, argv);
    if (cmd == "synth" && argc >= 4) return cmd_synth(std::atoi(argv[2]), std::strtoull(argv[3], nullptr, 10));
    if (cmd == "train" && argc >= 3) return cmd_train(argv[2]);
    if (cmd == "bench") return cmd_bench(argc, argv);
    if (cmd == "apibench") return cmd_apibench();
  } catch (const Error& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  } catch (const std::exception& e) {
    std::cerr << "internal error: " << e.what() << "\n";
    return 2;
  }
  std::cerr << "bad command\n";
  return 2;
}
