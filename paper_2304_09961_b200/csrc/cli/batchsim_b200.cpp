// Command-line front end with the reference CLI's subcommands, flags, output
// formats and exit codes (proj/tools/batchsim_main.cpp:434-496):
//
//   batchsim_b200 simulate        --profile P [sim flags] [--out outcomes.csv]
//   batchsim_b200 sweep-capacity  --profile P [sim flags] --rates lo:hi:step --schedulers a,b --seeds N [--out f]
//   batchsim_b200 validate-profile P
//   batchsim_b200 oracle-check    [--instances N] [--seed S] [--max-requests M] [--bounded] [--what W]
//
// The profile is any reference-schema table, in particular the h_k(b) tables
// measured on the B200 (tools/profile_latency.py), so a B200 latency table can
// be simulated, swept and validated exactly like the reference's synthetic
// ones. Exit codes: 0 success, 1 oracle failure, 2 usage or configuration error.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include <json.hpp>

#include "bsb/report.hpp"
#include "bsb/schedulers.hpp"
#include "bsb/selfcheck.hpp"
#include "bsb/server.hpp"

namespace {

using namespace batchsim;

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// --name value pairs (and bare flags) after the subcommand.
struct Args {
  std::map<std::string, std::string> opt;
  std::vector<std::string> positional;
  bool has(const std::string& k) const { return opt.count(k) != 0; }
  std::string str(const std::string& k, const std::string& dflt) const {
    auto it = opt.find(k);
    return it == opt.end() ? dflt : it->second;
  }
  double num(const std::string& k, double dflt) const { return has(k) ? std::stod(opt.at(k)) : dflt; }
  long long integer(const std::string& k, long long dflt) const { return has(k) ? std::stoll(opt.at(k)) : dflt; }
};

Args parse_args(int argc, char** argv, int first, const std::vector<std::string>& flags,
                const std::vector<std::string>& valued) {
  Args a;
  auto known = [](const std::vector<std::string>& v, const std::string& s) {
    return std::find(v.begin(), v.end(), s) != v.end();
  };
  for (int i = first; i < argc; ++i) {
    const std::string s = argv[i];
    if (s.rfind("--", 0) != 0) {
      a.positional.push_back(s);
      continue;
    }
    std::string key = s, val;
    if (const auto eq = s.find('='); eq != std::string::npos) {
      key = s.substr(0, eq);
      val = s.substr(eq + 1);
    }
    if (known(flags, key)) {
      a.opt[key] = "1";
    } else if (known(valued, key)) {
      if (val.empty()) {
        if (i + 1 >= argc) throw UsageError(key + " needs a value");
        val = argv[++i];
      }
      a.opt[key] = val;
    } else {
      throw UsageError("unknown option " + key);
    }
  }
  return a;
}

const std::vector<std::string> kSimFlags = {
    "--profile", "--workload", "--scheduler", "--process", "--rate", "--requests", "--deadline-ms", "--seed",
    "--trace", "--trace-scale", "--size-trace", "--clients", "--offload", "--client-profile", "--partial-rule",
    "--granularity", "--groups", "--max-batch", "--sched-latency-ms", "--step-overhead-ms", "--out"};

std::string resolve_profile(const std::string& arg) {
  namespace fs = std::filesystem;
  if (fs::exists(arg) || arg.find('/') != std::string::npos) return arg;
  if (const char* dir = std::getenv("BATCHSIM_PROFILE_DIR")) {
    const std::string c = std::string(dir) + "/" + arg + (arg.ends_with(".json") ? "" : ".json");
    if (fs::exists(c)) return c;
  }
  return arg;
}

// Workload JSON fields mirror the flags; flags given on the command line win
// (tools/batchsim_main.cpp:107-128).
void merge_workload(Args& a, std::vector<std::pair<std::string, double>>& mix) {
  if (!a.has("--workload")) return;
  std::ifstream in(a.str("--workload", ""));
  if (!in) throw std::runtime_error("cannot open workload file: " + a.str("--workload", ""));
  nlohmann::json doc;
  in >> doc;
  const std::map<std::string, std::string> fields = {
      {"process", "--process"}, {"rate", "--rate"},       {"requests", "--requests"}, {"deadline_ms", "--deadline-ms"},
      {"seed", "--seed"},       {"clients", "--clients"}, {"offload", "--offload"},   {"scheduler", "--scheduler"}};
  for (const auto& [field, flag] : fields) {
    if (!doc.contains(field) || a.has(flag)) continue;
    const auto& v = doc[field];
    a.opt[flag] = v.is_string() ? v.get<std::string>() : v.dump();
  }
  if (doc.contains("dnn_mix"))
    for (const auto& [name, frac] : doc["dnn_mix"].items()) mix.emplace_back(name, frac.get<double>());
}

WorkloadSpec make_spec(const Args& a, const std::vector<std::pair<std::string, double>>& mix) {
  WorkloadSpec s;
  s.process = parse_process(a.str("--process", "poisson"));
  s.rate = a.num("--rate", 100.0);
  s.count = static_cast<int>(a.integer("--requests", 5000));
  const double d = a.num("--deadline-ms", 0.0);
  s.relative_deadline = d > 0 ? d : kNoDeadline;
  s.seed = static_cast<std::uint64_t>(a.integer("--seed", 1));
  s.dnn_mix = mix;
  if (a.has("--size-trace")) s.size_trace = load_size_trace(a.str("--size-trace", ""));
  return s;
}

SimConfig make_config(const Args& a, const std::string& scheduler) {
  SimConfig c;
  c.scheduler = parse_scheduler(scheduler);
  const std::string g = a.str("--granularity", "group");
  if (g == "request") c.granularity = SplitGranularity::per_request;
  else if (g == "layer") c.granularity = SplitGranularity::per_layer;
  else if (g == "group") c.granularity = SplitGranularity::per_group;
  else throw std::runtime_error("unknown granularity '" + g + "'");
  c.groups = static_cast<int>(a.integer("--groups", 5));
  c.max_batch = static_cast<int>(a.integer("--max-batch", 90));
  c.scheduler_latency = a.num("--sched-latency-ms", 0.0);
  c.step_overhead = a.num("--step-overhead-ms", 0.0);
  c.offload = parse_offload(a.str("--offload", "none"));
  c.clients = static_cast<int>(a.integer("--clients", 0));
  c.partial_rule =
      a.str("--partial-rule", "min-completion") == "first-hide-wait" ? PartialRule::first_hide_wait : PartialRule::min_completion;
  return c;
}

std::optional<NetworkTrace> trace_of(const Args& a) {
  if (!a.has("--trace")) return std::nullopt;
  NetworkTrace t = load_trace(a.str("--trace", ""));
  const double scale = a.num("--trace-scale", 1.0);
  return scale != 1.0 ? scale_trace(t, scale) : t;
}

std::optional<ClientProfile> client_of(const Args& a) {
  if (!a.has("--client-profile")) return std::nullopt;
  return load_client_profile(a.str("--client-profile", ""));
}

std::string summary_path(const std::string& out) {
  const auto dot = out.rfind('.');
  return (dot == std::string::npos ? out : out.substr(0, dot)) + ".summary.json";
}

void print_summary(const SummaryMetrics& m) {
  std::printf("generated            %d\n", m.generated);
  std::printf("completed            %d\n", m.completed);
  std::printf("dropped              %d\n", m.dropped);
  std::printf("on-time ratio        %.4f\n", m.on_time_ratio);
  std::printf("mean completion      %.3f ms\n", m.mean_completion);
  std::printf("median completion    %.3f ms\n", m.median_completion);
  std::printf("p95 completion       %.3f ms\n", m.p95_completion);
  std::printf("locations            server=%d client-full=%d client-partial=%d\n", m.at_server, m.at_client_full,
              m.at_client_partial);
  std::printf("schedules computed   %d (mean solve %.3f ms)\n", m.schedules_computed, m.mean_solve_wall_ms);
}

int cmd_simulate(Args a) {
  if (!a.has("--profile")) throw UsageError("--profile is required");
  std::vector<std::pair<std::string, double>> mix;
  merge_workload(a, mix);
  const ProfileSet ps = load_profile(resolve_profile(a.str("--profile", "")));
  const auto trace = trace_of(a);
  const auto client = client_of(a);
  const SimResult res = run_sim(make_spec(a, mix), ps, make_config(a, a.str("--scheduler", "ours-time")),
                                trace ? &*trace : nullptr, client ? &*client : nullptr);
  if (a.has("--out")) {
    const std::string out = a.str("--out", "");
    std::ofstream f(out);
    if (!f) throw std::runtime_error("cannot write " + out);
    write_outcomes_csv(f, res.outcomes, ps);
    std::ofstream sj(summary_path(out));
    sj << summary_json(res.metrics).dump(1) << "\n";
    std::printf("wrote %s and %s\n", out.c_str(), summary_path(out).c_str());
  }
  print_summary(res.metrics);
  return 0;
}

std::vector<double> parse_rates(const std::string& text) {
  std::vector<double> rates;
  if (const auto c1 = text.find(':'); c1 != std::string::npos) {
    const auto c2 = text.find(':', c1 + 1);
    const double lo = std::stod(text.substr(0, c1));
    const double hi = std::stod(text.substr(c1 + 1, c2 - c1 - 1));
    const double step = c2 == std::string::npos ? 10.0 : std::stod(text.substr(c2 + 1));
    if (step <= 0 || hi < lo) throw UsageError("--rates: bad lo:hi:step range");
    for (double r = lo; r <= hi + 1e-9; r += step) rates.push_back(r);
    return rates;
  }
  std::istringstream in(text);
  for (std::string tok; std::getline(in, tok, ',');) rates.push_back(std::stod(tok));
  if (rates.empty()) throw UsageError("--rates: no rates given");
  return rates;
}

int cmd_sweep(Args a) {
  if (!a.has("--profile")) throw UsageError("--profile is required");
  std::vector<std::pair<std::string, double>> mix;
  merge_workload(a, mix);
  const ProfileSet ps = load_profile(resolve_profile(a.str("--profile", "")));
  const auto trace = trace_of(a);
  const auto client = client_of(a);
  const std::vector<double> rates = parse_rates(a.str("--rates", "10:350:10"));
  const int seeds = static_cast<int>(a.integer("--seeds", 1));
  std::vector<std::string> scheds;
  {
    std::istringstream in(a.str("--schedulers", "ours-time"));
    for (std::string tok; std::getline(in, tok, ',');) scheds.push_back(tok);
  }
  auto mean_std = [&](const std::vector<double>& v) {
    double m = 0, s = 0;
    for (double x : v) m += x;
    m /= static_cast<double>(v.size());
    for (double x : v) s += (x - m) * (x - m);
    return std::pair<double, double>{m, v.size() > 1 ? std::sqrt(s / static_cast<double>(v.size() - 1)) : 0.0};
  };
  std::vector<SweepRow> rows;
  for (const std::string& sched : scheds) {
    const SimConfig config = make_config(a, sched);
    std::vector<std::vector<double>> ratio(rates.size()), completion(rates.size());
    for (int s = 0; s < seeds; ++s) {
      WorkloadSpec spec = make_spec(a, mix);
      spec.seed += static_cast<std::uint64_t>(s);
      const CapacityCurve curve =
          capacity_sweep(spec, rates, ps, config, trace ? &*trace : nullptr, client ? &*client : nullptr);
      for (std::size_t r = 0; r < rates.size(); ++r) {
        ratio[r].push_back(curve.points[r].metrics.on_time_ratio);
        completion[r].push_back(curve.points[r].metrics.mean_completion / 1000.0);
      }
    }
    std::optional<double> capacity;
    for (std::size_t r = 0; r < rates.size(); ++r) {
      SweepRow row;
      row.scheduler = sched;
      row.rate = rates[r];
      std::tie(row.ratio_mean, row.ratio_std) = mean_std(ratio[r]);
      std::tie(row.mean_completion_s_mean, row.mean_completion_s_std) = mean_std(completion[r]);
      if (row.ratio_mean >= kCapacityThreshold) capacity = capacity ? std::max(*capacity, rates[r]) : rates[r];
      rows.push_back(row);
    }
    if (capacity) std::printf("capacity[%s] = %g req/s\n", sched.c_str(), *capacity);
    else
      std::printf("capacity[%s] = none (on-time ratio below %.2f at every tested rate)\n", sched.c_str(),
                  kCapacityThreshold);
  }
  if (a.has("--out")) {
    std::ofstream f(a.str("--out", ""));
    if (!f) throw std::runtime_error("cannot write " + a.str("--out", ""));
    write_sweep_csv(f, rows);
    std::printf("wrote %s\n", a.str("--out", "").c_str());
  } else {
    write_sweep_csv(std::cout, rows);
  }
  return 0;
}

int cmd_validate(const Args& a) {
  if (a.positional.size() != 1) throw UsageError("validate-profile takes one profile path");
  const ProfileSet ps = load_profile(resolve_profile(a.positional[0]));
  int total = 0;
  for (const auto& comp : ps.components) {
    const auto v = check_subadditivity(comp.cost);
    total += static_cast<int>(v.size());
    std::printf("component %-20s layers=%-3d  sub-additivity violations: %zu\n", comp.id.c_str(), comp.num_layers(),
                v.size());
    for (const auto& x : v)
      std::printf("  layer %d: h(%d+%d) exceeds h(%d)+h(%d) by %.4f ms\n", x.layer, x.b1, x.b2, x.b1, x.b2, x.excess);
  }
  std::printf("%d violation(s) across %zu component(s); schedulers do not require the property, batching gains may "
              "simply be absent there\n",
              total, ps.components.size());
  return 0;
}

void dump_instance(const RandomInstance& inst, int trial, const char* suite, std::uint64_t seed) {
  std::printf("oracle mismatch in %s (trial %d, seed %llu)\n", suite, trial, static_cast<unsigned long long>(seed));
  std::printf("  layers:");
  for (const auto& r : inst.requests) std::printf(" %d", r.layer);
  std::printf("\n  deadlines:");
  for (const auto& r : inst.requests) {
    if (r.deadline >= kNoDeadline) std::printf(" -");
    else std::printf(" %.0f", r.deadline);
  }
  std::printf("\n  table (layer: h(1..n)):\n");
  const int n_layers = inst.profile.dnns[0].num_layers();
  for (int k = 1; k <= n_layers; ++k) {
    std::printf("    %d:", k);
    for (int b = 1; b <= static_cast<int>(inst.requests.size()); ++b) std::printf(" %g", inst.profile.lookup(0, k, b));
    std::printf("\n");
  }
}

// Exhaustive-oracle self checks on random instances (the reference's
// oracle-check; instance streams identical for the same --seed).
int cmd_oracle(const Args& a) {
  const int instances = static_cast<int>(a.integer("--instances", 200));
  const auto seed = static_cast<std::uint64_t>(a.integer("--seed", 1));
  const int max_req = static_cast<int>(a.integer("--max-requests", 8));
  const bool bounded = a.has("--bounded");
  const std::string what = a.str("--what", "all");
  if (max_req < 1 || max_req > 10) throw std::runtime_error("--max-requests must be in [1, 10]");
  SplitMix64 rng(seed);
  int failures = 0;
  const bool all = what == "all";
  if (all || what == "time") {
    for (int t = 0; t < instances; ++t) {
      const auto inst = random_instance(rng, max_req, 5, TableStyle::arbitrary);
      const int n = static_cast<int>(inst.requests.size());
      const int bound = bounded ? rng.uniform_int(1, n) : n;
      const Schedule dp = compute_schedule(inst.requests, inst.profile, 0, bound);
      const ExhaustiveResult ex = exhaustive_min_completion(inst.requests, inst.profile, 0, bound);
      if (dp.objective != ex.objective) {
        dump_instance(inst, t, "completion-time DP", seed);
        std::printf("  expected %.6f got %.6f (bound %d)\n", ex.objective, dp.objective, bound);
        ++failures;
      }
    }
    std::printf("completion-time DP: %d instance(s) checked\n", instances);
  }
  if (all || what == "tardy") {
    for (int t = 0; t < instances; ++t) {
      const auto inst = random_instance(rng, max_req, 5, TableStyle::arbitrary, true, 0.0);
      const int n = static_cast<int>(inst.requests.size());
      const int bound = bounded ? rng.uniform_int(1, n) : n;
      const Schedule dp = tardy_dp(inst.requests, inst.profile, 0, bound, 0.0);
      const ExhaustiveResult ex = exhaustive_min_tardy(inst.requests, inst.profile, 0, bound, 0.0);
      if (dp.tardy_count != ex.tardy || dp.objective != ex.objective) {
        dump_instance(inst, t, "tardy DP", seed);
        std::printf("  expected tardy=%d sum=%.6f got tardy=%d sum=%.6f\n", ex.tardy, ex.objective, dp.tardy_count,
                    dp.objective);
        ++failures;
      }
    }
    std::printf("tardy DP: %d instance(s) checked\n", instances);
  }
  if (all || what == "multi") {
    for (int t = 0; t < instances; ++t) {
      ProfileSet ps;
      std::vector<Request> reqs;
      RequestId id = 1;
      Ms arrival = 0;
      for (int d = 0; d < 3; ++d) {
        SharedComponent comp;
        comp.id = "c" + std::to_string(d);
        comp.cost = random_cost_table(rng, 3, 9, TableStyle::arbitrary);
        comp.output_bits.assign(3, 100000);
        ps.components.push_back(std::move(comp));
        ps.dnns.emplace_back("m" + std::to_string(d), std::vector<StageRef>{{d, 1}}, 3);
        std::vector<int> layers(static_cast<std::size_t>(rng.uniform_int(1, 3)));
        for (int& l : layers) l = rng.uniform_int(1, 3);
        std::sort(layers.begin(), layers.end(), std::greater<int>());
        for (int l : layers) {
          Request r;
          r.id = id++;
          r.dnn = d;
          r.arrival = arrival;
          r.layer = l;
          arrival += 1.0;
          reqs.push_back(r);
        }
      }
      ps.max_batch = 9;
      const Schedule s = schedule_multi(reqs, ps, 9);
      const ExhaustiveResult ex = exhaustive_multi(reqs, ps, 9);
      if (s.objective != ex.objective) {
        std::printf("oracle mismatch in multi-DNN search (trial %d, seed %llu): expected %.6f got %.6f\n", t,
                    static_cast<unsigned long long>(seed), ex.objective, s.objective);
        ++failures;
      }
    }
    std::printf("multi-DNN permutation search: %d instance(s) checked\n", instances);
  }
  if (all || what == "lemma") {
    for (int t = 0; t < instances; ++t) {
      const auto inst = random_instance(rng, 4, 3, TableStyle::subadditive);
      const int n = static_cast<int>(inst.requests.size());
      const ExhaustiveResult ex = exhaustive_min_completion(inst.requests, inst.profile, 0, n);
      const Ms inter = interleaving_optimum(inst.requests, inst.profile, 0);
      if (inter < ex.objective) {
        dump_instance(inst, t, "run-to-completion check", seed);
        std::printf("  interleaving %.6f beats segmentation %.6f\n", inter, ex.objective);
        ++failures;
      }
    }
    std::printf("run-to-completion check: %d instance(s) checked\n", instances);
  }
  if (failures) {
    std::printf("%d failure(s); re-run with --seed %llu to reproduce\n", failures,
                static_cast<unsigned long long>(seed));
    return 1;
  }
  std::printf("all oracle checks passed\n");
  return 0;
}

void usage() {
  std::fprintf(stderr,
               "usage: batchsim_b200 <simulate|sweep-capacity|validate-profile|oracle-check> [options]\n"
               "  simulate        --profile P [--workload W] [--scheduler S] [--process P] [--rate R] ... [--out F]\n"
               "  sweep-capacity  --profile P [sim options] [--rates lo:hi:step] [--schedulers a,b] [--seeds N]\n"
               "  validate-profile PROFILE\n"
               "  oracle-check    [--instances N] [--seed S] [--max-requests M] [--bounded] [--what W]\n");
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    usage();
    return 2;
  }
  const std::string cmd = argv[1];
  try {
    if (cmd == "simulate") return cmd_simulate(parse_args(argc, argv, 2, {}, kSimFlags));
    if (cmd == "sweep-capacity") {
      std::vector<std::string> v = kSimFlags;
      v.insert(v.end(), {"--rates", "--schedulers", "--seeds"});
      return cmd_sweep(parse_args(argc, argv, 2, {}, v));
    }
    if (cmd == "validate-profile") return cmd_validate(parse_args(argc, argv, 2, {}, {}));
    if (cmd == "oracle-check")
      return cmd_oracle(parse_args(argc, argv, 2, {"--bounded"},
                                   {"--instances", "--seed", "--max-requests", "--what"}));
    if (cmd == "-h" || cmd == "--help") {
      usage();
      return 0;
    }
    usage();
    return 2;
  } catch (const UsageError& e) {
    std::fprintf(stderr, "usage error: %s\n", e.what());
    usage();
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
}
