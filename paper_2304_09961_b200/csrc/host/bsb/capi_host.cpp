// JSON C-ABI over the host scheduler library (libbs_host.so):
//
//   int   bs_host_call(const char* job_json, char** out_jsonl);
//   void  bs_host_free(char* p);
//   const char* bs_host_last_error(void);
//
// Job kinds mirror the reference's public entry points:
//   {"job":"sim", ...}     run_sim with a per-plan / per-step trace
//   {"job":"calls", ...}   compute_schedule_dp / tardy_dp / edf_batch /
//                          baselines / schedule_multi(_shared) / sweep /
//                          group_layers / lookup on given inputs
// Doubles in results are IEEE-754 bit patterns (16 hex digits) so callers
// can compare schedules bit for bit.
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <optional>
#include <sstream>
#include <string>
#include <typeinfo>

#include "jobs.hpp"

using json = nlohmann::json;
using namespace batchsim;

namespace {

thread_local std::string g_err;

std::vector<Request> requests_of(const json& arr) {
  std::vector<Request> v;
  for (const auto& a : arr) {
    Request r;
    r.id = a.at(0).get<RequestId>();
    r.dnn = a.at(1).get<int>();
    r.arrival = ms_from_json(a.at(2));
    r.deadline = ms_from_json(a.at(3));
    r.layer = a.at(4).get<int>();
    v.push_back(r);
  }
  return v;
}

ProfileSet profile_of(const json& j) {
  if (j.is_string()) return load_profile(j.get<std::string>());
  return parse_profile(j, "job");
}

json one_call(const json& c, const ProfileSet& ps) {
  const std::string fn = c.at("fn").get<std::string>();
  const std::vector<Request> reqs = requests_of(c.value("requests", json::array()));
  const int bound = c.value("bound", ps.max_batch);
  const int dnn = c.value("dnn", 0);
  DpOptions o;
  o.granularity = granularity_from_name(c.value("granularity", std::string("request")));
  o.groups = c.value("groups", 5);
  o.extra_active = c.value("extra_active", 0);
  const Ms now = c.contains("now") ? ms_from_json(c.at("now")) : 0.0;
  json out;
  try {
    if (fn == "dp") {
      out["result"] = schedule_to_json(compute_schedule_dp(reqs, ps, dnn, bound, o));
    } else if (fn == "tardy") {
      const Ms off = c.contains("start_offset") ? ms_from_json(c.at("start_offset")) : 0.0;
      out["result"] = schedule_to_json(tardy_dp(reqs, ps, dnn, bound, now, o, off));
    } else if (fn == "edf") {
      out["result"] = schedule_to_json(edf_batch(reqs, ps, bound, now));
    } else if (fn == "batch") {
      out["result"] = schedule_to_json(baseline_batch(reqs, ps, bound));
    } else if (fn == "no_batch") {
      out["result"] = schedule_to_json(baseline_no_batch(reqs, ps));
    } else if (fn == "multi" || fn == "multi_shared") {
      MultiOptions mo;
      mo.dp = o;
      mo.permutation_guard = c.value("guard", 6);
      mo.allow_heuristic = c.value("heuristic", true);
      out["result"] = schedule_to_json(fn == "multi" ? schedule_multi(reqs, ps, bound, mo)
                                            : schedule_multi_shared(reqs, ps, bound, mo));
    } else if (fn == "segment") {
      const std::vector<int> layers = c.at("layers").get<std::vector<int>>();
      const SweepResult r = segment_duration(layers, ps, dnn, bound);
      out["result"] = {{"duration", hexbits(r.duration)},
                       {"max_layer_batch", r.max_layer_batch},
                       {"layer_batch", r.layer_batch},
                       {"start_layer", r.start_layer},
                       {"feasible", r.feasible}};
    } else if (fn == "groups") {
      json g = json::array();
      for (const auto& lg : group_layers(ps, dnn, c.at("groups").get<int>()))
        g.push_back(json::array({lg.first, lg.last}));
      out["result"] = g;
    } else if (fn == "lookup") {
      json v = json::array();
      const int n = ps.dnns[static_cast<std::size_t>(dnn)].num_layers();
      for (int k = 1; k <= n; ++k)
        for (int b = 1; b <= bound + 1; ++b) v.push_back(hexbits(ps.lookup(dnn, k, b)));
      out["result"] = v;
    } else if (fn == "rng") {
      SplitMix64 g = c.contains("tag") ? SplitMix64::stream(c.at("seed").get<std::uint64_t>(), c.at("tag").get<std::uint64_t>())
                                       : SplitMix64(c.at("seed").get<std::uint64_t>());
      json v = json::array();
      for (int i = 0; i < c.value("count", 4); ++i) {
        const std::uint64_t a = g.next_u64();
        char buf[24];
        std::snprintf(buf, sizeof buf, "%016" PRIx64, a);
        v.push_back(std::string(buf));
        v.push_back(hexbits(g.next_double()));
        v.push_back(hexbits(g.exponential(3.5)));
        v.push_back(hexbits(g.pareto(1.25, 0.2)));
        v.push_back(g.uniform_int(-3, 17));
      }
      out["result"] = v;
    } else if (fn == "arrivals") {
      WorkloadSpec spec;
      spec.process = parse_process(c.value("process", std::string("poisson")));
      spec.rate = c.value("rate", 100.0);
      spec.count = c.value("count", 50);
      spec.seed = c.value("seed", std::uint64_t{1});
      if (c.contains("dnn_mix"))
        for (const auto& m : c.at("dnn_mix")) spec.dnn_mix.emplace_back(m.at(0).get<std::string>(), m.at(1).get<double>());
      json v = json::array();
      for (const auto& a : generate_arrivals(spec)) v.push_back(json::array({hexbits(a.time), a.dnn, a.size_bits}));
      out["result"] = v;
    } else {
      throw std::invalid_argument("unknown fn " + fn);
    }
  } catch (const std::exception& e) {
    out["error"] = std::string(typeid(e).name()) + ": " + e.what();
  }
  return out;
}

struct TraceWriter : SimObserver {
  std::ostream* out;
  bool plans, steps;
  void on_plan(Ms now, int plan_no, const Schedule& plan, const std::vector<detail::ExecStep>& st) override {
    if (!plans) return;
    json steps_j = json::array();
    for (const auto& s : st) steps_j.push_back(json::array({s.segment, s.layer_from, s.layer_to, hexbits(s.duration)}));
    json p = schedule_to_json(plan);
    p["ev"] = "plan";
    p["t"] = hexbits(now);
    p["n"] = plan_no;
    p["steps"] = steps_j;
    *out << p.dump() << '\n';
  }
  void on_step(Ms now, int plan_no, std::size_t index, Ms end, const detail::ExecStep& s) override {
    if (!steps) return;
    *out << json{{"ev", "step"}, {"t", hexbits(now)}, {"plan", plan_no}, {"i", index},
                 {"end", hexbits(end)}, {"from", s.layer_from}, {"to", s.layer_to}}
                .dump()
         << '\n';
  }
};

void sim_job(const json& j, std::ostream& out) {
  SimJob job = sim_job_from_json(j);
  TraceWriter tw;
  tw.out = &out;
  tw.plans = j.value("emit_plans", true);
  tw.steps = j.value("emit_steps", true);
  const auto t0 = std::chrono::steady_clock::now();
  Simulator sim(job.spec, job.ps, job.config, job.trace ? &*job.trace : nullptr, job.client ? &*job.client : nullptr);
  sim.set_observer(&tw);
  const SimResult res = sim.run();
  const double wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  json outs = json::array();
  for (const auto& o : res.outcomes) outs.push_back(outcome_to_json(o));
  out << json{{"ev", "outcomes"}, {"outcomes", outs}}.dump() << '\n';
  json sm = summary_to_json(res.metrics);
  sm["wall_ms"] = wall_ms;
  out << sm.dump() << '\n';
}

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

}  // namespace

extern "C" {

int bs_host_call(const char* job_json, char** out_jsonl) {
  if (!job_json || !out_jsonl) {
    g_err = "bs_host_call: null argument";
    return -1;
  }
  *out_jsonl = nullptr;
  try {
    const json job = json::parse(job_json);
    const std::string kind = job.at("job").get<std::string>();
    std::ostringstream out;
    if (kind == "sim") {
      sim_job(job, out);
    } else if (kind == "calls") {
      const ProfileSet ps = profile_of(job.at("profile"));
      for (const auto& c : job.at("calls")) {
        json r = one_call(c, ps);
        r["call"] = c;
        out << r.dump() << '\n';
      }
    } else {
      throw std::invalid_argument("unknown job " + kind);
    }
    *out_jsonl = dup(out.str());
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = std::string("invalid_argument: ") + e.what();
    return -1;
  } catch (const std::logic_error& e) {
    g_err = std::string("logic_error: ") + e.what();
    return -5;
  } catch (const std::exception& e) {
    g_err = std::string("runtime_error: ") + e.what();
    return -2;
  }
}

void bs_host_free(char* p) { std::free(p); }

const char* bs_host_last_error(void) { return g_err.c_str(); }

}  // extern "C"
