// Schedule oracle driver — TEST INFRASTRUCTURE ONLY.
//
// Compiled against the UNMODIFIED reference headers where they lie
// (/root/reference/proj/include/batchsim, see oracle/Makefile); nothing of the
// reference is copied into this repository. It runs the reference's own
// schedulers / simulator on a job description and prints JSON lines that the
// parity tests compare bit-for-bit against libbs_host.so (doubles are printed
// as their IEEE-754 bit patterns).
//
//   ref_dump JOB.json      (or "-" for stdin)
//
// Job kinds:
//   {"job":"sim", ...}     run_sim with a per-plan / per-step trace
//                          (the loop below is Simulator::run,
//                          simulator.hpp:221-241, with observation points)
//   {"job":"calls", "calls":[...]}  direct scheduler calls on given inputs
//                          (dp_time.hpp, deadline.hpp, multi_dnn.hpp, ...)
//   {"job":"random", ...}  random instances from reference.hpp:286-339 plus
//                          the calls above on them
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference
// legs may execute this binary.

#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>

#include <json.hpp>

// The simulator keeps its event loop state private; this oracle re-runs the
// same loop with observation points, so it needs to see it.
#define private public
#include <batchsim/batchsim.hpp>
#undef private

using json = nlohmann::json;
using namespace batchsim;

namespace {

std::string bits(double v) {
  std::uint64_t u;
  std::memcpy(&u, &v, sizeof u);
  char buf[24];
  std::snprintf(buf, sizeof buf, "%016" PRIx64, u);
  return buf;
}

double num(const json& j) {
  if (j.is_null()) return kNoDeadline;
  if (j.is_string()) {
    const std::string s = j.get<std::string>();
    if (s == "inf") return kNoDeadline;
    std::uint64_t u = std::stoull(s, nullptr, 16);
    double d;
    std::memcpy(&d, &u, sizeof d);
    return d;
  }
  return j.get<double>();
}

json rider_json(const Rider& r) {
  return json::array({r.id, r.dnn, r.join_layer, r.leave_layer, r.deposit_layer});
}

json schedule_json(const Schedule& s) {
  json segs = json::array();
  for (const auto& g : s.segments) {
    json riders = json::array();
    for (const auto& r : g.riders) riders.push_back(rider_json(r));
    segs.push_back({{"members", g.members},
                    {"dnn", g.dnn},
                    {"start_layer", g.start_layer},
                    {"duration", bits(g.duration)},
                    {"finish_offset", bits(g.finish_offset)},
                    {"max_layer_batch", g.max_layer_batch},
                    {"riders", riders}});
  }
  json offs = json::array();
  for (const auto& [id, off] : s.completion_offsets) offs.push_back(json::array({id, bits(off)}));
  return {{"segments", segs},
          {"completion_offsets", offs},
          {"objective", bits(s.objective)},
          {"total_duration", bits(s.total_duration)},
          {"tardy_count", s.tardy_count},
          {"drop_marks", s.drop_marks}};
}

json profile_json(const ProfileSet& ps) {
  json comps = json::array();
  for (const auto& c : ps.components) {
    json layers = json::array();
    for (int k = 1; k <= c.num_layers(); ++k) {
      json grid = json::array();
      for (const auto& [b, ms] : c.cost.grid(k)) grid.push_back(json::array({b, ms}));
      layers.push_back({{"output_bits", c.output_bits[static_cast<std::size_t>(k - 1)]},
                        {"runtime_ms", grid}});
    }
    comps.push_back({{"id", c.id}, {"layers", layers}});
  }
  json dnns = json::array();
  for (const auto& d : ps.dnns) {
    json stages = json::array();
    for (const auto& s : d.stages()) stages.push_back(ps.components[static_cast<std::size_t>(s.component)].id);
    dnns.push_back({{"id", d.name()}, {"stages", stages}});
  }
  return {{"max_batch", ps.max_batch}, {"components", comps}, {"dnns", dnns}};
}

json request_json(const Request& r) {
  json d = r.deadline >= kNoDeadline ? json(nullptr) : json(r.deadline);
  return json::array({r.id, r.dnn, r.arrival, d, r.layer});
}

std::vector<Request> requests_from(const json& arr) {
  std::vector<Request> out;
  for (const auto& a : arr) {
    Request r;
    r.id = a.at(0).get<RequestId>();
    r.dnn = a.at(1).get<int>();
    r.arrival = num(a.at(2));
    r.deadline = num(a.at(3));
    r.layer = a.at(4).get<int>();
    out.push_back(r);
  }
  return out;
}

SplitGranularity granularity_from(const std::string& s) {
  if (s == "request") return SplitGranularity::per_request;
  if (s == "layer") return SplitGranularity::per_layer;
  if (s == "group") return SplitGranularity::per_group;
  throw std::invalid_argument("granularity " + s);
}

ProfileSet profile_from(const json& j, const std::string& base) {
  if (j.is_string()) return load_profile(j.get<std::string>());
  return parse_profile(j, base);
}

// One scheduler call; returns {"result": schedule} or {"error": "..."}.
json do_call(const json& c, const ProfileSet& ps) {
  const std::string fn = c.at("fn").get<std::string>();
  const std::vector<Request> reqs = requests_from(c.value("requests", json::array()));
  const int bound = c.value("bound", ps.max_batch);
  const int dnn = c.value("dnn", 0);
  DpOptions opts;
  opts.granularity = granularity_from(c.value("granularity", std::string("request")));
  opts.groups = c.value("groups", 5);
  opts.extra_active = c.value("extra_active", 0);
  const Ms now = c.contains("now") ? num(c.at("now")) : 0.0;
  json out;
  try {
    if (fn == "dp") {
      out["result"] = schedule_json(compute_schedule_dp(reqs, ps, dnn, bound, opts));
    } else if (fn == "tardy") {
      const Ms off = c.contains("start_offset") ? num(c.at("start_offset")) : 0.0;
      out["result"] = schedule_json(tardy_dp(reqs, ps, dnn, bound, now, opts, off));
    } else if (fn == "edf") {
      out["result"] = schedule_json(edf_batch(reqs, ps, bound, now));
    } else if (fn == "batch") {
      out["result"] = schedule_json(baseline_batch(reqs, ps, bound));
    } else if (fn == "no_batch") {
      out["result"] = schedule_json(baseline_no_batch(reqs, ps));
    } else if (fn == "multi" || fn == "multi_shared") {
      MultiOptions mo;
      mo.dp = opts;
      mo.permutation_guard = c.value("guard", 6);
      mo.allow_heuristic = c.value("heuristic", true);
      out["result"] = schedule_json(fn == "multi" ? schedule_multi(reqs, ps, bound, mo)
                                                  : schedule_multi_shared(reqs, ps, bound, mo));
    } else if (fn == "segment") {
      std::vector<int> layers = c.at("layers").get<std::vector<int>>();
      const SweepResult r = segment_duration(layers, ps, dnn, bound);
      out["result"] = {{"duration", bits(r.duration)},
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
        for (int b = 1; b <= bound + 1; ++b) v.push_back(bits(ps.lookup(dnn, k, b)));
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
        v.push_back(bits(g.next_double()));
        v.push_back(bits(g.exponential(3.5)));
        v.push_back(bits(g.pareto(1.25, 0.2)));
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
      for (const auto& a : generate_arrivals(spec)) v.push_back(json::array({bits(a.time), a.dnn, a.size_bits}));
      out["result"] = v;
    } else {
      throw std::invalid_argument("unknown fn " + fn);
    }
  } catch (const std::exception& e) {
    out["error"] = std::string(typeid(e).name()) + ": " + e.what();
  }
  return out;
}

// ---------------------------------------------------------------- sim job

struct SimJob {
  WorkloadSpec spec;
  SimConfig config;
  ProfileSet ps;
  std::optional<NetworkTrace> trace;
  std::optional<ClientProfile> client;
};

SimJob sim_job_from(const json& j) {
  SimJob job;
  job.ps = profile_from(j.at("profile"), "job");
  const json& w = j.at("workload");
  job.spec.process = parse_process(w.value("process", std::string("poisson")));
  job.spec.rate = w.value("rate", 100.0);
  job.spec.count = w.value("count", 5000);
  job.spec.pareto_alpha = w.value("pareto_alpha", 1.25);
  if (w.contains("dnn_mix"))
    for (const auto& m : w.at("dnn_mix"))
      job.spec.dnn_mix.emplace_back(m.at(0).get<std::string>(), m.at(1).get<double>());
  job.spec.relative_deadline = w.contains("relative_deadline") ? num(w.at("relative_deadline")) : kNoDeadline;
  job.spec.seed = w.value("seed", std::uint64_t{1});
  job.spec.size_lo_bits = w.value("size_lo_bits", std::int64_t{120000});
  job.spec.size_hi_bits = w.value("size_hi_bits", std::int64_t{330000});
  if (w.contains("size_trace")) job.spec.size_trace = w.at("size_trace").get<std::vector<std::int64_t>>();
  if (w.contains("explicit_arrivals"))
    for (const auto& a : w.at("explicit_arrivals"))
      job.spec.explicit_arrivals.push_back({num(a.at(0)), a.at(1).get<int>(), a.at(2).get<std::int64_t>()});
  const json& s = j.at("sim");
  job.config.scheduler = parse_scheduler(s.value("scheduler", std::string("ours-time")));
  job.config.granularity = granularity_from(s.value("granularity", std::string("group")));
  job.config.groups = s.value("groups", 5);
  job.config.max_batch = s.value("max_batch", 90);
  job.config.window_cap = s.value("window_cap", 500);
  job.config.scheduler_latency = s.value("scheduler_latency", 0.0);
  job.config.step_overhead = s.value("step_overhead", 0.0);
  job.config.offload = parse_offload(s.value("offload", std::string("none")));
  job.config.partial_rule = s.value("partial_rule", std::string("min_completion")) == "first_hide_wait"
                                ? PartialRule::first_hide_wait
                                : PartialRule::min_completion;
  job.config.clients = s.value("clients", 0);
  job.config.shared_batching = s.value("shared_batching", true);
  if (j.contains("trace")) {
    NetworkTrace t = load_trace(j.at("trace").get<std::string>());
    const double scale = j.value("trace_scale", 1.0);
    job.trace = scale == 1.0 ? t : scale_trace(t, scale);
  } else if (j.contains("trace_points")) {
    std::vector<TracePoint> pts;
    for (const auto& p : j.at("trace_points")) pts.push_back({num(p.at(0)), num(p.at(1))});
    job.trace = NetworkTrace(std::move(pts));
  }
  if (j.contains("client_profile")) job.client = load_client_profile(j.at("client_profile").get<std::string>());
  return job;
}

json outcome_json(const RequestOutcome& o) {
  return json::array({o.id, o.dnn, bits(o.arrival), bits(o.completion), bits(o.deadline), o.on_time ? 1 : 0,
                      o.dropped ? 1 : 0, static_cast<int>(o.location), o.offload_groups, bits(o.network_delay),
                      bits(o.server_time), bits(o.client_time)});
}

void run_sim_job(const json& j, std::ostream& out) {
  const bool want_plans = j.value("emit_plans", true);
  const bool want_steps = j.value("emit_steps", true);
  SimJob job = sim_job_from(j);
  const auto t0 = std::chrono::steady_clock::now();
  Simulator sim(job.spec, job.ps, job.config, job.trace ? &*job.trace : nullptr,
                job.client ? &*job.client : nullptr);
  sim.setup();
  int plans_seen = 0;
  while (!sim.events_.empty()) {
    const Ms now = sim.events_.top().time;
    while (!sim.events_.empty() && sim.events_.top().time == now) {
      const detail::Ev ev = sim.events_.top();
      sim.events_.pop();
      sim.dispatch(ev);
    }
    const bool was_executing = sim.executing_;
    sim.end_of_instant(now);
    if (sim.schedules_computed_ != plans_seen) {
      plans_seen = sim.schedules_computed_;
      if (want_plans) {
        json steps = json::array();
        for (const auto& st : sim.steps_)
          steps.push_back(json::array({st.segment, st.layer_from, st.layer_to, bits(st.duration)}));
        json plan = schedule_json(sim.plan_);
        plan["ev"] = "plan";
        plan["t"] = bits(now);
        plan["n"] = plans_seen;
        plan["steps"] = steps;
        out << plan.dump() << '\n';
      }
    }
    if (!was_executing && sim.executing_ && want_steps) {
      const auto& st = sim.steps_[sim.next_step_];
      out << json{{"ev", "step"}, {"t", bits(now)}, {"plan", plans_seen}, {"i", sim.next_step_},
                  {"end", bits(sim.busy_until_)}, {"from", st.layer_from}, {"to", st.layer_to}}
                 .dump()
          << '\n';
    }
  }
  const double wall_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  SimResult result;
  for (const auto& b : sim.book_) result.outcomes.push_back(b.outcome);
  result.metrics = summarize(result.outcomes);
  json outs = json::array();
  for (const auto& o : result.outcomes) outs.push_back(outcome_json(o));
  const auto& m = result.metrics;
  out << json{{"ev", "outcomes"}, {"outcomes", outs}}.dump() << '\n';
  out << json{{"ev", "summary"},
              {"generated", m.generated},
              {"completed", m.completed},
              {"dropped", m.dropped},
              {"on_time", m.on_time},
              {"on_time_ratio", bits(m.on_time_ratio)},
              {"mean_completion", bits(m.mean_completion)},
              {"median_completion", bits(m.median_completion)},
              {"p95_completion", bits(m.p95_completion)},
              {"schedules_computed", sim.schedules_computed_},
              {"wall_ms", wall_ms}}
                 .dump()
      << '\n';
}

// ---------------------------------------------------------------- random job

TableStyle style_from(const std::string& s) {
  if (s == "arbitrary") return TableStyle::arbitrary;
  if (s == "subadditive") return TableStyle::subadditive;
  return TableStyle::strong_batching;
}

void run_random_job(const json& j, std::ostream& out) {
  SplitMix64 rng(j.value("seed", std::uint64_t{1}));
  const int trials = j.value("trials", 50);
  const int max_requests = j.value("max_requests", 8);
  const int max_layers = j.value("max_layers", 5);
  const TableStyle style = style_from(j.value("style", std::string("arbitrary")));
  const bool deadlines = j.value("deadlines", false);
  const int m = j.value("dnns", 1);
  const json fns = j.at("fns");
  for (int t = 0; t < trials; ++t) {
    ProfileSet ps;
    std::vector<Request> reqs;
    if (m == 1) {
      const Ms now = deadlines ? static_cast<Ms>(rng.uniform_int(0, 40)) : 0.0;
      RandomInstance inst = random_instance(rng, max_requests, max_layers, style, deadlines, now);
      ps = std::move(inst.profile);
      reqs = std::move(inst.requests);
    } else {
      // M private-component DNNs; FIFO per DNN, interleaved arrivals.
      const int layers_each = rng.uniform_int(1, max_layers);
      const int grid = rng.uniform_int(2, max_requests * m);
      for (int d = 0; d < m; ++d) {
        SharedComponent comp;
        comp.id = "c" + std::to_string(d);
        comp.cost = random_cost_table(rng, layers_each, grid, style);
        comp.output_bits.assign(static_cast<std::size_t>(layers_each), 100000);
        ps.components.push_back(std::move(comp));
        ps.dnns.emplace_back("m" + std::to_string(d), std::vector<StageRef>{{d, 1}}, layers_each);
      }
      ps.max_batch = grid;
      RequestId id = 1;
      std::vector<std::vector<int>> per(static_cast<std::size_t>(m));
      for (int d = 0; d < m; ++d) {
        const int n = rng.uniform_int(1, max_requests);
        for (int i = 0; i < n; ++i) per[static_cast<std::size_t>(d)].push_back(rng.uniform_int(1, layers_each));
        std::sort(per[static_cast<std::size_t>(d)].begin(), per[static_cast<std::size_t>(d)].end(), std::greater<int>());
      }
      std::vector<int> owner;
      for (int d = 0; d < m; ++d)
        for (std::size_t i = 0; i < per[static_cast<std::size_t>(d)].size(); ++i) owner.push_back(d);
      for (std::size_t i = owner.size(); i > 1; --i)
        std::swap(owner[i - 1], owner[static_cast<std::size_t>(rng.uniform_int(0, static_cast<int>(i) - 1))]);
      std::vector<std::size_t> next(static_cast<std::size_t>(m), 0);
      for (std::size_t i = 0; i < owner.size(); ++i) {
        const int d = owner[i];
        Request r;
        r.id = id++;
        r.dnn = d;
        r.arrival = static_cast<Ms>(i);
        r.layer = per[static_cast<std::size_t>(d)][next[static_cast<std::size_t>(d)]++];
        if (deadlines) r.deadline = static_cast<Ms>(rng.uniform_int(10, 150));
        reqs.push_back(r);
      }
    }
    json rq = json::array();
    for (const auto& r : reqs) rq.push_back(request_json(r));
    json line = {{"trial", t}, {"profile", profile_json(ps)}, {"requests", rq}};
    json calls = json::array();
    for (const auto& f : fns) {
      json c = f;
      c["requests"] = rq;
      if (deadlines && !c.contains("now")) c["now"] = 0.0;
      json r = do_call(c, ps);
      r["call"] = f;
      calls.push_back(r);
    }
    line["calls"] = calls;
    out << line.dump() << '\n';
  }
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ref_dump JOB.json|-\n");
    return 2;
  }
  json job;
  try {
    if (std::strcmp(argv[1], "-") == 0) {
      std::cin >> job;
    } else {
      std::ifstream in(argv[1]);
      in >> job;
    }
    const std::string kind = job.at("job").get<std::string>();
    std::ostringstream out;
    if (kind == "sim") {
      run_sim_job(job, out);
    } else if (kind == "report") {
      // The reference's own result writers (report.hpp:35-65) on run_sim:
      // outcome CSV, then a "--" line, then summary_json(...).dump(1).
      SimJob sj = sim_job_from(job);
      const SimResult res = run_sim(sj.spec, sj.ps, sj.config, sj.trace ? &*sj.trace : nullptr,
                                    sj.client ? &*sj.client : nullptr);
      write_outcomes_csv(out, res.outcomes, sj.ps);
      out << "--\n" << summary_json(res.metrics).dump(1) << '\n';
    } else if (kind == "sweep") {
      // capacity_sweep (simulator.hpp:806-820): per rate the on-time ratio and
      // mean completion (seconds) as IEEE bit patterns.
      SimJob sj = sim_job_from(job);
      const std::vector<double> rates = job.at("rates").get<std::vector<double>>();
      const auto curve = capacity_sweep(sj.spec, rates, sj.ps, sj.config, sj.trace ? &*sj.trace : nullptr,
                                        sj.client ? &*sj.client : nullptr);
      for (std::size_t r = 0; r < rates.size(); ++r)
        out << json{{"rate", rates[r]}, {"ratio", bits(curve.points[r].metrics.on_time_ratio)},
                    {"mean_completion_s", bits(curve.points[r].metrics.mean_completion / 1000.0)}}
                   .dump()
            << '\n';
    } else if (kind == "bench") {
      // bench.py --impl reference: the reference's run_sim (simulator.hpp:
      // 787-792) on the measured B200 table, one line per (rate, seed) run:
      // its outcome summary, its served req/s in simulated time (completed /
      // (last completion - first arrival), the formula bench.py uses for the
      // live server) and the host wall time of the run.
      for (const auto& r : job.at("runs")) {
        json one = job;
        one["workload"]["rate"] = r.at("rate");
        one["workload"]["seed"] = r.at("seed");
        SimJob sj = sim_job_from(one);
        const auto t0 = std::chrono::steady_clock::now();
        const SimResult res = run_sim(sj.spec, sj.ps, sj.config, sj.trace ? &*sj.trace : nullptr,
                                      sj.client ? &*sj.client : nullptr);
        const double wall = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        double first = res.outcomes.empty() ? 0.0 : res.outcomes.front().arrival, last = 0;
        for (const auto& o : res.outcomes) {
          first = std::min(first, o.arrival);
          if (!o.dropped) last = std::max(last, o.completion);
        }
        const auto& m = res.metrics;
        const double span = last - first;
        out << json{{"rate", r.at("rate")}, {"seed", r.at("seed")}, {"generated", m.generated},
                    {"completed", m.completed}, {"dropped", m.dropped}, {"on_time", m.on_time},
                    {"on_time_ratio", m.on_time_ratio}, {"mean_completion_ms", m.mean_completion},
                    {"p95_completion_ms", m.p95_completion}, {"span_ms", span},
                    {"served_rps", span > 0 ? m.completed / (span / 1000.0) : 0.0},
                    {"schedules_computed", m.schedules_computed}, {"mean_solve_wall_ms", m.mean_solve_wall_ms},
                    {"wall_ms", wall}}
                   .dump()
            << '\n';
      }
    } else if (kind == "random") {
      run_random_job(job, out);
    } else if (kind == "calls") {
      const ProfileSet ps = profile_from(job.at("profile"), "job");
      for (const auto& c : job.at("calls")) {
        json r = do_call(c, ps);
        r["call"] = c;
        out << r.dump() << '\n';
      }
    } else {
      throw std::invalid_argument("unknown job " + kind);
    }
    std::cout << out.str();
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_dump: %s\n", e.what());
    return 1;
  }
  return 0;
}
