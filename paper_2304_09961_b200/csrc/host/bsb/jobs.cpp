#include "jobs.hpp"

#include <cinttypes>
#include <cstdio>
#include <cstring>

namespace batchsim {

using json = nlohmann::json;

std::string hexbits(double v) {
  std::uint64_t u;
  std::memcpy(&u, &v, sizeof u);
  char buf[24];
  std::snprintf(buf, sizeof buf, "%016" PRIx64, u);
  return buf;
}

double ms_from_json(const json& j) {
  if (j.is_null()) return kNoDeadline;
  if (j.is_string()) {
    const std::string s = j.get<std::string>();
    if (s == "inf") return kNoDeadline;
    const std::uint64_t u = std::stoull(s, nullptr, 16);
    double d;
    std::memcpy(&d, &u, sizeof d);
    return d;
  }
  return j.get<double>();
}

json schedule_to_json(const Schedule& s) {
  json segs = json::array();
  for (const auto& g : s.segments) {
    json riders = json::array();
    for (const auto& r : g.riders)
      riders.push_back(json::array({r.id, r.dnn, r.join_layer, r.leave_layer, r.deposit_layer}));
    segs.push_back({{"members", g.members},
                    {"dnn", g.dnn},
                    {"start_layer", g.start_layer},
                    {"duration", hexbits(g.duration)},
                    {"finish_offset", hexbits(g.finish_offset)},
                    {"max_layer_batch", g.max_layer_batch},
                    {"riders", riders}});
  }
  json offs = json::array();
  for (const auto& [id, off] : s.completion_offsets) offs.push_back(json::array({id, hexbits(off)}));
  return {{"segments", segs},
          {"completion_offsets", offs},
          {"objective", hexbits(s.objective)},
          {"total_duration", hexbits(s.total_duration)},
          {"tardy_count", s.tardy_count},
          {"drop_marks", s.drop_marks}};
}

json outcome_to_json(const RequestOutcome& o) {
  return json::array({o.id, o.dnn, hexbits(o.arrival), hexbits(o.completion), hexbits(o.deadline),
                      o.on_time ? 1 : 0, o.dropped ? 1 : 0, static_cast<int>(o.location), o.offload_groups,
                      hexbits(o.network_delay), hexbits(o.server_time), hexbits(o.client_time)});
}

json summary_to_json(const SummaryMetrics& m) {
  return {{"ev", "summary"},
          {"generated", m.generated},
          {"completed", m.completed},
          {"dropped", m.dropped},
          {"on_time", m.on_time},
          {"on_time_ratio", hexbits(m.on_time_ratio)},
          {"mean_completion", hexbits(m.mean_completion)},
          {"median_completion", hexbits(m.median_completion)},
          {"p95_completion", hexbits(m.p95_completion)},
          {"schedules_computed", m.schedules_computed}};
}

SplitGranularity granularity_from_name(const std::string& s) {
  if (s == "request") return SplitGranularity::per_request;
  if (s == "layer") return SplitGranularity::per_layer;
  if (s == "group") return SplitGranularity::per_group;
  throw std::invalid_argument("granularity " + s);
}

SimJob sim_job_from_json(const json& j) {
  SimJob job;
  const json& pj = j.at("profile");
  job.ps = pj.is_string() ? load_profile(pj.get<std::string>()) : parse_profile(pj, "job");
  WorkloadSpec& spec = job.spec;
  const json& w = j.at("workload");
  spec.process = parse_process(w.value("process", std::string("poisson")));
  spec.rate = w.value("rate", 100.0);
  spec.count = w.value("count", 5000);
  spec.pareto_alpha = w.value("pareto_alpha", 1.25);
  if (w.contains("dnn_mix"))
    for (const auto& m : w.at("dnn_mix")) spec.dnn_mix.emplace_back(m.at(0).get<std::string>(), m.at(1).get<double>());
  spec.relative_deadline = w.contains("relative_deadline") ? ms_from_json(w.at("relative_deadline")) : kNoDeadline;
  spec.seed = w.value("seed", std::uint64_t{1});
  spec.size_lo_bits = w.value("size_lo_bits", std::int64_t{120000});
  spec.size_hi_bits = w.value("size_hi_bits", std::int64_t{330000});
  if (w.contains("size_trace")) spec.size_trace = w.at("size_trace").get<std::vector<std::int64_t>>();
  if (w.contains("explicit_arrivals"))
    for (const auto& a : w.at("explicit_arrivals"))
      spec.explicit_arrivals.push_back({ms_from_json(a.at(0)), a.at(1).get<int>(), a.at(2).get<std::int64_t>()});
  const json s = j.value("sim", json::object());
  SimConfig& cfg = job.config;
  cfg.scheduler = parse_scheduler(s.value("scheduler", std::string("ours-time")));
  cfg.granularity = granularity_from_name(s.value("granularity", std::string("group")));
  cfg.groups = s.value("groups", 5);
  cfg.max_batch = s.value("max_batch", 90);
  cfg.window_cap = s.value("window_cap", 500);
  cfg.scheduler_latency = s.value("scheduler_latency", 0.0);
  cfg.step_overhead = s.value("step_overhead", 0.0);
  cfg.offload = parse_offload(s.value("offload", std::string("none")));
  cfg.partial_rule = s.value("partial_rule", std::string("min_completion")) == "first_hide_wait"
                         ? PartialRule::first_hide_wait
                         : PartialRule::min_completion;
  cfg.clients = s.value("clients", 0);
  cfg.shared_batching = s.value("shared_batching", true);
  if (j.contains("trace")) {
    NetworkTrace t = load_trace(j.at("trace").get<std::string>());
    const double scale = j.value("trace_scale", 1.0);
    job.trace = scale == 1.0 ? t : scale_trace(t, scale);
  } else if (j.contains("trace_points")) {
    std::vector<TracePoint> pts;
    for (const auto& p : j.at("trace_points")) pts.push_back({ms_from_json(p.at(0)), ms_from_json(p.at(1))});
    job.trace = NetworkTrace(std::move(pts));
  }
  if (j.contains("client_profile")) {
    const json& c = j.at("client_profile");
    job.client = c.is_string() ? load_client_profile(c.get<std::string>())
                               : load_client_profile_string(c.dump(), "job");
  }
  return job;
}

}  // namespace batchsim
