// JSON job descriptions shared by the host C-ABI (bs_host_call) and the
// executor's replay / live servers (bs_replay, bs_serve).
#pragma once

#include <optional>
#include <string>

#include "json_io.hpp"
#include "server.hpp"

namespace batchsim {

struct SimJob {
  ProfileSet ps;
  WorkloadSpec spec;
  SimConfig config;
  std::optional<NetworkTrace> trace;
  std::optional<ClientProfile> client;
};

// {"profile": path | inline, "workload": {...}, "sim": {...},
//  "trace": csv path, "trace_scale": x | "trace_points": [[ms, bits/ms]...],
//  "client_profile": path}
SimJob sim_job_from_json(const nlohmann::json& j);
SplitGranularity granularity_from_name(const std::string& s);

std::string hexbits(double v);
double ms_from_json(const nlohmann::json& j);
nlohmann::json schedule_to_json(const Schedule& s);
nlohmann::json outcome_to_json(const RequestOutcome& o);
nlohmann::json summary_to_json(const SummaryMetrics& m);

}  // namespace batchsim
