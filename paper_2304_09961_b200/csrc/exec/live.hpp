// Live (wall-clock) serving and device latency profiling.
#pragma once

#include <json.hpp>

#include "executor.hpp"

namespace bs200 {

// Serves a generated arrival trace in real time on the GPU: requests are
// admitted at their arrival times, the batch-aware scheduler (the same
// Planner as the virtual-time simulator) plans on the MEASURED latency
// table, and steps are launched asynchronously with the plan for step k+1
// computed while step k runs. Returns outcomes and
// summary metrics (served req/s, on-time ratio, latency percentiles).
nlohmann::json serve_live(Executor& ex, const nlohmann::json& job);

// Measures h_k(b) for every layer of every component at the requested batch
// sizes and returns a profile in the reference schema
// (proj/include/batchsim/profile_io.hpp:3-18).
nlohmann::json measure_profile(Executor& ex, const nlohmann::json& opts);

}  // namespace bs200
