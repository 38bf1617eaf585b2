// Reference-style user code (the shape of proj/tests/test_simulator.cpp:31-66
// without Catch2): written against <batchsim/batchsim.hpp> and the reference's
// public names only. Built with -I<repo>/include and linked to libbs_host.so,
// i.e. the drop-in changes nothing but the include path.
#include <batchsim/batchsim.hpp>

#include <cmath>
#include <cstdio>
#include <vector>

using namespace batchsim;

static WorkloadSpec closed_instance(int n, std::int64_t size_bits = 200000) {
  WorkloadSpec spec;
  for (int i = 0; i < n; ++i) spec.explicit_arrivals.push_back({0.0, 0, size_bits});
  return spec;
}

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  int bad = 0;
  SimConfig config;
  config.scheduler = SchedulerKind::ours_time;
  config.granularity = SplitGranularity::per_request;
  config.max_batch = 90;
  // a single request: full runtime, then + network delay on a 10 Mbps link
  const ProfileSet ps = load_profile(argv[1]);
  auto result = run_sim(closed_instance(1), ps, config);
  const double c0 = result.outcomes.at(0).completion;
  NetworkTrace trace({{0.0, 10000.0}});
  result = run_sim(closed_instance(1), ps, config, &trace);
  const double c1 = result.outcomes.at(0).completion;
  std::printf("single request %.3f ms, over 10 Mbps %.3f ms\n", c0, c1);
  bad += std::fabs(c0 - 24.0) > 0.01 || std::fabs(c1 - 44.0) > 0.01;
  // closed instances reproduce the DP objective
  SplitMix64 rng(1001);
  for (int trial = 0; trial < 30; ++trial) {
    const auto inst = random_instance(rng, 8, 4, TableStyle::arbitrary);
    const int n = static_cast<int>(inst.requests.size());
    std::vector<Request> fresh;
    for (int i = 0; i < n; ++i) {
      Request r;
      r.id = i + 1;
      r.arrival = 0.0;
      r.layer = 1;
      fresh.push_back(r);
    }
    const auto dp = compute_schedule(fresh, inst.profile, 0, n);
    SimConfig cfg = config;
    cfg.max_batch = n;
    const auto res = run_sim(closed_instance(n), inst.profile, cfg);
    double total = 0;
    for (const auto& o : res.outcomes) total += o.completion - o.arrival;
    if (res.metrics.completed != n || std::fabs(total - dp.objective) > 1e-9 * std::fabs(dp.objective)) ++bad;
  }
  std::printf("%s\n", bad ? "FAIL" : "ok");
  return bad ? 1 : 0;
}
