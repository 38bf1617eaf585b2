// The batch-aware schedulers (paper Eq. 1-2 and the on-time objective).
// Drop-in for the reference's dp_time.hpp:34-415, deadline.hpp:21-282 and
// multi_dnn.hpp:28-301: same names, signatures, exceptions and results.
#pragma once

#include <functional>
#include <span>
#include <utility>
#include <vector>

#include "sweep.hpp"

namespace batchsim {

enum class SplitGranularity { per_request, per_layer, per_group };

struct DpOptions {
  SplitGranularity granularity = SplitGranularity::per_request;
  int groups = 5;
  int extra_active = 0;  // requests scheduled after this DNN's schedule
};

using RiderProvider = std::function<std::vector<Rider>(const Request& newest)>;

// A run of FIFO-adjacent requests that the DP may not split.
struct DpUnit {
  int first = 0;
  int last = 0;
  long long key = 0;
};

// Cached DP state for incremental re-scheduling (ref: dp_time.hpp:57-72).
struct DpTable {
  std::vector<std::pair<RequestId, int>> snapshot;
  int dnn = -1;
  int bound = 0;
  int extra_active = 0;
  SplitGranularity granularity = SplitGranularity::per_request;
  int groups = 0;
  std::vector<DpUnit> units;
  std::vector<std::vector<Ms>> durations;  // [e][s]
  std::vector<std::vector<int>> max_batch;
  std::vector<std::vector<Rider>> riders;
  std::vector<Ms> min_cost;
  std::vector<int> choice;
  Schedule schedule;
  bool valid = false;
};

namespace detail {
std::vector<Request> sorted_snapshot(std::span<const Request> requests);
std::vector<DpUnit> build_units(const std::vector<Request>& reqs, const ProfileSet& ps, int dnn,
                                SplitGranularity granularity, int groups, int bound);
[[noreturn]] void throw_infeasible(const std::vector<Request>& reqs, const ProfileSet& ps,
                                   int dnn, int bound, const DpUnit& unit);
}  // namespace detail

// Minimum total completion over contiguous FIFO segmentations of one DNN.
Schedule compute_schedule_dp(std::span<const Request> requests, const ProfileSet& ps, int dnn,
                             int bound, const DpOptions& opts = {}, DpTable* table = nullptr,
                             const RiderProvider& riders = nullptr);
Schedule compute_schedule(std::span<const Request> requests, const ProfileSet& ps, int dnn,
                          int bound, DpTable* table = nullptr);
Schedule compute_schedule_layer_units(std::span<const Request> requests, const ProfileSet& ps,
                                      int dnn, int bound, DpTable* table = nullptr);
Schedule compute_schedule_grouped(std::span<const Request> requests, const ProfileSet& ps,
                                  int dnn, int bound, int groups, DpTable* table = nullptr);
Schedule incremental_update(DpTable& table, std::span<const Request> requests,
                            const ProfileSet& ps, int dnn, int bound);

// Paper baselines: FIFO one-by-one; greedy fill of the head DNN.
Schedule baseline_no_batch(std::span<const Request> requests, const ProfileSet& ps);
Schedule baseline_batch(std::span<const Request> requests, const ProfileSet& ps, int bound);

// Deadline-aware schedulers.
std::pair<std::vector<Request>, std::vector<Request>> drop_expired(
    std::span<const Request> requests, Ms now);
Schedule edf_batch(std::span<const Request> requests, const ProfileSet& ps, int bound, Ms now);
Schedule tardy_dp(std::span<const Request> requests, const ProfileSet& ps, int dnn, int bound,
                  Ms now, const DpOptions& opts = {}, Ms start_offset = 0);

// Multi-DNN (model-wise permutation search) with optional shared-stage riders.
struct MultiOptions {
  DpOptions dp;
  int permutation_guard = 6;
  bool allow_heuristic = false;
};

inline bool reschedule_trigger(bool step_completed, bool arrivals_pending_since_last,
                               bool crossed_shared_boundary) {
  return crossed_shared_boundary || (step_completed && arrivals_pending_since_last);
}

namespace detail {
struct DnnGroup {
  int dnn = 0;
  std::vector<Request> requests;
};
std::vector<DnnGroup> group_by_dnn(std::span<const Request> requests);
std::vector<Rider> collect_riders(const Request& newest, int dnn, const ProfileSet& ps,
                                  const std::vector<Request>& foreign_pending);
}  // namespace detail

Schedule schedule_multi(std::span<const Request> requests, const ProfileSet& ps, int bound,
                        const MultiOptions& opts = {});
Schedule schedule_multi_shared(std::span<const Request> requests, const ProfileSet& ps,
                               int bound, const MultiOptions& opts = {});

}  // namespace batchsim
