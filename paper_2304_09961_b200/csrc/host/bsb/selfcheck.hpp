// Scheduler self-check: exhaustive searches kept independent of the DPs, and
// the random-instance generators that drive them. Restates the reference's
// proj/include/batchsim/reference.hpp:50-339 (brute_force_min_completion,
// brute_force_min_tardy, interleaving_min_completion, brute_force_multi,
// random_cost_table, random_instance): same objectives, same tie rules and
// the same SplitMix64 draw order, so `oracle-check --seed S` examines the
// same instances as the reference CLI (tools/batchsim_main.cpp:307-430).
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "profile.hpp"

namespace batchsim {

struct ExhaustiveResult {
  Ms objective = kInfeasible;
  int tardy = -1;
  std::uint64_t segmentations = 0;
};

// Min total completion over every contiguous FIFO segmentation.
ExhaustiveResult exhaustive_min_completion(std::span<const Request> requests, const ProfileSet& ps, int dnn,
                                           int bound);
// Fewest tardy jobs (finish strictly after the deadline, offset by now),
// then min total completion, over every contiguous FIFO segmentation.
ExhaustiveResult exhaustive_min_tardy(std::span<const Request> requests, const ProfileSet& ps, int dnn,
                                      int bound, Ms now);
// DNNs back to back in every order, each DNN's requests FIFO-segmented.
ExhaustiveResult exhaustive_multi(std::span<const Request> requests, const ProfileSet& ps, int bound);
// Min total completion over every layer-step interleaving that finishes
// requests in FIFO order (run-to-completion lemma check).
Ms interleaving_optimum(std::span<const Request> requests, const ProfileSet& ps, int dnn);

enum class TableStyle { arbitrary, subadditive, strong_batching };

CostTable random_cost_table(SplitMix64& rng, int num_layers, int grid_max, TableStyle style);

struct RandomInstance {
  ProfileSet profile;
  std::vector<Request> requests;
};

RandomInstance random_instance(SplitMix64& rng, int max_requests, int max_layers, TableStyle style,
                               bool with_deadlines = false, Ms now = 0);

}  // namespace batchsim
