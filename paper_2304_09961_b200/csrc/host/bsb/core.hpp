// Domain types of the batch-aware scheduler (drop-in for the reference's
// proj/include/batchsim/model.hpp:19-118 and rng.hpp:12-52).
//
// Times are double milliseconds. Build with -ffp-contract=off: every double
// expression in this library is evaluated in the same order as the
// reference so that schedules are bit-identical.
#pragma once

#include <cmath>
#include <cstdint>
#include <limits>
#include <span>
#include <string>
#include <vector>

namespace batchsim {

using Ms = double;
using RequestId = std::int64_t;

inline constexpr Ms kInfeasible = std::numeric_limits<double>::infinity();
inline constexpr Ms kNoDeadline = std::numeric_limits<double>::infinity();
inline constexpr int kRemoteOrigin = -1;

enum class RequestState { pending, running, completed, dropped };

// A request waiting at the server. `layer` is the next layer to execute
// (1-based; num_layers + 1 == finished). Ref: model.hpp:31-39.
struct Request {
  RequestId id = 0;
  int dnn = 0;
  Ms arrival = 0;
  Ms deadline = kNoDeadline;
  int layer = 1;
  RequestState state = RequestState::pending;
  int origin = kRemoteOrigin;
};

// FIFO order: generation time, then id. Ref: model.hpp:42-45.
inline bool arrives_before(const Request& a, const Request& b) {
  return a.arrival < b.arrival || (a.arrival == b.arrival && a.id < b.id);
}

void sort_by_arrival(std::vector<Request>& reqs);

struct ValidationIssue {
  enum class Kind { fifo_violation, layer_out_of_range, duplicate_id, bad_deadline };
  Kind kind;
  RequestId request = 0;
  std::string detail;
};

struct ValidationReport {
  std::vector<ValidationIssue> issues;
  bool ok() const { return issues.empty(); }
};

// Report-only FIFO/layer/id/deadline checks. Ref: model.hpp:65-101.
ValidationReport validate_request_set(std::span<const Request> requests, int num_layers);

enum class CompletionLocation { server, client_full, client_partial };

struct RequestOutcome {
  RequestId id = 0;
  int dnn = 0;
  Ms arrival = 0;
  Ms completion = kInfeasible;
  Ms deadline = kNoDeadline;
  bool on_time = false;
  bool dropped = false;
  CompletionLocation location = CompletionLocation::server;
  int offload_groups = 0;
  Ms network_delay = 0;
  Ms server_time = 0;
  Ms client_time = 0;
};

// SplitMix64 (Steele, Lea, Flood 2014): the portable, splittable generator
// all workload randomness flows through. Ref: rng.hpp:12-52 (the stream
// derivation and the 53-bit double construction are part of the contract:
// arrival traces must be bit-identical to the reference's).
class SplitMix64 {
 public:
  SplitMix64() = default;
  explicit SplitMix64(std::uint64_t seed) : s_(seed) {}

  std::uint64_t next_u64() {
    std::uint64_t z = (s_ += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * next_double(); }
  int uniform_int(int lo, int hi) {
    const auto span = static_cast<std::uint64_t>(hi - lo + 1);
    return lo + static_cast<int>(next_u64() % span);
  }
  double exponential(double mean) { return -mean * std::log(1.0 - next_double()); }
  double pareto(double alpha, double kappa) {
    return kappa * std::pow(1.0 - next_double(), -1.0 / alpha);
  }
  static SplitMix64 stream(std::uint64_t seed, std::uint64_t tag) {
    SplitMix64 mixer(seed ^ (0xA0761D6478BD642FULL * (tag + 1)));
    return SplitMix64(mixer.next_u64());
  }

 private:
  std::uint64_t s_ = 0;
};

}  // namespace batchsim
