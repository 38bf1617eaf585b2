// Request generation (Poisson / Pareto / constant gaps, DNN mix, image
// sizes) and the collaborative-mode models: network trace, EWMA estimator,
// client profiles and the offload decisions. Drop-in for the reference's
// workload.hpp:20-139, network.hpp:25-145 and offload.hpp:22-202.
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "core.hpp"

namespace batchsim {

// ------------------------------------------------------------- arrivals

enum class ArrivalProcess { poisson, pareto, constant };
ArrivalProcess parse_process(const std::string& name);
const char* process_name(ArrivalProcess p);

struct ArrivalRecord {
  Ms time = 0;
  int dnn = 0;  // index into the mix
  std::int64_t size_bits = 0;
};

struct WorkloadSpec {
  ArrivalProcess process = ArrivalProcess::poisson;
  double rate = 100.0;
  int count = 5000;
  double pareto_alpha = 1.25;
  std::vector<std::pair<std::string, double>> dnn_mix = {};
  Ms relative_deadline = kNoDeadline;
  std::uint64_t seed = 1;
  std::int64_t size_lo_bits = 120000;
  std::int64_t size_hi_bits = 330000;
  std::vector<std::int64_t> size_trace;
  std::vector<ArrivalRecord> explicit_arrivals;
};

inline constexpr std::uint64_t kArrivalStream = 1;
inline constexpr std::uint64_t kSizeStream = 2;
inline constexpr std::uint64_t kMixStream = 3;
// Synthetic-image stream of the B200 build; never drawn by
// the scheduler, so arrival traces are unaffected.
inline constexpr std::uint64_t kImageStream = 4;

std::vector<ArrivalRecord> generate_arrivals(const WorkloadSpec& spec);
std::vector<std::int64_t> load_size_trace(const std::string& path);

// --------------------------------------------------------------- network

struct TracePoint {
  Ms time = 0;
  double bits_per_ms = 0;
};

class NetworkTrace {
 public:
  NetworkTrace() = default;
  explicit NetworkTrace(std::vector<TracePoint> points);

  bool empty() const { return pts_.empty(); }
  const std::vector<TracePoint>& points() const { return pts_; }
  double throughput_at(Ms t) const { return pts_[segment_at(wrap(t))].bits_per_ms; }
  double span() const { return pts_.size() < 2 ? 0 : pts_.back().time - pts_.front().time; }

  // Position inside one trace period and the piece it falls in.
  Ms wrap(Ms t) const;
  std::size_t segment_at(Ms local) const;

 private:
  std::vector<TracePoint> pts_;
};

Ms transmission_delay(std::int64_t bits, Ms start, const NetworkTrace& trace);
NetworkTrace scale_trace(const NetworkTrace& trace, double factor);
NetworkTrace load_trace(const std::string& path);

// --------------------------------------------------------------- offload

class NetworkEstimator {
 public:
  static constexpr double kNewSampleWeight = 0.3;
  bool primed() const { return primed_; }
  double bits_per_ms() const { return est_; }
  void update(double sample_bits_per_ms);
  void prime(double bits_per_ms);
  Ms estimate_delay(std::int64_t bits) const {
    return (bits <= 0 || !primed_) ? 0 : static_cast<double>(bits) / est_;
  }

 private:
  double est_ = 0;
  bool primed_ = false;
};

double ewma_update(double estimate, double sample);

struct ClientDnnProfile {
  std::string dnn;
  std::vector<Ms> group_runtime_ms;
  std::vector<std::int64_t> group_output_bits;
  Ms full_runtime() const { return prefix_runtime(group_count()); }
  Ms prefix_runtime(int groups) const;
  int group_count() const { return static_cast<int>(group_runtime_ms.size()); }
};

struct ClientProfile {
  Ms compress_ms = 1.5;
  Ms decompress_ms = 0.6;
  std::vector<ClientDnnProfile> dnns;
  const ClientDnnProfile& for_dnn(const std::string& name) const;
  bool has_dnn(const std::string& name) const;
};

enum class OffloadDecision { local, offload };
OffloadDecision decide_binary(Ms local_estimate, Ms transmission_estimate, Ms server_estimate,
                              Ms deadline_remaining);

enum class PartialRule { min_completion, first_hide_wait };
struct PartialDecision {
  int groups_local = 0;
  Ms estimate = kInfeasible;
};
PartialDecision decide_partial(const std::vector<Ms>& client_ready,
                               const std::vector<Ms>& server_wait,
                               const std::vector<Ms>& server_rest,
                               const std::vector<Ms>& payload_delay,
                               PartialRule rule = PartialRule::min_completion);

ClientProfile load_client_profile(const std::string& path);
ClientProfile load_client_profile_string(const std::string& text, const std::string& origin);

}  // namespace batchsim
