#include "arrivals.hpp"

#include <algorithm>
#include <cmath>
#include <fstream>
#include <sstream>
#include <stdexcept>

#include <json.hpp>

namespace batchsim {

ArrivalProcess parse_process(const std::string& name) {
  if (name == "poisson") return ArrivalProcess::poisson;
  if (name == "pareto") return ArrivalProcess::pareto;
  if (name == "constant") return ArrivalProcess::constant;
  throw std::invalid_argument("unknown arrival process '" + name + "'");
}

const char* process_name(ArrivalProcess p) {
  return p == ArrivalProcess::poisson ? "poisson" : p == ArrivalProcess::pareto ? "pareto" : "constant";
}

// Ref: workload.hpp:65-125. Three independent SplitMix64 streams (gaps,
// sizes, mix) so that one concern never shifts another's draws.
std::vector<ArrivalRecord> generate_arrivals(const WorkloadSpec& spec) {
  if (!spec.explicit_arrivals.empty()) return spec.explicit_arrivals;
  if (spec.rate <= 0) throw std::invalid_argument("arrival rate must be positive");
  if (spec.count < 0) throw std::invalid_argument("request count must be >= 0");
  SplitMix64 gaps = SplitMix64::stream(spec.seed, kArrivalStream);
  SplitMix64 sizes = SplitMix64::stream(spec.seed, kSizeStream);
  SplitMix64 mix = SplitMix64::stream(spec.seed, kMixStream);
  const double mean_gap = 1000.0 / spec.rate;
  const double kappa = (spec.pareto_alpha - 1.0) / spec.rate * 1000.0;

  std::vector<double> cdf;
  double acc = 0;
  for (const auto& entry : spec.dnn_mix) cdf.push_back(acc += entry.second);
  if (!cdf.empty() && (acc < 0.999 || acc > 1.001))
    throw std::invalid_argument("dnn mix fractions must sum to 1");

  std::vector<ArrivalRecord> out(static_cast<std::size_t>(spec.count));
  Ms t = 0;
  for (int i = 0; i < spec.count; ++i) {
    ArrivalRecord& rec = out[static_cast<std::size_t>(i)];
    if (spec.process == ArrivalProcess::poisson)
      t += gaps.exponential(mean_gap);
    else if (spec.process == ArrivalProcess::pareto)
      t += gaps.pareto(spec.pareto_alpha, kappa);
    else
      t += mean_gap;
    rec.time = t;
    if (cdf.size() > 1) {
      const double x = mix.next_double();
      const auto it = std::find_if(cdf.begin(), cdf.end(), [x](double c) { return x < c; });
      rec.dnn = it == cdf.end() ? static_cast<int>(cdf.size()) - 1 : static_cast<int>(it - cdf.begin());
    }
    rec.size_bits = spec.size_trace.empty()
                        ? static_cast<std::int64_t>(sizes.uniform(static_cast<double>(spec.size_lo_bits),
                                                                  static_cast<double>(spec.size_hi_bits)))
                        : spec.size_trace[static_cast<std::size_t>(i) % spec.size_trace.size()];
  }
  return out;
}

std::vector<std::int64_t> load_size_trace(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open size trace: " + path);
  std::vector<std::int64_t> out;
  for (std::string line; std::getline(in, line);) {
    if (line.empty() || line.find("size") != std::string::npos) continue;
    out.push_back(std::stoll(line));
  }
  if (out.empty()) throw std::runtime_error(path + ": empty size trace");
  return out;
}

// ------------------------------------------------------------------ network

NetworkTrace::NetworkTrace(std::vector<TracePoint> points) : pts_(std::move(points)) {
  for (std::size_t i = 0; i < pts_.size(); ++i) {
    if (pts_[i].bits_per_ms <= 0) throw std::runtime_error("network trace throughput must be positive");
    if (i > 0 && pts_[i].time <= pts_[i - 1].time)
      throw std::runtime_error("network trace timestamps must be strictly increasing");
  }
}

Ms NetworkTrace::wrap(Ms t) const {
  if (pts_.size() < 2) return pts_.front().time;
  const Ms base = pts_.front().time;
  const Ms period = span();
  Ms x = t - base;
  x -= std::floor(x / period) * period;
  if (x < 0) x += period;
  return base + x;
}

std::size_t NetworkTrace::segment_at(Ms local) const {
  std::size_t i = 0;
  while (i + 1 < pts_.size() && pts_[i + 1].time <= local) ++i;
  if (pts_.size() > 1 && i + 1 == pts_.size()) i = pts_.size() - 2;
  return i;
}

// Integrates the piecewise-constant throughput from `start` (ref:
// network.hpp:83-111).
Ms transmission_delay(std::int64_t bits, Ms start, const NetworkTrace& trace) {
  if (bits <= 0 || trace.empty()) return 0;
  const auto& p = trace.points();
  if (p.size() == 1) return static_cast<Ms>(bits) / p[0].bits_per_ms;
  double left = static_cast<double>(bits);
  Ms t = start, delay = 0;
  while (left > 0) {
    const Ms local = trace.wrap(t);
    const std::size_t i = trace.segment_at(local);
    const double rate = p[i].bits_per_ms;
    const Ms width = p[i + 1].time - local;
    const double room = rate * width;
    if (room >= left) {
      delay += left / rate;
      left = 0;
    } else {
      left -= room;
      delay += width;
      t += width;
    }
  }
  return delay;
}

NetworkTrace scale_trace(const NetworkTrace& trace, double factor) {
  if (factor <= 0) throw std::invalid_argument("trace scale factor must be positive");
  std::vector<TracePoint> p = trace.points();
  for (TracePoint& x : p) x.bits_per_ms *= factor;
  return NetworkTrace(std::move(p));
}

NetworkTrace load_trace(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open trace file: " + path);
  std::vector<TracePoint> pts;
  bool header_possible = true;
  for (std::string line; std::getline(in, line);) {
    if (line.empty()) continue;
    if (header_possible) {
      header_possible = false;
      if (line.find("timestamp") != std::string::npos) continue;
    }
    const auto comma = line.find(',');
    if (comma == std::string::npos) throw std::runtime_error(path + ": malformed trace row: " + line);
    std::string thr = line.substr(comma + 1);
    if (const auto c2 = thr.find(','); c2 != std::string::npos) thr.resize(c2);
    if (thr.empty()) throw std::runtime_error(path + ": malformed trace row: " + line);
    TracePoint tp;
    tp.time = std::stod(line.substr(0, comma)) * 1000.0;  // s -> ms
    tp.bits_per_ms = std::stod(thr) * 1e6 / 1e3;           // Mbit/s -> bit/ms
    pts.push_back(tp);
  }
  if (pts.empty()) throw std::runtime_error(path + ": empty trace");
  return NetworkTrace(std::move(pts));
}

// ------------------------------------------------------------------ offload

void NetworkEstimator::update(double sample) {
  if (sample <= 0) return;
  if (!primed_) {
    est_ = sample;
    primed_ = true;
    return;
  }
  est_ = ewma_update(est_, sample);
}

void NetworkEstimator::prime(double bits_per_ms) {
  if (primed_ || bits_per_ms <= 0) return;
  est_ = bits_per_ms;
  primed_ = true;
}

double ewma_update(double estimate, double sample) {
  return NetworkEstimator::kNewSampleWeight * sample +
         (1.0 - NetworkEstimator::kNewSampleWeight) * estimate;
}

Ms ClientDnnProfile::prefix_runtime(int groups) const {
  Ms sum = 0;
  for (int g = 0; g < groups; ++g) sum += group_runtime_ms[static_cast<std::size_t>(g)];
  return sum;
}

const ClientDnnProfile& ClientProfile::for_dnn(const std::string& name) const {
  for (const auto& d : dnns)
    if (d.dnn == name) return d;
  throw std::invalid_argument("client profile has no entry for dnn '" + name + "'");
}

bool ClientProfile::has_dnn(const std::string& name) const {
  return std::any_of(dnns.begin(), dnns.end(), [&](const ClientDnnProfile& d) { return d.dnn == name; });
}

OffloadDecision decide_binary(Ms local_estimate, Ms transmission_estimate, Ms server_estimate,
                              Ms deadline_remaining) {
  if (local_estimate <= deadline_remaining) return OffloadDecision::local;
  return local_estimate < transmission_estimate + server_estimate ? OffloadDecision::local
                                                                  : OffloadDecision::offload;
}

// k local groups, then ship the k-boundary payload (ref: offload.hpp:133-161).
PartialDecision decide_partial(const std::vector<Ms>& client_ready,
                               const std::vector<Ms>& server_wait,
                               const std::vector<Ms>& server_rest,
                               const std::vector<Ms>& payload_delay, PartialRule rule) {
  const int g = static_cast<int>(client_ready.size()) - 1;
  PartialDecision pick;
  for (int k = 0; k <= g; ++k) {
    const std::size_t i = static_cast<std::size_t>(k);
    const Ms est = k == g ? client_ready[i]
                          : std::max(client_ready[i] + payload_delay[i], server_wait[i]) + server_rest[i];
    if (rule == PartialRule::min_completion) {
      if (est < pick.estimate) pick = {k, est};
    } else {
      pick = {k, est};
      if (client_ready[i] >= server_wait[i]) break;
    }
  }
  return pick;
}

static ClientProfile client_from_json(const nlohmann::json& doc, const std::string& origin) {
  ClientProfile cp;
  cp.compress_ms = doc.value("compress_ms", 1.5);
  cp.decompress_ms = doc.value("decompress_ms", 0.6);
  for (const auto& dj : doc.at("dnns")) {
    ClientDnnProfile d;
    d.dnn = dj.at("id").get<std::string>();
    for (const auto& g : dj.at("group_runtime_ms")) d.group_runtime_ms.push_back(g.get<double>());
    if (dj.contains("group_output_bits")) {
      for (const auto& g : dj.at("group_output_bits")) d.group_output_bits.push_back(g.get<std::int64_t>());
      if (d.group_output_bits.size() != d.group_runtime_ms.size())
        throw std::runtime_error(origin + ": dnn " + d.dnn +
                                 ": group_output_bits must match group_runtime_ms in length");
    }
    if (d.group_runtime_ms.empty()) throw std::runtime_error(origin + ": dnn " + d.dnn + " has no layer groups");
    cp.dnns.push_back(std::move(d));
  }
  return cp;
}

ClientProfile load_client_profile(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open client profile: " + path);
  nlohmann::json doc;
  try {
    in >> doc;
  } catch (const nlohmann::json::exception& e) {
    throw std::runtime_error(path + ": client profile parse error: " + e.what());
  }
  return client_from_json(doc, path);
}

ClientProfile load_client_profile_string(const std::string& text, const std::string& origin) {
  return client_from_json(nlohmann::json::parse(text), origin);
}

}  // namespace batchsim
