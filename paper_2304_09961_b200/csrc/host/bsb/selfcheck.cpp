#include "selfcheck.hpp"

#include <algorithm>
#include <functional>
#include <map>

namespace batchsim {

namespace {

// Direct-sum duration of one segment: from its shallowest member's layer to
// the last layer, batching every member whose layer has been reached
// (reference.hpp:30-45). +inf when a layer's batch exceeds the bound.
Ms segment_cost(const std::vector<int>& layers, std::size_t lo, std::size_t hi, const ProfileSet& ps, int dnn,
                int bound) {
  const int n_layers = ps.dnns[static_cast<std::size_t>(dnn)].num_layers();
  int first = n_layers + 1;
  for (std::size_t i = lo; i <= hi; ++i) first = std::min(first, layers[i]);
  Ms d = 0;
  for (int k = first; k <= n_layers; ++k) {
    int b = 0;
    for (std::size_t i = lo; i <= hi; ++i) b += layers[i] <= k ? 1 : 0;
    if (b > bound) return kInfeasible;
    d += ps.lookup(dnn, k, b);
  }
  return d;
}

std::vector<Request> fifo(std::span<const Request> requests) {
  std::vector<Request> v(requests.begin(), requests.end());
  sort_by_arrival(v);
  return v;
}

// Walks the segments of one FIFO segmentation (bit i of `cuts` = a segment
// ends after request i; the last request always closes one), calling
// on_segment(lo, hi, duration); false if a segment is infeasible.
template <typename F>
bool walk_segments(const std::vector<int>& layers, std::uint64_t cuts, const ProfileSet& ps, int dnn, int bound,
                   F&& on_segment) {
  const std::size_t n = layers.size();
  std::size_t lo = 0;
  for (std::size_t i = 0; i < n; ++i) {
    if (i + 1 != n && !((cuts >> i) & 1ULL)) continue;
    const Ms d = segment_cost(layers, lo, i, ps, dnn, bound);
    if (d >= kInfeasible) return false;
    on_segment(lo, i, d);
    lo = i + 1;
  }
  return true;
}

std::vector<int> layers_of(const std::vector<Request>& reqs) {
  std::vector<int> l;
  l.reserve(reqs.size());
  for (const Request& r : reqs) l.push_back(r.layer);
  return l;
}

}  // namespace

ExhaustiveResult exhaustive_min_completion(std::span<const Request> requests, const ProfileSet& ps, int dnn,
                                           int bound) {
  const std::vector<Request> reqs = fifo(requests);
  const std::vector<int> layers = layers_of(reqs);
  ExhaustiveResult best;
  if (reqs.empty()) {
    best.objective = 0;
    return best;
  }
  const std::uint64_t combos = 1ULL << (reqs.size() - 1);
  for (std::uint64_t cuts = 0; cuts < combos; ++cuts) {
    ++best.segmentations;
    Ms clock = 0, sum = 0;
    const bool ok = walk_segments(layers, cuts, ps, dnn, bound, [&](std::size_t lo, std::size_t hi, Ms d) {
      clock += d;
      sum += static_cast<Ms>(hi - lo + 1) * clock;
    });
    if (ok && sum < best.objective) best.objective = sum;
  }
  return best;
}

ExhaustiveResult exhaustive_min_tardy(std::span<const Request> requests, const ProfileSet& ps, int dnn,
                                      int bound, Ms now) {
  const std::vector<Request> reqs = fifo(requests);
  const std::vector<int> layers = layers_of(reqs);
  ExhaustiveResult best;
  if (reqs.empty()) {
    best.objective = 0;
    best.tardy = 0;
    return best;
  }
  const std::uint64_t combos = 1ULL << (reqs.size() - 1);
  for (std::uint64_t cuts = 0; cuts < combos; ++cuts) {
    ++best.segmentations;
    Ms clock = 0, sum = 0;
    int late = 0;
    const bool ok = walk_segments(layers, cuts, ps, dnn, bound, [&](std::size_t lo, std::size_t hi, Ms d) {
      clock += d;
      for (std::size_t j = lo; j <= hi; ++j) {
        sum += clock;
        late += now + clock > reqs[j].deadline ? 1 : 0;
      }
    });
    if (!ok) continue;
    if (best.tardy < 0 || late < best.tardy || (late == best.tardy && sum < best.objective)) {
      best.tardy = late;
      best.objective = sum;
    }
  }
  return best;
}

ExhaustiveResult exhaustive_multi(std::span<const Request> requests, const ProfileSet& ps, int bound) {
  const std::vector<Request> reqs = fifo(requests);
  std::vector<int> dnns;
  for (const Request& r : reqs)
    if (std::find(dnns.begin(), dnns.end(), r.dnn) == dnns.end()) dnns.push_back(r.dnn);
  std::sort(dnns.begin(), dnns.end());
  std::vector<std::vector<int>> layers(dnns.size());
  for (const Request& r : reqs)
    layers[static_cast<std::size_t>(std::find(dnns.begin(), dnns.end(), r.dnn) - dnns.begin())].push_back(r.layer);
  ExhaustiveResult best;
  std::vector<int> order(dnns.size());
  for (std::size_t i = 0; i < order.size(); ++i) order[i] = static_cast<int>(i);
  do {
    // One mixed-radix digit (a cut mask) per DNN.
    std::vector<std::uint64_t> digit(dnns.size(), 0), radix(dnns.size());
    for (std::size_t d = 0; d < dnns.size(); ++d) radix[d] = 1ULL << (layers[d].size() - 1);
    for (;;) {
      ++best.segmentations;
      Ms clock = 0, sum = 0;
      bool ok = true;
      for (std::size_t slot = 0; slot < order.size() && ok; ++slot) {
        const std::size_t d = static_cast<std::size_t>(order[slot]);
        ok = walk_segments(layers[d], digit[d], ps, dnns[d], bound, [&](std::size_t lo, std::size_t hi, Ms dur) {
          clock += dur;
          sum += static_cast<Ms>(hi - lo + 1) * clock;
        });
      }
      if (ok && sum < best.objective) best.objective = sum;
      std::size_t d = 0;
      for (; d < digit.size(); ++d) {
        if (++digit[d] < radix[d]) break;
        digit[d] = 0;
      }
      if (d == digit.size()) break;
    }
  } while (std::next_permutation(order.begin(), order.end()));
  return best;
}

Ms interleaving_optimum(std::span<const Request> requests, const ProfileSet& ps, int dnn) {
  const std::vector<Request> reqs = fifo(requests);
  const int n_layers = ps.dnns[static_cast<std::size_t>(dnn)].num_layers();
  std::map<std::vector<int>, Ms> memo;
  // A state is legal when finished requests form a FIFO prefix.
  auto fifo_finished = [&](const std::vector<int>& pos) {
    bool open = false;
    for (int p : pos) {
      const bool done = p > n_layers;
      if (done && open) return false;
      open = open || !done;
    }
    return true;
  };
  std::function<Ms(const std::vector<int>&)> value = [&](const std::vector<int>& pos) -> Ms {
    int waiting = 0;
    for (int p : pos) waiting += p <= n_layers ? 1 : 0;
    if (!waiting) return 0;
    if (auto hit = memo.find(pos); hit != memo.end()) return hit->second;
    Ms best = kInfeasible;
    for (int k = 1; k <= n_layers; ++k) {
      // Action: every request waiting at layer k runs through it together.
      std::vector<int> next = pos;
      int b = 0;
      for (int& p : next)
        if (p == k) {
          ++p;
          ++b;
        }
      if (!b || !fifo_finished(next)) continue;
      const Ms d = ps.lookup(dnn, k, b);
      if (d >= kInfeasible) continue;
      const Ms rest = value(next);
      if (rest >= kInfeasible) continue;
      best = std::min(best, static_cast<Ms>(waiting) * d + rest);
    }
    memo.emplace(pos, best);
    return best;
  };
  std::vector<int> start;
  for (const Request& r : reqs) start.push_back(r.layer);
  return value(start);
}

CostTable random_cost_table(SplitMix64& rng, int num_layers, int grid_max, TableStyle style) {
  CostTable t(num_layers, grid_max);
  for (int k = 1; k <= num_layers; ++k) {
    if (style == TableStyle::arbitrary) {
      for (int b = 1; b <= grid_max; ++b) t.add_point(k, b, static_cast<Ms>(rng.uniform_int(1, 30)));
      continue;
    }
    // Concave in b: non-increasing increments, hence sub-additive.
    int step = rng.uniform_int(5, 25);
    Ms h = static_cast<Ms>(step);
    t.add_point(k, 1, h);
    for (int b = 2; b <= grid_max; ++b) {
      step = rng.uniform_int(0, style == TableStyle::strong_batching && b == 2 ? step / 2 : step);
      h += static_cast<Ms>(step);
      t.add_point(k, b, h);
    }
  }
  t.finalize();
  return t;
}

RandomInstance random_instance(SplitMix64& rng, int max_requests, int max_layers, TableStyle style,
                               bool with_deadlines, Ms now) {
  const int n = rng.uniform_int(1, max_requests);
  const int n_layers = rng.uniform_int(1, max_layers);
  RandomInstance inst;
  SharedComponent comp;
  comp.id = "c0";
  comp.cost = random_cost_table(rng, n_layers, std::max(n, 2), style);
  comp.output_bits.assign(static_cast<std::size_t>(n_layers), 100000);
  inst.profile.components.push_back(std::move(comp));
  inst.profile.dnns.emplace_back("d0", std::vector<StageRef>{{0, 1}}, n_layers);
  inst.profile.max_batch = std::max(n, 2);
  std::vector<int> layers(static_cast<std::size_t>(n));
  for (int& l : layers) l = rng.uniform_int(1, n_layers);
  std::sort(layers.begin(), layers.end(), std::greater<int>());  // FIFO: older requests are deeper
  for (int i = 0; i < n; ++i) {
    Request r;
    r.id = i + 1;
    r.dnn = 0;
    r.arrival = static_cast<Ms>(i);
    r.layer = layers[static_cast<std::size_t>(i)];
    if (with_deadlines) r.deadline = now + static_cast<Ms>(rng.uniform_int(10, 120));
    inst.requests.push_back(r);
  }
  return inst;
}

}  // namespace batchsim
