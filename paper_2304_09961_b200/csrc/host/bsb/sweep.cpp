#include "sweep.hpp"

#include <algorithm>

namespace batchsim {

SegmentSweep::SegmentSweep(const ProfileSet& ps, int dnn, int batch_bound)
    : ps_(&ps),
      dnn_(dnn),
      bound_(batch_bound),
      last_(ps.dnns[static_cast<std::size_t>(dnn)].num_layers()),
      cnt_(static_cast<std::size_t>(last_) + 2, 0) {}

void SegmentSweep::reset() {
  std::fill(cnt_.begin(), cnt_.end(), 0);
  start_ = last_ + 1;
  dur_ = 0;
  peak_ = 0;
}

int SegmentSweep::absorb(int layer) {
  const int before = start_;
  int tail_from = layer;
  if (layer < before) {
    // Newly swept layers [layer, before): full runtime at the count that
    // already includes preloaded riders.
    const int stop = std::min(before, last_ + 1);
    for (int k = layer; k < stop; ++k) {
      int& c = cnt_[static_cast<std::size_t>(k)];
      ++c;
      if (c > peak_) peak_ = c;
      dur_ += h(k, c);
    }
    start_ = layer;
    tail_from = before;
  }
  for (int k = tail_from; k <= last_; ++k) dur_ += bump(k);
  return before;
}

void SegmentSweep::undo_absorb(int layer, int prev_start) {
  if (layer < prev_start) {
    for (int k = prev_start; k <= last_; ++k) dur_ -= unbump(k);
    const int stop = std::min(prev_start, last_ + 1);
    for (int k = layer; k < stop; ++k) {
      int& c = cnt_[static_cast<std::size_t>(k)];
      dur_ -= h(k, c);
      --c;
    }
    start_ = prev_start;
  } else {
    for (int k = layer; k <= last_; ++k) dur_ -= unbump(k);
  }
  peak_ = 0;
  for (int k = start_; k <= last_; ++k) peak_ = std::max(peak_, cnt_[static_cast<std::size_t>(k)]);
}

void SegmentSweep::add_rider_counts(int from, int to) {
  for (int k = from; k <= to; ++k) {
    if (k >= start_)
      dur_ += bump(k);
    else
      ++cnt_[static_cast<std::size_t>(k)];
  }
}

SweepResult segment_duration(std::span<const int> layers, const ProfileSet& ps, int dnn,
                             int batch_bound) {
  SweepResult res;
  if (layers.empty()) return res;
  const int n = ps.dnns[static_cast<std::size_t>(dnn)].num_layers();
  const int lo = std::min(n + 1, *std::min_element(layers.begin(), layers.end()));
  res.start_layer = lo;
  res.layer_batch.assign(static_cast<std::size_t>(n - lo + 1), 0);
  res.duration = 0;
  res.max_layer_batch = 0;
  for (int k = lo; k <= n; ++k) {
    const int b = static_cast<int>(std::count_if(layers.begin(), layers.end(),
                                                 [k](int l) { return l <= k; }));
    res.layer_batch[static_cast<std::size_t>(k - lo)] = b;
    res.max_layer_batch = std::max(res.max_layer_batch, b);
    if (b > batch_bound) {
      res.duration = kInfeasible;
      res.feasible = false;
      return res;
    }
    res.duration += ps.lookup(dnn, k, b);
  }
  res.feasible = res.duration < kInfeasible;
  return res;
}

}  // namespace batchsim
