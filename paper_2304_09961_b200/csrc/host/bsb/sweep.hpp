// Schedules, segments and the layer sweep that costs a segment.
// Drop-in for the reference's proj/include/batchsim/schedule.hpp:24-210.
//
// A segment sweeps from its newest member's layer to the DNN's last layer;
// a member joins the batch when the sweep reaches the layer it sits at. The
// incremental sweep charges each absorbed member its marginal cost; the
// floating-point evaluation order of those charges is part of the contract
// (schedules must match the reference bit for bit).
#pragma once

#include <span>
#include <utility>
#include <vector>

#include "profile.hpp"

namespace batchsim {

// Foreign request carried through a shared stage (ref: schedule.hpp:24-30).
struct Rider {
  RequestId id = 0;
  int dnn = 0;
  int join_layer = 0;     // segment DNN's layer space
  int leave_layer = 0;
  int deposit_layer = 0;  // rider's own layer space
};

struct ScheduledSegment {
  std::vector<RequestId> members;  // arrival order
  int dnn = 0;
  int start_layer = 1;
  Ms duration = 0;
  Ms finish_offset = 0;
  int max_layer_batch = 0;
  std::vector<Rider> riders;
};

struct Schedule {
  std::vector<ScheduledSegment> segments;
  std::vector<std::pair<RequestId, Ms>> completion_offsets;
  Ms objective = 0;
  Ms total_duration = 0;
  int tardy_count = 0;
  std::vector<RequestId> drop_marks;
  double solve_wall_ms = 0;

  Ms offset_of(RequestId id) const {
    for (const auto& [rid, off] : completion_offsets)
      if (rid == id) return off;
    return kInfeasible;
  }
};

// Incremental sweep over one DNN (ref: schedule.hpp:64-170).
class SegmentSweep {
 public:
  SegmentSweep(const ProfileSet& ps, int dnn, int batch_bound);

  void reset();
  int start_layer() const { return start_; }
  Ms duration() const { return dur_; }
  int max_count() const { return peak_; }
  bool feasible() const { return peak_ <= bound_; }
  int count_at(int layer) const { return cnt_[static_cast<std::size_t>(layer)]; }

  // Adds a member sitting at `layer`; returns the previous start layer.
  int absorb(int layer);
  // Immediate rollback of the latest absorb(layer) that returned prev_start.
  void undo_absorb(int layer, int prev_start);
  // Preloads rider counts on [from, to].
  void add_rider_counts(int from, int to);

 private:
  Ms h(int k, int b) const { return ps_->lookup(dnn_, k, b); }
  // Marginal cost of one more request at layer k (count goes c -> c+1).
  Ms bump(int k) {
    int& c = cnt_[static_cast<std::size_t>(k)];
    const Ms old = c == 0 ? 0 : h(k, c);
    ++c;
    if (c > peak_) peak_ = c;
    return h(k, c) - old;
  }
  Ms unbump(int k) {
    int& c = cnt_[static_cast<std::size_t>(k)];
    const Ms old = h(k, c);
    --c;
    return old - (c == 0 ? 0 : h(k, c));
  }

  const ProfileSet* ps_;
  int dnn_;
  int bound_;
  int last_;  // number of layers
  int start_ = 0;
  Ms dur_ = 0;
  int peak_ = 0;
  std::vector<int> cnt_;
};

struct SweepResult {
  Ms duration = kInfeasible;
  int max_layer_batch = 0;
  std::vector<int> layer_batch;
  int start_layer = 0;
  bool feasible = false;
};

// Direct sweep: duration = sum_{k >= min layer} h_k(#members with layer <= k).
SweepResult segment_duration(std::span<const int> layers, const ProfileSet& ps, int dnn,
                             int batch_bound);

}  // namespace batchsim
