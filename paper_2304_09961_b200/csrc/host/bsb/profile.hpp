// Cost model: per-layer batch-latency grids h_k(b), shared components, DNN
// stage layouts and layer grouping. Drop-in for the reference's
// proj/include/batchsim/cost_model.hpp:22-278 and profile_io.hpp:31-122.
//
// On the B200 build these tables hold MEASURED device latencies
// (bs_profile_layer / tools/profile_latency.py); the schema is unchanged so
// the reference can read the same file.
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "core.hpp"

namespace batchsim {

// h_k(b) grid for one component. Exact on measured points; linear between
// (and beyond) the two nearest measured batch sizes; +inf above the bound.
class CostTable {
 public:
  CostTable() = default;
  CostTable(int num_layers, int max_batch);

  int num_layers() const { return static_cast<int>(grids_.size()); }
  int max_batch() const { return bound_; }

  void add_point(int layer, int batch, Ms runtime_ms);
  // Sorts every grid by batch size and rejects duplicates; also builds the
  // dense [layer][b] cache the schedulers read.
  void finalize();
  const std::vector<std::pair<int, Ms>>& grid(int layer) const;

  Ms lookup(int layer, int batch) const {
    if (batch > bound_) return kInfeasible;
    if (dense_ready_) return dense_[static_cast<std::size_t>(layer - 1) * stride_ + batch];
    return interpolate(layer, batch);
  }

 private:
  Ms interpolate(int layer, int batch) const;

  int bound_ = 1;
  std::vector<std::vector<std::pair<int, Ms>>> grids_;
  std::vector<Ms> dense_;
  std::size_t stride_ = 0;
  bool dense_ready_ = false;
};

struct SubadditivityViolation {
  int layer;
  int b1;
  int b2;
  Ms excess;
};

// Measured (k, b1, b2) with h_k(b1 + b2) > h_k(b1) + h_k(b2); report only.
std::vector<SubadditivityViolation> check_subadditivity(const CostTable& table);

struct SharedComponent {
  std::string id;
  CostTable cost;
  std::vector<std::int64_t> output_bits;
  int num_layers() const { return cost.num_layers(); }
};

struct StageRef {
  int component = 0;
  int first_layer = 0;
};

struct LayerGroup {
  int first = 0;
  int last = 0;
};

class DnnProfile {
 public:
  struct Resolved {
    int stage;
    int component;
    int offset;  // 1-based inside the component
  };

  DnnProfile() = default;
  DnnProfile(std::string name, std::vector<StageRef> stages, int num_layers);

  const std::string& name() const { return name_; }
  int num_layers() const { return num_layers_; }
  const std::vector<StageRef>& stages() const { return stages_; }

  Resolved resolve(int layer) const { return where_[static_cast<std::size_t>(layer)]; }
  int stage_of(int layer) const { return resolve(layer).stage; }
  int stage_end(int layer) const;

 private:
  std::string name_;
  std::vector<StageRef> stages_;
  int num_layers_ = 0;
  std::vector<Resolved> where_;  // index 0 unused
};

class ProfileSet {
 public:
  std::vector<SharedComponent> components;
  std::vector<DnnProfile> dnns;
  int max_batch = 1;

  int dnn_index(const std::string& name) const;
  Ms lookup(int dnn, int layer, int batch) const {
    const auto r = dnns[static_cast<std::size_t>(dnn)].resolve(layer);
    return components[static_cast<std::size_t>(r.component)].cost.lookup(r.offset, batch);
  }
  Ms single_request_runtime(int dnn, int from_layer = 1) const;
  std::int64_t output_bits(int dnn, int layer) const;
  bool layer_is_shared(int dnn, int layer) const;
  int component_users(int component) const;
};

// Greedy contiguous G-partition with near-equal single-request runtime.
// Ref: cost_model.hpp:239-270.
std::vector<LayerGroup> group_layers(const ProfileSet& ps, int dnn, int groups);
int group_of_layer(const std::vector<LayerGroup>& groups, int layer);

// Profile JSON (reference schema, profile_io.hpp:3-18).
ProfileSet load_profile(const std::string& path);
ProfileSet load_profile_string(const std::string& text, const std::string& origin = "<string>");

}  // namespace batchsim
