#include "profile.hpp"

#include <algorithm>
#include <fstream>
#include <sstream>
#include <stdexcept>

#include "json_io.hpp"

namespace batchsim {

void sort_by_arrival(std::vector<Request>& reqs) {
  std::sort(reqs.begin(), reqs.end(), arrives_before);
}

ValidationReport validate_request_set(std::span<const Request> requests, int num_layers) {
  ValidationReport rep;
  std::vector<Request> fifo(requests.begin(), requests.end());
  sort_by_arrival(fifo);
  std::vector<RequestId> ids;
  for (const Request& r : fifo) ids.push_back(r.id);
  std::sort(ids.begin(), ids.end());
  for (std::size_t i = 1; i < ids.size(); ++i)
    if (ids[i] == ids[i - 1])
      rep.issues.push_back({ValidationIssue::Kind::duplicate_id, ids[i], "duplicate request id"});
  const Request* prev = nullptr;
  for (const Request& r : fifo) {
    if (r.layer < 1 || r.layer > num_layers + 1)
      rep.issues.push_back({ValidationIssue::Kind::layer_out_of_range, r.id,
                            "layer " + std::to_string(r.layer) + " outside [1, " +
                                std::to_string(num_layers + 1) + "]"});
    if (!(r.deadline > r.arrival))
      rep.issues.push_back({ValidationIssue::Kind::bad_deadline, r.id, "deadline not after arrival"});
    if (prev && prev->layer < r.layer)
      rep.issues.push_back({ValidationIssue::Kind::fifo_violation, r.id,
                            "arrives after request " + std::to_string(prev->id) +
                                " but sits at a deeper layer"});
    prev = &r;
  }
  return rep;
}

// ------------------------------------------------------------------ CostTable

CostTable::CostTable(int num_layers, int max_batch)
    : bound_(max_batch), grids_(static_cast<std::size_t>(num_layers)) {}

void CostTable::add_point(int layer, int batch, Ms runtime_ms) {
  grids_.at(static_cast<std::size_t>(layer - 1)).emplace_back(batch, runtime_ms);
  dense_ready_ = false;
}

const std::vector<std::pair<int, Ms>>& CostTable::grid(int layer) const {
  return grids_.at(static_cast<std::size_t>(layer - 1));
}

void CostTable::finalize() {
  for (auto& g : grids_) {
    std::sort(g.begin(), g.end());
    for (std::size_t i = 1; i < g.size(); ++i)
      if (g[i].first == g[i - 1].first)
        throw std::invalid_argument("duplicate batch size " + std::to_string(g[i].first) +
                                    " in cost table");
  }
  // Dense cache of the exact interpolation results for b in [1, bound].
  dense_ready_ = false;
  stride_ = static_cast<std::size_t>(bound_) + 1;
  dense_.assign(grids_.size() * stride_, kInfeasible);
  bool ok = true;
  for (std::size_t k = 0; k < grids_.size() && ok; ++k) {
    if (grids_[k].empty()) {
      ok = false;
      break;
    }
    for (int b = 1; b <= bound_; ++b)
      dense_[k * stride_ + static_cast<std::size_t>(b)] = interpolate(static_cast<int>(k) + 1, b);
  }
  dense_ready_ = ok && bound_ <= (1 << 16);
}

Ms CostTable::interpolate(int layer, int batch) const {
  const auto& g = grids_[static_cast<std::size_t>(layer - 1)];
  // First grid point with batch size >= b.
  std::size_t hi = 0;
  {
    std::size_t lo_i = 0, n = g.size();
    while (n > 0) {
      const std::size_t half = n / 2;
      if (g[lo_i + half].first < batch) {
        lo_i += half + 1;
        n -= half + 1;
      } else {
        n = half;
      }
    }
    hi = lo_i;
  }
  if (hi < g.size() && g[hi].first == batch) return g[hi].second;
  // Two nearest measured points; extrapolate at either end.
  std::size_t a, b;
  if (hi == 0) {
    a = 0;
    b = 1;
  } else if (hi == g.size()) {
    a = g.size() - 2;
    b = g.size() - 1;
  } else {
    a = hi - 1;
    b = hi;
  }
  if (b >= g.size()) return g[a].second;  // single-point grid: flat
  const double frac = static_cast<double>(batch - g[a].first) /
                      static_cast<double>(g[b].first - g[a].first);
  return g[a].second + (g[b].second - g[a].second) * frac;
}

std::vector<SubadditivityViolation> check_subadditivity(const CostTable& table) {
  std::vector<SubadditivityViolation> out;
  for (int k = 1; k <= table.num_layers(); ++k) {
    const auto& g = table.grid(k);
    for (std::size_t i = 0; i < g.size(); ++i) {
      for (std::size_t j = i; j < g.size(); ++j) {
        const int both = g[i].first + g[j].first;
        if (both > table.max_batch()) continue;
        const bool measured = std::any_of(g.begin(), g.end(),
                                          [both](const auto& p) { return p.first == both; });
        if (!measured) continue;
        const Ms together = table.lookup(k, both);
        const Ms apart = g[i].second + g[j].second;
        if (together > apart) out.push_back({k, g[i].first, g[j].first, together - apart});
      }
    }
  }
  return out;
}

// ---------------------------------------------------------------- DnnProfile

DnnProfile::DnnProfile(std::string name, std::vector<StageRef> stages, int num_layers)
    : name_(std::move(name)), stages_(std::move(stages)), num_layers_(num_layers) {
  where_.assign(static_cast<std::size_t>(num_layers_) + 1, Resolved{0, 0, 0});
  if (stages_.empty()) return;
  // Stage of a layer: the last stage that does not start after it, or the
  // first stage (ref: cost_model.hpp:157-163).
  for (int layer = 1; layer <= num_layers_; ++layer) {
    int s = static_cast<int>(stages_.size()) - 1;
    while (s > 0 && stages_[static_cast<std::size_t>(s)].first_layer > layer) --s;
    const StageRef& st = stages_[static_cast<std::size_t>(s)];
    where_[static_cast<std::size_t>(layer)] = {s, st.component, layer - st.first_layer + 1};
  }
}

int DnnProfile::stage_end(int layer) const {
  const std::size_t s = static_cast<std::size_t>(stage_of(layer));
  return s + 1 < stages_.size() ? stages_[s + 1].first_layer - 1 : num_layers_;
}

// ---------------------------------------------------------------- ProfileSet

int ProfileSet::dnn_index(const std::string& name) const {
  for (std::size_t i = 0; i < dnns.size(); ++i)
    if (dnns[i].name() == name) return static_cast<int>(i);
  throw std::invalid_argument("unknown dnn '" + name + "'");
}

Ms ProfileSet::single_request_runtime(int dnn, int from_layer) const {
  Ms sum = 0;
  const int n = dnns[static_cast<std::size_t>(dnn)].num_layers();
  for (int k = from_layer; k <= n; ++k) sum += lookup(dnn, k, 1);
  return sum;
}

std::int64_t ProfileSet::output_bits(int dnn, int layer) const {
  const auto r = dnns[static_cast<std::size_t>(dnn)].resolve(layer);
  return components[static_cast<std::size_t>(r.component)].output_bits[static_cast<std::size_t>(r.offset - 1)];
}

int ProfileSet::component_users(int component) const {
  int users = 0;
  for (const DnnProfile& d : dnns)
    users += std::any_of(d.stages().begin(), d.stages().end(),
                         [component](const StageRef& s) { return s.component == component; });
  return users;
}

bool ProfileSet::layer_is_shared(int dnn, int layer) const {
  return component_users(dnns[static_cast<std::size_t>(dnn)].resolve(layer).component) > 1;
}

// ------------------------------------------------------------- layer groups

std::vector<LayerGroup> group_layers(const ProfileSet& ps, int dnn, int groups) {
  const int n = ps.dnns[static_cast<std::size_t>(dnn)].num_layers();
  if (groups < 1) throw std::invalid_argument("group count must be >= 1");
  if (groups > n)
    throw std::invalid_argument("cannot split " + std::to_string(n) + " layers into " +
                                std::to_string(groups) + " groups");
  Ms total = 0;
  for (int k = 1; k <= n; ++k) total += ps.lookup(dnn, k, 1);
  const Ms target = total / groups;
  std::vector<LayerGroup> out;
  out.reserve(static_cast<std::size_t>(groups));
  int next = 1;
  for (int g = 0; g < groups; ++g) {
    LayerGroup grp{next, next};
    if (g + 1 == groups) {
      grp.last = n;
      out.push_back(grp);
      break;
    }
    // Close once the running sum reaches the target, but leave at least one
    // layer for every group still to come.
    const int still_to_form = groups - g - 1;
    Ms acc = ps.lookup(dnn, next, 1);
    ++next;
    while (acc < target && n - next + 1 > still_to_form) {
      acc += ps.lookup(dnn, next, 1);
      grp.last = next++;
    }
    out.push_back(grp);
  }
  return out;
}

int group_of_layer(const std::vector<LayerGroup>& groups, int layer) {
  for (std::size_t g = 0; g < groups.size(); ++g)
    if (groups[g].first <= layer && layer <= groups[g].last) return static_cast<int>(g);
  return static_cast<int>(groups.size());
}

// ---------------------------------------------------------------- profile IO

ProfileSet parse_profile(const nlohmann::json& doc, const std::string& origin) {
  if (!doc.contains("components") || !doc.contains("dnns"))
    throw std::runtime_error(origin + ": profile must declare components[] and dnns[]");
  ProfileSet ps;
  ps.max_batch = doc.value("max_batch", 90);
  if (ps.max_batch < 1) throw std::runtime_error(origin + ": max_batch must be >= 1");
  for (const auto& cj : doc.at("components")) {
    SharedComponent comp;
    comp.id = cj.at("id").get<std::string>();
    const auto& layers = cj.at("layers");
    comp.cost = CostTable(static_cast<int>(layers.size()), ps.max_batch);
    int idx = 0;
    for (const auto& lj : layers) {
      ++idx;
      const std::string lname = lj.value("name", "layer" + std::to_string(idx));
      bool have_b1 = false;
      for (const auto& pt : lj.at("runtime_ms")) {
        const int b = pt.at(0).get<int>();
        const double ms = pt.at(1).get<double>();
        const std::string where = origin + ": component " + comp.id + " layer " + lname;
        if (b < 1) throw std::runtime_error(where + " has batch size < 1");
        if (ms <= 0) throw std::runtime_error(where + " has non-positive runtime");
        have_b1 = have_b1 || b == 1;
        comp.cost.add_point(idx, b, ms);
      }
      if (!have_b1)
        throw std::runtime_error(origin + ": component " + comp.id + " layer " + lname +
                                 " is missing the batch-size-1 measurement");
      comp.output_bits.push_back(lj.value("output_bits", std::int64_t{0}));
    }
    comp.cost.finalize();
    ps.components.push_back(std::move(comp));
  }
  for (const auto& dj : doc.at("dnns")) {
    const std::string name = dj.at("id").get<std::string>();
    std::vector<StageRef> stages;
    int first = 1;
    for (const auto& sj : dj.at("stages")) {
      const std::string cid = sj.get<std::string>();
      auto it = std::find_if(ps.components.begin(), ps.components.end(),
                             [&](const SharedComponent& c) { return c.id == cid; });
      if (it == ps.components.end())
        throw std::runtime_error(origin + ": dnn " + name + " references undeclared component '" +
                                 cid + "'");
      stages.push_back({static_cast<int>(it - ps.components.begin()), first});
      first += it->num_layers();
    }
    if (stages.empty()) throw std::runtime_error(origin + ": dnn " + name + " has no stages");
    ps.dnns.emplace_back(name, std::move(stages), first - 1);
  }
  return ps;
}

ProfileSet load_profile(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open profile file: " + path);
  nlohmann::json doc;
  try {
    in >> doc;
  } catch (const nlohmann::json::exception& e) {
    throw std::runtime_error(path + ": profile parse error: " + e.what());
  }
  return parse_profile(doc, path);
}

ProfileSet load_profile_string(const std::string& text, const std::string& origin) {
  nlohmann::json doc;
  try {
    doc = nlohmann::json::parse(text);
  } catch (const nlohmann::json::exception& e) {
    throw std::runtime_error(origin + ": profile parse error: " + e.what());
  }
  return parse_profile(doc, origin);
}

}  // namespace batchsim
