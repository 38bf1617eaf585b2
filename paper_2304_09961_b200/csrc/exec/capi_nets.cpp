// C-ABI of libbs_nets.so: the networks' host-side definitions, calibrated
// weights and synthetic images, with no CUDA dependency (loads on any host).
// libbs_exec.so links the same objects and exports the same entry points.
// Used by the CPU oracles (tests/) and by bench.py's reference arm, which must
// not load the executor.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>

#include "bs_exec.h"
#include "image.hpp"
#include "nets_json.hpp"

namespace bs200 {

nlohmann::json suite_json(const Suite& s, std::size_t blob_floats) {
  nlohmann::json nets = nlohmann::json::array();
  for (const NetDef& n : s.nets) {
    nlohmann::json tensors = nlohmann::json::array();
    for (const TensorDef& t : n.tensors)
      tensors.push_back({{"name", t.name}, {"H", t.H}, {"W", t.W}, {"C", t.C}, {"off", t.off}});
    nlohmann::json ops = nlohmann::json::array();
    for (const OpDef& o : n.ops) {
      const char* kind = o.kind == OpKind::conv      ? "conv"
                         : o.kind == OpKind::maxpool ? "maxpool"
                         : o.kind == OpKind::avgpool ? "avgpool"
                         : o.kind == OpKind::dwconv  ? "dwconv"
                                                     : "softmax";
      auto ref = [](const TRef& r) { return nlohmann::json::array({r.t, r.coff, r.C}); };
      ops.push_back({{"kind", kind}, {"name", o.name}, {"in", ref(o.in)}, {"out", ref(o.out)}, {"res", ref(o.res)},
                     {"k", o.KH}, {"stride", o.stride}, {"pad", o.pad}, {"relu", o.relu},
                     {"round_out", o.round_out}, {"ceil", o.ceil_mode}, {"Kpad", o.Kpad}, {"w_off", o.w_off},
                     {"b_off", o.b_off}, {"Ho", o.Ho}, {"Wo", o.Wo}, {"flops", o.flops_per_image},
                     {"weight_floats", o.weight_floats}});
    }
    nlohmann::json layers = nlohmann::json::array();
    for (const LayerDef& l : n.layers)
      layers.push_back({{"name", l.name}, {"ops", l.ops}, {"component", l.component}, {"offset", l.offset}});
    nets.push_back({{"name", n.name}, {"components", n.components}, {"tensors", tensors}, {"ops", ops},
                    {"layers", layers}, {"input", n.input_t}, {"logits", n.logits_t}, {"probs", n.probs_t},
                    {"in_H", n.in_H}, {"in_W", n.in_W}, {"in_C", n.in_C}, {"classes", n.num_classes},
                    {"blob_floats", n.blob_floats}});
  }
  nlohmann::json comps = nlohmann::json::array();
  for (const ComponentDef& c : s.components) comps.push_back({{"id", c.id}, {"num_layers", c.num_layers}});
  return {{"suite", s.name}, {"components", comps}, {"nets", nets}, {"weights", s.weights.size()},
          {"slot_floats", blob_floats}, {"max_batch", s.max_batch}};
}

}  // namespace bs200

namespace {

std::string& nets_error() {
  thread_local std::string text;
  return text;
}

template <class F>
int nets_guarded(F&& f) {
  try {
    return f();
  } catch (const std::invalid_argument& e) {
    nets_error() = e.what();
    return BS_EINVAL;
  } catch (const std::exception& e) {
    nets_error() = e.what();
    return BS_ESTATE;
  }
}

}  // namespace

extern "C" {

const char* bs_nets_last_error(void) { return nets_error().c_str(); }

int bs_describe_suite(const char* suite, char** out) {
  return nets_guarded([&] {
    const bs200::Suite s = bs200::build_suite(suite);
    std::size_t slot = 0;
    for (const bs200::NetDef& n : s.nets) slot = std::max<std::size_t>(slot, static_cast<std::size_t>(n.blob_floats));
    const std::string text = bs200::suite_json(s, slot).dump();
    *out = static_cast<char*>(std::malloc(text.size() + 1));
    std::memcpy(*out, text.c_str(), text.size() + 1);
    return BS_OK;
  });
}

int bs_suite_weights_host(const char* suite, float* dst, size_t n) {
  return nets_guarded([&] {
    const bs200::Suite s = bs200::build_suite(suite);
    if (n < s.weights.size()) throw std::invalid_argument("bs_suite_weights_host: buffer too small");
    std::memcpy(dst, s.weights.data(), s.weights.size() * sizeof(float));
    return BS_OK;
  });
}

int bs_make_image(uint64_t seed, uint64_t index, int H, int W, int C, int real_c, float* out) {
  return nets_guarded([&] {
    bs200::synth_image(seed, index, H, W, C, real_c, out);
    return BS_OK;
  });
}

void bs_nets_free(void* p) { std::free(p); }

}  // extern "C"
