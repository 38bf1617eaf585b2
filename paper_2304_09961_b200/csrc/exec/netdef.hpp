// Network definitions for the executor: the scheduler's "layers" (the units
// of the reference's cost tables, h_k(b)) mapped to concrete NHWC ops.
//
// Every request owns ONE activation blob (an arena slot). A static memory
// plan assigns each tensor of a DNN an offset in that blob (greedy first-fit
// over op-index lifetimes), so a layer reads and writes its request's blob in
// place and the state at any layer boundary is simply the blob. Components
// shared between DNNs (config 3's ResNet-50 backbone) are DNN prefixes and are
// planned identically in every DNN that uses them, so a foreign request can
// ride a shared stage inside another DNN's segment.
//
// Layer decompositions follow SURVEY.md §7.3 (profile layer counts of the
// reference data: GoogLeNet 22, ResNet-50 50) and the builder's own
// SmallCNN (5), MobileNetV2 (53) and shared-backbone pair (49 + 1 / 49 + 2).
#pragma once

#include <cstdint>
#include <map>
#include <set>
#include <string>
#include <vector>

namespace bs200 {

enum class OpKind { conv, maxpool, avgpool, dwconv, softmax };

struct TensorDef {
  std::string name;
  int H = 1, W = 1, C = 0;  // C = channel stride (ldc) of the tensor
  long off = 0;             // element offset inside the request blob
  int born = 0, dies = 0;   // op-index lifetime (inclusive)
};

// A channel slice [coff, coff + C) of a planned tensor.
struct TRef {
  int t = -1;
  int coff = 0;
  int C = 0;
};

struct OpDef {
  OpKind kind = OpKind::conv;
  std::string name;
  TRef in, out, res;            // res.t < 0: no residual
  int KH = 1, KW = 1, stride = 1, pad = 0;
  int relu = 0;                 // 0 none, 1 relu, 2 relu6
  int round_out = 1;            // output feeds another tensor-core op
  bool ceil_mode = false;       // maxpool
  int Kpad = 0;                 // conv: padded K (row stride of the weight matrix)
  long w_off = -1, b_off = -1;  // offsets into the executor's weight pool (floats)
  int Ho = 0, Wo = 0;
  double wscale = 1.0;          // residual-branch gain (calibration target std)
  double flops_per_image = 0;   // algorithmic, 2*MACs
  long weight_floats = 0;
};

struct LayerDef {
  std::string name;
  std::vector<int> ops;  // indices into NetDef::ops
  int component = 0;     // index into Suite::components
  int offset = 0;        // 1-based layer index inside the component
};

struct NetDef {
  std::string name;
  std::vector<int> components;  // stage list (component indices)
  std::vector<TensorDef> tensors;
  std::vector<OpDef> ops;
  std::vector<LayerDef> layers;  // 1-based layer k -> layers[k-1]
  int input_t = -1, logits_t = -1, probs_t = -1;
  int in_H = 0, in_W = 0, in_C = 0;  // in_C padded to a multiple of 4
  int num_classes = 0;
  long blob_floats = 0;

  int num_layers() const { return static_cast<int>(layers.size()); }
};

struct ComponentDef {
  std::string id;
  int num_layers = 0;
};

// A set of DNNs served by one executor (one reference "profile set").
struct Suite {
  std::string name;
  std::vector<ComponentDef> components;
  std::vector<NetDef> nets;
  std::vector<float> weights;  // host copy of the weight pool, TF32-rounded
  std::map<std::string, std::pair<long, long>> weight_index;  // "component/op" -> (w_off, b_off)
  int max_batch = 90;
};

// Known suites: "small_cnn", "googlenet", "resnet50", "mobilenet_v2",
// "resnet50_pair" (shared backbone + two heads), "hetero3" (GoogLeNet +
// ResNet-50 + MobileNetV2), "collab" (GoogLeNet + ResNet-50).
// Weights are He-normal draws calibrated on a fixed batch (calib.cpp: BN
// folded with calibration statistics, classifier centred), then TF32-rounded.
// Built once per (name, seed) per process and copied out.
Suite build_suite(const std::string& name, std::uint64_t seed = 2304099610ULL);

// calib.cpp: calibrates the ops of `net` whose weights are not yet in
// `calibrated` (keyed by w_off), in forward order.
void calibrate_net(Suite& s, const NetDef& net, std::set<long>& calibrated);

// Bytes an op moves at batch b (weights once + activations per image) and
// its FLOPs: the algorithmic numerator of the roofline.
double op_bytes(const NetDef& net, const OpDef& op, int batch);
double op_flops(const OpDef& op, int batch);

}  // namespace bs200
