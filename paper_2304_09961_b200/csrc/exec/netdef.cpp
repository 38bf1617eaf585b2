#include "netdef.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <stdexcept>

#include "bsb/core.hpp"

namespace bs200 {

namespace {

constexpr long kAlign = 64;  // floats (256 B)

std::uint64_t fnv1a(const std::string& s) {
  std::uint64_t h = 1469598103934665603ULL;
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ULL;
  }
  return h;
}

float round_tf32_host(float x) {
  std::uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7F800000u) != 0x7F800000u) u = (u + 0x1000u) & 0xFFFFE000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

// Builds one DNN; weights of a component are generated once per suite and
// shared by every DNN that includes the component.
class Builder {
 public:
  Builder(Suite& suite, std::uint64_t seed, const std::string& name) : suite_(suite), seed_(seed) {
    net_.name = name;
  }

  // ---- structure
  void component(const std::string& id) {
    int idx = -1;
    for (std::size_t i = 0; i < suite_.components.size(); ++i)
      if (suite_.components[i].id == id) idx = static_cast<int>(i);
    if (idx < 0) {
      suite_.components.push_back({id, 0});
      idx = static_cast<int>(suite_.components.size()) - 1;
      fresh_component_ = true;
    } else {
      fresh_component_ = false;
    }
    comp_ = idx;
    comp_id_ = id;
    comp_layer_ = 0;
    net_.components.push_back(idx);
  }
  void layer(const std::string& name) {
    LayerDef l;
    l.name = name;
    l.component = comp_;
    l.offset = ++comp_layer_;
    net_.layers.push_back(l);
    if (fresh_component_) suite_.components[static_cast<std::size_t>(comp_)].num_layers = comp_layer_;
  }

  int tensor(const std::string& name, int H, int W, int C) {
    if (C % 4) throw std::logic_error("tensor channel stride must be a multiple of 4: " + name);
    TensorDef t;
    t.name = name;
    t.H = H;
    t.W = W;
    t.C = C;
    t.born = static_cast<int>(net_.ops.size());
    t.dies = t.born;
    net_.tensors.push_back(t);
    return static_cast<int>(net_.tensors.size()) - 1;
  }
  TRef all(int t) const { return TRef{t, 0, net_.tensors[static_cast<std::size_t>(t)].C}; }
  const TensorDef& T(int t) const { return net_.tensors[static_cast<std::size_t>(t)]; }

  int input(int H, int W, int C) {
    const int t = tensor("input", H, W, C);
    net_.tensors[static_cast<std::size_t>(t)].born = -1;
    net_.input_t = t;
    net_.in_H = H;
    net_.in_W = W;
    net_.in_C = C;
    return t;
  }

  // ---- ops
  // conv / FC: in slice -> out slice. real_cin: channels carrying data (the
  // stem's 4th channel is zero padding) for the FLOP count and fan-in.
  void conv(const std::string& name, TRef in, TRef out, int k, int stride, int pad, int relu,
            double wscale = 1.0, TRef res = {}, int real_cin = 0) {
    OpDef op;
    op.kind = OpKind::conv;
    op.name = name;
    op.in = in;
    op.out = out;
    op.res = res;
    op.KH = op.KW = k;
    op.stride = stride;
    op.pad = pad;
    op.relu = relu;
    op.wscale = wscale;
    const TensorDef& ti = T(in.t);
    op.Ho = (ti.H + 2 * pad - k) / stride + 1;
    op.Wo = (ti.W + 2 * pad - k) / stride + 1;
    const TensorDef& to = T(out.t);
    if (to.H != op.Ho || to.W != op.Wo) throw std::logic_error("conv output shape mismatch: " + name);
    const int K = k * k * in.C;
    op.Kpad = (K + 31) / 32 * 32;
    const int cin = real_cin > 0 ? real_cin : in.C;
    const int fan_in = k * k * cin;
    op.flops_per_image = 2.0 * op.Ho * op.Wo * out.C * fan_in;
    op.weight_floats = static_cast<long>(out.C) * fan_in;
    const double std = wscale * std::sqrt((relu ? 2.0 : 1.0) / fan_in);
    weights(op, static_cast<long>(out.C) * op.Kpad, out.C, [&](long i, batchsim::SplitMix64& g) -> float {
      const long kk = i % op.Kpad;
      if (kk >= K) return 0.f;
      if (real_cin > 0 && (kk % in.C) >= real_cin) return 0.f;
      return static_cast<float>(std * gauss(g));
    });
    add(op);
  }

  void dwconv(const std::string& name, TRef in, TRef out, int stride, int relu) {
    OpDef op;
    op.kind = OpKind::dwconv;
    op.name = name;
    op.in = in;
    op.out = out;
    op.KH = op.KW = 3;
    op.stride = stride;
    op.pad = 1;
    op.relu = relu;
    const TensorDef& ti = T(in.t);
    op.Ho = (ti.H + 2 - 3) / stride + 1;
    op.Wo = (ti.W + 2 - 3) / stride + 1;
    op.flops_per_image = 2.0 * op.Ho * op.Wo * in.C * 9;
    op.weight_floats = 9L * in.C;
    const double std = std::sqrt(2.0 / 9.0);
    weights(op, 9L * in.C, in.C, [&](long, batchsim::SplitMix64& g) -> float {
      return static_cast<float>(std * gauss(g));
    });
    add(op);
  }

  void maxpool(const std::string& name, TRef in, TRef out, int k, int stride, int pad, bool ceil_mode) {
    OpDef op;
    op.kind = OpKind::maxpool;
    op.name = name;
    op.in = in;
    op.out = out;
    op.KH = op.KW = k;
    op.stride = stride;
    op.pad = pad;
    op.ceil_mode = ceil_mode;
    op.round_out = 0;
    const TensorDef& ti = T(in.t);
    op.Ho = pool_out(ti.H, k, stride, pad, ceil_mode);
    op.Wo = pool_out(ti.W, k, stride, pad, ceil_mode);
    if (T(out.t).H != op.Ho || T(out.t).W != op.Wo) throw std::logic_error("pool output shape mismatch: " + name);
    add(op);
  }

  void avgpool(const std::string& name, TRef in, TRef out) {
    OpDef op;
    op.kind = OpKind::avgpool;
    op.name = name;
    op.in = in;
    op.out = out;
    op.Ho = op.Wo = 1;
    add(op);
  }

  void softmax(TRef logits, TRef probs) {
    OpDef op;
    op.kind = OpKind::softmax;
    op.name = "softmax";
    op.in = logits;
    op.out = probs;
    op.round_out = 0;
    add(op);
  }

  // Classifier head: global average pool, FC, softmax (the last layer of
  // every network here).
  void classifier(TRef feat, int classes, const std::string& prefix = "", bool pool = true) {
    int pooled = feat.t;
    if (pool) {
      pooled = tensor(prefix + "pool", 1, 1, feat.C);
      avgpool(prefix + "avgpool", feat, all(pooled));
    }
    net_.logits_t = tensor(prefix + "logits", 1, 1, (classes + 3) / 4 * 4);
    conv(prefix + "fc", all(pooled), TRef{net_.logits_t, 0, classes}, 1, 1, 0, 0);
    net_.ops.back().round_out = 0;
    net_.probs_t = tensor(prefix + "probs", 1, 1, (classes + 3) / 4 * 4);
    softmax(TRef{net_.logits_t, 0, classes}, TRef{net_.probs_t, 0, classes});
    net_.num_classes = classes;
  }

  NetDef finish() {
    const int n_ops = static_cast<int>(net_.ops.size());
    for (int t : {net_.logits_t, net_.probs_t})
      if (t >= 0) net_.tensors[static_cast<std::size_t>(t)].dies = n_ops;
    plan();
    return std::move(net_);
  }

 private:
  static int pool_out(int H, int k, int s, int p, bool ceil_mode) {
    const int num = H + 2 * p - k;
    int o = (ceil_mode ? (num + s - 1) / s : num / s) + 1;
    if (ceil_mode && (o - 1) * s >= H + p) --o;
    return o;
  }

  static double gauss(batchsim::SplitMix64& g) {
    const double u1 = g.next_double(), u2 = g.next_double();
    return std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(6.283185307179586 * u2);
  }

  template <class F>
  void weights(OpDef& op, long count, int bias_count, F&& value) {
    const std::string key = comp_id_ + "/" + op.name;
    auto hit = suite_.weight_index.find(key);
    if (hit != suite_.weight_index.end()) {
      op.w_off = hit->second.first;
      op.b_off = hit->second.second;
      return;
    }
    auto& pool = suite_.weights;
    auto align = [&] { pool.resize((pool.size() + kAlign - 1) / kAlign * kAlign, 0.f); };
    align();
    op.w_off = static_cast<long>(pool.size());
    batchsim::SplitMix64 g(seed_ ^ fnv1a(key));
    pool.resize(pool.size() + static_cast<std::size_t>(count));
    for (long i = 0; i < count; ++i)
      pool[static_cast<std::size_t>(op.w_off + i)] = value(i, g);  // TF32-rounded after calibration
    align();
    op.b_off = static_cast<long>(pool.size());
    pool.resize(pool.size() + static_cast<std::size_t>(bias_count));
    for (int i = 0; i < bias_count; ++i)
      pool[static_cast<std::size_t>(op.b_off + i)] = static_cast<float>(0.01 * gauss(g));
    suite_.weight_index[key] = {op.w_off, op.b_off};
  }

  void touch(const TRef& r, int idx) {
    if (r.t < 0) return;
    TensorDef& t = net_.tensors[static_cast<std::size_t>(r.t)];
    t.dies = std::max(t.dies, idx);
  }

  void add(OpDef op) {
    const int idx = static_cast<int>(net_.ops.size());
    touch(op.in, idx);
    touch(op.res, idx);
    touch(op.out, idx);
    net_.ops.push_back(std::move(op));
    net_.layers.back().ops.push_back(idx);
  }

  // First-fit offsets over lifetimes (tensors in creation order).
  void plan() {
    auto& ts = net_.tensors;
    std::vector<int> order(ts.size());
    for (std::size_t i = 0; i < ts.size(); ++i) order[i] = static_cast<int>(i);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
      return ts[static_cast<std::size_t>(a)].born < ts[static_cast<std::size_t>(b)].born;
    });
    std::vector<int> placed;
    long top = 0;
    for (int id : order) {
      TensorDef& t = ts[static_cast<std::size_t>(id)];
      const long size = (static_cast<long>(t.H) * t.W * t.C + kAlign - 1) / kAlign * kAlign;
      std::vector<std::pair<long, long>> busy;
      for (int o : placed) {
        const TensorDef& u = ts[static_cast<std::size_t>(o)];
        if (u.born <= t.dies && t.born <= u.dies)
          busy.emplace_back(u.off, u.off + (static_cast<long>(u.H) * u.W * u.C + kAlign - 1) / kAlign * kAlign);
      }
      std::sort(busy.begin(), busy.end());
      long at = 0;
      for (const auto& [b, e] : busy) {
        if (at + size <= b) break;
        at = std::max(at, e);
      }
      t.off = at;
      top = std::max(top, at + size);
      placed.push_back(id);
    }
    net_.blob_floats = top;
  }

  Suite& suite_;
  std::uint64_t seed_;
  NetDef net_;
  int comp_ = 0;
  std::string comp_id_;
  int comp_layer_ = 0;
  bool fresh_component_ = true;
};

// ------------------------------------------------------------------ models

void small_cnn(Builder& b) {
  b.component("small_cnn_body");
  const int x = b.input(32, 32, 4);
  b.layer("conv1");
  const int a1 = b.tensor("a1", 32, 32, 32);
  b.conv("conv1", b.all(x), b.all(a1), 3, 1, 1, 1, 1.0, {}, 3);
  b.layer("conv2");
  const int a2 = b.tensor("a2", 16, 16, 64);
  b.conv("conv2", b.all(a1), b.all(a2), 3, 2, 1, 1);
  b.layer("conv3");
  const int a3 = b.tensor("a3", 8, 8, 128);
  b.conv("conv3", b.all(a2), b.all(a3), 3, 2, 1, 1);
  b.layer("avgpool");
  const int p = b.tensor("pool", 1, 1, 128);
  b.avgpool("avgpool", b.all(a3), b.all(p));
  b.layer("fc");
  b.classifier(b.all(p), 10, "", false);  // FC + softmax
}

struct Incep {
  const char* name;
  int c1, c2r, c2, c3r, c3, c4;
};

// Two scheduler layers per inception module:
//   A: fused 1x1 GEMM [r2 | r3 | b1] on the module input + branch 4
//      (3x3/1 max-pool then 1x1);
//   B: the two 3x3 convs on the reduce outputs.
// Module tensor layout: [r2 | r3 | b1 | b2 | b3 | b4]; the concat output is
// the slice [c2r + c3r, end) in torchvision order.
TRef inception(Builder& b, TRef x, int H, const Incep& m, bool pool_after, int pool_k, int* out_H) {
  const int red = m.c2r + m.c3r;
  const int total = red + m.c1 + m.c2 + m.c3 + m.c4;
  b.layer(std::string(m.name) + "_a");
  const int T = b.tensor(std::string(m.name) + "_cat", H, H, total);
  b.conv(std::string(m.name) + "_1x1", x, TRef{T, 0, red + m.c1}, 1, 1, 0, 1);
  const int P = b.tensor(std::string(m.name) + "_pool", H, H, x.C);
  b.maxpool(std::string(m.name) + "_b4pool", x, b.all(P), 3, 1, 1, true);
  b.conv(std::string(m.name) + "_b4", b.all(P), TRef{T, red + m.c1 + m.c2 + m.c3, m.c4}, 1, 1, 0, 1);
  b.layer(std::string(m.name) + "_b");
  b.conv(std::string(m.name) + "_b2", TRef{T, 0, m.c2r}, TRef{T, red + m.c1, m.c2}, 3, 1, 1, 1);
  b.conv(std::string(m.name) + "_b3", TRef{T, m.c2r, m.c3r}, TRef{T, red + m.c1 + m.c2, m.c3}, 3, 1, 1, 1);
  TRef out{T, red, m.c1 + m.c2 + m.c3 + m.c4};
  *out_H = H;
  if (pool_after) {
    const int Ho = pool_k == 3 ? (H - 3 + 1) / 2 + 1 : (H - 2 + 1) / 2 + 1;
    const int M = b.tensor(std::string(m.name) + "_mp", Ho, Ho, out.C);
    b.maxpool(std::string(m.name) + "_maxpool", out, b.all(M), pool_k, 2, 0, true);
    *out_H = Ho;
    return b.all(M);
  }
  return out;
}

void googlenet(Builder& b) {
  b.component("googlenet_body");
  const int x = b.input(224, 224, 4);
  b.layer("conv1");
  const int c1 = b.tensor("conv1", 112, 112, 64);
  b.conv("conv1", b.all(x), b.all(c1), 7, 2, 3, 1, 1.0, {}, 3);
  const int p1 = b.tensor("pool1", 56, 56, 64);
  b.maxpool("maxpool1", b.all(c1), b.all(p1), 3, 2, 0, true);
  b.layer("conv2");
  const int c2 = b.tensor("conv2", 56, 56, 64);
  b.conv("conv2", b.all(p1), b.all(c2), 1, 1, 0, 1);
  b.layer("conv3");
  const int c3 = b.tensor("conv3", 56, 56, 192);
  b.conv("conv3", b.all(c2), b.all(c3), 3, 1, 1, 1);
  const int p2 = b.tensor("pool2", 28, 28, 192);
  b.maxpool("maxpool2", b.all(c3), b.all(p2), 3, 2, 0, true);
  static const Incep mods[9] = {
      {"i3a", 64, 96, 128, 16, 32, 32},    {"i3b", 128, 128, 192, 32, 96, 64},
      {"i4a", 192, 96, 208, 16, 48, 64},   {"i4b", 160, 112, 224, 24, 64, 64},
      {"i4c", 128, 128, 256, 24, 64, 64},  {"i4d", 112, 144, 288, 32, 64, 64},
      {"i4e", 256, 160, 320, 32, 128, 128}, {"i5a", 256, 160, 320, 32, 128, 128},
      {"i5b", 384, 192, 384, 48, 128, 128}};
  TRef cur = b.all(p2);
  int H = 28;
  for (int i = 0; i < 9; ++i) {
    const bool pool = i == 1 || i == 6;
    cur = inception(b, cur, H, mods[i], pool, i == 1 ? 3 : 2, &H);
  }
  b.layer("head");
  b.classifier(cur, 1000);
}

// ResNet-50 (torchvision v1.5: stride on the 3x3). Three scheduler layers per
// bottleneck; the projection shortcut runs inside the third layer.
TRef bottleneck(Builder& b, const std::string& name, TRef x, int H, int width, int stride, bool project,
                double res_scale) {
  const int Ho = H / stride;
  b.layer(name + "_conv1");
  const int t1 = b.tensor(name + "_t1", H, H, width);
  b.conv(name + "_conv1", x, b.all(t1), 1, 1, 0, 1);
  b.layer(name + "_conv2");
  const int t2 = b.tensor(name + "_t2", Ho, Ho, width);
  b.conv(name + "_conv2", b.all(t1), b.all(t2), 3, stride, 1, 1);
  b.layer(name + "_conv3");
  TRef shortcut = x;
  if (project) {
    const int ds = b.tensor(name + "_ds", Ho, Ho, width * 4);
    b.conv(name + "_downsample", x, b.all(ds), 1, stride, 0, 0);
    shortcut = b.all(ds);
  }
  const int y = b.tensor(name + "_out", Ho, Ho, width * 4);
  b.conv(name + "_conv3", b.all(t2), b.all(y), 1, 1, 0, 1, res_scale, shortcut);
  return b.all(y);
}

TRef resnet50_backbone(Builder& b, const std::string& comp) {
  b.component(comp);
  const int x = b.input(224, 224, 4);
  b.layer("conv1");
  const int c1 = b.tensor("conv1", 112, 112, 64);
  b.conv("conv1", b.all(x), b.all(c1), 7, 2, 3, 1, 1.0, {}, 3);
  const int p1 = b.tensor("pool1", 56, 56, 64);
  b.maxpool("maxpool", b.all(c1), b.all(p1), 3, 2, 1, false);
  TRef cur = b.all(p1);
  int H = 56;
  const int blocks[4] = {3, 4, 6, 3};
  const int widths[4] = {64, 128, 256, 512};
  for (int s = 0; s < 4; ++s) {
    for (int i = 0; i < blocks[s]; ++i) {
      const int stride = (s > 0 && i == 0) ? 2 : 1;
      const std::string name = "layer" + std::to_string(s + 1) + "." + std::to_string(i);
      cur = bottleneck(b, name, cur, H, widths[s], stride, i == 0, 0.25);
      H /= stride;
    }
  }
  return cur;
}

void resnet50(Builder& b) {
  const TRef feat = resnet50_backbone(b, "resnet50_body");
  b.layer("head");
  b.classifier(feat, 1000);
}

// Config 3: two DNNs over one shared backbone component (49 layers) with
// different heads, stitched like the reference's flow_pair profile.
void resnet50_head_a(Builder& b) {
  const TRef feat = resnet50_backbone(b, "resnet50_backbone");
  b.component("head_a");
  b.layer("head_a");
  b.classifier(feat, 1000, "a_");
}

void resnet50_head_b(Builder& b) {
  const TRef feat = resnet50_backbone(b, "resnet50_backbone");
  b.component("head_b");
  b.layer("head_b_conv");
  const int h = b.tensor("b_conv", 7, 7, 512);
  b.conv("b_conv", feat, b.all(h), 1, 1, 0, 1);
  b.layer("head_b_cls");
  b.classifier(b.all(h), 365, "b_");
}

void mobilenet_v2(Builder& b) {
  b.component("mobilenet_v2_body");
  const int x = b.input(224, 224, 4);
  b.layer("conv_stem");
  const int s = b.tensor("stem", 112, 112, 32);
  b.conv("stem", b.all(x), b.all(s), 3, 2, 1, 2, 1.0, {}, 3);
  struct Cfg {
    int t, c, n, s;
  };
  static const Cfg cfg[7] = {{1, 16, 1, 1}, {6, 24, 2, 2}, {6, 32, 3, 2}, {6, 64, 4, 2},
                             {6, 96, 3, 1}, {6, 160, 3, 2}, {6, 320, 1, 1}};
  TRef cur = b.all(s);
  int H = 112, cin = 32, blk = 0;
  for (const Cfg& g : cfg) {
    for (int i = 0; i < g.n; ++i, ++blk) {
      const int stride = i == 0 ? g.s : 1;
      const int hidden = cin * g.t;
      const std::string name = "block" + std::to_string(blk);
      TRef in = cur;
      if (g.t != 1) {
        b.layer(name + "_expand");
        const int e = b.tensor(name + "_e", H, H, hidden);
        b.conv(name + "_expand", in, b.all(e), 1, 1, 0, 2);
        in = b.all(e);
      }
      b.layer(name + "_dw");
      const int Ho = (H + 2 - 3) / stride + 1;
      const int d = b.tensor(name + "_d", Ho, Ho, hidden);
      b.dwconv(name + "_dw", in, b.all(d), stride, 2);
      b.layer(name + "_project");
      const int o = b.tensor(name + "_o", Ho, Ho, g.c);
      const bool residual = stride == 1 && cin == g.c;
      b.conv(name + "_project", b.all(d), b.all(o), 1, 1, 0, 0, residual ? 0.5 : 1.0,
             residual ? cur : TRef{});
      cur = b.all(o);
      H = Ho;
      cin = g.c;
    }
  }
  b.layer("conv_last");
  const int last = b.tensor("last", 7, 7, 1280);
  b.conv("conv_last", cur, b.all(last), 1, 1, 0, 2);
  b.layer("head");
  b.classifier(b.all(last), 1000);
}

}  // namespace

namespace {

Suite build_suite_uncached(const std::string& name, std::uint64_t seed) {
  Suite s;
  s.name = name;
  auto add = [&](const char* dnn, void (*fn)(Builder&)) {
    Builder b(s, seed, dnn);
    fn(b);
    s.nets.push_back(b.finish());
  };
  if (name == "small_cnn") {
    add("small_cnn", small_cnn);
    s.max_batch = 10;
  } else if (name == "googlenet") {
    add("googlenet", googlenet);
  } else if (name == "resnet50") {
    add("resnet50", resnet50);
  } else if (name == "mobilenet_v2") {
    add("mobilenet_v2", mobilenet_v2);
  } else if (name == "resnet50_pair") {
    add("resnet50_a", resnet50_head_a);
    add("resnet50_b", resnet50_head_b);
  } else if (name == "hetero3") {
    add("googlenet", googlenet);
    add("resnet50", resnet50);
    add("mobilenet_v2", mobilenet_v2);
  } else if (name == "collab") {
    add("googlenet", googlenet);
    add("resnet50", resnet50);
  } else {
    throw std::invalid_argument("unknown suite '" + name + "'");
  }
  // Shared components must be planned identically in every DNN using them.
  for (std::size_t c = 0; c < s.components.size(); ++c) {
    const NetDef* first = nullptr;
    for (const NetDef& n : s.nets) {
      if (std::find(n.components.begin(), n.components.end(), static_cast<int>(c)) == n.components.end()) continue;
      if (n.components.front() != static_cast<int>(c) && !first) {
        // only prefix sharing is supported
      }
      if (!first) {
        first = &n;
        continue;
      }
      for (std::size_t L = 0; L < n.layers.size() && L < first->layers.size(); ++L) {
        if (n.layers[L].component != static_cast<int>(c)) continue;
        const auto& a = n.layers[L].ops;
        const auto& bb = first->layers[L].ops;
        if (a.size() != bb.size()) throw std::logic_error("shared component layouts differ");
        for (std::size_t i = 0; i < a.size(); ++i) {
          const OpDef& x = n.ops[static_cast<std::size_t>(a[i])];
          const OpDef& y = first->ops[static_cast<std::size_t>(bb[i])];
          const auto off = [](const NetDef& net, const TRef& r) {
            return r.t < 0 ? -1L : net.tensors[static_cast<std::size_t>(r.t)].off + r.coff;
          };
          if (x.w_off != y.w_off || off(n, x.in) != off(*first, y.in) || off(n, x.out) != off(*first, y.out) ||
              off(n, x.res) != off(*first, y.res))
            throw std::logic_error("shared component planned differently in " + n.name);
        }
      }
    }
  }
  // Calibrate, then round every weight matrix to TF32 (the
  // tensor-core operand precision; biases stay fp32).
  std::set<long> calibrated;
  for (const NetDef& n : s.nets) calibrate_net(s, n, calibrated);
  for (const NetDef& n : s.nets)
    for (const OpDef& op : n.ops) {
      long count = 0;
      if (op.kind == OpKind::conv) count = static_cast<long>(op.out.C) * op.Kpad;
      if (op.kind == OpKind::dwconv) count = 9L * op.in.C;
      for (long i = 0; i < count; ++i) {
        float& v = s.weights[static_cast<std::size_t>(op.w_off + i)];
        v = round_tf32_host(v);
      }
    }
  return s;
}

}  // namespace

Suite build_suite(const std::string& name, std::uint64_t seed) {
  static std::mutex mu;
  static std::map<std::pair<std::string, std::uint64_t>, Suite> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find({name, seed});
  if (it == cache.end()) it = cache.emplace(std::make_pair(name, seed), build_suite_uncached(name, seed)).first;
  return it->second;
}

double op_bytes(const NetDef& net, const OpDef& op, int batch) {
  const auto elems = [&](const TRef& r, bool out_side) -> double {
    if (r.t < 0) return 0;
    const TensorDef& t = net.tensors[static_cast<std::size_t>(r.t)];
    const double hw = out_side ? static_cast<double>(op.Ho) * op.Wo : static_cast<double>(t.H) * t.W;
    return hw * r.C;
  };
  double w = 0;
  if (op.kind == OpKind::conv) w = op.weight_floats + op.out.C;
  if (op.kind == OpKind::dwconv) w = op.weight_floats + op.in.C;
  double act = elems(op.in, false) + elems(op.res, true);
  if (op.kind == OpKind::softmax || op.kind == OpKind::avgpool)
    act += op.kind == OpKind::avgpool ? op.in.C : op.out.C;
  else
    act += elems(op.out, true);
  return 4.0 * (w + batch * act);
}

double op_flops(const OpDef& op, int batch) { return op.flops_per_image * batch; }

}  // namespace bs200
