// Deterministic weight calibration of the synthetic networks.
//
// He-normal random weights on white-noise images give input-INDEPENDENT
// outputs: every image's pooled features sit within a few percent of their
// expectation, so one class wins for every input and "identical top-1" checks
// nothing (round-1 verdict: 1 distinct GoogLeNet top-1 over 24 inputs, 3% of
// the logit magnitude input-dependent). This pass folds batch-norm with
// statistics of a fixed calibration batch into every conv / depthwise conv,
// the way a trained network's BN leaves them:
//   * per output channel c: pre-activation z_c (conv without bias, residual
//     excluded) gets mean 0 and std = gain over (calibration images x pixels);
//     gain = the op's residual-branch scale (ResNet 0.25, MobileNetV2 0.5),
//     else 1: w_c *= gain / sigma_c, b_c = -mu_c * gain / sigma_c (+ one std
//     before a ReLU, kReluShift);
//   * the classifier FC is centred per class on the calibration batch (its
//     logits are the input-dependent part only) and scaled by one scalar so
//     the logits have std kLogitStd.
// This is weight INITIALISATION, run once per suite on the host; the serving
// path never computes a layer on the CPU. The forward used here is a plain
// multithreaded fp32 loop nest whose every output element has a fixed
// accumulation order, so the weights are bit-identical for any thread count
// and on any host running this binary.
// -O3: the axpy loops need the vectoriser's runtime alias checks (-O2 skips them).
#pragma GCC optimize("O3")
#include <algorithm>
#include <cmath>
#include <cstring>
#include <set>
#include <thread>
#include <vector>

#include "image.hpp"
#include "netdef.hpp"

namespace bs200 {

namespace {

constexpr std::uint64_t kCalibSeed = 0x0CA11B4A7E5EEDULL;
constexpr int kCalibImages = 8;
constexpr double kLogitStd = 1.0;
// ReLU layers: pre-activation mean kReluShift (in units of its std), not 0.
// Fully centred ReLUs put the random network in the chaotic regime, where the
// fp32-vs-fp64 accumulation difference of every layer is amplified ~100x by
// the end (GoogLeNet logits 4e-5 on a CPU fp32 forward, 5e-4 on the tensor
// cores); a shift of one std cuts that 2.5-3x (ResNet-50 / GoogLeNet /
// MobileNetV2 <= 3e-5) while >= 99 of 128 inputs still get distinct top-1
// classes and every layer's RMS stays in [1, 6.2].
constexpr double kReluShift = 1.0;

template <class F>
void parallel_for(long n, F&& body) {
  const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  const long parts = std::min<long>(n, hw);
  if (parts <= 1) {
    for (long i = 0; i < n; ++i) body(i);
    return;
  }
  std::vector<std::thread> th;
  for (long t = 0; t < parts; ++t)
    th.emplace_back([&, t] {
      for (long i = t; i < n; i += parts) body(i);
    });
  for (auto& x : th) x.join();
}

struct View {
  float* base;  // tensor origin inside the blob
  int H, W, ldc, coff, C;
  float* px(int h, int w) const { return base + (static_cast<long>(h) * W + w) * ldc + coff; }
};

View view(const NetDef& net, std::vector<float>& blob, const TRef& r) {
  const TensorDef& t = net.tensors[static_cast<std::size_t>(r.t)];
  return View{blob.data() + t.off, t.H, t.W, t.C, r.coff, r.C};
}

// One output row of an implicit-GEMM conv: acc[ow][co] += x * wt[tap][ci][co]
// (no contraction: -ffp-contract=off; identical results with or without AVX
// because every lane is an independent mul + add in a fixed order).
__attribute__((target_clones("avx2", "default"))) void conv_row(const View& in, const float* __restrict wt,
                                                                 float* __restrict z, int oh, int Wo, int k,
                                                                 int stride, int pad, int cout) {
  const int cin = in.C;
  for (int ow = 0; ow < Wo; ++ow) {
    float* __restrict acc = z + static_cast<long>(ow) * cout;
    for (int kh = 0; kh < k; ++kh) {
      const int ih = oh * stride - pad + kh;
      if (ih < 0 || ih >= in.H) continue;
      for (int kw = 0; kw < k; ++kw) {
        const int iw = ow * stride - pad + kw;
        if (iw < 0 || iw >= in.W) continue;
        const float* x = in.px(ih, iw);
        const float* wrow = wt + static_cast<long>((kh * k + kw) * cin) * cout;
        for (int ci = 0; ci < cin; ++ci) {
          const float a = x[ci];
          if (a == 0.f) continue;
          const float* __restrict w = wrow + static_cast<long>(ci) * cout;
          for (int co = 0; co < cout; ++co) acc[co] += a * w[co];
        }
      }
    }
  }
}

// z[img][pixel][co] = sum_k col(img, pixel)[k] * W[co][k]  (no bias)
std::vector<float> conv_raw(const NetDef& net, const OpDef& op, std::vector<std::vector<float>>& blobs,
                            const float* w) {
  const int cin = op.in.C, cout = op.out.C, k = op.KH;
  const int K = k * k * cin;
  std::vector<float> wt(static_cast<std::size_t>(K) * cout);  // [K][Cout]
  for (int co = 0; co < cout; ++co)
    for (int kk = 0; kk < K; ++kk) wt[static_cast<std::size_t>(kk) * cout + co] = w[static_cast<long>(co) * op.Kpad + kk];
  const long P = static_cast<long>(op.Ho) * op.Wo;
  const int nb = static_cast<int>(blobs.size());
  std::vector<float> z(static_cast<std::size_t>(nb) * P * cout, 0.f);
  parallel_for(static_cast<long>(nb) * op.Ho, [&](long job) {
    const int b = static_cast<int>(job / op.Ho), oh = static_cast<int>(job % op.Ho);
    const View in = view(net, blobs[static_cast<std::size_t>(b)], op.in);
    conv_row(in, wt.data(), z.data() + (static_cast<std::size_t>(b) * P + static_cast<long>(oh) * op.Wo) * cout, oh,
             op.Wo, k, op.stride, op.pad, cout);
  });
  return z;
}

std::vector<float> dw_raw(const NetDef& net, const OpDef& op, std::vector<std::vector<float>>& blobs,
                          const float* w) {
  const int C = op.in.C;
  const long P = static_cast<long>(op.Ho) * op.Wo;
  const int nb = static_cast<int>(blobs.size());
  std::vector<float> z(static_cast<std::size_t>(nb) * P * C, 0.f);
  parallel_for(static_cast<long>(nb) * op.Ho, [&](long job) {
    const int b = static_cast<int>(job / op.Ho), oh = static_cast<int>(job % op.Ho);
    const View in = view(net, blobs[static_cast<std::size_t>(b)], op.in);
    for (int ow = 0; ow < op.Wo; ++ow) {
      float* acc = z.data() + (static_cast<std::size_t>(b) * P + static_cast<long>(oh) * op.Wo + ow) * C;
      for (int kh = 0; kh < 3; ++kh) {
        const int ih = oh * op.stride - 1 + kh;
        if (ih < 0 || ih >= in.H) continue;
        for (int kw = 0; kw < 3; ++kw) {
          const int iw = ow * op.stride - 1 + kw;
          if (iw < 0 || iw >= in.W) continue;
          const float* x = in.px(ih, iw);
          const float* wt = w + (kh * 3 + kw) * C;  // [3][3][C]
          for (int c = 0; c < C; ++c) acc[c] += x[c] * wt[c];
        }
      }
    }
  });
  return z;
}

// y = act(z + bias + res) into the op's output slice of every blob.
void finish_op(const NetDef& net, const OpDef& op, std::vector<std::vector<float>>& blobs,
               const std::vector<float>& z, const float* bias) {
  const int C = op.out.C;
  const long P = static_cast<long>(op.Ho) * op.Wo;
  for (std::size_t b = 0; b < blobs.size(); ++b) {
    const View out = view(net, blobs[b], op.out);
    for (long p = 0; p < P; ++p) {
      const int h = static_cast<int>(p / op.Wo), w = static_cast<int>(p % op.Wo);
      float* y = out.px(h, w);
      const float* zz = z.data() + (b * P + p) * C;
      const float* r = op.res.t >= 0 ? view(net, blobs[b], op.res).px(h, w) : nullptr;
      for (int c = 0; c < C; ++c) {
        float v = zz[c] + bias[c];
        if (r) v += r[c];
        if (op.relu == 1) v = std::max(v, 0.f);
        if (op.relu == 2) v = std::min(std::max(v, 0.f), 6.f);
        y[c] = v;
      }
    }
  }
}

void pool_op(const NetDef& net, const OpDef& op, std::vector<std::vector<float>>& blobs) {
  for (auto& blob : blobs) {
    const View in = view(net, blob, op.in), out = view(net, blob, op.out);
    if (op.kind == OpKind::avgpool) {
      float* y = out.px(0, 0);
      for (int c = 0; c < in.C; ++c) {
        double s = 0;
        for (int h = 0; h < in.H; ++h)
          for (int w = 0; w < in.W; ++w) s += in.px(h, w)[c];
        y[c] = static_cast<float>(s / (static_cast<double>(in.H) * in.W));
      }
      continue;
    }
    if (op.kind == OpKind::softmax) {
      const float* x = in.px(0, 0);
      float* y = out.px(0, 0);
      double mx = x[0], s = 0;
      for (int c = 1; c < in.C; ++c) mx = std::max<double>(mx, x[c]);
      for (int c = 0; c < in.C; ++c) s += std::exp(x[c] - mx);
      for (int c = 0; c < in.C; ++c) y[c] = static_cast<float>(std::exp(x[c] - mx) / s);
      continue;
    }
    for (int oh = 0; oh < op.Ho; ++oh)
      for (int ow = 0; ow < op.Wo; ++ow) {
        float* y = out.px(oh, ow);
        const int h0 = oh * op.stride - op.pad, w0 = ow * op.stride - op.pad;
        for (int c = 0; c < in.C; ++c) {
          float m = -INFINITY;
          for (int h = std::max(h0, 0); h < std::min(h0 + op.KH, in.H); ++h)
            for (int w = std::max(w0, 0); w < std::min(w0 + op.KW, in.W); ++w) m = std::max(m, in.px(h, w)[c]);
          y[c] = m;
        }
      }
  }
}

}  // namespace

void calibrate_net(Suite& s, const NetDef& net, std::set<long>& calibrated) {
  std::vector<std::vector<float>> blobs(kCalibImages, std::vector<float>(static_cast<std::size_t>(net.blob_floats), 0.f));
  const TensorDef& tin = net.tensors[static_cast<std::size_t>(net.input_t)];
  for (int i = 0; i < kCalibImages; ++i)
    synth_image(kCalibSeed, static_cast<std::uint64_t>(i), net.in_H, net.in_W, net.in_C, 3,
                blobs[static_cast<std::size_t>(i)].data() + tin.off);
  for (const OpDef& op : net.ops) {
    if (op.kind != OpKind::conv && op.kind != OpKind::dwconv) {
      pool_op(net, op, blobs);
      continue;
    }
    float* w = s.weights.data() + op.w_off;
    float* bias = s.weights.data() + op.b_off;
    std::vector<float> z = op.kind == OpKind::conv ? conv_raw(net, op, blobs, w) : dw_raw(net, op, blobs, w);
    const int C = op.out.C;
    if (!calibrated.count(op.w_off)) {
      calibrated.insert(op.w_off);
      const long n = static_cast<long>(z.size() / static_cast<std::size_t>(C));
      std::vector<double> mu(static_cast<std::size_t>(C), 0.0), var(static_cast<std::size_t>(C), 0.0);
      for (long i = 0; i < n; ++i)
        for (int c = 0; c < C; ++c) mu[static_cast<std::size_t>(c)] += z[static_cast<std::size_t>(i) * C + c];
      for (auto& m : mu) m /= static_cast<double>(n);
      for (long i = 0; i < n; ++i)
        for (int c = 0; c < C; ++c) {
          const double d = z[static_cast<std::size_t>(i) * C + c] - mu[static_cast<std::size_t>(c)];
          var[static_cast<std::size_t>(c)] += d * d;
        }
      double mean_var = 0;
      for (auto& v : var) mean_var += (v /= static_cast<double>(n));
      mean_var /= C;
      const bool classifier = op.out.t == net.logits_t;
      std::vector<double> scale(static_cast<std::size_t>(C));
      for (int c = 0; c < C; ++c) {
        // few samples per class at the classifier: one scalar scale
        const double sd = std::sqrt(classifier ? mean_var : std::max(var[static_cast<std::size_t>(c)], 1e-12 * mean_var));
        const double gain = classifier ? kLogitStd : (op.res.t >= 0 ? op.wscale : 1.0);
        scale[static_cast<std::size_t>(c)] = sd > 0 ? gain / sd : 1.0;
      }
      if (op.kind == OpKind::conv) {
        for (int c = 0; c < C; ++c)
          for (int kk = 0; kk < op.Kpad; ++kk)
            w[static_cast<long>(c) * op.Kpad + kk] =
                static_cast<float>(w[static_cast<long>(c) * op.Kpad + kk] * scale[static_cast<std::size_t>(c)]);
      } else {
        for (int t = 0; t < 9; ++t)
          for (int c = 0; c < C; ++c)
            w[t * C + c] = static_cast<float>(w[t * C + c] * scale[static_cast<std::size_t>(c)]);
      }
      const double shift = (op.relu && !classifier) ? kReluShift : 0.0;
      for (int c = 0; c < C; ++c)
        bias[c] = static_cast<float>(-mu[static_cast<std::size_t>(c)] * scale[static_cast<std::size_t>(c)] + shift);
      for (std::size_t i = 0; i < z.size(); ++i)
        z[i] = static_cast<float>(z[i] * scale[i % static_cast<std::size_t>(C)]);
    }
    finish_op(net, op, blobs, z, bias);
  }
}

}  // namespace bs200
