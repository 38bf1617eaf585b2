#include "executor.hpp"

#include <cstdlib>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>

#include "../kernels/conv_tc.cuh"
#include "../kernels/simple_ops.cuh"
#include "bsb/core.hpp"
#include "image.hpp"

namespace bs200 {

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

constexpr int kChunks = 64;

}  // namespace

Executor::Executor(int device, const std::string& suite_name, int max_batch, int max_requests)
    : suite_(build_suite(suite_name)), device_(device), max_batch_(max_batch) {
  ck(cudaSetDevice(device), "cudaSetDevice");
  ck(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "stream");
  // Admission and client-prefix streams at the highest priority: their
  // kernels are small and gate the next steps (ready events); at high load the
  // serving stream's persistent kernels -- and, with PDL, the next kernel's
  // CTAs parked in griddepcontrol.wait -- otherwise keep them waiting for SMs.
  {
    int lo = 0, hi = 0;
    ck(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
    ck(cudaStreamCreateWithPriority(&copy_, cudaStreamNonBlocking, hi), "copy stream");
    ck(cudaStreamCreateWithPriority(&side_, cudaStreamNonBlocking, hi), "side stream");
  }
  ck(cudaMalloc(&d_weights_, suite_.weights.size() * sizeof(float)), "weights");
  ck(cudaMemcpy(d_weights_, suite_.weights.data(), suite_.weights.size() * sizeof(float), cudaMemcpyHostToDevice),
     "weights H2D");
  for (const NetDef& n : suite_.nets) slot_floats_ = std::max<std::size_t>(slot_floats_, static_cast<std::size_t>(n.blob_floats));
  slot_floats_ = (slot_floats_ + 63) / 64 * 64;
  n_slots_ = max_requests;
  ready_ring_.resize(static_cast<std::size_t>(n_slots_) + 256);
  for (auto& e : ready_ring_) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "ready ring");
  {
    std::size_t mx = 0;
    for (const NetDef& n : suite_.nets) mx = std::max<std::size_t>(mx, static_cast<std::size_t>(n.in_H) * n.in_W * 3);
    staging_floats_ = (mx + 63) / 64 * 64;
    staging_n_ = 64;
    ck(cudaMalloc(&staging_, staging_floats_ * staging_n_), "rgb staging");
    ck(cudaMallocHost(&pack_host_, staging_floats_ * staging_n_), "rgb pack");
    pack_seq_.assign(static_cast<std::size_t>(staging_n_), 0);
    pack_ev_.resize(128);
    for (auto& e : pack_ev_) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "pack event");
  }
  // One slot space: [request slots | ride buffers | profiler scratch], so a
  // single TMA tensor map per layer input addresses every blob by slot index.
  n_ride_ = std::max(2 * max_batch_, 16);
  total_slots_ = static_cast<long>(n_slots_) + n_ride_ + max_batch_;
  ck(cudaMalloc(&arena_, static_cast<std::size_t>(total_slots_) * slot_floats_ * sizeof(float)), "arena");
  for (int i = n_slots_ - 1; i >= 0; --i) free_.push_back(i);
  // A freed slot may still be read by work queued on the serving stream (the
  // retiring request's D2H copy of its probabilities); its next admission
  // writes it from the copy or side stream, so it first waits on this event.
  slot_free_.assign(static_cast<std::size_t>(n_slots_), FreeMark{});
  free_ring_.resize(4096);
  for (auto& e : free_ring_) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "slot event");
  ride_arena_ = arena_ + static_cast<std::size_t>(n_slots_) * slot_floats_;
  for (int i = n_ride_ - 1; i >= 0; --i) ride_free_.push_back(i);
  int max_layers = 1;
  for (const NetDef& n : suite_.nets) max_layers = std::max(max_layers, n.num_layers());
  chunk_cap_ = static_cast<std::size_t>(max_layers) * static_cast<std::size_t>(max_batch_ + n_ride_) + 64;
  ck(cudaMalloc(&stamps_, kStampCap * sizeof(unsigned long long)), "step stamps");
  ck(cudaMemset(stamps_, 0, kStampCap * sizeof(unsigned long long)), "step stamps");
  chunks_.resize(kChunks);
  for (auto& c : chunks_) {
    ck(cudaMallocHost(&c.host, chunk_cap_ * sizeof(float*)), "pinned table");
    ck(cudaMalloc(&c.dev, chunk_cap_ * sizeof(float*)), "device table");
    ck(cudaEventCreateWithFlags(&c.done, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&c.uploaded, cudaEventDisableTiming), "event");
  }
  {
    const char* tm = std::getenv("BS_TABLE_MODE");
    if (tm && tm[0] >= '0' && tm[0] <= '2') table_mode_ = tm[0] - '0';
    int lo = 0, hi = 0;
    ck(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
    ck(cudaStreamCreateWithPriority(&table_, cudaStreamNonBlocking, hi), "table stream");
  }
  // Scratch blobs for the profiler (max_batch of them) + an L2 flush buffer.
  scratch_ = ride_arena_ + static_cast<std::size_t>(n_ride_) * slot_floats_;
  ck(cudaMemset(scratch_, 0, static_cast<std::size_t>(max_batch_) * slot_floats_ * sizeof(float)), "scratch zero");
  ck(cudaMalloc(&scratch_ptrs_, max_batch_ * sizeof(float*)), "scratch ptrs");
  std::vector<float*> hp(static_cast<std::size_t>(max_batch_));
  for (int i = 0; i < max_batch_; ++i) hp[static_cast<std::size_t>(i)] = scratch_ + static_cast<std::size_t>(i) * slot_floats_;
  ck(cudaMemcpy(scratch_ptrs_, hp.data(), hp.size() * sizeof(float*), cudaMemcpyHostToDevice), "scratch ptrs H2D");
  pool_.assign(suite_.nets.size(), nullptr);
  pool_n_.assign(suite_.nets.size(), 0);
  // One TMA descriptor per conv/FC weight matrix (weights never move).
  wmaps_.resize(suite_.nets.size());
  wmaps_wide_.resize(suite_.nets.size());
  wmaps_mid_.resize(suite_.nets.size());
  wmaps_mid160_.resize(suite_.nets.size());
  for (std::size_t n = 0; n < suite_.nets.size(); ++n) {
    const NetDef& net = suite_.nets[n];
    wmaps_[n].resize(net.ops.size());
    wmaps_wide_[n].resize(net.ops.size());
    wmaps_mid_[n].resize(net.ops.size());
    wmaps_mid160_[n].resize(net.ops.size());
    for (std::size_t i = 0; i < net.ops.size(); ++i) {
      const OpDef& op = net.ops[i];
      if (op.kind != OpKind::conv) continue;
      if (!encode_weight_map(&wmaps_[n][i], d_weights_ + op.w_off, op.out.C, op.Kpad))
        throw std::runtime_error("cuTensorMapEncodeTiled failed for " + op.name);
      if (op.out.C > 128 &&
          !encode_weight_map(&wmaps_wide_[n][i], d_weights_ + op.w_off, op.out.C, op.Kpad, 256))
        throw std::runtime_error("cuTensorMapEncodeTiled (wide) failed for " + op.name);
      if (op.out.C > 128 &&
          !encode_weight_map(&wmaps_mid_[n][i], d_weights_ + op.w_off, op.out.C, op.Kpad, 192))
        throw std::runtime_error("cuTensorMapEncodeTiled (mid) failed for " + op.name);
      if (op.out.C > 128 &&
          !encode_weight_map(&wmaps_mid160_[n][i], d_weights_ + op.w_off, op.out.C, op.Kpad, 160))
        throw std::runtime_error("cuTensorMapEncodeTiled (mid160) failed for " + op.name);
    }
  }
  // Tap-row mode for the stems (default; BS_CONV_TAPROW=0 disables): one K
  // tile per filter row, so the A gather is one contiguous 128-byte segment
  // per output pixel and K tile. Weights re-laid to match.
  {
    const char* tr_env = std::getenv("BS_CONV_TAPROW");
    const bool use_tr = !(tr_env && tr_env[0] == '0');
    taps_.resize(suite_.nets.size());
    std::vector<float> pool;
    std::vector<std::pair<std::size_t, std::size_t>> where;
    for (std::size_t n = 0; n < suite_.nets.size() && use_tr; ++n) {
      const NetDef& net = suite_.nets[n];
      taps_[n].resize(net.ops.size());
      for (std::size_t i = 0; i < net.ops.size(); ++i) {
        const OpDef& op = net.ops[i];
        if (op.kind != OpKind::conv || op.out.C > 128 || !conv_tap_rows_eligible(op.in.C, op.KW)) continue;
        TapRowMap& tm = taps_[n][i];
        tm.w_off = pool.size();
        pool.resize(pool.size() + static_cast<std::size_t>(op.out.C) * op.KH * 32);
        conv_tap_row_weights(suite_.weights.data() + op.w_off, op.out.C, op.Kpad, op.KH, op.KW, op.in.C,
                             pool.data() + tm.w_off);
        where.emplace_back(n, i);
      }
    }
    tap_pool_floats_ = pool.size();
    if (!pool.empty()) {
      ck(cudaMalloc(&d_tap_weights_, pool.size() * sizeof(float)), "tap-row weights");
      ck(cudaMemcpy(d_tap_weights_, pool.data(), pool.size() * sizeof(float), cudaMemcpyHostToDevice),
         "tap-row weights H2D");
    }
    for (const auto& [n, i] : where) {
      const OpDef& op = suite_.nets[n].ops[i];
      TapRowMap& tm = taps_[n][i];
      tm.ok = encode_weight_map(&tm.wmap, d_tap_weights_ + tm.w_off, op.out.C, op.KH * 32);
      if (!tm.ok) throw std::runtime_error("tap-row weight map failed for " + op.name);
    }
  }
  plan_groups();
}

// Launch order per layer. Two convs of a layer are grouped into one launch
// when neither reads or writes what the other writes (channel slices of one
// tensor, or the arena ranges of different tensors, which the planner may
// alias): the two branch convs of an inception block, or -- by running a
// pooling op first -- the merged 1x1 conv and the pool projection.
void Executor::plan_groups() {
  const char* env = std::getenv("BS_CONV_GROUP");
  const bool on = !(env && env[0] == '0');
  plans_.assign(suite_.nets.size(), {});
  gmaps_.assign(suite_.nets.size(), {});
  gmap_ok_.assign(suite_.nets.size(), {});
  gmaps192_.assign(suite_.nets.size(), {});
  gmap192_ok_.assign(suite_.nets.size(), {});
  for (std::size_t n = 0; n < suite_.nets.size(); ++n) {
    const NetDef& net = suite_.nets[n];
    gmaps_[n].resize(net.ops.size());
    gmap_ok_[n].assign(net.ops.size(), 0);
    gmaps192_[n].resize(net.ops.size());
    gmap192_ok_[n].assign(net.ops.size(), 0);
    auto overlap = [&](const TRef& x, const TRef& y) {
      if (x.t < 0 || y.t < 0) return false;
      if (x.t == y.t) return x.coff < y.coff + y.C && y.coff < x.coff + x.C;
      const TensorDef& a = net.tensors[static_cast<std::size_t>(x.t)];
      const TensorDef& b = net.tensors[static_cast<std::size_t>(y.t)];
      const long ae = a.off + static_cast<long>(a.H) * a.W * a.C, be = b.off + static_cast<long>(b.H) * b.W * b.C;
      return a.off < be && b.off < ae;
    };
    // No ordering constraint between x and y (either may run first / both at once).
    auto indep = [&](const OpDef& x, const OpDef& y) {
      return !overlap(x.out, y.in) && !overlap(x.out, y.res) && !overlap(y.out, x.in) && !overlap(y.out, x.res) &&
             !overlap(x.out, y.out);
    };
    auto groupable = [&](int i) {
      const OpDef& op = net.ops[static_cast<std::size_t>(i)];
      const auto k = static_cast<std::size_t>(i);
      return op.kind == OpKind::conv && !(n < taps_.size() && k < taps_[n].size() && taps_[n][k].ok);
    };
    for (const LayerDef& L : net.layers) {
      std::vector<LayerItem> items;
      const std::vector<int>& o = L.ops;
      std::size_t i = 0;
      while (i < o.size()) {
        const int a = o[i];
        if (on && groupable(a)) {
          if (i + 1 < o.size() && groupable(o[i + 1]) &&
              indep(net.ops[static_cast<std::size_t>(a)], net.ops[static_cast<std::size_t>(o[i + 1])])) {
            items.push_back({a, o[i + 1]});
            i += 2;
            continue;
          }
          if (i + 2 < o.size() && net.ops[static_cast<std::size_t>(o[i + 1])].kind != OpKind::conv &&
              groupable(o[i + 2]) &&
              indep(net.ops[static_cast<std::size_t>(a)], net.ops[static_cast<std::size_t>(o[i + 1])]) &&
              indep(net.ops[static_cast<std::size_t>(a)], net.ops[static_cast<std::size_t>(o[i + 2])])) {
            items.push_back({o[i + 1], -1});  // the pool runs first
            items.push_back({a, o[i + 2]});
            i += 3;
            continue;
          }
        }
        items.push_back({a, -1});
        ++i;
      }
      // Weight maps at the group's tile width for the narrower conv of a pair.
      for (const LayerItem& it : items) {
        if (it.b < 0) continue;
        const OpDef& x = net.ops[static_cast<std::size_t>(it.a)];
        const OpDef& y = net.ops[static_cast<std::size_t>(it.b)];
        const int bn = std::max(conv_tile_n(x.out.C), conv_tile_n(y.out.C));
        for (int k : {it.a, it.b}) {
          const OpDef& op = net.ops[static_cast<std::size_t>(k)];
          if (conv_tile_n(op.out.C) == bn) continue;
          if (!encode_weight_map(&gmaps_[n][static_cast<std::size_t>(k)], d_weights_ + op.w_off, op.out.C, op.Kpad, bn))
            throw std::runtime_error("group weight map failed for " + op.name);
          gmap_ok_[n][static_cast<std::size_t>(k)] = 1;
        }
        // 192-row maps of both convs when the wider one spans more than one
        // 128-wide tile (the launcher may run the pair as 128 x 192 tiles)
        if (std::max(x.out.C, y.out.C) > 128)
          for (int k : {it.a, it.b}) {
            const OpDef& op = net.ops[static_cast<std::size_t>(k)];
            if (!encode_weight_map(&gmaps192_[n][static_cast<std::size_t>(k)], d_weights_ + op.w_off, op.out.C,
                                   op.Kpad, 192))
              throw std::runtime_error("group weight map (192) failed for " + op.name);
            gmap192_ok_[n][static_cast<std::size_t>(k)] = 1;
          }
      }
      plans_[n].push_back(std::move(items));
    }
  }
}

Executor::~Executor() {
  cudaSetDevice(device_);
  if (stream_) cudaStreamSynchronize(stream_);
  if (side_) cudaStreamSynchronize(side_);
  for (auto& c : chunks_) {
    cudaFreeHost(c.host);
    cudaFree(c.dev);
    cudaEventDestroy(c.done);
    cudaEventDestroy(c.uploaded);
  }
  if (copy_) cudaStreamSynchronize(copy_);
  cudaFree(stamps_);
  for (cudaEvent_t e : ready_ring_) cudaEventDestroy(e);
  for (cudaEvent_t e : free_ring_) cudaEventDestroy(e);
  cudaFree(staging_);
  cudaFreeHost(pack_host_);
  for (cudaEvent_t e : pack_ev_) cudaEventDestroy(e);
  for (cudaEvent_t e : event_pool_) cudaEventDestroy(e);
  for (float* p : pool_) cudaFree(p);
  cudaFree(d_weights_);
  cudaFree(d_tap_weights_);
  cudaFree(d_weights_bf16_);
  cudaFree(d_tap_weights_bf16_);
  cudaFree(arena_);
  cudaFree(scratch_ptrs_);
  cudaFree(flush_);
  cudaStreamDestroy(stream_);
  cudaStreamDestroy(side_);
  cudaStreamDestroy(copy_);
  cudaStreamDestroy(table_);
}

cudaEvent_t Executor::next_ready_event() {
  cudaEvent_t e = ready_ring_[ready_next_];
  ready_next_ = (ready_next_ + 1) % ready_ring_.size();
  return e;
}

std::vector<std::uint64_t> Executor::stamps() {
  std::vector<std::uint64_t> v(kStampCap);
  ck(cudaMemcpy(v.data(), stamps_, v.size() * sizeof(std::uint64_t), cudaMemcpyDeviceToHost), "stamps D2H");
  return v;
}

void Executor::sync() {
  ck(cudaStreamSynchronize(copy_), "sync copy");
  ck(cudaStreamSynchronize(stream_), "sync");
}

void Executor::set_precision(const std::string& mode) {
  if (mode == "tf32x2") prec_ = 1;
  else if (mode == "tf32") prec_ = 0;
  else if (mode == "bf16") {
    build_bf16();
    prec_ = 2;
  } else {
    throw std::invalid_argument("unknown precision '" + mode + "' (tf32x2 | tf32 | bf16)");
  }
}

void Executor::build_bf16() {
  if (bf16_ready_) return;
  ck(cudaMalloc(&d_weights_bf16_, suite_.weights.size() * 2), "bf16 weights");
  ck(launch_to_bf16(d_weights_, d_weights_bf16_, suite_.weights.size(), stream_), "bf16 weights");
  if (tap_pool_floats_) {
    ck(cudaMalloc(&d_tap_weights_bf16_, tap_pool_floats_ * 2), "bf16 tap-row weights");
    ck(launch_to_bf16(d_tap_weights_, d_tap_weights_bf16_, tap_pool_floats_, stream_), "bf16 tap-row weights");
  }
  ck(cudaStreamSynchronize(stream_), "bf16 weights");
  wmaps_bf_.assign(suite_.nets.size(), {});
  wmaps_wide_bf_.assign(suite_.nets.size(), {});
  gmaps_bf_.assign(suite_.nets.size(), {});
  for (std::size_t n = 0; n < suite_.nets.size(); ++n) {
    const NetDef& net = suite_.nets[n];
    wmaps_bf_[n].resize(net.ops.size());
    wmaps_wide_bf_[n].resize(net.ops.size());
    gmaps_bf_[n].resize(net.ops.size());
    for (std::size_t i = 0; i < net.ops.size(); ++i) {
      const OpDef& op = net.ops[i];
      if (op.kind != OpKind::conv) continue;
      const std::uint16_t* w = d_weights_bf16_ + op.w_off;
      bool ok = encode_weight_map_bf16(&wmaps_bf_[n][i], w, op.out.C, op.Kpad);
      if (op.out.C > 128) ok = ok && encode_weight_map_bf16(&wmaps_wide_bf_[n][i], w, op.out.C, op.Kpad, 256);
      if (gmap_ok_[n][i]) {
        // the group's tile width: the wider of the pair (plan_groups)
        int bn = conv_tile_n(op.out.C);
        for (const auto& items : plans_[n])
          for (const LayerItem& it : items)
            if (it.b >= 0 && (it.a == static_cast<int>(i) || it.b == static_cast<int>(i)))
              bn = std::max(conv_tile_n(net.ops[static_cast<std::size_t>(it.a)].out.C),
                            conv_tile_n(net.ops[static_cast<std::size_t>(it.b)].out.C));
        ok = ok && encode_weight_map_bf16(&gmaps_bf_[n][i], w, op.out.C, op.Kpad, bn);
      }
      if (n < taps_.size() && i < taps_[n].size() && taps_[n][i].ok)
        ok = ok && encode_weight_map_bf16(&taps_[n][i].wmap_bf, d_tap_weights_bf16_ + taps_[n][i].w_off, op.out.C,
                                          op.KH * 32);
      if (!ok) throw std::runtime_error("bf16 weight tensor maps failed for " + op.name);
    }
  }
  bf16_ready_ = true;
}

// ------------------------------------------------------------------ tables

float** Executor::table_alloc(std::size_t n, float*** host_view) {
  if (n > chunk_cap_) throw std::runtime_error("pointer table overflow");
  if (chunk_used_ + n > chunk_cap_) throw std::runtime_error("pointer chunk overflow");
  TableChunk& c = chunks_[chunk_];
  *host_view = c.host + chunk_used_;
  float** d = c.dev + chunk_used_;
  chunk_used_ += n;
  return d;
}

// ------------------------------------------------------------------ launch

ConvParams Executor::conv_params(const NetDef& net, const OpDef& op, float* const* d_ptrs, int batch) const {
  const auto off = [&](const TRef& r) -> long {
    return r.t < 0 ? 0 : net.tensors[static_cast<std::size_t>(r.t)].off + r.coff;
  };
  const auto ldc = [&](const TRef& r) -> int { return r.t < 0 ? 0 : net.tensors[static_cast<std::size_t>(r.t)].C; };
  const TensorDef& ti = net.tensors[static_cast<std::size_t>(op.in.t)];
  ConvParams p{};
  const bool bf = prec_ == 2;
  {
    const std::size_t ni = static_cast<std::size_t>(&net - suite_.nets.data());
    const std::size_t oi = static_cast<std::size_t>(&op - net.ops.data());
    p.wmap = bf ? wmaps_bf_[ni][oi] : wmaps_[ni][oi];
    if (op.out.C > 128) conv_add_wide_map(p, bf ? wmaps_wide_bf_[ni][oi] : wmaps_wide_[ni][oi]);
    if (op.out.C > 128 && !bf) conv_add_mid_map(p, wmaps_mid_[ni][oi]);
    if (op.out.C > 128 && !bf) conv_add_mid160_map(p, wmaps_mid160_[ni][oi]);
  }
  p.nimg = batch;
  p.H = ti.H;
  p.W = ti.W;
  p.Cin = op.in.C;
  p.Ho = op.Ho;
  p.Wo = op.Wo;
  p.KH = op.KH;
  p.KW = op.KW;
  p.stride = op.stride;
  p.pad = op.pad;
  p.K = op.KH * op.KW * op.in.C;
  p.Kpad = op.Kpad;
  p.N = op.out.C;
  p.in_ptrs = input_ptrs(net, op, d_ptrs);
  p.in_off = off(op.in);
  p.in_ldc = ldc(op.in);
  p.wgt = d_weights_ + op.w_off;
  p.bias = d_weights_ + op.b_off;
  p.out_ptrs = d_ptrs;
  p.out_off = off(op.out);
  p.out_ldc = ldc(op.out);
  p.res_ptrs = op.res.t >= 0 ? d_ptrs : nullptr;
  p.res_off = off(op.res);
  p.res_ldc = ldc(op.res);
  p.relu = op.relu;
  p.round_out = prec_ == 0 ? op.round_out : 0;
  p.prec = prec_;
  {
    const std::size_t ni = static_cast<std::size_t>(&net - suite_.nets.data());
    const std::size_t oi = static_cast<std::size_t>(&op - net.ops.data());
    ConvChoice c{};
    if (static_cast<int>(ni) == tune_net_ && static_cast<int>(oi) == tune_op_) {
      c = tune_choice_;
    } else {
      const int t = tuned_index(batch);
      if (t >= 0 && ni < conv_pref_.size() && oi < conv_pref_[ni].size() && !conv_pref_[ni][oi].empty())
        c = conv_pref_[ni][oi][static_cast<std::size_t>(t)];
    }
    p.wide_pref = c.wide;
    p.ks_force = c.ks;
  }
  {
    const std::size_t ni = static_cast<std::size_t>(&net - suite_.nets.data());
    const std::size_t oi = static_cast<std::size_t>(&op - net.ops.data());
    if (ni < taps_.size() && oi < taps_[ni].size() && taps_[ni][oi].ok) {
      p.tap_rows = 1;
      p.Kpad = op.KH * 32;
      p.wmap = bf ? taps_[ni][oi].wmap_bf : taps_[ni][oi].wmap;
      p.wgt = d_tap_weights_ + taps_[ni][oi].w_off;
    }
  }
  return p;
}

void Executor::launch_group(const NetDef& net, int layer, int item, const OpDef& a, const OpDef& b,
                            float* const* d_ptrs, int batch) {
  const std::size_t ni = static_cast<std::size_t>(&net - suite_.nets.data());
  // Grouped or separate: the tuning override, else the tuned choice of the
  // nearest batch, else the launcher's rule (declines for split / wide).
  int pref = 0;
  if (static_cast<int>(ni) == tune_net_ && layer == tune_layer_ && item == tune_item_) {
    pref = tune_group_;
  } else {
    const int t = tuned_index(batch);
    if (t >= 0 && ni < group_pref_.size()) {
      const auto& g = group_pref_[ni][static_cast<std::size_t>(layer - 1)][static_cast<std::size_t>(item)];
      if (!g.empty()) pref = g[static_cast<std::size_t>(t)];
    }
  }
  if (pref < 0) {
    launch_op(net, a, d_ptrs, batch);
    launch_op(net, b, d_ptrs, batch);
    return;
  }
  ConvParams pa = conv_params(net, a, d_ptrs, batch), pb = conv_params(net, b, d_ptrs, batch);
  const std::size_t ia = static_cast<std::size_t>(&a - net.ops.data()), ib = static_cast<std::size_t>(&b - net.ops.data());
  if (gmap_ok_[ni][ia]) pa.wmap = prec_ == 2 ? gmaps_bf_[ni][ia] : gmaps_[ni][ia];
  if (gmap_ok_[ni][ib]) pb.wmap = prec_ == 2 ? gmaps_bf_[ni][ib] : gmaps_[ni][ib];
  // group maps at 192 rows (launch_conv_tc_group's 128 x 192 option)
  pa.wmap_mid = prec_ != 2 && gmap192_ok_[ni][ia] ? &gmaps192_[ni][ia] : nullptr;
  pb.wmap_mid = prec_ != 2 && gmap192_ok_[ni][ib] ? &gmaps192_[ni][ib] : nullptr;
  pa.wmap_mid160 = pb.wmap_mid160 = nullptr;
  LaunchStat st{};
  const bool sample = stats_on_ && (++stats_seen_ % stats_every_ == 0) && ev_next_ + 2 <= event_pool_.size();
  if (sample) {
    st.kind = OpKind::conv;
    st.batch = batch;
    st.bytes = op_bytes(net, a, batch) + op_bytes(net, b, batch);
    st.flops = op_flops(a, batch) + op_flops(b, batch);
    st.t0 = event_pool_[ev_next_++];
    st.t1 = event_pool_[ev_next_++];
    ck(cudaEventRecord(st.t0, stream_), "ev rec");
  }
  const cudaError_t e = launch_conv_tc_group(pa, pb, stream_, pref > 0, std::max(1, pref));
  if (e == cudaErrorNotSupported) {  // split-K / wide tiles win at this batch
    if (sample) {
      ev_next_ -= 2;
      --stats_seen_;
    }
    launch_op(net, a, d_ptrs, batch);
    launch_op(net, b, d_ptrs, batch);
    return;
  }
  ck(e, (a.name + "+" + b.name).c_str());
  ++launches_;
  if (sample) {
    ck(cudaEventRecord(st.t1, stream_), "ev rec");
    stats_.push_back(st);
  }
}

void Executor::launch_op(const NetDef& net, const OpDef& op, float* const* d_ptrs, int batch) {
  const auto off = [&](const TRef& r) -> long {
    return r.t < 0 ? 0 : net.tensors[static_cast<std::size_t>(r.t)].off + r.coff;
  };
  const auto ldc = [&](const TRef& r) -> int { return r.t < 0 ? 0 : net.tensors[static_cast<std::size_t>(r.t)].C; };
  const TensorDef& ti = net.tensors[static_cast<std::size_t>(op.in.t)];
  LaunchStat st{};
  const bool sample = stats_on_ && (++stats_seen_ % stats_every_ == 0) && ev_next_ + 2 <= event_pool_.size();
  if (sample) {
    st.kind = op.kind;
    st.batch = batch;
    st.bytes = op_bytes(net, op, batch);
    st.flops = op_flops(op, batch);
    st.t0 = event_pool_[ev_next_++];
    st.t1 = event_pool_[ev_next_++];
    ck(cudaEventRecord(st.t0, stream_), "ev rec");
  }
  cudaError_t e = cudaSuccess;
  switch (op.kind) {
    case OpKind::conv: {
      const ConvParams cp = conv_params(net, op, d_ptrs, batch);
      // small-batch FC: weight-streaming GEMV (BS_FC_GEMV=0 keeps conv_tc)
      static const bool gemv_on = [] {
        const char* v = std::getenv("BS_FC_GEMV");
        return !(v && std::atoi(v) == 0);
      }();
      if (gemv_on && prec_ != 2 && cp.H == 1 && cp.W == 1 && cp.KH == 1 && cp.KW == 1 && cp.nimg <= kFcMaxImg &&
          !cp.res_ptrs && !cp.round_out && cp.in_off % 4 == 0 && cp.K % 4 == 0 && cp.K <= 4096) {
        FcParams fp{cp.nimg, cp.K, cp.Kpad, cp.N, cp.relu, cp.in_ptrs, cp.in_off, cp.wgt, cp.bias, cp.out_ptrs, cp.out_off};
        st.gemv = true;
        e = launch_fc_gemv(fp, stream_);
      } else {
        e = launch_conv_tc(cp, stream_);
      }
      break;
    }
    case OpKind::maxpool: {
      PoolParams p{batch, ti.H, ti.W, op.in.C, op.Ho, op.Wo, op.KH, op.stride, op.pad,
                   input_ptrs(net, op, d_ptrs), off(op.in), ldc(op.in), d_ptrs, off(op.out), ldc(op.out)};
      e = launch_maxpool(p, stream_);
      break;
    }
    case OpKind::avgpool: {
      AvgPoolParams p{batch, ti.H * ti.W, op.in.C, input_ptrs(net, op, d_ptrs), off(op.in), ldc(op.in), d_ptrs, off(op.out), prec_ == 0 ? 1 : 0};
      e = launch_avgpool(p, stream_);
      break;
    }
    case OpKind::dwconv: {
      DwParams p{batch, ti.H, ti.W, op.in.C, op.Ho, op.Wo, op.stride, input_ptrs(net, op, d_ptrs), off(op.in), ldc(op.in),
                 d_weights_ + op.w_off, d_weights_ + op.b_off, d_ptrs, off(op.out), ldc(op.out), op.relu,
                 prec_ == 0 ? op.round_out : 0};
      e = launch_dwconv(p, stream_);
      break;
    }
    case OpKind::softmax: {
      SoftmaxParams p{batch, op.in.C, d_ptrs, off(op.in), off(op.out)};
      e = launch_softmax(p, stream_);
      break;
    }
  }
  ck(e, op.name.c_str());
  ++launches_;
  if (sample) {
    ck(cudaEventRecord(st.t1, stream_), "ev rec");
    stats_.push_back(st);
  }
}

void Executor::run_layer(int dnn, int layer, float* const* d_ptrs, int batch) {
  if (batch <= 0) return;
  const NetDef& net = suite_.nets[static_cast<std::size_t>(dnn)];
  const auto& items = plans_[static_cast<std::size_t>(dnn)][static_cast<std::size_t>(layer - 1)];
  for (std::size_t i = 0; i < items.size(); ++i) {
    const LayerItem& it = items[i];
    if (it.b < 0) launch_op(net, net.ops[static_cast<std::size_t>(it.a)], d_ptrs, batch);
    else
      launch_group(net, layer, static_cast<int>(i), net.ops[static_cast<std::size_t>(it.a)],
                   net.ops[static_cast<std::size_t>(it.b)], d_ptrs, batch);
  }
}

// --------------------------------------------------------------- requests

void Executor::admit(std::int64_t id, int dnn, int entry_layer, const float* image, bool on_device) {
  if (slot_of_.count(id)) throw std::logic_error("request admitted twice: " + std::to_string(id));
  if (free_.empty()) throw std::runtime_error("activation arena full");
  const NetDef& net = suite_.nets[static_cast<std::size_t>(dnn)];
  Slot s;
  s.index = free_.back();
  free_.pop_back();
  s.dnn = dnn;
  s.blob = slot_ptr(s.index);
  const TensorDef& in = net.tensors[static_cast<std::size_t>(net.input_t)];
  const std::size_t bytes = static_cast<std::size_t>(in.H) * in.W * in.C * sizeof(float);
  cudaStream_t st = entry_layer > 1 ? side_ : copy_;
  wait_slot_free(s.index, st);
  ck(cudaMemcpyAsync(s.blob + in.off, image, bytes, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st),
     "admit copy");
  if (entry_layer == 1) {
    s.ready = next_ready_event();
    ck(cudaEventRecord(s.ready, copy_), "ready rec");
    s.pending_ready = true;
    s.ready_seq = ++ready_seq_;
    s.ready_stream = 0;
  } else {
    // Collaborative mode: the client's layer prefix, emulated on a side
    // stream so it stays off the server's critical path.
    TableChunk& c = chunks_[chunk_];
    (void)c;
    float** host;
    chunk_ = (chunk_ + 1) % chunks_.size();
    TableChunk& mine = chunks_[chunk_];
    if (mine.in_use) ck(cudaEventSynchronize(mine.done), "chunk wait");
    chunk_used_ = 0;
    float** d = table_alloc(1, &host);
    host[0] = s.blob;
    ck(cudaMemcpyAsync(d, host, sizeof(float*), cudaMemcpyHostToDevice, side_), "table H2D");
    std::swap(stream_, side_);
    try {
      for (int k = 1; k < entry_layer; ++k) run_layer(dnn, k, d, 1);
    } catch (...) {
      std::swap(stream_, side_);
      throw;
    }
    std::swap(stream_, side_);
    ck(cudaEventRecord(mine.done, side_), "chunk done");
    mine.in_use = true;
    s.ready = next_ready_event();
    ck(cudaEventRecord(s.ready, side_), "ready rec");
    s.pending_ready = true;
    s.ready_seq = ++ready_seq_;
    s.ready_stream = 1;
  }
  slot_of_.emplace(id, s);
}

void Executor::admit_ref(std::int64_t id, int dnn, const float* image) {
  if (slot_of_.count(id)) throw std::logic_error("request admitted twice: " + std::to_string(id));
  if (free_.empty()) throw std::runtime_error("activation arena full");
  if (!image) throw std::invalid_argument("admit_ref: null image");
  Slot s;
  s.index = free_.back();
  free_.pop_back();
  s.dnn = dnn;
  s.blob = slot_ptr(s.index);
  s.image = image;
  // Nothing is written now: the first layer's kernels write the blob on the
  // serving stream, after any earlier work that read the slot.
  slot_free_[static_cast<std::size_t>(s.index)].seq = 0;
  slot_of_.emplace(id, s);
}

void Executor::admit_rgb(std::int64_t id, int dnn, const std::uint8_t* rgb) {
  if (slot_of_.count(id)) throw std::logic_error("request admitted twice: " + std::to_string(id));
  if (free_.empty()) throw std::runtime_error("activation arena full");
  const NetDef& net = suite_.nets[static_cast<std::size_t>(dnn)];
  const TensorDef& in = net.tensors[static_cast<std::size_t>(net.input_t)];
  if (in.C != 4) throw std::invalid_argument("admit_rgb needs a 4-channel padded input");
  Slot s;
  s.index = free_.back();
  free_.pop_back();
  s.dnn = dnn;
  s.blob = slot_ptr(s.index);
  const int hw = in.H * in.W;
  std::uint8_t* stage = staging_ + static_cast<std::size_t>(staging_next_) * staging_floats_;
  staging_next_ = (staging_next_ + 1) % staging_n_;  // ring reuse is ordered on copy_
  ck(cudaMemcpyAsync(stage, rgb, static_cast<std::size_t>(hw) * 3, cudaMemcpyHostToDevice, copy_), "admit rgb H2D");
  wait_slot_free(s.index, copy_);
  ck(launch_expand_rgb(stage, s.blob + in.off, hw, copy_), "expand rgb");
  s.ready = next_ready_event();
  ck(cudaEventRecord(s.ready, copy_), "ready rec");
  s.pending_ready = true;
  s.ready_seq = ++ready_seq_;
  s.ready_stream = 0;
  slot_of_.emplace(id, s);
}

void Executor::admit_rgb_many(const std::int64_t* ids, int dnn, const std::uint8_t* const* rgb, int k, bool pinned_src) {
  if (k <= 0) return;
  const NetDef& net = suite_.nets[static_cast<std::size_t>(dnn)];
  const TensorDef& in = net.tensors[static_cast<std::size_t>(net.input_t)];
  if (in.C != 4) throw std::invalid_argument("admit_rgb needs a 4-channel padded input");
  const int hw = in.H * in.W;
  const std::size_t bytes = static_cast<std::size_t>(hw) * 3;
  for (int i = 0; i < k; ++i)
    if (slot_of_.count(ids[i])) throw std::logic_error("request admitted twice: " + std::to_string(ids[i]));
  if (free_.size() < static_cast<std::size_t>(k)) throw std::runtime_error("activation arena full");
  int done = 0;
  while (done < k) {
    // consecutive staging slots (no wrap inside one copy), at most kExpandMax
    const int first = staging_next_;
    const int take = std::min({k - done, staging_n_ - first, kExpandMax});
    // The host regions were last read by earlier batches' H2D copies on copy_
    // (in order): waiting for the newest of them covers the rest.
    std::uint8_t* dev = staging_ + static_cast<std::size_t>(first) * staging_floats_;
    if (pinned_src) {
      for (int q = 0; q < take; ++q)
        ck(cudaMemcpyAsync(dev + static_cast<std::size_t>(q) * staging_floats_, rgb[done + q], bytes,
                           cudaMemcpyHostToDevice, copy_), "admit rgb H2D");
    } else {
      long newest = 0;
      for (int q = 0; q < take; ++q) newest = std::max(newest, pack_seq_[static_cast<std::size_t>(first + q)]);
      if (newest > pack_synced_) {
        ck(cudaEventSynchronize(pack_ev_[static_cast<std::size_t>(newest % 128)]), "pack reuse");
        pack_synced_ = newest;
      }
      std::uint8_t* host = pack_host_ + static_cast<std::size_t>(first) * staging_floats_;
      for (int q = 0; q < take; ++q) std::memcpy(host + static_cast<std::size_t>(q) * staging_floats_, rgb[done + q], bytes);
      ck(cudaMemcpyAsync(dev, host, static_cast<std::size_t>(take - 1) * staging_floats_ + bytes, cudaMemcpyHostToDevice,
                         copy_), "admit rgb batch H2D");
      const long seq = ++pack_batches_;
      ck(cudaEventRecord(pack_ev_[static_cast<std::size_t>(seq % 128)], copy_), "pack rec");
      for (int q = 0; q < take; ++q) pack_seq_[static_cast<std::size_t>(first + q)] = seq;
    }
    staging_next_ = (first + take) % staging_n_;
    ExpandManyParams ep;
    ep.rgb = dev;
    ep.stride = static_cast<long>(staging_floats_);
    ep.hw = hw;
    ep.n = take;
    std::vector<Slot> slots(static_cast<std::size_t>(take));
    for (int q = 0; q < take; ++q) {
      Slot& s = slots[static_cast<std::size_t>(q)];
      s.index = free_.back();
      free_.pop_back();
      s.dnn = dnn;
      s.blob = slot_ptr(s.index);
      wait_slot_free(s.index, copy_);
      ep.dst[q] = s.blob + in.off;
    }
    ck(launch_expand_rgb_many(ep, copy_), "expand rgb batch");
    const cudaEvent_t ready = next_ready_event();
    ck(cudaEventRecord(ready, copy_), "ready rec");
    for (int q = 0; q < take; ++q) {
      Slot& s = slots[static_cast<std::size_t>(q)];
      s.ready = ready;
      s.pending_ready = true;
      s.ready_seq = ++ready_seq_;
      s.ready_stream = 0;
      slot_of_.emplace(ids[done + q], s);
    }
    done += take;
  }
}

void Executor::wait_ready(const std::vector<Slot*>& pending) {
  Slot* latest[2] = {nullptr, nullptr};
  for (Slot* s : pending) {
    Slot*& l = latest[s->ready_stream];
    if (!l || s->ready_seq > l->ready_seq) l = s;
  }
  for (Slot* l : latest)
    if (l) {
      // an input copy that has already landed needs no device-side wait (a
      // cross-stream wait costs the next kernel its programmatic launch)
      if (cudaEventQuery(l->ready) == cudaSuccess) continue;
      ck(cudaStreamWaitEvent(stream_, l->ready, 0), "wait ready");
      pdl::suppress_next();
    }
  for (Slot* s : pending) s->pending_ready = false;
}

Executor::FreeMark Executor::record_free() {
  // A re-recorded ring event (after 4096 frees) only waits for a later point.
  FreeMark m{free_ring_[free_next_], ++free_seq_};
  free_next_ = (free_next_ + 1) % free_ring_.size();
  ck(cudaEventRecord(m.ev, stream_), "slot free rec");
  return m;
}

void Executor::wait_slot_free(int index, cudaStream_t st) {
  FreeMark& f = slot_free_[static_cast<std::size_t>(index)];
  if (!f.seq) return;
  long& waited = waited_free_[st == side_ ? 1 : 0];
  if (f.seq > waited) {
    ck(cudaStreamWaitEvent(st, f.ev, 0), "wait slot free");
    pdl::suppress_next();
    waited = f.seq;  // every free up to this one is covered on st
  }
  f.seq = 0;
}

const float* Executor::blob(std::int64_t id) const {
  auto it = slot_of_.find(id);
  return it == slot_of_.end() ? nullptr : it->second.blob;
}

void Executor::retire(std::int64_t id, float* out, int n, bool logits) {
  auto it = slot_of_.find(id);
  if (it == slot_of_.end()) throw std::logic_error("retire of unknown request " + std::to_string(id));
  const NetDef& net = suite_.nets[static_cast<std::size_t>(it->second.dnn)];
  const TensorDef& t = net.tensors[static_cast<std::size_t>(logits ? net.logits_t : net.probs_t)];
  const int cnt = std::min(n, net.num_classes);
  ck(cudaMemcpyAsync(out, it->second.blob + t.off, static_cast<std::size_t>(cnt) * sizeof(float),
                     cudaMemcpyDeviceToHost, stream_),
     "retire copy");
  ck(cudaStreamSynchronize(stream_), "retire sync");
  drop(id);
}

void Executor::retire_async(std::int64_t id, float* out, int n) {
  auto it = slot_of_.find(id);
  if (it == slot_of_.end()) throw std::logic_error("retire of unknown request " + std::to_string(id));
  const NetDef& net = suite_.nets[static_cast<std::size_t>(it->second.dnn)];
  const TensorDef& t = net.tensors[static_cast<std::size_t>(net.probs_t)];
  const int cnt = std::min(n, net.num_classes);
  ck(cudaMemcpyAsync(out, it->second.blob + t.off, static_cast<std::size_t>(cnt) * sizeof(float),
                     cudaMemcpyDeviceToHost, stream_),
     "retire copy");
  drop(id);  // the slot's next admission waits for this copy (slot_free_)
}

void Executor::retire_many_async(const std::vector<std::int64_t>& ids, const std::vector<float*>& outs, int n) {
  for (std::size_t b = 0; b < ids.size(); b += kGatherMax) {
    GatherParams g{};
    g.n = 0;
    g.cnt = n;
    for (std::size_t i = b; i < ids.size() && i < b + kGatherMax; ++i) {
      auto it = slot_of_.find(ids[i]);
      if (it == slot_of_.end()) throw std::logic_error("retire of unknown request " + std::to_string(ids[i]));
      const NetDef& net = suite_.nets[static_cast<std::size_t>(it->second.dnn)];
      const TensorDef& t = net.tensors[static_cast<std::size_t>(net.probs_t)];
      g.cnt = std::min(g.cnt, net.num_classes);
      g.src[g.n] = it->second.blob + t.off;
      g.dst[g.n] = outs[i];
      ++g.n;
    }
    ck(launch_gather_out(g, stream_), "retire gather");
  }
  // One release mark after the gather for all of them (slot reuse waits for it).
  if (ids.empty()) return;
  for (std::int64_t id : ids) {
    auto it = slot_of_.find(id);
    if (it != slot_of_.end() && it->second.pending_ready) {
      ck(cudaStreamWaitEvent(stream_, it->second.ready, 0), "wait ready");
      pdl::suppress_next();
      it->second.pending_ready = false;
    }
  }
  const FreeMark m = record_free();
  for (std::int64_t id : ids) release_slot(id, &m);
}

void Executor::drop(std::int64_t id) { release_slot(id, nullptr); }

void Executor::release_slot(std::int64_t id, const FreeMark* shared) {
  auto it = slot_of_.find(id);
  if (it == slot_of_.end()) return;
  if (it->second.pending_ready) {
    // a pending input copy / prefix must finish before the slot can be reused
    ck(cudaStreamWaitEvent(stream_, it->second.ready, 0), "wait ready");
    pdl::suppress_next();
  }
  const std::size_t idx = static_cast<std::size_t>(it->second.index);
  slot_free_[idx] = shared ? *shared : record_free();
  free_.push_back(it->second.index);
  slot_of_.erase(it);
  auto r = ride_of_.find(id);
  if (r != ride_of_.end()) {
    ride_free_.push_back(r->second);
    ride_of_.erase(r);
  }
}

// ------------------------------------------------------------------ steps

void Executor::new_plan(int plan_no) {
  // Rides in progress are discarded: the rider keeps its committed blob.
  for (auto& [id, idx] : ride_of_) ride_free_.push_back(idx);
  ride_of_.clear();
  ride_plan_ = plan_no;
}

void Executor::step(int plan_no, int segment, int dnn, int from, int to,
                    const std::vector<std::pair<std::int64_t, int>>& members,
                    const std::vector<batchsim::Rider>& riders) {
  if (plan_no != ride_plan_) new_plan(plan_no);
  const NetDef& net = suite_.nets[static_cast<std::size_t>(dnn)];
  // Members whose input copy / client prefix may still be running.
  std::vector<Slot*> pending;
  for (const auto& [id, layer] : members) {
    auto it = slot_of_.find(id);
    if (it == slot_of_.end()) throw std::logic_error("step member not admitted: " + std::to_string(id));
    if (it->second.pending_ready) pending.push_back(&it->second);
  }
  // Members sorted by current layer: the batch at layer k is a prefix.
  struct Mem {
    int first;
    float* blob;
    const float* image;  // admit_ref input (nullptr: the input tensor is in the blob)
  };
  std::vector<Mem> mem;
  mem.reserve(members.size());
  bool any_ref = false;
  for (const auto& [id, layer] : members) {
    const Slot& sl = slot_of_.at(id);
    mem.push_back({layer, sl.blob, sl.image});
    any_ref = any_ref || sl.image;
  }
  std::stable_sort(mem.begin(), mem.end(), [](const Mem& a, const Mem& b) { return a.first < b.first; });

  // Ride buffers for riders joining inside this step; riders that joined in
  // an earlier step of the same plan continue on their buffer.
  struct RideRun {
    int join, leave;
    float* buf;
    float* committed;
    const float* image;
  };
  std::vector<RideRun> rides;
  for (const batchsim::Rider& r : riders) {
    if (r.join_layer > to || r.leave_layer < from) continue;
    auto it = slot_of_.find(r.id);
    if (it == slot_of_.end()) continue;  // dropped meanwhile
    if (it->second.pending_ready) pending.push_back(&it->second);
    auto rb = ride_of_.find(r.id);
    float* buf;
    if (rb == ride_of_.end()) {
      if (ride_free_.empty()) throw std::runtime_error("ride arena full");
      const int idx = ride_free_.back();
      ride_free_.pop_back();
      ride_of_[r.id] = idx;
      buf = ride_arena_ + static_cast<std::size_t>(idx) * slot_floats_;
    } else {
      buf = ride_arena_ + static_cast<std::size_t>(rb->second) * slot_floats_;
    }
    rides.push_back({r.join_layer, r.leave_layer, buf, it->second.blob, it->second.image});
    any_ref = any_ref || it->second.image;
  }

  wait_ready(pending);

  // One pointer chunk per step.
  chunk_ = (chunk_ + 1) % chunks_.size();
  TableChunk& c = chunks_[chunk_];
  if (c.in_use) ck(cudaEventSynchronize(c.done), "chunk wait");
  chunk_used_ = 0;
  struct LayerRun {
    int k;
    float** d;
    int b;
    float** din;  // input-tensor table (admit_ref members), or nullptr
  };
  const long in_off = net.tensors[static_cast<std::size_t>(net.input_t)].off;
  std::vector<LayerRun> runs;
  std::vector<std::pair<int, RideRun>> copies;  // (layer before which to copy, ride)
  std::size_t mi = 0;
  // The reference DP sets a segment's start layer to its newest member's
  // layer (dp_time.hpp:279), assuming FIFO order implies non-increasing
  // layers. With collaborative admission an older request can arrive later
  // at a lower layer; the simulator then advances it to layer_to + 1
  // (simulator.hpp:475-516) although layers [its layer, from) never ran.
  // Schedules stay bit-exact; the executor runs those layers for such members
  // inside this step, so outputs remain the network's.
  int first = from;
  for (const auto& m : mem) first = std::min(first, m.first);
  for (int k = first; k <= to; ++k) {
    while (mi < mem.size() && mem[mi].first <= k) ++mi;
    int nr = 0;
    for (const RideRun& rr : rides)
      if (rr.join <= k && k <= rr.leave) ++nr;
    const int b = static_cast<int>(mi) + nr;
    if (b == 0) continue;
    if (b > max_batch_) throw std::logic_error("step batch exceeds the configured bound");
    float** host;
    float** d = table_alloc(static_cast<std::size_t>(b), &host);
    for (std::size_t i = 0; i < mi; ++i) host[i] = mem[i].blob;
    int j = static_cast<int>(mi);
    for (const RideRun& rr : rides)
      if (rr.join <= k && k <= rr.leave) host[j++] = rr.buf;
    float** din = nullptr;
    if (any_ref && k == 1) {
      // bases such that base + input offset = the referenced image
      float** hin;
      din = table_alloc(static_cast<std::size_t>(b), &hin);
      for (std::size_t i = 0; i < mi; ++i) hin[i] = mem[i].image ? const_cast<float*>(mem[i].image) - in_off : mem[i].blob;
      int jj = static_cast<int>(mi);
      for (const RideRun& rr : rides)
        if (rr.join <= k && k <= rr.leave) hin[jj++] = rr.image ? const_cast<float*>(rr.image) - in_off : rr.buf;
    }
    runs.push_back({k, d, b, din});
  }
  if (table_mode_ == 2) {
    // the chunk's previous step has finished (host-synchronised above)
    ck(launch_table_write(c.dev, c.host, chunk_used_, stream_, stamps_, ++step_seq_, kStampCap), "table write");
    launches_ += static_cast<long>((chunk_used_ + kTableWriteMax - 1) / kTableWriteMax);
  } else if (table_mode_ == 1) {
    // the chunk's previous step has finished (host-synchronised above), so
    // the upload may overwrite it at once; the serving stream waits for it
    ck(cudaMemcpyAsync(c.dev, c.host, chunk_used_ * sizeof(float*), cudaMemcpyHostToDevice, table_), "table H2D");
    ck(cudaEventRecord(c.uploaded, table_), "table uploaded");
    ck(cudaStreamWaitEvent(stream_, c.uploaded, 0), "wait table");
    pdl::suppress_next();
  } else {
    ck(cudaMemcpyAsync(c.dev, c.host, chunk_used_ * sizeof(float*), cudaMemcpyHostToDevice, stream_), "table H2D");
  }
  for (const LayerRun& lr : runs) {
    for (const RideRun& rr : rides)
      if (rr.join == lr.k)
        ck(cudaMemcpyAsync(rr.buf, rr.committed, slot_floats_ * sizeof(float), cudaMemcpyDeviceToDevice, stream_),
           "ride copy");
    in_override_ = lr.din;
    run_layer(dnn, lr.k, lr.d, lr.b);
    in_override_ = nullptr;
  }
  ck(cudaEventRecord(c.done, stream_), "chunk done");
  c.in_use = true;
  (void)net;
  (void)segment;
}

void Executor::step_done(const std::vector<std::int64_t>& deposited) {
  // Commit: the ride buffer becomes the rider's state (blob copy back so
  // the slot keeps its fixed address).
  for (std::int64_t id : deposited) {
    auto rb = ride_of_.find(id);
    auto it = slot_of_.find(id);
    if (rb == ride_of_.end() || it == slot_of_.end()) continue;
    ck(cudaMemcpyAsync(it->second.blob, ride_arena_ + static_cast<std::size_t>(rb->second) * slot_floats_,
                       slot_floats_ * sizeof(float), cudaMemcpyDeviceToDevice, stream_),
       "ride commit");
    ride_free_.push_back(rb->second);
    ride_of_.erase(rb);
  }
}

// -------------------------------------------------------------- measurement

void Executor::enable_stats(bool on, int every) {
  stats_on_ = on;
  stats_every_ = std::max(1, every);
  if (on && event_pool_.empty()) {
    event_pool_.resize(1 << 16);
    for (auto& e : event_pool_) ck(cudaEventCreate(&e), "event pool");
  }
}

void Executor::clear_stats() {
  stats_.clear();
  ev_next_ = 0;
}

int Executor::tuned_index(int batch) const {
  if (tune_batches_.empty()) return -1;
  // nearest tuned batch by ratio
  std::size_t best = 0;
  double bd = 1e30;
  for (std::size_t t = 0; t < tune_batches_.size(); ++t) {
    const double d = std::fabs(std::log(static_cast<double>(tune_batches_[t]) / batch));
    if (d < bd) {
      bd = d;
      best = t;
    }
  }
  return static_cast<int>(best);
}

std::string Executor::tune_tiles(const std::vector<int>& batches, int reps) {
  tune_batches_.clear();
  conv_pref_.assign(suite_.nets.size(), {});
  group_pref_.assign(suite_.nets.size(), {});
  std::vector<int> bs;
  for (int b : batches)
    if (b >= 1 && b <= max_batch_) bs.push_back(b);
  std::sort(bs.begin(), bs.end());
  bs.erase(std::unique(bs.begin(), bs.end()), bs.end());
  // Choices apply as soon as they are made (an untuned entry is the
  // launcher's rule), so a pair's "separate" timing uses its tuned convs.
  tune_batches_ = bs;
  std::string log = "[";
  auto note = [&](const std::string& what, int b, const char* choice, double ms) {
    char buf[200];
    std::snprintf(buf, sizeof buf, "%s[\"%s\",%d,\"%s\",%.4f]", log.size() > 1 ? "," : "", what.c_str(), b, choice, ms);
    log += buf;
  };
  for (std::size_t n = 0; n < suite_.nets.size(); ++n) {
    const NetDef& net = suite_.nets[n];
    conv_pref_[n].assign(net.ops.size(), std::vector<ConvChoice>(bs.size()));
    group_pref_[n].resize(plans_[n].size());
    for (std::size_t k = 0; k < plans_[n].size(); ++k)
      group_pref_[n][k].assign(plans_[n][k].size(), std::vector<signed char>(bs.size(), 0));
    for (int k = 1; k <= net.num_layers(); ++k) {
      const auto& items = plans_[n][static_cast<std::size_t>(k - 1)];
      for (std::size_t t = 0; t < bs.size(); ++t) {
        const int b = bs[t];
        auto time_layer = [&] { return profile_layer(static_cast<int>(n), k, b, reps, false); };
        for (std::size_t ii = 0; ii < items.size(); ++ii) {
          const LayerItem& it = items[ii];
          const bool pair = it.b >= 0;
          tune_net_ = static_cast<int>(n);
          if (pair) {  // tune the two convs as separate launches first
            tune_layer_ = k;
            tune_item_ = static_cast<int>(ii);
            tune_group_ = -1;
          }
          for (int oi : {it.a, it.b}) {
            if (oi < 0) continue;
            const OpDef& op = net.ops[static_cast<std::size_t>(oi)];
            if (op.kind != OpKind::conv) continue;
            // candidates: the launcher's own choice first, then forced splits
            // (narrow tiles), then 128 x 256 tiles unsplit (N > 128)
            std::vector<ConvChoice> cands{{0, 0}};
            for (signed char ks : {1, 2, 4, 8}) cands.push_back({2, ks});
            if (op.out.C > 128) cands.push_back({1, 1});
            if (op.out.C > 128 && prec_ != 2) cands.push_back({3, 1});
            if (op.out.C > 128 && prec_ != 2) cands.push_back({4, 1});
            tune_op_ = oi;
            ConvChoice best{};
            double best_ms = 1e30;
            for (const ConvChoice& c : cands) {
              tune_choice_ = c;
              const double ms = time_layer();
              char name[16];
              std::snprintf(name, sizeof name, "w%d/k%d", c.wide, c.ks);
              note(op.name, b, name, ms);
              if (ms < 0.98 * best_ms) {  // switch only on a clear win
                best_ms = ms;
                best = c;
              }
            }
            conv_pref_[n][static_cast<std::size_t>(oi)][t] = best;
            tune_op_ = -1;
          }
          if (pair) {
            const std::string nm =
                net.ops[static_cast<std::size_t>(it.a)].name + "+" + net.ops[static_cast<std::size_t>(it.b)].name;
            signed char best_g = -1;
            double best_ms = time_layer();  // separate, with the tuned convs
            note(nm, b, "separate", best_ms);
            for (signed char g : {1, 2, 4, 8}) {
              tune_group_ = g;
              const double ms = time_layer();
              char name[16];
              std::snprintf(name, sizeof name, "grouped/k%d", g);
              note(nm, b, name, ms);
              if (ms < 0.98 * best_ms) {
                best_ms = ms;
                best_g = g;
              }
            }
            group_pref_[n][static_cast<std::size_t>(k - 1)][ii][t] = best_g;
          }
          tune_net_ = tune_layer_ = tune_item_ = -1;
          tune_group_ = 0;
        }
      }
    }
  }
  return log + "]";
}

double Executor::profile_layer(int dnn, int layer, int batch, int reps, bool flush_l2) {
  if (batch < 1 || batch > max_batch_) throw std::invalid_argument("profile batch out of range");
  if (flush_l2 && !flush_) {
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device_);
    flush_bytes_ = static_cast<std::size_t>(std::max(l2, 1 << 20)) * 2;
    ck(cudaMalloc(&flush_, flush_bytes_), "flush");
  }
  cudaEvent_t a, b;
  ck(cudaEventCreate(&a), "ev");
  ck(cudaEventCreate(&b), "ev");
  std::vector<float> ms;
  for (int r = -2; r < reps; ++r) {
    if (flush_l2) ck(cudaMemsetAsync(flush_, r & 0xff, flush_bytes_, stream_), "flush");
    ck(cudaEventRecord(a, stream_), "ev");
    run_layer(dnn, layer, scratch_ptrs_, batch);
    ck(cudaEventRecord(b, stream_), "ev");
    ck(cudaEventSynchronize(b), "ev sync");
    float t = 0;
    ck(cudaEventElapsedTime(&t, a, b), "elapsed");
    if (r >= 0) ms.push_back(t);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  std::sort(ms.begin(), ms.end());
  return ms[ms.size() / 2];
}

double Executor::profile_pass_total(int dnn, int batch, int reps) {
  if (batch < 1 || batch > max_batch_) throw std::invalid_argument("profile batch out of range");
  const int L = suite_.nets[static_cast<std::size_t>(dnn)].num_layers();
  std::vector<cudaEvent_t> ev(static_cast<std::size_t>(reps) + 1);
  for (auto& e : ev) ck(cudaEventCreate(&e), "ev");
  for (int w = 0; w < 2; ++w)
    for (int k = 1; k <= L; ++k) run_layer(dnn, k, scratch_ptrs_, batch);
  ck(cudaEventRecord(ev[0], stream_), "ev");
  for (int r = 0; r < reps; ++r) {
    for (int k = 1; k <= L; ++k) run_layer(dnn, k, scratch_ptrs_, batch);
    ck(cudaEventRecord(ev[static_cast<std::size_t>(r) + 1], stream_), "ev");
  }
  ck(cudaStreamSynchronize(stream_), "pass sync");
  std::vector<double> v(static_cast<std::size_t>(reps));
  for (int r = 0; r < reps; ++r) {
    float t = 0;
    ck(cudaEventElapsedTime(&t, ev[static_cast<std::size_t>(r)], ev[static_cast<std::size_t>(r) + 1]), "elapsed");
    v[static_cast<std::size_t>(r)] = t;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

std::vector<double> Executor::profile_pass(int dnn, int batch, int reps) {
  if (batch < 1 || batch > max_batch_) throw std::invalid_argument("profile batch out of range");
  const int L = suite_.nets[static_cast<std::size_t>(dnn)].num_layers();
  std::vector<cudaEvent_t> ev(static_cast<std::size_t>(reps) * (L + 1));
  for (auto& e : ev) ck(cudaEventCreate(&e), "ev");
  for (int w = 0; w < 2; ++w)
    for (int k = 1; k <= L; ++k) run_layer(dnn, k, scratch_ptrs_, batch);
  for (int r = 0; r < reps; ++r) {
    cudaEvent_t* er = ev.data() + static_cast<std::size_t>(r) * (L + 1);
    ck(cudaEventRecord(er[0], stream_), "ev");
    for (int k = 1; k <= L; ++k) {
      run_layer(dnn, k, scratch_ptrs_, batch);
      ck(cudaEventRecord(er[k], stream_), "ev");
    }
  }
  ck(cudaStreamSynchronize(stream_), "pass sync");
  std::vector<double> out(static_cast<std::size_t>(L));
  std::vector<double> v(static_cast<std::size_t>(reps));
  for (int k = 1; k <= L; ++k) {
    for (int r = 0; r < reps; ++r) {
      float t = 0;
      const cudaEvent_t* er = ev.data() + static_cast<std::size_t>(r) * (L + 1);
      ck(cudaEventElapsedTime(&t, er[k - 1], er[k]), "elapsed");
      v[static_cast<std::size_t>(r)] = t;
    }
    std::sort(v.begin(), v.end());
    out[static_cast<std::size_t>(k - 1)] = v[v.size() / 2];
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return out;
}

std::vector<double> Executor::profile_steps(int dnn, int batch, int reps) {
  if (batch < 1 || batch > max_batch_) throw std::invalid_argument("profile batch out of range");
  const NetDef& net = suite_.nets[static_cast<std::size_t>(dnn)];
  const int L = net.num_layers();
  float** tab = nullptr;
  ck(cudaMalloc(&tab, static_cast<std::size_t>(max_batch_) * sizeof(float*)), "step table");
  std::vector<float*> hp(static_cast<std::size_t>(batch));
  for (int i = 0; i < batch; ++i) hp[static_cast<std::size_t>(i)] = scratch_ + static_cast<std::size_t>(i) * slot_floats_;
  const int classes = net.num_classes;
  float* outs = nullptr;
  ck(cudaHostAlloc(&outs, static_cast<std::size_t>(batch) * classes * sizeof(float), cudaHostAllocMapped), "step outs");
  const long probs_off = net.tensors[static_cast<std::size_t>(net.probs_t)].off;
  std::vector<std::uint64_t> seq;  // table-write (step start) numbers, reps x L
  auto pass = [&](bool keep) {
    for (int k = 1; k <= L; ++k) {
      ck(launch_table_write(tab, hp.data(), hp.size(), stream_, stamps_, ++step_seq_, kStampCap), "step table");
      ++launches_;
      if (keep) seq.push_back(step_seq_);
      run_layer(dnn, k, tab, batch);
      if (k == L)  // the finishing requests' results copy-out
        for (int b0 = 0; b0 < batch; b0 += kGatherMax) {
          GatherParams g{};
          g.n = std::min(kGatherMax, batch - b0);
          g.cnt = classes;
          for (int i = 0; i < g.n; ++i) {
            g.src[i] = hp[static_cast<std::size_t>(b0 + i)] + probs_off;
            g.dst[i] = outs + static_cast<std::size_t>(b0 + i) * classes;
          }
          ck(launch_gather_out(g, stream_), "step gather");
        }
    }
  };
  pass(false);
  pass(false);
  for (int r = 0; r < reps; ++r) pass(true);
  ck(launch_table_write(tab, hp.data(), hp.size(), stream_, stamps_, ++step_seq_, kStampCap), "step table");
  sync();
  const std::vector<std::uint64_t> st = stamps();
  std::vector<double> out(static_cast<std::size_t>(L));
  std::vector<double> v(static_cast<std::size_t>(reps));
  for (int k = 0; k < L; ++k) {
    for (int r = 0; r < reps; ++r) {
      const std::uint64_t q = seq[static_cast<std::size_t>(r) * L + k];
      v[static_cast<std::size_t>(r)] = static_cast<double>(st[(q + 1) % kStampCap] - st[q % kStampCap]) * 1e-6;
    }
    std::sort(v.begin(), v.end());
    out[static_cast<std::size_t>(k)] = v[v.size() / 2];
  }
  cudaFreeHost(outs);
  cudaFree(tab);
  return out;
}

void Executor::profile_span(int dnn, int from, int to, int batch, int reps, double out[3]) {
  if (batch < 1 || batch > max_batch_) throw std::invalid_argument("profile batch out of range");
  cudaEvent_t a, b;
  ck(cudaEventCreate(&a), "ev");
  ck(cudaEventCreate(&b), "ev");
  auto pass = [&] {
    for (int k = from; k <= to; ++k) run_layer(dnn, k, scratch_ptrs_, batch);
  };
  auto elapsed = [&] {
    float t = 0;
    ck(cudaEventSynchronize(b), "ev sync");
    ck(cudaEventElapsedTime(&t, a, b), "elapsed");
    return static_cast<double>(t);
  };
  pass();
  sync();
  std::vector<double> v;
  for (int r = 0; r < reps; ++r) {
    ck(cudaEventRecord(a, stream_), "ev");
    pass();
    ck(cudaEventRecord(b, stream_), "ev");
    v.push_back(elapsed());
  }
  std::sort(v.begin(), v.end());
  out[0] = v[v.size() / 2];
  // BS_SPAN_STEP (diagnostic bitmask) runs the back-to-back passes as the
  // serving loop's one-layer steps: 1 a table-write kernel before each layer
  // (the layer reads its pointers from that table), 4 an event record after
  // it, 8 the table by H2D on the table stream + a cross-stream event wait.
  const char* se = std::getenv("BS_SPAN_STEP");
  const int step_bits = se ? std::atoi(se) : 0;
  float** tab = nullptr;
  cudaEvent_t sev = nullptr;
  if (step_bits) {
    ck(cudaMalloc(&tab, static_cast<std::size_t>(max_batch_) * sizeof(float*)), "span table");
    ck(cudaEventCreateWithFlags(&sev, cudaEventDisableTiming), "ev");
  }
  std::vector<float*> hp(static_cast<std::size_t>(batch));
  for (int i = 0; i < batch; ++i) hp[static_cast<std::size_t>(i)] = scratch_ + static_cast<std::size_t>(i) * slot_floats_;
  if (step_bits & 8) std::copy(hp.begin(), hp.end(), chunks_[0].host);
  auto step_pass = [&] {
    for (int k = from; k <= to; ++k) {
      if (step_bits & 1) ck(launch_table_write(tab, hp.data(), hp.size(), stream_), "span table");
      if (step_bits & 8) {
        ck(cudaMemcpyAsync(tab, chunks_[0].host, hp.size() * sizeof(float*), cudaMemcpyHostToDevice, table_), "span H2D");
        ck(cudaEventRecord(chunks_[0].uploaded, table_), "ev");
        ck(cudaStreamWaitEvent(stream_, chunks_[0].uploaded, 0), "wait");
        pdl::suppress_next();
      }
      run_layer(dnn, k, (step_bits & 9) ? tab : scratch_ptrs_, batch);
      if (step_bits & 4) ck(cudaEventRecord(sev, stream_), "ev");
    }
  };
  ck(cudaEventRecord(a, stream_), "ev");
  for (int r = 0; r < reps; ++r) step_bits ? step_pass() : pass();
  ck(cudaEventRecord(b, stream_), "ev");
  out[1] = elapsed() / reps;
  if (tab) {
    sync();
    cudaFree(tab);
    cudaEventDestroy(sev);
  }
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge = nullptr;
  ck(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal), "capture");
  pass();
  ck(cudaStreamEndCapture(stream_, &g), "end capture");
  ck(cudaGraphInstantiate(&ge, g, 0), "instantiate");
  ck(cudaGraphLaunch(ge, stream_), "graph launch");
  sync();
  ck(cudaEventRecord(a, stream_), "ev");
  for (int r = 0; r < reps; ++r) ck(cudaGraphLaunch(ge, stream_), "graph launch");
  ck(cudaEventRecord(b, stream_), "ev");
  out[2] = elapsed() / reps;
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
}

// ------------------------------------------------------------- image pools

void Executor::make_image_pool(int dnn, int count, std::uint64_t seed) {
  const NetDef& net = suite_.nets[static_cast<std::size_t>(dnn)];
  const std::size_t per = static_cast<std::size_t>(net.in_H) * net.in_W * net.in_C;
  std::vector<float> host(per * static_cast<std::size_t>(count));
  for (int i = 0; i < count; ++i)
    synth_image(seed, static_cast<std::uint64_t>(i), net.in_H, net.in_W, net.in_C, 3, host.data() + per * static_cast<std::size_t>(i));
  if (pool_[static_cast<std::size_t>(dnn)]) cudaFree(pool_[static_cast<std::size_t>(dnn)]);
  ck(cudaMalloc(&pool_[static_cast<std::size_t>(dnn)], host.size() * sizeof(float)), "image pool");
  ck(cudaMemcpy(pool_[static_cast<std::size_t>(dnn)], host.data(), host.size() * sizeof(float), cudaMemcpyHostToDevice),
     "image pool H2D");
  pool_n_[static_cast<std::size_t>(dnn)] = count;
}

const float* Executor::pool_image(int dnn, int index) const {
  const NetDef& net = suite_.nets[static_cast<std::size_t>(dnn)];
  const std::size_t per = static_cast<std::size_t>(net.in_H) * net.in_W * net.in_C;
  return pool_[static_cast<std::size_t>(dnn)] + per * static_cast<std::size_t>(index % pool_n_[static_cast<std::size_t>(dnn)]);
}

int Executor::pool_size(int dnn) const { return pool_n_[static_cast<std::size_t>(dnn)]; }

}  // namespace bs200
