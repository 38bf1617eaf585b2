#include <cstdio>
#include <cstdlib>
// C-ABI of libbs_exec.so (declared in include/bs_exec.h).
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>

#include "bs_exec.h"
#include "bsb/jobs.hpp"
#include "errors.hpp"
#include "executor.hpp"
#include "image.hpp"
#include "live.hpp"
#include "nets_json.hpp"

using json = nlohmann::json;
using namespace bs200;

struct bs_handle {
  std::unique_ptr<Executor> ex;
  int window_cap = 0;              // default sim window for bs_replay / bs_serve jobs (0: job's own / 500)
  cudaEvent_t step_done = nullptr;  // bs_step_ex completion event (owned)
  ~bs_handle() {
    if (step_done) cudaEventDestroy(step_done);
  }
};

namespace {

char* dup_str(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const std::invalid_argument& e) {
    return bs_fail(BS_EINVAL, e.what());
  } catch (const std::logic_error& e) {
    return bs_fail(BS_ESTATE, e.what());
  } catch (const std::bad_alloc& e) {
    return bs_fail(BS_ENOMEM, e.what());
  } catch (const std::exception& e) {
    const std::string w = e.what();
    return bs_fail(w.find("full") != std::string::npos ? BS_ENOMEM : BS_ECUDA, w);
  }
}

// Virtual-time serving (the reference's event loop, bit-exact schedules)
// with every step executed on the GPU.
struct ReplayHook : batchsim::StepHook {
  Executor* ex;
  std::vector<int> dnn_map;  // profile dnn -> suite net
  std::uint64_t image_seed = 1;
  bool pool = true;
  float* results = nullptr;  // pinned [count][classes]
  int classes = 0;
  std::vector<float> host_img;
  int max_batch_seen = 0;
  int rider_steps = 0;  // steps carrying >= 1 foreign request through a shared stage
  int riders_total = 0;
  long steps = 0;

  bool log = std::getenv("BS_REPLAY_LOG") != nullptr;
  void admit(batchsim::RequestId id, int dnn, int entry_layer, batchsim::Ms t) override {
    const int net = dnn_map[static_cast<std::size_t>(dnn)];
    if (log) std::fprintf(stderr, "t=%.3f admit %lld net %d entry %d\n", t, static_cast<long long>(id), net, entry_layer);
    const NetDef& nd = ex->suite().nets[static_cast<std::size_t>(net)];
    if (pool && ex->pool_size(net) > 0) {
      const float* img = ex->pool_image(net, static_cast<int>((id - 1) % ex->pool_size(net)));
      if (entry_layer == 1) ex->admit_ref(id, net, img);
      else ex->admit(id, net, entry_layer, img, true);
    } else {
      host_img.resize(static_cast<std::size_t>(nd.in_H) * nd.in_W * nd.in_C);
      synth_image(image_seed, static_cast<std::uint64_t>(id - 1), nd.in_H, nd.in_W, nd.in_C, 3, host_img.data());
      ex->admit(id, net, entry_layer, host_img.data(), false);
      ex->sync();  // host buffer is reused
    }
  }
  void plan(int plan_no, batchsim::Ms) override { ex->new_plan(plan_no); }
  void step(const batchsim::StepView& v) override {
    if (log) {
      std::fprintf(stderr, "t=%.3f step plan %d seg %d net %d [%d,%d]:", v.start, v.plan, v.segment,
                   dnn_map[static_cast<std::size_t>(v.dnn)], v.from, v.to);
      for (const auto& [id, layer] : v.members) std::fprintf(stderr, " %lld@%d", static_cast<long long>(id), layer);
      std::fprintf(stderr, "\n");
    }
    ex->step(v.plan, v.segment, dnn_map[static_cast<std::size_t>(v.dnn)], v.from, v.to, v.members, v.riders);
    max_batch_seen = std::max(max_batch_seen, static_cast<int>(v.members.size() + v.riders.size()));
    if (!v.riders.empty()) ++rider_steps;
    riders_total += static_cast<int>(v.riders.size());
    ++steps;
  }
  void step_done(const batchsim::StepView&, const std::vector<batchsim::RequestId>& dep) override {
    ex->step_done(dep);
  }
  void finish(batchsim::RequestId id, batchsim::Ms) override {
    if (ex->has(id)) ex->retire_async(id, results + static_cast<std::size_t>(id - 1) * classes, classes);
  }
  void drop(batchsim::RequestId id, batchsim::Ms) override { ex->drop(id); }
};

std::vector<int> map_dnns(const batchsim::ProfileSet& ps, const Suite& s) {
  std::vector<int> m;
  for (const auto& d : ps.dnns) {
    int idx = -1;
    for (std::size_t i = 0; i < s.nets.size(); ++i)
      if (s.nets[i].name == d.name()) idx = static_cast<int>(i);
    if (idx < 0) throw std::invalid_argument("profile dnn '" + d.name() + "' is not in suite " + s.name);
    if (s.nets[static_cast<std::size_t>(idx)].num_layers() != d.num_layers())
      throw std::invalid_argument("profile dnn '" + d.name() + "' layer count differs from the network");
    m.push_back(idx);
  }
  return m;
}

}  // namespace

extern "C" {

int bs_create(int device, const char* suite, int max_batch, int max_requests, bs_handle** out) {
  return guarded([&] {
    if (!suite || !out || max_batch < 1 || max_requests < 1) throw std::invalid_argument("bs_create: bad argument");
    auto h = std::make_unique<bs_handle>();
    h->ex = std::make_unique<Executor>(device, suite, max_batch, max_requests);
    *out = h.release();
    return BS_OK;
  });
}

int bs_create_ex(int device, const char* suite, int max_batch, int max_requests, int window_cap, const char* dtype,
                 bs_handle** out) {
  return guarded([&] {
    if (window_cap < 0) throw std::invalid_argument("bs_create_ex: window_cap < 0");
    bs_handle* h = nullptr;
    const int rc = bs_create(device, suite, max_batch, max_requests, &h);
    if (rc != BS_OK) return rc;
    std::unique_ptr<bs_handle> own(h);
    h->window_cap = window_cap;
    if (dtype && *dtype) h->ex->set_precision(dtype);
    *out = own.release();
    return static_cast<int>(BS_OK);
  });
}

int bs_destroy(bs_handle* h) {
  return guarded([&] {
    delete h;
    return BS_OK;
  });
}

int bs_suite_json(bs_handle* h, char** out) {
  return guarded([&] {
    *out = dup_str(suite_json(h->ex->suite(), h->ex->blob_floats()).dump());
    return BS_OK;
  });
}

int bs_read_weights(bs_handle* h, float* dst, size_t n) {
  return guarded([&] {
    const auto& w = h->ex->suite().weights;
    if (n < w.size()) throw std::invalid_argument("bs_read_weights: buffer too small");
    std::memcpy(dst, w.data(), w.size() * sizeof(float));
    return BS_OK;
  });
}

int bs_admit(bs_handle* h, int64_t id, int dnn, int entry_layer, const float* image_host) {
  return guarded([&] {
    h->ex->admit(id, dnn, entry_layer, image_host, false);
    h->ex->sync();
    return BS_OK;
  });
}

int bs_set_precision(bs_handle* h, const char* mode) {
  return guarded([&] {
    h->ex->set_precision(mode ? mode : "");
    return BS_OK;
  });
}

int bs_admit_device(bs_handle* h, int64_t id, int dnn, const float* image_device) {
  return guarded([&] {
    h->ex->admit_ref(id, dnn, image_device);
    return BS_OK;
  });
}

int bs_admit_rgb(bs_handle* h, int64_t id, int dnn, const uint8_t* rgb_pinned) {
  return guarded([&] {
    if (!rgb_pinned) throw std::invalid_argument("bs_admit_rgb: null image");
    h->ex->admit_rgb(id, dnn, rgb_pinned);
    return BS_OK;
  });
}

int bs_admit_rgb_many(bs_handle* h, const int64_t* ids, int dnn, const uint8_t* const* rgb, int k) {
  return guarded([&] {
    if (k < 0 || (k > 0 && (!ids || !rgb))) throw std::invalid_argument("bs_admit_rgb_many: bad arrays");
    h->ex->admit_rgb_many(ids, dnn, rgb, k);
    return BS_OK;
  });
}

int bs_plan(bs_handle* h, int plan_no) {
  return guarded([&] {
    h->ex->new_plan(plan_no);
    return BS_OK;
  });
}

int bs_step(bs_handle* h, int plan_no, int segment, int dnn, int layer_from, int layer_to, const bs_member* m, int nm,
            const bs_rider* r, int nr) {
  return guarded([&] {
    std::vector<std::pair<std::int64_t, int>> members;
    for (int i = 0; i < nm; ++i) members.emplace_back(m[i].id, m[i].layer);
    std::vector<batchsim::Rider> riders;
    for (int i = 0; i < nr; ++i)
      riders.push_back({r[i].id, r[i].dnn, r[i].join_layer, r[i].leave_layer, r[i].deposit_layer});
    h->ex->step(plan_no, segment, dnn, layer_from, layer_to, members, riders);
    return BS_OK;
  });
}

int bs_step_ex(bs_handle* h, int plan_no, int segment, int dnn, int layer_from, int layer_to, const bs_member* m,
               int nm, const bs_rider* r, int nr, void* stream, bs_step_result* out) {
  return guarded([&] {
    if (!h || (nm > 0 && !m) || (nr > 0 && !r)) throw std::invalid_argument("bs_step_ex: bad argument");
    cudaStream_t user = static_cast<cudaStream_t>(stream);
    Executor& ex = *h->ex;
    if (!h->step_done && cudaEventCreateWithFlags(&h->step_done, cudaEventDisableTiming) != cudaSuccess)
      throw std::runtime_error("bs_step_ex: event");
    if (user) {  // the step follows the work already enqueued on the caller's stream
      if (cudaEventRecord(h->step_done, user) != cudaSuccess ||
          cudaStreamWaitEvent(ex.stream(), h->step_done, 0) != cudaSuccess)
        throw std::runtime_error("bs_step_ex: stream order");
    }
    const long k0 = ex.launches();
    const int rc = bs_step(h, plan_no, segment, dnn, layer_from, layer_to, m, nm, r, nr);
    if (rc != BS_OK) return rc;
    if (cudaEventRecord(h->step_done, ex.stream()) != cudaSuccess) throw std::runtime_error("bs_step_ex: event");
    if (user && cudaStreamWaitEvent(user, h->step_done, 0) != cudaSuccess)
      throw std::runtime_error("bs_step_ex: stream order");
    if (out) {
      // the batch rule of step_duration (simulator.hpp:705-713), as Executor::step applies it
      int first = layer_from;
      for (int i = 0; i < nm; ++i) first = std::min(first, m[i].layer);
      out->layers_run = 0;
      out->max_batch = 0;
      for (int k = first; k <= layer_to; ++k) {
        int b = 0;
        for (int i = 0; i < nm; ++i) b += m[i].layer <= k;
        for (int i = 0; i < nr; ++i) b += r[i].join_layer <= k && k <= r[i].leave_layer;
        out->layers_run += b > 0;
        out->max_batch = std::max(out->max_batch, b);
      }
      out->kernels = static_cast<int>(ex.launches() - k0);
      out->done_event = h->step_done;
    }
    return static_cast<int>(BS_OK);
  });
}

int bs_step_done(bs_handle* h, const int64_t* deposited, int n) {
  return guarded([&] {
    h->ex->step_done(std::vector<std::int64_t>(deposited, deposited + n));
    return BS_OK;
  });
}

int bs_retire(bs_handle* h, int64_t id, float* out, int n, int logits) {
  return guarded([&] {
    h->ex->retire(id, out, n, logits != 0);
    return BS_OK;
  });
}

int bs_drop(bs_handle* h, int64_t id) {
  return guarded([&] {
    h->ex->drop(id);
    return BS_OK;
  });
}

int bs_read_blob(bs_handle* h, int64_t id, float* dst, size_t n) {
  return guarded([&] {
    const float* b = h->ex->blob(id);
    if (!b) throw std::logic_error("unknown request");
    h->ex->sync();
    const std::size_t cnt = std::min(n, h->ex->blob_floats());
    if (cudaMemcpy(dst, b, cnt * sizeof(float), cudaMemcpyDeviceToHost) != cudaSuccess)
      throw std::runtime_error("blob copy failed");
    return BS_OK;
  });
}

int bs_sync(bs_handle* h) {
  return guarded([&] {
    h->ex->sync();
    return BS_OK;
  });
}

int bs_profile_layer(bs_handle* h, int dnn, int layer, int batch, int reps, int flush_l2, double* ms) {
  return guarded([&] {
    *ms = h->ex->profile_layer(dnn, layer, batch, reps, flush_l2 != 0);
    return BS_OK;
  });
}

int bs_profile_span(bs_handle* h, int dnn, int from, int to, int batch, int reps, double* ms3) {
  return guarded([&] {
    h->ex->profile_span(dnn, from, to, batch, reps, ms3);
    return BS_OK;
  });
}

namespace {
// bs_create_ex's window_cap is the default of the job's sim window.
json with_window_cap(const bs_handle* h, json j) {
  if (h->window_cap > 0 && j.contains("sim") && j["sim"].is_object() && !j["sim"].contains("window_cap"))
    j["sim"]["window_cap"] = h->window_cap;
  return j;
}
}  // namespace

int bs_replay(bs_handle* h, const char* job_json, char** out) {
  return guarded([&] {
    const json j = with_window_cap(h, json::parse(job_json));
    batchsim::SimJob job = batchsim::sim_job_from_json(j);
    Executor& ex = *h->ex;
    ReplayHook hook;
    hook.ex = &ex;
    hook.dnn_map = map_dnns(job.ps, ex.suite());
    hook.image_seed = j.value("image_seed", std::uint64_t{1});
    hook.pool = j.value("image_pool", 0) > 0;
    if (hook.pool)
      for (int net : hook.dnn_map) ex.make_image_pool(net, j.value("image_pool", 0), hook.image_seed);
    for (const NetDef& n : ex.suite().nets) hook.classes = std::max(hook.classes, n.num_classes);
    const std::size_t count = batchsim::generate_arrivals(job.spec).size();
    float* results = nullptr;
    if (cudaMallocHost(&results, std::max<std::size_t>(1, count) * hook.classes * sizeof(float)) != cudaSuccess)
      throw std::runtime_error("pinned results");
    std::memset(results, 0, count * hook.classes * sizeof(float));
    hook.results = results;
    const long launches0 = ex.launches();
    const auto t0 = std::chrono::steady_clock::now();
    batchsim::Simulator sim(job.spec, job.ps, job.config, job.trace ? &*job.trace : nullptr,
                            job.client ? &*job.client : nullptr);
    sim.set_hook(&hook);
    batchsim::SimResult res;
    try {
      res = sim.run();
      ex.sync();
    } catch (...) {
      cudaFreeHost(results);
      throw;
    }
    const double wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    std::ostringstream os;
    json outs = json::array();
    for (const auto& o : res.outcomes) outs.push_back(batchsim::outcome_to_json(o));
    os << json{{"ev", "outcomes"}, {"outcomes", outs}}.dump() << '\n';
    json top1 = json::array();
    for (std::size_t i = 0; i < count; ++i) {
      const float* p = results + i * hook.classes;
      int best = 0;
      for (int c = 1; c < hook.classes; ++c)
        if (p[c] > p[best]) best = c;
      top1.push_back(p[best] > 0 ? best : -1);
    }
    json dumped = json::object();
    for (const auto& idj : j.value("dump_ids", json::array())) {
      const std::int64_t id = idj.get<std::int64_t>();
      if (id >= 1 && static_cast<std::size_t>(id) <= count)
        dumped[std::to_string(id)] =
            std::vector<float>(results + (id - 1) * hook.classes, results + id * hook.classes);
    }
    cudaFreeHost(results);
    json sm = batchsim::summary_to_json(res.metrics);
    sm["wall_ms"] = wall_ms;
    os << json{{"ev", "results"}, {"top1", top1}, {"probs", dumped}, {"launches", ex.launches() - launches0},
               {"steps", hook.steps}, {"max_step_batch", hook.max_batch_seen},
               {"rider_steps", hook.rider_steps}, {"riders", hook.riders_total}}
              .dump()
       << '\n';
    os << sm.dump() << '\n';
    *out = dup_str(os.str());
    return BS_OK;
  });
}

int bs_serve(bs_handle* h, const char* job_json, char** out) {
  return guarded([&] {
    *out = dup_str(serve_live(*h->ex, with_window_cap(h, json::parse(job_json))).dump());
    return BS_OK;
  });
}

int bs_profile_table(bs_handle* h, const char* opts_json, char** out) {
  return guarded([&] {
    *out = dup_str(measure_profile(*h->ex, json::parse(opts_json)).dump());
    return BS_OK;
  });
}

int bs_stats(bs_handle* h, int enable, int every) {
  return guarded([&] {
    h->ex->sync();
    h->ex->clear_stats();
    h->ex->enable_stats(enable != 0, every);
    return BS_OK;
  });
}

// Per-kind sums over the sampled launches: count, device ms, algorithmic
// bytes and FLOPs, plus ideal time at the given peaks.
int bs_stats_summary(bs_handle* h, double hbm_gbs, double tensor_tflops, char** out) {
  return guarded([&] {
    h->ex->sync();
    json kinds = json::object();
    for (const LaunchStat& st : h->ex->stats()) {
      float ms = 0;
      if (cudaEventElapsedTime(&ms, st.t0, st.t1) != cudaSuccess) continue;
      const char* k = st.gemv                      ? "fc_gemv"
                      : st.kind == OpKind::conv    ? "conv_tc"
                      : st.kind == OpKind::maxpool ? "maxpool"
                      : st.kind == OpKind::avgpool ? "avgpool"
                      : st.kind == OpKind::dwconv  ? "dwconv"
                                                   : "softmax";
      json& e = kinds[k];
      if (e.is_null()) e = {{"launches", 0}, {"ms", 0.0}, {"bytes", 0.0}, {"flops", 0.0}, {"ideal_ms", 0.0},
                            {"ideal_hbm_ms", 0.0}, {"ideal_tensor_ms", 0.0}};
      const double t_hbm = st.bytes / (hbm_gbs * 1e9) * 1e3;
      const double t_tc = st.flops / (tensor_tflops * 1e12) * 1e3;
      e["launches"] = e["launches"].get<int>() + 1;
      e["ms"] = e["ms"].get<double>() + ms;
      e["bytes"] = e["bytes"].get<double>() + st.bytes;
      e["flops"] = e["flops"].get<double>() + st.flops;
      e["ideal_ms"] = e["ideal_ms"].get<double>() + std::max(t_hbm, t_tc);
      e["ideal_hbm_ms"] = e["ideal_hbm_ms"].get<double>() + t_hbm;
      e["ideal_tensor_ms"] = e["ideal_tensor_ms"].get<double>() + t_tc;
    }
    *out = dup_str(kinds.dump());
    return BS_OK;
  });
}

void bs_free(char* p) { std::free(p); }

}  // extern "C"
