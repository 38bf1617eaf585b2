#include "live.hpp"

#include <algorithm>
#include <array>
#include <chrono>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <stdexcept>
#include <thread>
#include <vector>

#include "bsb/jobs.hpp"
#include "image.hpp"

using json = nlohmann::json;

namespace bs200 {

namespace {

using Clock = std::chrono::steady_clock;

double ms_since(Clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

struct Book {
  int dnn = 0;
  double arrival = 0, deadline = 0, completion = -1;
  bool dropped = false, done = false;
  batchsim::CompletionLocation location = batchsim::CompletionLocation::server;
};

struct InFlight {
  cudaEvent_t ev = nullptr;
  double expected_end = 0;
  std::vector<batchsim::RequestId> finishing;
};

}  // namespace

json serve_live(Executor& ex, const json& j) {
  using namespace batchsim;
  SimJob job = sim_job_from_json(j);
  const Suite& suite = ex.suite();
  std::vector<int> dnn_map;
  for (const auto& d : job.ps.dnns) {
    int idx = -1;
    for (std::size_t i = 0; i < suite.nets.size(); ++i)
      if (suite.nets[i].name == d.name()) idx = static_cast<int>(i);
    if (idx < 0 || suite.nets[static_cast<std::size_t>(idx)].num_layers() != d.num_layers())
      throw std::invalid_argument("profile dnn '" + d.name() + "' does not match suite " + suite.name);
    dnn_map.push_back(idx);
  }
  const int pool = j.value("image_pool", 32);
  const bool h2d = j.value("h2d", false);
  const std::uint64_t image_seed = j.value("image_seed", std::uint64_t{1});
  const int depth = std::max(1, j.value("pipeline_depth", 2));
  const bool deadlines = job.spec.relative_deadline < kNoDeadline;

  // Inputs: device-resident pool (kernel-level runs) or pinned host images
  // copied H2D at admission (end-to-end runs).
  std::vector<std::uint8_t*> host_pool(suite.nets.size(), nullptr);
  std::vector<std::size_t> img_floats(suite.nets.size(), 0);  // bytes per packed 8-bit RGB image
  for (std::size_t d = 0; d < dnn_map.size(); ++d) {
    const int net = dnn_map[d];
    const NetDef& nd = suite.nets[static_cast<std::size_t>(net)];
    // e2e runs ship the images as decoded 8-bit RGB from pinned host memory
    // (csrc/exec/image.hpp: the same pixels the device-resident pool holds).
    img_floats[static_cast<std::size_t>(net)] = static_cast<std::size_t>(nd.in_H) * nd.in_W * 3;
    if (h2d) {
      if (!host_pool[static_cast<std::size_t>(net)]) {
        std::uint8_t* p = nullptr;
        if (cudaMallocHost(&p, img_floats[static_cast<std::size_t>(net)] * pool) != cudaSuccess)
          throw std::runtime_error("pinned image pool");
        for (int i = 0; i < pool; ++i)
          synth_image_bytes(image_seed, static_cast<std::uint64_t>(i), nd.in_H, nd.in_W, 3,
                            p + img_floats[static_cast<std::size_t>(net)] * static_cast<std::size_t>(i));
        host_pool[static_cast<std::size_t>(net)] = p;
      }
    } else if (ex.pool_size(net) < pool) {
      ex.make_image_pool(net, pool, image_seed);
    }
  }

  const std::vector<ArrivalRecord> arrivals = generate_arrivals(job.spec);
  const std::size_t n = arrivals.size();
  // ids follow arrival order (the pending queue's binary search relies on it)
  for (std::size_t i = 1; i < n; ++i)
    if (arrivals[i].time < arrivals[i - 1].time) throw std::logic_error("serve: arrivals out of time order");

  // Server admissions: (time at the server, id, entry layer). Without
  // offload every request arrives at layer 1 at its generation time. In
  // collaborative mode (config 5) the client side -- per-client compute
  // queues, the uplink trace, the EWMA throughput estimate and the
  // binary / partial offload decision (reference simulator.hpp:286-433,
  // offload.hpp:22-161) -- does not depend on the server, so it is replayed
  // in virtual time by the reference-semantics Simulator with a recording
  // hook, and its server arrivals (request id, entry layer) are served live:
  // the intermediate activation of the client's prefix is computed on the
  // executor's side stream at admission (Executor::admit, entry_layer > 1).
  // Requests the client finishes on its own complete at their client time.
  struct Admission {
    double time;
    RequestId id;
    int entry_layer;
  };
  std::vector<Admission> adm;
  std::vector<double> client_done(n, -1.0);
  std::vector<CompletionLocation> client_loc(n, CompletionLocation::server);
  const bool collab = job.config.offload != OffloadMode::none;
  if (collab) {
    struct Recorder : StepHook {
      std::vector<Admission>* adm = nullptr;
      void admit(RequestId id, int, int entry_layer, Ms now) override { adm->push_back({now, id, entry_layer}); }
    } rec;
    rec.adm = &adm;
    Simulator client_side(job.spec, job.ps, job.config, job.trace ? &*job.trace : nullptr,
                          job.client ? &*job.client : nullptr);
    client_side.set_hook(&rec);
    const SimResult res = client_side.run();
    std::vector<char> at_server(n + 1, 0);
    for (const Admission& a : adm) at_server[static_cast<std::size_t>(a.id)] = 1;
    for (const RequestOutcome& o : res.outcomes)
      if (!at_server[static_cast<std::size_t>(o.id)] && !o.dropped) {
        client_done[static_cast<std::size_t>(o.id - 1)] = o.completion;
        client_loc[static_cast<std::size_t>(o.id - 1)] = o.location;
      }
    std::sort(adm.begin(), adm.end(),
              [](const Admission& x, const Admission& y) { return x.time < y.time || (x.time == y.time && x.id < y.id); });
  } else {
    adm.reserve(n);
    for (std::size_t i = 0; i < n; ++i) adm.push_back({arrivals[i].time, static_cast<RequestId>(i) + 1, 1});
  }
  const std::size_t n_adm = adm.size();
  std::vector<Book> book(n);
  std::vector<int> mix;
  if (job.spec.dnn_mix.empty()) {
    mix.push_back(0);
  } else {
    for (const auto& m : job.spec.dnn_mix) mix.push_back(job.ps.dnn_index(m.first));
  }
  int classes = 0;
  for (const NetDef& nd : suite.nets) classes = std::max(classes, nd.num_classes);
  float* results = nullptr;
  if (cudaMallocHost(&results, std::max<std::size_t>(n, 1) * classes * sizeof(float)) != cudaSuccess)
    throw std::runtime_error("pinned results");

  Planner planner(job.ps, job.config);
  std::vector<Request> pending;
  Schedule plan;
  std::vector<detail::ExecStep> steps;
  std::size_t next_step = 0;
  int plan_no = 0;
  bool needs_schedule = false;
  int arrivals_since = 0;
  std::deque<InFlight> inflight;
  std::vector<cudaEvent_t> ev_free;
  std::size_t ai = 0, resolved = 0;
  long n_steps = 0, n_plans = 0, h2d_bytes = 0, d2h_bytes = 0;
  double sched_ms = 0, max_sched_ms = 0;
  double predicted_ms = 0;  // sum of the launched steps' table durations (what the scheduler assumed)
  double host_admit_ms = 0, host_step_ms = 0;  // host time in admissions / step issue (+ bookkeeping)
  const long launches0 = ex.launches();
  std::vector<int> step_batch_hist;
  // BS_LIVE_STEP_TIMES=1 (diagnostics, pointer-table mode 2): per step, its
  // predicted duration and its device time from the table-write kernels'
  // global-timer stamps (each stamps the end of all earlier work, so step k
  // lasted stamp(k + 1) - stamp(k); no extra launch or event).
  const char* st_env = std::getenv("BS_LIVE_STEP_TIMES");
  const bool step_times = st_env && std::atoi(st_env) != 0;
  std::vector<std::uint64_t> st_seq;
  std::vector<std::array<double, 8>> st_info;  // from, to, batch, predicted ms, in flight, new members, finishing, riders

  auto finish = [&](RequestId id, double t) {
    Book& b = book[static_cast<std::size_t>(id - 1)];
    b.completion = t;
    b.done = true;
    ++resolved;
  };
  auto drop = [&](RequestId id) {
    Book& b = book[static_cast<std::size_t>(id - 1)];
    if (b.done || b.dropped) return;
    b.dropped = true;
    ++resolved;
    ex.drop(id);
  };
  auto layer_shared = [&](int dnn, int layer) { return job.ps.layer_is_shared(dnn, layer); };

  // Every request's generation-time facts; client-finished requests resolve
  // at their client completion time.
  for (std::size_t i = 0; i < n; ++i) {
    Book& b = book[i];
    b.dnn = mix[static_cast<std::size_t>(arrivals[i].dnn) % mix.size()];
    b.arrival = arrivals[i].time;
    b.deadline = deadlines ? arrivals[i].time + job.spec.relative_deadline : kNoDeadline;
    if (client_done[i] >= 0) {
      b.location = client_loc[i];
      finish(static_cast<RequestId>(i) + 1, client_done[i]);
    }
  }
  ex.sync();
  // H2D images up to this size are admitted in batches per loop iteration
  // (Executor::admit_rgb_many: SmallCNN's 3 KB images at ~100k req/s made one
  // copy + launch + event per request the host loop's bound); larger ones
  // (GoogLeNet's 150 KB) keep one DMA straight from the pinned pool each.
  const long batch_admit_bytes = [] {
    const char* e = std::getenv("BS_BATCH_ADMIT_BYTES");
    return e ? std::atol(e) : 16384L;
  }();
  // BS_BATCH_ADMIT_LARGE=1: larger images batched too (per-image DMA, shared
  // expansion launch and ready event) -- A/B switch
  const bool batch_admit_large = [] {
    const char* e = std::getenv("BS_BATCH_ADMIT_LARGE");
    return e && std::atoi(e) != 0;
  }();
  std::vector<std::vector<RequestId>> batch_ids(ex.suite().nets.size());
  std::vector<std::vector<const std::uint8_t*>> batch_src(ex.suite().nets.size());
  cudaEvent_t dev0, dev1;
  cudaEventCreate(&dev0);
  cudaEventCreate(&dev1);
  const Clock::time_point t0 = Clock::now();
  cudaEventRecord(dev0, ex.stream());
  while (resolved < n) {
    double now = ms_since(t0);
    // 1. admissions
    const auto ha0 = Clock::now();
    while (ai < n_adm && adm[ai].time <= now) {
      const RequestId id = adm[ai].id;
      const std::size_t i = static_cast<std::size_t>(id - 1);
      Book& b = book[i];
      const int net = dnn_map[static_cast<std::size_t>(b.dnn)];
      const int img = static_cast<int>(i % static_cast<std::size_t>(pool));
      if (h2d && adm[ai].entry_layer == 1) {
        const std::uint8_t* src = host_pool[static_cast<std::size_t>(net)] + img_floats[static_cast<std::size_t>(net)] * img;
        if (static_cast<long>(img_floats[static_cast<std::size_t>(net)]) <= batch_admit_bytes || batch_admit_large) {
          batch_ids[static_cast<std::size_t>(net)].push_back(id);
          batch_src[static_cast<std::size_t>(net)].push_back(src);
        } else {
          ex.admit_rgb(id, net, src);
        }
        h2d_bytes += static_cast<long>(img_floats[static_cast<std::size_t>(net)]);
      } else {
        if (adm[ai].entry_layer == 1)
          ex.admit_ref(id, net, ex.pool_image(net, img));  // HBM-resident input: read in place by layer 1
        else
          ex.admit(id, net, adm[ai].entry_layer, ex.pool_image(net, img), true);
      }
      Request r;
      r.id = id;
      r.dnn = b.dnn;
      r.arrival = b.arrival;
      r.deadline = b.deadline;
      r.layer = adm[ai].entry_layer;
      if (collab) r.origin = static_cast<int>((id - 1) % static_cast<RequestId>(job.config.clients));
      pending.insert(std::upper_bound(pending.begin(), pending.end(), r, arrives_before), r);
      ++arrivals_since;
      ++ai;
    }
    // small images arrived in this iteration: one packed copy + expansion per DNN
    for (std::size_t q = 0; q < batch_ids.size(); ++q) {
      if (batch_ids[q].empty()) continue;
      // images above the packing size come from the pinned pool: DMA'd one by
      // one into consecutive staging slots, one expansion + event per batch
      ex.admit_rgb_many(batch_ids[q].data(), static_cast<int>(q), batch_src[q].data(),
                        static_cast<int>(batch_ids[q].size()),
                        static_cast<long>(img_floats[q]) > batch_admit_bytes);
      batch_ids[q].clear();
      batch_src[q].clear();
    }
    host_admit_ms += std::chrono::duration<double, std::milli>(Clock::now() - ha0).count();
    // 2. completions (in stream order)
    while (!inflight.empty() && cudaEventQuery(inflight.front().ev) == cudaSuccess) {
      now = ms_since(t0);
      for (RequestId id : inflight.front().finishing) finish(id, now);
      ev_free.push_back(inflight.front().ev);
      inflight.pop_front();
    }
    // 3. plan + launch while the pipeline has room
    if (static_cast<int>(inflight.size()) < depth && !pending.empty()) {
      const double start_est = inflight.empty() ? now : std::max(now, inflight.back().expected_end);
      if ((needs_schedule || next_step >= steps.size())) {
        const auto s0 = Clock::now();
        needs_schedule = false;
        arrivals_since = 0;
        next_step = 0;
        steps.clear();
        Planner::Result r = planner.plan(pending, start_est, deadlines);
        for (RequestId id : r.dropped) drop(id);
        if (r.computed) {
          plan = std::move(r.plan);
          steps = std::move(r.steps);
          ++plan_no;
          ++n_plans;
          ex.new_plan(plan_no);
        }
        const double dt = std::chrono::duration<double, std::milli>(Clock::now() - s0).count();
        sched_ms += dt;
        max_sched_ms = std::max(max_sched_ms, dt);
      }
      if (next_step < steps.size()) {
        const auto hs0 = Clock::now();
        const detail::ExecStep st = steps[next_step];
        const std::uint64_t seq0 = ex.step_seq();
        const ScheduledSegment& seg = plan.segments[static_cast<std::size_t>(st.segment)];
        // pending is FIFO by (arrival, id) and live ids are assigned in
        // arrival order, so it is sorted by id: members are found by binary
        // search (was a linear scan of pending per member).
        auto find_pending = [&](RequestId id) {
          auto it = std::lower_bound(pending.begin(), pending.end(), id,
                                     [](const Request& r, RequestId v) { return r.id < v; });
          return (it != pending.end() && it->id == id) ? it : pending.end();
        };
        std::vector<std::pair<std::int64_t, int>> members;
        members.reserve(seg.members.size());
        for (RequestId id : seg.members) {
          auto it = find_pending(id);
          if (it != pending.end()) members.emplace_back(id, it->layer);
        }
        ex.step(plan_no, st.segment, dnn_map[static_cast<std::size_t>(seg.dnn)], st.layer_from, st.layer_to, members,
                seg.riders);
        ++n_steps;
        step_batch_hist.push_back(static_cast<int>(members.size() + seg.riders.size()));
        // Effects apply at launch (the stream guarantees completion order);
        // completion times are stamped when the step's event fires.
        InFlight f;
        bool crossed = false;
        for (RequestId id : seg.members) {
          auto it = find_pending(id);
          if (it == pending.end() || it->layer > st.layer_to) continue;
          const int was = it->layer;
          it->layer = st.layer_to + 1;
          const int nl = job.ps.dnns[static_cast<std::size_t>(it->dnn)].num_layers();
          if (it->layer > nl) {
            d2h_bytes += classes * static_cast<long>(sizeof(float));
            f.finishing.push_back(id);
            pending.erase(it);
          } else if (planner.has_shared() && layer_shared(it->dnn, was) != layer_shared(it->dnn, it->layer)) {
            crossed = true;
          }
        }
        std::vector<std::int64_t> deposited;
        for (const Rider& rider : seg.riders) {
          if (rider.leave_layer > st.layer_to || rider.join_layer > st.layer_to) continue;
          auto it = find_pending(rider.id);
          if (it == pending.end() || it->dnn != rider.dnn || it->layer >= rider.deposit_layer) continue;
          it->layer = rider.deposit_layer;
          crossed = true;
          deposited.push_back(rider.id);
        }
        ex.step_done(deposited);
        for (std::int64_t id : deposited) {
          auto it = find_pending(id);
          if (it != pending.end() && it->layer > job.ps.dnns[static_cast<std::size_t>(it->dnn)].num_layers()) {
            d2h_bytes += classes * static_cast<long>(sizeof(float));
            f.finishing.push_back(id);
            pending.erase(it);
          }
        }
        // One copy-out kernel for the step's finishing requests (a DMA per
        // request serialised ~3 us each on the serving stream).
        if (!f.finishing.empty()) {
          std::vector<float*> outs;
          outs.reserve(f.finishing.size());
          for (RequestId id : f.finishing) outs.push_back(results + static_cast<std::size_t>(id - 1) * classes);
          ex.retire_many_async(f.finishing, outs, classes);
        }
        if (ev_free.empty()) {
          cudaEvent_t e;
          cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
          ev_free.push_back(e);
        }
        f.ev = ev_free.back();
        ev_free.pop_back();
        cudaEventRecord(f.ev, ex.stream());
        if (step_times && ex.step_seq() > seq0) {
          int fresh = 0;
          for (const auto& m : members) fresh += m.second == 1;
          st_seq.push_back(ex.step_seq());
          int riding = 0;
          for (const Rider& rd : seg.riders) riding += rd.join_layer <= st.layer_to && rd.leave_layer >= st.layer_from;
          st_info.push_back({static_cast<double>(st.layer_from), static_cast<double>(st.layer_to),
                             static_cast<double>(members.size() + seg.riders.size()), st.duration,
                             static_cast<double>(inflight.size()), static_cast<double>(fresh),
                             static_cast<double>(f.finishing.size()), static_cast<double>(riding)});
        }
        f.expected_end = start_est + st.duration;
        predicted_ms += st.duration;
        inflight.push_back(std::move(f));
        ++next_step;
        if (reschedule_trigger(true, arrivals_since > 0, crossed)) needs_schedule = true;
        host_step_ms += std::chrono::duration<double, std::milli>(Clock::now() - hs0).count();
        continue;
      }
    }
    // 4. idle: wait for the next event
    if (inflight.empty() && pending.empty() && ai < n_adm) {
      const double wait = adm[ai].time - ms_since(t0);
      if (wait > 0.2) std::this_thread::sleep_for(std::chrono::microseconds(static_cast<long>((wait - 0.1) * 1000)));
    }
  }
  cudaEventRecord(dev1, ex.stream());
  ex.sync();
  const double wall = ms_since(t0);
  float device_ms = 0;
  cudaEventElapsedTime(&device_ms, dev0, dev1);
  json step_rows = json::array();
  if (!st_seq.empty()) {
    const std::vector<std::uint64_t> stamp = ex.stamps();
    const auto at = [&](std::uint64_t q) { return stamp[q % Executor::kStampCap]; };
    for (std::size_t k = 0; k + 1 < st_seq.size(); ++k) {
      if (st_seq[k + 1] - st_seq[0] >= static_cast<std::uint64_t>(Executor::kStampCap)) break;
      json row = json::array();
      for (double v : st_info[k]) row.push_back(v);
      row.push_back(static_cast<double>(at(st_seq[k + 1]) - at(st_seq[k])) * 1e-6);
      step_rows.push_back(row);
    }
  }
  cudaEventDestroy(dev0);
  cudaEventDestroy(dev1);
  for (cudaEvent_t e : ev_free) cudaEventDestroy(e);

  // Outcomes (reference semantics: drops count against on-time).
  std::vector<RequestOutcome> outs(n);
  double first_arrival = n ? arrivals.front().time : 0, last_completion = 0;
  int on_time_completed = 0, server_completed = 0;
  json top1 = json::array();
  for (std::size_t i = 0; i < n; ++i) {
    RequestOutcome& o = outs[i];
    const Book& b = book[i];
    o.id = static_cast<RequestId>(i) + 1;
    o.dnn = b.dnn;
    o.arrival = b.arrival;
    o.deadline = b.deadline;
    o.dropped = b.dropped;
    o.location = b.location;
    if (b.done) {
      o.completion = b.completion;
      o.on_time = b.deadline >= kNoDeadline || b.completion <= b.deadline;
      last_completion = std::max(last_completion, b.completion);
      if (o.on_time) ++on_time_completed;
      if (b.location != CompletionLocation::server) {  // finished on its client: no server output
        top1.push_back(-1);
        continue;
      }
      ++server_completed;
      const float* p = results + i * classes;
      int best = 0;
      for (int c = 1; c < classes; ++c)
        if (p[c] > p[best]) best = c;
      top1.push_back(best);
    } else {
      top1.push_back(-1);
    }
  }
  json dumped = json::object();
  for (const auto& idj : j.value("dump_ids", json::array())) {
    const std::int64_t id = idj.get<std::int64_t>();
    if (id >= 1 && static_cast<std::size_t>(id) <= n && book[static_cast<std::size_t>(id - 1)].done &&
        book[static_cast<std::size_t>(id - 1)].location == CompletionLocation::server)
      dumped[std::to_string(id)] = std::vector<float>(results + (id - 1) * classes, results + id * classes);
  }
  cudaFreeHost(results);
  for (std::uint8_t* p : host_pool)
    if (p) cudaFreeHost(p);
  const SummaryMetrics m = summarize(outs);
  const double span_s = (last_completion - first_arrival) / 1000.0;
  json out = summary_to_json(m);
  out["on_time_ratio_f"] = m.on_time_ratio;
  out["mean_completion_ms"] = m.mean_completion;
  out["median_completion_ms"] = m.median_completion;
  out["p95_completion_ms"] = m.p95_completion;
  out["served_rps"] = span_s > 0 ? m.completed / span_s : 0.0;
  out["goodput_rps"] = span_s > 0 ? on_time_completed / span_s : 0.0;
  out["offered_rps"] = job.spec.rate;
  out["server_completed"] = server_completed;
  out["predicted_step_ms_total"] = predicted_ms;
  out["server_admissions"] = n_adm;
  out["admitted_mid_network"] = std::count_if(adm.begin(), adm.end(), [](const Admission& a) { return a.entry_layer > 1; });  // completed on the GPU (collab: excludes client-finished)
  out["server_served_rps"] = span_s > 0 ? server_completed / span_s : 0.0;
  out["wall_ms"] = wall;
  out["host_admit_ms"] = host_admit_ms;
  out["host_step_ms"] = host_step_ms;
  out["device_ms"] = device_ms;  // CUDA events on the serving stream, first admission to last retire
  out["span_ms"] = last_completion - first_arrival;
  out["steps"] = n_steps;
  if (step_times) out["step_times"] = step_rows;  // [from, to, batch, predicted, in flight, new, finishing, riders, device ms]
  out["plans"] = n_plans;
  out["sched_ms_total"] = sched_ms;
  out["sched_ms_max"] = max_sched_ms;
  out["launches"] = ex.launches() - launches0;
  {
    // step size distribution (members + riders of each launched step)
    double sum = 0;
    json hist = json::object();
    for (int b : step_batch_hist) {
      sum += b;
      const int bucket = b <= 1 ? 1 : b <= 4 ? 4 : b <= 16 ? 16 : b <= 48 ? 48 : 90;
      hist[std::to_string(bucket)] = hist.value(std::to_string(bucket), 0) + 1;
    }
    out["step_members_mean"] = step_batch_hist.empty() ? 0.0 : sum / static_cast<double>(step_batch_hist.size());
    out["step_members_hist"] = hist;
  }
  out["h2d_bytes"] = h2d_bytes;
  out["d2h_bytes"] = d2h_bytes;
  out["top1"] = top1;
  out["probs"] = dumped;
  if (!dumped.empty()) {  // suite network of every request (to check dumped outputs)
    std::vector<int> nets(n);
    for (std::size_t i = 0; i < n; ++i) nets[i] = dnn_map[static_cast<std::size_t>(book[i].dnn)];
    out["dnn_of"] = nets;
  }
  return out;
}

json measure_profile(Executor& ex, const json& opts) {
  const Suite& s = ex.suite();
  std::vector<int> batches = opts.value("batches", std::vector<int>{1, 2, 4, 8, 16, 32, 64, 90});
  batches.erase(std::remove_if(batches.begin(), batches.end(), [&](int b) { return b < 1 || b > ex.max_batch(); }),
                batches.end());
  if (std::find(batches.begin(), batches.end(), 1) == batches.end()) batches.insert(batches.begin(), 1);
  const int reps = opts.value("reps", 10);
  const bool flush = opts.value("flush_l2", false);
  json tuned = nullptr;
  if (opts.value("tune_tiles", false)) tuned = json::parse(ex.tune_tiles(batches, std::max(3, reps / 2)));
  // "step" (default): each layer as a one-layer serving step inside
  // back-to-back passes run as such steps (pointer-table kernel + layer,
  // results copy-out after the last; device stamps, Executor::profile_steps)
  // -- what the live loop's layer-granular steps cost; "pass": each layer's latency inside back-to-back passes with
  // events between the layers, columns scaled to the whole-pass time
  // (round-2 tables); "layer": each layer alone, synchronised (adds launch
  // latency and idle gaps per layer; the only mode with flush_l2, which needs
  // an L2 flush before every timed layer). BS_TABLE_TIMING overrides.
  const char* tt_env = std::getenv("BS_TABLE_TIMING");
  const std::string timing = flush ? "layer" : (tt_env && tt_env[0]) ? std::string(tt_env) : opts.value("timing", std::string("step"));
  if (timing != "pass" && timing != "layer" && timing != "step") throw std::invalid_argument("timing: step | pass | layer");
  // pass timings of every net at every batch: [net][batch index][layer - 1]
  std::vector<std::vector<std::vector<double>>> pass_ms(s.nets.size());
  // The events between layers break the programmatic-dependent-launch
  // overlap a multi-layer step has, so the per-layer medians sum above what
  // the same layers cost back to back. With scale_to_pass (default; env
  // BS_TABLE_SCALE=0 disables) each (net, batch) column is scaled so that it
  // sums to the median whole-pass time measured without inner events: the
  // layers' relative costs come from the events, the total from the chain.
  const char* sc_env = std::getenv("BS_TABLE_SCALE");
  const bool scale = opts.value("scale_to_pass", true) && !(sc_env && sc_env[0] == '0');
  json scales = json::array();
  if (timing == "step")
    for (std::size_t i = 0; i < s.nets.size(); ++i)
      for (int b : batches) pass_ms[i].push_back(ex.profile_steps(static_cast<int>(i), b, reps));
  if (timing == "pass")
    for (std::size_t i = 0; i < s.nets.size(); ++i)
      for (int b : batches) {
        std::vector<double> col = ex.profile_pass(static_cast<int>(i), b, reps);
        if (scale) {
          double sum = 0;
          for (double v : col) sum += v;
          const double whole = ex.profile_pass_total(static_cast<int>(i), b, reps);
          const double f = sum > 0 ? whole / sum : 1.0;
          for (double& v : col) v *= f;
          scales.push_back(json::array({s.nets[i].name, b, f}));
        }
        pass_ms[i].push_back(std::move(col));
      }
  json comps = json::array();
  for (std::size_t c = 0; c < s.components.size(); ++c) {
    // measure a component inside the first DNN that contains it
    const NetDef* net = nullptr;
    int net_idx = 0;
    for (std::size_t i = 0; i < s.nets.size() && !net; ++i)
      for (int cc : s.nets[i].components)
        if (cc == static_cast<int>(c)) {
          net = &s.nets[i];
          net_idx = static_cast<int>(i);
          break;
        }
    json layers = json::array();
    for (int k = 1; k <= net->num_layers(); ++k) {
      const LayerDef& L = net->layers[static_cast<std::size_t>(k - 1)];
      if (L.component != static_cast<int>(c)) continue;
      json grid = json::array();
      for (std::size_t bi = 0; bi < batches.size(); ++bi) {
        const int b = batches[bi];
        const double ms = timing != "layer" ? pass_ms[static_cast<std::size_t>(net_idx)][bi][static_cast<std::size_t>(k - 1)]
                                           : ex.profile_layer(net_idx, k, b, reps, flush);
        grid.push_back(json::array({b, ms}));
      }
      const OpDef& last = net->ops[static_cast<std::size_t>(L.ops.back())];
      const long bits = 32L * last.Ho * std::max(last.Wo, 1) * last.out.C;
      layers.push_back({{"name", L.name}, {"output_bits", bits}, {"runtime_ms", grid}});
    }
    comps.push_back({{"id", s.components[c].id}, {"layers", layers}});
  }
  json dnns = json::array();
  for (const NetDef& n : s.nets) {
    json stages = json::array();
    for (int c : n.components) stages.push_back(s.components[static_cast<std::size_t>(c)].id);
    dnns.push_back({{"id", n.name}, {"stages", stages}});
  }
  json prof = {{"max_batch", ex.max_batch()}, {"components", comps}, {"dnns", dnns}};
  if (!tuned.is_null()) prof["tile_tune"] = tuned;  // [op, batch, choice, layer ms] (extra key; opt-in)
  prof["timing"] = timing;                          // extra key (ignored by the profile parsers)
  if (!scales.empty()) prof["pass_scale"] = scales;  // [net, batch, whole pass / sum of layers]
  return prof;
}

}  // namespace bs200
