// The serving event loop: request queue, per-DNN layer progress, plan ->
// steps -> batched step -> progress, re-scheduling at step boundaries.
// Drop-in for the reference's proj/include/batchsim/simulator.hpp:35-820.
//
// Two additions for the B200 build, neither of which changes a scheduling
// decision:
//   * StepHook — the batched step is *executed*: the hook receives the exact
//     batch membership of every layer of every step (members + riders), the
//     admissions, completions and drops (bs_exec.h wires libbs_exec.so here);
//   * SimObserver — plan/step trace for bit-exact parity checks.
// Time here is the virtual clock of the cost table (replay mode); the live
// wall-clock server lives in the executor library (live_server.cu).
#pragma once

#include <cstdint>
#include <deque>
#include <optional>
#include <queue>
#include <string>
#include <vector>

#include "arrivals.hpp"
#include "schedulers.hpp"

namespace batchsim {

enum class SchedulerKind { ours_time, ours_tardy, edf, batch, no_batch };
SchedulerKind parse_scheduler(const std::string& name);
const char* scheduler_name(SchedulerKind k);

enum class OffloadMode { none, binary, partial };
OffloadMode parse_offload(const std::string& name);

struct SimConfig {
  SchedulerKind scheduler = SchedulerKind::ours_time;
  SplitGranularity granularity = SplitGranularity::per_group;
  int groups = 5;
  int max_batch = 90;
  int window_cap = 500;
  Ms scheduler_latency = 0;
  Ms step_overhead = 0;
  OffloadMode offload = OffloadMode::none;
  PartialRule partial_rule = PartialRule::min_completion;
  int clients = 0;
  bool shared_batching = true;
};

struct SummaryMetrics {
  int generated = 0;
  int completed = 0;
  int dropped = 0;
  int on_time = 0;
  double on_time_ratio = 0;
  Ms mean_completion = 0;
  Ms median_completion = 0;
  Ms p95_completion = 0;
  int at_server = 0;
  int at_client_full = 0;
  int at_client_partial = 0;
  Ms mean_network_delay = 0;
  double mean_solve_wall_ms = 0;
  int schedules_computed = 0;
};

SummaryMetrics summarize(const std::vector<RequestOutcome>& outcomes);

struct SimResult {
  std::vector<RequestOutcome> outcomes;
  SummaryMetrics metrics;
};

namespace detail {
struct ExecStep {
  int segment = 0;
  int layer_from = 0;
  int layer_to = 0;
  Ms duration = 0;
};
}  // namespace detail

// One batched step as the executor sees it. Layer k of [from, to] runs on
// {members with layer <= k} U {riders with join <= k <= leave}
// (ref: simulator.hpp:705-713).
struct StepView {
  int plan = 0;     // plan number (rides do not survive a new plan)
  int segment = 0;
  int dnn = 0;
  int from = 0, to = 0;
  Ms start = 0, end = 0;  // virtual times
  std::vector<std::pair<RequestId, int>> members;  // (id, layer at step start), arrival order
  std::vector<Rider> riders;
};

struct StepHook {
  virtual ~StepHook() = default;
  virtual void admit(RequestId id, int dnn, int entry_layer, Ms now) {}
  virtual void plan(int plan_no, Ms now) {}
  virtual void step(const StepView& s) {}
  // Riders that were deposited at the end of the step (their ride commits).
  virtual void step_done(const StepView& s, const std::vector<RequestId>& deposited) {}
  virtual void finish(RequestId id, Ms when) {}
  virtual void drop(RequestId id, Ms now) {}
};

// The reference's plan -> steps pipeline (simulator.hpp:541-721):
// expiry drops, window cap, scheduler dispatch (incl. the Our-Tardy drop
// loop), and the expansion of a schedule into executable steps with their
// cost-table durations. Shared by the virtual-time Simulator and the live
// wall-clock server so both make identical decisions on identical state.
class Planner {
 public:
  Planner(const ProfileSet& ps, const SimConfig& config);
  struct Result {
    bool computed = false;  // false: the window emptied through expiry drops
    Schedule plan;
    std::vector<detail::ExecStep> steps;
    std::vector<RequestId> dropped;  // expiry drops first, then tardy drops
  };
  Result plan(std::vector<Request>& pending, Ms now, bool deadlines);
  Ms step_duration(const ScheduledSegment& seg, int from, int to, const std::vector<int>& layer_of) const;
  bool has_shared() const { return has_shared_; }

 private:
  Schedule run_scheduler(std::vector<Request>& window, std::vector<Request>& pending, Ms now,
                         std::vector<RequestId>& dropped);
  Schedule tardy_multi(std::span<const Request> window, Ms now, const DpOptions& dp);
  std::vector<detail::ExecStep> build_steps(const Schedule& plan, const std::vector<Request>& pending) const;

  const ProfileSet& ps_;
  SimConfig config_;
  bool has_shared_ = false;
  DpTable dp_cache_;
};

struct SimObserver {
  virtual ~SimObserver() = default;
  virtual void on_plan(Ms now, int plan_no, const Schedule& plan,
                       const std::vector<detail::ExecStep>& steps) {}
  virtual void on_step(Ms now, int plan_no, std::size_t index, Ms end,
                       const detail::ExecStep& step) {}
};

class Simulator {
 public:
  Simulator(const WorkloadSpec& spec, const ProfileSet& ps, const SimConfig& config,
            const NetworkTrace* trace = nullptr, const ClientProfile* client_profile = nullptr);

  void set_hook(StepHook* hook) { hook_ = hook; }
  void set_observer(SimObserver* obs) { obs_ = obs; }
  SimResult run();

 private:
  enum class Kind : int { step_complete = 0, client_complete = 1, transmission_complete = 2, request_arrival = 3 };
  struct Event {
    Ms time;
    Kind kind;
    RequestId id;
    std::uint64_t seq;
  };
  struct Later {
    bool operator()(const Event& a, const Event& b) const {
      if (a.time != b.time) return a.time > b.time;
      if (a.kind != b.kind) return static_cast<int>(a.kind) > static_cast<int>(b.kind);
      if (a.id != b.id) return a.id > b.id;
      return a.seq > b.seq;
    }
  };
  struct ClientJob {
    RequestId id = 0;
    Ms compute_ms = 0;
    bool partial = false;
  };
  struct Client {
    bool busy = false;
    Ms busy_until = 0;
    std::deque<ClientJob> queue;
    ClientJob current;
    NetworkEstimator estimator;
    Ms backlog(Ms now) const;
  };
  struct Book {
    RequestOutcome outcome;
    std::int64_t size_bits = 0;
    Ms server_arrival = 0;
    int entry_layer = 1;
  };

  void setup();
  void dispatch(const Event& ev);
  void on_generated(const Event& ev);
  void on_client_done(const Event& ev);
  void on_step_complete(const Event& ev);
  void end_of_instant(Ms now);
  void start_step(Ms now);
  void compute_plan(Ms now);
  std::int64_t payload_bits(const ClientDnnProfile& local, int dnn,
                            const std::vector<LayerGroup>& bounds, int k) const;
  void enqueue_client(int client, ClientJob job, Ms now);
  void start_transmission(RequestId id, std::int64_t bits, Ms now, int entry_layer, Ms decompress);
  void send_to_server(RequestId id, Ms now, int entry_layer);
  void arrive_at_server(RequestId id, Ms now);
  Ms server_remaining_makespan(Ms now) const;
  void finish(RequestId id, Ms when);
  void mark_dropped(RequestId id, Ms now);
  StepView view_of(const detail::ExecStep& st, Ms start, Ms end) const;

  Book& book(RequestId id) { return book_[static_cast<std::size_t>(id - 1)]; }
  Request* find_pending(RequestId id);
  void erase_pending(RequestId id);
  void push(Ms t, Kind k, RequestId id) { events_.push(Event{t, k, id, seq_++}); }
  int client_of(RequestId id) const { return static_cast<int>((id - 1) % static_cast<RequestId>(clients_.size())); }

  const WorkloadSpec& spec_;
  const ProfileSet& ps_;
  SimConfig config_;
  const NetworkTrace* trace_;
  const ClientProfile* client_profile_;
  Planner planner_;
  StepHook* hook_ = nullptr;
  SimObserver* obs_ = nullptr;

  std::vector<int> mix_dnn_;
  bool has_shared_ = false;
  std::priority_queue<Event, std::vector<Event>, Later> events_;
  std::uint64_t seq_ = 0;
  std::vector<Book> book_;
  std::vector<Client> clients_;

  std::vector<Request> pending_;  // FIFO order
  Schedule plan_;
  std::vector<detail::ExecStep> steps_;
  std::size_t next_step_ = 0;
  bool executing_ = false;
  Ms busy_until_ = 0;
  Ms step_started_ = 0;
  Ms plan_ready_at_ = 0;
  bool needs_schedule_ = false;
  int arrivals_since_schedule_ = 0;
  int schedules_computed_ = 0;
  double solve_wall_total_ = 0;
};

SimResult run_sim(const WorkloadSpec& spec, const ProfileSet& ps, const SimConfig& config,
                  const NetworkTrace* trace = nullptr, const ClientProfile* client_profile = nullptr);

struct RatePoint {
  double rate = 0;
  SummaryMetrics metrics;
};

struct CapacityCurve {
  std::vector<RatePoint> points;
  std::optional<double> capacity;
};

inline constexpr double kCapacityThreshold = 0.90;

CapacityCurve capacity_sweep(WorkloadSpec spec, const std::vector<double>& rates,
                             const ProfileSet& ps, const SimConfig& config,
                             const NetworkTrace* trace = nullptr,
                             const ClientProfile* client_profile = nullptr);

}  // namespace batchsim
