// The B200 batched-layer executor.
//
//   * weights: one device pool per suite (TF32-rounded fp32), shared by every
//     DNN that includes a component;
//   * activation arena: one blob per admitted request (slot); a layer runs in
//     place on its members' blobs; riders ride on a copy (ride buffer) that is
//     committed only when the simulator deposits them (simulator.hpp:497-511
//     "riders rewind");
//   * a step = layers [from, to] of one DNN, layer k on {members with
//     layer <= k} U {riders with join <= k <= leave} (simulator.hpp:705-713),
//     all launched asynchronously on one stream; per-layer blob-pointer
//     tables are uploaded once per step.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include <cuda.h>
#include <cuda_runtime.h>

#include "bsb/schedulers.hpp"
#include "netdef.hpp"
#include "../kernels/conv_tc.cuh"

namespace bs200 {

struct LaunchStat {
  OpKind kind;
  int batch;
  double bytes;   // algorithmic
  double flops;
  cudaEvent_t t0, t1;
  bool gemv = false;  // a small-batch FC ran as the weight-streaming GEMV (not conv_tc)
};

struct RideKey {
  std::int64_t id;
  bool operator==(const RideKey& o) const { return id == o.id; }
};

class Executor {
 public:
  Executor(int device, const std::string& suite_name, int max_batch, int max_requests);
  ~Executor();
  Executor(const Executor&) = delete;
  Executor& operator=(const Executor&) = delete;

  const Suite& suite() const { return suite_; }
  cudaStream_t stream() const { return stream_; }
  int max_batch() const { return max_batch_; }

  // ---- request lifecycle
  // image: NHWC [in_H][in_W][in_C] floats, on host (copied H2D) or device.
  void admit(std::int64_t id, int dnn, int entry_layer, const float* image, bool on_device);
  // Packed 8-bit RGB [H][W][3] in pinned host memory (csrc/exec/image.hpp
  // encoding): H2D on the copy stream into a staging ring, expanded to the
  // padded fp32 input tensor on the device; the request's first step waits
  // for it (copies overlap compute).
  void admit_rgb(std::int64_t id, int dnn, const std::uint8_t* rgb_pinned);
  // k images of one DNN admitted together: packed into a pinned staging
  // region on the host, one H2D copy, one expansion launch and one ready event
  // for the batch (for small images, where per-request copies, launches and
  // events bound the host loop).
  // pinned_src: the images are in pinned host memory -- each is DMA'd straight
  // into its staging slot (no host packing; for large images), and the batch
  // still shares one expansion launch and one ready event.
  void admit_rgb_many(const std::int64_t* ids, int dnn, const std::uint8_t* const* rgb, int k, bool pinned_src = false);
  // Device-resident input (e.g. an image pool in HBM) admitted by reference:
  // no copy into the blob and no admission event; the request's first layer
  // reads its input tensor straight from `image` (same NHWC layout), which
  // must stay valid until that layer has run.
  void admit_ref(std::int64_t id, int dnn, const float* image_device);
  void retire(std::int64_t id, float* probs_host, int n, bool logits = false);  // synchronous copy
  void retire_async(std::int64_t id, float* probs_pinned, int n);               // stream-ordered copy + free
  // Batched retire: one copy-out kernel for all ids (pinned, device-mapped
  // destinations), then the slots are freed in stream order.
  void retire_many_async(const std::vector<std::int64_t>& ids, const std::vector<float*>& outs, int n);
  void drop(std::int64_t id);
  bool has(std::int64_t id) const { return slot_of_.count(id) != 0; }
  const float* blob(std::int64_t id) const;
  std::size_t blob_floats() const { return slot_floats_; }
  int free_slots() const { return static_cast<int>(free_.size()); }

  // ---- batched step (async on stream())
  void new_plan(int plan_no);
  void step(int plan_no, int segment, int dnn, int from, int to,
            const std::vector<std::pair<std::int64_t, int>>& members,
            const std::vector<batchsim::Rider>& riders);
  void step_done(const std::vector<std::int64_t>& deposited);
  // Step stamps (diagnostics, table mode 2): step number `step_seq()` of the
  // last step; its table-write kernel stamps the global timer (ns) once
  // every earlier kernel has completed, i.e. the previous step's end.
  // stamps() copies the ring (valid for the last kStampCap steps).
  static constexpr int kStampCap = 1 << 16;
  std::uint64_t step_seq() const { return step_seq_; }
  std::vector<std::uint64_t> stamps();

  // Runs layers [from, to] of `dnn` on an explicit batch of blob pointers
  // (the inner loop of step(); also used by the profiler).
  void run_layer(int dnn, int layer, float* const* d_ptrs, int batch);

  // ---- measurement
  // Median of `reps` CUDA-event timings of one layer at batch b (cold L2 if
  // flush), on scratch blobs.
  double profile_layer(int dnn, int layer, int batch, int reps, bool flush_l2);
  // Per-layer latency inside back-to-back whole-network passes (ms, median
  // over reps): events between the layers of a pass, the stream kept full
  // -- the cost a layer has in a multi-layer serving step, without the
  // launch latency and idle gaps a synchronised single-layer timing adds.
  std::vector<double> profile_pass(int dnn, int batch, int reps);
  // Per-layer latency of one-layer serving steps back to back (ms, median
  // over reps): each step is the pointer-table kernel + the layer, as step()
  // issues it, the last layer followed by the results' copy-out kernel.
  // Timed by the table kernels' device stamps, so nothing between two steps
  // breaks the programmatic-launch overlap a serving step has.
  std::vector<double> profile_steps(int dnn, int batch, int reps);
  // Median time of one whole-network pass at batch b, passes back to back
  // with events only between passes (ms).
  double profile_pass_total(int dnn, int batch, int reps);
  // Layers [from, to] at one batch on scratch blobs, per pass (ms):
  // out[0] = synchronised per pass (launch latency included), out[1] = reps
  // passes queued back to back, out[2] = one CUDA graph of the pass replayed.
  void profile_span(int dnn, int from, int to, int batch, int reps, double out[3]);
  // Sampled launch timing: every `every`-th conv launch (and every other
  // kernel) gets an event pair from a preallocated pool.
  void enable_stats(bool on, int every = 1);
  std::vector<LaunchStat>& stats() { return stats_; }
  void clear_stats();
  long launches() const { return launches_; }

  void sync();

  // "tf32x2" (default): split-A 2xTF32 GEMMs, fp32 activations (fp32 parity);
  // "tf32": one TF32 MMA per K step, activations rounded to TF32;
  // "bf16": bf16 operands (activations rounded to bf16 on their way into
  // TMEM, bf16 copies of the weights), fp32 accumulation and fp32
  // activations in HBM -- the separately reported bf16 path.
  void set_precision(const std::string& mode);
  const char* precision() const { return prec_ == 1 ? "tf32x2" : prec_ == 2 ? "bf16" : "tf32"; }

  // Device-resident synthetic image pool (inputs resident in HBM for the
  // bench); image i of dnn d.
  void make_image_pool(int dnn, int count, std::uint64_t seed);
  const float* pool_image(int dnn, int index) const;
  int pool_size(int dnn) const;

 private:
  struct Slot {
    int index = -1;
    int dnn = 0;
    float* blob = nullptr;
    cudaEvent_t ready = nullptr;  // input copy / client prefix finished (ring-owned)
    bool pending_ready = false;
    // order of its ready event on its admission stream (0 copy_, 1 side_):
    // events on one stream complete in order, so a step waits only on the
    // latest pending one per stream
    long ready_seq = 0;
    int ready_stream = 0;
    const float* image = nullptr;  // admit_ref: the input tensor lives here, not in the blob
  };
  float* slot_ptr(int index) const { return arena_ + static_cast<std::size_t>(index) * slot_floats_; }
  float** table_alloc(std::size_t n, float*** host_view);
  void launch_op(const NetDef& net, const OpDef& op, float* const* d_ptrs, int batch);
  ConvParams conv_params(const NetDef& net, const OpDef& op, float* const* d_ptrs, int batch) const;
  // Ops reading the network's input tensor take their blob bases from this
  // table when set (step(): admit_ref members point at image - input offset).
  float* const* in_override_ = nullptr;
  float* const* input_ptrs(const NetDef& net, const OpDef& op, float* const* d_ptrs) const {
    return in_override_ && op.in.t == net.input_t ? in_override_ : d_ptrs;
  }
  // Two independent convs of one layer in one persistent launch (falls back
  // to two launches when the launcher declines: split-K or wide tiles win).
  void launch_group(const NetDef& net, int layer, int item, const OpDef& a, const OpDef& b, float* const* d_ptrs,
                    int batch);
  void plan_groups();

 public:
  // Profile-time autotune of the conv launch choices, per conv and per
  // batch in `batches`: the K split (1 / 2 / 4 / 8 or the launcher's cost
  // model), 128 x 256 vs 128-wide tiles (N > 128), and for the conv pairs of
  // grouped launches whether one grouped launch beats two separate ones.
  // Each candidate is timed on its whole layer; launches then use the
  // fastest choice of the nearest tuned batch. Returns the timings as JSON.
  std::string tune_tiles(const std::vector<int>& batches, int reps);

 private:
  struct ConvChoice {
    signed char wide = 0;  // 0 launcher rule, 1 128 x 256, 2 128-wide, 3 128 x 192, 4 128 x 160
    signed char ks = 0;    // 0 launcher cost model, else forced K split
  };
  int tuned_index(int batch) const;                              // nearest tuned batch, -1 if none
  std::vector<int> tune_batches_;                                // sorted tuned batch sizes
  std::vector<std::vector<std::vector<ConvChoice>>> conv_pref_;  // [net][op][tuned batch]
  // [net][layer - 1][item][tuned batch]: 0 launcher rule, -1 separate,
  // k >= 1 grouped with a k-way K split
  std::vector<std::vector<std::vector<std::vector<signed char>>>> group_pref_;
  // overrides while tuning
  int tune_net_ = -1, tune_op_ = -1;
  ConvChoice tune_choice_{};
  int tune_layer_ = -1, tune_item_ = -1, tune_group_ = 0;

  Suite suite_;
  int device_ = 0;
  int max_batch_ = 90;
  cudaStream_t stream_ = nullptr;
  cudaStream_t side_ = nullptr;  // client-prefix emulation
  cudaStream_t copy_ = nullptr;  // admissions (H2D / D2D input copies)
  std::vector<cudaEvent_t> ready_ring_;
  std::size_t ready_next_ = 0;
  std::uint8_t* staging_ = nullptr;  // 8-bit RGB staging ring
  std::size_t staging_floats_ = 0;      // bytes per staging slot
  int staging_n_ = 0, staging_next_ = 0;
  std::uint8_t* pack_host_ = nullptr;  // pinned host mirror of the staging ring (batched admissions)
  std::vector<long> pack_seq_;         // per staging slot: batch that last copied from its host region
  std::vector<cudaEvent_t> pack_ev_;   // per batch (ring of 128): its H2D copy is done
  long pack_batches_ = 0, pack_synced_ = 0;
  cudaEvent_t next_ready_event();
  long ready_seq_ = 0;
  // One stream wait per admission stream for the pending members / riders
  // of a step (the latest-admitted one's ready event covers the rest).
  void wait_ready(const std::vector<Slot*>& pending);
  float* d_weights_ = nullptr;
  float* arena_ = nullptr;
  std::size_t slot_floats_ = 0;
  int n_slots_ = 0;
  std::vector<int> free_;
  // Slot release marks: a ring event recorded on stream_ when slots are
  // freed (one per batched retire, shared by its slots) and its sequence
  // number. Frees are ordered on stream_, so an admission stream that has
  // waited on free #S needs no wait for any slot freed at or before S.
  struct FreeMark {
    cudaEvent_t ev = nullptr;
    long seq = 0;  // 0: nothing pending
  };
  std::vector<FreeMark> slot_free_;
  std::vector<cudaEvent_t> free_ring_;
  std::size_t free_next_ = 0;
  long free_seq_ = 0;
  long waited_free_[2] = {0, 0};  // copy_, side_
  FreeMark record_free();
  void release_slot(std::int64_t id, const FreeMark* shared);
  void wait_slot_free(int index, cudaStream_t st);
  std::unordered_map<std::int64_t, Slot> slot_of_;
  // ride buffers: rider id -> ride slot index (valid for the current plan)
  float* ride_arena_ = nullptr;
  int n_ride_ = 0;
  std::vector<int> ride_free_;
  std::unordered_map<std::int64_t, int> ride_of_;
  int ride_plan_ = -1;
  // pointer tables: ring of pinned host + device chunks
  struct TableChunk {
    float** host = nullptr;
    float** dev = nullptr;
    cudaEvent_t done = nullptr;      // recorded on the serving stream after the step
    cudaEvent_t uploaded = nullptr;  // recorded on table_ after the H2D upload
    bool in_use = false;
  };
  unsigned long long* stamps_ = nullptr;  // device, kStampCap entries
  std::uint64_t step_seq_ = 0;
  // How a step's pointer table reaches the device (BS_TABLE_MODE):
  // 2 (default) a table-write kernel on the serving stream with the pointers
  // as launch parameters (keeps the programmatic-launch chain across steps);
  // 1 an H2D copy on its own top-priority stream, the serving stream waiting
  // on its event; 0 an H2D copy on the serving stream.
  cudaStream_t table_ = nullptr;
  int table_mode_ = 2;
  std::vector<TableChunk> chunks_;
  std::size_t chunk_cap_ = 0;
  std::size_t chunk_ = 0;
  std::size_t chunk_used_ = 0;
  // scratch for profiling
  float* scratch_ = nullptr;
  float** scratch_ptrs_ = nullptr;
  float* flush_ = nullptr;
  std::size_t flush_bytes_ = 0;
  // image pools
  std::vector<float*> pool_;
  std::vector<int> pool_n_;
  std::vector<std::vector<CUtensorMap>> wmaps_;  // [net][op] weight tensor maps
  std::vector<std::vector<CUtensorMap>> wmaps_wide_;  // [net][op] 256-row boxes (N > 128)
  std::vector<std::vector<CUtensorMap>> wmaps_mid_;   // [net][op] 192-row boxes (N > 128)
  std::vector<std::vector<CUtensorMap>> wmaps_mid160_;  // [net][op] 160-row boxes (N > 128)
  struct TapRowMap {
    bool ok = false;
    CUtensorMap wmap{};
    CUtensorMap wmap_bf{};  // bf16 copy (BF16 precision)
    std::size_t w_off = 0;  // into d_tap_weights_
  };
  std::vector<std::vector<TapRowMap>> taps_;      // [net][op] tap-row mode (stems)
  // Per layer, the launch order: single ops, or (a, b) conv pairs run as one
  // grouped launch (independent branch convs; BS_CONV_GROUP=0 disables).
  struct LayerItem {
    int a = -1, b = -1;
  };
  std::vector<std::vector<std::vector<LayerItem>>> plans_;  // [net][layer - 1]
  std::vector<std::vector<CUtensorMap>> gmaps_;              // [net][op] weights at the group's tile width
  std::vector<std::vector<CUtensorMap>> gmaps192_;           // [net][op] 192-row boxes for 128 x 192 grouped launches
  std::vector<std::vector<char>> gmap192_ok_;
  std::vector<std::vector<char>> gmap_ok_;
  float* d_tap_weights_ = nullptr;                // (kh, kw < 32 / Cin, ci) copies of the stem weights
  long total_slots_ = 0;
  int prec_ = 1;  // 0 tf32, 1 tf32x2, 2 bf16 (ConvParams::prec)
  // BF16 precision: bf16 copies of the weight pools and their tensor maps
  // (built on the first set_precision("bf16")).
  void build_bf16();
  bool bf16_ready_ = false;
  std::uint16_t* d_weights_bf16_ = nullptr;
  std::uint16_t* d_tap_weights_bf16_ = nullptr;
  std::size_t tap_pool_floats_ = 0;
  std::vector<std::vector<CUtensorMap>> wmaps_bf_, wmaps_wide_bf_, gmaps_bf_;
  bool stats_on_ = false;
  int stats_every_ = 1;
  long stats_seen_ = 0;
  std::size_t ev_next_ = 0;
  std::vector<LaunchStat> stats_;
  std::vector<cudaEvent_t> event_pool_;
  long launches_ = 0;
};

}  // namespace bs200
