/* C ABI of the B200 batched-layer executor (libbs_exec.so).
 *
 * The reference (batchsim, arXiv 2304.09961) has no executor: a batched step
 * is a cost-table lookup scheduled as a completion event. Each entry point
 * below replaces one point of the reference's serving loop
 * (proj/include/batchsim/simulator.hpp):
 *
 *   bs_admit      arrive_at_server        simulator.hpp:447-465 (request enters the
 *                                         queue at entry_layer; entry_layer > 1 is the
 *                                         collaborative path, :325-371 / :393-419)
 *   bs_plan       compute_plan            simulator.hpp:541-570 (a new plan discards
 *                                         in-progress rides: riders rewind)
 *   bs_step       start_step              simulator.hpp:533-539 (instead of
 *                                         scheduling now + sum_k h_k(b), run layers
 *                                         [from, to] with the batch rule of
 *                                         step_duration, :702-721)
 *   bs_step_done  on_step_complete        simulator.hpp:497-511 (rider deposits)
 *   bs_retire     finish                  simulator.hpp:740-751
 *   bs_drop       drop_expired / tardy    deadline.hpp:21-35, simulator.hpp:611-628
 *   bs_profile_layer / bs_profile_table   the h_k(b) grids of the cost model
 *                                         (cost_model.hpp:22-82, profile_io.hpp:3-18)
 *   bs_replay     run_sim                 simulator.hpp:787-792, every step executed
 *   bs_serve      (new) the same loop on the wall clock
 *
 * Plain C types only; every function returns a status code (BS_OK == 0) and
 * bs_last_error() holds the text of the most recent failure on this thread.
 * Calls on one handle must be serialised by the caller (one host thread per
 * GPU); GPU work is asynchronous on the handle's stream.
 */
#ifndef BS_EXEC_H_
#define BS_EXEC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  BS_OK = 0,
  BS_EINVAL = -1,   /* invalid argument        -> std::invalid_argument */
  BS_ENOMEM = -2,   /* device or arena OOM     -> std::runtime_error    */
  BS_ECUDA = -3,    /* CUDA runtime failure    -> std::runtime_error    */
  BS_EBOUND = -4,   /* step batch > bound      -> std::logic_error      */
  BS_ESTATE = -5    /* unknown request / order -> std::logic_error      */
};

typedef struct bs_handle bs_handle;

/* A segment member: request id and the layer it currently sits at. */
typedef struct bs_member {
  int64_t id;
  int layer;
} bs_member;

/* A foreign request carried through a shared stage (schedule.hpp:24-30). */
typedef struct bs_rider {
  int64_t id;
  int dnn;
  int join_layer;
  int leave_layer;
  int deposit_layer;
} bs_rider;

const char* bs_last_error(void);
void bs_free(char* p);

/* ---------------------------------------------------------------- handle */

/* suite: "small_cnn", "googlenet", "resnet50", "mobilenet_v2",
 * "resnet50_pair", "hetero3", "collab". max_requests = arena slots. */
int bs_create(int device, const char* suite, int max_batch, int max_requests, bs_handle** out);
/* SURVEY.md §8(b) form: also the scheduler window cap (the default "window_cap"
 * of the sim jobs given to bs_replay / bs_serve; 0 = theirs or the
 * reference's 500, simulator.hpp SimConfig::window_cap) and the arithmetic
 * type ("tf32x2" / "tf32" / "bf16", as bs_set_precision; NULL = "tf32x2"). */
int bs_create_ex(int device, const char* suite, int max_batch, int max_requests, int window_cap,
                 const char* dtype, bs_handle** out);
int bs_destroy(bs_handle* h);
/* "tf32x2" (default; split-A 2xTF32 GEMMs, fp32 activations, fp32 parity),
 * "tf32" (one TF32 MMA per K step, TF32-rounded activations) or "bf16"
 * (bf16 operands, fp32 accumulation and activations; reported separately). */
int bs_set_precision(bs_handle* h, const char* mode);
/* JSON: DNNs, layers, ops, tensor plan, weight offsets (for checkers). */
int bs_suite_json(bs_handle* h, char** out_json);
int bs_read_weights(bs_handle* h, float* dst, size_t n);
/* Same description without a device (builds the suite on the host only). */
int bs_describe_suite(const char* suite, char** out_json);
/* The suite's weight pool built on the host (no device). */
int bs_suite_weights_host(const char* suite, float* dst, size_t n);
/* The deterministic synthetic image for (seed, index). */
int bs_make_image(uint64_t seed, uint64_t index, int H, int W, int C, int real_c, float* out);

/* ------------------------------------------------------------- requests */

int bs_admit(bs_handle* h, int64_t id, int dnn, int entry_layer, const float* image_host);
/* Same arrival (entry_layer 1) with the NHWC fp32 input already in device
 * memory: admitted by reference -- no copy; the request's first layer reads
 * the image in place, so it must stay valid and unchanged until that layer
 * has run (e.g. until the request retires). */
int bs_admit_device(bs_handle* h, int64_t id, int dnn, const float* image_device);
/* Arrivals shipped as packed 8-bit RGB [H][W][3] (value (byte - 128) / 32,
 * csrc/exec/image.hpp) in PINNED host memory, for DNNs with a 4-channel padded
 * input: H2D on the handle's admission stream into a staging ring, expanded
 * on the device into the request's input tensor; its first step waits for it.
 * The caller keeps `rgb` unchanged until the copy has run (the next
 * bs_step_ex's done event covers it). */
int bs_admit_rgb(bs_handle* h, int64_t id, int dnn, const uint8_t* rgb_pinned);
/* k arrivals of one DNN at once (any host memory): packed into a pinned staging
 * region, one H2D copy, one expansion launch and one ready event for the
 * batch -- for small images, where per-request copies bound the host loop. */
int bs_admit_rgb_many(bs_handle* h, const int64_t* ids, int dnn, const uint8_t* const* rgb, int k);
int bs_plan(bs_handle* h, int plan_no);
int bs_step(bs_handle* h, int plan_no, int segment, int dnn, int layer_from, int layer_to,
            const bs_member* members, int n_members, const bs_rider* riders, int n_riders);
int bs_step_done(bs_handle* h, const int64_t* deposited, int n);

/* What bs_step_ex launched. done_event is a cudaEvent_t recorded on the
 * handle's stream after the step (owned by the handle, re-recorded by the next
 * bs_step_ex): the on_step_complete signal of simulator.hpp:475-516. */
typedef struct bs_step_result {
  int layers_run;     /* layers with a non-empty batch (step_duration's rule, :705-713) */
  int max_batch;      /* largest per-layer batch of the step */
  int kernels;        /* kernel launches the step issued */
  void* done_event;   /* cudaEvent_t */
} bs_step_result;
/* bs_step with the §8(b) stream and result: `stream` (a cudaStream_t, or
 * NULL) orders the step after the work already enqueued on it, and the
 * stream waits for the step's completion (dependent work can follow on it). */
int bs_step_ex(bs_handle* h, int plan_no, int segment, int dnn, int layer_from, int layer_to,
               const bs_member* members, int n_members, const bs_rider* riders, int n_riders, void* stream,
               bs_step_result* out);
/* Copies the request's class probabilities (or logits) out and frees its slot. */
int bs_retire(bs_handle* h, int64_t id, float* out, int n, int logits);
int bs_drop(bs_handle* h, int64_t id);
int bs_read_blob(bs_handle* h, int64_t id, float* dst, size_t n);
int bs_sync(bs_handle* h);

/* ----------------------------------------------------------- measurement */

int bs_profile_layer(bs_handle* h, int dnn, int layer, int batch, int reps, int flush_l2, double* ms);
/* Layers [from, to] at one batch (scratch blobs), ms per pass: ms3[0] synchronised per pass (host launch
 * latency included), ms3[1] passes queued back to back, ms3[2] one CUDA graph of the pass replayed. */
int bs_profile_span(bs_handle* h, int dnn, int from, int to, int batch, int reps, double* ms3);
/* opts: {"batches": [...], "reps": r, "flush_l2": bool} -> reference-schema profile JSON */
int bs_profile_table(bs_handle* h, const char* opts_json, char** out_json);

/* Sampled per-launch CUDA-event timing (every `every`-th launch). */
int bs_stats(bs_handle* h, int enable, int every);
/* JSON per kernel kind: launches, device ms, algorithmic bytes / FLOPs and
 * the roofline-ideal time at the given HBM GB/s and tensor TFLOP/s. */
int bs_stats_summary(bs_handle* h, double hbm_gbs, double tensor_tflops, char** out_json);

/* ------------------------------------------------------------- serving */

/* Virtual-time run_sim (bit-exact reference schedules) with every step
 * executed; job JSON as bs_host_call's "sim" job plus "image_seed",
 * "image_pool", "dump_ids". Returns JSONL (outcomes, results, summary). */
int bs_replay(bs_handle* h, const char* job_json, char** out_jsonl);
/* Live wall-clock serving of the same job description on the GPU. */
int bs_serve(bs_handle* h, const char* job_json, char** out_json);

/* ---------------------------------------------------------------- kernels */

/* One convolution / FC layer (NHWC, implicit GEMM on tcgen05 TF32). */
typedef struct bs_conv_desc {
  int H, W, Cin;      /* input spatial size, padded channel count (%4 == 0) */
  int Ho, Wo;
  int KH, KW, stride, pad;
  int N;              /* output channels */
  int in_ldc, in_coff;
  int out_ldc, out_coff;
  int res_ldc, res_coff;
  int relu;           /* 0 none, 1 relu, 2 relu6 */
  int round_out;      /* round outputs to TF32 */
  int split;          /* precision: 0 TF32, 1 2xTF32 split-A GEMM, 2 BF16 operands */
} bs_conv_desc;

/* Runs the conv kernel once on host buffers (weights [N][Kpad], Kpad =
 * roundup(KH*KW*Cin, 32)); optionally times `reps` further launches. */
int bs_kernel_conv(const bs_conv_desc* d, int nimg, const float* in_host, const float* w_host,
                   const float* bias_host, const float* res_host, float* out_host, int reps,
                   float* ms_per_launch);

/* Max-pool (k <= 3) on host NHWC buffers; stride_pad = 16 * stride + pad. */
int bs_kernel_maxpool(int nimg, int H, int W, int C, int Ho, int Wo, int k, int stride_pad, const float* in_host,
                      float* out_host);

#ifdef __cplusplus
}
#endif

#endif /* BS_EXEC_H_ */
