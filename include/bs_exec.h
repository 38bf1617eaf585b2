/* C ABI of the B200 batched-layer executor (libbs_exec.so).
 *
 * The reference (batchsim, arXiv 2304.09961) has no executor: a batched step
 * is a cost-table lookup scheduled as a completion event
 * (proj/include/batchsim/simulator.hpp:533-539 start_step,
 *  :702-721 step_duration, :475-516 on_step_complete).
 * These entry points are what replaces that lookup: the host event loop calls
 * bs_admit where arrive_at_server runs (simulator.hpp:447-465), bs_step where
 * start_step fires, bs_retire where finish runs (simulator.hpp:740-751) and
 * bs_drop where drop_expired / tardy drops resolve a request
 * (simulator.hpp:548-559, :611-628).
 *
 * Plain C types only; every function returns a status code (BS_OK == 0) and
 * bs_last_error() holds the text of the most recent failure on this thread.
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

const char* bs_last_error(void);

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
} bs_conv_desc;

/* Runs the conv kernel once on host buffers (weights [N][Kpad], Kpad =
 * roundup(KH*KW*Cin, 32)); optionally times `reps` further launches. */
int bs_kernel_conv(const bs_conv_desc* d, int nimg, const float* in_host, const float* w_host,
                   const float* bias_host, const float* res_host, float* out_host, int reps,
                   float* ms_per_launch);

#ifdef __cplusplus
}
#endif

#endif /* BS_EXEC_H_ */
