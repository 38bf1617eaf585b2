#include <algorithm>
// Kernel-level C-ABI hooks: run one layer kernel on host buffers. Used by the
// per-kernel parity tests (tests/test_kernels_gpu.py) and by the latency
// profiler; the serving path goes through bs_step instead.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../kernels/conv_tc.cuh"
#include "../kernels/simple_ops.cuh"
#include "bs_exec.h"
#include "errors.hpp"

using bs200::ConvParams;

extern "C" int bs_kernel_conv(const bs_conv_desc* d, int nimg, const float* in_host,
                              const float* w_host, const float* bias_host, const float* res_host,
                              float* out_host, int reps, float* ms_per_launch) {
  using namespace bs200;
  if (!d || nimg <= 0 || !in_host || !w_host || !out_host) return bs_fail(BS_EINVAL, "bs_kernel_conv: null argument");
  const int K = d->KH * d->KW * d->Cin;
  const int Kpad = (K + 31) / 32 * 32;
  const size_t in_img = static_cast<size_t>(d->H) * d->W * d->in_ldc;
  const size_t out_img = static_cast<size_t>(d->Ho) * d->Wo * d->out_ldc;
  const size_t res_img = res_host ? static_cast<size_t>(d->Ho) * d->Wo * d->res_ldc : 0;
  float *dwin = nullptr;
  float *din = nullptr, *dw = nullptr, *db = nullptr, *dout = nullptr, *dres = nullptr;
  float** ptrs = nullptr;
  std::uint16_t* dbf = nullptr;  // bf16 weight copy (d->split == 2)
  CUtensorMap wide;              // 256-row weight box (the launcher keeps a pointer)
  CUtensorMap mid;               // 192-row weight box
  CUtensorMap mid160;            // 160-row weight box
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  int rc = BS_OK;
#define CK(x)                                           \
  do {                                                  \
    cudaError_t _e = (x);                               \
    if (_e != cudaSuccess) {                            \
      rc = bs_fail_cuda(_e, #x);                        \
      goto done;                                        \
    }                                                   \
  } while (0)
  {
    CK(cudaMalloc(&din, in_img * nimg * sizeof(float)));
    CK(cudaMalloc(&dw, static_cast<size_t>(d->N) * Kpad * sizeof(float)));
    CK(cudaMalloc(&dout, out_img * nimg * sizeof(float)));
    if (bias_host) CK(cudaMalloc(&db, d->N * sizeof(float)));
    if (res_host) CK(cudaMalloc(&dres, res_img * nimg * sizeof(float)));
    CK(cudaMalloc(&ptrs, 3 * nimg * sizeof(float*)));
    CK(cudaMemcpy(din, in_host, in_img * nimg * sizeof(float), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dw, w_host, static_cast<size_t>(d->N) * Kpad * sizeof(float), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dout, out_host, out_img * nimg * sizeof(float), cudaMemcpyHostToDevice));
    if (bias_host) CK(cudaMemcpy(db, bias_host, d->N * sizeof(float), cudaMemcpyHostToDevice));
    if (res_host) CK(cudaMemcpy(dres, res_host, res_img * nimg * sizeof(float), cudaMemcpyHostToDevice));
    std::vector<float*> hp(3 * nimg);
    for (int i = 0; i < nimg; ++i) {
      hp[i] = din + in_img * i;
      hp[nimg + i] = dout + out_img * i;
      hp[2 * nimg + i] = dres ? dres + res_img * i : nullptr;
    }
    CK(cudaMemcpy(ptrs, hp.data(), hp.size() * sizeof(float*), cudaMemcpyHostToDevice));
    ConvParams p{};
    p.nimg = nimg;
    p.H = d->H; p.W = d->W; p.Cin = d->Cin; p.Ho = d->Ho; p.Wo = d->Wo;
    p.KH = d->KH; p.KW = d->KW; p.stride = d->stride; p.pad = d->pad;
    p.K = K; p.Kpad = Kpad; p.N = d->N;
    p.in_ptrs = ptrs; p.in_ldc = d->in_ldc; p.in_off = d->in_coff;
    p.wgt = dw; p.bias = db;
    if (!encode_weight_map(&p.wmap, dw, d->N, Kpad)) {
      rc = bs_fail(BS_ECUDA, "cuTensorMapEncodeTiled failed");
      goto done;
    }
    if (d->N > 128) {
      if (!encode_weight_map(&wide, dw, d->N, Kpad, 256)) {
        rc = bs_fail(BS_ECUDA, "cuTensorMapEncodeTiled (wide) failed");
        goto done;
      }
      conv_add_wide_map(p, wide);
      if (!encode_weight_map(&mid, dw, d->N, Kpad, 192)) {
        rc = bs_fail(BS_ECUDA, "cuTensorMapEncodeTiled (mid) failed");
        goto done;
      }
      conv_add_mid_map(p, mid);
      if (!encode_weight_map(&mid160, dw, d->N, Kpad, 160)) {
        rc = bs_fail(BS_ECUDA, "cuTensorMapEncodeTiled (mid160) failed");
        goto done;
      }
      conv_add_mid160_map(p, mid160);
    }
    p.out_ptrs = ptrs + nimg; p.out_ldc = d->out_ldc; p.out_off = d->out_coff;
    p.res_ptrs = dres ? ptrs + 2 * nimg : nullptr; p.res_ldc = d->res_ldc; p.res_off = d->res_coff;
    p.relu = d->relu; p.round_out = d->round_out; p.prec = d->split;
    // test hook: force a K split (the executor's autotune sets ks_force per conv)
    if (const char* ksf = std::getenv("BS_CONV_KS_FORCE")) p.ks_force = std::atoi(ksf);
    {
      if (d->N <= 128 && conv_tap_rows_eligible(d->Cin, d->KW) &&
          !(std::getenv("BS_CONV_TAPROW") && std::getenv("BS_CONV_TAPROW")[0] == '0')) {
        // Tap-row mode (the executor's rule for the stems): re-laid weights.
        std::vector<float> hw(static_cast<size_t>(d->N) * d->KH * 32);
        conv_tap_row_weights(w_host, d->N, Kpad, d->KH, d->KW, d->Cin, hw.data());
        CK(cudaMalloc(&dwin, hw.size() * sizeof(float)));
        CK(cudaMemcpy(dwin, hw.data(), hw.size() * sizeof(float), cudaMemcpyHostToDevice));
        if (!encode_weight_map(&p.wmap, dwin, d->N, d->KH * 32)) {
          rc = bs_fail(BS_ECUDA, "tap-row weight map failed");
          goto done;
        }
        p.tap_rows = 1;
        p.Kpad = d->KH * 32;
        p.wgt = dwin;
      }
    }
    if (d->split == 2) {
      // BF16: the kernel reads a bf16 copy of the (possibly re-laid) weights.
      const int kp = p.tap_rows ? d->KH * 32 : Kpad;
      CK(cudaMalloc(&dbf, static_cast<size_t>(d->N) * kp * 2));
      CK(launch_to_bf16(p.tap_rows ? dwin : dw, dbf, static_cast<size_t>(d->N) * kp, 0));
      if (!encode_weight_map_bf16(&p.wmap, dbf, d->N, kp)) {
        rc = bs_fail(BS_ECUDA, "bf16 weight map failed");
        goto done;
      }
      if (d->N > 128 && !p.tap_rows) {
        if (!encode_weight_map_bf16(&wide, dbf, d->N, kp, 256)) {
          rc = bs_fail(BS_ECUDA, "bf16 weight map (wide) failed");
          goto done;
        }
        conv_add_wide_map(p, wide);
      }
    }
    unsigned long long* trace = nullptr;
    if (std::getenv("BS_CONV_TRACE")) {
      CK(cudaMalloc(&trace, 8 * 3600));
      CK(cudaMemset(trace, 0, 8 * 3600));
      p.trace = trace;
      CK(launch_conv_tc(p, 0));  // warm-up (TMEM/TMA descriptors, L2)
      CK(cudaDeviceSynchronize());
      CK(cudaMemset(trace, 0, 8 * 3600));
    }
    CK(launch_conv_tc(p, 0));
    if (trace && std::getenv("BS_CONV_TRACE")[0] == '2') CK(launch_conv_tc(p, 0));  // trace the 2nd of a pair
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(out_host, dout, out_img * nimg * sizeof(float), cudaMemcpyDeviceToHost));
    if (trace) {
      unsigned long long h[3600];
      CK(cudaMemcpy(h, trace, sizeof h, cudaMemcpyDeviceToHost));
      unsigned long long t0 = ~0ULL;
      for (int b = 0; b < 254; ++b)
        if (h[8 + 4 * b] && h[8 + 4 * b] < t0) t0 = h[8 + 4 * b];
      auto rel = [&](unsigned long long v) { return v ? static_cast<long long>(v - t0) : -1LL; };
      {
        long long smin = 1LL << 60, smax = 0, emin = 1LL << 60, emax = 0;
        int nb = 0;
        for (int b = 0; b < 254 && h[8 + 4 * b]; ++b, ++nb) {
          smin = std::min(smin, rel(h[8 + 4 * b])); smax = std::max(smax, rel(h[8 + 4 * b]));
          emin = std::min(emin, rel(h[11 + 4 * b])); emax = std::max(emax, rel(h[11 + 4 * b]));
        }
        std::fprintf(stderr, "  ctas %d start [%lld, %lld] end [%lld, %lld]\n", nb, smin, smax, emin, emax);
      }
      for (int b = 0; b < 254 && h[8 + 4 * b]; ++b)
        if (b < 2)
          std::fprintf(stderr, "  cta %3d start %7lld setup %7lld firstA %7lld end %7lld\n", b, rel(h[8 + 4 * b]),
                       rel(h[9 + 4 * b]), rel(h[10 + 4 * b]), rel(h[11 + 4 * b]));
      for (int it = 0; it < 48 && h[1024 + it * 5 + 4]; ++it)
        std::fprintf(stderr, "  it %2d A %7lld B %7lld landed %7lld split %7lld mma %7lld | ta_ok %7lld b_ok %7lld\n", it,
                     rel(h[1024 + it * 5]), rel(h[1025 + it * 5]), rel(h[1026 + it * 5]), rel(h[1027 + it * 5]),
                     rel(h[1028 + it * 5]), rel(h[2048 + it * 4]), rel(h[2049 + it * 4]));
      for (int j = 0; j < 32 && h[3072 + j * 8]; ++j)
        std::fprintf(stderr, "  unit %2d epi wait %7lld acc_full %7lld chunks %7lld %7lld %7lld %7lld\n", j,
                     rel(h[3072 + j * 8]), rel(h[3073 + j * 8]), rel(h[3074 + j * 8]), rel(h[3075 + j * 8]),
                     rel(h[3076 + j * 8]), rel(h[3077 + j * 8]));
      for (int c = 0; c < 2 && h[3300 + c * 8]; ++c)
        std::fprintf(stderr, "  epi chunk %d: start %7lld tmem_ld %7lld staged %7lld bias %7lld stored %7lld\n", c,
                     rel(h[3300 + c * 8]), rel(h[3301 + c * 8]), rel(h[3302 + c * 8]), rel(h[3303 + c * 8]),
                     rel(h[3304 + c * 8]));
      for (int j = 0; j < 32 && h[3400 + j * 4]; ++j)
        std::fprintf(stderr, "  producer unit %2d top %7lld ptrs %7lld tap %7lld | b-warp loop entry %7lld\n", j,
                     rel(h[3400 + j * 4]), rel(h[3401 + j * 4]), rel(h[3402 + j * 4]), rel(h[3403]));
      p.trace = nullptr;
      cudaFree(trace);
    }
    if (reps > 0 && ms_per_launch) {
      CK(cudaEventCreate(&e0));
      CK(cudaEventCreate(&e1));
      CK(cudaEventRecord(e0));
      for (int r = 0; r < reps; ++r) CK(launch_conv_tc(p, 0));
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      *ms_per_launch = ms / reps;
    }
  }
#undef CK
done:
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  cudaFree(dbf);
  cudaFree(din); cudaFree(dw); cudaFree(dwin); cudaFree(db); cudaFree(dout); cudaFree(dres); cudaFree(ptrs);
  return rc;
}

// Max-pool on host buffers (stride_pad = 16 * stride + pad), for the kernel tests.
extern "C" int bs_kernel_maxpool(int nimg, int H, int W, int C, int Ho, int Wo, int k, int stride_pad,
                                 const float* in_host, float* out_host) {
  using namespace bs200;
  const std::size_t in_n = static_cast<std::size_t>(nimg) * H * W * C, out_n = static_cast<std::size_t>(nimg) * Ho * Wo * C;
  float *din = nullptr, *dout = nullptr;
  float** ptrs = nullptr;
  int rc = BS_OK;
  std::vector<float*> hp(2 * nimg);
  cudaError_t e = cudaMalloc(&din, in_n * 4);
  if (e == cudaSuccess) e = cudaMalloc(&dout, out_n * 4);
  if (e == cudaSuccess) e = cudaMalloc(&ptrs, 2 * nimg * sizeof(float*));
  if (e == cudaSuccess) e = cudaMemcpy(din, in_host, in_n * 4, cudaMemcpyHostToDevice);
  for (int i = 0; i < nimg; ++i) {
    hp[i] = din + static_cast<std::size_t>(H) * W * C * i;
    hp[nimg + i] = dout + static_cast<std::size_t>(Ho) * Wo * C * i;
  }
  if (e == cudaSuccess) e = cudaMemcpy(ptrs, hp.data(), hp.size() * sizeof(float*), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    PoolParams p{nimg, H, W, C, Ho, Wo, k, stride_pad / 16, stride_pad % 16, ptrs, 0, C, ptrs + nimg, 0, C};
    e = launch_maxpool(p, 0);
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(out_host, dout, out_n * 4, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) rc = bs_fail_cuda(e, "bs_kernel_maxpool");
  cudaFree(din); cudaFree(dout); cudaFree(ptrs);
  return rc;
}
