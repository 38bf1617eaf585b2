// Implicit-GEMM convolution / fully-connected layer on the sm_100a tensor
// cores (tcgen05.mma kind::tf32, accumulator in TMEM).
//
//   D[m, n] = sum_k A[m, k] * W[n, k]      m = (image, ho, wo), n = out channel,
//                                          k = (kh, kw, ci) with ci fastest
//
// Mixed TMA / cp.async mainloop:
//   * B (weights, a dense [N][Kpad] matrix) arrives by TMA, one 2D box per
//     stage, 128B-swizzled — one instruction from one thread;
//   * A is never materialised: producer warps gather 16-byte channel chunks of
//     the NHWC input straight into 128B-swizzled shared memory with cp.async
//     (zero-fill = spatial padding and M/K tails). Every image of the merged
//     batch has its own base pointer, so requests stay in their own arena
//     slots: the batch is "gathered" by the loader and "scattered" by the
//     epilogue, with no copy kernels (gather/scatter row).
//     Row addresses are computed once per filter tap (kh, kw); completion is
//     signalled with cp.async.mbarrier.arrive.noinc, so producers never block
//     on their own copies and the ring runs STAGES deep.
//   * 2xTF32 split-A (default precision): the weights are exactly TF32 (they
//     are generated that way), so A*W = A_hi*W + A_lo*W with A_hi = rn_tf32(A)
//     recovers ~fp32 accuracy for two MMAs per K step and no extra HBM bytes.
//     Splitter warps rewrite each landed A stage into [A_hi | A_lo].
//
// Warp roles:
//   warps 0-3   A producers (cp.async gather)
//   warp  4     TMEM allocation; lane 0 issues tcgen05.mma
//   warp  5     lane 0 issues the B TMA loads
//   warps 4-7   epilogue: tcgen05.ld -> bias / residual / ReLU(6) / rounding
//               -> per-image output slot (channel-slice writes = concat)
//   warps 8-11  splitters (2xTF32 only)
#pragma once
#include <cstdint>

#include <cuda.h>

#include "ptx.cuh"

namespace bs200 {

struct ConvParams {
  CUtensorMap wmap;             // weights [N][Kpad] (2D, box {32, BN}, SWIZZLE_128B)
  int nimg;                     // images in the merged batch
  int H, W, Cin;                // input spatial size; Cin = padded channel count (% 4 == 0)
  int Ho, Wo;                   // output spatial size
  int KH, KW, stride, pad;
  int K;                        // KH * KW * Cin
  int Kpad;                     // K rounded up to 32 (row stride of the weights)
  int N;                        // output channels
  const float* const* in_ptrs;  // [nimg] per-request blob base pointers
  long in_off;                  // element offset of (pixel 0, first channel) in the blob
  int in_ldc;                   // floats per pixel
  const float* wgt;             // weights (for the tensor map; also a valid dummy address)
  const float* bias;            // [N] or nullptr
  float* const* out_ptrs;       // [nimg]
  long out_off;
  int out_ldc;
  const float* const* res_ptrs; // [nimg] or nullptr (residual add before ReLU)
  long res_off;
  int res_ldc;
  int relu;                     // 0 none, 1 ReLU, 2 ReLU6
  int round_out;                // round outputs to TF32 (they feed another GEMM)
  int split;                    // 1: 2xTF32 (A = A_hi + A_lo, near-fp32 accuracy)
  unsigned long long* trace;    // debug timeline of CTA (0,0) (nullptr in production)
};

namespace conv_tc {

constexpr int kBM = 128;
constexpr int kBK = 32;  // fp32 elements per 128-byte swizzle row

template <int BN, int STAGES, bool SPLIT>
struct Smem {
  static constexpr int kThreads = SPLIT ? 384 : 256;
  static constexpr int kABytes = kBM * 128;
  static constexpr int kBBytes = BN * 128;
  static constexpr int kStageBytes = kABytes * (SPLIT ? 2 : 1) + kBBytes;  // [A_hi | A_lo | B]
  static constexpr int kBarOffset = STAGES * kStageBytes;
  static constexpr int kTotal = kBarOffset + 512 + 1024;  // barriers + alignment slack
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// trace layout: [0] start, [1] setup done, [2] epilogue start, [3] end,
// [8 + 4 kt + {0: A issued, 1: B issued, 2: MMA got data, 3: split done}]
#define BS_TRACE(slot)                                                         \
  do {                                                                         \
    if (p.trace && blockIdx.x == 0 && blockIdx.y == 0) p.trace[(slot)] = gtime(); \
  } while (0)

__device__ __forceinline__ uint32_t swz(int row, int chunk) {
  return static_cast<uint32_t>(row * 128 + ((chunk ^ (row & 7)) << 4));
}

template <int BN, int STAGES, bool SPLIT>
__global__ void __launch_bounds__(Smem<BN, STAGES, SPLIT>::kThreads, 1)
    conv_tc_kernel(const __grid_constant__ ConvParams p) {
  using S = Smem<BN, STAGES, SPLIT>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* raw_full = reinterpret_cast<uint64_t*>(smem + S::kBarOffset);
  uint64_t* split_full = raw_full + STAGES;
  uint64_t* empty_bar = split_full + STAGES;
  uint64_t* accum_bar = empty_bar + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum_bar + 1);
  uint64_t* mma_full = SPLIT ? split_full : raw_full;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int M = p.nimg * p.Ho * p.Wo;
  const int m_base = blockIdx.x * kBM;
  const int n_base = blockIdx.y * BN;
  const int KT = p.Kpad / kBK;
  const uint32_t smem_base = ptx::smem_u32(smem);
  if (threadIdx.x == 0) BS_TRACE(0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&raw_full[s], 128 + 1);  // 128 cp.async arrivals + the TMA expect_tx
      ptx::mbar_init(&split_full[s], 128);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    ptx::mbar_init(accum_bar, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 5 && lane == 0) ptx::prefetch_tmap(&p.wmap);
  if (warp == 4) ptx::tmem_alloc<BN>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) BS_TRACE(1);

  if (warp < 4) {
    // ------------------------------------------------------------ A gather
    const int t = threadIdx.x;
    const int c = t & 7;    // 16-byte chunk inside the 128-byte K row
    const int r0 = t >> 3;  // rows r0 + 16 i
    const int HoWo = p.Ho * p.Wo;
    const float* row_base[8];
    int row_h[8], row_w[8];
    bool row_ok[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int m = m_base + r0 + 16 * i;
      row_ok[i] = m < M;
      const int mm = row_ok[i] ? m : 0;
      const int n = mm / HoWo;
      const int rem = mm - n * HoWo;
      const int ho = rem / p.Wo;
      const int wo = rem - ho * p.Wo;
      row_h[i] = ho * p.stride - p.pad;
      row_w[i] = wo * p.stride - p.pad;
      row_base[i] = p.in_ptrs[n] + p.in_off;
    }
    const float* dummy = p.wgt;
    auto wait_slot = [&](int kt, int s) {
      if (kt >= STAGES) ptx::mbar_wait(&empty_bar[s], ((kt / STAGES) - 1) & 1);
    };
    if (p.Cin % kBK == 0) {
      // Filter-tap-major walk: row addresses once per (kh, kw), then the
      // channel chunks are consecutive K tiles.
      int kt = 0;
      for (int kh = 0; kh < p.KH; ++kh) {
        for (int kw = 0; kw < p.KW; ++kw) {
          const float* src[8];
          bool ok[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int h = row_h[i] + kh, w = row_w[i] + kw;
            ok[i] = row_ok[i] && h >= 0 && h < p.H && w >= 0 && w < p.W;
            src[i] = ok[i] ? row_base[i] + (static_cast<long>(h) * p.W + w) * p.in_ldc + c * 4 : dummy;
          }
          for (int ci = 0; ci < p.Cin; ci += kBK, ++kt) {
            const int s = kt % STAGES;
            wait_slot(kt, s);
            const uint32_t a_tile = smem_base + s * S::kStageBytes;
#pragma unroll
            for (int i = 0; i < 8; ++i)
              ptx::cp_async16(a_tile + swz(r0 + 16 * i, c), ok[i] ? src[i] + ci : dummy, ok[i] ? 16u : 0u);
            ptx::cp_async_arrive_noinc(&raw_full[s]);
            if (t == 0 && kt < 64) BS_TRACE(8 + 4 * kt);
          }
        }
      }
    } else {
      // Generic K decomposition (stem Cin = 4, narrow 1x1 inputs).
      for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % STAGES;
        wait_slot(kt, s);
        const uint32_t a_tile = smem_base + s * S::kStageBytes;
        const int k0 = kt * kBK + c * 4;
        const bool k_ok = k0 < p.K;
        int ci = 0, kh = 0, kw = 0;
        if (k_ok) {
          const int q = k0 / p.Cin;
          ci = k0 - q * p.Cin;
          kh = q / p.KW;
          kw = q - kh * p.KW;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int h = row_h[i] + kh, w = row_w[i] + kw;
          const bool ok = k_ok && row_ok[i] && h >= 0 && h < p.H && w >= 0 && w < p.W;
          const float* srcp = ok ? row_base[i] + (static_cast<long>(h) * p.W + w) * p.in_ldc + ci : dummy;
          ptx::cp_async16(a_tile + swz(r0 + 16 * i, c), srcp, ok ? 16u : 0u);
        }
        ptx::cp_async_arrive_noinc(&raw_full[s]);
        if (t == 0 && kt < 64) BS_TRACE(8 + 4 * kt);
      }
    }
  } else if (warp >= 8) {
    // --------------------------------------------------- 2xTF32 splitters
    if constexpr (SPLIT) {
      const int t = threadIdx.x - 256;
      const int c = t & 7;
      const int r0 = t >> 3;
      for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % STAGES;
        ptx::mbar_wait(&raw_full[s], (kt / STAGES) & 1);
        const uint32_t a_hi = smem_base + s * S::kStageBytes;
        const uint32_t a_lo = a_hi + S::kABytes;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint32_t o = swz(r0 + 16 * i, c);
          const float4 v = ptx::lds128(a_hi + o);
          const float4 h = make_float4(ptx::round_tf32(v.x), ptx::round_tf32(v.y), ptx::round_tf32(v.z),
                                       ptx::round_tf32(v.w));
          ptx::sts128(a_hi + o, h);
          ptx::sts128(a_lo + o, make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w));
        }
        ptx::fence_proxy_async_smem();
        ptx::mbar_arrive(&split_full[s]);
        if (t == 0 && kt < 64) BS_TRACE(8 + 4 * kt + 3);
      }
    }
  } else {
    if (warp == 4) {
      // ---------------------------------------------------------- MMA issue
      constexpr uint32_t idesc = ptx::make_idesc(2, kBM, BN);
      for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % STAGES;
        ptx::mbar_wait(&mma_full[s], (kt / STAGES) & 1);
        ptx::tc_fence_after();
        if (lane == 0 && kt < 64) BS_TRACE(8 + 4 * kt + 2);
        if (lane == 0) {
          const uint32_t a_tile = smem_base + s * S::kStageBytes;
          const uint32_t b_tile = a_tile + S::kABytes * (SPLIT ? 2 : 1);
          const uint64_t a_desc = ptx::sw128_kmajor_desc(a_tile);
          const uint64_t b_desc = ptx::sw128_kmajor_desc(b_tile);
#pragma unroll
          for (int k = 0; k < kBK / 8; ++k) {
            // +32 bytes per K=8 step inside the swizzled row (>>4 -> +2).
            ptx::mma_tf32(tmem_base, a_desc + 2 * k, b_desc + 2 * k, idesc, (kt | k) != 0);
            if constexpr (SPLIT) {
              const uint64_t lo_desc = ptx::sw128_kmajor_desc(a_tile + S::kABytes);
              ptx::mma_tf32(tmem_base, lo_desc + 2 * k, b_desc + 2 * k, idesc, 1);
            }
          }
          ptx::mma_commit(&empty_bar[s]);
          if (kt == KT - 1) ptx::mma_commit(accum_bar);
        }
        __syncwarp();
      }
    } else if (warp == 5 && lane == 0) {
      // ------------------------------------------------------------ B TMA
      for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % STAGES;
        if (kt >= STAGES) ptx::mbar_wait(&empty_bar[s], ((kt / STAGES) - 1) & 1);
        const uint32_t b_tile = smem_base + s * S::kStageBytes + S::kABytes * (SPLIT ? 2 : 1);
        ptx::mbar_arrive_expect_tx(&raw_full[s], S::kBBytes);
        ptx::tma_load_2d(b_tile, &p.wmap, kt * kBK, n_base, &raw_full[s]);
        if (kt < 64) BS_TRACE(8 + 4 * kt + 1);
      }
    }
    __syncwarp();
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 4;
    const int row = ew * 32 + lane;
    const int m = m_base + row;
    const bool m_ok = m < M;
    int n_img = 0, pix = 0;
    if (m_ok) {
      const int HoWo = p.Ho * p.Wo;
      n_img = m / HoWo;
      pix = m - n_img * HoWo;
    }
    ptx::mbar_wait(accum_bar, 0);
    ptx::tc_fence_after();
    if (warp == 4 && lane == 0) BS_TRACE(2);
    float* out_row = m_ok ? p.out_ptrs[n_img] + p.out_off + static_cast<long>(pix) * p.out_ldc : nullptr;
    const float* res_row =
        (m_ok && p.res_ptrs) ? p.res_ptrs[n_img] + p.res_off + static_cast<long>(pix) * p.res_ldc : nullptr;
#pragma unroll 1
    for (int j = 0; j < BN / 32; ++j) {
      uint32_t v[32];
      ptx::tmem_ld32(tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + j * 32, v);
      ptx::tmem_ld_wait();
      const int n0 = n_base + j * 32;
      if (!m_ok || n0 >= p.N) continue;
      const int ncols = min(32, p.N - n0);
      float o[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        float x = __uint_as_float(v[q]);
        if (q < ncols) {
          if (p.bias) x += __ldg(p.bias + n0 + q);
          if (res_row) x += res_row[n0 + q];
          if (p.relu == 1) x = fmaxf(x, 0.f);
          else if (p.relu == 2) x = fminf(fmaxf(x, 0.f), 6.f);
          if (p.round_out) x = ptx::round_tf32(x);
        }
        o[q] = x;
      }
      float* dst = out_row + n0;
      if (ncols == 32 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
        for (int q = 0; q < 32; q += 4)
          *reinterpret_cast<float4*>(dst + q) = make_float4(o[q], o[q + 1], o[q + 2], o[q + 3]);
      } else {
#pragma unroll
        for (int q = 0; q < 32; ++q)
          if (q < ncols) dst[q] = o[q];
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) BS_TRACE(3);
  if (warp == 4) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<BN>(tmem_base);
  }
}

}  // namespace conv_tc

// N tile the launcher uses for N output channels.
int conv_tile_n(int N);
// Encodes a weight tensor map for w ([N][Kpad] floats) and the tile conv_tile_n(N).
bool encode_weight_map(CUtensorMap* map, const float* w, int N, int Kpad);
// Host-side launcher (p.wmap must be encoded for conv_tile_n(p.N)).
cudaError_t launch_conv_tc(const ConvParams& p, cudaStream_t stream);

}  // namespace bs200
