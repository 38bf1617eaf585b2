#include <cfloat>
#include <cstdlib>

#include "pdl.cuh"
#include "ptx.cuh"
#include "simple_ops.cuh"

#include <cuda_bf16.h>
#include <algorithm>

namespace bs200 {

namespace {

constexpr int kThreads = 256;

int grid_for(long work) {
  long blocks = (work + kThreads - 1) / kThreads;
  // Grid-stride loops: cap at a few waves of 148 SMs.
  const long cap = 148L * 16;
  return static_cast<int>(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
}

__device__ __forceinline__ float4 max4(float4 a, float4 b) {
  return make_float4(fmaxf(a.x, b.x), fmaxf(a.y, b.y), fmaxf(a.z, b.z), fmaxf(a.w, b.w));
}

// One thread per (image, output pixel, 4 channels); 32-bit index math
// (every pooled tensor of a 90-request batch has < 2^31 float4s).
__global__ void maxpool_kernel(const PoolParams p) {
  pdl::launch_dependents();
  pdl::wait();
  const int C4 = p.C >> 2;
  const int total = p.nimg * p.Ho * p.Wo * C4;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int c4 = i % C4;
    int r = i / C4;
    const int wo = r % p.Wo;
    r /= p.Wo;
    const int ho = r % p.Ho;
    const int n = r / p.Ho;
    const float* in = p.in_ptrs[n] + p.in_off + c4 * 4;
    const int h0 = ho * p.stride - p.pad, w0 = wo * p.stride - p.pad;
    const int hs = max(h0, 0), ws = max(w0, 0);
    const int he = min(h0 + p.k, p.H), we = min(w0 + p.k, p.W);
    float4 m = make_float4(-FLT_MAX, -FLT_MAX, -FLT_MAX, -FLT_MAX);
    for (int h = hs; h < he; ++h)
      for (int w = ws; w < we; ++w) m = max4(m, __ldg(reinterpret_cast<const float4*>(in + (h * p.W + w) * p.in_ldc)));
    *reinterpret_cast<float4*>(p.out_ptrs[n] + p.out_off + (ho * p.Wo + wo) * p.out_ldc + c4 * 4) = m;
  }
}

// k x k max-pool, fully unrolled: one thread per (image, output pixel, 4
// channels), consecutive threads on consecutive channel quads (coalesced
// 16-byte loads/stores); all k*k window loads are independent and predicated
// so they are in flight together.
template <int K>
__global__ void __launch_bounds__(256) maxpool_unrolled_kernel(const PoolParams p) {
  pdl::launch_dependents();
  pdl::wait();
  const int C4 = p.C >> 2;
  const int total = p.nimg * p.Ho * p.Wo * C4;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int c4 = i % C4;
    int r = i / C4;
    const int wo = r % p.Wo;
    r /= p.Wo;
    const int ho = r % p.Ho;
    const int n = r / p.Ho;
    const float* in = p.in_ptrs[n] + p.in_off + c4 * 4;
    const int h0 = ho * p.stride - p.pad, w0 = wo * p.stride - p.pad;
    float4 v[K * K];
#pragma unroll
    for (int kh = 0; kh < K; ++kh)
#pragma unroll
      for (int kw = 0; kw < K; ++kw) {
        const int h = h0 + kh, w = w0 + kw;
        const bool ok = h >= 0 && h < p.H && w >= 0 && w < p.W;
        v[kh * K + kw] = ok ? __ldg(reinterpret_cast<const float4*>(in + (h * p.W + w) * p.in_ldc))
                            : make_float4(-FLT_MAX, -FLT_MAX, -FLT_MAX, -FLT_MAX);
      }
    float4 m = v[0];
#pragma unroll
    for (int j = 1; j < K * K; ++j) m = max4(m, v[j]);
    *reinterpret_cast<float4*>(p.out_ptrs[n] + p.out_off + (ho * p.Wo + wo) * p.out_ldc + c4 * 4) = m;
  }
}

// 3x3 max-pool, 2x2 output block per thread (one channel quad): the
// (S + 3)^2 input window is walked row by row and folded into the four
// running maxima, so a stride-1 pool loads 16 inputs per 4 outputs (9 each
// in the one-output form) and stride 2 loads 25 per 4. Consecutive threads
// take consecutive channel quads (coalesced 16-byte accesses).
template <int S>
__global__ void __launch_bounds__(256) maxpool3_block_kernel(const PoolParams p) {
  pdl::launch_dependents();
  pdl::wait();
  constexpr int IN = S + 3;  // input rows / cols of a 2x2 output block (windows [0,3) and [S,S+3))
  const int C4 = p.C >> 2;
  const int Bw = (p.Wo + 1) >> 1, Bh = (p.Ho + 1) >> 1;
  const int total = p.nimg * Bh * Bw * C4;
  const float4 ninf = make_float4(-FLT_MAX, -FLT_MAX, -FLT_MAX, -FLT_MAX);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int c4 = i % C4;
    int r = i / C4;
    const int bw = r % Bw;
    r /= Bw;
    const int bh = r % Bh;
    const int n = r / Bh;
    const int oh0 = 2 * bh, ow0 = 2 * bw;
    const int h0 = oh0 * S - p.pad, w0 = ow0 * S - p.pad;
    const float* in = p.in_ptrs[n] + p.in_off + c4 * 4;
    float4 m[2][2] = {{ninf, ninf}, {ninf, ninf}};
#pragma unroll
    for (int dy = 0; dy < IN; ++dy) {
      const int h = h0 + dy;
      const bool hok = h >= 0 && h < p.H;
      float4 v[IN];
#pragma unroll
      for (int dx = 0; dx < IN; ++dx) {
        const int w = w0 + dx;
        v[dx] = (hok && w >= 0 && w < p.W) ? __ldg(reinterpret_cast<const float4*>(in + (h * p.W + w) * p.in_ldc))
                                            : ninf;
      }
      // column maxima of the two output columns' windows (cols [0,3), [S, S+3))
      const float4 c0 = max4(max4(v[0], v[1]), v[2]);
      const float4 c1 = max4(max4(v[S], v[S + 1]), v[S + 2]);
      if (dy < 3) {
        m[0][0] = max4(m[0][0], c0);
        m[0][1] = max4(m[0][1], c1);
      }
      if (dy >= S) {
        m[1][0] = max4(m[1][0], c0);
        m[1][1] = max4(m[1][1], c1);
      }
    }
    float* out = p.out_ptrs[n] + p.out_off + c4 * 4;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int oh = oh0 + a, ow = ow0 + b;
        if (oh < p.Ho && ow < p.Wo) *reinterpret_cast<float4*>(out + (oh * p.Wo + ow) * p.out_ldc) = m[a][b];
      }
  }
}

// 3x3 max-pool, BH x BW output tile per thread (one channel quad): each of
// the (BH-1)S+3 input rows is loaded once, folded into the BW column-window
// maxima and those into the output rows whose window covers it. Stride 1 at
// 2x4 loads 3 inputs per output (2x2: 4). Opt-in (BS_POOL_BLOCK=24 / 44):
// measured slower than 2x2 on the GoogLeNet pools at b=90 (stride-1 pool
// time 474 / 505 / 649 us over 3 passes for 2x2 / 2x4 / 4x4) -- the fewer
// threads in flight cost more than the saved L2 reads.
template <int S, int BH, int BW>
__global__ void __launch_bounds__(256) maxpool3_tile_kernel(const PoolParams p) {
  pdl::launch_dependents();
  pdl::wait();
  constexpr int IH = (BH - 1) * S + 3, IW = (BW - 1) * S + 3;
  const int C4 = p.C >> 2;
  const int Bw = (p.Wo + BW - 1) / BW, Bh = (p.Ho + BH - 1) / BH;
  const int total = p.nimg * Bh * Bw * C4;
  const float4 ninf = make_float4(-FLT_MAX, -FLT_MAX, -FLT_MAX, -FLT_MAX);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int c4 = i % C4;
    int r = i / C4;
    const int bw = r % Bw;
    r /= Bw;
    const int bh = r % Bh;
    const int n = r / Bh;
    const int oh0 = BH * bh, ow0 = BW * bw;
    const int h0 = oh0 * S - p.pad, w0 = ow0 * S - p.pad;
    const float* in = p.in_ptrs[n] + p.in_off + c4 * 4;
    float4 m[BH][BW];
#pragma unroll
    for (int a = 0; a < BH; ++a)
#pragma unroll
      for (int b = 0; b < BW; ++b) m[a][b] = ninf;
#pragma unroll
    for (int dy = 0; dy < IH; ++dy) {
      const int h = h0 + dy;
      const bool hok = h >= 0 && h < p.H;
      float4 v[IW];
#pragma unroll
      for (int dx = 0; dx < IW; ++dx) {
        const int w = w0 + dx;
        v[dx] = (hok && w >= 0 && w < p.W) ? __ldg(reinterpret_cast<const float4*>(in + (h * p.W + w) * p.in_ldc))
                                            : ninf;
      }
#pragma unroll
      for (int b = 0; b < BW; ++b) {
        const float4 cm = max4(max4(v[b * S], v[b * S + 1]), v[b * S + 2]);
#pragma unroll
        for (int a = 0; a < BH; ++a)
          if (dy >= a * S && dy < a * S + 3) m[a][b] = max4(m[a][b], cm);
      }
    }
    float* out = p.out_ptrs[n] + p.out_off + c4 * 4;
#pragma unroll
    for (int a = 0; a < BH; ++a)
#pragma unroll
      for (int b = 0; b < BW; ++b) {
        const int oh = oh0 + a, ow = ow0 + b;
        if (oh < p.Ho && ow < p.Wo) *reinterpret_cast<float4*>(out + (oh * p.Wo + ow) * p.out_ldc) = m[a][b];
      }
  }
}

// Row-sliding max-pool (k <= 3): a thread owns one output row of 4 channels
// and walks it left to right; each input column's k-row maximum is computed
// once and kept in a 3-entry ring, so a stride-1 3x3 pool loads every input
// element once per output row (3 loads per output instead of 9) and the
// index math is per row, not per output.
__global__ void maxpool_rows_kernel(const PoolParams p) {
  pdl::launch_dependents();
  pdl::wait();
  const int C4 = p.C >> 2;
  const long total = static_cast<long>(p.nimg) * p.Ho * C4;
  const float4 ninf = make_float4(-FLT_MAX, -FLT_MAX, -FLT_MAX, -FLT_MAX);
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const int c4 = static_cast<int>(i % C4);
    const long r = i / C4;
    const int ho = static_cast<int>(r % p.Ho);
    const int n = static_cast<int>(r / p.Ho);
    const float* in = p.in_ptrs[n] + p.in_off + c4 * 4;
    float* out = p.out_ptrs[n] + p.out_off + static_cast<long>(ho) * p.Wo * p.out_ldc + c4 * 4;
    const int h0 = ho * p.stride - p.pad;
    const int hs = max(h0, 0), he = min(h0 + p.k, p.H);
    float4 ring[3] = {ninf, ninf, ninf};
    int last = -1000000;
    for (int wo = 0; wo < p.Wo; ++wo) {
      const int w0 = wo * p.stride - p.pad;
      const int need = w0 + p.k - 1;
      for (int col = max(last + 1, w0); col <= need; ++col) {
        float4 m = ninf;
        if (col >= 0 && col < p.W)
          for (int h = hs; h < he; ++h)
            m = max4(m, __ldg(reinterpret_cast<const float4*>(in + (static_cast<long>(h) * p.W + col) * p.in_ldc)));
        ring[((col % 3) + 3) % 3] = m;
      }
      last = max(last, need);
      float4 o = ring[((w0 % 3) + 3) % 3];
      for (int kw = 1; kw < p.k; ++kw) o = max4(o, ring[(((w0 + kw) % 3) + 3) % 3]);
      *reinterpret_cast<float4*>(out + static_cast<long>(wo) * p.out_ldc) = o;
    }
  }
}

// One thread per (image, 4 channels); sums the H*W pixels in fp32.
// Global average pool. One CTA per (image, 32 channel quads): the 8 warps
// split the pixels (lane = channel quad, so each pixel row read is 512
// contiguous bytes), then the 8 partial sums are folded in shared memory in
// a fixed order. At small batches this keeps ~8 CTAs per image in flight
// instead of one thread per channel quad walking all pixels serially.
__global__ void avgpool_kernel(const AvgPoolParams p) {
  pdl::launch_dependents();
  pdl::wait();
  __shared__ float4 part[8][32];
  const int C4 = p.C >> 2;
  const int chunks = (C4 + 31) / 32;
  const int n = blockIdx.x / chunks;
  const int c4 = (blockIdx.x - n * chunks) * 32 + (threadIdx.x & 31);
  const int wg = threadIdx.x >> 5;  // pixel group 0..7
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  if (c4 < C4) {
    const float* in = p.in_ptrs[n] + p.in_off + c4 * 4;
#pragma unroll 4
    for (int q = wg; q < p.HW; q += 8) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(in + static_cast<long>(q) * p.in_ldc));
      s.x += v.x;
      s.y += v.y;
      s.z += v.z;
      s.w += v.w;
    }
  }
  part[wg][threadIdx.x & 31] = s;
  __syncthreads();
  if (wg == 0 && c4 < C4) {
    float4 t = part[0][threadIdx.x];
#pragma unroll
    for (int g = 1; g < 8; ++g) {
      const float4 v = part[g][threadIdx.x];
      t.x += v.x;
      t.y += v.y;
      t.z += v.z;
      t.w += v.w;
    }
    const float inv = 1.0f / static_cast<float>(p.HW);
    float4 o = make_float4(t.x * inv, t.y * inv, t.z * inv, t.w * inv);
    if (p.round_out) {
      o.x = ptx::round_tf32(o.x);
      o.y = ptx::round_tf32(o.y);
      o.z = ptx::round_tf32(o.z);
      o.w = ptx::round_tf32(o.w);
    }
    *reinterpret_cast<float4*>(p.out_ptrs[n] + p.out_off + c4 * 4) = o;
  }
}

__device__ __forceinline__ float act(float x, int relu) {
  if (relu == 1) return fmaxf(x, 0.f);
  if (relu == 2) return fminf(fmaxf(x, 0.f), 6.f);
  return x;
}

__global__ void dwconv_kernel(const DwParams p) {
  pdl::launch_dependents();
  pdl::wait();
  const int C4 = p.C >> 2;
  const long total = static_cast<long>(p.nimg) * p.Ho * p.Wo * C4;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const int c4 = static_cast<int>(i % C4);
    long r = i / C4;
    const int wo = static_cast<int>(r % p.Wo);
    r /= p.Wo;
    const int ho = static_cast<int>(r % p.Ho);
    const int n = static_cast<int>(r / p.Ho);
    const float* in = p.in_ptrs[n] + p.in_off + c4 * 4;
    float4 acc = __ldg(reinterpret_cast<const float4*>(p.bias + c4 * 4));
#pragma unroll
    for (int kh = 0; kh < 3; ++kh) {
      const int h = ho * p.stride - 1 + kh;
      if (h < 0 || h >= p.H) continue;
#pragma unroll
      for (int kw = 0; kw < 3; ++kw) {
        const int w = wo * p.stride - 1 + kw;
        if (w < 0 || w >= p.W) continue;
        const float4 v = __ldg(reinterpret_cast<const float4*>(in + (static_cast<long>(h) * p.W + w) * p.in_ldc));
        const float4 k = __ldg(reinterpret_cast<const float4*>(p.wgt + (kh * 3 + kw) * p.C + c4 * 4));
        acc.x = fmaf(v.x, k.x, acc.x);
        acc.y = fmaf(v.y, k.y, acc.y);
        acc.z = fmaf(v.z, k.z, acc.z);
        acc.w = fmaf(v.w, k.w, acc.w);
      }
    }
    acc.x = act(acc.x, p.relu);
    acc.y = act(acc.y, p.relu);
    acc.z = act(acc.z, p.relu);
    acc.w = act(acc.w, p.relu);
    if (p.round_out) {
      acc.x = ptx::round_tf32(acc.x);
      acc.y = ptx::round_tf32(acc.y);
      acc.z = ptx::round_tf32(acc.z);
      acc.w = ptx::round_tf32(acc.w);
    }
    float* out = p.out_ptrs[n] + p.out_off + (static_cast<long>(ho) * p.Wo + wo) * p.out_ldc + c4 * 4;
    *reinterpret_cast<float4*>(out) = acc;
  }
}

// Depthwise 3x3 (pad 1), 2x2 output block per thread and channel quad: the
// (S + 3)^2 input window is loaded once (16 loads per 4 outputs at stride 1,
// 25 at stride 2, against 36) and the nine weight quads once per block.
template <int S>
__global__ void __launch_bounds__(256) dwconv3_block_kernel(const DwParams p) {
  pdl::launch_dependents();
  pdl::wait();
  constexpr int IN = S + 3;
  const int C4 = p.C >> 2;
  const int Bw = (p.Wo + 1) >> 1, Bh = (p.Ho + 1) >> 1;
  const long total = static_cast<long>(p.nimg) * Bh * Bw * C4;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const int c4 = static_cast<int>(i % C4);
    long r = i / C4;
    const int bw = static_cast<int>(r % Bw);
    r /= Bw;
    const int bh = static_cast<int>(r % Bh);
    const int n = static_cast<int>(r / Bh);
    const int oh0 = 2 * bh, ow0 = 2 * bw;
    const int h0 = oh0 * S - 1, w0 = ow0 * S - 1;
    const float* in = p.in_ptrs[n] + p.in_off + c4 * 4;
    float4 k[9];
#pragma unroll
    for (int t = 0; t < 9; ++t) k[t] = __ldg(reinterpret_cast<const float4*>(p.wgt + t * p.C + c4 * 4));
    const float4 b = __ldg(reinterpret_cast<const float4*>(p.bias + c4 * 4));
    float4 acc[2][2] = {{b, b}, {b, b}};
#pragma unroll
    for (int dy = 0; dy < IN; ++dy) {
      const int h = h0 + dy;
      const bool hok = h >= 0 && h < p.H;
#pragma unroll
      for (int dx = 0; dx < IN; ++dx) {
        const int w = w0 + dx;
        if (!(hok && w >= 0 && w < p.W)) continue;
        const float4 v = __ldg(reinterpret_cast<const float4*>(in + (static_cast<long>(h) * p.W + w) * p.in_ldc));
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int kh = dy - a * S, kw = dx - c * S;
            if (kh < 0 || kh > 2 || kw < 0 || kw > 2) continue;  // compile-time after unrolling
            const float4 kk = k[kh * 3 + kw];
            acc[a][c].x = fmaf(v.x, kk.x, acc[a][c].x);
            acc[a][c].y = fmaf(v.y, kk.y, acc[a][c].y);
            acc[a][c].z = fmaf(v.z, kk.z, acc[a][c].z);
            acc[a][c].w = fmaf(v.w, kk.w, acc[a][c].w);
          }
      }
    }
    float* out = p.out_ptrs[n] + p.out_off + c4 * 4;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int oh = oh0 + a, ow = ow0 + c;
        if (oh >= p.Ho || ow >= p.Wo) continue;
        float4 o = acc[a][c];
        o.x = act(o.x, p.relu);
        o.y = act(o.y, p.relu);
        o.z = act(o.z, p.relu);
        o.w = act(o.w, p.relu);
        if (p.round_out) {
          o.x = ptx::round_tf32(o.x);
          o.y = ptx::round_tf32(o.y);
          o.z = ptx::round_tf32(o.z);
          o.w = ptx::round_tf32(o.w);
        }
        *reinterpret_cast<float4*>(out + (static_cast<long>(oh) * p.Wo + ow) * p.out_ldc) = o;
      }
  }
}

// One warp per image: max, sum of exp, normalise.
// Softmax over N classes, one CTA (256 threads) per image: block max and
// block sum through shared memory (fixed reduction order).
__global__ void softmax_kernel(const SoftmaxParams p) {
  pdl::launch_dependents();
  pdl::wait();
  __shared__ float red[8];
  const int n = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float* x = p.ptrs[n] + p.in_off;
  float* y = const_cast<float*>(p.ptrs[n]) + p.out_off;
  float m = -FLT_MAX;
  for (int j = threadIdx.x; j < p.N; j += blockDim.x) m = fmaxf(m, x[j]);
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) red[warp] = m;
  __syncthreads();
  m = red[0];
#pragma unroll
  for (int w = 1; w < 8; ++w) m = fmaxf(m, red[w]);
  __syncthreads();
  float s = 0.f;
  for (int j = threadIdx.x; j < p.N; j += blockDim.x) s += __expf(x[j] - m);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) red[warp] = s;
  __syncthreads();
  s = red[0];
#pragma unroll
  for (int w = 1; w < 8; ++w) s += red[w];
  const float inv = 1.f / s;
  for (int j = threadIdx.x; j < p.N; j += blockDim.x) y[j] = __expf(x[j] - m) * inv;
}

__global__ void gather_out_kernel(const GatherParams p) {
  pdl::launch_dependents();
  pdl::wait();
  const float* src = p.src[blockIdx.x];
  float* dst = p.dst[blockIdx.x];
  for (int j = threadIdx.x; j < p.cnt; j += blockDim.x) dst[j] = src[j];
}

__global__ void table_write_kernel(const __grid_constant__ TableWriteParams p) {
  for (int i = threadIdx.x; i < p.n; i += blockDim.x) p.dst[i] = p.src[i];
  pdl::launch_dependents();
  pdl::wait();  // completes after the previous kernel: keeps the stream's completion order
  if (p.stamps && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.stamps[p.seq % static_cast<unsigned long long>(p.cap)] = t;
  }
}

__global__ void expand_rgb_kernel(const unsigned char* __restrict__ rgb, float* __restrict__ dst, int hw) {
  pdl::launch_dependents();
  pdl::wait();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < hw; i += gridDim.x * blockDim.x) {
    const float r = (static_cast<int>(rgb[3 * i]) - 128) * (1.0f / 32.0f);
    const float g = (static_cast<int>(rgb[3 * i + 1]) - 128) * (1.0f / 32.0f);
    const float b = (static_cast<int>(rgb[3 * i + 2]) - 128) * (1.0f / 32.0f);
    reinterpret_cast<float4*>(dst)[i] = make_float4(r, g, b, 0.f);
  }
}

__global__ void expand_rgb_many_kernel(const ExpandManyParams p) {
  pdl::launch_dependents();
  pdl::wait();
  const unsigned char* __restrict__ rgb = p.rgb + blockIdx.y * p.stride;
  float* __restrict__ dst = p.dst[blockIdx.y];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p.hw; i += gridDim.x * blockDim.x) {
    const float r = (static_cast<int>(rgb[3 * i]) - 128) * (1.0f / 32.0f);
    const float g = (static_cast<int>(rgb[3 * i + 1]) - 128) * (1.0f / 32.0f);
    const float b = (static_cast<int>(rgb[3 * i + 2]) - 128) * (1.0f / 32.0f);
    reinterpret_cast<float4*>(dst)[i] = make_float4(r, g, b, 0.f);
  }
}

__global__ void to_bf16_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst, std::size_t n) {
  for (std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::size_t>(gridDim.x) * blockDim.x)
    dst[i] = __float2bfloat16_rn(src[i]);
}

}  // namespace

cudaError_t launch_to_bf16(const float* src, std::uint16_t* dst, std::size_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const unsigned blocks = static_cast<unsigned>(std::min<std::size_t>((n + 255) / 256, 148 * 16));
  to_bf16_kernel<<<blocks, 256, 0, s>>>(src, reinterpret_cast<__nv_bfloat16*>(dst), n);
  return cudaGetLastError();
}

cudaError_t launch_expand_rgb(const unsigned char* rgb, float* dst, int hw, cudaStream_t s) {
  cudaError_t e = cudaSuccess;
  pdl::suppress_next();  // admission copy stream: after an H2D copy / event wait
  e = pdl::launch(expand_rgb_kernel, dim3(grid_for(hw)), dim3(kThreads), 0, s, rgb, dst, hw);
  return e;
}

cudaError_t launch_expand_rgb_many(const ExpandManyParams& p, cudaStream_t s) {
  if (p.n <= 0) return cudaSuccess;
  if (p.n > kExpandMax) return cudaErrorInvalidValue;
  pdl::suppress_next();  // admission copy stream: after an H2D copy / event wait
  const unsigned bx = static_cast<unsigned>(std::min<long>(grid_for(p.hw), 16));
  return pdl::launch(expand_rgb_many_kernel, dim3(bx, p.n), dim3(kThreads), 0, s, p);
}

namespace {
// One block per output column: its 256 threads split the weight row (K / 256
// float4 each, all loads issued up front, so a whole 4-8 MB matrix is in
// flight at once), per-image partial sums reduced across the block.
__global__ void __launch_bounds__(256) fc_gemv_kernel(const FcParams p) {
  pdl::launch_dependents();
  const int n = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const float* w = p.wgt + static_cast<long>(n) * p.Kpad;
  constexpr int kMaxPer = 4;  // K <= 4096
  float4 wv[kMaxPer];
  // weights are immutable: loaded before waiting for the previous kernel
#pragma unroll
  for (int u = 0; u < kMaxPer; ++u) {
    const int k = (u * 256 + t) * 4;
    wv[u] = k < p.K ? __ldg(reinterpret_cast<const float4*>(w + k)) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  pdl::wait();
  __shared__ float part[8][kFcMaxImg];
#pragma unroll
  for (int m = 0; m < kFcMaxImg; ++m) {
    if (m >= p.nimg) break;
    const float* a = p.in_ptrs[m] + p.in_off;
    float acc = 0.f;
#pragma unroll
    for (int u = 0; u < kMaxPer; ++u) {
      const int k = (u * 256 + t) * 4;
      if (k < p.K) {
        const float4 x = *reinterpret_cast<const float4*>(a + k);
        acc = fmaf(x.x, wv[u].x, acc);
        acc = fmaf(x.y, wv[u].y, acc);
        acc = fmaf(x.z, wv[u].z, acc);
        acc = fmaf(x.w, wv[u].w, acc);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) part[warp][m] = acc;
  }
  __syncthreads();
  if (t < p.nimg) {
    float v = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) v += part[q][t];
    if (p.bias) v += __ldg(p.bias + n);
    if (p.relu == 1) v = fmaxf(v, 0.f);
    else if (p.relu == 2) v = fminf(fmaxf(v, 0.f), 6.f);
    p.out_ptrs[t][p.out_off + n] = v;
  }
}
}  // namespace

cudaError_t launch_fc_gemv(const FcParams& p, cudaStream_t s) {
  if (p.nimg <= 0 || p.nimg > kFcMaxImg || p.K % 4 || p.Kpad % 4 || p.in_off % 4 || p.K > 4096)
    return cudaErrorInvalidValue;
  return pdl::launch(fc_gemv_kernel, dim3(p.N), dim3(256), 0, s, p);
}

cudaError_t launch_maxpool(const PoolParams& p, cudaStream_t s) {
  cudaError_t e = cudaSuccess;
  if (p.C % 4 || p.k > 3) return cudaErrorInvalidValue;
  const long rows = static_cast<long>(p.nimg) * p.Ho * (p.C / 4);
  // The row-sliding form loads each input once per row but serialises a
  // row's outputs; it pays only when rows alone fill the GPU several times.
  const long outs = static_cast<long>(p.nimg) * p.Ho * p.Wo * (p.C / 4);
  if (p.stride == 1 && rows >= 148L * 2048 * 2)
    e = pdl::launch(maxpool_rows_kernel, dim3(grid_for(rows)), dim3(kThreads), 0, s, p);
  else if (p.k == 3 && (p.stride == 1 || p.stride == 2) && !std::getenv("BS_POOL_SIMPLE")) {
    // Output tile per thread (BS_POOL_BLOCK = 22 / 24 / 44 for stride 1).
    const char* be = std::getenv("BS_POOL_BLOCK");  // per launch: tests toggle it
    const int blk = be ? std::atoi(be) : 22;
    const auto tiles = [&](int bh, int bw) {
      return static_cast<long>(p.nimg) * ((p.Ho + bh - 1) / bh) * ((p.Wo + bw - 1) / bw) * (p.C / 4);
    };
    if (p.stride == 1 && blk == 24)
      e = pdl::launch(maxpool3_tile_kernel<1, 2, 4>, dim3(grid_for(tiles(2, 4))), dim3(kThreads), 0, s, p);
    else if (p.stride == 1 && blk == 44)
      e = pdl::launch(maxpool3_tile_kernel<1, 4, 4>, dim3(grid_for(tiles(4, 4))), dim3(kThreads), 0, s, p);
    else if (p.stride == 1)
      e = pdl::launch(maxpool3_block_kernel<1>, dim3(grid_for(tiles(2, 2))), dim3(kThreads), 0, s, p);
    else
      e = pdl::launch(maxpool3_block_kernel<2>, dim3(grid_for(tiles(2, 2))), dim3(kThreads), 0, s, p);
  } else if (p.k == 3)
    e = pdl::launch(maxpool_unrolled_kernel<3>, dim3(grid_for(outs)), dim3(kThreads), 0, s, p);
  else if (p.k == 2)
    e = pdl::launch(maxpool_unrolled_kernel<2>, dim3(grid_for(outs)), dim3(kThreads), 0, s, p);
  else
    e = pdl::launch(maxpool_kernel, dim3(grid_for(outs)), dim3(kThreads), 0, s, p);
  return e;
}

cudaError_t launch_avgpool(const AvgPoolParams& p, cudaStream_t s) {
  cudaError_t e = cudaSuccess;
  if (p.C % 4) return cudaErrorInvalidValue;
  e = pdl::launch(avgpool_kernel, dim3(p.nimg * ((p.C / 4 + 31) / 32)), dim3(256), 0, s, p);
  return e;
}

cudaError_t launch_dwconv(const DwParams& p, cudaStream_t s) {
  cudaError_t e = cudaSuccess;
  if (p.C % 4) return cudaErrorInvalidValue;
  const long blocks = static_cast<long>(p.nimg) * ((p.Ho + 1) / 2) * ((p.Wo + 1) / 2) * (p.C / 4);
  if (p.stride == 1 && !std::getenv("BS_DW_SIMPLE"))
    e = pdl::launch(dwconv3_block_kernel<1>, dim3(grid_for(blocks)), dim3(kThreads), 0, s, p);
  else if (p.stride == 2 && !std::getenv("BS_DW_SIMPLE"))
    e = pdl::launch(dwconv3_block_kernel<2>, dim3(grid_for(blocks)), dim3(kThreads), 0, s, p);
  else
    e = pdl::launch(dwconv_kernel, dim3(grid_for(static_cast<long>(p.nimg) * p.Ho * p.Wo * (p.C / 4))), dim3(kThreads), 0, s, p);
  return e;
}

cudaError_t launch_gather_out(const GatherParams& p, cudaStream_t s) {
  if (p.n <= 0) return cudaSuccess;
  if (p.n > kGatherMax) return cudaErrorInvalidValue;
  return pdl::launch(gather_out_kernel, dim3(p.n), dim3(kThreads), 0, s, p);
}

cudaError_t launch_table_write(float** dst, float* const* src, std::size_t n, cudaStream_t s,
                               unsigned long long* stamps, unsigned long long seq, int cap) {
  for (std::size_t b = 0; b < n; b += kTableWriteMax) {
    TableWriteParams p;
    p.dst = dst + b;
    p.stamps = b == 0 ? stamps : nullptr;
    p.seq = seq;
    p.cap = cap;
    p.n = static_cast<int>(std::min<std::size_t>(kTableWriteMax, n - b));
    for (int i = 0; i < p.n; ++i) p.src[i] = src[b + static_cast<std::size_t>(i)];
    const cudaError_t e = pdl::launch(table_write_kernel, dim3(1), dim3(128), 0, s, p);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_softmax(const SoftmaxParams& p, cudaStream_t s) {
  cudaError_t e = cudaSuccess;
  e = pdl::launch(softmax_kernel, dim3(p.nimg), dim3(256), 0, s, p);
  return e;
}

}  // namespace bs200
