#include <cfloat>

#include "ptx.cuh"
#include "simple_ops.cuh"

namespace bs200 {

namespace {

constexpr int kThreads = 256;

int grid_for(long work) {
  long blocks = (work + kThreads - 1) / kThreads;
  // Grid-stride loops: cap at a few waves of 148 SMs.
  const long cap = 148L * 16;
  return static_cast<int>(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
}

__global__ void maxpool_kernel(const PoolParams p) {
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
    const int h0 = ho * p.stride - p.pad, w0 = wo * p.stride - p.pad;
    const int hs = max(h0, 0), ws = max(w0, 0);
    const int he = min(h0 + p.k, p.H), we = min(w0 + p.k, p.W);
    float4 m = make_float4(-FLT_MAX, -FLT_MAX, -FLT_MAX, -FLT_MAX);
    for (int h = hs; h < he; ++h)
      for (int w = ws; w < we; ++w) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(in + (static_cast<long>(h) * p.W + w) * p.in_ldc));
        m.x = fmaxf(m.x, v.x);
        m.y = fmaxf(m.y, v.y);
        m.z = fmaxf(m.z, v.z);
        m.w = fmaxf(m.w, v.w);
      }
    float* out = p.out_ptrs[n] + p.out_off + (static_cast<long>(ho) * p.Wo + wo) * p.out_ldc + c4 * 4;
    *reinterpret_cast<float4*>(out) = m;
  }
}

// One thread per (image, 4 channels); sums the H*W pixels in fp32.
__global__ void avgpool_kernel(const AvgPoolParams p) {
  const int C4 = p.C >> 2;
  const long total = static_cast<long>(p.nimg) * C4;
  const float inv = 1.0f / static_cast<float>(p.HW);
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const int c4 = static_cast<int>(i % C4);
    const int n = static_cast<int>(i / C4);
    const float* in = p.in_ptrs[n] + p.in_off + c4 * 4;
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int q = 0; q < p.HW; ++q) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(in + static_cast<long>(q) * p.in_ldc));
      s.x += v.x;
      s.y += v.y;
      s.z += v.z;
      s.w += v.w;
    }
    float4 o = make_float4(s.x * inv, s.y * inv, s.z * inv, s.w * inv);
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

// One warp per image: max, sum of exp, normalise.
__global__ void softmax_kernel(const SoftmaxParams p) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= p.nimg) return;
  const float* x = p.ptrs[warp] + p.in_off;
  float* y = const_cast<float*>(p.ptrs[warp]) + p.out_off;
  float m = -FLT_MAX;
  for (int j = lane; j < p.N; j += 32) m = fmaxf(m, x[j]);
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float s = 0.f;
  for (int j = lane; j < p.N; j += 32) s += __expf(x[j] - m);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float inv = 1.f / s;
  for (int j = lane; j < p.N; j += 32) y[j] = __expf(x[j] - m) * inv;
}

}  // namespace

cudaError_t launch_maxpool(const PoolParams& p, cudaStream_t s) {
  if (p.C % 4) return cudaErrorInvalidValue;
  maxpool_kernel<<<grid_for(static_cast<long>(p.nimg) * p.Ho * p.Wo * (p.C / 4)), kThreads, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_avgpool(const AvgPoolParams& p, cudaStream_t s) {
  if (p.C % 4) return cudaErrorInvalidValue;
  avgpool_kernel<<<grid_for(static_cast<long>(p.nimg) * (p.C / 4)), kThreads, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_dwconv(const DwParams& p, cudaStream_t s) {
  if (p.C % 4) return cudaErrorInvalidValue;
  dwconv_kernel<<<grid_for(static_cast<long>(p.nimg) * p.Ho * p.Wo * (p.C / 4)), kThreads, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_softmax(const SoftmaxParams& p, cudaStream_t s) {
  const int blocks = (p.nimg * 32 + kThreads - 1) / kThreads;
  softmax_kernel<<<blocks, kThreads, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace bs200
