// A-operand gather paths for the conv kernel, measured without MMAs: per
// iteration 128 rows x 128 B (one K tile of A) land in an 8-stage ring; the
// rows are pixels `stride` bytes apart (NHWC with stride / 4 channels), the
// tile origin moves through a buffer of `mb` MB. 148 CTAs, one per SM.
//   ldgsts : 128 threads x 8 x cp.async 16 B (today's gather)
//   bulk1w : one warp, 4 x cp.async.bulk 128 B per lane
//   bulk4w : four warps, one cp.async.bulk 128 B per thread
//   tma2d  : one 2D TMA box {32 channels, 128 pixels} (best case, contiguous pixels)
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o tools/micro/gather_micro tools/micro/gather_micro.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../../paper_2304_09961_b200/csrc/kernels/ptx.cuh"
using namespace bs200;

constexpr int RA = 8;
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(ptx::smem_u32(bar))
               : "memory");
}

__global__ void __launch_bounds__(192, 1) k(const __grid_constant__ CUtensorMap map, const uint8_t* buf, long npix,
                                            int stride, int iters, int mode, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t af[RA], ae[RA];
  if (threadIdx.x == 0) {
    for (int s = 0; s < RA; ++s) {
      ptx::mbar_init(&af[s], mode == 0 ? 128 : 1);
      ptx::mbar_init(&ae[s], 1);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const uint32_t abase = ptx::smem_u32(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, t = threadIdx.x;
  auto origin = [&](int it) { return (static_cast<long>(blockIdx.x) * 7919 + static_cast<long>(it) * 131) % (npix - 128); };
  if (warp < 4) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % RA;
      if (it >= RA) ptx::mbar_wait(&ae[s], ((it / RA) - 1) & 1);
      const long p0 = origin(it);
      const uint32_t st = abase + s * 16384;
      if (mode == 0) {
        const int c = t & 7, r0 = t >> 3;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          ptx::cp_async16(st + (r0 + 16 * i) * 128 + c * 16, buf + (p0 + r0 + 16 * i) * stride + c * 16, 16);
        ptx::cp_async_arrive_noinc(&af[s]);
      } else if (mode == 1) {
        if (warp == 0) {
          if (lane == 0) ptx::mbar_arrive_expect_tx(&af[s], 16384);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int r = lane + 32 * i;
            bulk_g2s(st + r * 128, buf + (p0 + r) * stride, 128, &af[s]);
          }
        }
      } else if (mode == 2) {
        if (t == 0) ptx::mbar_arrive_expect_tx(&af[s], 16384);
        bulk_g2s(st + t * 128, buf + (p0 + t) * stride, 128, &af[s]);
      } else {
        if (t == 0) {
          ptx::mbar_arrive_expect_tx(&af[s], 16384);
          ptx::tma_load_2d(st, &map, 0, static_cast<int>(p0), &af[s]);
        }
      }
    }
  } else if (threadIdx.x == 128) {
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      ptx::mbar_wait(&af[it % RA], (it / RA) & 1);
      ptx::mbar_arrive(&ae[it % RA]);
    }
    cyc[blockIdx.x] = clock64() - t0;
  }
}

int main() {
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<EncodeFn>(fp);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* cyc = nullptr;
  cudaMalloc(&cyc, sms * sizeof(long long));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, RA * 16384 + 1024);
  const char* names[] = {"ldgsts 8x16B/thread", "bulk 128B, 1 warp", "bulk 128B, 4 warps", "tma2d box 32x128"};
  for (int mb : {32, 512}) {
    for (int stride : {128, 1024}) {
      const long bytes = static_cast<long>(mb) << 20;
      uint8_t* buf = nullptr;
      cudaMalloc(&buf, bytes);
      cudaMemset(buf, 1, bytes);
      const long npix = bytes / stride;
      CUtensorMap map;
      cuuint64_t dims[2] = {32, static_cast<cuuint64_t>(npix)};
      cuuint64_t strides[1] = {static_cast<cuuint64_t>(stride)};
      cuuint32_t box[2] = {32, 128}, el[2] = {1, 1};
      encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, buf, dims, strides, box, el, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      for (int mode = 0; mode < 4; ++mode) {
        const int iters = 2000;
        k<<<sms, 192, RA * 16384 + 1024>>>(map, buf, npix, stride, 50, mode, cyc);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k<<<sms, 192, RA * 16384 + 1024>>>(map, buf, npix, stride, iters, mode, cyc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        long long h[256];
        cudaMemcpy(h, cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < sms; ++i) avg += h[i];
        avg /= sms;
        std::printf("buf %3d MB row stride %4d B  %-22s: %6.1f cyc/K tile  %5.1f B/cyc/SM  chip %6.0f GB/s  (%s)\n", mb,
                    stride, names[mode], avg / iters, 16384.0 * iters / avg, 16384.0 * iters * sms / (ms * 1e6),
                    cudaGetErrorString(cudaGetLastError()));
      }
      cudaFree(buf);
    }
  }
  return 0;
}
