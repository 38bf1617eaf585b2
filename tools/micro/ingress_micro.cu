// Per-SM ingest of the conv kernel's load mix without MMAs: per iteration a
// TMA box of `bbytes` (weights) into an NB ring plus a 16 KB cp.async gather
// (128 threads x 8 x 16 B, 128-byte rows) into an RA ring; one consumer
// thread releases stages. L2-resident sources (every CTA reads the same 4 MB).
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a ingress_micro.cu -o ingress_micro
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#include "../../paper_2304_09961_b200/csrc/kernels/ptx.cuh"
using namespace bs200;

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
constexpr int NB = 4, RA = 4;

__global__ void __launch_bounds__(192, 1) k(const __grid_constant__ CUtensorMap map, const float* asrc, int iters,
                                            int bbytes, int use_a, int use_b, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bf[NB], be[NB], af[RA], ae[RA];
  if (threadIdx.x == 0) {
    for (int s = 0; s < NB; ++s) { ptx::mbar_init(&bf[s], 1); ptx::mbar_init(&be[s], 1); }
    for (int s = 0; s < RA; ++s) { ptx::mbar_init(&af[s], 128); ptx::mbar_init(&ae[s], 1); }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const uint32_t bbase = ptx::smem_u32(smem), abase = bbase + NB * 32768;
  const int warp = threadIdx.x >> 5;
  if (warp < 4) {  // A gather
    if (!use_a) return;
    const int t = threadIdx.x, c = t & 7, r0 = t >> 3;
    for (int it = 0; it < iters; ++it) {
      const int s = it % RA;
      if (it >= RA) ptx::mbar_wait(&ae[s], ((it / RA) - 1) & 1);
      const float* src = asrc + (static_cast<size_t>((blockIdx.x * 37 + it) % 256) * 128) * 32;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        ptx::cp_async16(abase + s * 16384 + (r0 + 16 * i) * 128 + c * 16, src + (r0 + 16 * i) * 32 + c * 4, 16);
      ptx::cp_async_arrive_noinc(&af[s]);
    }
  } else if (warp == 4 && threadIdx.x == 128) {  // B TMA
    if (!use_b) return;
    for (int it = 0; it < iters; ++it) {
      const int s = it % NB;
      if (it >= NB) ptx::mbar_wait(&be[s], ((it / NB) - 1) & 1);
      ptx::mbar_arrive_expect_tx(&bf[s], bbytes);
      ptx::tma_load_2d(bbase + s * 32768, &map, 0, (it % 64) * (bbytes / 128), &bf[s]);
    }
  } else if (threadIdx.x == 160) {  // consumer
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (use_b) { ptx::mbar_wait(&bf[it % NB], (it / NB) & 1); ptx::mbar_arrive(&be[it % NB]); }
      if (use_a) { ptx::mbar_wait(&af[it % RA], (it / RA) & 1); ptx::mbar_arrive(&ae[it % RA]); }
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
  float* d = nullptr;
  const size_t rows = 64 * 256 + 256;
  cudaMalloc(&d, rows * 32 * sizeof(float));
  cudaMemset(d, 0, rows * 32 * sizeof(float));
  long long* cyc = nullptr;
  cudaMalloc(&cyc, sms * sizeof(long long));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, NB * 32768 + RA * 16384 + 1024);
  for (int bb : {16384, 32768}) {
    CUtensorMap map;
    cuuint64_t dims[2] = {32, rows};
    cuuint64_t str[1] = {128};
    cuuint32_t box[2] = {32, static_cast<cuuint32_t>(bb / 128)}, el[2] = {1, 1};
    encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, el, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int mode = 1; mode <= 3; ++mode) {
      const int use_a = mode & 1, use_b = (mode >> 1) & 1, iters = 2048;
      for (int grid : {1, sms}) {
        k<<<grid, 192, NB * 32768 + RA * 16384 + 1024>>>(map, d, iters, bb, use_a, use_b, cyc);
        k<<<grid, 192, NB * 32768 + RA * 16384 + 1024>>>(map, d, iters, bb, use_a, use_b, cyc);
        cudaDeviceSynchronize();
        std::vector<long long> h(grid);
        cudaMemcpy(h.data(), cyc, grid * sizeof(long long), cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (long long v : h) mx = v > mx ? v : mx;
        const double bytes = iters * ((use_a ? 16384.0 : 0) + (use_b ? bb : 0));
        std::printf("B=%5d A=%d B=%d grid=%3d: %6.0f cycles/iter, %.1f B/cycle/SM  (%s)\n", bb, use_a, use_b, grid,
                    double(mx) / iters, bytes / mx, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
