// Per-SM TMA ingest rate for the conv kernel's box shapes: one CTA per SM,
// one producer thread issuing 16 KB boxes into an S-stage ring, one consumer
// thread releasing stages. Prints GB/s per SM and for the chip.
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a tma_micro.cu -o tma_micro
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

constexpr int kStages = 8;
constexpr int kBox = 16384;

// mode 0: 2D box {32, 128}; mode 1: 4D box {32, 16, 8, 1}; mode 2: 4D box
// {32, 128, 1, 1}; coordinates walk a per-CTA region (hbm) or one shared
// region (l2).
__global__ void tma_kernel(const __grid_constant__ CUtensorMap map, int mode, int iters, int shared_region,
                           long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[kStages], empty[kStages];
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const uint32_t base = ptx::smem_u32(smem);
  const int region = shared_region ? 0 : blockIdx.x;
  if (threadIdx.x == 0) {
    ptx::prefetch_tmap(&map);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int s = it % kStages;
      if (it >= kStages) ptx::mbar_wait(&empty[s], ((it / kStages) - 1) & 1);
      ptx::mbar_arrive_expect_tx(&full[s], kBox);
      const int blk = it % 64;  // 64 distinct boxes per region (1 MB)
      if (mode == 0) ptx::tma_load_2d(base + s * kBox, &map, 0, (region * 64 + blk) * 128, &full[s]);
      else if (mode == 1)
        ptx::tma_load_4d(base + s * kBox, &map, 0, 0, (blk % 8) * 8, region * 8 + blk / 8, &full[s]);
      else ptx::tma_load_4d(base + s * kBox, &map, 0, 0, blk, region, &full[s]);
    }
    ptx::mbar_wait(&full[(iters - 1) % kStages], ((iters - 1) / kStages) & 1);
    cycles[blockIdx.x] = clock64() - t0;
  } else if (threadIdx.x == 32) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % kStages;
      ptx::mbar_wait(&full[s], (it / kStages) & 1);
      ptx::mbar_arrive(&empty[s]);
    }
  }
}

// Cluster multicast: CS CTAs each load 1/CS of every 16 KB box (2D
// {32, 128/CS}) and multicast it to all CS CTAs; every CTA receives the full
// 16 KB per stage. Empty barriers are cluster-wide (count CS).
template <int CS>
__global__ void __cluster_dims__(CS, 1, 1) tma_mc_kernel(const __grid_constant__ CUtensorMap map, int iters,
                                                         long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[kStages], empty[kStages];
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], CS);
    }
    ptx::fence_mbar_init();
  }
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  const uint32_t base = ptx::smem_u32(smem);
  const int cluster = blockIdx.x / CS;
  if (threadIdx.x == 0) {
    ptx::prefetch_tmap(&map);
    const long long t0 = clock64();
    const uint16_t mask = (1u << CS) - 1;
    for (int it = 0; it < iters; ++it) {
      const int s = it % kStages;
      if (it >= kStages) ptx::mbar_wait(&empty[s], ((it / kStages) - 1) & 1);
      ptx::mbar_arrive_expect_tx(&full[s], kBox);
      const int blk = it % 64;
      const uint32_t dst = base + s * kBox + rank * (kBox / CS);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
          " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
          "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"((cluster * 64 + blk) * 128 + rank * (128 / CS)),
          "r"(ptx::smem_u32(&full[s])), "h"(mask)
          : "memory");
    }
    ptx::mbar_wait(&full[(iters - 1) % kStages], ((iters - 1) / kStages) & 1);
    cycles[blockIdx.x] = clock64() - t0;
  } else if (threadIdx.x == 32) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % kStages;
      ptx::mbar_wait(&full[s], (it / kStages) & 1);
      for (int r = 0; r < CS; ++r) {
        uint32_t remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(ptx::smem_u32(&empty[s])), "r"(r));
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
      }
    }
  }
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int CS>
void run_mc(EncodeFn encode, float* d, size_t rows, int sms, long long* cyc) {
  CUtensorMap map;
  cuuint64_t dims[2] = {32, rows};
  cuuint64_t str[1] = {128};
  cuuint32_t box[2] = {32, 128 / CS}, el[2] = {1, 1};
  encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, el, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(tma_mc_kernel<CS>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kBox + 1024);
  const int grid = sms / CS * CS, iters = 2048;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    tma_mc_kernel<CS><<<grid, 64, kStages * kBox + 1024>>>(map, iters, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<long long> h(grid);
    cudaMemcpy(h.data(), cyc, grid * sizeof(long long), cudaMemcpyDeviceToHost);
    double mx = 0;
    for (long long v : h) mx = v > mx ? v : mx;
    const double bytes = static_cast<double>(iters) * kBox;
    if (rep)
      std::printf("multicast CS=%d    grid=%3d: %.1f B/cycle/SM received (%.0f cyc per 16KB stage), chip %.0f GB/s received  err=%s\n",
                  CS, grid, bytes / mx, mx / iters, bytes * grid / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<EncodeFn>(fp);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  // 148 regions x 1 MB (fp32 [rows][32]) = 155 MB > L2.
  const size_t rows = static_cast<size_t>(sms) * 64 * 128;
  float* d = nullptr;
  cudaMalloc(&d, rows * 32 * sizeof(float));
  cudaMemset(d, 0, rows * 32 * sizeof(float));
  long long* cyc = nullptr;
  cudaMalloc(&cyc, sms * sizeof(long long));
  cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kBox + 1024);
  const char* names[3] = {"2D {32,128}", "4D {32,16,8,1}", "4D {32,128,1,1}"};
  for (int mode = 0; mode < 3; ++mode) {
    CUtensorMap map;
    if (mode == 0) {
      cuuint64_t dims[2] = {32, rows};
      cuuint64_t str[1] = {128};
      cuuint32_t box[2] = {32, 128}, el[2] = {1, 1};
      encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, el, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else if (mode == 1) {
      // images of 16 x 64 pixels (1 region = 8 images = 1 MB)
      cuuint64_t dims[4] = {32, 16, 64, static_cast<cuuint64_t>(sms) * 8};
      cuuint64_t str[3] = {128, 16 * 128, 16 * 64 * 128};
      cuuint32_t box[4] = {32, 16, 8, 1}, el[4] = {1, 1, 1, 1};
      encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d, dims, str, box, el, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      cuuint64_t dims[4] = {32, 128, 64, static_cast<cuuint64_t>(sms)};
      cuuint64_t str[3] = {128, 128 * 128, 128 * 128 * 64};
      cuuint32_t box[4] = {32, 128, 1, 1}, el[4] = {1, 1, 1, 1};
      encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d, dims, str, box, el, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    for (int shared = 0; shared < 2; ++shared) {
      for (int grid : {1, sms}) {
        const int iters = 2048;
        tma_kernel<<<grid, 64, kStages * kBox + 1024>>>(map, mode, iters, shared, cyc);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        tma_kernel<<<grid, 64, kStages * kBox + 1024>>>(map, mode, iters, shared, cyc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        std::vector<long long> h(grid);
        cudaMemcpy(h.data(), cyc, grid * sizeof(long long), cudaMemcpyDeviceToHost);
        double mx = 0;
        for (long long v : h) mx = v > mx ? v : mx;
        const double bytes = static_cast<double>(iters) * kBox;
        std::printf("%-16s %s grid=%3d: %.1f B/cycle/SM (%.0f cyc per 16KB box), chip %.0f GB/s  err=%s\n",
                    names[mode], shared ? "L2 " : "HBM", grid, bytes / mx, mx / iters, bytes * grid / (ms * 1e6),
                    cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  run_mc<2>(encode, d, rows, sms, cyc);
  run_mc<4>(encode, d, rows, sms, cyc);
  return 0;
}
