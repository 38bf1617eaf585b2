// Launch-overhead microbenchmark: which kernel ingredient costs ~50 us per launch?
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

struct Big { alignas(64) unsigned long long m[16]; int x[64]; };

__global__ void k_empty(int* o) { if (threadIdx.x == 0 && o) o[blockIdx.x] = 1; }
__global__ void k_smem(int* o) {
  extern __shared__ uint8_t s[];
  if (threadIdx.x == 0) { s[0] = 1; if (o) o[blockIdx.x] = s[0]; }
}
template <int COLS>
__global__ void k_tmem(int* o) {
  extern __shared__ uint8_t s[];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(&slot))), "n"(COLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x == 0) { s[0] = 1; if (o) o[blockIdx.x] = s[0] + slot; }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "n"(COLS) : "memory");
}
__global__ void k_big(const __grid_constant__ Big b, int* o) {
  extern __shared__ uint8_t s[];
  if (threadIdx.x == 0) { s[0] = 1; if (o) o[blockIdx.x] = s[0] + b.x[blockIdx.x & 63]; }
}

template <class F>
void timeit(const char* name, F&& launch, int reps = 100) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 5; ++i) launch();
  cudaDeviceSynchronize();
  auto h0 = std::chrono::steady_clock::now();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) launch();
  cudaEventRecord(b);
  auto h1 = std::chrono::steady_clock::now();
  cudaEventSynchronize(b);
  float ms = 0; cudaEventElapsedTime(&ms, a, b);
  double host_us = std::chrono::duration<double, std::micro>(h1 - h0).count() / reps;
  printf("%-40s gpu %8.2f us/launch   host-issue %6.2f us/launch  err=%s\n", name, ms * 1000 / reps, host_us,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int* o; cudaMalloc(&o, 4096 * 4);
  const int big = 194 * 1024;
  cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  cudaFuncSetAttribute(k_tmem<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  cudaFuncSetAttribute(k_tmem<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  cudaFuncSetAttribute(k_big, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  Big bb{};
  for (int grid : {7, 148}) {
    printf("grid %d, 448 threads\n", grid);
    timeit("empty", [&] { k_empty<<<grid, 448>>>(o); });
    timeit("smem 194KB", [&] { k_smem<<<grid, 448, big>>>(o); });
    timeit("smem 48KB", [&] { k_smem<<<grid, 448, 48 * 1024>>>(o); });
    timeit("tmem 256 + smem 194KB", [&] { k_tmem<256><<<grid, 448, big>>>(o); });
    timeit("tmem 32 + smem 8KB", [&] { k_tmem<32><<<grid, 448, 8192>>>(o); });
    timeit("grid_constant 640B + smem 194KB", [&] { k_big<<<grid, 448, big>>>(bb, o); });
    timeit("alternating smem 194KB / empty", [&] { k_smem<<<grid, 448, big>>>(o); k_empty<<<grid, 256>>>(o); }, 50);
  }
  return 0;
}
