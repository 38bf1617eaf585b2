// MMA issue loop in the kernel's context: per group wait(already complete) +
// fence + 4 MMAs + commit, with optional spinning warps sharing the SMSPs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2304_09961_b200/csrc/kernels/ptx.cuh"
using namespace bs200;

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
  return pred != 0;
}

template <int SPIN, int ELECT, int WAITFULL>
__global__ void k(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full, empty, never;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { ptx::mbar_init(&full, 1); ptx::mbar_init(&empty, 1); ptx::mbar_init(&never, 1); ptx::fence_mbar_init(); }
  if (warp == 0) ptx::tmem_alloc<256>(&slot);
  ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
  if (threadIdx.x == 0) ptx::mbar_arrive(&full);  // phase 0 complete
  __syncthreads();
  const uint32_t tmem = slot;
  const uint32_t a = ptx::smem_u32(smem), b = a + 16384;
  const uint64_t ad = ptx::sw128_kmajor_desc(a), bd = ptx::sw128_kmajor_desc(b);
  constexpr uint32_t idesc = ptx::make_idesc(2, 128, 128);
  if (warp == 0) {
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (WAITFULL) ptx::mbar_wait(&full, 0);  // already complete
      ptx::tc_fence_after();
      const bool leader = ELECT ? elect_one() : lane == 0;
      if (leader) {
        for (int kk = 0; kk < 4; ++kk) ptx::mma_tf32(tmem, ad + 2 * kk, bd + 2 * kk, idesc, (it | kk) != 0);
        ptx::mma_commit(&empty);
      }
      __syncwarp();
    }
    ptx::mbar_wait(&empty, (iters - 1) & 1);
    long long t1 = clock64();
    if (lane == 0) out[0] = t1 - t0;
    if (lane == 0) ptx::mbar_arrive(&never);  // release spinners
  } else if (SPIN) {
    ptx::mbar_wait(&never, 0);  // spin like the epilogue / splitter warps do
  }
  ptx::tc_fence_before(); __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc<256>(tmem); }
}

template <int SPIN, int ELECT, int WAITFULL>
void run(const char* name, int threads) {
  long long* d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(k<SPIN, ELECT, WAITFULL>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int r = 0; r < 2; ++r) k<SPIN, ELECT, WAITFULL><<<1, threads, 100 * 1024>>>(d, 256);
  cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-52s %7.1f cycles per k-tile (%s)\n", name, double(h) / 256, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<0, 0, 0>("lane0, no wait, alone", 32);
  run<0, 0, 1>("lane0, wait(done) + fence, alone", 32);
  run<0, 1, 1>("elect, wait(done) + fence, alone", 32);
  run<1, 0, 1>("lane0, wait(done) + fence, 13 spinning warps", 448);
  run<1, 1, 1>("elect, wait(done) + fence, 13 spinning warps", 448);
  return 0;
}
