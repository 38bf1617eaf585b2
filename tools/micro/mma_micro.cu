// tcgen05.mma issue/commit cost: same accumulator, 128x128x8 TF32 (and bf16 K=16).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2304_09961_b200/csrc/kernels/ptx.cuh"
using namespace bs200;

template <int N, int MODE, int KIND>
__global__ void k(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (warp == 0) ptx::tmem_alloc<512>(&slot);
  ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t a = ptx::smem_u32(smem), b = a + 16384;
  const uint64_t ad = ptx::sw128_kmajor_desc(a), bd = ptx::sw128_kmajor_desc(b);
  constexpr uint32_t idesc = KIND != 1 ? ptx::make_idesc(2, 128, N) : ptx::make_idesc(1, 128, N);
  long long t0 = 0, t1 = 0;
  if (warp == 0) {
    uint32_t phase = 0;
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (lane == 0) {
        for (int kk = 0; kk < 4; ++kk) {
          if (KIND == 0) ptx::mma_tf32(tmem, ad + 2 * kk, bd + 2 * kk, idesc, (it | kk) != 0);
          else if (KIND == 1) ptx::mma_f16(tmem, ad + 2 * kk, bd + 2 * kk, idesc, (it | kk) != 0);
          else ptx::mma_tf32_ts(tmem, tmem + 256 + 8 * kk, bd + 2 * kk, idesc, (it | kk) != 0);
        }
        if (MODE >= 1) ptx::mma_commit(&bar);
      }
      __syncwarp();
      if (MODE == 2) { ptx::mbar_wait(&bar, phase); phase ^= 1; }
    }
    if (lane == 0 && MODE == 0) ptx::mma_commit(&bar);
    __syncwarp();
    if (MODE == 0) ptx::mbar_wait(&bar, 0);
    if (MODE == 1) { /* wait for the last commit */ ptx::mbar_wait(&bar, (iters - 1) & 1); }
    t1 = clock64();
    if (lane == 0) out[blockIdx.x] = t1 - t0;
  }
  ptx::tc_fence_before(); __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc<512>(tmem); }
}

template <int N, int MODE, int KIND>
void run(const char* name, int iters) {
  long long* d; cudaMalloc(&d, 8 * 148);
  cudaFuncSetAttribute(k<N, MODE, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  k<N, MODE, KIND><<<1, 128, 100 * 1024>>>(d, iters);
  cudaDeviceSynchronize();
  k<N, MODE, KIND><<<1, 128, 100 * 1024>>>(d, iters);
  long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-44s N=%3d: %7.1f cycles per 4-MMA group (%s)\n", name, N, double(h) / iters,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<128, 0, 0>("tf32 4 MMAs/group, one commit at end", 256);
  run<128, 1, 0>("tf32 4 MMAs + commit per group", 256);
  run<128, 2, 0>("tf32 4 MMAs + commit + wait per group", 256);
  run<256, 0, 0>("tf32 4 MMAs/group, one commit at end", 256);
  run<64, 0, 0>("tf32 4 MMAs/group, one commit at end", 256);
  run<128, 0, 1>("bf16 4 MMAs(K=16)/group, one commit", 256);
  run<128, 2, 1>("bf16 4 MMAs + commit + wait per group", 256);
  run<256, 0, 1>("bf16 4 MMAs(K=16)/group, one commit", 256);
  run<128, 0, 2>("tf32 TS (A in TMEM) 4 MMAs/group, one commit", 256);
  run<128, 1, 2>("tf32 TS 4 MMAs + commit per group", 256);
  run<128, 2, 2>("tf32 TS 4 MMAs + commit + wait per group", 256);
  run<64, 0, 2>("tf32 TS (A in TMEM) 4 MMAs/group, one commit", 256);
  return 0;
}
