// Is the instruction cache cold at every kernel launch? A kernel runs a long
// straight-line block of independent ALU instructions twice and stamps
// %globaltimer around each pass; launched back to back, pass 1 vs pass 2
// shows the fetch cost of code not yet cached.
//   python tools/gen_icache_body.py && nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O2 -o tools/micro/icache_micro tools/micro/icache_micro.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

#include "icache_body.inc"
template <int N>
__global__ void k(unsigned long long* t, unsigned* out) {
  unsigned x = threadIdx.x;
  unsigned long long t0 = gt();
  for (int pass = 0; pass < 3; ++pass) {
    x = body<N>(x);
    __syncwarp();
    if (threadIdx.x == 0 && blockIdx.x == 0) t[pass] = gt() - t0;
    t0 = gt();
  }
  if (x == 0x12345) out[0] = x;
}

template <int N>
void run(unsigned long long* t, unsigned* out) {
  unsigned long long h[3];
  for (int l = 0; l < 4; ++l) {
    k<N><<<1, 32>>>(t, out);
    cudaMemcpy(h, t, sizeof h, cudaMemcpyDeviceToHost);
    std::printf("N=%5d instr (%3d KB) launch %d: pass1 %6llu ns  pass2 %6llu ns  pass3 %6llu ns\n", N, N * 16 / 1024, l,
                h[0], h[1], h[2]);
  }
  // back-to-back without host sync in between
  for (int l = 0; l < 3; ++l) k<N><<<1, 32>>>(t, out);
  cudaMemcpy(h, t, sizeof h, cudaMemcpyDeviceToHost);
  std::printf("N=%5d back-to-back 3rd launch: pass1 %6llu ns  pass2 %6llu ns\n", N, h[0], h[1]);
}

int main() {
  unsigned long long* t;
  unsigned* out;
  cudaMalloc(&t, 64);
  cudaMalloc(&out, 64);
  run<1024>(t, out);
  run<4096>(t, out);
  run<8192>(t, out);
  return 0;
}
