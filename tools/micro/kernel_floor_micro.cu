// Fixed per-launch cost of the conv kernel's launch shape, isolated:
// back-to-back launches of near-empty kernels that add one ingredient of
// conv_tc at a time (608 threads, ~200 KB dynamic smem, a ~1.3 KB
// __grid_constant__ parameter block, TMEM alloc/dealloc of 512 columns,
// a global load of a pointer table), with and without PDL, eager and in a
// CUDA graph.
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O2 -o tools/micro/kernel_floor_micro tools/micro/kernel_floor_micro.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#ifndef PARAM_BYTES
#define PARAM_BYTES 1320
#endif
struct Big {
  unsigned char bytes[PARAM_BYTES];
};

template <int TMEM, int LOADS>
__global__ void k_probe(const __grid_constant__ Big p, float* const* tab, float* out, int use_pdl) {
  __shared__ uint32_t slot;
  if (use_pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (TMEM && threadIdx.x < 32) {
    uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&slot));
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(dst));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  if (use_pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (LOADS && threadIdx.x == 0) {
    float* o = tab[blockIdx.x];
    o[0] = static_cast<float>(p.bytes[blockIdx.x % PARAM_BYTES]);
  }
  __syncthreads();
  if (TMEM && threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
  (void)out;
}

template <int TMEM, int LOADS>
static void run(const char* name, int grid, int threads, int smem, int pdl, float* const* tab) {
  auto k = k_probe<TMEM, LOADS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  Big b{};
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[0].val.programmaticStreamSerializationAllowed = pdl;
  cfg.attrs = a;
  cfg.numAttrs = 1;
  const int n = 200;
  for (int i = 0; i < 20; ++i) cudaLaunchKernelEx(&cfg, k, b, tab, nullptr, pdl);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  for (int i = 0; i < n; ++i) cudaLaunchKernelEx(&cfg, k, b, tab, nullptr, pdl);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  // graph of n launches
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < n; ++i) cudaLaunchKernelEx(&cfg, k, b, tab, nullptr, pdl);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEventRecord(e0, s);
  cudaGraphLaunch(ge, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float gms = 0;
  cudaEventElapsedTime(&gms, e0, e1);
  std::printf("%-44s grid %3d thr %3d smem %6d pdl %d: eager %6.2f us  graph %6.2f us  (%s)\n", name, grid, threads,
              smem, pdl, ms * 1000 / n, gms * 1000 / n, cudaGetErrorString(cudaGetLastError()));
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaStreamDestroy(s);
}

int main() {
  float* buf;
  cudaMalloc(&buf, 1 << 20);
  float** tab;
  cudaMalloc(&tab, 1024 * sizeof(float*));
  float* h[1024];
  for (int i = 0; i < 1024; ++i) h[i] = buf + i * 16;
  cudaMemcpy(tab, h, sizeof(h), cudaMemcpyHostToDevice);
  std::printf("param block %d bytes\n", PARAM_BYTES);
  for (int pdl = 0; pdl < 2; ++pdl) {
    run<0, 0>("plain 128 thr", 8, 128, 0, pdl, tab);
    run<0, 0>("608 thr", 8, 608, 0, pdl, tab);
    run<0, 0>("608 thr + 200KB smem", 8, 608, 200 * 1024, pdl, tab);
    run<1, 0>("608 thr + 200KB smem + TMEM 512", 8, 608, 200 * 1024, pdl, tab);
    run<1, 1>("... + pointer-table load", 8, 608, 200 * 1024, pdl, tab);
    run<1, 1>("... grid 148", 148, 608, 200 * 1024, pdl, tab);
  }
  return 0;
}
