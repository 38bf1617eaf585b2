// Per-launch floor of a conv_tc-shaped kernel (608 threads, ~200 KB dynamic
// smem, TMEM 512 columns) when it alternates with a small pool-shaped kernel
// (256 threads, no smem): does the L1/shared carveout switch between them
// cost time, and what does a cluster launch add?
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O2 -o tools/micro/launch_mix_micro tools/micro/launch_mix_micro.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void big_probe(float* out) {
  __shared__ uint32_t slot;
  extern __shared__ float dyn[];
  if (threadIdx.x < 32) {
    uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&slot));
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(dst));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  if (threadIdx.x == 0) dyn[0] = 1.f;
  __syncthreads();
  if (threadIdx.x == 0 && out) out[blockIdx.x] = dyn[0];
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

__global__ void small_probe(float* out) {
  if (threadIdx.x == 0 && out) out[blockIdx.x + 1024] = 2.f;
}

struct Cfg {
  const char* name;
  int big_grid, cluster, small_every, carve;
};

static float run(const Cfg& c, bool graph) {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  float* out;
  cudaMalloc(&out, 1 << 16);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(big_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(small_probe, cudaFuncAttributePreferredSharedMemoryCarveout, c.carve);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(c.big_grid);
  cfg.blockDim = dim3(608);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = c.cluster;
  a[0].val.clusterDim.y = 1;
  a[0].val.clusterDim.z = 1;
  cfg.attrs = a;
  cfg.numAttrs = c.cluster > 1 ? 1 : 0;
  const int n = 200;
  auto body = [&] {
    for (int i = 0; i < n; ++i) {
      cudaLaunchKernelEx(&cfg, big_probe, out);
      if (c.small_every && i % c.small_every == 0) small_probe<<<32, 256, 0, s>>>(out);
    }
  };
  body();
  cudaStreamSynchronize(s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0;
  if (!graph) {
    cudaEventRecord(e0, s);
    body();
    cudaEventRecord(e1, s);
  } else {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    body();
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    cudaEventRecord(e0, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
  }
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  cudaStreamDestroy(s);
  cudaFree(out);
  return ms * 1000 / n;
}

int main() {
  const Cfg cs[] = {
      {"big only grid 8", 8, 1, 0, -1},
      {"big only grid 148", 148, 1, 0, -1},
      {"big grid 8 cluster 4 (grid 32)", 32, 4, 0, -1},
      {"big grid 8 cluster 8 (grid 64)", 64, 8, 0, -1},
      {"big + small each (small carve default)", 8, 1, 1, -1},
      {"big + small each (small carve 100 = max smem)", 8, 1, 1, 100},
      {"big + small each (small carve 0)", 8, 1, 1, 0},
      {"big cluster 4 + small each, carve 100", 32, 4, 1, 100},
  };
  for (const Cfg& c : cs) {
    const float e = run(c, false), g = run(c, true);
    std::printf("%-48s per big launch: eager %6.2f us  graph %6.2f us  (%s)\n", c.name, e, g,
                cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
