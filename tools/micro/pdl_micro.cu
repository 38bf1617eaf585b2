// Host cost of a kernel launch with / without programmatic stream
// serialization, and device time of a chain of dependent small kernels.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/micro/pdl_micro tools/micro/pdl_micro.cu
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_small(float* x, int n, int use) {
  if (use) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (use) asm volatile("griddepcontrol.wait;" ::: "memory");
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = x[i] * 0.999f + 1.f;
}

static double run(float* d, int n, int pdl, int launches, cudaStream_t s, cudaEvent_t e0, cudaEvent_t e1,
                  float* dev_ms) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((n + 255) / 256);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[0].val.programmaticStreamSerializationAllowed = pdl;
  cfg.attrs = a;
  cfg.numAttrs = 1;
  cudaStreamSynchronize(s);
  cudaEventRecord(e0, s);
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < launches; ++i) cudaLaunchKernelEx(&cfg, k_small, d, n, pdl);
  auto t1 = std::chrono::steady_clock::now();
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(dev_ms, e0, e1);
  return std::chrono::duration<double, std::micro>(t1 - t0).count() / launches;
}

int main() {
  float* d;
  cudaMalloc(&d, 1 << 24);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1, ev;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  for (int n : {256, 1 << 20}) {
    for (int pdl : {0, 1, 0, 1}) {
      float ms;
      double host_us = run(d, n, pdl, 2000, s, e0, e1, &ms);
      std::printf("n=%8d pdl=%d host %.2f us/launch, device %.2f us/launch\n", n, pdl, host_us, ms * 1000 / 2000);
    }
  }
  // Launch after a cross-stream event wait.
  cudaStream_t s2;
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  for (int pdl : {0, 1, 0, 1}) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a[0].val.programmaticStreamSerializationAllowed = pdl;
    cfg.attrs = a;
    cfg.numAttrs = 1;
    cudaDeviceSynchronize();
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < 500; ++i) {
      cudaEventRecord(ev, s2);
      cudaStreamWaitEvent(s, ev, 0);
      cudaLaunchKernelEx(&cfg, k_small, d, 256, pdl);
      cudaLaunchKernelEx(&cfg, k_small, d, 256, pdl);
    }
    cudaDeviceSynchronize();
    auto t1 = std::chrono::steady_clock::now();
    std::printf("event-wait + 2 launches, pdl=%d: %.2f us per iteration (wall)\n", pdl,
                std::chrono::duration<double, std::micro>(t1 - t0).count() / 500);
  }
  // Host polling of an event recorded after a PDL kernel.
  for (int pdl : {0, 1, 0, 1}) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a[0].val.programmaticStreamSerializationAllowed = pdl;
    cfg.attrs = a;
    cfg.numAttrs = 1;
    cudaDeviceSynchronize();
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < 500; ++i) {
      cudaLaunchKernelEx(&cfg, k_small, d, 256, pdl);
      cudaEventRecord(ev, s);
      while (cudaEventQuery(ev) == cudaErrorNotReady) {
      }
    }
    auto t1 = std::chrono::steady_clock::now();
    std::printf("launch + record + poll, pdl=%d: %.2f us per iteration (wall)\n", pdl,
                std::chrono::duration<double, std::micro>(t1 - t0).count() / 500);
  }
  return 0;
}
