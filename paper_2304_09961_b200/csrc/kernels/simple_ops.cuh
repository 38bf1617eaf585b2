// Bandwidth-bound NHWC ops on merged batches: max-pool, global average
// pool, depthwise 3x3 conv, softmax. Every image has its own blob base
// pointer (activation-arena slot) plus an element offset, exactly like the
// tensor-core conv. Channels are processed four at a time (float4) so warps
// issue 512-byte coalesced requests along the channel axis.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace bs200 {

struct PoolParams {
  int nimg, H, W, C, Ho, Wo;
  int k, stride, pad;
  const float* const* in_ptrs;
  long in_off;
  int in_ldc;
  float* const* out_ptrs;
  long out_off;
  int out_ldc;
};

struct AvgPoolParams {
  int nimg, HW, C;
  const float* const* in_ptrs;
  long in_off;
  int in_ldc;
  float* const* out_ptrs;
  long out_off;
  int round_out;
};

struct DwParams {
  int nimg, H, W, C, Ho, Wo, stride;  // 3x3, pad 1
  const float* const* in_ptrs;
  long in_off;
  int in_ldc;
  const float* wgt;   // [9][C]
  const float* bias;  // [C]
  float* const* out_ptrs;
  long out_off;
  int out_ldc;
  int relu;  // 0 none, 1 relu, 2 relu6
  int round_out;
};

struct SoftmaxParams {
  int nimg, N;
  const float* const* ptrs;
  long in_off, out_off;
};

// Packed RGB [HW][3] -> padded NHWC [HW][4] (4th channel zero), the request's
// input tensor. Lets clients ship 3 channels over PCIe.
// 8-bit packed RGB [hw][3] -> padded fp32 [hw][4] with value (b - 128) / 32
// (the synthetic images' pixel encoding, csrc/exec/image.hpp).
cudaError_t launch_expand_rgb(const unsigned char* rgb, float* dst, int hw, cudaStream_t s);
// The same for k <= kExpandMax images packed at `stride` bytes in one staging
// region (one launch per batch of small admitted images).
constexpr int kExpandMax = 64;
struct ExpandManyParams {
  const unsigned char* rgb;
  long stride;
  int hw, n;
  float* dst[kExpandMax];
};
cudaError_t launch_expand_rgb_many(const ExpandManyParams& p, cudaStream_t s);
// Fully connected layer at small batch (1x1 conv on a 1x1 input, nimg <=
// kFcMaxImg): weight streaming GEMV, one warp per output column reading its
// weight row once for every image of the batch, fp32 FMA accumulation. At
// b <= 8 the tcgen05 tile is almost empty and the layer is a pure weight
// stream (GoogLeNet's 4 MB, ResNet-50's 8 MB).
constexpr int kFcMaxImg = 8;
struct FcParams {
  int nimg, K, Kpad, N, relu;
  const float* const* in_ptrs;
  long in_off;
  const float* wgt;   // [N][Kpad]
  const float* bias;  // [N] or nullptr
  float* const* out_ptrs;
  long out_off;
};
cudaError_t launch_fc_gemv(const FcParams& p, cudaStream_t s);
cudaError_t launch_maxpool(const PoolParams& p, cudaStream_t s);
cudaError_t launch_avgpool(const AvgPoolParams& p, cudaStream_t s);
cudaError_t launch_dwconv(const DwParams& p, cudaStream_t s);
cudaError_t launch_softmax(const SoftmaxParams& p, cudaStream_t s);
// Result copy-out of up to kGatherMax requests in one launch: request i's
// cnt floats from src[i] to dst[i] (host-mapped pinned memory under UVA), so
// a step's finishing requests cost one kernel instead of one DMA each.
constexpr int kGatherMax = 64;
struct GatherParams {
  const float* src[kGatherMax];
  float* dst[kGatherMax];
  int n, cnt;
};
cudaError_t launch_gather_out(const GatherParams& p, cudaStream_t s);
// A step's pointer table written by a kernel on the serving stream: the
// pointers travel as launch parameters, so no H2D copy and no cross-stream
// event wait sits between two steps' kernels (either one ends the
// programmatic-launch overlap of the previous step's tail with the next
// step's prologue). dst must not be read by work still in flight (the
// executor's chunk ring guarantees it), since the kernel writes before it
// waits on the previous kernel. stamps != null: once every earlier kernel
// of the stream has completed, the global timer (ns) goes to
// stamps[seq % cap] (diagnostics: the previous step's end, no extra launch).
constexpr int kTableWriteMax = 480;
struct TableWriteParams {
  float** dst;
  unsigned long long* stamps;
  unsigned long long seq;
  int cap;
  int n;
  float* src[kTableWriteMax];
};
cudaError_t launch_table_write(float** dst, float* const* src, std::size_t n, cudaStream_t s,
                               unsigned long long* stamps = nullptr, unsigned long long seq = 0, int cap = 1);
// dst[i] = bf16 round-to-nearest-even of src[i] (weight copies for BF16 precision).
cudaError_t launch_to_bf16(const float* src, std::uint16_t* dst, std::size_t n, cudaStream_t s);

}  // namespace bs200
