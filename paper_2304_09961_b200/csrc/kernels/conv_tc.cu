#include "conv_tc.cuh"

namespace bs200 {

namespace {

template <int BN, int STAGES, bool SPLIT>
cudaError_t launch_bn(const ConvParams& p, cudaStream_t stream) {
  using S = conv_tc::Smem<BN, STAGES, SPLIT>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(conv_tc::conv_tc_kernel<BN, STAGES, SPLIT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, S::kTotal);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int M = p.nimg * p.Ho * p.Wo;
  dim3 grid((M + conv_tc::kBM - 1) / conv_tc::kBM, (p.N + BN - 1) / BN);
  conv_tc::conv_tc_kernel<BN, STAGES, SPLIT><<<grid, S::kThreads, S::kTotal, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace

int conv_tile_n(int N) { return N <= 32 ? 32 : N <= 64 ? 64 : 128; }

namespace {
// The driver entry point is resolved through the runtime, so the library has
// no link-time dependency on libcuda (it loads on hosts without a GPU).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeTiledFn>(nullptr);
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}
}  // namespace

bool encode_weight_map(CUtensorMap* map, const float* w, int N, int Kpad) {
  const EncodeTiledFn encode = encode_fn();
  if (!encode) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(Kpad), static_cast<cuuint64_t>(N)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(Kpad) * sizeof(float)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(conv_tc::kBK), static_cast<cuuint32_t>(conv_tile_n(N))};
  const cuuint32_t elem[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(w), dims, strides, box,
                                elem, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t launch_conv_tc(const ConvParams& p, cudaStream_t stream) {
  if (p.Cin % 4 != 0 || p.Kpad % conv_tc::kBK != 0 || p.Kpad < p.K || p.nimg <= 0)
    return cudaErrorInvalidValue;
  const int bn = conv_tile_n(p.N);
  if (p.split) {
    if (bn == 32) return launch_bn<32, 4, true>(p, stream);
    if (bn == 64) return launch_bn<64, 4, true>(p, stream);
    return launch_bn<128, 4, true>(p, stream);
  }
  if (bn == 32) return launch_bn<32, 4, false>(p, stream);
  if (bn == 64) return launch_bn<64, 4, false>(p, stream);
  return launch_bn<128, 4, false>(p, stream);
}

}  // namespace bs200
