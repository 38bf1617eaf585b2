#include "conv_tc.cuh"

namespace bs200 {

namespace {

template <int BN, int STAGES>
cudaError_t launch_bn(const ConvParams& p, cudaStream_t stream) {
  using S = conv_tc::Smem<BN, STAGES>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(conv_tc::conv_tc_kernel<BN, STAGES>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, S::kTotal);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int M = p.nimg * p.Ho * p.Wo;
  dim3 grid((M + conv_tc::kBM - 1) / conv_tc::kBM, (p.N + BN - 1) / BN);
  conv_tc::conv_tc_kernel<BN, STAGES><<<grid, conv_tc::kThreads, S::kTotal, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_conv_tc(const ConvParams& p, cudaStream_t stream) {
  if (p.Cin % 4 != 0 || p.Kpad % conv_tc::kBK != 0 || p.Kpad < p.K || p.nimg <= 0)
    return cudaErrorInvalidValue;
  if (p.N <= 32) return launch_bn<32, 4>(p, stream);
  if (p.N <= 64) return launch_bn<64, 4>(p, stream);
  return launch_bn<128, 4>(p, stream);
}

}  // namespace bs200
