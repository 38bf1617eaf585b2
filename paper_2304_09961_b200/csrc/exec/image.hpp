// Deterministic synthetic images: NHWC fp32 N(0,1), keyed
// by (seed, image index) through SplitMix64 stream kImageStream, zero in the
// padding channels. Host-side so every shard and every checker regenerates
// identical inputs.
#pragma once

#include <cmath>
#include <cstdint>

#include "bsb/core.hpp"

namespace bs200 {

inline void synth_image(std::uint64_t seed, std::uint64_t index, int H, int W, int C, int real_c, float* out) {
  batchsim::SplitMix64 g = batchsim::SplitMix64::stream(seed ^ (index * 0x9E3779B97F4A7C15ULL), 4);
  const long n = static_cast<long>(H) * W;
  for (long p = 0; p < n; ++p) {
    for (int c = 0; c < C; ++c) {
      float v = 0.f;
      if (c < real_c) {
        const double u1 = g.next_double(), u2 = g.next_double();
        v = static_cast<float>(std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(6.283185307179586 * u2));
        // inputs feed a TF32 GEMM: round once here (cvt.rna semantics)
        std::uint32_t u;
        __builtin_memcpy(&u, &v, 4);
        u = (u + 0x1000u) & 0xFFFFE000u;
        __builtin_memcpy(&v, &u, 4);
      }
      out[p * C + c] = v;
    }
  }
}

}  // namespace bs200
