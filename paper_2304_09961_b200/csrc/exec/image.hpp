// Deterministic synthetic images, keyed by (seed, image
// index) through SplitMix64 stream kImageStream: 8-bit RGB pixels -- a
// N(0,1) draw quantised to k / 32 with k = round(32 x) clamped to
// [-128, 127], stored as the byte k + 128 -- and the network input is their
// exact fp32 value k / 32 (zero in the padding channels; exactly TF32). The
// end-to-end path ships the bytes over PCIe (as decoded images are) and
// expands them on the device to the same values the device-resident path
// uses. Host-side so every shard and every checker regenerates identical
// inputs.
#pragma once

#include <cmath>
#include <cstdint>

#include "bsb/core.hpp"

namespace bs200 {

inline void synth_image_bytes(std::uint64_t seed, std::uint64_t index, int H, int W, int real_c, std::uint8_t* out) {
  batchsim::SplitMix64 g = batchsim::SplitMix64::stream(seed ^ (index * 0x9E3779B97F4A7C15ULL), 4);
  const long n = static_cast<long>(H) * W * real_c;
  for (long i = 0; i < n; ++i) {
    const double u1 = g.next_double(), u2 = g.next_double();
    const double v = std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(6.283185307179586 * u2);
    const long k = std::lround(v * 32.0);
    out[i] = static_cast<std::uint8_t>((k < -128 ? -128 : k > 127 ? 127 : k) + 128);
  }
}

// The fp32 network input of an 8-bit pixel (exact: k / 32).
inline float pixel_value(std::uint8_t b) { return static_cast<float>(static_cast<int>(b) - 128) * (1.0f / 32.0f); }

inline void synth_image(std::uint64_t seed, std::uint64_t index, int H, int W, int C, int real_c, float* out) {
  const long n = static_cast<long>(H) * W;
  std::uint8_t px[16];
  batchsim::SplitMix64 g = batchsim::SplitMix64::stream(seed ^ (index * 0x9E3779B97F4A7C15ULL), 4);
  for (long p = 0; p < n; ++p) {
    // the same draw order as synth_image_bytes (pixel-major, real channels)
    for (int c = 0; c < real_c; ++c) {
      const double u1 = g.next_double(), u2 = g.next_double();
      const double v = std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(6.283185307179586 * u2);
      const long k = std::lround(v * 32.0);
      px[c] = static_cast<std::uint8_t>((k < -128 ? -128 : k > 127 ? 127 : k) + 128);
    }
    for (int c = 0; c < C; ++c) out[p * C + c] = c < real_c ? pixel_value(px[c]) : 0.f;
  }
}

}  // namespace bs200
