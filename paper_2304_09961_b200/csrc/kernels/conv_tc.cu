#include "conv_tc.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace bs200 {

namespace {

constexpr int kMaxDevices = 64;

int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev < 0 || dev >= kMaxDevices ? 0 : dev;
}

// Per-device caches (a process may drive several GPUs).
int sm_count() {
  static int n[kMaxDevices] = {};
  const int dev = current_device();
  if (!n[dev]) {
    int v = 148;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) v = 148;
    n[dev] = v;
  }
  return n[dev];
}

template <int BN, int PREC, bool GROUP>
cudaError_t launch_bn(const ConvParams& p, const ConvParams& p2, int grid, cudaStream_t stream) {
  using S = conv_tc::Cfg<BN, PREC>;
  static bool configured[kMaxDevices] = {};
  const int dev = current_device();
  if (!configured[dev]) {
    cudaError_t e = cudaFuncSetAttribute(conv_tc::conv_tc_kernel<BN, PREC, GROUP>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, S::kTotal);
    if (e != cudaSuccess) return e;
    configured[dev] = true;
  }
  // Split-K launches are clusters of ksplits CTAs (one per split of a tile).
  const int cluster = p.ksplits > 1 ? p.ksplits : 1;
  conv_tc::ConvArgs<GROUP> args;
  args.a = p;
  if constexpr (GROUP) args.b = p2;
  return pdl::launch_ex(conv_tc::conv_tc_kernel<BN, PREC, GROUP>, dim3(grid), dim3(S::kThreads), S::kTotal, stream,
                        cluster, args);
}

}  // namespace

int conv_tile_n(int N) { return N <= 32 ? 32 : N <= 64 ? 64 : 128; }

namespace {
// 128 x 256 tiles for N > 128. The A path (gather + conversion) costs about
// the same per K tile whatever the tile width, so the wide tile halves it per
// FLOP, but it has a single TMEM accumulator (epilogue not overlapped) and
// half the tiles. Measured on B200 (profiles/r01/layers_b90_bn*.csv): a wide
// K tile costs ~1.8x a narrow one, so wide pays when it cuts the N tiles by
// more than 1.8x, the K loop is long (K >= 512) and the tiles still fill the
// GPU. BS_CONV_BN256=0 disables, =2 forces (when a wide weight map exists).
bool use_wide(const ConvParams& p, int sms) {
  const char* env = std::getenv("BS_CONV_BN256");  // read per launch (tests toggle it)
  if (!p.wmap_wide || (env && env[0] == '0')) return false;
  if (env && env[0] == '2') return true;
  if (p.wide_pref == 1) return true;
  if (p.wide_pref == 2) return false;
  const int narrow = (p.N + 127) / 128, wide = (p.N + 255) / 256;
  return p.N > 128 && p.K >= 512 && wide * 1.8 < narrow && p.m_tiles * wide * 10 >= sms * 9;
}
}  // namespace

void conv_add_wide_map(ConvParams& p, const CUtensorMap& wide) { p.wmap_wide = &wide; }
void conv_add_mid_map(ConvParams& p, const CUtensorMap& mid) { p.wmap_mid = &mid; }
void conv_add_mid160_map(ConvParams& p, const CUtensorMap& mid160) { p.wmap_mid160 = &mid160; }

namespace {
// 128 x 192 tiles (two TMEM accumulators, 2xTF32 / TF32 only): the tuned
// choice (wide_pref 3), else by rule when 192 divides N and 128 does not
// (N = 192: one exact tile instead of 25% padding at 256 or 128 + 64).
// BS_CONV_BN192=0 never, =2 always (when a 192-row map exists).
bool use_mid(const ConvParams& p) {
  const char* env = std::getenv("BS_CONV_BN192");  // read per launch (tests toggle it)
  if (!p.wmap_mid || p.prec == 2 || (env && env[0] == '0')) return false;
  if (env && env[0] == '2') return true;
  if (p.wide_pref) return p.wide_pref == 3;
  return p.N > 128 && p.N % 192 == 0 && p.N % 128 != 0;
}
// 128 x 160 tiles: tuned (wide_pref 4), else when 160 divides N and neither
// 128 nor 192 does (N = 160, 320, 480). BS_CONV_BN160=0 never, =2 always.
bool use_mid160(const ConvParams& p) {
  const char* env = std::getenv("BS_CONV_BN160");
  if (!p.wmap_mid160 || p.prec == 2 || (env && env[0] == '0')) return false;
  if (env && env[0] == '2') return true;
  if (p.wide_pref) return p.wide_pref == 4;
  return p.N > 128 && p.N % 160 == 0 && p.N % 128 != 0 && p.N % 192 != 0;
}
}  // namespace

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

bool encode_weight_map(CUtensorMap* map, const float* w, int N, int Kpad, int box_n) {
  const EncodeTiledFn encode = encode_fn();
  if (!encode) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(Kpad), static_cast<cuuint64_t>(N)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(Kpad) * sizeof(float)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(conv_tc::kBK),
                             static_cast<cuuint32_t>(box_n > 0 ? box_n : conv_tile_n(N))};
  const cuuint32_t elem[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(w), dims, strides, box,
                                elem, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool encode_weight_map_bf16(CUtensorMap* map, const void* w, int N, int Kpad, int box_n) {
  const EncodeTiledFn encode = encode_fn();
  if (!encode) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(Kpad), static_cast<cuuint64_t>(N)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(Kpad) * 2};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(conv_tc::kBK),
                             static_cast<cuuint32_t>(box_n > 0 ? box_n : conv_tile_n(N))};
  const cuuint32_t elem[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(w), dims, strides, box, elem,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool conv_tap_rows_eligible(int Cin, int KW) {
  if (Cin != 4 && Cin != 8 && Cin != 16) return false;
  const int taps = conv_tc::kBK / Cin;
  return KW <= taps && KW + 1 >= taps;
}

void conv_tap_row_weights(const float* w, int N, int Kpad_src, int KH, int KW, int Cin, float* out) {
  const int taps = conv_tc::kBK / Cin;
  for (int n = 0; n < N; ++n) {
    float* o = out + static_cast<std::size_t>(n) * KH * conv_tc::kBK;
    const float* src = w + static_cast<std::size_t>(n) * Kpad_src;
    for (int kh = 0; kh < KH; ++kh)
      for (int kw = 0; kw < taps; ++kw)
        for (int ci = 0; ci < Cin; ++ci)
          o[(kh * taps + kw) * Cin + ci] = kw < KW ? src[(kh * KW + kw) * Cin + ci] : 0.f;
  }
}

namespace {
// Split-K cost model. The splits of a tile are one thread-block cluster
// (<= 8 CTAs, the portable cluster size) whose partial tiles are reduced over
// DSMEM at the end of the kernel; a split unit costs its K tiles plus a fixed
// overhead (partial tile into shared memory, two cluster barriers, the
// reduction of 128 / ks rows from ks peers), in K-tile units (BS_CONV_KS_OVH,
// default fitted on the GoogLeNet / ResNet-50 layer sums at small batches;
// BS_CONV_KS_MAX caps the split). Splits only when the tiles cannot cover the
// SMs, one unit per CTA.
int choose_ksplits(int tiles, int KT, int sms) {
  int ks = 1;
  static const int ks_max = std::min(8, std::getenv("BS_CONV_KS_MAX") ? std::atoi(std::getenv("BS_CONV_KS_MAX")) : 8);
  static const int ks_ovh = std::getenv("BS_CONV_KS_OVH") ? std::atoi(std::getenv("BS_CONV_KS_OVH")) : 16;
  if (tiles < sms) {
    auto cost = [&](int k) {
      const int per = (KT + k - 1) / k;
      const int units = tiles * k;
      const int waves = (units + sms - 1) / sms;
      return waves * (per + (k > 1 ? ks_ovh : 0));
    };
    int best = cost(1);
    for (int k = 2; k <= ks_max && tiles * k <= sms && k <= KT; ++k) {
      const int c = cost(k);
      if (c < best) {
        best = c;
        ks = k;
      }
    }
  }
  return ks;
}

template <int PREC>
cudaError_t launch_prec(const ConvParams& p, const ConvParams& p2, int bn, int grid, cudaStream_t stream) {
  if (p.group_units) {  // grouped launches use tile widths <= 128, or 192
    if constexpr (PREC != 2)
      if (bn == 192) return launch_bn<192, PREC, true>(p, p2, grid, stream);
    if (bn == 32) return launch_bn<32, PREC, true>(p, p2, grid, stream);
    if (bn == 64) return launch_bn<64, PREC, true>(p, p2, grid, stream);
    return launch_bn<128, PREC, true>(p, p2, grid, stream);
  }
  if (bn == 32) return launch_bn<32, PREC, false>(p, p2, grid, stream);
  if (bn == 64) return launch_bn<64, PREC, false>(p, p2, grid, stream);
  if (bn == 128) return launch_bn<128, PREC, false>(p, p2, grid, stream);
  if constexpr (PREC != 2) {
    if (bn == 192) return launch_bn<192, PREC, false>(p, p2, grid, stream);
    if (bn == 160) return launch_bn<160, PREC, false>(p, p2, grid, stream);
  }
  return launch_bn<256, PREC, false>(p, p2, grid, stream);
}

cudaError_t launch_dispatch(const ConvParams& p, const ConvParams& p2, int bn, int grid, cudaStream_t stream) {
  if (p.prec == 1) return launch_prec<1>(p, p2, bn, grid, stream);
  if (p.prec == 2) return launch_prec<2>(p, p2, bn, grid, stream);
  return launch_prec<0>(p, p2, bn, grid, stream);
}
}  // namespace

cudaError_t launch_conv_tc(ConvParams p, cudaStream_t stream) {
  if (p.Cin % 4 != 0 || p.Kpad % conv_tc::kBK != 0 || p.Kpad < p.K || p.nimg <= 0)
    return cudaErrorInvalidValue;
  int bn = conv_tile_n(p.N);
  const int sms = sm_count();
  const int KT = p.Kpad / conv_tc::kBK;
  if (p.tap_rows && (!conv_tap_rows_eligible(p.Cin, p.KW) || p.Kpad != p.KH * conv_tc::kBK))
    return cudaErrorInvalidValue;
  p.m_tiles = (p.nimg * p.Ho * p.Wo + conv_tc::kBM - 1) / conv_tc::kBM;
  if (use_mid(p)) {
    bn = 192;
    p.wmap = *p.wmap_mid;
  } else if (use_mid160(p)) {
    bn = 160;
    p.wmap = *p.wmap_mid160;
  } else if (use_wide(p, sms)) {
    bn = 256;
    p.wmap = *p.wmap_wide;
  }
  p.n_tiles = (p.N + bn - 1) / bn;
  const int tiles = p.m_tiles * p.n_tiles;
  // Split K when the tiles cannot cover the SMs (small merged batches):
  // minimise the estimated makespan waves(units) * (K tiles per unit +
  // overhead); a split launch has one CTA per unit (cluster = the splits).
  int ks = choose_ksplits(tiles, KT, sms);
  if (p.ks_force > 0) ks = std::min({p.ks_force, 8, KT});  // measured choice (executor autotune)
  // n-minor unit order (opt-in BS_CONV_NMINOR=1): an M tile's activations
  // are re-read for each N tile while still in L2 (1x1 56x56 64->256 +
  // residual at b=90: 190 -> 184 us; ResNet-50 layer sum -1%), but the e2e
  // (H2D admission) serving capacity came out lower in both bench runs with
  // it (29.6k / 31.6k vs 35.2k-37.0k req/s with m-minor).
  const char* nm = std::getenv("BS_CONV_NMINOR");  // per launch (A/B)
  p.n_minor = nm ? (nm[0] == '1') : 0;
  p.ksplits = std::max(1, ks);
  const int units = tiles * p.ksplits;
  const int grid = p.ksplits > 1 ? units : std::min(units, sms);
  static const bool log = std::getenv("BS_CONV_LOG") != nullptr;
  if (log)
    std::fprintf(stderr, "conv M=%d N=%d K=%d KT=%d bn=%d tiles=%d ks=%d grid=%d tap_rows=%d\n",
                 p.nimg * p.Ho * p.Wo, p.N, p.K, KT, bn, tiles, p.ksplits, grid, p.tap_rows);
  p.group_units = 0;
  return launch_dispatch(p, p, bn, grid, stream);
}

cudaError_t launch_conv_tc_group(ConvParams a, ConvParams b, cudaStream_t stream, bool force, int ks) {
  for (const ConvParams* q : {&a, &b})
    if (q->Cin % 4 != 0 || q->Kpad % conv_tc::kBK != 0 || q->Kpad < q->K || q->nimg <= 0 || q->tap_rows ||
        q->prec != a.prec)
      return cudaErrorInvalidValue;
  int bn = std::max(conv_tile_n(a.N), conv_tile_n(b.N));
  // 128 x 192 tiles for the pair (group maps at 192 rows in wmap_mid) when
  // they cut the wider conv's N tiles (N = 176 / 192 / 288 / 320 / 384 ...);
  // BS_CONV_G192=0 disables.
  const char* e192 = std::getenv("BS_CONV_G192");
  // Only when the pair still fills the GPU with the wider tiles (at small
  // batches fewer, wider tiles cost parallelism: GoogLeNet b=8 +4%).
  const int big = std::max(a.N, b.N);
  const int big_m = (a.N >= b.N ? a.nimg * a.Ho * a.Wo : b.nimg * b.Ho * b.Wo);
  const bool g192 = !(e192 && e192[0] == '0') && a.prec != 2 && a.wmap_mid && b.wmap_mid && big > 128 &&
                    (big + 191) / 192 < (big + 127) / 128 &&
                    ((big_m + conv_tc::kBM - 1) / conv_tc::kBM) * ((big + 191) / 192) >= sm_count();
  if (g192) {
    bn = 192;
    a.wmap = *a.wmap_mid;
    b.wmap = *b.wmap_mid;
  }
  // Unforced, a group is unsplit: decline (the caller launches the two convs
  // separately) when either conv would be split on its own.
  for (const ConvParams* q : {&a, &b}) {
    if (force) break;
    const int qbn = conv_tile_n(q->N);
    const int tiles = ((q->nimg * q->Ho * q->Wo + conv_tc::kBM - 1) / conv_tc::kBM) * ((q->N + qbn - 1) / qbn);
    if (choose_ksplits(tiles, q->Kpad / conv_tc::kBK, sm_count()) > 1) return cudaErrorNotSupported;
    ConvParams t = *q;
    t.m_tiles = (q->nimg * q->Ho * q->Wo + conv_tc::kBM - 1) / conv_tc::kBM;
    // 128 x 256 / 160 / 192 tiles beat the group (192: unless the group itself runs 192-wide)
    if (use_wide(t, sm_count()) || (use_mid(t) && !g192) || use_mid160(t)) return cudaErrorNotSupported;
  }
  ks = force ? std::max(1, std::min({ks, 8, a.Kpad / conv_tc::kBK, b.Kpad / conv_tc::kBK})) : 1;
  for (ConvParams* q : {&a, &b}) {
    q->m_tiles = (q->nimg * q->Ho * q->Wo + conv_tc::kBM - 1) / conv_tc::kBM;
    q->n_tiles = (q->N + bn - 1) / bn;
    q->ksplits = ks;
    q->group_units = 0;
    const char* nm = std::getenv("BS_CONV_NMINOR");
    q->n_minor = nm ? (nm[0] == '1') : 0;
  }
  b.trace = a.trace;
  a.group_units = b.m_tiles * b.n_tiles * ks;
  const int units = a.m_tiles * a.n_tiles * ks + a.group_units;
  const int grid = ks > 1 ? units : std::min(units, sm_count());
  static const bool log = std::getenv("BS_CONV_LOG") != nullptr;
  if (log)
    std::fprintf(stderr, "conv M=%d N=%d K=%d KT=%d bn=%d units=%d ks=%d grid=%d group=M%dN%dK%d\n",
                 a.nimg * a.Ho * a.Wo, a.N, a.K, a.Kpad / conv_tc::kBK, bn, units, ks, grid, b.nimg * b.Ho * b.Wo,
                 b.N, b.K);
  return launch_dispatch(a, b, bn, grid, stream);
}

}  // namespace bs200
