// Implicit-GEMM convolution / fully-connected layer on the sm_100a tensor
// cores (tcgen05.mma kind::tf32, accumulator in TMEM).
//
//   D[m, n] = sum_k A[m, k] * W[n, k]      m = (image, ho, wo), n = out channel,
//                                          k = (kh, kw, ci) with ci fastest
//
// Persistent, one CTA per SM. The launcher cuts the GEMM into work units =
// (128 x BN output tile) x (K split); CTA c walks units c, c + G, c + 2G, ...
// with one continuous shared-memory ring across units, so loads for the next
// unit overlap the MMAs and epilogue of the current one. The accumulator is
// double-buffered in TMEM (2 x BN columns): the epilogue of unit i drains one
// buffer while the MMAs of unit i+1 fill the other. Small-M layers (batches
// of a few requests) are split along K so the grid still covers all SMs:
// the splits of a tile form one thread-block cluster, park their partial
// tiles in their own shared memory and reduce them over DSMEM in fixed split
// order (deterministic results, no global workspace, no cross-CTA spin).
//
// Loads and operands:
//   * B (weights, dense [N][Kpad]) by TMA, one 128B-swizzled 2D box per stage,
//     read by the tensor core from shared memory;
//   * A gathered straight from the NHWC request blobs with cp.async (zero-fill
//     = spatial padding and M/K tails) into a raw shared-memory ring. Every
//     image of a merged batch has its own base pointer, so requests stay in
//     their own arena slots: the batch is gathered by the loader and
//     scattered by the epilogue with no copy kernels.
//     Completion: cp.async.mbarrier.arrive.noinc.
//   * Converter warps move each landed raw A stage into TMEM (tcgen05.st) as
//     the MMA's A operand (tcgen05.mma ... [a_tmem] form) and free the raw
//     stage at once, so the gather runs RA stages ahead of the converters
//     instead of waiting for the MMAs of the stage it overwrites.
//   * 2xTF32 split-A (default precision): weights are exactly TF32, so
//     A*W = A_hi*W + A_lo*W with A_hi = rn_tf32(A) recovers ~fp32 accuracy at
//     two MMAs per K step and no extra HBM or shared-memory traffic (A_lo
//     lives in TMEM next to A_hi).
//
// Warp roles: 0-3 A cp.async producers, 4-7 epilogue (TMEM lanes 0-127),
// 8 MMA issuer (+ TMEM owner), 9 B TMA issuer, 10-13 A converters (group 0),
// 14 idle, 15-18 A converters (group 1).
#pragma once
#include <cmath>
#include <cstdint>
#include <type_traits>

#include <cuda.h>

#include "pdl.cuh"
#include "ptx.cuh"

namespace bs200 {

struct ConvParams {
  CUtensorMap wmap;             // weights [N][Kpad] (2D, box {32, BN}, SWIZZLE_128B)
  int nimg;                     // images in the merged batch
  int H, W, Cin;                // input spatial size; Cin = padded channel count (% 4 == 0)
  int Ho, Wo;                   // output spatial size
  int KH, KW, stride, pad;
  int K;                        // KH * KW * Cin
  int Kpad;                     // K rounded up to 32 (row stride of the weights)
  int N;                        // output channels
  const float* const* in_ptrs;  // [nimg] per-request blob base pointers
  long in_off;                  // element offset of (pixel 0, first channel) in the blob
  int in_ldc;                   // floats per pixel
  const float* wgt;             // weights (for the tensor map; also a valid dummy address)
  const float* bias;            // [N] or nullptr
  float* const* out_ptrs;       // [nimg]
  long out_off;
  int out_ldc;
  const float* const* res_ptrs; // [nimg] or nullptr (residual add before ReLU)
  long res_off;
  int res_ldc;
  int relu;                     // 0 none, 1 ReLU, 2 ReLU6
  int round_out;                // round outputs to TF32 (they feed another GEMM)
  int prec;                     // 0 TF32, 1 2xTF32 (A = A_hi + A_lo, near-fp32 accuracy), 2 BF16
  // work decomposition (filled by launch_conv_tc)
  int m_tiles, n_tiles, ksplits;  // K tiles of split s: [s KT / ksplits, (s + 1) KT / ksplits)
  unsigned long long* trace;    // debug timeline of CTA 0 (nullptr in production)
  // Tap-row mode (Cin * 32 / Cin taps = one K tile per filter row): K order
  // (kh, kw < 32 / Cin, ci) with zero weights past KW, Kpad = KH * 32. Each
  // output pixel's A row of a K tile is 32 / Cin consecutive input pixels
  // (128 contiguous bytes); only the input row advances per K tile.
  int tap_rows;
  // Grouped launch: units past this problem's own belong to the kernel's
  // second ConvParams (an independent conv of the same layer, e.g. the two
  // branch convs of an inception block), so one persistent launch covers
  // both and the small one stops paying a launch + pipeline fill of its own.
  int group_units;
  // Tile-width preference from the executor's profile-time autotune:
  // 0 = launcher rule, 1 = 128 x 256 tiles (needs wmap_wide), 2 = 128-wide,
  // 3 = 128 x 192 tiles (needs wmap_mid), 4 = 128 x 160 (needs wmap_mid160).
  int wide_pref;
  // K-split override from the same autotune: 0 = launcher cost model, else
  // the split count (clamped to the K tiles and the cluster limit of 8).
  int ks_force;
  int n_minor;                  // unit order (see unit_of)
  // Host side only (the launcher swaps it into wmap for 128 x 256 tiles):
  // weights map with a 256-row box (N > 128), owned by the caller.
  const CUtensorMap* wmap_wide;
  // Host side only: weights map with a 192-row box (N > 128) for 128 x 192
  // tiles -- N = 192 in one tile, or 384 / 576 in exact tiles, with two TMEM
  // accumulators (the 256-wide tile has one); owned by the caller.
  const CUtensorMap* wmap_mid;
  // Host side only: the same with a 160-row box (128 x 160 tiles: N = 320 in
  // two exact tiles instead of 128 + 128 + 64), owned by the caller.
  const CUtensorMap* wmap_mid160;
};


namespace conv_tc {

constexpr int kBM = 128;
constexpr int kBK = 32;  // fp32 elements per 128-byte K row

// Pipeline geometry per N tile (TF32 / BF16). Three rings decouple the
// stages so no load waits on an MMA it does not feed:
//   raw A  (smem, RA x 16 KB): cp.async gather target; freed as soon as the
//          converter warps have read a stage (not when the MMA finishes);
//   B      (smem, NB x BN*128 B): weights by TMA, 128B-swizzled for UMMA
//          (bf16: BN*64 B stages, 64B-swizzled);
//   A op   (TMEM, TA slots): converted A operand, [hi | lo] for 2xTF32,
//          packed bf16 pairs for BF16; the MMAs read A from TMEM, so shared
//          memory only serves B to the tensor core.
// PREC: 0 = TF32 (one MMA), 1 = 2xTF32 (split A, ~fp32 accuracy),
//       2 = BF16 (A rounded to bf16 by the converters, bf16 weights).
// 2xTF32 ("HIS", hi in shared memory): the tensor core reads fp32 data as
// TF32 by dropping the 13 low mantissa bits, i.e. exactly A_hi, so the A_hi
// MMAs read the raw gathered stage from shared memory (SS form, the same
// 128B-swizzled K-major layout as the weights) and only A_lo = A - A_hi goes
// through the converters into TMEM (TS form). The A_hi MMAs need no
// conversion, the converters and TMEM stores do half the work, and raw A,
// B and the A_lo slot of a K tile live in one ring of D stages freed by the
// K tile's single commit.

template <int BN, int PREC>
struct Cfg {
  static constexpr int kThreads = 608;
  // 2xTF32 reads A_hi straight from the raw gathered stage (HIS, see below).
  static constexpr bool HIS = PREC == 1;
  // BN = 256: one accumulator (256 columns) so the A slots still fit in TMEM;
  // the raw A ring shrinks to make room for the 32 KB B stages.
  static constexpr int kAcc = BN == 256 ? 1 : 2;                 // TMEM accumulator buffers
  // TMEM columns per A slot: A_lo only for 2xTF32 (A_hi is read from shared
  // memory), TF32 operand for TF32, packed bf16 pairs for BF16.
  static constexpr int kACols = PREC == 2 ? kBK / 2 : kBK;
  static constexpr int kTA0 = kAcc * BN;                         // first A column (after the accumulators)
  // One operand stage = (TMEM A slot, B smem stage), released by a single
  // tcgen05.commit per K tile (each commit costs the tensor pipe ~84 cycles).
  static constexpr int kTAmax = (512 - kTA0) / kACols;
  // Per epilogue warp: bias [2][BN] fp32, blob-table entries [2][32] (out,
  // residual) and the unit's final row pointers [32] (out, residual).
  static constexpr int kEpiWarpBytes = 8 * BN + 1536;
  static constexpr int kBRow = PREC == 2 ? 64 : 128;             // bytes per weight row of a K tile
  static constexpr int kFixed = 1024 + 512 + kBM * 32 * 4 + 4 * kEpiWarpBytes;
  static constexpr int kABytes = kBM * 128;
  static constexpr int kBBytes = BN * kBRow;
  static constexpr int min3(int a, int b, int c) { return a < b ? (a < c ? a : c) : (b < c ? b : c); }
  // HIS: one ring of D stages (raw A, B, TMEM A_lo) freed by one commit.
  static constexpr int kD = min3(kTAmax, (232448 - kFixed) / (kABytes + kBBytes), 8);
  static constexpr int RA = HIS ? kD : (BN == 32 ? 10 : BN == 256 ? 6 : 8);
  static constexpr int kNBmax = (232448 - kFixed - RA * kABytes) / kBBytes;
  static constexpr int TA = HIS ? kD : min3(kTAmax, kNBmax, 8);
  static constexpr int NB = TA;
  static constexpr int kBOffset = RA * kABytes;
  static constexpr int kStagingOffset = kBOffset + NB * kBBytes;  // epilogue staging, 128 x 32 fp32
  static constexpr int kEpiOffset = kStagingOffset + kBM * 32 * 4;
  static constexpr int kBarOffset = kEpiOffset + 4 * kEpiWarpBytes;
  static constexpr int kTotal = kBarOffset + 512 + 1024;        // barriers + alignment slack
  static_assert(kTotal <= 232448, "shared memory budget");
  static_assert(TA >= 2, "TMEM budget");
  static_assert(!HIS || (RA == TA && NB == TA), "HIS rings share one index");
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t swz(int row, int chunk) {
  return static_cast<uint32_t>(row * 128 + ((chunk ^ (row & 7)) << 4));
}

__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

struct Unit {
  int mt, m_base, n_base, tile, split, kt0, kt1;
};

__device__ __forceinline__ Unit unit_of(const ConvParams& p, int u, int BN, int KT) {
  Unit w;
  w.split = u % p.ksplits;
  w.tile = u / p.ksplits;
  // m-minor: consecutive tiles share a weight slice; n-minor: the N tiles of
  // an M tile run back to back, so its activations are re-read from L2.
  const int mt = p.n_minor ? w.tile / p.n_tiles : w.tile % p.m_tiles;
  const int nt = p.n_minor ? w.tile % p.n_tiles : w.tile / p.m_tiles;
  w.mt = mt;
  w.m_base = mt * kBM;
  w.n_base = nt * BN;
  // balanced: every split has >= 1 K tile when ksplits <= KT
  w.kt0 = (w.split * KT) / p.ksplits;
  w.kt1 = ((w.split + 1) * KT) / p.ksplits;
  return w;
}

// Output pixel of row r of M tile mt: image and pixel index, false for
// padding rows (M tail).
__device__ __forceinline__ bool row_pixel(const ConvParams& p, int mt, int r, int& img, int& pix) {
  const int m = mt * kBM + r;
  const int HoWo = p.Ho * p.Wo;
  img = m / HoWo;
  pix = m - img * HoWo;
  return m < p.nimg * HoWo;
}

// A operand conversion. 2xTF32: hi = x with the 13 low mantissa bits
// cleared (exactly TF32), lo = x - hi (exact in fp32; the tensor core keeps
// its top 11 bits, so |error| <= 2^-21 |x|). Plain TF32: round to nearest
// (ties away) by integer add + mask, valid for finite x.
template <bool SPLIT>
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
  const uint32_t u = __float_as_uint(x);
  if constexpr (SPLIT) {
    hi = u & 0xffffe000u;
    lo = __float_as_uint(x - __uint_as_float(hi));
  } else {
    hi = (u + 0x1000u) & 0xffffe000u;
    (void)lo;
  }
}

// One K-tile row of A (32 fp32 values, this thread's TMEM lane) -> operand
// registers: TF32 / 2xTF32 hi (+ lo) words, or (BF16) 16 packed bf16 pairs.
template <int PREC>
__device__ __forceinline__ void a_operand(const float4 (&v)[8], uint32_t (&hi)[32], uint32_t (&lo)[32]) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    if constexpr (PREC == 2) {
      hi[2 * c] = ptx::pack_bf16x2(v[c].x, v[c].y);
      hi[2 * c + 1] = ptx::pack_bf16x2(v[c].z, v[c].w);
    } else {
      const float x[4] = {v[c].x, v[c].y, v[c].z, v[c].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) split_tf32<PREC == 1>(x[e], hi[4 * c + e], lo[4 * c + e]);
    }
  }
}
template <int PREC>
__device__ __forceinline__ void a_store(uint32_t dst, const uint32_t (&hi)[32], const uint32_t (&lo)[32]) {
  if constexpr (PREC == 2) {
    ptx::tmem_st16(dst, *reinterpret_cast<const uint32_t(*)[16]>(hi));
  } else {
    ptx::tmem_st32(dst, hi);
    if constexpr (PREC == 1) ptx::tmem_st32(dst + kBK, lo);
  }
}

__device__ __forceinline__ float epilogue_op(const ConvParams& p, float x, int n, const float* res_row) {
  if (p.bias) x += __ldg(p.bias + n);
  if (res_row) x += res_row[n];
  if (p.relu == 1) x = fmaxf(x, 0.f);
  else if (p.relu == 2) x = fminf(fmaxf(x, 0.f), 6.f);
  if (p.round_out) x = ptx::round_tf32(x);
  return x;
}

// Kernel parameters: one problem, or two for a grouped launch (an ungrouped
// launch does not ship a second ConvParams: the parameter block is what the
// host pays per launch).
template <bool GROUP>
struct ConvArgs {
  ConvParams a;
};
template <>
struct ConvArgs<true> {
  ConvParams a, b;
};
template <bool GROUP>
__device__ __forceinline__ const ConvParams& second_problem(const ConvArgs<GROUP>& k) {
  if constexpr (GROUP) return k.b;
  else return k.a;
}

template <int BN, int PREC, bool GROUP>
__global__ void __launch_bounds__(Cfg<BN, PREC>::kThreads, 1)
    conv_tc_kernel(const __grid_constant__ ConvArgs<GROUP> args) {
  // Roles take the problem of each unit from BS_UNIT_PROBLEM (p_a for the
  // first units0 units, p_b after); outside unit loops p is p_a.
  const ConvParams& p_a = args.a;
  const ConvParams& p_b = second_problem<GROUP>(args);
  const ConvParams& p = p_a;
  using S = Cfg<BN, PREC>;
  constexpr bool SPLIT = PREC == 1, BF16 = PREC == 2;
  constexpr int RA = S::RA, NB = S::NB, TA = S::TA;
  extern __shared__ uint8_t smem_raw[];
  // Align by pointer arithmetic on the __shared__ array (not via uintptr_t)
  // so accesses through `smem` stay LDS/STS instead of generic LD/ST.
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* ra_full = reinterpret_cast<uint64_t*>(smem + S::kBarOffset);
  uint64_t* ra_empty = ra_full + RA;
  uint64_t* b_full = ra_empty + RA;
  uint64_t* ta_full = b_full + NB;
  uint64_t* ta_empty = ta_full + TA;
  uint64_t* b_empty = S::HIS ? ra_empty : ta_empty;  // same ring: one commit frees slot and stage(s)
  uint64_t* acc_full = ta_empty + TA;  // [2]
  uint64_t* acc_empty = acc_full + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int M = p.nimg * p.Ho * p.Wo;
  const int KT = p.Kpad / kBK;
  const int units0 = p.m_tiles * p.n_tiles * p.ksplits;
  const int units = units0 + (GROUP ? p.group_units : 0);
  // GROUP is a template flag so an ungrouped launch binds p to p_a at compile
  // time (constant-bank loads); a runtime-selected reference turns every
  // parameter read into a generic load (measured +5% on ResNet-50).
#define BS_UNIT_PROBLEM(uv)                                                   \
  const ConvParams& p = (!GROUP || (uv) < units0) ? p_a : p_b;                \
  const int KT = p.Kpad / kBK;                                                \
  [[maybe_unused]] const int M = p.nimg * p.Ho * p.Wo;                        \
  const int lu = (!GROUP || (uv) < units0) ? (uv) : (uv) - units0;
  const uint32_t smem_base = ptx::smem_u32(smem);
  // trace: [8 + 4 b + {0 start, 1 setup done, 2 first A issued, 3 end}]
  if (p.trace && threadIdx.x == 0) p.trace[8 + 4 * blockIdx.x] = gtime();

  if (threadIdx.x == 0) {
    for (int s = 0; s < RA; ++s) {
      // one cp.async .noinc arrival per producer thread; freed by the
      // converters' reads (TF32 / BF16) or by the K tile's commit (HIS)
      ptx::mbar_init(&ra_full[s], 128);
      ptx::mbar_init(&ra_empty[s], S::HIS ? 1 : 128);
    }
    for (int s = 0; s < NB; ++s) {
      ptx::mbar_init(&b_full[s], 1);
    }
    for (int s = 0; s < TA; ++s) {
      ptx::mbar_init(&ta_full[s], 4);  // one arrival per converter warp
      ptx::mbar_init(&ta_empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&acc_full[a], 1);
      ptx::mbar_init(&acc_empty[a], 4);  // one arrival per epilogue warp
    }
    ptx::fence_mbar_init();
  }
  if (warp == 9 && lane == 0) {
    ptx::prefetch_tmap(&p_a.wmap);
    if (GROUP) ptx::prefetch_tmap(&p_b.wmap);
  }
  if (warp == 8) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Everything above overlapped the previous kernel's tail (PDL). Only the
  // roles that read activations wait for the previous kernel: the A gather
  // (here) and the epilogue (after it has prefetched its immutable blob-table
  // entries and bias, before residual reads). The weight TMA warp reads only
  // immutable weights; the MMA issuer and the converters touch shared memory
  // and TMEM only, fed by those roles, so they start at once. Every output
  // store follows the gather's wait (it depends on the gathered A), and the
  // kernel cannot complete before its producers passed the wait, so
  // completion stays ordered along the stream. The gather waits right
  // before its first copy, so its first unit's row setup and blob-table loads
  // (immutable for the kernel) overlap the previous kernel too.
  if (p.trace && threadIdx.x == 0) p.trace[8 + 4 * blockIdx.x + 1] = gtime();

  // Converter: thread = one A row (TMEM lane). Reads its 128-byte row of a
  // landed raw stage, frees the stage, and writes the MMA operand into its
  // TMEM lane (TF32 hi (+ lo for 2xTF32), or packed bf16 pairs). Two
  // converter groups (warps 10-13 and 15-18) take alternate K tiles so the
  // conversion latency overlaps.
  auto convert = [&](int group, int ngroups, int trace_tid) {
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row = q * 32 + lane;
    uint32_t roff[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) roff[c] = swz(row, c);
    const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + S::kTA0;
    int it = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      BS_UNIT_PROBLEM(u)
      const Unit w = unit_of(p, lu, BN, KT);
      for (int kt = w.kt0; kt < w.kt1; ++kt, ++it) {
        if (it % ngroups != group) continue;
        const int s = it % RA;
        ptx::mbar_wait(&ra_full[s], (it / RA) & 1);
        if (p.trace && threadIdx.x == trace_tid && blockIdx.x == 0 && it < 48) p.trace[1024 + it * 5 + 2] = gtime();
        const uint32_t a_raw = smem_base + s * S::kABytes;
        float4 v[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) v[c] = ptx::lds128(a_raw + roff[c]);
        const int sa = it % TA;
        if constexpr (S::HIS) {
          // A_lo only. Slot sa (== s) is free: this stage's gather was issued
          // after the commit of K tile it - D, which retired the slot's MMAs.
          uint32_t lo[32];
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float x[4] = {v[c].x, v[c].y, v[c].z, v[c].w};
#pragma unroll
            for (int e = 0; e < 4; ++e)
              lo[4 * c + e] = __float_as_uint(x[e] - __uint_as_float(__float_as_uint(x[e]) & 0xffffe000u));
          }
          ptx::tc_fence_after();
          ptx::tmem_st32(lane_base + sa * S::kACols, lo);
        } else {
          ptx::mbar_arrive(&ra_empty[s]);
          uint32_t hi[32];
          [[maybe_unused]] uint32_t lo[32];
          a_operand<PREC>(v, hi, lo);
          if (it >= TA) ptx::mbar_wait(&ta_empty[sa], ((it / TA) - 1) & 1);
          ptx::tc_fence_after();
          const uint32_t dst = lane_base + sa * S::kACols;
          a_store<PREC>(dst, hi, lo);
        }
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        // one arrival per warp after the warp's stores are fenced (each
        // barrier arrival is a shared-memory atomic on the K loop's path)
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&ta_full[sa]);
        if (p.trace && threadIdx.x == trace_tid && blockIdx.x == 0 && it < 48) p.trace[1024 + it * 5 + 3] = gtime();
      }
    }
  };

  if (warp < 4) {
    // ------------------------------------------------------------ A gather  } else if (warp < 4) {
    // ------------------------------------------------------------ A gather
    const int t = threadIdx.x;
    const int c = t & 7;    // 16-byte chunk inside the 128-byte K row
    const int r0 = t >> 3;  // rows r0 + 16 i
    const int HoWo = p.Ho * p.Wo;
    const float* dummy = p.wgt;
    int it = 0;  // ring position across units
    bool waited = false;
    auto wait_once = [&] {
      if (!waited) pdl::wait();
      waited = true;
    };
    // (image, ho, wo) of rows r0 + 16 i of the tile at m_base: one division
    // pair, then a 16-row walk (was 16 divisions per unit; the unit switch
    // stalled the stem's producer ~1.4 us). Rows past M: ok = false, image 0.
    auto walk_rows = [&](const ConvParams& q, int m_base, int (&n)[8], int (&ho)[8], int (&wo)[8], bool (&ok)[8]) {
      const int qHoWo = q.Ho * q.Wo, qM = q.nimg * qHoWo;
      int m = m_base + r0;
      int nn = m / qHoWo;
      const int rem = m - nn * qHoWo;
      int h = rem / q.Wo;
      int ww = rem - h * q.Wo;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        ok[i] = m < qM;
        n[i] = ok[i] ? nn : 0;
        ho[i] = h;
        wo[i] = ww;
        m += 16;
        ww += 16;
        while (ww >= q.Wo) {
          ww -= q.Wo;
          if (++h == q.Ho) {
            h = 0;
            ++nn;
          }
        }
      }
    };
    if (p.tap_rows) {
      // One K tile per filter row kh. Warp pw owns tile rows 32 pw .. +31:
      // lane l works out row 32 pw + l (image, input row / column origin)
      // once per unit, and the 8 row groups a lane copies (rows 4 i + l / 8,
      // 16 bytes = tap kw, channels ci..ci+3) come from shuffles; the row
      // state was computed 8x redundantly per lane before (~480 SASS per
      // unit on the producer, which paces the stems).
      const int pw = warp;
      const int cc = lane & 7;
      const int kw = (cc * 4) / p.Cin, ci = cc * 4 - kw * p.Cin;
      const long hstride = static_cast<long>(p.W) * p.in_ldc;
      // Own-row state of the next unit (its image pointer load is issued a
      // unit ahead of its use).
      int nx_h0 = 0, nx_w0 = 0;
      bool nx_ok = false;
      const float* nx_img = nullptr;
      auto own_row = [&](int u) {
        const int m = unit_of(p, u, BN, KT).m_base + 32 * pw + lane;
        nx_ok = m < M;
        const int mm = nx_ok ? m : 0;
        const int n = mm / HoWo;
        const int rem = mm - n * HoWo;
        const int ho = rem / p.Wo;
        nx_h0 = ho * p.stride - p.pad;
        nx_w0 = (rem - ho * p.Wo) * p.stride - p.pad;
        nx_img = p.in_ptrs[n] + p.in_off;
      };
      uint32_t doff[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) doff[i] = swz(32 * pw + 4 * i + (lane >> 3), cc);
      if (static_cast<int>(blockIdx.x) < units) own_row(blockIdx.x);
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const Unit w = unit_of(p, u, BN, KT);
        const int my_h0 = nx_h0, my_w0 = nx_w0;
        const bool my_ok = nx_ok;
        const float* my_img = nx_img;
        if (u + static_cast<int>(gridDim.x) < units) own_row(u + gridDim.x);
        const float* base[8];
        int h0[8];
        bool ok_w[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int src = 4 * i + (lane >> 3);
          const int rh = __shfl_sync(0xffffffffu, my_h0, src);
          const int wi = __shfl_sync(0xffffffffu, my_w0, src) + kw;
          const bool rok = __shfl_sync(0xffffffffu, static_cast<int>(my_ok), src) != 0;
          const float* img = reinterpret_cast<const float*>(
              __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(my_img), src));
          h0[i] = rh + w.kt0;
          ok_w[i] = rok && kw < p.KW && wi >= 0 && wi < p.W;
          base[i] = img + (static_cast<long>(h0[i]) * p.W + wi) * p.in_ldc + ci;
        }
        wait_once();
        for (int kt = w.kt0; kt < w.kt1; ++kt, ++it) {
          const int s = it % RA;
          if (it >= RA) ptx::mbar_wait(&ra_empty[s], ((it / RA) - 1) & 1);
          const uint32_t a_tile = smem_base + s * S::kABytes;
          // The copies read the loop-carried row pointers (an out-of-image
          // tap keeps its address and copies 0 bytes: cp.async zero-fills
          // without reading).
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const bool ok = ok_w[i] && static_cast<unsigned>(h0[i]) < static_cast<unsigned>(p.H);
            ptx::cp_async16(a_tile + doff[i], base[i], ok ? 16u : 0u);
            base[i] += hstride;
            ++h0[i];
          }
          ptx::cp_async_arrive_noinc(&ra_full[s]);
          if (p.trace && threadIdx.x == 0 && blockIdx.x == 0 && it < 48) p.trace[1024 + it * 5 + 0] = gtime();
        }
      }
    }
    for (int u = blockIdx.x; u < units && !p.tap_rows; u += gridDim.x) {
      BS_UNIT_PROBLEM(u)
      const bool aligned = p.Cin % kBK == 0;
      const Unit w = unit_of(p, lu, BN, KT);
      const bool ptr_tr = p.trace && t == 0 && blockIdx.x == 0 && u < 32 * static_cast<int>(gridDim.x);
      const int ptr_j = u / static_cast<int>(gridDim.x);
      if (ptr_tr) p.trace[3400 + ptr_j * 4 + 0] = gtime();
      const float* row_base[8];
      int row_h[8], row_w[8];
      bool row_ok[8];
      {
        int rn[8], rho[8], rwo[8];
        walk_rows(p, w.m_base, rn, rho, rwo, row_ok);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          row_h[i] = rho[i] * p.stride - p.pad;
          row_w[i] = rwo[i] * p.stride - p.pad;
          row_base[i] = p.in_ptrs[rn[i]] + p.in_off;
        }
      }
      if (ptr_tr) p.trace[3400 + ptr_j * 4 + 1] = gtime() + (reinterpret_cast<uintptr_t>(row_base[0]) & 1);
      uint32_t doff[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) doff[i] = swz(r0 + 16 * i, c);
      if (aligned) {
        // Filter-tap-major walk: per (kh, kw) the 8 row sources and byte
        // counts are computed once; each K tile is then 8 independent
        // cp.async with hoisted smem offsets (no divisions, no selects).
        int tap = (w.kt0 * kBK) / p.Cin;
        int ci = w.kt0 * kBK - tap * p.Cin;
        int kh = tap / p.KW, kw = tap - kh * p.KW;
        const float* src[8];
        uint32_t nbytes[8];
        auto set_tap = [&] {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int h = row_h[i] + kh, ww = row_w[i] + kw;
            const bool ok = row_ok[i] && h >= 0 && h < p.H && ww >= 0 && ww < p.W;
            src[i] = row_base[i] + (h * p.W + ww) * p.in_ldc + c * 4 + ci;  // 0 bytes when !ok
            nbytes[i] = ok ? 16u : 0u;
          }
        };
        set_tap();
        if (ptr_tr) p.trace[3400 + ptr_j * 4 + 2] = gtime() + (nbytes[7] & 1);
        wait_once();
        for (int kt = w.kt0; kt < w.kt1; ++kt, ++it) {
          const int s = it % RA;
          if (it >= RA) ptx::mbar_wait(&ra_empty[s], ((it / RA) - 1) & 1);
          const uint32_t a_tile = smem_base + s * S::kABytes;
          // src[i] already points at this K tile (ci folded in): each LDGSTS
          // reads a loop-carried register, never a reused temporary.
          ptx::cp_async16x8(a_tile + doff[0], 16 * 128, src, nbytes);
          ptx::cp_async_arrive_noinc(&ra_full[s]);
          if (p.trace && t == 0 && it == 0) p.trace[8 + 4 * blockIdx.x + 2] = gtime();
          if (p.trace && t == 0 && blockIdx.x == 0 && it < 48) p.trace[1024 + it * 5 + 0] = gtime();
          ci += kBK;
          if (ci == p.Cin) {
            if (kt + 1 < w.kt1) {
              ci = 0;
              if (++kw == p.KW) {
                kw = 0;
                ++kh;
              }
              set_tap();
            }
          } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) src[i] += kBK;
          }
        }
      } else {
        // Generic K walk (stem Cin = 4, narrow inputs): this thread's 4
        // channels start at k = kt * 32 + 4c; the (ci, kw, kh) position is
        // stepped by 32 per K tile without divisions.
        int k0 = w.kt0 * kBK + c * 4;
        int q = k0 / p.Cin;
        int ci = k0 - q * p.Cin;
        int kh = q / p.KW;
        int kw = q - kh * p.KW;
        wait_once();
        for (int kt = w.kt0; kt < w.kt1; ++kt, ++it) {
          const int s = it % RA;
          if (it >= RA) ptx::mbar_wait(&ra_empty[s], ((it / RA) - 1) & 1);
          const uint32_t a_tile = smem_base + s * S::kABytes;
          const bool k_ok = k0 < p.K;
          // All 8 addresses first (fresh IMAD.WIDE pairs), then one 8-copy
          // statement: interleaving address math with the copies made every
          // address wait for the previous LDGSTS to release a reused pair.
          const float* srcs[8];
          uint32_t nb[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int h = row_h[i] + kh, ww = row_w[i] + kw;
            const bool ok = k_ok && row_ok[i] && h >= 0 && h < p.H && ww >= 0 && ww < p.W;
            srcs[i] = row_base[i] + (h * p.W + ww) * p.in_ldc + ci;  // 0 bytes when !ok
            nb[i] = ok ? 16u : 0u;
          }
          ptx::cp_async16x8(a_tile + doff[0], 16 * 128, srcs, nb);
          ptx::cp_async_arrive_noinc(&ra_full[s]);
          if (p.trace && t == 0 && blockIdx.x == 0 && it < 48) p.trace[1024 + it * 5 + 0] = gtime();
          k0 += kBK;
          ci += kBK;
          while (ci >= p.Cin) {
            ci -= p.Cin;
            if (++kw == p.KW) {
              kw = 0;
              ++kh;
            }
          }
        }
      }
    }
    wait_once();  // (every CTA has >= 1 unit; kept so completion order never depends on it)
    // The next kernel may be scheduled once every CTA has issued its last
    // gather (its prologue then overlaps this CTA's last K tiles and
    // epilogue). Triggering at entry let a whole step's kernels become
    // resident at once, parked in griddepcontrol.wait, and starve the other
    // streams' kernels (admission, client prefixes) of SMs.
    pdl::launch_dependents();
  } else if (warp < 8) {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 4;
    const int row = ew * 32 + lane;
    const int et = threadIdx.x - 128;  // 0..127
    // The epilogue's global loads (row base pointers from the per-request
    // blob tables, the unit's bias slice) are issued one unit ahead: when the
    // epilogue is the critical role (short-K layers) a load issued at the
    // top of the unit sits behind the producers' traffic in L1 and stalls
    // every chunk (measured ~1 us per chunk on 1x1 layers at b=90).
    // They land by cp.async in this warp's double-buffered area, so they
    // take no registers (held in registers they were spilled at once).
    const uint32_t epi_s = smem_base + S::kEpiOffset + ew * S::kEpiWarpBytes;
    uint8_t* epi_g = smem + S::kEpiOffset + ew * S::kEpiWarpBytes;
    constexpr int kTabB = 8 * BN, kFinB = 8 * BN + 1024;
    const unsigned long long* fin_out = reinterpret_cast<const unsigned long long*>(epi_g + kFinB);
    const unsigned long long* fin_res = fin_out + 32;
    auto prefetch = [&](int u, int buf) {
      BS_UNIT_PROBLEM(u)
      const Unit w = unit_of(p, lu, BN, KT);
      int n_img = 0, pix = 0;
      const bool m_ok = row_pixel(p, w.mt, row, n_img, pix);
      const int ic = m_ok ? n_img : 0;
      ptx::cp_async8(epi_s + kTabB + (buf * 32 + lane) * 8, p.out_ptrs + ic, m_ok ? 8u : 0u);
      if (p.res_ptrs) ptx::cp_async8(epi_s + kTabB + 512 + (buf * 32 + lane) * 8, p.res_ptrs + ic, m_ok ? 8u : 0u);
#pragma unroll
      for (int i = 0; i < BN / 32; ++i) {
        const int n = w.n_base + i * 32 + lane;
        const bool ok = p.bias && n < p.N;
        ptx::cp_async4(epi_s + (buf * BN + i * 32 + lane) * 4, ok ? static_cast<const void*>(p.bias + n) : p.out_ptrs,
                       ok ? 4u : 0u);
      }
      ptx::cp_async_commit();
    };
    if (static_cast<int>(blockIdx.x) < units) prefetch(blockIdx.x, 0);
    pdl::wait();  // residual rows (L1 prefetch / loads) come from earlier kernels
    int j = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      BS_UNIT_PROBLEM(u)
      const Unit w = unit_of(p, lu, BN, KT);
      const int acc = j % S::kAcc;
      const int buf = j & 1;
      // Buffer buf ^ 1 was last read by the previous unit's chunks (this
      // warp, program order); issue the next unit's copies into it, then
      // wait for this unit's group.
      if (u + static_cast<int>(gridDim.x) < units) prefetch(u + gridDim.x, buf ^ 1);
      else ptx::cp_async_commit();  // empty group keeps wait_group<1> exact
      ptx::cp_async_wait<1>();
      __syncwarp();
      const float* bias_st = reinterpret_cast<const float*>(epi_g) + buf * BN;
      float* out_row = nullptr;
      const float* res_row = nullptr;
      {
        int n_img = 0, pix = 0;
        if (row_pixel(p, w.mt, row, n_img, pix)) {
          const auto* tab = reinterpret_cast<const unsigned long long*>(epi_g + kTabB);
          float* ob = reinterpret_cast<float*>(tab[buf * 32 + lane]);
          out_row = ob ? ob + p.out_off + static_cast<long>(pix) * p.out_ldc : nullptr;
          if (p.res_ptrs) {
            const float* rb = reinterpret_cast<const float*>(tab[64 + buf * 32 + lane]);
            res_row = rb ? rb + p.res_off + static_cast<long>(pix) * p.res_ldc : nullptr;
          }
        }
        auto* fin = reinterpret_cast<unsigned long long*>(epi_g + kFinB);
        fin[lane] = reinterpret_cast<unsigned long long>(out_row);
        fin[32 + lane] = reinterpret_cast<unsigned long long>(res_row);
      }
      __syncwarp();
      // Fast path (no split-K, 16-byte aligned rows, N % 4 == 0).
      bool fast = false;
      if (p.ksplits == 1) {
        const bool ok = (reinterpret_cast<uintptr_t>(out_row) & 15) == 0 &&
                        (reinterpret_cast<uintptr_t>(res_row) & 15) == 0 && (!p.res_ptrs || !out_row || res_row);
        fast = __all_sync(0xffffffffu, ok) && (p.N & 3) == 0;
      }
      // Residual rows: this lane's row segment of a 32-column chunk into L1
      // one chunk ahead (the quads are read right after the TMEM load).
      auto prefetch_res = [&](int c) {
        const int n0 = w.n_base + c * 32;
        if (res_row && n0 < p.N) {
          ptx::prefetch_l1(res_row + n0);
          ptx::prefetch_l1(res_row + min(n0 + 31, p.N - 1));
        }
      };
      if (p.ksplits == 1) prefetch_res(0);
      const bool etr = p.trace && threadIdx.x == 128 && blockIdx.x == 0 && j < 32;
      if (etr) p.trace[3072 + j * 8 + 0] = gtime();
      ptx::mbar_wait(&acc_full[acc], (j / S::kAcc) & 1);
      if (etr) p.trace[3072 + j * 8 + 1] = gtime();
      ptx::tc_fence_after();
      const uint32_t tbase = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * BN;
      if (p.ksplits == 1) {
        // Coalesced epilogue: each warp stages its 32 rows x 32 columns in
        // shared memory (16B chunks XOR-swizzled by row), then writes whole
        // 128-byte row segments (8 lanes per row, 4 rows per instruction).
        const uint32_t stage = smem_base + S::kStagingOffset + ew * 32 * 128;
        // One 32-column chunk; RES (a compile-time tag) selects the residual
        // variant so the plain epilogue keeps its registers and schedule.
        auto chunk = [&](int jj, auto res_tag) {
          constexpr bool RES = decltype(res_tag)::value;
          // Residual quads of this chunk (rows rq*4 + lane/8, 16-byte column
          // chunk lane%8): all eight loads issued before the TMEM load so
          // their latency overlaps it instead of serialising the store loop
          // (measured: residual layers ran 3x slower than the same shape
          // without a residual).
          [[maybe_unused]] float4 rv[8];
          if constexpr (RES) {
            if (jj + 1 < BN / 32) prefetch_res(jj + 1);
            const int nc = w.n_base + jj * 32 + (lane & 7) * 4;
#pragma unroll
            for (int rq = 0; rq < 8; ++rq) {
              const unsigned long long rp = fin_res[rq * 4 + (lane >> 3)];
              const float* rr = reinterpret_cast<const float*>(rp);
              const bool ok = rr && nc + 3 < p.N && (reinterpret_cast<uintptr_t>(rr + nc) & 15) == 0;
              rv[rq] = ok ? __ldg(reinterpret_cast<const float4*>(rr + nc)) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
          }
          const bool ctr = etr && j == 0 && jj < 2;
          if (ctr) p.trace[3300 + jj * 8 + 0] = gtime();
          uint32_t v[32];
          ptx::tmem_ld32(tbase + jj * 32, v);
          ptx::tmem_ld_wait();
          if (ctr) p.trace[3300 + jj * 8 + 1] = gtime() + (v[31] & 1);
          if (jj == BN / 32 - 1) {
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&acc_empty[acc]);  // TMEM buffer free for unit j + kAcc
          }
          const int n0 = w.n_base + jj * 32;
          if (n0 >= p.N) return;  // warp-uniform
#pragma unroll
          for (int q = 0; q < 8; ++q)
            ptx::sts128(stage + lane * 128 + ((q ^ (lane & 7)) << 4),
                        make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                                    __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3])));
          __syncwarp();
          if (ctr) p.trace[3300 + jj * 8 + 2] = gtime();
          const int cq = lane & 7;          // 16-byte chunk of the row segment
          const int nc = n0 + cq * 4;       // first column of the chunk
          const bool col_ok = nc < p.N;
          const bool full4 = nc + 3 < p.N;
          // Zero past N (the prefetch stored 0 there), so no test is needed.
          const float4 b4 = *reinterpret_cast<const float4*>(bias_st + jj * 32 + cq * 4);
          if (fast) {
            const float* st = reinterpret_cast<const float*>(smem + S::kStagingOffset + ew * 32 * 128);
            // Rows in batches of RB: all staging / row-pointer loads of a
            // batch are issued before the first use, so their shared-memory
            // latencies overlap (one dependent LDS chain per row cost ~60
            // cycles x 8 rows per chunk before). The activation is a runtime
            // clamp (one code copy instead of one per activation kind).
            const float lo = p.relu ? 0.f : -INFINITY, hi = p.relu == 2 ? 6.f : INFINITY;
            constexpr int RB = RES ? 4 : 8;
            if (ctr) p.trace[3300 + jj * 8 + 3] = gtime();
#pragma unroll
            for (int g = 0; g < 8; g += RB) {
              float4 x[RB];
              unsigned long long o[RB];
#pragma unroll
              for (int i = 0; i < RB; ++i) {
                const int rl = (g + i) * 4 + (lane >> 3);
                x[i] = *reinterpret_cast<const float4*>(st + rl * 32 + ((cq ^ (rl & 7)) << 2));
                o[i] = fin_out[rl];
              }
#pragma unroll
              for (int i = 0; i < RB; ++i) {
                float4& y = x[i];
                y.x += b4.x; y.y += b4.y; y.z += b4.z; y.w += b4.w;
                if constexpr (RES) {
                  y.x += rv[g + i].x; y.y += rv[g + i].y; y.z += rv[g + i].z; y.w += rv[g + i].w;
                }
                y.x = fminf(fmaxf(y.x, lo), hi); y.y = fminf(fmaxf(y.y, lo), hi);
                y.z = fminf(fmaxf(y.z, lo), hi); y.w = fminf(fmaxf(y.w, lo), hi);
                if (p.round_out) {
                  y.x = ptx::round_tf32(y.x); y.y = ptx::round_tf32(y.y);
                  y.z = ptx::round_tf32(y.z); y.w = ptx::round_tf32(y.w);
                }
              }
#pragma unroll
              for (int i = 0; i < RB; ++i)
                if (o[i] && col_ok) ptx::stg128(reinterpret_cast<float*>(o[i]) + nc, x[i]);
            }
            __syncwarp();
            if (ctr) p.trace[3300 + jj * 8 + 4] = gtime();
            return;
          }
          auto store_row = [&](int rq, const float4& r4) {
            const int rl = rq * 4 + (lane >> 3);  // row inside the warp's 32
            const unsigned long long op = fin_out[rl];
            const unsigned long long rp = fin_res[rl];
            if (!op || !col_ok) return;
            float4 x = ptx::lds128(stage + rl * 128 + ((cq ^ (rl & 7)) << 4));
            float* dst = reinterpret_cast<float*>(op) + nc;
            const float* rr = reinterpret_cast<const float*>(rp);
            const bool vec = full4 && ((reinterpret_cast<uintptr_t>(dst) | (rr ? reinterpret_cast<uintptr_t>(rr + nc) : 0)) & 15) == 0;
            if (vec) {
              x.x += b4.x; x.y += b4.y; x.z += b4.z; x.w += b4.w;
              if (rr) {  // r4 was prefetched with the same rows / columns / alignment test
                x.x += r4.x; x.y += r4.y; x.z += r4.z; x.w += r4.w;
              }
              if (p.relu == 1) {
                x.x = fmaxf(x.x, 0.f); x.y = fmaxf(x.y, 0.f); x.z = fmaxf(x.z, 0.f); x.w = fmaxf(x.w, 0.f);
              } else if (p.relu == 2) {
                x.x = fminf(fmaxf(x.x, 0.f), 6.f); x.y = fminf(fmaxf(x.y, 0.f), 6.f);
                x.z = fminf(fmaxf(x.z, 0.f), 6.f); x.w = fminf(fmaxf(x.w, 0.f), 6.f);
              }
              if (p.round_out) {
                x.x = ptx::round_tf32(x.x); x.y = ptx::round_tf32(x.y);
                x.z = ptx::round_tf32(x.z); x.w = ptx::round_tf32(x.w);
              }
              *reinterpret_cast<float4*>(dst) = x;
            } else {
              const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
              for (int q = 0; q < 4; ++q)
                if (nc + q < p.N) dst[q] = epilogue_op(p, xs[q], nc + q, rr);
            }
          };
          if constexpr (RES) {
#pragma unroll
            for (int rq = 0; rq < 8; ++rq) store_row(rq, rv[rq]);
          } else {
            const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
            for (int rq = 0; rq < 8; ++rq) store_row(rq, zero);
          }
          __syncwarp();
        };
        if (p.res_ptrs) {
#pragma unroll 1
          for (int jj = 0; jj < BN / 32; ++jj) chunk(jj, std::true_type{});
        } else {
#pragma unroll 1
          for (int jj = 0; jj < BN / 32; ++jj) {
            chunk(jj, std::false_type{});
            if (etr && jj < 6) p.trace[3072 + j * 8 + 2 + jj] = gtime();
          }
        }
      } else {
        // Split-K (cluster launch, CTA rank = split, one unit per CTA): park
        // this split's raw partial tile in OWN shared memory -- the A ring,
        // idle once the unit's MMAs are done -- as [row][BN] fp32 with the
        // 16-byte chunks XOR-swizzled by row (conflict-free stores). The
        // cluster reduces the tile over DSMEM after the role loops (below).
        const uint32_t prow = smem_base + static_cast<uint32_t>(row * BN * 4);
#pragma unroll 1
        for (int jj = 0; jj < BN / 32; ++jj) {
          uint32_t v[32];
          ptx::tmem_ld32(tbase + jj * 32, v);
          ptx::tmem_ld_wait();
          if (jj == BN / 32 - 1) {
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&acc_empty[acc]);
          }
#pragma unroll
          for (int q = 0; q < 8; ++q)
            ptx::sts128(prow + static_cast<uint32_t>(((jj * 8 + q) ^ (row & 7)) << 4),
                        make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                                    __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3])));
        }
      }
    }
  } else if (warp == 8) {
    // ---------------------------------------------------------- MMA issue
    constexpr uint32_t idesc = ptx::make_idesc(BF16 ? 1 : 2, kBM, BN);
    const uint32_t a_tmem0 = tmem_base + S::kTA0;
    int it = 0, j = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      BS_UNIT_PROBLEM(u)
      const Unit w = unit_of(p, lu, BN, KT);
      const int acc = j % S::kAcc;
      if (j >= S::kAcc) ptx::mbar_wait(&acc_empty[acc], ((j / S::kAcc) - 1) & 1);
      ptx::tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kt = w.kt0; kt < w.kt1; ++kt, ++it) {
        const int sa = it % TA, sb = it % NB;
        if constexpr (S::HIS) {
          // A_hi = the raw stage read as TF32 (SS form), as soon as the
          // gather and the weights have landed; then A_lo from TMEM (TS).
          ptx::mbar_wait(&ra_full[sa], (it / TA) & 1);
          ptx::mbar_wait(&b_full[sb], (it / NB) & 1);
          ptx::fence_proxy_async_smem();  // cp.async (generic proxy) data -> tensor core (async proxy)
          ptx::tc_fence_after();
          if (p.trace && lane == 0 && blockIdx.x == 0 && it < 48) p.trace[1024 + it * 5 + 4] = gtime();
          const uint64_t a_desc = ptx::sw128_kmajor_desc(smem_base + sa * S::kABytes);
          const uint64_t b_desc = ptx::sw128_kmajor_desc(smem_base + S::kBOffset + sb * S::kBBytes);
          if (ptx::elect_one()) {
#pragma unroll
            for (int k = 0; k < kBK / 8; ++k)
              ptx::mma_tf32(d_tmem, a_desc + 2 * k, b_desc + 2 * k, idesc, (kt != w.kt0) || k != 0);
          }
          __syncwarp();
          ptx::mbar_wait(&ta_full[sa], (it / TA) & 1);
          ptx::tc_fence_after();
          if (ptx::elect_one()) {
            const uint32_t a_slot = a_tmem0 + sa * S::kACols;
#pragma unroll
            for (int k = 0; k < kBK / 8; ++k) ptx::mma_tf32_ts(d_tmem, a_slot + 8 * k, b_desc + 2 * k, idesc, 1);
            ptx::mma_commit(&ra_empty[sa]);  // frees raw stage, B stage and A_lo slot
            if (kt == w.kt1 - 1) ptx::mma_commit(&acc_full[acc]);
          }
          __syncwarp();
          continue;
        }
        ptx::mbar_wait(&ta_full[sa], (it / TA) & 1);
        if (p.trace && lane == 0 && blockIdx.x == 0 && it < 48) p.trace[2048 + it * 4 + 0] = gtime();
        ptx::mbar_wait(&b_full[sb], (it / NB) & 1);
        if (p.trace && lane == 0 && blockIdx.x == 0 && it < 48) p.trace[2048 + it * 4 + 1] = gtime();
        ptx::tc_fence_after();
        if (p.trace && lane == 0 && blockIdx.x == 0 && it < 48) p.trace[1024 + it * 5 + 4] = gtime();
        if (ptx::elect_one()) {
          const uint32_t a_slot = a_tmem0 + sa * S::kACols;
          const uint32_t b_addr = smem_base + S::kBOffset + sb * S::kBBytes;
          if constexpr (BF16) {
            // K = 16 bf16 per MMA: A 8 TMEM columns, B +32 bytes in the 64-byte row.
            const uint64_t b_desc = ptx::sw64_kmajor_desc(b_addr);
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k)
              ptx::mma_bf16_ts(d_tmem, a_slot + 8 * k, b_desc + 2 * k, idesc, (kt != w.kt0) || k != 0);
          } else {
            const uint64_t b_desc = ptx::sw128_kmajor_desc(b_addr);
#pragma unroll
            for (int k = 0; k < kBK / 8; ++k) {
              // A: 8 TMEM columns per K=8 step; B: +32 bytes inside the swizzled row.
              ptx::mma_tf32_ts(d_tmem, a_slot + 8 * k, b_desc + 2 * k, idesc, (kt != w.kt0) || k != 0);
            }
          }
          ptx::mma_commit(&ta_empty[sa]);  // == b_empty[sb]
          if (kt == w.kt1 - 1) ptx::mma_commit(&acc_full[acc]);
        }
        __syncwarp();
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------ B TMA
    if (lane == 0) {
      int it = 0;
      if (p.trace && blockIdx.x == 0) p.trace[3400 + 3] = gtime();
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        BS_UNIT_PROBLEM(u)
        const Unit w = unit_of(p, lu, BN, KT);
        for (int kt = w.kt0; kt < w.kt1; ++kt, ++it) {
          const int s = it % NB;
          if (it >= NB) ptx::mbar_wait(&b_empty[s], ((it / NB) - 1) & 1);
          ptx::mbar_arrive_expect_tx(&b_full[s], S::kBBytes);
          ptx::tma_load_2d(smem_base + S::kBOffset + s * S::kBBytes, &p.wmap, kt * kBK, w.n_base, &b_full[s]);
          if (p.trace && blockIdx.x == 0 && it < 48) p.trace[1024 + it * 5 + 1] = gtime();
        }
      }
    }
    __syncwarp();
  } else if (warp >= 10 && warp < 14) {
    convert(0, 2, 320);
  } else if (warp >= 15 && warp < 19) {
    convert(1, 2, 480);
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (p.trace && threadIdx.x == 0) p.trace[8 + 4 * blockIdx.x + 3] = gtime();
  if (warp == 8) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem_base);
  }
  if (p.ksplits > 1) {
    // ------------------------------------------ split-K reduction over DSMEM
    // The ks CTAs of a cluster hold the ks K-splits of one tile (the
    // hardware co-schedules a cluster, so no CTA ever waits for one that is
    // not resident -- unlike a grid-wide spin, this cannot deadlock against
    // other work on the GPU). After the barrier every partial is visible;
    // CTA `rank` reduces rows [rank * 128 / ks, ...) in fixed split order
    // (deterministic), applies bias / residual / activation and writes them.
    // The second barrier keeps every CTA's shared memory alive until all
    // peers have read it.
    ptx::cluster_sync_all();
    const int rank = static_cast<int>(ptx::cluster_ctarank());
    BS_UNIT_PROBLEM(static_cast<int>(blockIdx.x))
    const Unit w = unit_of(p, lu, BN, KT);
    const int rows_per = (kBM + p.ksplits - 1) / p.ksplits;
    const int r_lo = rank * rows_per, r_hi = min(kBM, r_lo + rows_per);
    constexpr int kVec = BN / 4;  // 16-byte chunks per row
    for (int idx = threadIdx.x; idx < (r_hi - r_lo) * kVec; idx += blockDim.x) {
      const int rr = r_lo + idx / kVec;
      const int c4 = idx - (idx / kVec) * kVec;
      const int n0 = w.n_base + c4 * 4;
      int img, px;
      if (!row_pixel(p, w.mt, rr, img, px) || n0 >= p.N) continue;
      const uint32_t off = smem_base + static_cast<uint32_t>(rr * BN * 4 + ((c4 ^ (rr & 7)) << 4));
      float4 acc4 = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int sp = 0; sp < p.ksplits; ++sp) {
        const float4 x = ptx::ld_dsmem128(ptx::mapa_shared(off, static_cast<uint32_t>(sp)));
        acc4.x += x.x;
        acc4.y += x.y;
        acc4.z += x.z;
        acc4.w += x.w;
      }
      float* orow = p.out_ptrs[img] + p.out_off + static_cast<long>(px) * p.out_ldc;
      const float* rrow = p.res_ptrs ? p.res_ptrs[img] + p.res_off + static_cast<long>(px) * p.res_ldc : nullptr;
      const float vals[4] = {acc4.x, acc4.y, acc4.z, acc4.w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (n0 + q < p.N) orow[n0 + q] = epilogue_op(p, vals[q], n0 + q, rrow);
    }
    ptx::cluster_sync_all();
  }
}

}  // namespace conv_tc

// Narrow N tile for N output channels (the launcher may widen to 192 / 256,
// see conv_add_wide_map / conv_add_mid_map).
int conv_tile_n(int N);

// Tap-row mode eligibility (Cin 4 / 8 / 16 and at most one padded tap per
// filter row: the stems) and the matching weight layout out[N][KH * 32].
bool conv_tap_rows_eligible(int Cin, int KW);
void conv_tap_row_weights(const float* w, int N, int Kpad_src, int KH, int KW, int Cin, float* out);
// Encodes a weight tensor map for w ([N][Kpad] floats) and the tile conv_tile_n(N).
bool encode_weight_map(CUtensorMap* map, const float* w, int N, int Kpad, int box_n = 0);
// The same for a bf16 copy of the weights (BF16 precision): box {32, BN},
// 64-byte swizzle.
bool encode_weight_map_bf16(CUtensorMap* map, const void* w_bf16, int N, int Kpad, int box_n = 0);
// Offers the launcher 128 x 256 tiles (weights map with box_n = 256; the map
// must outlive the launch call).
void conv_add_wide_map(ConvParams& p, const CUtensorMap& wide);
// Offers the launcher 128 x 192 / 128 x 160 tiles (weights maps with
// box_n = 192 / 160).
void conv_add_mid_map(ConvParams& p, const CUtensorMap& mid);
void conv_add_mid160_map(ConvParams& p, const CUtensorMap& mid160);
// Grouped launch of two independent convs (no data flow between them; same
// precision; cp.async gather path, no split-K): one persistent grid walks the
// units of a, then of b, with a common tile width.
// force: launch grouped even where the launcher's rules would decline (the
// executor's autotune measured the group faster at this batch).
// ks > 0 (with force): split both convs ks ways (cluster of ks CTAs per tile;
// clamped to the shorter K loop).
cudaError_t launch_conv_tc_group(ConvParams a, ConvParams b, cudaStream_t stream, bool force = false, int ks = 1);
// Host-side launcher: chooses the K split (a split-K launch is a cluster
// launch, one CTA per split, reduced over DSMEM) and the grid
// (p.wmap must be encoded for conv_tile_n(p.N)).
cudaError_t launch_conv_tc(ConvParams p, cudaStream_t stream);

}  // namespace bs200
