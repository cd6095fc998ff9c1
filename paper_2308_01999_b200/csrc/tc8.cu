// tc8.cu — k = 4/5-qubit dense gates (optionally with the fold fuser's
// outside-coupled pre-phase) on the 5th-generation tensor cores, complex64,
// through EXACT 8-bit integer products (tcgen05.mma kind::i8, int32 accumulate).
//
// Replaces apply_dense_bits (reference statevec.py:44-60) for the same windows
// as tc.cu (the bf16-limb kernel, kept for A/B via DSV_TC8=0).  Same dataflow
// (persistent CTA per SM, two 128-thread groups on alternate 128-group tiles,
// cp.async rings, A operand in TMEM, gate operand in SW128 shared memory, one
// thread issues the MMAs and commits to an mbarrier); what changes is the
// arithmetic, which is cheaper on every side:
//
//   * A (the amplitudes): a row of the tile is scaled by its own power of two
//     so |y| < 2^22 and rounded to an integer I with ONE fma against the magic
//     1.5 * 2^23 (the float's low mantissa bits are then I + 2^22).  One
//     integer add turns the bits into I' = I + 0x8080, whose bytes are the
//     balanced base-256 digits of I: a0 = byte0 ^ 0x80, a1 = byte1 ^ 0x80
//     (in [-128, 127]), a2 = byte2 (in [-64, 64]); byte permutes pack four
//     values' digits per 32-bit TMEM column.  ~4 integer/fp ops per value
//     instead of 9 fp ops + packing for three bf16 limbs.
//   * B (the gate's real embedding) is split the same way on the host:
//     X = B 2^(23 - e_b) = b2 2^16 + b1 2^8 + b0, digits in [-128, 127].
//   * products of digit weight >= 2^16 (a2 b2, a2 b1, a1 b2, a2 b0, a1 b1, a0 b2)
//     land in three int32 accumulators hi / mid / lo (exact: |acc| < 2^22);
//     3 MMAs per 32-wide K step (N = 3, 2, 1 x 2^(k+1)) instead of 10 bf16 ones,
//     at twice the bf16 tensor rate.  The dropped products (a1 b0, a0 b1, a0 b0)
//     are zero-mean and below 2^-22 of the row's scale: measured (U then U^dagger,
//     tools/tc_precision.py) 1.8e-6 max relative error per round vs 4.2e-7 for
//     the fp32 CUDA-core kernels and 2.4e-7 for tc.cu — inside the c64 bound
//     (1e-5 absolute, fidelity 1 - 1e-6) but not fp32-identical; DSV_TC8=0
//     selects tc.cu where that matters.
//   * the accumulators start at the float bits of 1.5 * 2^23 (tcgen05.st of a
//     constant), so each int32 sum reads back directly as the float
//     1.5 * 2^23 + acc: the epilogue is 1 add + 3 fma per value, no conversion.
#include <cmath>
#include <cstring>

#include "common.cuh"
#include "launch.h"
#include "tcgen05.cuh"

namespace dsv {

using namespace tcx;

#ifndef DSV_TC8_FILL
#define DSV_TC8_FILL 0  // accumulator start value: 0 per-thread tcgen05.st, 1/2 tcgen05.cp (diagnostics)
#endif
template <int K>
struct Tc8P {
  Geom g;                 // groups (amplitude index space, holes = targets + controls)
  uint64_t ntiles;        // g.nwork / 128
  int nnib;               // phase-table nibbles (0: plain dense)
  int e_b;                // gate scale: |B| < 2^e_b, X = B 2^(23 - e_b)
  int emin, emax;         // row-exponent clamp (keeps every power of two normal)
  int coop;               // phase uniform over a tile's 128 rows: computed once per tile
  int nnib_row;           // leading nibbles that vary over the rows (the rest: tile-uniform sums)
  int nib_shift[16];      // amplitude-index shift of nibble c
  int tshift;             // member j at offset j << tshift (contiguous targets), else -1: offs[]
  int jpos;               // row-pair copies: thread-index bit that selects the member parity (see issue())
  uint64_t offs[1 << K];  // member offsets (amplitudes)
  float4 ctab[kTcMaxNib * 16 * 2];  // tile-uniform phase table (constant bank, broadcast reads)
  int tma_shift[5];       // kTcTma: tile coordinate of map dim q = (tile >> shift[q]) & mask[q]
  uint32_t tma_mask[5];
  int nrb;                // row-phase bits (<= 3): per tile, 2^nrb vectors = tile vector x R_v
  int rb_bit[3];
  const float2* rvec;     // [2^nrb][D] launch-constant row phase factors
  int pairswap;           // plain row-pair windows: lanes swap one member and store 16 bytes (A/B; default 8-byte rows)
};

template <int K>
struct Tc8Layout {
  static constexpr int D = 1 << K;
  static constexpr int N0 = 2 * D;                // real outputs = real inputs (GEMM K)
  static constexpr int KSTEPS = N0 / 32;          // MMA K = 32 (8-bit)
  static constexpr int B_BYTES = 3 * N0 * 128;    // [b2 | b1 | b0] rows of 128 B (K <= 64 used)
  static constexpr int BAR = B_BYTES;             // 2 mbarriers + TMEM slot
  static constexpr int MAG = BAR + 256;           // 128 x 32 B of the accumulator start value (tcgen05.cp source)
  static constexpr int TMABAR = BAR + 64;         // kTcTma: full[grp][stage] mbarriers (<= 2 x 8)
  static constexpr int PBUF = MAG + (DSV_TC8_FILL ? 4096 : 0);  // tile-uniform phases: [group][2][D] float2
  static constexpr int PBV = 8;                   // phase vectors per tile slot (2^nrb, nrb <= 3)
  static constexpr int PBD = D + 1;               // vector stride (float2): rows of one warp read 8 vectors
                                                  // at once, the pad puts them in different banks
  static constexpr int RING = PBUF + 2 * 2 * PBV * PBD * 8;
  static constexpr int STAGE = 128 * D * 8;
  static constexpr int SMEM_MAX = 227 * 1024 - 1024;
  static constexpr int NS_FIT = (SMEM_MAX - RING) / (2 * STAGE);
  static constexpr int NSTAGE = NS_FIT > 6 ? 6 : NS_FIT;
  static_assert(NSTAGE >= 3, "ring must hold three tiles per group");
  static_assert(N0 <= 64, "B rows are one 128-byte K block");
  static constexpr int BYTES = RING + 2 * NSTAGE * STAGE;
  // TMEM per group (256 columns): A digits a2, a1, a0 (4 per column), then hi | mid | lo
  static constexpr int ACOLS = N0 / 4;
  static constexpr int T_A2 = 0, T_A1 = ACOLS, T_A0 = 2 * ACOLS;
  static constexpr int T_HI = 64, T_MID = T_HI + N0, T_LO = T_HI + 2 * N0;
  static_assert(3 * ACOLS <= T_HI && T_LO + N0 <= 256, "TMEM plan");
};

constexpr uint32_t kAccInit = 0x4B400000u;           // float bits of 1.5 * 2^23
constexpr uint32_t kDigitOff = 0x8080u - 0x4B400000u;  // float bits of M + I -> I + 0x8080

//   [hi | mid | lo] += a2 [b2 | b1 | b0];  [mid | lo] += a1 [b2 | b1];  lo += a0 b2
template <int K, int GRP>
__device__ __forceinline__ void issue_mma8(uint32_t sbase) {
  using L = Tc8Layout<K>;
  constexpr uint32_t T0 = GRP * 256;
  constexpr uint32_t ID3 = idesc_i8<3 * L::N0, 1, 1>(), ID2 = idesc_i8<2 * L::N0, 1, 1>(),
                     ID1 = idesc_i8<L::N0, 1, 1>();
#pragma unroll
  for (int s = 0; s < L::KSTEPS; ++s) {
    const uint64_t bd = sw128_desc(sbase + s * 32);
    mma_ts_i8(T0 + L::T_HI, T0 + L::T_A2 + s * 8, bd, ID3, 1u);
    mma_ts_i8(T0 + L::T_MID, T0 + L::T_A1 + s * 8, bd, ID2, 1u);
    mma_ts_i8(T0 + L::T_LO, T0 + L::T_A0 + s * 8, bd, ID1, 1u);
  }
}

template <int K, bool PHASED, int MODE>
__global__ void __launch_bounds__(256, 1)
k_dense_tc8(const __grid_constant__ Tc8P<K> p, const __grid_constant__ CUtensorMap tmap,
            const uint4* __restrict__ bmat, const float4* __restrict__ tab, float2* __restrict__ sv) {
  using L = Tc8Layout<K>;
  constexpr bool TMA = MODE == kTcTma;  // loads by tensor map; otherwise as kTcPair
  constexpr bool PAIR = MODE == kTcPair || TMA;
  constexpr bool LOWT = MODE == kTcLow;
  constexpr bool ROW2 = MODE == kTcRow2;  // stage layout [member pair m][row] x 16 B
  constexpr int D = L::D;
  constexpr int N0 = L::N0;
  constexpr int S = L::NSTAGE;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t raw_base = smem_u32(smem_raw);
  const uint32_t sbase = (raw_base + 1023u) & ~1023u;
  unsigned char* sm = smem_raw + (sbase - raw_base);
  const int tid = threadIdx.x;
  // warp / group index through a lane-0 shuffle: provably warp-uniform, so the
  // TMEM addresses derived from it live in uniform registers (ncu showed ~2.5
  // R2UR per amplitude moving them there for every tcgen05.ld / st)
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int grp = warp >> 2;
  const int row = tid & 127;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + L::BAR + 16);
  const uint32_t bar = sbase + L::BAR + 8 * grp;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid < 2) reinterpret_cast<uint32_t*>(sm + L::BAR + 32)[tid] = kAccInit;
  if (tid == 32) {
    mbar_init(sbase + L::BAR, 1);
    mbar_init(sbase + L::BAR + 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (TMA && row == 0) {  // each group's TMA issuer owns its stage barriers (initialised before its first load)
    for (int q = 0; q < S; ++q) mbar_init(sbase + L::TMABAR + 8 * (grp * S + q), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (TMA && tid == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
  static_assert(!TMA || 2 * S * 8 <= 192, "TMA barriers fit the barrier block");
  // gate digits, host layout [3 N0 rows][8 x 16 B] -> 128-byte swizzled rows
  for (int i = tid; i < 3 * N0 * 8; i += 256) {
    const int r = i / 8, c16 = i % 8;
    *reinterpret_cast<uint4*>(sm + r * 128 + ((c16 ^ (r & 7)) << 4)) = bmat[i];
  }
  if (DSV_TC8_FILL)
    for (int i = tid; i < 1024; i += 256) reinterpret_cast<uint32_t*>(sm + L::MAG)[i] = kAccInit;

  const uint64_t step = gridDim.x;
  auto tile_of = [&](int i) { return uint64_t(blockIdx.x) + (2 * uint64_t(i) + grp) * step; };
  const uint64_t e0 = expand(p.g, 0);
  const uint64_t rowoff = expand(p.g, row) ^ e0;
  // row-pair copies: thread-index bit jpos picks the member parity, the other
  // six bits the row pair.  jpos = (lowest target - 1) capped at 6, so a
  // warp's 16-byte copies cover whole contiguous runs (with the lowest target
  // at bit 1 adjacent threads take the two members of one 32-byte sector).
  const int prow = 2 * ((row & ((1 << p.jpos) - 1)) | ((row >> (p.jpos + 1)) << p.jpos));
  const int jpar = (row >> p.jpos) & 1;
  const uint64_t prowoff = expand(p.g, prow) ^ e0;
  int vrow = 0;  // this row's value of the row-phase bits (rows are the same index bits in every tile)
  for (int q = 0; q < p.nrb; ++q) vrow |= int((rowoff >> p.rb_bit[q]) & 1u) << q;
  auto issue = [&](int i) -> uint64_t {
    const uint64_t tl = tile_of(i);
    uint64_t tb = 0;
    if (tl < p.ntiles) {
      tb = expand(p.g, tl * 128);
      const uint32_t st0 = sbase + L::RING + ((grp * S) + (i % S)) * L::STAGE;
      if constexpr (TMA) {
        if (row == 0) {  // the whole 128-row x 2^k-member tile in one bulk tensor load
          int c[5];
#pragma unroll
          for (int q = 0; q < 5; ++q) c[q] = int(uint32_t(tl >> p.tma_shift[q]) & p.tma_mask[q]);
          const uint32_t fb = sbase + L::TMABAR + 8 * (grp * S + (i % S));
          mbar_expect_tx(fb, L::STAGE);
          tma_load_5d(st0, &tmap, c, fb);
        }
      } else if constexpr (LOWT) {
#pragma unroll
        for (int m = 0; m < D / 2; ++m) {
          const int q = row + 128 * m;
          const int r = q / (D / 2), c = q % (D / 2);
          cp_async16(st0 + r * (D * 8) + ((c ^ (r & 7)) << 4), sv + tb + 2 * q);
        }
      } else if constexpr (ROW2) {  // this row's member pairs: 16-byte copies, lanes 16 bytes apart
        const uint64_t b = tb | rowoff;
#pragma unroll
        for (int m = 0; m < D / 2; ++m) cp_async16(st0 + m * 2048 + row * 16, sv + b + p.offs[2 * m]);
      } else if constexpr (PAIR) {
        const uint64_t b = tb | prowoff;
        if (p.tshift >= 0) {  // member j at j << tshift: one strided pointer
          const float2* src = sv + b + (uint64_t(jpar) << p.tshift);
          const uint64_t stride = uint64_t(2) << p.tshift;
#pragma unroll
          for (int jj = 0; jj < D / 2; ++jj) cp_async16(st0 + prow * 8 + (2 * jj + jpar) * 1024, src + jj * stride);
        } else {
#pragma unroll
          for (int jj = 0; jj < D / 2; ++jj) {
            const uint64_t o = jpar ? p.offs[2 * jj + 1] : p.offs[2 * jj];
            cp_async16(st0 + prow * 8 + (2 * jj + jpar) * 1024, sv + b + o);
          }
        }
      } else {
        const uint64_t b = tb | rowoff;
        if (p.tshift >= 0) {
          const float2* src = sv + b;
          const uint64_t stride = uint64_t(1) << p.tshift;
#pragma unroll
          for (int j = 0; j < D; ++j) cp_async8(st0 + row * 8 + j * 1024, src + j * stride);
        } else {
#pragma unroll
          for (int j = 0; j < D; ++j) cp_async8(st0 + row * 8 + j * 1024, sv + b + p.offs[j]);
        }
      }
    }
    cp_async_commit();
    return tb;
  };
  float2* Pb = reinterpret_cast<float2*>(sm + L::PBUF) + grp * 2 * L::PBV * L::PBD;
  auto coop_phase = [&](int i, uint64_t tb) {
    const int j = row - (128 - D);
    if (PHASED && !p.coop && j == 0 && tile_of(i) < p.ntiles) {
      float a[8];
#pragma unroll
      for (int s = 0; s < 8; ++s) a[s] = 0.f;
#pragma unroll
      for (int c = 0; c < kTcMaxNib; ++c) {
        if (c >= p.nnib_row && c < p.nnib) {
          const int r = (c * 16 + int((tb >> p.nib_shift[c]) & 15u)) * 2;
          const float4 x = p.ctab[r], y = p.ctab[r + 1];
          a[0] += x.x; a[1] += x.y; a[2] += x.z; a[3] += x.w;
          a[4] += y.x; a[5] += y.y; a[6] += y.z; a[7] += y.w;
        }
      }
      float4* hb = reinterpret_cast<float4*>(Pb + (i & 1) * L::PBV * L::PBD);
      hb[0] = make_float4(a[0], a[1], a[2], a[3]);
      hb[1] = make_float4(a[4], a[5], a[6], a[7]);
    }
    if (PHASED && p.coop && j >= 0 && tile_of(i) < p.ntiles) {
      float a[8];
#pragma unroll
      for (int s = 0; s < 8; ++s) a[s] = 0.f;
#pragma unroll
      for (int c = 0; c < kTcMaxNib; ++c) {
        if (c < p.nnib) {
          const int r = (c * 16 + int((tb >> p.nib_shift[c]) & 15u)) * 2;
          const float4 x = p.ctab[r], y = p.ctab[r + 1];
          a[0] += x.x; a[1] += x.y; a[2] += x.z; a[3] += x.w;
          a[4] += y.x; a[5] += y.y; a[6] += y.z; a[7] += y.w;
        }
      }
      float ang = a[K];
#pragma unroll
      for (int m = 0; m < K; ++m) ang += ((j >> m) & 1) ? a[m] : 0.f;
      float sn, cs;
      sincos_unit(ang, &sn, &cs);
      if (p.nrb == 0) {
        Pb[(i & 1) * L::PBV * L::PBD + j] = make_float2(cs, sn);
      } else {  // one vector per value of the row-phase bits: tile vector x launch-constant row factor
        for (int v = 0; v < (1 << p.nrb); ++v) {
          const float2 r = __ldg(p.rvec + v * D + j);
          Pb[((i & 1) * L::PBV + v) * L::PBD + j] = make_float2(cs * r.x - sn * r.y, cs * r.y + sn * r.x);
        }
      }
    }
  };
  uint64_t tq[S - 1];
#pragma unroll
  for (int s = 0; s < S - 1; ++s) tq[s] = issue(s);
  coop_phase(0, tq[0]);
  coop_phase(1, tq[1]);
  // per-row phase slots (row-varying nibbles) of this thread's row in the
  // NEXT tile, loaded one iteration ahead so the table latency stays off the
  // critical path
  float ra[8];
  auto row_angles = [&](uint64_t b) {
#pragma unroll
    for (int s = 0; s < 8; ++s) ra[s] = 0.f;
#pragma unroll
    for (int c = 0; c < kTcMaxNib; ++c) {
      if (c < p.nnib_row) {
        const int r = (c * 16 + int((b >> p.nib_shift[c]) & 15u)) * 2;
        const float4 x = __ldg(tab + r), y = __ldg(tab + r + 1);
        ra[0] += x.x; ra[1] += x.y; ra[2] += x.z; ra[3] += x.w;
        ra[4] += y.x; ra[5] += y.y; ra[6] += y.z; ra[7] += y.w;
      }
    }
  };
  if (PHASED && !p.coop) row_angles(tq[0] | rowoff);
  cp_async_wait<S - 2>();

  const uint32_t tlane = uint32_t(grp * 256) + (uint32_t((warp & 3) * 32) << 16);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  fence_before();
  __syncthreads();
  fence_after();
  // read only after the barrier: warp 0's tcgen05.alloc wrote the slot
  // (compute-sanitizer racecheck flagged the earlier pre-barrier read)
  if (*tmem_slot != 0u) __trap();  // whole-TMEM allocation starts at lane 0, column 0

  // out = scale (hi 2^16 + mid 2^8 + lo): the accumulators read back as
  // M + acc (M = 1.5 * 2^23); t2 = V + 257 M, removed by the last fma
  auto combine = [](float h, float m, float l, float scale, float cm) {
    const float t1 = __fmaf_rn(__fadd_rn(h, -kMagic), 256.f, m);
    return __fmaf_rn(__fmaf_rn(t1, 256.f, l), scale, cm);
  };
  auto epilogue = [&](uint64_t b, float scale, float cm) {
#pragma unroll
    for (int h = 0; h < N0 / 32; ++h) {
      float ch[32], cmid[32], cl[32];
      tmem_ld32(tlane + uint32_t(L::T_HI + h * 32), ch);
      tmem_ld32(tlane + uint32_t(L::T_MID + h * 32), cmid);
      tmem_ld32(tlane + uint32_t(L::T_LO + h * 32), cl);
      auto val = [&](int c) { return combine(ch[c], cmid[c], cl[c], scale, cm); };
      if constexpr (LOWT) {  // this row is contiguous: 32-byte stores, one full sector per lane
#pragma unroll
        for (int i = 0; i < 4; ++i)
          stcs32(sv + b + h * 16 + 4 * i, val(8 * i), val(8 * i + 1), val(8 * i + 2), val(8 * i + 3), val(8 * i + 4),
                 val(8 * i + 5), val(8 * i + 6), val(8 * i + 7));
      } else if constexpr (ROW2) {  // member pairs (2m, 2m+1) are adjacent amplitudes: 16-byte stores
#pragma unroll
        for (int i = 0; i < 8; ++i)
          __stcs(reinterpret_cast<float4*>(sv + b + p.offs[h * 16 + 2 * i]),
                 make_float4(val(4 * i), val(4 * i + 1), val(4 * i + 2), val(4 * i + 3)));
      } else if (PAIR && !PHASED && p.pairswap) {
        // lanes 2t', 2t'+1 hold adjacent amplitudes: swap one member per pair
        // and store 16 bytes each (even lane: member 2q of both rows, odd: 2q+1)
        const bool odd = row & 1;
        const uint64_t be = b - (odd ? 1 : 0);
        float2* dst = sv + be + (p.tshift >= 0 ? (uint64_t(h * 16 + (odd ? 1 : 0)) << p.tshift) : 0);
        const uint64_t stride = p.tshift >= 0 ? (uint64_t(2) << p.tshift) : 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float o[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) o[c] = val(4 * q + c);
          const float sx = odd ? o[0] : o[2], sy = odd ? o[1] : o[3];
          const float rx = __shfl_xor_sync(0xffffffffu, sx, 1), ry = __shfl_xor_sync(0xffffffffu, sy, 1);
          const float4 w = odd ? make_float4(rx, ry, o[2], o[3]) : make_float4(o[0], o[1], rx, ry);
          if (p.tshift >= 0) {
            __stcs(reinterpret_cast<float4*>(dst + q * stride), w);
          } else {
            const uint64_t oj = odd ? p.offs[h * 16 + 2 * q + 1] : p.offs[h * 16 + 2 * q];
            __stcs(reinterpret_cast<float4*>(sv + be + oj), w);
          }
        }
      } else {
        // 8-byte stores of this row's members: with index bit 0 free (PAIR)
        // adjacent lanes hold adjacent amplitudes, so each warp store is one
        // contiguous 256-byte run without any lane exchange (measured faster
        // than the 16-byte pair exchange for the phased windows, slower for
        // plain ones)
        if (p.tshift >= 0) {
          float2* dst = sv + b + (uint64_t(h * 16) << p.tshift);
          const uint64_t stride = uint64_t(1) << p.tshift;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            __stcs(dst, make_float2(val(2 * i), val(2 * i + 1)));
            dst += stride;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) __stcs(sv + b + p.offs[h * 16 + i], make_float2(val(2 * i), val(2 * i + 1)));
        }
      }
    }
  };

  // (loaded from shared memory so the compiler keeps them in registers rather
  // than re-materialising eight immediates for every store)
  uint32_t mg[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) mg[i] = reinterpret_cast<const uint32_t*>(sm + L::BAR + 32)[i & 1];
  uint64_t prev_base = 0;
  float prev_scale = 0.f, prev_cm = 0.f;
  int it = 0, stage = 0;
#pragma unroll 1
  for (;; ++it) {
    const uint64_t tile = tile_of(it);
    if (tile >= p.ntiles) break;
    const uint64_t tb_new = issue(it + S - 1);
    const uint64_t base = tq[0] | rowoff;
#pragma unroll
    for (int s = 0; s + 1 < S - 1; ++s) tq[s] = tq[s + 1];
    tq[S - 2] = tb_new;
    if constexpr (TMA) mbar_wait(sbase + L::TMABAR + 8 * (grp * S + stage), uint32_t(it / S) & 1u);
    const unsigned char* stg = sm + L::RING + (grp * S + stage) * L::STAGE;
    stage = stage + 1 == S ? 0 : stage + 1;
    float2 v[D];
    if constexpr (ROW2) {
#pragma unroll
      for (int m = 0; m < D / 2; ++m) {
        const float4 x = *reinterpret_cast<const float4*>(stg + m * 2048 + row * 16);
        v[2 * m] = make_float2(x.x, x.y);
        v[2 * m + 1] = make_float2(x.z, x.w);
      }
    } else if constexpr (LOWT) {
#pragma unroll
      for (int c = 0; c < D / 2; ++c) {
        const float4 x = *reinterpret_cast<const float4*>(stg + row * (D * 8) + ((c ^ (row & 7)) << 4));
        v[2 * c] = make_float2(x.x, x.y);
        v[2 * c + 1] = make_float2(x.z, x.w);
      }
    } else {
      const float2* raw = reinterpret_cast<const float2*>(stg) + row;
#pragma unroll
      for (int j = 0; j < D; ++j) v[j] = raw[j * 128];
    }
    if constexpr (PHASED) {
      if (p.coop) {
        const float2* P = Pb + ((it & 1) * L::PBV + vrow) * L::PBD;
#pragma unroll
        for (int j = 0; j < D; ++j) {
          const float2 x = v[j], f = P[j];
          v[j] = make_float2(x.x * f.x - x.y * f.y, x.x * f.y + x.y * f.x);
        }
      } else {
        float a[8];
        const float4* hb = reinterpret_cast<const float4*>(Pb + (it & 1) * L::PBV * L::PBD);
        const float4 h0 = hb[0], h1 = hb[1];
        a[0] = h0.x + ra[0]; a[1] = h0.y + ra[1]; a[2] = h0.z + ra[2]; a[3] = h0.w + ra[3];
        a[4] = h1.x + ra[4]; a[5] = h1.y + ra[5]; a[6] = h1.z + ra[6]; a[7] = h1.w + ra[7];
        float2 P[D];
        sincos_red(a[K], &P[0].y, &P[0].x);
#pragma unroll
        for (int m = 0; m < K; ++m) {
          float es, ec;
          sincos_red(a[m], &es, &ec);
#pragma unroll
          for (int j = 0; j < (1 << m); ++j) {
            const float2 q = P[j];
            P[j + (1 << m)] = make_float2(q.x * ec - q.y * es, q.x * es + q.y * ec);
          }
        }
#pragma unroll
        for (int j = 0; j < D; ++j) {
          const float2 x = v[j];
          v[j] = make_float2(x.x * P[j].x - x.y * P[j].y, x.x * P[j].y + x.y * P[j].x);
        }
      }
    }
    // row exponent: max |x| < 2^e_row
    float mx = 0.f;
#pragma unroll
    for (int j = 0; j < D; ++j) mx = fmaxf(mx, fmaxf(fabsf(v[j].x), fabsf(v[j].y)));
    const int e_row = min(max(int((__float_as_uint(mx) >> 23) & 0xFF) - 126, p.emin), p.emax);
    const float sc_in = pow2f(22 - e_row);
    const float scale = pow2f(e_row + p.e_b - 29);
    const float cm = -771.f * pow2f(e_row + p.e_b - 7);  // -257 M scale
    if (it > 0) {  // MMA(i-1) done: A is free and its accumulators are ready
      mbar_wait(bar, (it - 1) & 1);
      fence_after();
      epilogue(prev_base, prev_scale, prev_cm);
    }
#if DSV_TC8_FILL == 0
    // accumulators back to M for this tile's MMAs (8 columns per store from
    // registers that stay live across the loop: no per-tile materialisation)
#pragma unroll
    for (int q = 0; q < 3 * N0 / 8; ++q) tmem_st8(tlane + uint32_t(L::T_HI + 8 * q), mg);
#endif
    // digits -> TMEM: column c holds K = 4c..4c+3 = (re, im) of members 2c, 2c+1
    uint32_t la2[N0 / 4], la1[N0 / 4], la0[N0 / 4];
#pragma unroll
    for (int c = 0; c < N0 / 4; ++c) {
      const uint32_t w0 = __float_as_uint(__fmaf_rn(v[2 * c].x, sc_in, kMagic)) + kDigitOff;
      const uint32_t w1 = __float_as_uint(__fmaf_rn(v[2 * c].y, sc_in, kMagic)) + kDigitOff;
      const uint32_t w2 = __float_as_uint(__fmaf_rn(v[2 * c + 1].x, sc_in, kMagic)) + kDigitOff;
      const uint32_t w3 = __float_as_uint(__fmaf_rn(v[2 * c + 1].y, sc_in, kMagic)) + kDigitOff;
      const uint32_t p01 = __byte_perm(w0, w1, 0x5140), p23 = __byte_perm(w2, w3, 0x5140);
      la0[c] = __byte_perm(p01, p23, 0x5410) ^ 0x80808080u;
      la1[c] = __byte_perm(p01, p23, 0x7632) ^ 0x80808080u;
      la2[c] = __byte_perm(__byte_perm(w0, w1, 0x0062), __byte_perm(w2, w3, 0x0062), 0x5410);
    }
    if constexpr (N0 / 4 == 16) {
      tmem_st16(tlane + uint32_t(L::T_A2), la2);
      tmem_st16(tlane + uint32_t(L::T_A1), la1);
      tmem_st16(tlane + uint32_t(L::T_A0), la0);
    } else {
      tmem_st8(tlane + uint32_t(L::T_A2), la2);
      tmem_st8(tlane + uint32_t(L::T_A1), la1);
      tmem_st8(tlane + uint32_t(L::T_A0), la0);
    }
    cp_async_wait<S - 2>();
    tmem_wait_st();
    fence_before();
    group_sync(grp);
    if (row == 0) {
      fence_after();
#if DSV_TC8_FILL == 1
      // accumulators back to M (tcgen05.cp of a constant block, ordered before the MMAs)
      const uint64_t md = plain_desc(sbase + L::MAG, 128, 128);
#pragma unroll
      for (int q = 0; q < 3 * N0 / 4; ++q) tmem_cp_x4(uint32_t(grp * 256 + L::T_HI + 4 * q), md);
#elif DSV_TC8_FILL == 2
      const uint64_t md = plain_desc(sbase + L::MAG, 128, 256);
#pragma unroll
      for (int q = 0; q < 3 * N0 / 8; ++q) tmem_cp_128x256(uint32_t(grp * 256 + L::T_HI + 8 * q), md);
#endif
      if (grp == 0) issue_mma8<K, 0>(sbase);
      else issue_mma8<K, 1>(sbase);
      mma_commit(bar);
    }
    coop_phase(it + 2, tq[S - 2 >= 1 ? 1 : 0]);
    if (PHASED && !p.coop) row_angles(tq[0] | rowoff);  // tile i+1
    prev_base = base;
    prev_scale = scale;
    prev_cm = cm;
  }
  if (it > 0) {
    mbar_wait(bar, (it - 1) & 1);
    fence_after();
    epilogue(prev_base, prev_scale, prev_cm);
  }
  cp_async_wait<0>();
  fence_before();
  __syncthreads();
  if (warp == 0) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmem_slot), "r"(512) : "memory");
  }
}

// ---- warp-specialised pipeline ---------------------------------------------------------
// The same arithmetic as k_dense_tc8, with the per-tile work split over three
// warp roles that run concurrently on different tiles (14 warps per SM instead
// of 8; a role never waits on another role's instruction latency):
//   warps 0-1  loaders: cp.async two rows each of the tile into a ring stage,
//              arrive on full[stage] when the copies land; phased windows
//              also compute the tile's phase data into the stage;
//   warps 2-5  converters (thread = row, TMEM lane quarter = warp % 4): read
//              the row, apply the phase, scale and split into int8 digits,
//              tcgen05.st them into TMEM slot (i & 1), free the stage; one
//              thread issues the 3 x KSTEPS MMAs and commits;
//   warps 6-13 epilogue (two warps per lane quarter, one per half of the
//              output columns): wait for the MMAs, tcgen05.ld the three
//              accumulators, combine, store to HBM, reset the accumulators
//              to the magic start value and hand the TMEM slot back.
// mbarriers: full[s] (64 cp.async arrivals + 64 loader arrivals), empty[s]
// (128 converters), slot_free[t] (256 epilogue threads; completion 0 = the
// initial accumulator fill), acc_full[t] (MMA commit), meta_full[t] (the
// converters' per-row scale / offset for the epilogue).  The epilogue has the
// most dependent work per tile (ncu: converters waited on slot_free and
// loaders on empty with one epilogue warp per quarter), hence two per quarter.
template <int K, bool PHASED>
struct Tc8WsLayout {
  static constexpr int D = 1 << K;
  static constexpr int N0 = 2 * D;
  static constexpr int B_BYTES = 3 * N0 * 128;
  static constexpr int BAR = B_BYTES;              // barriers + TMEM slot + magic words (256 B)
  static constexpr int META = BAR + 256;           // [2 slots][128 rows] float2 (scale, cm)
  static constexpr int PST = META + 2 * 128 * 8;   // per-stage phase data
  static constexpr int PSTAGE = PHASED ? (32 + D * 8) : 0;  // tile-uniform angle sums [8] + phase vector [D]
  static constexpr int STAGE = 128 * D * 8;
  static constexpr int SMEM_MAX = 227 * 1024 - 1024;
  static constexpr int NS_FIT = (SMEM_MAX - PST - 1024) / (STAGE + PSTAGE);
  static constexpr int NSTAGE = NS_FIT > 8 ? 8 : NS_FIT;
  static constexpr int RING = ((PST + NSTAGE * PSTAGE + 1023) / 1024) * 1024;
  static constexpr int BYTES = RING + NSTAGE * STAGE;
  static_assert(NSTAGE >= 3, "ring must hold three tiles");
  static_assert(BYTES <= SMEM_MAX, "shared memory plan");
};

template <int K, bool PHASED, int MODE>
__global__ void __launch_bounds__(448, 1)
k_dense_tc8ws(const __grid_constant__ Tc8P<K> p, const uint4* __restrict__ bmat, const float4* __restrict__ tab,
              float2* __restrict__ sv) {
  using L = Tc8WsLayout<K, PHASED>;
  using LM = Tc8Layout<K>;  // TMEM plan and MMA shapes
  constexpr bool PAIR = MODE == kTcPair;
  constexpr bool LOWT = MODE == kTcLow;
  constexpr bool ROW2 = MODE == kTcRow2;
  constexpr int D = L::D;
  constexpr int N0 = L::N0;
  constexpr int S = L::NSTAGE;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t raw_base = smem_u32(smem_raw);
  const uint32_t sbase = (raw_base + 1023u) & ~1023u;
  unsigned char* sm = smem_raw + (sbase - raw_base);
  const int tid = threadIdx.x;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);  // warp-uniform (TMEM addresses in uniform registers)
  const int role = warp < 2 ? 0 : (warp < 6 ? 1 : 2);
  // converters / epilogue: the row is this thread's TMEM lane (quarter = warp % 4)
  const int row = role == 0 ? tid : (((warp & 3) << 5) | (tid & 31));
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + L::BAR + 192);
  auto FULL = [&](int s) { return sbase + L::BAR + 8 * s; };
  auto EMPTY = [&](int s) { return sbase + L::BAR + 64 + 8 * s; };
  auto SLOTFREE = [&](int t) { return sbase + L::BAR + 128 + 8 * t; };
  auto ACCFULL = [&](int t) { return sbase + L::BAR + 144 + 8 * t; };
  auto METAFULL = [&](int t) { return sbase + L::BAR + 160 + 8 * t; };

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid < 2) reinterpret_cast<uint32_t*>(sm + L::BAR + 200)[tid] = kAccInit;
  if (tid == 32) {
    for (int s = 0; s < S; ++s) {
      mbar_init(FULL(s), 128);
      mbar_init(EMPTY(s), 128);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(SLOTFREE(t), 256);
      mbar_init(ACCFULL(t), 1);
      mbar_init(METAFULL(t), 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < 3 * N0 * 8; i += 448) {
    const int r = i / 8, c16 = i % 8;
    *reinterpret_cast<uint4*>(sm + r * 128 + ((c16 ^ (r & 7)) << 4)) = bmat[i];
  }
  const uint64_t step = gridDim.x;
  auto tile_of = [&](int i) { return uint64_t(blockIdx.x) + uint64_t(i) * step; };
  const uint64_t e0 = expand(p.g, 0);
  const uint64_t rowoff = expand(p.g, row) ^ e0;
  float2* meta = reinterpret_cast<float2*>(sm + L::META);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  fence_before();
  __syncthreads();
  fence_after();
  if (*tmem_slot != 0u) __trap();  // whole-TMEM allocation starts at lane 0, column 0
  const uint32_t tq = uint32_t((warp & 3) * 32) << 16;

  if (role == 0) {
    // ===== loaders =====
#pragma unroll 1
    for (int i = 0;; ++i) {
      const uint64_t tl = tile_of(i);
      if (tl >= p.ntiles) break;
      const int s = i % S;
      if (i >= S) mbar_wait(EMPTY(s), uint32_t((i / S) - 1) & 1u);
      const uint64_t tb = expand(p.g, tl * 128);
      const uint32_t st0 = sbase + L::RING + s * L::STAGE;
#pragma unroll 1
      for (int rr = 0; rr < 2; ++rr) {
      const int row = tid + 64 * rr;  // this loader's two rows
      const uint64_t rowoff = expand(p.g, row) ^ e0;
      const int prow = 2 * (row & 63);  // (the jpos mapping measured slower in this pipeline)
      const int jpar = row >> 6;
      const uint64_t prowoff = expand(p.g, prow) ^ e0;
      if constexpr (LOWT) {
#pragma unroll
        for (int m = 0; m < D / 2; ++m) {
          const int q = row + 128 * m;
          const int r = q / (D / 2), c = q % (D / 2);
          cp_async16(st0 + r * (D * 8) + ((c ^ (r & 7)) << 4), sv + tb + 2 * q);
        }
      } else if constexpr (ROW2) {
        const uint64_t b = tb | rowoff;
#pragma unroll
        for (int m = 0; m < D / 2; ++m) cp_async16(st0 + m * 2048 + row * 16, sv + b + p.offs[2 * m]);
      } else if constexpr (PAIR) {
        const uint64_t b = tb | prowoff;
        if (p.tshift >= 0) {
          const float2* src = sv + b + (uint64_t(jpar) << p.tshift);
          const uint64_t stride = uint64_t(2) << p.tshift;
#pragma unroll
          for (int jj = 0; jj < D / 2; ++jj) cp_async16(st0 + prow * 8 + (2 * jj + jpar) * 1024, src + jj * stride);
        } else {
#pragma unroll
          for (int jj = 0; jj < D / 2; ++jj) {
            const uint64_t o = jpar ? p.offs[2 * jj + 1] : p.offs[2 * jj];
            cp_async16(st0 + prow * 8 + (2 * jj + jpar) * 1024, sv + b + o);
          }
        }
      } else {
        const uint64_t b = tb | rowoff;
        if (p.tshift >= 0) {
          const float2* src = sv + b;
          const uint64_t stride = uint64_t(1) << p.tshift;
#pragma unroll
          for (int j = 0; j < D; ++j) cp_async8(st0 + row * 8 + j * 1024, src + j * stride);
        } else {
#pragma unroll
          for (int j = 0; j < D; ++j) cp_async8(st0 + row * 8 + j * 1024, sv + b + p.offs[j]);
        }
      }
      }
      cp_async_mbar_arrive(FULL(s));
      if constexpr (PHASED) {
        // tile-uniform angle sums (constant bank, the same for every thread);
        // row-varying nibbles are added by the converters (rows' own part)
        unsigned char* ps = sm + L::PST + s * L::PSTAGE;
        float a[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) a[q] = 0.f;
#pragma unroll
        for (int c = 0; c < kTcMaxNib; ++c) {
          if (c >= p.nnib_row && c < p.nnib) {
            const int r = (c * 16 + int((tb >> p.nib_shift[c]) & 15u)) * 2;
            const float4 x = p.ctab[r], y = p.ctab[r + 1];
            a[0] += x.x; a[1] += x.y; a[2] += x.z; a[3] += x.w;
            a[4] += y.x; a[5] += y.y; a[6] += y.z; a[7] += y.w;
          }
        }
        if (p.coop) {  // one phase vector per tile: member j = tid - (64 - D)
          const int j = tid - (64 - D);
          if (j >= 0) {
            float ang = a[K];
#pragma unroll
            for (int m = 0; m < K; ++m) ang += ((j >> m) & 1) ? a[m] : 0.f;
            float sn, cs;
            sincos_unit(ang, &sn, &cs);
            reinterpret_cast<float2*>(ps + 32)[j] = make_float2(cs, sn);
          }
        } else if (tid == 0) {
          float4* au = reinterpret_cast<float4*>(ps);
          au[0] = make_float4(a[0], a[1], a[2], a[3]);
          au[1] = make_float4(a[4], a[5], a[6], a[7]);
        }
      }
      mbar_arrive(FULL(s));
    }
    cp_async_wait<0>();
  } else if (role == 1) {
    // ===== converters + MMA issue =====
    // row-varying phase nibbles (non-coop windows): this row's angle sums from
    // the global table, loaded one tile ahead so the latency is off the path
    float ra[8];
    auto row_part = [&](uint64_t tl) {
#pragma unroll
      for (int q = 0; q < 8; ++q) ra[q] = 0.f;
      if (tl >= p.ntiles) return;
      const uint64_t b = expand(p.g, tl * 128) | rowoff;
#pragma unroll
      for (int c = 0; c < kTcMaxNib; ++c) {
        if (c < p.nnib_row) {
          const int r = (c * 16 + int((b >> p.nib_shift[c]) & 15u)) * 2;
          const float4 x = __ldg(tab + r), y = __ldg(tab + r + 1);
          ra[0] += x.x; ra[1] += x.y; ra[2] += x.z; ra[3] += x.w;
          ra[4] += y.x; ra[5] += y.y; ra[6] += y.z; ra[7] += y.w;
        }
      }
    };
    if (PHASED && !p.coop) row_part(tile_of(0));
#pragma unroll 1
    for (int i = 0;; ++i) {
      const uint64_t tl = tile_of(i);
      if (tl >= p.ntiles) break;
      const int s = i % S;
      const int t = i & 1;
      mbar_wait(FULL(s), uint32_t(i / S) & 1u);
      const unsigned char* stg = sm + L::RING + s * L::STAGE;
      float2 v[D];
      if constexpr (ROW2) {
#pragma unroll
        for (int m = 0; m < D / 2; ++m) {
          const float4 x = *reinterpret_cast<const float4*>(stg + m * 2048 + row * 16);
          v[2 * m] = make_float2(x.x, x.y);
          v[2 * m + 1] = make_float2(x.z, x.w);
        }
      } else if constexpr (LOWT) {
#pragma unroll
        for (int c = 0; c < D / 2; ++c) {
          const float4 x = *reinterpret_cast<const float4*>(stg + row * (D * 8) + ((c ^ (row & 7)) << 4));
          v[2 * c] = make_float2(x.x, x.y);
          v[2 * c + 1] = make_float2(x.z, x.w);
        }
      } else {
        const float2* raw = reinterpret_cast<const float2*>(stg) + row;
#pragma unroll
        for (int j = 0; j < D; ++j) v[j] = raw[j * 128];
      }
      if constexpr (PHASED) {
        const unsigned char* ps = sm + L::PST + s * L::PSTAGE;
        if (p.coop) {
          const float2* P = reinterpret_cast<const float2*>(ps + 32);
#pragma unroll
          for (int j = 0; j < D; ++j) {
            const float2 x = v[j], f = P[j];
            v[j] = make_float2(x.x * f.x - x.y * f.y, x.x * f.y + x.y * f.x);
          }
        } else {
          const float4* au = reinterpret_cast<const float4*>(ps);
          const float4 h0 = au[0], h1 = au[1];
          const float a[8] = {h0.x + ra[0], h0.y + ra[1], h0.z + ra[2], h0.w + ra[3],
                              h1.x + ra[4], h1.y + ra[5], h1.z + ra[6], h1.w + ra[7]};
          row_part(tile_of(i + 1));  // next tile's row part (loads in flight during this tile)
          float2 P[D];
          sincos_red(a[K], &P[0].y, &P[0].x);
#pragma unroll
          for (int m = 0; m < K; ++m) {
            float es, ec;
            sincos_red(a[m], &es, &ec);
#pragma unroll
            for (int j = 0; j < (1 << m); ++j) {
              const float2 q = P[j];
              P[j + (1 << m)] = make_float2(q.x * ec - q.y * es, q.x * es + q.y * ec);
            }
          }
#pragma unroll
          for (int j = 0; j < D; ++j) {
            const float2 x = v[j];
            v[j] = make_float2(x.x * P[j].x - x.y * P[j].y, x.x * P[j].y + x.y * P[j].x);
          }
        }
      }
      mbar_arrive(EMPTY(s));  // the row (and its phase data) is in registers: stage free
      float mx = 0.f;
#pragma unroll
      for (int j = 0; j < D; ++j) mx = fmaxf(mx, fmaxf(fabsf(v[j].x), fabsf(v[j].y)));
      const int e_row = min(max(int((__float_as_uint(mx) >> 23) & 0xFF) - 126, p.emin), p.emax);
      const float sc_in = pow2f(22 - e_row);
      // slot t: the epilogue has drained tile i - 2 (completion 0 = initial fill)
      mbar_wait(SLOTFREE(t), uint32_t(i >> 1) & 1u);
      fence_after();
      meta[t * 128 + row] = make_float2(pow2f(e_row + p.e_b - 29), -197379.f * pow2f(e_row + p.e_b - 7));
      const uint32_t tl0 = uint32_t(t * 256) + tq;
      // digits -> TMEM in blocks of 8 columns (column c: K = 4c..4c+3 = (re, im) of members 2c, 2c+1)
#pragma unroll
      for (int cb = 0; cb < N0 / 4; cb += 8) {
        uint32_t la2[8], la1[8], la0[8];
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {
          const int c = cb + cc;
          const uint32_t w0 = __float_as_uint(__fmaf_rn(v[2 * c].x, sc_in, kMagic)) + kDigitOff;
          const uint32_t w1 = __float_as_uint(__fmaf_rn(v[2 * c].y, sc_in, kMagic)) + kDigitOff;
          const uint32_t w2 = __float_as_uint(__fmaf_rn(v[2 * c + 1].x, sc_in, kMagic)) + kDigitOff;
          const uint32_t w3 = __float_as_uint(__fmaf_rn(v[2 * c + 1].y, sc_in, kMagic)) + kDigitOff;
          const uint32_t p01 = __byte_perm(w0, w1, 0x5140), p23 = __byte_perm(w2, w3, 0x5140);
          la0[cc] = __byte_perm(p01, p23, 0x5410) ^ 0x80808080u;
          la1[cc] = __byte_perm(p01, p23, 0x7632) ^ 0x80808080u;
          la2[cc] = __byte_perm(__byte_perm(w0, w1, 0x0062), __byte_perm(w2, w3, 0x0062), 0x5410);
        }
        tmem_st8(tl0 + uint32_t(LM::T_A2 + cb), la2);
        tmem_st8(tl0 + uint32_t(LM::T_A1 + cb), la1);
        tmem_st8(tl0 + uint32_t(LM::T_A0 + cb), la0);
      }
      mbar_arrive(METAFULL(t));
      tmem_wait_st();
      fence_before();
      named_sync(1, 128);
      if (row == 0) {
        fence_after();
        if (t == 0) issue_mma8<K, 0>(sbase);
        else issue_mma8<K, 1>(sbase);
        mma_commit(ACCFULL(t));
      }
    }
  } else {
    // ===== epilogue =====
    uint32_t mg[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) mg[q] = reinterpret_cast<const uint32_t*>(sm + L::BAR + 200)[q & 1];
    // this warp's half of the output columns (k = 4: one half of 32 columns
    // per accumulator, the second warp of the quarter only resets)
    constexpr int NH = N0 / 32 > 0 ? N0 / 32 : 1;
    const int half = (warp - 6) >> 2;
    auto reset = [&](uint32_t tlane) {
      if constexpr (NH == 1) {  // k = 4: the first warp of the quarter owns all 32 columns
        if (half == 0)
#pragma unroll
          for (int q = 0; q < 3 * N0 / 8; ++q) tmem_st8(tlane + uint32_t(LM::T_HI + 8 * q), mg);
      } else {
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int q = 0; q < N0 / 16; ++q)
            tmem_st8(tlane + uint32_t(LM::T_HI + a * N0 + half * (N0 / 2) + 8 * q), mg);
      }
    };
    // accumulators of both slots start at the magic value: completion 0 of slot_free
    reset(tq);
    reset(uint32_t(256) + tq);
    tmem_wait_st();
    fence_before();
    mbar_arrive(SLOTFREE(0));
    mbar_arrive(SLOTFREE(1));
    // out = scale (acc_h 2^16 + acc_m 2^8 + acc_l): the accumulators read
    // back as M + acc, so with cm = -65793 M scale three fmas do it, hi first
    // (acc_h 2^16 - 257 M is exact; the two later sums round once each)
    auto combine = [](float h, float m, float l, float scale, float s8, float s16, float cm) {
      return __fmaf_rn(l, scale, __fmaf_rn(m, s8, __fmaf_rn(h, s16, cm)));
    };
#pragma unroll 1
    for (int i = 0;; ++i) {
      const uint64_t tl = tile_of(i);
      if (tl >= p.ntiles) break;
      const int t = i & 1;
      const uint64_t b = expand(p.g, tl * 128) | rowoff;
      mbar_wait(ACCFULL(t), uint32_t(i >> 1) & 1u);
      mbar_wait(METAFULL(t), uint32_t(i >> 1) & 1u);
      fence_after();
      const float2 mt = meta[t * 128 + row];
      const float scale = mt.x, cm = mt.y;
      const float s8 = scale * 256.f, s16 = scale * 65536.f;
      const uint32_t tlane = uint32_t(t * 256) + tq;
#pragma unroll
      for (int hh = 0; hh < (NH + 1) / 2; ++hh) {
        const int h = NH == 1 ? 0 : half;
        if (NH == 1 && half == 1) break;
        float ch[32], cmid[32], cl[32];
        tmem_ld32(tlane + uint32_t(LM::T_HI + h * 32), ch);
        tmem_ld32(tlane + uint32_t(LM::T_MID + h * 32), cmid);
        tmem_ld32(tlane + uint32_t(LM::T_LO + h * 32), cl);
        auto val = [&](int c) { return combine(ch[c], cmid[c], cl[c], scale, s8, s16, cm); };
        if constexpr (LOWT) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            stcs32(sv + b + h * 16 + 4 * q, val(8 * q), val(8 * q + 1), val(8 * q + 2), val(8 * q + 3),
                   val(8 * q + 4), val(8 * q + 5), val(8 * q + 6), val(8 * q + 7));
        } else if constexpr (ROW2) {
#pragma unroll
          for (int q = 0; q < 8; ++q)
            __stcs(reinterpret_cast<float4*>(sv + b + p.offs[h * 16 + 2 * q]),
                   make_float4(val(4 * q), val(4 * q + 1), val(4 * q + 2), val(4 * q + 3)));
        } else if constexpr (PAIR && !PHASED) {  // (pair-swapped stores win here: 31.5 -> 28.7 ms on (1,9,17,22,30), dense state)
          const bool odd = row & 1;
          const uint64_t be = b - (odd ? 1 : 0);
          float2* dst = sv + be + (p.tshift >= 0 ? (uint64_t(h * 16 + (odd ? 1 : 0)) << p.tshift) : 0);
          const uint64_t stride = p.tshift >= 0 ? (uint64_t(2) << p.tshift) : 0;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            float o[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) o[c] = val(4 * q + c);
            const float sx = odd ? o[0] : o[2], sy = odd ? o[1] : o[3];
            const float rx = __shfl_xor_sync(0xffffffffu, sx, 1), ry = __shfl_xor_sync(0xffffffffu, sy, 1);
            const float4 w = odd ? make_float4(rx, ry, o[2], o[3]) : make_float4(o[0], o[1], rx, ry);
            if (p.tshift >= 0) {
              __stcs(reinterpret_cast<float4*>(dst + q * stride), w);
            } else {
              const uint64_t oj = odd ? p.offs[h * 16 + 2 * q + 1] : p.offs[h * 16 + 2 * q];
              __stcs(reinterpret_cast<float4*>(sv + be + oj), w);
            }
          }
        } else {
          if (p.tshift >= 0) {
            float2* dst = sv + b + (uint64_t(h * 16) << p.tshift);
            const uint64_t stride = uint64_t(1) << p.tshift;
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              __stcs(dst, make_float2(val(2 * q), val(2 * q + 1)));
              dst += stride;
            }
          } else {
#pragma unroll
            for (int q = 0; q < 16; ++q) __stcs(sv + b + p.offs[h * 16 + q], make_float2(val(2 * q), val(2 * q + 1)));
          }
        }
      }
      // accumulators back to the magic start value, slot handed back
      reset(tlane);
      tmem_wait_st();
      fence_before();
      mbar_arrive(SLOTFREE(t));
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 0) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmem_slot), "r"(512) : "memory");
  }
}

template <int K, bool PHASED, int MODE>
static cudaError_t tc8_go(const TcDesc& d, const void* d_bmat, const void* d_tab, void* sv, cudaStream_t st) {
  using L = Tc8Layout<K>;
  Tc8P<K> p;
  std::memset(&p, 0, sizeof p);
  p.g = d.g;
  p.ntiles = d.g.nwork / 128;
  p.pairswap = d.pairswap;
  p.nnib = d.nnib;
  p.e_b = d.e_b;
  // every power of two the kernel forms stays normal: 22 - e_row, e_row + e_b - 29, e_row + e_b - 7
  // every power of two the kernel forms stays normal: 22 - e_row, e_row + e_b - 29,
  // 771 * 2^(e_row + e_b - 7)
  p.emin = std::max(-100, -97 - d.e_b);
  p.emax = std::min(100, 124 - d.e_b);
  p.coop = d.coop;
  p.nnib_row = d.nnib_row;
  p.tshift = d.tshift;
  p.jpos = 6;
  {  // lowest target bit (the first hole above bit 0 in PAIR mode): member parity sits at thread bit t - 1
    int lo = 64;
    for (int j = 1; j < (1 << K); ++j) {
      const uint64_t o = d.offs[j];
      if (o) lo = std::min(lo, __builtin_ctzll(o));
    }
    if (lo >= 1 && lo <= 7) p.jpos = lo - 1;
  }
#ifdef DSV_TC8_NOSTRIDE
  p.tshift = -1;
#endif
  for (int c = 0; c < 16; ++c) p.nib_shift[c] = d.nib_shift[c];
  for (int q = 0; q < 5; ++q) {
    p.tma_shift[q] = d.tma_shift[q];
    p.tma_mask[q] = d.tma_mask[q];
  }
  p.nrb = d.nrb;
  for (int q = 0; q < 3; ++q) p.rb_bit[q] = d.rb_bit[q];
  p.rvec = static_cast<const float2*>(d.d_rvec);
  for (int j = 0; j < (1 << K); ++j) p.offs[j] = d.offs[j];
  if (d.htab && d.nnib > 0) std::memcpy(p.ctab, d.htab, size_t(d.nnib) * 16 * 2 * sizeof(float4));
  int dev = 0;
  cudaGetDevice(&dev);
  if (MODE != kTcTma && d.ws) {
    using LW = Tc8WsLayout<K, PHASED>;
    const int smem = LW::BYTES + 1024;
    static bool attr_ws[64] = {false};
    if (dev >= 0 && dev < 64 && !attr_ws[dev]) {
      cudaError_t e =
          cudaFuncSetAttribute(k_dense_tc8ws<K, PHASED, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return e;
      attr_ws[dev] = true;
    }
    uint64_t blocks = uint64_t(device_sm_count());
    if (blocks > p.ntiles) blocks = p.ntiles;
    if (blocks == 0) return cudaSuccess;
    k_dense_tc8ws<K, PHASED, MODE><<<unsigned(blocks), 448, smem, st>>>(p, static_cast<const uint4*>(d_bmat),
                                                                      static_cast<const float4*>(d_tab),
                                                                      static_cast<float2*>(sv));
    return cudaGetLastError();
  }
  const int smem = L::BYTES + 1024;
  static bool attr_set[64] = {false};
  if (dev >= 0 && dev < 64 && !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_dense_tc8<K, PHASED, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr_set[dev] = true;
  }
  uint64_t blocks = uint64_t(device_sm_count());
  const uint64_t need = (p.ntiles + 1) / 2;
  if (blocks > need) blocks = need;
  if (blocks == 0) return cudaSuccess;
  k_dense_tc8<K, PHASED, MODE><<<unsigned(blocks), 256, smem, st>>>(p, d.tmap, static_cast<const uint4*>(d_bmat),
                                                                static_cast<const float4*>(d_tab),
                                                                static_cast<float2*>(sv));
  return cudaGetLastError();
}

template <int K>
static cudaError_t tc8_k(const TcDesc& d, const void* d_bmat, const void* d_tab, void* sv, cudaStream_t st) {
  const bool ph = d.nnib > 0 || d.nrb > 0;
  switch (d.mode) {
    case kTcPair: return ph ? tc8_go<K, true, kTcPair>(d, d_bmat, d_tab, sv, st) : tc8_go<K, false, kTcPair>(d, d_bmat, d_tab, sv, st);
    case kTcLow: return ph ? tc8_go<K, true, kTcLow>(d, d_bmat, d_tab, sv, st) : tc8_go<K, false, kTcLow>(d, d_bmat, d_tab, sv, st);
    case kTcRow2: return ph ? tc8_go<K, true, kTcRow2>(d, d_bmat, d_tab, sv, st) : tc8_go<K, false, kTcRow2>(d, d_bmat, d_tab, sv, st);
    case kTcTma: return ph ? tc8_go<K, true, kTcTma>(d, d_bmat, d_tab, sv, st) : tc8_go<K, false, kTcTma>(d, d_bmat, d_tab, sv, st);
  }
  return ph ? tc8_go<K, true, kTcRow>(d, d_bmat, d_tab, sv, st) : tc8_go<K, false, kTcRow>(d, d_bmat, d_tab, sv, st);
}

cudaError_t launch_dense_tc8(int k, const TcDesc& d, const void* d_bmat, const void* d_tab, void* sv,
                             cudaStream_t st) {
  switch (k) {
    case 4: return tc8_k<4>(d, d_bmat, d_tab, sv, st);
    case 5: return tc8_k<5>(d, d_bmat, d_tab, sv, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace dsv
