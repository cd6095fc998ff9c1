// tc8d.cu — complex128 5-qubit windows on the tensor cores through exact
// 8-bit digits (tcgen05.mma kind::i8, int32 accumulation): the digit
// arithmetic of tc8.cu / tc68.cu widened to fp64 precision.  Replaces
// apply_dense_bits (reference statevec.py:44-60) for complex128 k = 5 fused
// windows, which on the CUDA cores are FP64-FMA bound (2^(k-2) = 8 flop per
// byte against a ~5 flop/B FP64 ridge: 0.31-0.34 of the copy peak).
//
// Arithmetic.  Each tile row (one amplitude group, 64 reals) is scaled by a
// power of two so its largest |value| is < 2^51 and rounded to an integer I
// with ONE fma against the magic M = 1.5 * 2^52.  The bits of M + I are
// (0x4338 + s) 2^48 + (I mod 2^48) with s = I >> 48: bytes 0..5 are the
// unsigned base-256 digits of I (planes 6..1, u8) and, after subtracting
// 0x38 from byte 6, s is the signed top digit (plane 0, s8 in [-8, 8]) — no
// integer work per value beyond that one subtraction.  The gate's real
// embedding is split on the host into balanced signed digits b0 (|b0| <= 8)
// .. b6 in [-128, 127].
// Products a_i b_j with i + j = L accumulate exactly in int32 in level L
// (|acc| < 2^24); levels 0..7 are kept (34 digit products), the dropped
// levels >= 8 weigh ~2^-52 of the row-times-column scale; the rounding of
// the inputs to 52-bit integers (2^-52 of the row maximum) is the same order:
// a few times the native FP64 kernel's rounding error.
// Readback: H = acc0 2^24 + acc1 2^16 + acc2 2^8 + acc3 and
// Lo = acc4 2^24 + ... + acc7 are exact int64 (< 2^49), made doubles by the
// same magic (bits(M) + H as a double, minus M) and combined with one fma:
//   out = (H 2^32 + Lo) 2^(e_row + e_b - 62).
//
// Layout (one persistent CTA per SM, NT = 512 threads by default, 256 with
// dsv_config_set("tc8d512", 0); P = NT / 128 parts per tile row):
//   * loader / epilogue: thread (row = tid % 128, part = tid / 128) copies
//     and stores members 32 part / P .. of tile row `row` (its TMEM lane);
//   * converters: warp w takes rows 32 w / P .., the P lanes of a row share
//     its maximum by shuffles (no block barrier) and publish the row exponent
//     in shared memory for the epilogue;
//   * 2-stage cp.async ring of 64 KB tiles ([member][row] x 16 B);
//   * A digits in shared memory, K-major 128-byte swizzled: block q holds
//     planes 2q (bytes 0..63) and 2q + 1 (bytes 64..127) of all 128 rows;
//   * gate digits: 256 rows x 128 B, row n: bytes 0..63 = plane n / 64
//     (b0..b3) of output real n % 64, bytes 64..127 = plane 4 + n / 64 (b4..b6);
//   * TMEM: the CTA's 512 columns = levels 0..7 x 64 output reals;
//     a_i [b_j .. b_j'] lands on levels i + j .. i + j' (contiguous columns),
//     so 23 MMAs (N = 64..256) cover the 34 products per 128-row tile;
//   * with index bit 0 a target, member pairs (2i, 2i + 1) leave as one
//     32-byte store (STG.256): full sectors (n = 32, (0,5,11,19,28): 36 -> 33 ms).
// Bound: the 23 MMAs read ~230 KB of shared memory per tile (A 4 KB + B
// N x 32 B each), ~1800 cycles at 128 B/clk, and the single 512-column
// accumulator serialises them with the epilogue's TMEM reads: 0.75-0.8 of the
// copy peak on a dense random state.  Rejected on the same box (A/B at
// n = 32): a warp-specialised split (8 converter + 4 epilogue warps, mbarrier
// handshakes: 25 -> 29 ms), output-half TMEM split so half 0's MMAs overlap
// half 1's epilogue (46 narrower MMAs: 25 -> 30 ms), a third ring stage
// holding A in the consumed stage (25 -> 29 ms), member-fastest loads for
// index-bit-0 windows (slower: the cp.async smem writes or per-unit row
// offsets cost more than the sectors saved).
#include <cmath>
#include <cstring>

#include "common.cuh"
#include "launch.h"
#include "tcgen05.cuh"

namespace dsv {

using namespace tcx;

struct Tc8dP {
  Geom g;
  uint64_t ntiles;
  int e_b;
  int tshift;
  int mlo;  // targets occupy index bits 0 .. mlo - 1 (0: bit 0 free)
  int nchunk;               // PHASED: index bytes carrying phase terms
  int chunk_shift[8];       // their amplitude-index shifts (8 c)
  const double2* ftab;      // PHASED: [nchunk][256][6] unit factors exp(i angle) per (byte value, slot)
  uint64_t offs[32];
};

__device__ __forceinline__ double2 cmul_d(double2 a, double2 b) {
  return make_double2(__fma_rn(a.x, b.x, -__dmul_rn(a.y, b.y)), __fma_rn(a.x, b.y, __dmul_rn(a.y, b.x)));
}



struct Tc8dLayout {
  static constexpr int D = 32;
  static constexpr int B_OFF = 0;
  static constexpr int B_BYTES = 256 * 128;        // 32 KB
  static constexpr int A_OFF = B_OFF + B_BYTES;    // 4 blocks x 128 rows x 128 B
  static constexpr int A_BYTES = 4 * 128 * 128;    // 64 KB
  static constexpr int BAR = A_OFF + A_BYTES;      // MMA mbarrier + TMEM slot
  static constexpr int MX = BAR + 128;             // row exponents [3][128] int
  static constexpr int RING = (MX + 3 * 128 * 4 + 1023) / 1024 * 1024;
  static constexpr int STAGE = 128 * D * 16;       // 64 KB
  static constexpr int NSTAGE = 2;
  static constexpr int BYTES = RING + NSTAGE * STAGE;
  static_assert(BYTES + 1024 <= 227 * 1024, "shared memory budget");
};

constexpr unsigned long long kMagicBitsD = 0x4338000000000000ull;  // bits of 1.5 * 2^52
constexpr double kMagicD = 6755399441055744.0;                      // 1.5 * 2^52

// one 32-byte streaming store (STG.256)
__device__ __forceinline__ void st_cs_v4d(void* p, double a, double b, double c, double d) {
  asm volatile("st.global.cs.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

__device__ __forceinline__ double pow2d(int e) { return __longlong_as_double((long long)(e + 1023) << 52); }

__device__ __forceinline__ void issue_mma8d(uint32_t sbase) {
  using L = Tc8dLayout;
  // A plane 0 signed (s in [-8, 7]), planes 1..6 unsigned bytes; B balanced signed digits
  constexpr uint32_t S64 = idesc_i8<64, 1, 1>(), S192 = idesc_i8<192, 1, 1>(), S256 = idesc_i8<256, 1, 1>();
  constexpr uint32_t U64 = idesc_i8<64, 0, 1>(), U128 = idesc_i8<128, 0, 1>(), U192 = idesc_i8<192, 0, 1>(),
                     U256 = idesc_i8<256, 0, 1>();
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    auto A = [&](int i) { return sw128_desc(sbase + L::A_OFF + (i >> 1) * 16384 + 64 * (i & 1) + 32 * s); };
    // half 0: planes b0..b3 from row 64 j; half 1: planes b4..b6 from row 64 (j - 4)
    auto B0 = [&](int j) { return sw128_desc(sbase + L::B_OFF + j * 64 * 128 + 32 * s); };
    auto B1 = [&](int j) { return sw128_desc(sbase + L::B_OFF + (j - 4) * 64 * 128 + 64 + 32 * s); };
    const uint32_t acc = s > 0 ? 1u : 0u;
    auto col = [](int level) { return uint32_t(64 * level); };
    if (s == 0) {
      mma_ss_i8(col(0), A(0), B0(0), S64, 0u);    // level 0        (zeroes cols 0..63)
    } else {
      mma_ss_i8(col(0), A(0), B0(0), S256, 1u);   // levels 0..3
    }
    mma_ss_i8(col(1), A(1), B0(0), U256, acc);    // levels 1..4    (s = 0: zeroes cols 64..319)
    mma_ss_i8(col(5), A(1), B1(4), U192, acc);    // levels 5..7    (s = 0: zeroes cols 320..511)
    if (s == 0) mma_ss_i8(col(1), A(0), B0(1), S192, 1u);  // levels 1..3
    mma_ss_i8(col(4), A(0), B1(4), S192, 1u);     // levels 4..6
    mma_ss_i8(col(2), A(2), B0(0), U256, 1u);     // levels 2..5
    mma_ss_i8(col(6), A(2), B1(4), U128, 1u);     // levels 6..7
    mma_ss_i8(col(3), A(3), B0(0), U256, 1u);     // levels 3..6
    mma_ss_i8(col(7), A(3), B1(4), U64, 1u);      // level 7
    mma_ss_i8(col(4), A(4), B0(0), U256, 1u);     // levels 4..7
    mma_ss_i8(col(5), A(5), B0(0), U192, 1u);     // levels 5..7
    mma_ss_i8(col(6), A(6), B0(0), U128, 1u);     // levels 6..7
  }
}

// NT threads = P parts per tile row (P = 2: 256 threads, P = 4: 512 threads
// with half the values per thread and twice the warps to hide latency)
template <int NT, bool PHASED>
__global__ void __launch_bounds__(NT, 1)
k_dense_tc8d(const __grid_constant__ Tc8dP p, const uint4* __restrict__ bmat, double2* __restrict__ sv) {
  using L = Tc8dLayout;
  constexpr int S = L::NSTAGE;
  constexpr int P = NT / 128;   // parts per row
  constexpr int MP = 32 / P;    // members per part
  constexpr int RP = 64 / P;    // reals per part
  constexpr int RW = 32 / P;    // rows per warp in the input phase
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t raw_base = smem_u32(smem_raw);
  const uint32_t sbase = (raw_base + 1023u) & ~1023u;
  unsigned char* sm = smem_raw + (sbase - raw_base);
  const int tid = threadIdx.x;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int row = tid & 127;
  const int part = tid >> 7;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + L::BAR + 16);
  const uint32_t bar = sbase + L::BAR;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 32) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // gate digits, host layout [256 rows][8 x 16 B] -> 128-byte swizzled rows
  for (int i = tid; i < 256 * 8; i += NT) {
    const int r = i / 8, c16 = i % 8;
    *reinterpret_cast<uint4*>(sm + L::B_OFF + r * 128 + ((c16 ^ (r & 7)) << 4)) = bmat[i];
  }

  const uint64_t step = gridDim.x;
  auto tile_of = [&](int i) { return uint64_t(blockIdx.x) + uint64_t(i) * step; };
  const uint64_t e0 = expand(p.g, 0);
  const uint64_t rowoff = expand(p.g, row) ^ e0;
  auto issue = [&](int i) -> uint64_t {
    const uint64_t tl = tile_of(i);
    uint64_t tb = 0;
    if (tl < p.ntiles) {
      tb = expand(p.g, tl * 128);
      const uint32_t st0 = sbase + L::RING + (i % S) * L::STAGE + row * 16;
      const uint64_t b = tb | rowoff;
      if (p.tshift >= 0) {
        const double2* src = sv + b + (uint64_t(MP * part) << p.tshift);
        const uint64_t stride = uint64_t(1) << p.tshift;
#pragma unroll
        for (int mm = 0; mm < MP; ++mm) cp_async16(st0 + (MP * part + mm) * 2048, src + mm * stride);
      } else {
#pragma unroll
        for (int mm = 0; mm < MP; ++mm) {
          const int j = MP * part + mm;
          cp_async16(st0 + j * 2048, sv + b + p.offs[j]);
        }
      }
    }
    cp_async_commit();
    return tb;
  };

  uint64_t tq = issue(0);
  cp_async_wait<0>();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  fence_before();
  __syncthreads();
  fence_after();
  if (*tmem_slot != 0u) __trap();
  const uint32_t tlane = uint32_t((warp & 3) * 32) << 16;

  // out = (H 2^32 + Lo) 2^(e_row + e_b - 62); H, Lo exact int64 < 2^49
  // chunk = 8 output reals starting at real c0 (members c0 / 2 .. + 3); level
  // L of real c at TMEM column 64 L + c
  auto load_chunk = [&](int c0, uint32_t (&acc)[8][8]) {
#pragma unroll
    for (int l = 0; l < 8; ++l) tmem_ld8(tlane + uint32_t(64 * l + c0), acc[l]);
    tmem_wait_ld();
#pragma unroll
    for (int l = 0; l < 8; ++l) reg_fence(acc[l]);
  };
  auto finish_chunk = [&](const uint32_t (&acc)[8][8], int c0, uint64_t b, int e_row) {
    const double s_lo = pow2d(e_row + p.e_b - 62), s_hi = pow2d(e_row + p.e_b - 30);
    double o[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const long long H = (long long)int(acc[0][c]) * 16777216ll + (long long)int(acc[1][c]) * 65536ll +
                          (long long)int(acc[2][c]) * 256ll + (long long)int(acc[3][c]) + (long long)kMagicBitsD;
      const long long Lw = (long long)int(acc[4][c]) * 16777216ll + (long long)int(acc[5][c]) * 65536ll +
                           (long long)int(acc[6][c]) * 256ll + (long long)int(acc[7][c]) + (long long)kMagicBitsD;
      const double hd = __dadd_rn(__longlong_as_double(H), -kMagicD);
      const double ld = __dadd_rn(__longlong_as_double(Lw), -kMagicD);
      o[c] = __fma_rn(hd, s_hi, __dmul_rn(ld, s_lo));
    }
    const int m0 = c0 / 2;
    if (p.mlo >= 1) {  // index bit 0 a target: members 2i, 2i + 1 are one 32-byte sector
#pragma unroll
      for (int i = 0; i < 4; i += 2) {
        double2* dst = p.tshift >= 0 ? sv + b + (uint64_t(m0 + i) << p.tshift) : sv + b + p.offs[m0 + i];
        st_cs_v4d(dst, o[2 * i], o[2 * i + 1], o[2 * i + 2], o[2 * i + 3]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        double2* dst = p.tshift >= 0 ? sv + b + (uint64_t(m0 + i) << p.tshift) : sv + b + p.offs[m0 + i];
        __stcs(dst, make_double2(o[2 * i], o[2 * i + 1]));
      }
    }
  };
  // this thread's output reals RP part .. RP part + RP - 1
  auto epilogue = [&](uint64_t b, int e_row) {
#pragma unroll 1
    for (int c0 = RP * part; c0 < RP * part + RP; c0 += 8) {
      uint32_t acc[8][8];
      load_chunk(c0, acc);
      finish_chunk(acc, c0, b, e_row);
    }
  };

  // input phase: warp w converts rows RW w .. RW w + RW - 1, lanes l, l + RW,
  // ... share row RW w + l (parts 0 .. P - 1), so the row maximum is a
  // shuffle; the epilogue keeps the TMEM lane mapping (row = tid & 127) and
  // reads the row's exponent from shared memory (double-buffered per tile)
  const int irow = RW * warp + (tid & (RW - 1));
  const int ipart = (tid & 31) / RW;
  const uint64_t irowoff = expand(p.g, irow) ^ e0;  // PHASED: group index of row irow within its tile
  int* ebuf = reinterpret_cast<int*>(sm + L::MX);  // [2][128] row exponents
  uint64_t prev_tb = 0;
  int it = 0;
#pragma unroll 1
  for (;; ++it) {
    const uint64_t tile = tile_of(it);
    if (tile >= p.ntiles) break;
    const uint64_t tb_cur = tq;
    tq = issue(it + 1);
    const double2* raw = reinterpret_cast<const double2*>(sm + L::RING + (it % S) * L::STAGE) + irow;
    double v[RP];
#pragma unroll
    for (int mm = 0; mm < MP; ++mm) {
      const double2 x = raw[(MP * ipart + mm) * 128];
      v[2 * mm] = x.x;
      v[2 * mm + 1] = x.y;
    }
    if constexpr (PHASED) {
      // the fold fuser's pre-phase (phased.cu's model): member j of the row
      // with group index x takes exp(i (gamma(x) + sum_m j_m alpha_m(x))); the
      // slot factors F_s = exp(i alpha_s(x)) (F_5 = exp(i gamma(x))) are
      // products of tabulated unit factors per index byte, applied factor by
      // factor to this thread's MP members (no sin/cos on the device)
      const uint64_t x = tb_cur | irowoff;
      double2 F[6];
#pragma unroll
      for (int t = 0; t < 6; ++t) F[t] = make_double2(1.0, 0.0);
#pragma unroll 1
      for (int c = 0; c < p.nchunk; ++c) {
        const double2* tr = p.ftab + (c * 256 + int((x >> p.chunk_shift[c]) & 255u)) * 6;
#pragma unroll
        for (int t = 0; t < 6; ++t) F[t] = cmul_d(F[t], __ldg(tr + t));
      }
      constexpr int LMP = MP == 16 ? 4 : (MP == 8 ? 3 : 2);
      double2 base = F[5];
#pragma unroll
      for (int m = LMP; m < 5; ++m)
        if (((MP * ipart) >> m) & 1) base = cmul_d(base, F[m]);
      // members in Gray-code order: one factor (or its conjugate) per step
      double2 f = base;
#pragma unroll
      for (int i = 0; i < MP; ++i) {
        const int mm = i ^ (i >> 1);
        if (i > 0) {
          // the bit that changed (folds to a constant after unrolling)
          const int m = (i & 1) ? 0 : ((i & 2) ? 1 : ((i & 4) ? 2 : 3));
          const double2 q = m == 0 ? F[0] : (m == 1 ? F[1] : (m == 2 ? F[2] : F[3]));
          f = cmul_d(f, ((mm >> m) & 1) ? q : make_double2(q.x, -q.y));
        }
        const double2 y = cmul_d(f, make_double2(v[2 * mm], v[2 * mm + 1]));
        v[2 * mm] = y.x;
        v[2 * mm + 1] = y.y;
      }
    }
    uint32_t mx = 0;
#pragma unroll
    for (int c = 0; c < RP; ++c) mx = max(mx, uint32_t(__double2hiint(v[c])) & 0x7FFFFFFFu);
#pragma unroll
    for (int o = RW; o < 32; o *= 2) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    // |values| < 2^e_row; the clamp keeps 2^(51 - e_row) and the output scales normal
    const int e_row = min(max(int(mx >> 20) - 1022, -900), 900);
    if (ipart == 0) ebuf[(it & 1) * 128 + irow] = e_row;
    const double sc_in = pow2d(51 - e_row);
    // digits straight from the bits of M + I (|I| <= 2^51, M = 1.5 * 2^52;
    // bits(M + I) = bits(M) + I holds up to 2^53): bytes 0..5 are the
    // unsigned base-256 digits of I mod 2^48 (planes 6..1, u8), byte 6 is
    // 0x38 + s with s = I >> 48 in [-8, 8] (plane 0, s8 once 0x38 is
    // subtracted from the high word).  Word g of plane i = the plane-i bytes
    // of reals 4g .. 4g + 3.
    uint32_t dg[7][RP / 4];
#pragma unroll
    for (int g = 0; g < RP / 4; ++g) {
      uint32_t lo[4], hi[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const double x = __fma_rn(v[4 * g + r], sc_in, kMagicD);
        lo[r] = uint32_t(__double2loint(x));
        hi[r] = uint32_t(__double2hiint(x)) - 0x00380000u;
      }
      const uint32_t t01 = __byte_perm(lo[0], lo[1], 0x5140), t23 = __byte_perm(lo[2], lo[3], 0x5140);
      const uint32_t u01 = __byte_perm(lo[0], lo[1], 0x7362), u23 = __byte_perm(lo[2], lo[3], 0x7362);
      const uint32_t h01 = __byte_perm(hi[0], hi[1], 0x5140), h23 = __byte_perm(hi[2], hi[3], 0x5140);
      const uint32_t g01 = __byte_perm(hi[0], hi[1], 0x0062), g23 = __byte_perm(hi[2], hi[3], 0x0062);
      dg[6][g] = __byte_perm(t01, t23, 0x5410);
      dg[5][g] = __byte_perm(t01, t23, 0x7632);
      dg[4][g] = __byte_perm(u01, u23, 0x5410);
      dg[3][g] = __byte_perm(u01, u23, 0x7632);
      dg[2][g] = __byte_perm(h01, h23, 0x5410);
      dg[1][g] = __byte_perm(h01, h23, 0x7632);
      dg[0][g] = __byte_perm(g01, g23, 0x5410);
    }
    if (it > 0) {  // MMA(i-1) done: A is free and its accumulators are ready
      mbar_wait(bar, (it - 1) & 1);
      fence_after();
      epilogue(prev_tb | rowoff, ebuf[((it - 1) & 1) * 128 + row]);
    }
#pragma unroll
    for (int i = 0; i < 7; ++i) {
      unsigned char* rowp = sm + L::A_OFF + (i >> 1) * 16384 + irow * 128;
#pragma unroll
      for (int h = 0; h < RP / 16; ++h) {
        const int c16 = 4 * (i & 1) + (RP / 16) * ipart + h;
        *reinterpret_cast<uint4*>(rowp + ((c16 ^ (irow & 7)) << 4)) =
            make_uint4(dg[i][4 * h], dg[i][4 * h + 1], dg[i][4 * h + 2], dg[i][4 * h + 3]);
      }
    }
    cp_async_wait<0>();  // tile i+1 landed (this thread's part)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // A digits visible to the tensor core
    fence_before();
    __syncthreads();  // B2
    if (tid == 0) {
      fence_after();
      issue_mma8d(sbase);
      mma_commit(bar);
    }
    prev_tb = tb_cur;
  }
  if (it > 0) {
    mbar_wait(bar, (it - 1) & 1);
    fence_after();
    epilogue(prev_tb | rowoff, ebuf[((it - 1) & 1) * 128 + row]);
  }
  cp_async_wait<0>();
  fence_before();
  __syncthreads();
  if (warp == 0) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmem_slot), "r"(512) : "memory");
  }
}

template <int NT, bool PHASED>
static cudaError_t tc8d_go(const Tc8dP& p, unsigned blocks, int smem, const void* d_bmat, void* sv, cudaStream_t st) {
  static bool attr_set[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_dense_tc8d<NT, PHASED>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr_set[dev] = true;
  }
  k_dense_tc8d<NT, PHASED><<<blocks, NT, smem, st>>>(p, static_cast<const uint4*>(d_bmat), static_cast<double2*>(sv));
  return cudaGetLastError();
}

int tc8d_smem_bytes() { return Tc8dLayout::BYTES + 1024; }

cudaError_t launch_dense_tc8d(const TcDesc& d, const void* d_bmat, const void* d_ftab, void* sv, cudaStream_t st) {
  Tc8dP p;
  std::memset(&p, 0, sizeof p);
  p.g = d.g;
  p.ntiles = d.g.nwork / 128;
  p.e_b = d.e_b;
  p.tshift = d.tshift;
  while (p.mlo < 5 && d.offs[1 << p.mlo] == (uint64_t(1) << p.mlo)) ++p.mlo;  // targets 0 .. mlo - 1
  for (int j = 0; j < 32; ++j) p.offs[j] = d.offs[j];
  p.nchunk = d.nnib;  // byte chunks (TcDesc reuses its nibble fields)
  for (int c = 0; c < d.nnib && c < 8; ++c) p.chunk_shift[c] = d.nib_shift[c];
  p.ftab = static_cast<const double2*>(d_ftab);
  const int smem = tc8d_smem_bytes();
  uint64_t blocks = uint64_t(device_sm_count());
  if (blocks > p.ntiles) blocks = p.ntiles;
  if (blocks == 0) return cudaSuccess;
  const unsigned nb = unsigned(blocks);
  // 512 threads (4 parts per row): twice the warps of the 256-thread
  // layout to hide latency, 0-4 % faster on the same box (tools/tc8d_probe.py)
  if (p.nchunk > 0)
    return d.ws ? tc8d_go<512, true>(p, nb, smem, d_bmat, sv, st) : tc8d_go<256, true>(p, nb, smem, d_bmat, sv, st);
  return d.ws ? tc8d_go<512, false>(p, nb, smem, d_bmat, sv, st) : tc8d_go<256, false>(p, nb, smem, d_bmat, sv, st);
}

}  // namespace dsv
