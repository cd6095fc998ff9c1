// tc68.cu — 6-qubit complex64 windows (plain or with the fold fuser's
// pre-phase) on the tensor cores through exact 8-bit digits (tcgen05.mma
// kind::i8, int32 accumulation) — the arithmetic of tc8.cu on the layout of
// tc6.cu.  Replaces apply_dense_bits (reference statevec.py:44-60) for
// 6-qubit fused windows; with the bf16 limbs of tc6.cu these were
// tensor-bound (40 MMAs per tile, 0.72 of the copy peak), the int8 digits
// need 16 MMAs at twice the rate, so k = 6 windows run at HBM speed and a
// 33-qubit QFT needs 6 passes instead of 7.
//
//   * one persistent CTA per SM, ONE group of 256 threads: thread (row, half)
//     owns members 32 half .. 32 half + 31 of tile row `row` (warps w and
//     w + 4 share TMEM lane quarter w); the halves exchange their row maxima
//     through shared memory so the whole row has one digit scale;
//   * A digits a2 | a1 | a0 in TMEM (3 x 32 columns, 4 per column), gate
//     digits [b2 | b1 | b0] (384 rows x 128 B = one SW128 K block, 48 KB),
//     accumulators hi | mid | lo (3 x 128 columns): the CTA owns all 512;
//       [hi | mid] += a2 [b2 | b1]   (N = 256)    lo += a2 b0   (N = 128)
//       [mid | lo] += a1 [b2 | b1]   (N = 256)    lo += a0 b2   (N = 128)
//     4 K steps x 4 = 16 MMAs per 128-row tile (64 KB of state);
//   * hi and mid start at the float bits of 1.5 * 2^23 (read back as floats),
//     lo starts at zero (its K = 128 sum may exceed the magic's 2^22 range)
//     and is converted with I2FP;
//   * 2-stage cp.async ring (one 64 KB tile in flight while one is consumed).
#include <cmath>
#include <cstring>

#include "common.cuh"
#include "launch.h"
#include "tcgen05.cuh"

namespace dsv {

using namespace tcx;

struct Tc68P {
  Geom g;
  uint64_t ntiles;
  int nnib;
  int e_b;
  int emin, emax;
  int coop;
  int tshift;
  int jpos;  // PAIR copies: thread-index bit that selects the member parity
  int row2;  // !PAIR, index bit 0 the lowest target: member pairs (2m, 2m+1) move as 16-byte units
  int nib_shift[16];
  uint64_t offs[64];
  float4 ctab[kTcMaxNib * 16 * 2];
};

struct Tc68Layout {
  static constexpr int D = 64;
  static constexpr int N0 = 128;               // reals per row
  static constexpr int KSTEPS = 4;             // K = 128 int8 = 4 x 32
  static constexpr int B_BYTES = 3 * 128 * 128;  // [b2 | b1 | b0] rows of 128 B (SW128)
  static constexpr int BAR = B_BYTES;          // MMA mbarrier + TMEM slot + accumulator start value
  static constexpr int PBUF = BAR + 128;       // tile-uniform phase factors [64] float2
  static constexpr int MX = PBUF + 64 * 8;     // row maxima [half][row] float
  static constexpr int RING = (MX + 2 * 128 * 4 + 1023) / 1024 * 1024;
  static constexpr int STAGE = 128 * D * 8;    // 64 KB
  static constexpr int SMEM_MAX = 227 * 1024 - 1024;
  static constexpr int NSTAGE = (SMEM_MAX - RING) / STAGE;
  static_assert(NSTAGE >= 2, "ring must hold two 64 KB tiles");
  static constexpr int BYTES = RING + NSTAGE * STAGE;
  static constexpr int T_A = 0;                // digit l at 32 l
  static constexpr int T_HI = 128, T_MID = 256, T_LO = 384;
};

constexpr uint32_t kAcc68Init = 0x4B400000u;           // float bits of 1.5 * 2^23
constexpr uint32_t kDigit68Off = 0x8080u - 0x4B400000u;  // float bits of M + I -> I + 0x8080

__device__ __forceinline__ void issue_mma68(uint32_t sbase) {
  using L = Tc68Layout;
  constexpr uint32_t ID2 = idesc_i8<256, 1, 1>(), ID1 = idesc_i8<128, 1, 1>();
#pragma unroll
  for (int s = 0; s < L::KSTEPS; ++s) {
    const uint64_t b21 = sw128_desc(sbase + s * 32);              // rows 0..255: b2 | b1
    const uint64_t b0 = sw128_desc(sbase + 256 * 128 + s * 32);   // rows 256..383: b0
    const uint32_t ta = L::T_A + s * 8;
    mma_ts_i8(L::T_HI, ta + 0 * 32, b21, ID2, 1u);                 // [hi | mid] += a2 [b2 | b1]
    mma_ts_i8(L::T_LO, ta + 0 * 32, b0, ID1, s > 0 ? 1u : 0u);     // lo (+)= a2 b0 (zeroes lo first)
    mma_ts_i8(L::T_MID, ta + 1 * 32, b21, ID2, 1u);                // [mid | lo] += a1 [b2 | b1]
    mma_ts_i8(L::T_LO, ta + 2 * 32, b21, ID1, 1u);                 // lo += a0 b2
  }
}

template <bool PHASED, bool PAIR>
__global__ void __launch_bounds__(256, 1)
k_dense_tc68(const __grid_constant__ Tc68P p, const uint4* __restrict__ bmat, const float4* __restrict__ tab,
             float2* __restrict__ sv) {
  using L = Tc68Layout;
  constexpr int S = L::NSTAGE;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t raw_base = smem_u32(smem_raw);
  const uint32_t sbase = (raw_base + 1023u) & ~1023u;
  unsigned char* sm = smem_raw + (sbase - raw_base);
  const int tid = threadIdx.x;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);  // warp-uniform (TMEM addresses in uniform registers)
  const int row = tid & 127;
  const int half = tid >> 7;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + L::BAR + 16);
  const uint32_t bar = sbase + L::BAR;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid < 2) reinterpret_cast<uint32_t*>(sm + L::BAR + 32)[tid] = kAcc68Init;
  if (tid == 32) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // gate digits, host layout [384 rows][8 x 16 B] -> 128-byte swizzled rows
  for (int i = tid; i < 384 * 8; i += 256) {
    const int r = i / 8, c16 = i % 8;
    *reinterpret_cast<uint4*>(sm + r * 128 + ((c16 ^ (r & 7)) << 4)) = bmat[i];
  }

  const uint64_t step = gridDim.x;
  auto tile_of = [&](int i) { return uint64_t(blockIdx.x) + uint64_t(i) * step; };
  const uint64_t e0 = expand(p.g, 0);
  const uint64_t rowoff = expand(p.g, row) ^ e0;
  // PAIR: thread moves rows (2p, 2p+1) of members j = 4 jj + jq (16-byte
  // copies).  As in tc8.cu, thread-index bit jpos (= lowest target - 1,
  // capped at 6) picks the member parity, so with the lowest target at bit 1
  // adjacent lanes fetch the two halves of one 32-byte sector (whole sectors
  // per lane pair; the window's time barely moves: 16.6 -> 16.2 ms at n = 32)
  const int pp = tid & 127;
  const int prow = 2 * ((pp & ((1 << p.jpos) - 1)) | ((pp >> (p.jpos + 1)) << p.jpos));
  const int jq = 2 * (tid >> 7) + ((pp >> p.jpos) & 1);
  const uint64_t prowoff = expand(p.g, prow) ^ e0;
  auto issue = [&](int i) -> uint64_t {
    const uint64_t tl = tile_of(i);
    uint64_t tb = 0;
    if (tl < p.ntiles) {
      tb = expand(p.g, tl * 128);
      const uint32_t st0 = sbase + L::RING + (i % S) * L::STAGE;
      if constexpr (PAIR) {
        const uint64_t b = tb | prowoff;
        if (p.tshift >= 0) {
          const float2* src = sv + b + (uint64_t(jq) << p.tshift);
          const uint64_t stride = uint64_t(4) << p.tshift;
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) cp_async16(st0 + (4 * jj + jq) * 1024 + prow * 8, src + jj * stride);
        } else {
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) {
            const int j = 4 * jj + jq;
            cp_async16(st0 + j * 1024 + prow * 8, sv + b + p.offs[j]);
          }
        }
      } else if (p.row2) {  // index bit 0 the lowest target: [member pair][row] x 16 B
        const uint64_t b = tb | rowoff;
#pragma unroll
        for (int mm = 0; mm < 16; ++mm) {
          const int m = 16 * half + mm;
          cp_async16(st0 + m * 2048 + row * 16, sv + b + p.offs[2 * m]);
        }
      } else {  // index bit 0 a target or control: this thread's half row, 8 B per member
        const uint64_t b = tb | rowoff;
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) {
          const int j = 32 * half + jj;
          cp_async8(st0 + j * 1024 + row * 8, sv + b + p.offs[j]);
        }
      }
    }
    cp_async_commit();
    return tb;
  };
  auto phase_angles = [&](uint64_t b, float (&a)[8], bool from_const) {
#pragma unroll
    for (int s = 0; s < 8; ++s) a[s] = 0.f;
#pragma unroll
    for (int c = 0; c < kTcMaxNib; ++c) {
      if (c < p.nnib) {
        const int r = (c * 16 + int((b >> p.nib_shift[c]) & 15u)) * 2;
        const float4 x = from_const ? p.ctab[r] : __ldg(tab + r);
        const float4 y = from_const ? p.ctab[r + 1] : __ldg(tab + r + 1);
        a[0] += x.x; a[1] += x.y; a[2] += x.z; a[3] += x.w;
        a[4] += y.x; a[5] += y.y; a[6] += y.z; a[7] += y.w;
      }
    }
  };
  // tile-uniform phases: the last warp's 32 lanes x 2 compute the 64 factors of tile i
  float2* Pb = reinterpret_cast<float2*>(sm + L::PBUF);
  auto coop_phase = [&](int i, uint64_t tb) {
    if (PHASED && p.coop && warp == 7 && tile_of(i) < p.ntiles) {
      float a[8];
      phase_angles(tb, a, true);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = (tid & 31) + 32 * h;
        float ang = a[6];
#pragma unroll
        for (int m = 0; m < 6; ++m) ang += ((j >> m) & 1) ? a[m] : 0.f;
        float sn, cs;
        sincos_unit(ang, &sn, &cs);
        Pb[j] = make_float2(cs, sn);
      }
    }
  };
  float* mxs = reinterpret_cast<float*>(sm + L::MX);

  uint64_t tq = issue(0);
  coop_phase(0, tq);
  cp_async_wait<0>();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  fence_before();
  __syncthreads();
  fence_after();
  if (*tmem_slot != 0u) __trap();
  const uint32_t tlane = uint32_t((warp & 3) * 32) << 16;
  uint32_t mg[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) mg[i] = reinterpret_cast<const uint32_t*>(sm + L::BAR + 32)[i & 1];

  // out = scale (hi 2^16 + mid 2^8 + lo): hi and mid read back as M + acc,
  // lo is a plain int32; t2 = V + 256 M, removed by the last fma
  auto combine = [](float h, float m, float l, float scale, float cm) {
    const float t1 = __fmaf_rn(__fadd_rn(h, -kMagic), 256.f, m);
    return __fmaf_rn(__fmaf_rn(t1, 256.f, l), scale, cm);
  };
  auto epilogue = [&](uint64_t b, float scale, float cm) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int col = 64 * half + 32 * h;  // members 32 half + 16 h .. + 15
      float ch[32], cmid[32], cl[32];
      tmem_ld32(tlane + uint32_t(L::T_HI + col), ch);
      tmem_ld32(tlane + uint32_t(L::T_MID + col), cmid);
      tmem_ld32(tlane + uint32_t(L::T_LO + col), cl);
      auto val = [&](int c) {
        return combine(ch[c], cmid[c], __int2float_rn(__float_as_int(cl[c])), scale, cm);
      };
      const int jb = 32 * half + 16 * h;
      if (!PAIR && p.row2) {  // member pairs (2m, 2m+1) are adjacent amplitudes: 16-byte stores
#pragma unroll
        for (int i = 0; i < 8; ++i)
          __stcs(reinterpret_cast<float4*>(sv + b + p.offs[jb + 2 * i]),
                 make_float4(val(4 * i), val(4 * i + 1), val(4 * i + 2), val(4 * i + 3)));
      } else if (PAIR && p.jpos == 0) {
        // lowest target at bit 1: rows (r, r+1) x members (m, m+1) are one
        // 32-byte sector held by lanes r, r+1 — swap one value per lane pair
        // and store 16 bytes each (even lane: member m of both rows, odd: m+1)
        const bool odd = row & 1;
        const uint64_t be = b - (odd ? 1 : 0);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float o0 = val(4 * q), o1 = val(4 * q + 1), o2 = val(4 * q + 2), o3 = val(4 * q + 3);
          const float sx = odd ? o0 : o2, sy = odd ? o1 : o3;
          const float rx = __shfl_xor_sync(0xffffffffu, sx, 1), ry = __shfl_xor_sync(0xffffffffu, sy, 1);
          const float4 w = odd ? make_float4(rx, ry, o2, o3) : make_float4(o0, o1, rx, ry);
          const uint64_t oj = odd ? p.offs[jb + 2 * q + 1] : p.offs[jb + 2 * q];
          __stcs(reinterpret_cast<float4*>(sv + be + oj), w);
        }
      } else if (p.tshift >= 0) {
        float2* dst = sv + b + (uint64_t(jb) << p.tshift);
        const uint64_t stride = uint64_t(1) << p.tshift;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          __stcs(dst, make_float2(val(2 * i), val(2 * i + 1)));
          dst += stride;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) __stcs(sv + b + p.offs[jb + i], make_float2(val(2 * i), val(2 * i + 1)));
      }
    }
  };

  uint64_t prev_base = 0;
  float prev_scale = 0.f, prev_cm = 0.f;
  int it = 0;
#pragma unroll 1
  for (;; ++it) {
    const uint64_t tile = tile_of(it);
    if (tile >= p.ntiles) break;
    const uint64_t tb_cur = tq;
    tq = issue(it + 1);
    const uint64_t base = tb_cur | rowoff;
    const float2* raw = reinterpret_cast<const float2*>(sm + L::RING + (it % S) * L::STAGE) + row;
    float2 v[32];
    if (!PAIR && p.row2) {
      const float4* raw2 = reinterpret_cast<const float4*>(sm + L::RING + (it % S) * L::STAGE) + row;
#pragma unroll
      for (int mm = 0; mm < 16; ++mm) {
        const float4 x = raw2[(16 * half + mm) * 128];
        v[2 * mm] = make_float2(x.x, x.y);
        v[2 * mm + 1] = make_float2(x.z, x.w);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = raw[(32 * half + j) * 128];
    }
    if constexpr (PHASED) {
      if (p.coop) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float2 x = v[j], f = Pb[32 * half + j];
          v[j] = make_float2(x.x * f.x - x.y * f.y, x.x * f.y + x.y * f.x);
        }
      } else {
        float a[8];
        phase_angles(base, a, false);
        float2 P[32];
        float es, ec;
        sincos_red(a[6] + (half ? a[5] : 0.f), &P[0].y, &P[0].x);
#pragma unroll
        for (int m = 0; m < 5; ++m) {
          sincos_red(a[m], &es, &ec);
#pragma unroll
          for (int j = 0; j < (1 << m); ++j) {
            const float2 q = P[j];
            P[j + (1 << m)] = make_float2(q.x * ec - q.y * es, q.x * es + q.y * ec);
          }
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float2 x = v[j];
          v[j] = make_float2(x.x * P[j].x - x.y * P[j].y, x.x * P[j].y + x.y * P[j].x);
        }
      }
    }
    float mx = 0.f;
#pragma unroll
    for (int j = 0; j < 32; ++j) mx = fmaxf(mx, fmaxf(fabsf(v[j].x), fabsf(v[j].y)));
    mxs[half * 128 + row] = mx;
    __syncthreads();  // B1: both halves' maxima (and every P read above) done
    mx = fmaxf(mx, mxs[(half ^ 1) * 128 + row]);
    coop_phase(it + 1, tq);  // next tile's factors; P was read before B1, published by B2
    const int e_row = min(max(int((__float_as_uint(mx) >> 23) & 0xFF) - 126, p.emin), p.emax);
    const float sc_in = pow2f(22 - e_row);
    const float scale = pow2f(e_row + p.e_b - 29);
    const float cm = -3.f * pow2f(e_row + p.e_b + 1);  // -256 M scale
    // digits of this thread's 32 members: word c = (re, im) of members 2c, 2c+1
    uint32_t la[3][16];
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const uint32_t w0 = __float_as_uint(__fmaf_rn(v[2 * c].x, sc_in, kMagic)) + kDigit68Off;
      const uint32_t w1 = __float_as_uint(__fmaf_rn(v[2 * c].y, sc_in, kMagic)) + kDigit68Off;
      const uint32_t w2 = __float_as_uint(__fmaf_rn(v[2 * c + 1].x, sc_in, kMagic)) + kDigit68Off;
      const uint32_t w3 = __float_as_uint(__fmaf_rn(v[2 * c + 1].y, sc_in, kMagic)) + kDigit68Off;
      const uint32_t p01 = __byte_perm(w0, w1, 0x5140), p23 = __byte_perm(w2, w3, 0x5140);
      la[2][c] = __byte_perm(p01, p23, 0x5410) ^ 0x80808080u;
      la[1][c] = __byte_perm(p01, p23, 0x7632) ^ 0x80808080u;
      la[0][c] = __byte_perm(__byte_perm(w0, w1, 0x0062), __byte_perm(w2, w3, 0x0062), 0x5410);
    }
    if (it > 0) {  // MMA(i-1) done: A is free and its accumulators are ready
      mbar_wait(bar, (it - 1) & 1);
      fence_after();
      epilogue(prev_base, prev_scale, prev_cm);
    }
    // hi and mid back to M (this thread's 2 x 64 columns); lo is zeroed by the first MMA
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      tmem_st8(tlane + uint32_t(L::T_HI + 64 * half + 8 * q), mg);
      tmem_st8(tlane + uint32_t(L::T_MID + 64 * half + 8 * q), mg);
    }
#pragma unroll
    for (int l = 0; l < 3; ++l) tmem_st16(tlane + uint32_t(L::T_A + 32 * l + 16 * half), la[l]);
    cp_async_wait<0>();  // tile i+1 landed (this thread's part)
    tmem_wait_st();
    fence_before();
    __syncthreads();  // B2
    if (tid == 0) {
      fence_after();
      issue_mma68(sbase);
      mma_commit(bar);
    }
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

template <bool PHASED, bool PAIR>
static cudaError_t tc68_go(const TcDesc& d, const void* d_bmat, const void* d_tab, void* sv, cudaStream_t st) {
  using L = Tc68Layout;
  Tc68P p;
  std::memset(&p, 0, sizeof p);
  p.g = d.g;
  p.ntiles = d.g.nwork / 128;
  p.nnib = d.nnib;
  p.e_b = d.e_b;
  // every power of two the kernel forms stays normal: 22 - e_row, e_row + e_b - 29, 3 * 2^(e_row + e_b + 1)
  p.emin = std::max(-100, -97 - d.e_b);
  p.emax = std::min(100, 124 - d.e_b);
  p.coop = d.coop;
  p.tshift = d.tshift;
  p.row2 = d.mode == kTcRow2 ? 1 : 0;
  p.jpos = 6;
  for (int lo = 0; lo < 7; ++lo)  // lowest target bit = lowest set bit of offs[1]
    if (d.offs[1] == (uint64_t(1) << lo)) p.jpos = lo >= 1 ? std::min(lo - 1, 6) : 6;
  for (int c = 0; c < 16; ++c) p.nib_shift[c] = d.nib_shift[c];
  for (int j = 0; j < 64; ++j) p.offs[j] = d.offs[j];
  if (d.htab && d.nnib > 0) std::memcpy(p.ctab, d.htab, size_t(d.nnib) * 16 * 2 * sizeof(float4));
  const int smem = L::BYTES + 1024;
  static bool attr_set[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_dense_tc68<PHASED, PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr_set[dev] = true;
  }
  uint64_t blocks = uint64_t(device_sm_count());
  if (blocks > p.ntiles) blocks = p.ntiles;
  if (blocks == 0) return cudaSuccess;
  k_dense_tc68<PHASED, PAIR><<<unsigned(blocks), 256, smem, st>>>(p, static_cast<const uint4*>(d_bmat),
                                                                  static_cast<const float4*>(d_tab),
                                                                  static_cast<float2*>(sv));
  return cudaGetLastError();
}

cudaError_t launch_dense_tc68(const TcDesc& d, const void* d_bmat, const void* d_tab, void* sv, cudaStream_t st) {
  const bool ph = d.nnib > 0;
  if (d.mode == kTcPair) return ph ? tc68_go<true, true>(d, d_bmat, d_tab, sv, st) : tc68_go<false, true>(d, d_bmat, d_tab, sv, st);
  return ph ? tc68_go<true, false>(d, d_bmat, d_tab, sv, st) : tc68_go<false, false>(d, d_bmat, d_tab, sv, st);
}

}  // namespace dsv
