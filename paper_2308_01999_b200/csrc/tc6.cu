// tc6.cu — 6-qubit complex64 windows (plain or with the fold fuser's
// pre-phase) on the tensor cores.  Same arithmetic as tc.cu (exact bf16
// integer limbs, partial sums below 2^23, two TMEM accumulators combined with
// round-to-nearest FMAs), re-laid out for a 64-member group:
//
//   * one persistent CTA per SM, ONE group of 256 threads: thread (row, half)
//     owns members 32 half .. 32 half + 31 of tile row `row` (warps w and
//     w + 4 share TMEM lane quarter w), so per-thread registers match the
//     k = 5 kernel; the two halves exchange their row maxima through shared
//     memory (one extra barrier) so the whole row has one limb scale;
//   * A limbs a0, a1, a2 / 2^8, a1 / 2^8 in TMEM (4 x 64 columns), gate limbs
//     b0, b1, b2 / 2^8 (96 KB, K-block-major SW128), accumulators acc0 |
//     acc12 (2 x 128 columns): the CTA owns all 512 TMEM columns;
//       [acc0 | acc12] = a0 [b0 | b1]            (N = 256)
//       acc12 += a0 b2' + a1 b0 + a1' b1 + a2' b0 (N = 128)
//     8 K steps x 5 = 40 MMAs per 128-row tile (64 KB of state);
//   * 2-stage cp.async ring (one 64 KB tile in flight while one is consumed).
//
// Replaces apply_dense_bits (reference statevec.py:44-60) for 6-qubit fused
// windows, which the CUDA-core path can only run through its generic
// one-CTA-per-group kernel.
#include <cmath>
#include <cstring>

#include "common.cuh"
#include "launch.h"
#include "tcgen05.cuh"

namespace dsv {

using namespace tcx;

struct Tc6P {
  Geom g;
  uint64_t ntiles;
  int nnib;
  int e_b;
  int coop;
  int nib_shift[16];
  uint64_t offs[64];
  float4 ctab[kTcMaxNib * 16 * 2];
};

struct Tc6Layout {
  static constexpr int D = 64;
  static constexpr int N = 128;
  static constexpr int KSTEPS = 8;
  static constexpr int B_KB = 3 * 128 * 128;  // one 128-byte K block of all three limbs
  static constexpr int B0 = 0;                // [kb 0..1][limb 0..2][row 0..127] x 128 B
  static constexpr int BAR = 2 * B_KB;        // MMA mbarrier + TMEM slot
  static constexpr int PBUF = BAR + 128;      // tile-uniform phase factors [64] float2
  static constexpr int MX = PBUF + 64 * 8;    // row maxima [half][row] float
  static constexpr int RING = MX + 2 * 128 * 4;
  static constexpr int STAGE = 128 * D * 8;   // 64 KB
  static constexpr int SMEM_MAX = 227 * 1024 - 1024;
  static constexpr int NSTAGE = (SMEM_MAX - RING) / STAGE;
  static_assert(NSTAGE >= 2, "ring must hold two 64 KB tiles");
  static constexpr int BYTES = RING + NSTAGE * STAGE;
  static constexpr int T_A = 0;               // limbs at 0, 64, 128, 192
  static constexpr int T_ACC0 = 256;
  static constexpr int T_ACC12 = 384;
};

__device__ __forceinline__ void issue_mma6(uint32_t sbase) {
  using L = Tc6Layout;
  constexpr uint32_t ID1 = idesc_bf16<128>(), ID2 = idesc_bf16<256>();
#pragma unroll
  for (int s = 0; s < L::KSTEPS; ++s) {
    const uint32_t bk = sbase + L::B0 + (s >> 2) * L::B_KB + (s & 3) * 32;
    const uint32_t ta = L::T_A + s * 8;
    mma_ts(L::T_ACC0, ta + 0 * 64, sw128_desc(bk + 0 * 16384), ID2, s > 0);  // a0 [b0 | b1]
    mma_ts(L::T_ACC12, ta + 0 * 64, sw128_desc(bk + 2 * 16384), ID1, 1u);    // a0 b2'
    mma_ts(L::T_ACC12, ta + 1 * 64, sw128_desc(bk + 0 * 16384), ID1, 1u);    // a1 b0
    mma_ts(L::T_ACC12, ta + 3 * 64, sw128_desc(bk + 1 * 16384), ID1, 1u);    // a1' b1
    mma_ts(L::T_ACC12, ta + 2 * 64, sw128_desc(bk + 0 * 16384), ID1, 1u);    // a2' b0
  }
}

template <bool PHASED, bool PAIR>
__global__ void __launch_bounds__(256, 1)
k_dense_tc6(const __grid_constant__ Tc6P p, const uint4* __restrict__ bmat, const float4* __restrict__ tab,
            float2* __restrict__ sv) {
  using L = Tc6Layout;
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
  if (tid == 32) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // gate limbs, host layout [3][128 rows][128 cols] bf16 -> [kb][limb][row] swizzled 128-byte rows
  for (int i = tid; i < 3 * 128 * 16; i += 256) {
    const int limb = i / (128 * 16);
    const int r = (i / 16) % 128;
    const int c16 = i % 16;
    const int off = L::B0 + (c16 >> 3) * L::B_KB + limb * 16384 + r * 128 + (((c16 & 7) ^ (r & 7)) << 4);
    *reinterpret_cast<uint4*>(sm + off) = bmat[i];
  }

  const uint64_t step = gridDim.x;
  auto tile_of = [&](int i) { return uint64_t(blockIdx.x) + uint64_t(i) * step; };
  const uint64_t e0 = expand(p.g, 0);
  const uint64_t rowoff = expand(p.g, row) ^ e0;
  // PAIR: thread moves rows (2p, 2p+1) of members j = 4 jj + quarter (16-byte copies)
  const int prow = 2 * (tid & 63);
  const int jq = tid >> 6;
  const uint64_t prowoff = expand(p.g, prow) ^ e0;
  auto issue = [&](int i) -> uint64_t {
    const uint64_t tl = tile_of(i);
    uint64_t tb = 0;
    if (tl < p.ntiles) {
      tb = expand(p.g, tl * 128);
      const uint32_t st0 = sbase + L::RING + (i % S) * L::STAGE;
      if constexpr (PAIR) {
        const uint64_t b = tb | prowoff;
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const int j = 4 * jj + jq;
          cp_async16(st0 + j * 1024 + prow * 8, sv + b + p.offs[j]);
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
  const bool odd = row & 1;

  // out = 2^(e_row + e_b - 16) (acc0 + acc12 / 2^8): this thread's 32 members
  auto epilogue = [&](uint64_t b, float scale) {
    const uint64_t be = b - (odd ? 1 : 0);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int col = 64 * half + 32 * h;  // members 32 half + 16 h .. + 15
      float c0[32], c1[32];
      tmem_ld32(tlane + uint32_t(L::T_ACC0 + col), c0);
      tmem_ld32(tlane + uint32_t(L::T_ACC12 + col), c1);
      const int jb = 32 * half + 16 * h;
      if constexpr (PAIR) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float o[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) o[c] = __fmaf_rn(c1[4 * q + c], 1.f / 256.f, c0[4 * q + c]) * scale;
          const float sx = odd ? o[0] : o[2], sy = odd ? o[1] : o[3];
          const float rx = __shfl_xor_sync(0xffffffffu, sx, 1), ry = __shfl_xor_sync(0xffffffffu, sy, 1);
          const uint64_t oj = odd ? p.offs[jb + 2 * q + 1] : p.offs[jb + 2 * q];
          const float4 w = odd ? make_float4(rx, ry, o[2], o[3]) : make_float4(o[0], o[1], rx, ry);
          __stcs(reinterpret_cast<float4*>(sv + be + oj), w);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float re = __fmaf_rn(c1[2 * i], 1.f / 256.f, c0[2 * i]) * scale;
          const float im = __fmaf_rn(c1[2 * i + 1], 1.f / 256.f, c0[2 * i + 1]) * scale;
          __stcs(sv + b + p.offs[jb + i], make_float2(re, im));
        }
      }
    }
  };

  uint64_t prev_base = 0;
  float prev_scale = 0.f;
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
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = raw[(32 * half + j) * 128];
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
    const int e_row = min(max(int((__float_as_uint(mx) >> 23) & 0xFF) - 126, -100), 120);
    const float s8 = pow2f(8 - e_row), s16 = pow2f(16 - e_row);
    const float scale = pow2f(e_row + p.e_b - 16);
    if (it > 0) {
      mbar_wait(bar, (it - 1) & 1);
      fence_after();
      epilogue(prev_base, prev_scale);
    }
    // limbs of this thread's 32 members -> TMEM columns 32 half .. + 31 of each limb
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint32_t l0[16], l1[16], l2[16], l3[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        float a0[2], a1[2], a2[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const float x = c ? v[h * 16 + q].y : v[h * 16 + q].x;
          a0[c] = __fadd_rn(__fmaf_rn(x, s8, kMagic), -kMagic);
          const float r1 = __fmaf_rn(a0[c], -256.f, x * s16);
          a1[c] = __fadd_rn(__fadd_rn(r1, kMagic), -kMagic);
          a2[c] = __fadd_rn(__fadd_rn(__fadd_rn(r1, -a1[c]), kMagic16), -kMagic16);
        }
        l0[q] = pack2(a0[0], a0[1]);
        l1[q] = pack2(a1[0], a1[1]);
        l2[q] = pack2(a2[0], a2[1]);
        l3[q] = pack2(a1[0] * (1.f / 256.f), a1[1] * (1.f / 256.f));
      }
      const uint32_t c = uint32_t(32 * half + 16 * h);
      tmem_st16(tlane + L::T_A + 0 * 64 + c, l0);
      tmem_st16(tlane + L::T_A + 1 * 64 + c, l1);
      tmem_st16(tlane + L::T_A + 2 * 64 + c, l2);
      tmem_st16(tlane + L::T_A + 3 * 64 + c, l3);
    }
    cp_async_wait<0>();  // tile i+1 landed (this thread's part)
    tmem_wait_st();
    fence_before();
    __syncthreads();  // B2
    if (tid == 0) {
      fence_after();
      issue_mma6(sbase);
      mma_commit(bar);
    }
    prev_base = base;
    prev_scale = scale;
  }
  if (it > 0) {
    mbar_wait(bar, (it - 1) & 1);
    fence_after();
    epilogue(prev_base, prev_scale);
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
static cudaError_t tc6_go(const TcDesc& d, const void* d_bmat, const void* d_tab, void* sv, cudaStream_t st) {
  using L = Tc6Layout;
  Tc6P p;
  std::memset(&p, 0, sizeof p);
  p.g = d.g;
  p.ntiles = d.g.nwork / 128;
  p.nnib = d.nnib;
  p.e_b = d.e_b;
  p.coop = d.coop;
  for (int c = 0; c < 16; ++c) p.nib_shift[c] = d.nib_shift[c];
  for (int j = 0; j < 64; ++j) p.offs[j] = d.offs[j];
  if (d.htab && d.nnib > 0) std::memcpy(p.ctab, d.htab, size_t(d.nnib) * 16 * 2 * sizeof(float4));
  const int smem = L::BYTES + 1024;
  static bool attr_set[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_dense_tc6<PHASED, PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr_set[dev] = true;
  }
  uint64_t blocks = uint64_t(device_sm_count());
  if (blocks > p.ntiles) blocks = p.ntiles;
  if (blocks == 0) return cudaSuccess;
  k_dense_tc6<PHASED, PAIR><<<unsigned(blocks), 256, smem, st>>>(p, static_cast<const uint4*>(d_bmat),
                                                                 static_cast<const float4*>(d_tab),
                                                                 static_cast<float2*>(sv));
  return cudaGetLastError();
}

cudaError_t launch_dense_tc6(const TcDesc& d, const void* d_bmat, const void* d_tab, void* sv, cudaStream_t st) {
  const bool ph = d.nnib > 0;
  if (d.mode == kTcPair) return ph ? tc6_go<true, true>(d, d_bmat, d_tab, sv, st) : tc6_go<false, true>(d, d_bmat, d_tab, sv, st);
  return ph ? tc6_go<true, false>(d, d_bmat, d_tab, sv, st) : tc6_go<false, false>(d, d_bmat, d_tab, sv, st);
}

}  // namespace dsv
