// tc.cu — k = 4/5-qubit dense gates (optionally with the fold fuser's
// outside-coupled pre-phase) on the 5th-generation tensor cores, complex64.
//
// Replaces apply_dense_bits (reference statevec.py:44-60) for fused windows
// whose 2^k x 2^k complex product is FMA-bound on the CUDA cores (k = 5 needs
// 16 flop/B, i.e. ~100 TFLOP/s of FP32 FMA at HBM speed — more than the
// CUDA cores have).
//
// Arithmetic: exact-integer tensor-core products (Ozaki-style split).  A row
// of the tile (one amplitude group, 2^(k+1) reals) is scaled by its own power
// of two so |y| < 256 and rounded to 24 significant bits as bf16 integer
// limbs y = a0 + a1/2^8 + a2/2^16 (|a0| <= 256, |a1|, |a2| <= 128); the gate's
// real embedding is split the same way with one global exponent.
// tcgen05.mma.kind::f16 (bf16 in, fp32 accumulate) then sums
//   acc0  = sum a0 b0                                  (integers < 2^22: exact)
//   acc12 = sum a0 b1 + a1 b0 + (a0 b2 + a1 b1 + a2 b0) / 2^8
// (integer part < 2^23, so the tensor core's truncating accumulation can only
// drop bits 2^-31 below the result), and the epilogue forms
// 2^(e_row + e_b - 16) (acc0 + acc12 / 2^8) with round-to-nearest FMAs.
// fp32-level accuracy without the systematic norm drift of a 3xTF32 split
// (measured -2e-6 per gate from accumulator truncation; this path: ~1e-8).
//
// Dataflow (one persistent CTA per SM, 256 threads = two independent groups
// of 128; in a group thread t = row t = group t of a 128-group tile; the two
// groups take alternate tiles and share the gate operand in shared memory):
//   * per-group ring of S raw tiles in shared memory, filled by cp.async
//     (16 B = one member of two adjacent groups, coalesced), S-1 tiles of
//     loads always in flight;
//   * thread t: phase polynomial in registers (phased windows), row exponent,
//     limb split, tcgen05.st of its own TMEM lane (the A operand lives in
//     tensor memory: no shared-memory staging, no swizzle, no bank conflicts);
//   * thread 0 of the group issues 20 MMAs (M = 128, N = 2^(k+1..k+2), K = 16)
//     and commits to the group's mbarrier; the MMAs overlap the next tile's
//     copy issue and phase work and the other group's work; then each thread
//     reads its TMEM lane (tcgen05.ld 32x32b) and streams its 2^k outputs out.
#include <cmath>
#include <cstring>

#include "common.cuh"
#include "launch.h"
#include "tcgen05.cuh"

namespace dsv {

using namespace tcx;

template <int K>
struct TcP {
  Geom g;                 // groups (amplitude index space, holes = targets + controls)
  uint64_t ntiles;        // g.nwork / 128
  int nnib;               // phase-table nibbles (0: plain dense)
  int e_b;                // gate limb exponent: |B| < 2^e_b
  int coop;               // phase uniform over a tile's 128 rows: computed once per tile
  int nnib_row;           // leading nibbles that vary over the rows (the rest: tile-uniform sums)
  int nib_shift[16];      // amplitude-index shift of nibble c
  uint64_t offs[1 << K];  // member offsets (amplitudes)
  // tile-uniform (coop) phase table in the kernel-parameter constant bank:
  // every lane of the computing warp reads the same entries (broadcast), no
  // global-memory latency on the path to the group barrier
  float4 ctab[kTcMaxNib * 16 * 2];
};

template <int K>
struct TcLayout {
  static constexpr int D = 1 << K;
  static constexpr int N = 2 * D;                 // GEMM N = real outputs, K = real inputs
  static constexpr int KSTEPS = N / 16;           // MMA K = 16 (bf16)
  static constexpr int NBL = 4;                   // B limbs: b0, b1, b2 / 2^8, b1 / 2^8
  static constexpr int B_LIMB = N * 128;          // one limb: N rows of one 128-byte bf16 row (K <= 64)
  static constexpr int B0 = 0;
  static constexpr int BAR = B0 + NBL * B_LIMB;   // 2 mbarriers + TMEM slot
  static constexpr int PBUF = BAR + 128;          // tile-uniform phases: [group][2][D] float2
  static constexpr int RING = PBUF + 2 * 2 * D * 8;  // raw tiles: [group][stage][member j][row t] float2
  static constexpr int STAGE = 128 * D * 8;
  static constexpr int SMEM_MAX = 227 * 1024 - 1024;  // minus the 1 KB alignment slack
  static constexpr int NS_FIT = (SMEM_MAX - RING) / (2 * STAGE);
  static constexpr int NSTAGE = NS_FIT > 6 ? 6 : NS_FIT;  // per group
  static_assert(NSTAGE >= 3, "ring must hold three tiles per group");
  static_assert(N <= 64, "B operand is one 128-byte K block");
  static constexpr int BYTES = RING + 2 * NSTAGE * STAGE;
  // TMEM per group (256 columns): A limbs a0, a1, a2 / 2^8 (D columns each:
  // one complex member = two bf16 per 32-bit column), acc0, acc12
  static constexpr int T_A = 0;
  static constexpr int T_ACC0 = 128;
  static constexpr int T_ACC12 = T_ACC0 + N;     // adjacent: one N = 2^(k+2) MMA fills both
  static_assert(3 * D <= T_ACC0 && T_ACC12 + N <= 256, "TMEM plan");
};

// The group's 20 MMAs for one tile (thread 0 of the group).  TMEM addresses
// are compile-time constants (the CTA owns all 512 columns, base 0, checked at
// start).
//   [acc0 | acc12]  = a0 [b0 | b1]             (one N = 2^(k+2) MMA per K step)
//   acc12          += a0 b2' + a1 b0 + a1 b1' + a2' b0      (' = / 2^8)
template <int K, int GRP>
__device__ __forceinline__ void issue_mma(uint32_t sbase) {
  using L = TcLayout<K>;
  constexpr int D = L::D;
  constexpr int N = L::N;
  constexpr uint32_t T0 = GRP * 256;
  constexpr uint32_t ID1 = idesc_bf16<N>(), ID2 = idesc_bf16<2 * N>();
  const uint32_t bs = sbase + L::B0;
#pragma unroll
  for (int s = 0; s < L::KSTEPS; ++s)
    mma_ts(T0 + L::T_ACC0, T0 + L::T_A + 0 * D + s * 8, sw128_desc(bs + 0 * L::B_LIMB + s * 32), ID2, s > 0);
  constexpr int al[4] = {0, 1, 1, 2};
  constexpr int bl[4] = {2, 0, 3, 0};
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int s = 0; s < L::KSTEPS; ++s)
      mma_ts(T0 + L::T_ACC12, T0 + L::T_A + al[q] * D + s * 8, sw128_desc(bs + bl[q] * L::B_LIMB + s * 32), ID1,
             1u);
}

// Per group and iteration i (the group's i-th tile):
//   issue tile i+S-1's member copies (cp.async into its ring stage)
//   wait for tile i's copies; phase-multiply in registers; row exponent
//   wait MMA(i-1); epilogue(i-1): TMEM accumulators -> HBM
//   limbs of tile i -> TMEM (A); group barrier; thread 0 issues MMA(i), commit
template <int K, bool PHASED, int MODE>
__global__ void __launch_bounds__(256, 1)
k_dense_tc(const __grid_constant__ TcP<K> p, const uint4* __restrict__ bmat, const float4* __restrict__ tab,
           float2* __restrict__ sv) {
  using L = TcLayout<K>;
  // MODE: kTcRow (8-byte copies/stores of each thread's own row), kTcPair
  // (index bit 0 free: 16-byte row pairs), kTcLow (targets = bits 0..k-1:
  // tiles are contiguous, staged row-major with a 16-byte-chunk swizzle)
  constexpr bool PAIR = MODE == kTcPair;
  constexpr bool LOWT = MODE == kTcLow;
  constexpr int D = L::D;
  constexpr int N = L::N;
  constexpr int S = L::NSTAGE;
  constexpr uint32_t IDESC = idesc_bf16<N>();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // 1 KB-aligned base, kept as an offset from smem_raw so the compiler still
  // sees shared-space accesses (LDS, not generic loads)
  const uint32_t raw_base = smem_u32(smem_raw);
  const uint32_t sbase = (raw_base + 1023u) & ~1023u;
  unsigned char* sm = smem_raw + (sbase - raw_base);
  const int tid = threadIdx.x;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);  // warp-uniform (TMEM addresses in uniform registers)
  const int grp = warp >> 2;  // consumer group
  const int row = tid & 127;  // TMEM lane = tile row = amplitude group within the tile
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + L::BAR + 16);
  const uint32_t bar = sbase + L::BAR + 8 * grp;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 32) {
    mbar_init(sbase + L::BAR, 1);
    mbar_init(sbase + L::BAR + 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // gate limbs, host layout [4][N rows][64 cols] bf16 -> 128-byte swizzled rows
  for (int i = tid; i < L::NBL * N * 8; i += 256) {
    const int limb = i / (N * 8);
    const int r = (i / 8) % N;
    const int c16 = i % 8;
    const int off = L::B0 + limb * L::B_LIMB + r * 128 + ((c16 ^ (r & 7)) << 4);
    *reinterpret_cast<uint4*>(sm + off) = bmat[i];
  }

  const uint64_t step = gridDim.x;
  // this group's i-th tile
  auto tile_of = [&](int i) { return uint64_t(blockIdx.x) + (2 * uint64_t(i) + grp) * step; };
  // rows are the lowest 7 free index bits: index(tile, r) = expand(tile * 128) | rowoff(r)
  const uint64_t e0 = expand(p.g, 0);
  const uint64_t rowoff = expand(p.g, row) ^ e0;
  // ring: the group's tile i into stage i % S, 16-byte copies: thread t moves
  // rows (2t', 2t'+1) (adjacent amplitudes, index bit 0) of members j = 2i + t / 64
  const int prow = 2 * (row & 63);
  const int jpar = row >> 6;
  const uint64_t prowoff = expand(p.g, prow) ^ e0;
  auto issue = [&](int i) -> uint64_t {  // returns the tile's base index
    const uint64_t tl = tile_of(i);
    uint64_t tb = 0;
    if (tl < p.ntiles) {
      tb = expand(p.g, tl * 128);
      if constexpr (LOWT) {  // contiguous 128 x D amplitudes: chunk q -> row q / (D/2), swizzled column
        const uint32_t st0 = sbase + L::RING + ((grp * S) + (i % S)) * L::STAGE;
#pragma unroll
        for (int m = 0; m < D / 2; ++m) {
          const int q = row + 128 * m;
          const int r = q / (D / 2), c = q % (D / 2);
          cp_async16(st0 + r * (D * 8) + ((c ^ (r & 7)) << 4), sv + tb + 2 * q);
        }
      } else if constexpr (PAIR) {
        const uint64_t b = tb | prowoff;
        const uint32_t dst = sbase + L::RING + ((grp * S) + (i % S)) * L::STAGE + prow * 8;
#pragma unroll
        for (int jj = 0; jj < D / 2; ++jj) {
          const uint64_t o = jpar ? p.offs[2 * jj + 1] : p.offs[2 * jj];  // static indices: no LDC
          cp_async16(dst + (2 * jj + jpar) * 1024, sv + b + o);
        }
      } else {  // index bit 0 is a target or control: each thread copies its own row, 8 B per member
        const uint64_t b = tb | rowoff;
        const uint32_t dst = sbase + L::RING + ((grp * S) + (i % S)) * L::STAGE + row * 8;
#pragma unroll
        for (int j = 0; j < D; ++j) cp_async8(dst + j * 1024, sv + b + p.offs[j]);
      }
    }
    cp_async_commit();
    return tb;
  };
  // phase slots of the row at amplitude index `b`: a[m] (target m), a[K] (outside)
  auto phase_angles = [&](uint64_t b, float (&a)[8]) {
#pragma unroll
    for (int s = 0; s < 8; ++s) a[s] = 0.f;
    // small table, L1-resident; unrolled to the maximum nibble count so all
    // loads issue before the first add
#pragma unroll
    for (int c = 0; c < kTcMaxNib; ++c) {
      if (c < p.nnib) {
        const int r = (c * 16 + int((b >> p.nib_shift[c]) & 15u)) * 2;
        const float4 x = __ldg(tab + r), y = __ldg(tab + r + 1);
        a[0] += x.x; a[1] += x.y; a[2] += x.z; a[3] += x.w;
        a[4] += y.x; a[5] += y.y; a[6] += y.z; a[7] += y.w;
      }
    }
  };
  // tile-uniform phases: thread 128 - D + j of the group computes factor j of
  // the group's tile i (base tb) into buffer i & 1 (published by a later group barrier)
  float2* Pb = reinterpret_cast<float2*>(sm + L::PBUF) + grp * 2 * D;
  auto phase_angles_c = [&](uint64_t b, float (&a)[8]) {
#pragma unroll
    for (int s = 0; s < 8; ++s) a[s] = 0.f;
#pragma unroll
    for (int c = 0; c < kTcMaxNib; ++c) {
      if (c < p.nnib) {
        const int r = (c * 16 + int((b >> p.nib_shift[c]) & 15u)) * 2;
        const float4 x = p.ctab[r], y = p.ctab[r + 1];
        a[0] += x.x; a[1] += x.y; a[2] += x.z; a[3] += x.w;
        a[4] += y.x; a[5] += y.y; a[6] += y.z; a[7] += y.w;
      }
    }
  };
  auto coop_phase = [&](int i, uint64_t tb) {
    const int j = row - (128 - D);
    if (PHASED && !p.coop && j == 0 && tile_of(i) < p.ntiles) {
      // per-row phases: the tile-uniform part of the angle sums (nibbles past
      // the row-varying ones) once per tile, from the constant bank
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
      float4* hb = reinterpret_cast<float4*>(Pb + (i & 1) * D);
      hb[0] = make_float4(a[0], a[1], a[2], a[3]);
      hb[1] = make_float4(a[4], a[5], a[6], a[7]);
    }
    if (PHASED && p.coop && j >= 0 && tile_of(i) < p.ntiles) {
      float a[8];
      phase_angles_c(tb, a);
      float ang = a[K];
#pragma unroll
      for (int m = 0; m < K; ++m) ang += ((j >> m) & 1) ? a[m] : 0.f;
      float sn, cs;
      sincos_unit(ang, &sn, &cs);
      Pb[(i & 1) * D + j] = make_float2(cs, sn);
    }
  };
  uint64_t tq[S - 1];  // bases of the tiles in flight (static indices only)
#pragma unroll
  for (int s = 0; s < S - 1; ++s) tq[s] = issue(s);
  coop_phase(0, tq[0]);
  coop_phase(1, tq[1]);
  cp_async_wait<S - 2>();  // tile 0 landed (this thread's part; the barrier below publishes it)

  const uint32_t tmem = uint32_t(grp * 256);
  const uint32_t tlane = tmem + (uint32_t((warp & 3) * 32) << 16);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // B operand: generic -> async proxy
  fence_before();
  __syncthreads();
  fence_after();
  // read only after the barrier: warp 0's tcgen05.alloc wrote the slot
  // (compute-sanitizer racecheck flagged the earlier pre-barrier read)
  if (*tmem_slot != 0u) __trap();  // whole-TMEM allocation starts at lane 0, column 0

  // out = 2^(e_row + e_b - 16) (acc0 + acc12 / 2^8); columns 2i (re), 2i+1 (im).
  // Lanes 2t', 2t'+1 hold adjacent amplitudes: they swap one member per pair
  // and store 16 bytes each (even lane: member 2q of both rows, odd: 2q+1).
  const bool odd = row & 1;
  auto epilogue = [&](uint64_t b, float scale) {
#ifdef DSV_AB_NOEPI
    return;
#endif
    if constexpr (LOWT) {  // this row's members are contiguous: 16-byte stores
#pragma unroll
      for (int h = 0; h < N / 32; ++h) {
        float c0[32], c1[32];
        tmem_ld32(tlane + uint32_t(L::T_ACC0 + h * 32), c0);
        tmem_ld32(tlane + uint32_t(L::T_ACC12 + h * 32), c1);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float o[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) o[c] = __fmaf_rn(c1[4 * i + c], 1.f / 256.f, c0[4 * i + c]) * scale;
          __stcs(reinterpret_cast<float4*>(sv + b) + h * 8 + i, make_float4(o[0], o[1], o[2], o[3]));
        }
      }
      return;
    }
    if constexpr (!PAIR) {  // 8-byte stores of this row's members
#pragma unroll
      for (int h = 0; h < N / 32; ++h) {
        float c0[32], c1[32];
        tmem_ld32(tlane + uint32_t(L::T_ACC0 + h * 32), c0);
        tmem_ld32(tlane + uint32_t(L::T_ACC12 + h * 32), c1);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float re = __fmaf_rn(c1[2 * i], 1.f / 256.f, c0[2 * i]) * scale;
          const float im = __fmaf_rn(c1[2 * i + 1], 1.f / 256.f, c0[2 * i + 1]) * scale;
          __stcs(sv + b + p.offs[h * 16 + i], make_float2(re, im));
        }
      }
      return;
    }
    const uint64_t be = b - (odd ? 1 : 0);
#pragma unroll
    for (int h = 0; h < N / 32; ++h) {
      float c0[32], c1[32];
      tmem_ld32(tlane + uint32_t(L::T_ACC0 + h * 32), c0);
      tmem_ld32(tlane + uint32_t(L::T_ACC12 + h * 32), c1);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float o[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) o[c] = __fmaf_rn(c1[4 * q + c], 1.f / 256.f, c0[4 * q + c]) * scale;
        // o = (re, im) of members 2q, 2q+1 (of this half)
        const float sx = odd ? o[0] : o[2], sy = odd ? o[1] : o[3];
        const float rx = __shfl_xor_sync(0xffffffffu, sx, 1), ry = __shfl_xor_sync(0xffffffffu, sy, 1);
        const uint64_t oj = odd ? p.offs[h * 16 + 2 * q + 1] : p.offs[h * 16 + 2 * q];
        const float4 w = odd ? make_float4(rx, ry, o[2], o[3]) : make_float4(o[0], o[1], rx, ry);
        __stcs(reinterpret_cast<float4*>(sv + be + oj), w);
      }
    }
  };

  uint64_t prev_base = 0;
  float prev_scale = 0.f;
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
    const unsigned char* stg = sm + L::RING + (grp * S + stage) * L::STAGE;
    stage = stage + 1 == S ? 0 : stage + 1;
    float2 v[D];
    if constexpr (LOWT) {
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
      if (p.coop) {  // the tile's D phase factors, computed last iteration by the last warp
        const float2* P = Pb + (it & 1) * D;
#pragma unroll
        for (int j = 0; j < D; ++j) {
          const float2 x = v[j], f = P[j];
          v[j] = make_float2(x.x * f.x - x.y * f.y, x.x * f.y + x.y * f.x);
        }
      } else {
        // tile-uniform part (computed two tiles ahead) + this row's nibbles
        float a[8];
        const float4* hb = reinterpret_cast<const float4*>(Pb + (it & 1) * D);
        const float4 h0 = hb[0], h1 = hb[1];
        a[0] = h0.x; a[1] = h0.y; a[2] = h0.z; a[3] = h0.w;
        a[4] = h1.x; a[5] = h1.y; a[6] = h1.z; a[7] = h1.w;
#pragma unroll
        for (int c = 0; c < kTcMaxNib; ++c) {
          if (c < p.nnib_row) {
            const int r = (c * 16 + int((base >> p.nib_shift[c]) & 15u)) * 2;
            const float4 x = __ldg(tab + r), y = __ldg(tab + r + 1);
            a[0] += x.x; a[1] += x.y; a[2] += x.z; a[3] += x.w;
            a[4] += y.x; a[5] += y.y; a[6] += y.z; a[7] += y.w;
          }
        }
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
    // row exponent: max |x| < 2^e_row (rows below 2^-100 flush to zero)
    float mx = 0.f;
#pragma unroll
    for (int j = 0; j < D; ++j) mx = fmaxf(mx, fmaxf(fabsf(v[j].x), fabsf(v[j].y)));
    const int e_row = min(max(int((__float_as_uint(mx) >> 23) & 0xFF) - 126, -100), 120);
    const float s8 = pow2f(8 - e_row), s16 = pow2f(16 - e_row);
    const float scale = pow2f(e_row + p.e_b - 16);
    if (it > 0) {  // MMA(i-1) done: A is free and its accumulators are ready
      mbar_wait(bar, (it - 1) & 1);
      fence_after();
      epilogue(prev_base, prev_scale);
    }
    // limbs -> TMEM: column j of limb l = member j (re | im << 16).
    // y = x 2^(8 - e_row), |y| < 256:  a0 = rint(y), r1 = (y - a0) 2^8 (exact),
    // a1 = rint(r1), a2' = (r1 - a1) rounded to 2^-8 (= a2 / 2^8, |a2| <= 128):
    // y = a0 + a1 / 2^8 + a2 / 2^16 to 2^-17 (24 significant bits of the row
    // maximum), 9 full-rate FP32 ops per value (magic-number rounding).
#pragma unroll
    for (int h = 0; h < D / 16; ++h) {
      uint32_t l0[16], l1[16], l2[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        float a0[2], a1[2], a2[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const float x = c ? v[h * 16 + q].y : v[h * 16 + q].x;
#ifndef DSV_AB_NOSPLIT
          a0[c] = __fadd_rn(__fmaf_rn(x, s8, kMagic), -kMagic);
          const float r1 = __fmaf_rn(a0[c], -256.f, x * s16);
          a1[c] = __fadd_rn(__fadd_rn(r1, kMagic), -kMagic);
          a2[c] = __fadd_rn(__fadd_rn(__fadd_rn(r1, -a1[c]), kMagic16), -kMagic16);
#else
          a0[c] = x;
          a1[c] = x;
          a2[c] = x;
#endif
        }
        l0[q] = pack2(a0[0], a0[1]);
        l1[q] = pack2(a1[0], a1[1]);
        l2[q] = pack2(a2[0], a2[1]);
      }
      tmem_st16(tlane + uint32_t(L::T_A + 0 * D + h * 16), l0);
      tmem_st16(tlane + uint32_t(L::T_A + 1 * D + h * 16), l1);
      tmem_st16(tlane + uint32_t(L::T_A + 2 * D + h * 16), l2);
    }
    cp_async_wait<S - 2>();  // tile i+1 landed (this thread's part)
    tmem_wait_st();
    fence_before();
    group_sync(grp);
    if (row == 0) {
      fence_after();
#ifndef DSV_AB_NOMMA
      if (grp == 0) issue_mma<K, 0>(sbase);
      else issue_mma<K, 1>(sbase);
#endif
      mma_commit(bar);
    }
    // two tiles ahead, after the barrier: off the barrier's critical path,
    // published by the next iteration's barrier (buffer (i + 2) & 1 = i & 1
    // was read before this iteration's barrier)
    coop_phase(it + 2, tq[S - 2 >= 1 ? 1 : 0]);
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

template <int K, bool PHASED, int MODE>
static cudaError_t tc_go(const TcDesc& d, const void* d_bmat, const void* d_tab, void* sv, cudaStream_t st) {
  using L = TcLayout<K>;
  TcP<K> p;
  std::memset(&p, 0, sizeof p);
  p.g = d.g;
  p.ntiles = d.g.nwork / 128;
  p.nnib = d.nnib;
  p.e_b = d.e_b;
  p.coop = d.coop;
  p.nnib_row = d.nnib_row;
  for (int c = 0; c < 16; ++c) p.nib_shift[c] = d.nib_shift[c];
  for (int j = 0; j < (1 << K); ++j) p.offs[j] = d.offs[j];
  if (d.htab && d.nnib > 0) std::memcpy(p.ctab, d.htab, size_t(d.nnib) * 16 * 2 * sizeof(float4));
  const int smem = L::BYTES + 1024;
  static bool attr_set[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_dense_tc<K, PHASED, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr_set[dev] = true;
  }
  uint64_t blocks = uint64_t(device_sm_count());  // persistent: one CTA per SM
  const uint64_t need = (p.ntiles + 1) / 2;        // two tiles in flight per CTA
  if (blocks > need) blocks = need;
  if (blocks == 0) return cudaSuccess;
  k_dense_tc<K, PHASED, MODE><<<unsigned(blocks), 256, smem, st>>>(p, static_cast<const uint4*>(d_bmat),
                                                              static_cast<const float4*>(d_tab),
                                                              static_cast<float2*>(sv));
  return cudaGetLastError();
}

int tc_smem_bytes(int k) {
  switch (k) {
    case 4: return TcLayout<4>::BYTES + 1024;
    case 5: return TcLayout<5>::BYTES + 1024;
  }
  return 0;
}

template <int K>
static cudaError_t tc_k(const TcDesc& d, const void* d_bmat, const void* d_tab, void* sv, cudaStream_t st) {
  const bool ph = d.nnib > 0;
  switch (d.mode) {
    case kTcPair: return ph ? tc_go<K, true, kTcPair>(d, d_bmat, d_tab, sv, st) : tc_go<K, false, kTcPair>(d, d_bmat, d_tab, sv, st);
    case kTcLow: return ph ? tc_go<K, true, kTcLow>(d, d_bmat, d_tab, sv, st) : tc_go<K, false, kTcLow>(d, d_bmat, d_tab, sv, st);
  }
  return ph ? tc_go<K, true, kTcRow>(d, d_bmat, d_tab, sv, st) : tc_go<K, false, kTcRow>(d, d_bmat, d_tab, sv, st);
}

cudaError_t launch_dense_tc(int k, const TcDesc& d, const void* d_bmat, const void* d_tab, void* sv,
                            cudaStream_t st) {
  switch (k) {
    case 4: return tc_k<4>(d, d_bmat, d_tab, sv, st);
    case 5: return tc_k<5>(d, d_bmat, d_tab, sv, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace dsv
