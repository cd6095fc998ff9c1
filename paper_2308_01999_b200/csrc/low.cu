// low.cu — complex64 dense k-qubit gates (k = 1..3) whose targets are exactly
// the LOWEST k index bits, optionally preceded by the fold fuser's
// outside-coupled phase polynomial (the last window of a folded QFT, e.g.
// QFT-33 at k = 5 ends on qubits (0, 1, 2)).  Replaces apply_dense_bits
// (reference statevec.py:44-60) for that layout.
//
// A group (2^k consecutive amplitudes, 2^(k+3) bytes) is spread over
// L = 2^(k-1) lanes, one 16-byte float4 (two members) each, so every warp
// load/store is a fully coalesced 512-byte run — the register path's
// one-thread-per-group layout strides 64 bytes between lanes here.  Each lane
// applies the phase to its own two members (one sincos each: the member's
// angle is the outside angle plus the cross angles of its set target bits),
// gathers the group with L-1 float4 shuffles and computes its two output rows
// from matrix rows held in registers for the whole persistent loop.
#include <cmath>
#include <cstring>

#include "common.cuh"
#include "launch.h"

namespace dsv {

constexpr int kLowItems = 4;

template <int K>
struct Low128P {
  int nchunk;              // phase-table index bytes (0: plain dense)
  int chunk_shift[8];
  cplx<double> m[(1 << K) * (1 << K)];
};

template <int K>
struct LowP {
  Geom g;                 // groups: holes = targets (bits 0..k-1) + controls
  int nchunk;             // phase-table index bytes in use (0: plain dense)
  int plain;              // no controls: group w starts at amplitude w << k
  uint32_t used;          // bit c: index byte c carries phase terms (table row block c)
  cplx<float> m[(1 << K) * (1 << K)];
};

__device__ __forceinline__ void sincos_low(float a, float* sn, float* cs) {
  const float t = a - 6.28318530717958647692f * rintf(a * 0.15915494309189533577f);
  __sincosf(t, sn, cs);
}

template <int K, bool PHASED>
__global__ void __launch_bounds__(256)
k_dense_low(const __grid_constant__ LowP<K> p, const float4* __restrict__ tab, float4* __restrict__ sv4) {
  constexpr int D = 1 << K;
  constexpr int L = D / 2;  // lanes per group
  extern __shared__ float4 stab[];  // [index byte 0..7][256] phase slots (target m: slot m, outside: slot K)
  if constexpr (PHASED) {
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) stab[i] = tab[i];
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int sub = lane & (L - 1);
  const int gl0 = lane & ~(L - 1);
  // this lane's two output rows, 2 sub and 2 sub + 1, kept in registers
  float mr[2][D][2];
#pragma unroll
  for (int rr = 0; rr < 2; ++rr)
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const cplx<float> z = p.m[(2 * sub + rr) * D + c];
      mr[rr][c][0] = z.x;
      mr[rr][c][1] = z.y;
    }
  // U lane-items per thread per pass, all loads first (memory-level parallelism);
  // the host guarantees nwork * L is a multiple of 256 U: no per-item guards,
  // so the shuffles stay convergent
  constexpr int U = kLowItems;
  const uint64_t npass = p.g.nwork * L / (256 * U);
  // block-uniform trip count: the compiler sees convergent shuffles
  const int warp = threadIdx.x >> 5;
  for (uint64_t pass = blockIdx.x; pass < npass; pass += gridDim.x) {
    // a warp's U x 32 lane-items = 256 consecutive amplitudes (256-aligned):
    // without controls, index bytes 1..7 are uniform over the warp's items
    const uint64_t t0 = pass * (256 * U) + warp * (32 * U) + lane;
    uint64_t base[U];
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t t = t0 + uint64_t(u) * 32;
      base[u] = p.plain ? (t / L) << K : expand(p.g, t / L);  // multiple of 2^k
      v[u] = __ldcs(sv4 + (base[u] >> 1) + sub);
    }
    float4 hi = make_float4(0.f, 0.f, 0.f, 0.f);  // phase slots from index bytes 1..7
    if constexpr (PHASED) {
      if (p.plain) {
#pragma unroll
        for (int c = 1; c < 8; ++c) {
          if ((p.used >> c) & 1u) {  // warp-uniform row: broadcast
            const float4 x = stab[c * 256 + int((base[0] >> (8 * c)) & 255u)];
            hi.x += x.x; hi.y += x.y; hi.z += x.z; hi.w += x.w;
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if constexpr (PHASED) {
        float a[4] = {hi.x, hi.y, hi.z, hi.w};
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          if ((p.used >> c) & 1u && (c == 0 || !p.plain)) {  // compile-time byte position
            const float4 x = stab[c * 256 + int((base[u] >> (8 * c)) & 255u)];
            a[0] += x.x; a[1] += x.y; a[2] += x.z; a[3] += x.w;
          }
        }
        float ang[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int j = 2 * sub + h;
          ang[h] = a[K];
#pragma unroll
          for (int m = 0; m < K; ++m) ang[h] += ((j >> m) & 1) ? a[m] : 0.f;
        }
        float s0, c0, s1, c1;
        sincos_low(ang[0], &s0, &c0);
        sincos_low(ang[1], &s1, &c1);
        const float4 x = v[u];
        v[u] = make_float4(x.x * c0 - x.y * s0, x.x * s0 + x.y * c0, x.z * c1 - x.w * s1, x.z * s1 + x.w * c1);
      }
      float in[D][2];
#pragma unroll
      for (int i = 0; i < L; ++i) {
        float4 w;
        if constexpr (L == 1) {
          w = v[u];
        } else {
          w.x = __shfl_sync(0xffffffffu, v[u].x, gl0 + i);
          w.y = __shfl_sync(0xffffffffu, v[u].y, gl0 + i);
          w.z = __shfl_sync(0xffffffffu, v[u].z, gl0 + i);
          w.w = __shfl_sync(0xffffffffu, v[u].w, gl0 + i);
        }
        in[2 * i][0] = w.x;
        in[2 * i][1] = w.y;
        in[2 * i + 1][0] = w.z;
        in[2 * i + 1][1] = w.w;
      }
      float o[2][2];
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        float re = 0.f, im = 0.f;
#pragma unroll
        for (int c = 0; c < D; ++c) {
          re = fmaf(mr[rr][c][0], in[c][0], re);
          re = fmaf(-mr[rr][c][1], in[c][1], re);
          im = fmaf(mr[rr][c][0], in[c][1], im);
          im = fmaf(mr[rr][c][1], in[c][0], im);
        }
        o[rr][0] = re;
        o[rr][1] = im;
      }
      __stcs(sv4 + (base[u] >> 1) + sub, make_float4(o[0][0], o[0][1], o[1][0], o[1][1]));
    }
  }
}

// k = 3 without controls: each warp moves a contiguous 512-amplitude run
// (4 KB, 16-byte coalesced loads) into its own shared-memory slice (16-byte
// units XOR-swizzled by their 128-byte line: the group reads below are
// conflict-free), every lane then applies the phase and the full 8 x 8 matrix
// (kernel-parameter constant bank, warp-uniform FFMA operands) to two whole
// groups, and the run streams back out.  No shuffles: ~45 instructions per
// amplitude instead of ~80 for the lane-split kernel above.
constexpr int kLowtRun = 512;  // amplitudes per warp run

__device__ __forceinline__ uint32_t lowt_slot(uint32_t u) { return u ^ ((u >> 3) & 7u); }

template <int K, bool PHASED>
__global__ void __launch_bounds__(256)
k_dense_lowt(const __grid_constant__ LowP<K> p, uint64_t nruns, const float4* __restrict__ tab,
             float4* __restrict__ sv4) {
  constexpr int D = 1 << K;
  constexpr int G = kLowtRun / D / 32;  // groups per lane per run
  extern __shared__ float4 lsm[];  // [8 warps][256 units] run slices, then [8][256] phase slots
  float4* stab = lsm + 8 * 256;
  if constexpr (PHASED) {
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) stab[i] = tab[i];
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  float4* slice = lsm + warp * 256;
  const uint64_t nwarps = uint64_t(gridDim.x) * 8;
  for (uint64_t run = uint64_t(blockIdx.x) * 8 + warp; run < nruns; run += nwarps) {
    float4* g4 = sv4 + run * (kLowtRun / 2);
    float4 t[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) t[i] = __ldcs(g4 + i * 32 + lane);
#pragma unroll
    for (int i = 0; i < 8; ++i) slice[lowt_slot(i * 32 + lane)] = t[i];
    __syncwarp();
    // index bytes 2..7 of the run: uniform
    float4 hi = make_float4(0.f, 0.f, 0.f, 0.f);
    const uint64_t rb = run * kLowtRun;
    if constexpr (PHASED) {
#pragma unroll
      for (int c = 2; c < 8; ++c)
        if ((p.used >> c) & 1u) {
          const float4 x = stab[c * 256 + int((rb >> (8 * c)) & 255u)];
          hi.x += x.x; hi.y += x.y; hi.z += x.z; hi.w += x.w;
        }
    }
#pragma unroll
    for (int q = 0; q < G; ++q) {
      const int g = lane + 32 * q;  // group: amplitudes D g .. D g + D - 1 of the run
      float in[D][2];
#pragma unroll
      for (int c = 0; c < D / 2; ++c) {
        const float4 x = slice[lowt_slot((D / 2) * g + c)];
        in[2 * c][0] = x.x; in[2 * c][1] = x.y; in[2 * c + 1][0] = x.z; in[2 * c + 1][1] = x.w;
      }
      if constexpr (PHASED) {
        float a[4] = {hi.x, hi.y, hi.z, hi.w};
        const uint64_t b = rb + uint64_t(D) * g;
#pragma unroll
        for (int c = 0; c < 2; ++c)
          if ((p.used >> c) & 1u) {
            const float4 x = stab[c * 256 + int((b >> (8 * c)) & 255u)];
            a[0] += x.x; a[1] += x.y; a[2] += x.z; a[3] += x.w;
          }
        float ang[D];
        ang[0] = a[K];
#pragma unroll
        for (int m = 0; m < K; ++m)
#pragma unroll
          for (int j = 0; j < (1 << m); ++j) ang[j + (1 << m)] = ang[j] + a[m];
#pragma unroll
        for (int j = 0; j < D; ++j) {
          float sn, cs;
          sincos_low(ang[j], &sn, &cs);
          const float xr = in[j][0], xi = in[j][1];
          in[j][0] = xr * cs - xi * sn;
          in[j][1] = xr * sn + xi * cs;
        }
      }
      float o[D][2];
#pragma unroll
      for (int r = 0; r < D; ++r) {
        float re = 0.f, im = 0.f;
#pragma unroll
        for (int c = 0; c < D; ++c) {
          const float mr = p.m[r * D + c].x, mi = p.m[r * D + c].y;
          re = fmaf(mr, in[c][0], re);
          re = fmaf(-mi, in[c][1], re);
          im = fmaf(mr, in[c][1], im);
          im = fmaf(mi, in[c][0], im);
        }
        o[r][0] = re;
        o[r][1] = im;
      }
#pragma unroll
      for (int c = 0; c < D / 2; ++c)
        slice[lowt_slot((D / 2) * g + c)] = make_float4(o[2 * c][0], o[2 * c][1], o[2 * c + 1][0], o[2 * c + 1][1]);
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 8; ++i) __stcs(g4 + i * 32 + lane, slice[lowt_slot(i * 32 + lane)]);
    __syncwarp();
  }
}

template <int K, bool PHASED>
static cudaError_t lowt_go(const LowDesc& d, uint64_t namps, const void* matrix, const void* d_tab, void* sv,
                           cudaStream_t st) {
  LowP<K> p;
  std::memset(&p, 0, sizeof p);
  p.g = d.g;
  p.nchunk = d.nchunk;
  p.plain = d.plain;
  for (int c = 0; c < d.nchunk; ++c) p.used |= 1u << (d.chunk_shift[c] / 8);
  std::memcpy(p.m, matrix, sizeof(p.m));
  const uint64_t nruns = namps / kLowtRun;
  const int smem = (8 * 256 + (PHASED ? 8 * 256 : 0)) * 16;
  static bool attr_set[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_dense_lowt<K, PHASED>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr_set[dev] = true;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dense_lowt<K, PHASED>, 256, smem);
  if (per_sm < 1) per_sm = 1;
  uint64_t blocks = (nruns + 7) / 8;
  const uint64_t cap = uint64_t(device_sm_count()) * per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) return cudaSuccess;
  k_dense_lowt<K, PHASED><<<unsigned(blocks), 256, smem, st>>>(p, nruns, static_cast<const float4*>(d_tab),
                                                             static_cast<float4*>(sv));
  return cudaGetLastError();
}

cudaError_t launch_dense_lowt(int k, const LowDesc& d, uint64_t namps, const void* matrix, const void* d_tab,
                              void* sv, cudaStream_t st) {
  if (!d.plain || namps % kLowtRun) return cudaErrorInvalidValue;
  const bool ph = d.nchunk > 0;
  switch (k) {
    case 1: return ph ? lowt_go<1, true>(d, namps, matrix, d_tab, sv, st) : lowt_go<1, false>(d, namps, matrix, d_tab, sv, st);
    case 2: return ph ? lowt_go<2, true>(d, namps, matrix, d_tab, sv, st) : lowt_go<2, false>(d, namps, matrix, d_tab, sv, st);
    case 3: return ph ? lowt_go<3, true>(d, namps, matrix, d_tab, sv, st) : lowt_go<3, false>(d, namps, matrix, d_tab, sv, st);
  }
  return cudaErrorInvalidValue;
}

template <int K, bool PHASED>
static cudaError_t low_go(const LowDesc& d, const void* matrix, const void* d_tab, void* sv, cudaStream_t st) {
  LowP<K> p;
  std::memset(&p, 0, sizeof p);
  p.g = d.g;
  p.nchunk = d.nchunk;
  p.plain = d.plain;
  for (int c = 0; c < d.nchunk; ++c) p.used |= 1u << (d.chunk_shift[c] / 8);
  std::memcpy(p.m, matrix, sizeof(p.m));
  const int smem = PHASED ? 8 * 256 * 16 : 0;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dense_low<K, PHASED>, 256, smem);
  if (per_sm < 1) per_sm = 1;
  constexpr int L = (1 << K) / 2;
  uint64_t blocks = (d.g.nwork * L + 256 * kLowItems - 1) / (256 * kLowItems);
  const uint64_t cap = uint64_t(device_sm_count()) * per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) return cudaSuccess;
  k_dense_low<K, PHASED><<<unsigned(blocks), 256, smem, st>>>(p, static_cast<const float4*>(d_tab),
                                                             static_cast<float4*>(sv));
  return cudaGetLastError();
}

cudaError_t launch_dense_low(int k, const LowDesc& d, const void* matrix, const void* d_tab, void* sv,
                             cudaStream_t st) {
  const bool ph = d.nchunk > 0;
  switch (k) {
    case 1: return ph ? low_go<1, true>(d, matrix, d_tab, sv, st) : low_go<1, false>(d, matrix, d_tab, sv, st);
    case 2: return ph ? low_go<2, true>(d, matrix, d_tab, sv, st) : low_go<2, false>(d, matrix, d_tab, sv, st);
    case 3: return ph ? low_go<3, true>(d, matrix, d_tab, sv, st) : low_go<3, false>(d, matrix, d_tab, sv, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace dsv

namespace dsv {

// complex128 k = 1..4 windows (plain or phased) on the lowest k bits, no
// controls: the warp-transposed scheme of k_dense_lowt with 16-byte units of
// one amplitude and 512-amplitude (8 KB) runs, and the phased.cu tables of
// unit factors exp(i angle) per (index byte, value, slot) — no sin/cos per
// group: index bytes 2.. are uniform over a run (one product per run), bytes
// 0 and 1 vary per group.  Replaces apply_dense_bits (statevec.py:44-60) for
// the last window of a complex128 fold-fused QFT.
constexpr int kLowt128Run = 512;

template <int K, bool PHASED>
__global__ void __launch_bounds__(256)
k_dense_lowt128(const __grid_constant__ Low128P<K> p, uint64_t nruns, const cplx<double>* __restrict__ tab,
                double2* __restrict__ sv2) {
  constexpr int D = 1 << K;
  constexpr int S = K + 1;
  constexpr int G = kLowt128Run / D / 32;  // groups per lane per run
  extern __shared__ double2 lsm2[];  // [8 warps][512] run slices, then [nchunk][256][S] factors
  cplx<double>* stab = reinterpret_cast<cplx<double>*>(lsm2 + 8 * kLowt128Run);
  if constexpr (PHASED) {
    for (int i = threadIdx.x; i < p.nchunk * 256 * S; i += blockDim.x) stab[i] = tab[i];
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  double2* slice = lsm2 + warp * kLowt128Run;
  const uint64_t nwarps = uint64_t(gridDim.x) * 8;
  for (uint64_t run = uint64_t(blockIdx.x) * 8 + warp; run < nruns; run += nwarps) {
    double2* g2 = sv2 + run * kLowt128Run;
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // two batches of 8 loads in flight (register budget)
      double2 t[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) t[i] = __ldcs(g2 + (8 * h + i) * 32 + lane);
#pragma unroll
      for (int i = 0; i < 8; ++i) slice[lowt_slot((8 * h + i) * 32 + lane)] = t[i];
    }
    __syncwarp();
    const uint64_t rb = run * kLowt128Run;
    double hr[S], hi[S];  // run-uniform factors (index bytes >= 2)
#pragma unroll
    for (int s = 0; s < S; ++s) {
      hr[s] = 1.0;
      hi[s] = 0.0;
    }
    if constexpr (PHASED) {
      for (int c = 0; c < p.nchunk; ++c) {
        if (p.chunk_shift[c] < 16) continue;
        const cplx<double>* row = stab + (size_t(c) * 256 + ((rb >> p.chunk_shift[c]) & 255u)) * S;
#pragma unroll
        for (int s = 0; s < S; ++s) {
          const double xr = hr[s] * row[s].x - hi[s] * row[s].y;
          hi[s] = hr[s] * row[s].y + hi[s] * row[s].x;
          hr[s] = xr;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < G; ++q) {
      const int g = lane + 32 * q;  // group: amplitudes D g .. D g + D - 1 of the run
      double in[D][2];
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const double2 x = slice[lowt_slot(D * g + j)];
        in[j][0] = x.x;
        in[j][1] = x.y;
      }
      if constexpr (PHASED) {
        double fr[S], fi[S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
          fr[s] = hr[s];
          fi[s] = hi[s];
        }
        const uint64_t b = rb + uint64_t(D) * g;
        for (int c = 0; c < p.nchunk; ++c) {
          if (p.chunk_shift[c] >= 16) continue;
          const cplx<double>* row = stab + (size_t(c) * 256 + ((b >> p.chunk_shift[c]) & 255u)) * S;
#pragma unroll
          for (int s = 0; s < S; ++s) {
            const double xr = fr[s] * row[s].x - fi[s] * row[s].y;
            fi[s] = fr[s] * row[s].y + fi[s] * row[s].x;
            fr[s] = xr;
          }
        }
        // member j: exp(i gamma) prod_{m in j} exp(i alpha_m)
#pragma unroll
        for (int j = 0; j < D; ++j) {
          double er = fr[K], ei = fi[K];
#pragma unroll
          for (int m = 0; m < K; ++m)
            if ((j >> m) & 1) {
              const double xr = er * fr[m] - ei * fi[m];
              ei = er * fi[m] + ei * fr[m];
              er = xr;
            }
          const double xr = in[j][0], xi = in[j][1];
          in[j][0] = xr * er - xi * ei;
          in[j][1] = xr * ei + xi * er;
        }
      }
      // each output row goes straight back to its slot (the inputs are in registers)
#pragma unroll
      for (int r = 0; r < D; ++r) {
        double re = 0.0, im = 0.0;
#pragma unroll
        for (int c = 0; c < D; ++c) {
          const double mr = p.m[r * D + c].x, mi = p.m[r * D + c].y;
          re = fma(mr, in[c][0], re);
          re = fma(-mi, in[c][1], re);
          im = fma(mr, in[c][1], im);
          im = fma(mi, in[c][0], im);
        }
        slice[lowt_slot(D * g + r)] = make_double2(re, im);
      }
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 16; ++i) __stcs(g2 + i * 32 + lane, slice[lowt_slot(i * 32 + lane)]);
    __syncwarp();
  }
}

template <int K, bool PHASED>
static cudaError_t lowt128_go(const PhasedDesc& d, uint64_t namps, const void* matrix, const void* d_tab,
                              void* sv, cudaStream_t st) {
  Low128P<K> p;
  std::memset(&p, 0, sizeof p);
  p.nchunk = PHASED ? d.nchunk : 0;
  for (int c = 0; c < 8; ++c) p.chunk_shift[c] = d.chunk_shift[c];
  std::memcpy(p.m, matrix, sizeof(p.m));
  const uint64_t nruns = namps / kLowt128Run;
  const int smem = 8 * kLowt128Run * 16 + (PHASED ? d.nchunk * 256 * (K + 1) * 16 : 0);
  cudaError_t e = cudaFuncSetAttribute(k_dense_lowt128<K, PHASED>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dense_lowt128<K, PHASED>, 256, smem);
  if (per_sm < 1) per_sm = 1;
  uint64_t blocks = (nruns + 7) / 8;
  const uint64_t cap = uint64_t(device_sm_count()) * per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) return cudaSuccess;
  k_dense_lowt128<K, PHASED><<<unsigned(blocks), 256, smem, st>>>(p, nruns, static_cast<const cplx<double>*>(d_tab),
                                                                 static_cast<double2*>(sv));
  return cudaGetLastError();
}

cudaError_t launch_dense_lowt128(int k, bool phased, const PhasedDesc& d, uint64_t namps, const void* matrix,
                                 const void* d_tab, void* sv, cudaStream_t st) {
  if (namps % kLowt128Run) return cudaErrorInvalidValue;
  switch (k) {
    case 1: return phased ? lowt128_go<1, true>(d, namps, matrix, d_tab, sv, st) : lowt128_go<1, false>(d, namps, matrix, d_tab, sv, st);
    case 2: return phased ? lowt128_go<2, true>(d, namps, matrix, d_tab, sv, st) : lowt128_go<2, false>(d, namps, matrix, d_tab, sv, st);
    case 3: return phased ? lowt128_go<3, true>(d, namps, matrix, d_tab, sv, st) : lowt128_go<3, false>(d, namps, matrix, d_tab, sv, st);
    case 4: return phased ? lowt128_go<4, true>(d, namps, matrix, d_tab, sv, st) : lowt128_go<4, false>(d, namps, matrix, d_tab, sv, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace dsv
