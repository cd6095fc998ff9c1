// wt.cu — dense k-qubit gates whose targets all sit in the lowest six index
// bits, through a per-warp shared-memory transpose.  Replaces
// apply_dense_bits (reference statevec.py:44-60) for those layouts.
//
// When a group's 2^k members lie inside one 64-amplitude block, the register
// path's one-thread-per-group loads give every lane its own 128-byte line per
// instruction (e.g. complex64 targets (1,2,3), complex128 (0,1,2): ~0.6 of
// HBM bandwidth).  Here each warp instead moves a contiguous 4-8 KB run with
// 16-byte coalesced loads into its own shared-memory slice (16-byte units
// XOR-swizzled by their 128-byte line so the group reads are conflict-free),
// every lane applies the matrix to its 512/(32 D) groups in place, and the
// warp streams the run back out.  HBM traffic stays one read + one write.
#include <cstring>

#include "common.cuh"
#include "launch.h"

namespace dsv {

template <typename R, int K>
struct WtP {
  uint64_t npass;             // runs of RUN amplitudes
  uint64_t run_amps;
  int ngpl;                   // groups per lane per run
  uint16_t gbase[256];        // group g's first member within the run (amplitudes)
  uint16_t offs[1 << K];      // member offsets
  cplx<R> m[(1 << K) * (1 << K)];
};

// 16-byte unit u of a warp slice -> swizzled slot (XOR the line's 3 low unit bits)
__device__ __forceinline__ uint32_t wt_slot(uint32_t u) { return u ^ ((u >> 3) & 7u); }

template <typename R, int K, int UNITS>
__global__ void __launch_bounds__(256)
k_dense_wt(const __grid_constant__ WtP<R, K> p, R* __restrict__ sv_r) {
  constexpr int D = 1 << K;
  constexpr int APU = 16 / (2 * int(sizeof(R)));  // amplitudes per 16-byte unit
  using U = float4;                                // 16-byte unit
  extern __shared__ __align__(16) float4 wsm[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  U* slice = wsm + warp * UNITS;
  U* svu = reinterpret_cast<U*>(sv_r);
  const uint64_t nwarps = uint64_t(gridDim.x) * (blockDim.x >> 5);
  for (uint64_t run = uint64_t(blockIdx.x) * (blockDim.x >> 5) + warp; run < p.npass; run += nwarps) {
    U* g = svu + run * UNITS;
    U t[UNITS / 32];
#pragma unroll
    for (int i = 0; i < UNITS / 32; ++i) t[i] = __ldcs(g + i * 32 + lane);
#pragma unroll
    for (int i = 0; i < UNITS / 32; ++i) slice[wt_slot(i * 32 + lane)] = t[i];
    __syncwarp();
    for (int q = 0; q < p.ngpl; ++q) {
      const uint32_t b = p.gbase[q * 32 + lane];
      R ar[D], ai[D];
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const uint32_t a = b + p.offs[j];
        const R* e = reinterpret_cast<const R*>(slice + wt_slot(a / APU)) + 2 * (a % APU);
        ar[j] = e[0];
        ai[j] = e[1];
      }
#pragma unroll
      for (int r = 0; r < D; ++r) {
        R xr = R(0), xi = R(0);
#pragma unroll
        for (int c = 0; c < D; ++c) {
          const R mr = p.m[r * D + c].x, mi = p.m[r * D + c].y;
          xr = fma(mr, ar[c], xr);
          xr = fma(-mi, ai[c], xr);
          xi = fma(mr, ai[c], xi);
          xi = fma(mi, ar[c], xi);
        }
        const uint32_t a = b + p.offs[r];
        R* e = reinterpret_cast<R*>(slice + wt_slot(a / APU)) + 2 * (a % APU);
        e[0] = xr;
        e[1] = xi;
      }
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < UNITS / 32; ++i) __stcs(g + i * 32 + lane, slice[wt_slot(i * 32 + lane)]);
    __syncwarp();
  }
}

template <typename R, int K>
static cudaError_t wt_t(int nbits, const int* tb, const void* matrix, void* sv, cudaStream_t st) {
  constexpr int D = 1 << K;
  // 8 units (128 B) per lane: 512 complex64 / 256 complex128 amplitudes per run;
  // complex128 k = 4 takes 16 units per lane (512 amplitudes: one group per lane)
  constexpr int UNITS = (sizeof(R) == 8 && K == 4) ? 512 : 256;
  constexpr int APU = 16 / (2 * int(sizeof(R)));
  const uint64_t run_amps = uint64_t(UNITS) * APU;
  if ((uint64_t(1) << nbits) < run_amps) return cudaErrorInvalidValue;
  WtP<R, K> p;
  std::memset(&p, 0, sizeof p);
  p.run_amps = run_amps;
  p.npass = (uint64_t(1) << nbits) / run_amps;
  uint32_t tmask = 0;
  for (int m = 0; m < K; ++m) tmask |= 1u << tb[m];
  for (int j = 0; j < D; ++j) {
    uint32_t o = 0;
    for (int m = 0; m < K; ++m) o |= uint32_t((j >> m) & 1) << tb[m];
    p.offs[j] = uint16_t(o);
  }
  const int ngroups = int(run_amps / D);
  if (ngroups % 32 || ngroups > 256) return cudaErrorInvalidValue;
  p.ngpl = ngroups / 32;
  // group g -> base: g's bits deposited into the non-target bits; lane l takes g = q * 32 + l
  for (int g = 0; g < ngroups; ++g) {
    uint32_t base = 0;
    for (int bit = 0, src = 0; src < 16; ++bit)
      if (!(tmask >> bit & 1)) base |= uint32_t((g >> src++) & 1) << bit;
    p.gbase[g] = uint16_t(base);
  }
  std::memcpy(p.m, matrix, sizeof(p.m));
  const int smem = 8 * UNITS * 16;  // 8 warps x 4 KB (8 KB for complex128 k = 4)
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_dense_wt<R, K, UNITS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dense_wt<R, K, UNITS>, 256, smem);
  if (per_sm < 1) per_sm = 1;
  uint64_t blocks = (p.npass + 7) / 8;
  const uint64_t cap = uint64_t(device_sm_count()) * per_sm;
  if (blocks > cap) blocks = cap;
  k_dense_wt<R, K, UNITS><<<unsigned(blocks), 256, smem, st>>>(p, static_cast<R*>(sv));
  return cudaGetLastError();
}

// Generalised permutation (out[perm[j]] = d[j] in[j], NumPy FMA-form complex
// product: bit-exact) on the same warp-transposed runs, for tables whose
// targets all sit in the lowest six bits (the register path strides lanes 64+
// bytes apart there: perm2 on bits (0,1) ran at 0.59 of the copy peak).
// Replaces apply_permutation_bits (reference statevec.py:63-81) for that layout.
template <typename R, int K>
struct WtPermP {
  uint64_t npass;
  int ngpl;
  uint32_t active;
  uint16_t gbase[256];
  uint16_t offs[1 << K];
  uint8_t pout[1 << K];  // member j goes to member pout[j]
  cplx<R> d[1 << K];
};

template <typename R, int K, int UNITS>
__global__ void __launch_bounds__(256)
k_perm_wt(const __grid_constant__ WtPermP<R, K> p, R* __restrict__ sv_r) {
  constexpr int D = 1 << K;
  constexpr int APU = 16 / (2 * int(sizeof(R)));
  using U = float4;
  extern __shared__ __align__(16) float4 wsm[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  U* slice = wsm + warp * UNITS;
  U* svu = reinterpret_cast<U*>(sv_r);
  const uint64_t nwarps = uint64_t(gridDim.x) * (blockDim.x >> 5);
  for (uint64_t run = uint64_t(blockIdx.x) * (blockDim.x >> 5) + warp; run < p.npass; run += nwarps) {
    U* g = svu + run * UNITS;
    U t[UNITS / 32];
#pragma unroll
    for (int i = 0; i < UNITS / 32; ++i) t[i] = __ldcs(g + i * 32 + lane);
#pragma unroll
    for (int i = 0; i < UNITS / 32; ++i) slice[wt_slot(i * 32 + lane)] = t[i];
    __syncwarp();
    for (int q = 0; q < p.ngpl; ++q) {
      const uint32_t b = p.gbase[q * 32 + lane];
      R ar[D], ai[D];
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const uint32_t a = b + p.offs[j];
        const R* e = reinterpret_cast<const R*>(slice + wt_slot(a / APU)) + 2 * (a % APU);
        ar[j] = e[0];
        ai[j] = e[1];
      }
#pragma unroll
      for (int j = 0; j < D; ++j) {
        if (!((p.active >> j) & 1u)) continue;
        R orr, oi;
        cmul_numpy(p.d[j].x, p.d[j].y, ar[j], ai[j], orr, oi);
        const uint32_t a = b + p.offs[p.pout[j]];
        R* e = reinterpret_cast<R*>(slice + wt_slot(a / APU)) + 2 * (a % APU);
        e[0] = orr;
        e[1] = oi;
      }
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < UNITS / 32; ++i) __stcs(g + i * 32 + lane, slice[wt_slot(i * 32 + lane)]);
    __syncwarp();
  }
}

template <typename R, int K>
static cudaError_t perm_wt_t(int nbits, const int* tb, const uint64_t* pout, const void* diag, uint64_t active,
                             void* sv, cudaStream_t st) {
  constexpr int D = 1 << K;
  constexpr int UNITS = 256;
  constexpr int APU = 16 / (2 * int(sizeof(R)));
  const uint64_t run_amps = uint64_t(UNITS) * APU;
  if ((uint64_t(1) << nbits) < run_amps) return cudaErrorInvalidValue;
  WtPermP<R, K> p;
  std::memset(&p, 0, sizeof p);
  p.npass = (uint64_t(1) << nbits) / run_amps;
  p.active = uint32_t(active);
  uint32_t tmask = 0;
  for (int m = 0; m < K; ++m) tmask |= 1u << tb[m];
  for (int j = 0; j < D; ++j) {
    uint32_t o = 0;
    for (int m = 0; m < K; ++m) o |= uint32_t((j >> m) & 1) << tb[m];
    p.offs[j] = uint16_t(o);
    p.pout[j] = uint8_t(pout[j]);
    p.d[j] = static_cast<const cplx<R>*>(diag)[j];
  }
  const int ngroups = int(run_amps / D);
  if (ngroups % 32 || ngroups > 256) return cudaErrorInvalidValue;
  p.ngpl = ngroups / 32;
  for (int g = 0; g < ngroups; ++g) {
    uint32_t base = 0;
    for (int bit = 0, src = 0; src < 16; ++bit)
      if (!(tmask >> bit & 1)) base |= uint32_t((g >> src++) & 1) << bit;
    p.gbase[g] = uint16_t(base);
  }
  const int smem = 8 * UNITS * 16;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_perm_wt<R, K, UNITS>, 256, smem);
  if (per_sm < 1) per_sm = 1;
  uint64_t blocks = (p.npass + 7) / 8;
  const uint64_t cap = uint64_t(device_sm_count()) * per_sm;
  if (blocks > cap) blocks = cap;
  k_perm_wt<R, K, UNITS><<<unsigned(blocks), 256, smem, st>>>(p, static_cast<R*>(sv));
  return cudaGetLastError();
}

cudaError_t launch_perm_wt(int dtype, int nbits, int k, const int* tb, const uint64_t* pout, const void* diag,
                           uint64_t active, void* sv, cudaStream_t st) {
  if (dtype == 1) {
    switch (k) {
      case 1: return perm_wt_t<double, 1>(nbits, tb, pout, diag, active, sv, st);
      case 2: return perm_wt_t<double, 2>(nbits, tb, pout, diag, active, sv, st);
      case 3: return perm_wt_t<double, 3>(nbits, tb, pout, diag, active, sv, st);
    }
  } else {
    switch (k) {
      case 1: return perm_wt_t<float, 1>(nbits, tb, pout, diag, active, sv, st);
      case 2: return perm_wt_t<float, 2>(nbits, tb, pout, diag, active, sv, st);
      case 3: return perm_wt_t<float, 3>(nbits, tb, pout, diag, active, sv, st);
      case 4: return perm_wt_t<float, 4>(nbits, tb, pout, diag, active, sv, st);
    }
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_dense_wt(int dtype, int nbits, int k, const int* tb, const void* matrix, void* sv,
                            cudaStream_t st) {
  if (dtype == 1) {
    switch (k) {
      case 1: return wt_t<double, 1>(nbits, tb, matrix, sv, st);
      case 2: return wt_t<double, 2>(nbits, tb, matrix, sv, st);
      case 3: return wt_t<double, 3>(nbits, tb, matrix, sv, st);
      case 4: return wt_t<double, 4>(nbits, tb, matrix, sv, st);
    }
  } else {
    switch (k) {
      case 1: return wt_t<float, 1>(nbits, tb, matrix, sv, st);
      case 2: return wt_t<float, 2>(nbits, tb, matrix, sv, st);
      case 3: return wt_t<float, 3>(nbits, tb, matrix, sv, st);
      case 4: return wt_t<float, 4>(nbits, tb, matrix, sv, st);
    }
  }
  return cudaErrorInvalidValue;
}

}  // namespace dsv
