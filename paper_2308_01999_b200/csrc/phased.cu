// phased.cu — dense k-qubit gate preceded by a phase polynomial that couples
// the targets to OUTSIDE qubits (the fold fuser's window, fusion_fold.py):
//
//   psi_g[j] <- sum_c M[j][c] * exp(i (gamma(x) + sum_m c_m alpha_m(x))) psi_g[c]
//
// where x are the group's outside index bits, alpha_m(x) = sum_b theta_mb x_b
// (cross terms t_ab x_a x_b with a = target m, b outside) and gamma(x) =
// sum_b theta_b x_b (outside linear terms).  All alpha_m and gamma are linear
// in the outside bits, so they are evaluated per group from byte tables
//   T[c][v][s] = sum over terms of slot s whose bit lies in byte c of the index
// (s = 0..k-1: alpha_m, s = k: gamma), kept in shared memory by a persistent
// grid.  One sincos per target per group, D-1 complex products for the member
// phases — ~10% on top of the 2^k x 2^k matrix, and it deletes the separate
// HBM pass every folded controlled-phase would otherwise cost (QFT-33: 152
// reference windows -> 7 phased windows).
#include <cmath>

#include "common.cuh"
#include "launch.h"

namespace dsv {

template <int K, typename R>
struct PhasedP {
  Geom g;                  // holes = targets (unit space)
  int nchunk;              // active index bytes
  int chunk_shift[8];      // amp-index shift of each active byte
  uint64_t offs[1 << K];   // member offsets (units)
  cplx<R> m[(1 << K) * (1 << K)];
  R msum[(1 << K) * (1 << K)];
};

// sin/cos after explicit reduction to [-pi, pi]: the fast float path is then
// accurate to ~1e-6 (c64 tolerance 1e-5); doubles keep the libm sincos
__device__ __forceinline__ void sincos_red(float a, float* sn, float* cs) {
  const float t = a - 6.28318530717958647692f * rintf(a * 0.15915494309189533577f);
  __sincosf(t, sn, cs);
}
__device__ __forceinline__ void sincos_red(double a, double* sn, double* cs) {
  const double t = a - 6.28318530717958647692 * rint(a * 0.15915494309189533577);
  sincos(t, sn, cs);
}

template <typename R>
__device__ __forceinline__ void cmul_into(R& xr, R& xi, R er, R ei) {
  const R r = xr * er - xi * ei;
  xi = xr * ei + xi * er;
  xr = r;
}

template <int K, class VT, bool M3>
__global__ void __launch_bounds__(256)
k_dense_phased(const __grid_constant__ PhasedP<K, typename VT::R> p, const cplx<typename VT::R>* __restrict__ tab,
               typename VT::V* __restrict__ sv) {
  using V = typename VT::V;
  using R = typename VT::R;
  constexpr int D = 1 << K;
  constexpr int L = VT::L;
  constexpr int S = K + 1;
  extern __shared__ __align__(16) unsigned char smem[];
  cplx<R>* st = reinterpret_cast<cplx<R>*>(smem);  // [nchunk][256][S] unit factors exp(i angle)
  const int ntab = p.nchunk * 256 * S;
  for (int i = threadIdx.x; i < ntab; i += blockDim.x) st[i] = tab[i];
  __syncthreads();
  for (uint64_t w = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; w < p.g.nwork;
       w += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t base = expand(p.g, w);
    V in[D];
#pragma unroll
    for (int j = 0; j < D; ++j) in[j] = ldg_s(sv + base + p.offs[j]);
#pragma unroll
    for (int l = 0; l < L; ++l) {
      const uint64_t amp = (L == 2) ? ((base << 1) | uint64_t(l)) : base;
      // per-slot factors exp(i alpha_s) = product over the index bytes of the
      // tabulated unit factors (no sin/cos per group: for complex128 the libm
      // pair cost more than the 2^k x 2^k product)
      R fr[S], fi[S];
      {
        const cplx<R>* row = st + size_t((amp >> p.chunk_shift[0]) & 255u) * S;
#pragma unroll
        for (int s = 0; s < S; ++s) {
          fr[s] = row[s].x;
          fi[s] = row[s].y;
        }
      }
      for (int c = 1; c < p.nchunk; ++c) {
        const cplx<R>* row = st + (size_t(c) * 256 + ((amp >> p.chunk_shift[c]) & 255u)) * S;
#pragma unroll
        for (int s = 0; s < S; ++s) cmul_into(fr[s], fi[s], row[s].x, row[s].y);
      }
      // P_j = exp(i gamma) * prod_{m in j} exp(i alpha_m), applied factor by factor
      R er = fr[K], ei = fi[K];
#pragma unroll
      for (int j = 0; j < D; ++j) {
        R ar, ai;
        VT::get(in[j], l, ar, ai);
        cmul_into(ar, ai, er, ei);
        VT::set(in[j], l, ar, ai);
      }
#pragma unroll
      for (int m = 0; m < K; ++m) {
        er = fr[m];
        ei = fi[m];
#pragma unroll
        for (int j = 0; j < D; ++j) {
          if (!((j >> m) & 1)) continue;
          R ar, ai;
          VT::get(in[j], l, ar, ai);
          cmul_into(ar, ai, er, ei);
          VT::set(in[j], l, ar, ai);
        }
      }
    }
    if constexpr (M3)
      matvec3m_store<D, VT>(p.m, p.msum, in, sv, base, p.offs);
    else
      matvec4m_store<D, VT>(p.m, in, sv, base, p.offs);
  }
}

template <int K, class VT, bool M3>
static cudaError_t phased_go(const PhasedP<K, typename VT::R>& p, size_t smem, uint64_t nwork,
                             const void* d_tab, void* sv, cudaStream_t st) {
  using R = typename VT::R;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_dense_phased<K, VT, M3>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dense_phased<K, VT, M3>, 256, smem);
  if (per_sm < 1) per_sm = 1;
  uint64_t blocks = (nwork + 255) / 256;
  const uint64_t cap = uint64_t(device_sm_count()) * per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) return cudaSuccess;
  k_dense_phased<K, VT, M3><<<unsigned(blocks), 256, smem, st>>>(p, static_cast<const cplx<R>*>(d_tab),
                                                                 static_cast<typename VT::V*>(sv));
  return cudaGetLastError();
}

template <int K, class VT>
static cudaError_t phased_t(const PhasedDesc& d, const void* matrix, const void* d_tab, void* sv,
                            cudaStream_t st) {
  using R = typename VT::R;
  constexpr int D = 1 << K;
  PhasedP<K, R> p;
  p.g = d.g;
  p.nchunk = d.nchunk;
  for (int c = 0; c < 8; ++c) p.chunk_shift[c] = c < d.nchunk ? d.chunk_shift[c] : 0;
  for (int j = 0; j < D; ++j) p.offs[j] = d.offs[j];
  const cplx<R>* m = static_cast<const cplx<R>*>(matrix);
  for (int i = 0; i < D * D; ++i) {
    p.m[i] = m[i];
    p.msum[i] = m[i].x + m[i].y;
  }
  const size_t smem = 2 * sizeof(R) * size_t(d.nchunk) * 256 * (K + 1);
  if (use_3m()) return phased_go<K, VT, true>(p, smem, d.g.nwork, d_tab, sv, st);
  return phased_go<K, VT, false>(p, smem, d.g.nwork, d_tab, sv, st);
}

template <class VT>
static cudaError_t phased_mode(int k, const PhasedDesc& d, const void* m, const void* tab, void* sv,
                               cudaStream_t st) {
  switch (k) {
    case 1: return phased_t<1, VT>(d, m, tab, sv, st);
    case 2: return phased_t<2, VT>(d, m, tab, sv, st);
    case 3: return phased_t<3, VT>(d, m, tab, sv, st);
    case 4: return phased_t<4, VT>(d, m, tab, sv, st);
    case 5: return phased_t<5, VT>(d, m, tab, sv, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_dense_phased(int dtype, int mode, int k, const PhasedDesc& d, const void* matrix,
                                const void* d_tab, void* sv, cudaStream_t st) {
  if (dtype == 1) return phased_mode<C128x1>(k, d, matrix, d_tab, sv, st);
  if (mode == MODE_VEC2) return phased_mode<C64x2>(k, d, matrix, d_tab, sv, st);
  return phased_mode<C64x1>(k, d, matrix, d_tab, sv, st);
}

}  // namespace dsv
