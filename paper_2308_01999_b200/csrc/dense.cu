// dense.cu — dense k-qubit gate application (replaces apply_dense_bits,
// reference statevec.py:44-60) and the fused dense expectation value
// (replaces StateVector.expectation's copy+apply+vdot, statevec.py:241-245).
//
// Register path (k <= 5): each thread owns ITEMS amplitude groups (two per
// unit in C64x2 mode), issues all 2^k loads of every group first (memory-
// level parallelism), then streams the 2^k outputs out row by row.  The
// 2^k x 2^k matrix lives in the kernel parameter block, i.e. the constant
// bank: every FFMA takes its matrix operand straight from c[0x0][...], warp-
// uniform, no shared memory.  Traffic is exactly one read + one write of the
// control-satisfied amplitudes, the algorithmic minimum 2*s*2^(n-c).
#include "common.cuh"
#include "launch.h"

namespace dsv {

template <int K, typename R>
struct DenseP {
  Geom g;
  int cached;  // members share 128-byte lines (low targets): L1-cached loads, not streaming
  int lanectl;  // 16-byte units with index bit 0 a CONTROL: only lane lanectl is transformed, else -1
  uint64_t offs[1 << K];
  cplx<R> m[(1 << K) * (1 << K)];
  R msum[(1 << K) * (1 << K)];  // re + im of m (3-multiplication products)
};

template <class VT, int K>
struct DenseItems {
  // aim for >= 64 B of loads in flight per thread
  static constexpr int bytes = int(sizeof(typename VT::V)) << K;
  static constexpr int value = bytes >= 64 ? 1 : 64 / bytes;
};

template <int K, class VT, int ITEMS, bool M3>
__global__ void __launch_bounds__(256)
k_dense(const __grid_constant__ DenseP<K, typename VT::R> p, typename VT::V* __restrict__ sv) {
  using V = typename VT::V;
  using R = typename VT::R;
  constexpr int D = 1 << K;
  constexpr int L = VT::L;
  const uint64_t w0 = uint64_t(blockIdx.x) * (uint64_t(blockDim.x) * ITEMS) + threadIdx.x;
  V in[ITEMS][D];
  uint64_t base[ITEMS];
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const uint64_t w = w0 + uint64_t(it) * blockDim.x;
    base[it] = expand(p.g, w);
    if (w < p.g.nwork) {
#pragma unroll
      for (int j = 0; j < D; ++j) in[it][j] = p.cached ? __ldg(sv + base[it] + p.offs[j]) : ldg_s(sv + base[it] + p.offs[j]);
    }
  }
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const uint64_t w = w0 + uint64_t(it) * blockDim.x;
    if (w >= p.g.nwork) continue;
    if constexpr (M3) {  // FMA-bound regime: 3-multiplication complex products
      matvec3m_store<D, VT>(p.m, p.msum, in[it], sv, base[it], p.offs, p.lanectl);
      continue;
    }
#pragma unroll
    for (int r = 0; r < D; ++r) {
      R accr[L], acci[L];
#pragma unroll
      for (int l = 0; l < L; ++l) { accr[l] = R(0); acci[l] = R(0); }
#pragma unroll
      for (int c = 0; c < D; ++c) {
        const R mr = p.m[r * D + c].x, mi = p.m[r * D + c].y;
#pragma unroll
        for (int l = 0; l < L; ++l) {
          R ar, ai;
          VT::get(in[it][c], l, ar, ai);
          accr[l] = fma(mr, ar, accr[l]);
          accr[l] = fma(-mi, ai, accr[l]);
          acci[l] = fma(mr, ai, acci[l]);
          acci[l] = fma(mi, ar, acci[l]);
        }
      }
      V out;
#pragma unroll
      for (int l = 0; l < L; ++l) VT::set(out, l, accr[l], acci[l]);
      if (L == 2 && p.lanectl >= 0) {  // control on index bit 0 not met: that lane keeps its input
        R xr, xi;
        VT::get(in[it][r], 1 - p.lanectl, xr, xi);
        VT::set(out, 1 - p.lanectl, xr, xi);
      }
      stg_s(sv + base[it] + p.offs[r], out);
    }
  }
}

template <int K, class VT>
static cudaError_t dense_reg_t(const Geom& g, const uint64_t* offs, const void* matrix, void* sv,
                               cudaStream_t st, int lanectl = -1) {
  using R = typename VT::R;
  constexpr int D = 1 << K;
  constexpr int ITEMS = DenseItems<VT, K>::value;
  DenseP<K, R> p;
  p.g = g;
  p.lanectl = lanectl;
  uint64_t span = 0;
  for (int j = 0; j < D; ++j) {
    p.offs[j] = offs[j];
    span |= offs[j];
  }
  p.cached = span != 0 && span * sizeof(typename VT::V) < 256;
  const cplx<R>* m = static_cast<const cplx<R>*>(matrix);
  for (int i = 0; i < D * D; ++i) {
    p.m[i] = m[i];
    p.msum[i] = m[i].x + m[i].y;
  }
  const uint64_t per_block = 256ull * ITEMS;
  const uint64_t blocks = (g.nwork + per_block - 1) / per_block;
  if (blocks == 0) return cudaSuccess;
  if (K >= 3 && use_3m())
    k_dense<K, VT, ITEMS, (K >= 3)><<<dim3(unsigned(blocks)), 256, 0, st>>>(p, static_cast<typename VT::V*>(sv));
  else
    k_dense<K, VT, ITEMS, false><<<dim3(unsigned(blocks)), 256, 0, st>>>(p, static_cast<typename VT::V*>(sv));
  return cudaGetLastError();
}

template <class VT>
static cudaError_t dense_reg_mode(int k, const Geom& g, const uint64_t* offs, const void* m,
                                  void* sv, cudaStream_t st) {
  switch (k) {
    case 0: return dense_reg_t<0, VT>(g, offs, m, sv, st);
    case 1: return dense_reg_t<1, VT>(g, offs, m, sv, st);
    case 2: return dense_reg_t<2, VT>(g, offs, m, sv, st);
    case 3: return dense_reg_t<3, VT>(g, offs, m, sv, st);
    case 4: return dense_reg_t<4, VT>(g, offs, m, sv, st);
    case 5: return dense_reg_t<5, VT>(g, offs, m, sv, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_dense_lanectl(int k, const Geom& g, const uint64_t* offs, const void* matrix, int lanectl,
                                 void* sv, cudaStream_t st) {
  switch (k) {
    case 1: return dense_reg_t<1, C64x2>(g, offs, matrix, sv, st, lanectl);
    case 2: return dense_reg_t<2, C64x2>(g, offs, matrix, sv, st, lanectl);
    case 3: return dense_reg_t<3, C64x2>(g, offs, matrix, sv, st, lanectl);
    case 4: return dense_reg_t<4, C64x2>(g, offs, matrix, sv, st, lanectl);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_dense_reg(int dtype, int mode, int k, const Geom& g, const uint64_t* offs,
                             const void* matrix, void* sv, cudaStream_t st) {
  if (dtype == 1) return dense_reg_mode<C128x1>(k, g, offs, matrix, sv, st);
  if (mode == MODE_VEC2) return dense_reg_mode<C64x2>(k, g, offs, matrix, sv, st);
  return dense_reg_mode<C64x1>(k, g, offs, matrix, sv, st);
}

// ---- generic path: any k <= 10 ----------------------------------------------
template <typename R>
__global__ void __launch_bounds__(256)
k_dense_generic(const __grid_constant__ Geom g, int k, const uint64_t* __restrict__ offs,
                const cplx<R>* __restrict__ mt, cplx<R>* __restrict__ sv) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx<R>* sh = reinterpret_cast<cplx<R>*>(smem_raw);
  const int D = 1 << k;
  for (uint64_t w = blockIdx.x; w < g.nwork; w += gridDim.x) {
    const uint64_t base = expand(g, w);
    for (int j = threadIdx.x; j < D; j += blockDim.x) sh[j] = sv[base + offs[j]];
    __syncthreads();
    for (int r = threadIdx.x; r < D; r += blockDim.x) {
      R ar = 0, ai = 0;
      for (int c = 0; c < D; ++c) {
        const cplx<R> m = mt[uint64_t(c) * D + r];
        const cplx<R> x = sh[c];
        ar = fma(m.x, x.x, ar);
        ar = fma(-m.y, x.y, ar);
        ai = fma(m.x, x.y, ai);
        ai = fma(m.y, x.x, ai);
      }
      sv[base + offs[r]] = cplx<R>{ar, ai};
    }
    __syncthreads();
  }
}

// ---- batched path: complex128 k = 6, complex64 k = 7 ---------------------------
// A CTA keeps the whole transposed matrix in shared memory and applies it to
// 32 groups at a time: thread (g, rb) loads members rb*RB .. of groups g and
// g + 16 into the [member][group] stage (consecutive lanes = consecutive
// groups, so loads and stores are coalesced when index bit 0 is free), then
// computes output rows rb*RB .. rb*RB + RB - 1 of both groups (each matrix
// entry, broadcast to the 16 lanes of a row block, feeds two groups).  FP64-FMA bound for complex128 (256 DFMA per
// amplitude: ~0.3 of the copy peak vs ~0.05 for the one-CTA-per-group
// generic kernel).
template <typename R, int K>
__global__ void __launch_bounds__(256)
k_dense_batched(const __grid_constant__ Geom g, const uint64_t* __restrict__ offs, const cplx<R>* __restrict__ mt,
                cplx<R>* __restrict__ sv) {
  constexpr int D = 1 << K;
  constexpr int G = 32;       // groups per batch; thread (gi, rb) takes groups gi and gi + 16
  constexpr int RB = D / 16;  // rows (and loaded members) per thread
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx<R>* Ms = reinterpret_cast<cplx<R>*>(smem_raw);  // [c][r]
  cplx<R>* X = Ms + D * D;                              // [c][g]
  uint64_t* os = reinterpret_cast<uint64_t*>(X + D * G);
  for (int i = threadIdx.x; i < D * D; i += blockDim.x) Ms[i] = mt[i];
  for (int i = threadIdx.x; i < D; i += blockDim.x) os[i] = offs[i];
  __syncthreads();
  const int gi = threadIdx.x & 15;
  const int r0 = (threadIdx.x >> 4) * RB;
  for (uint64_t b = blockIdx.x; b * G < g.nwork; b += gridDim.x) {
    uint64_t base[2];
    bool valid[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint64_t w = b * G + uint64_t(gi + 16 * h);
      valid[h] = w < g.nwork;
      base[h] = expand(g, valid[h] ? w : 0);
#pragma unroll
      for (int i = 0; i < RB; ++i) {
        const int c = r0 + i;
        X[c * G + gi + 16 * h] = valid[h] ? sv[base[h] + os[c]] : cplx<R>{R(0), R(0)};
      }
    }
    __syncthreads();
    R ar[2][RB], ai[2][RB];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int i = 0; i < RB; ++i) { ar[h][i] = R(0); ai[h][i] = R(0); }
#pragma unroll 2
    for (int c = 0; c < D; ++c) {
      const cplx<R> x0 = X[c * G + gi], x1 = X[c * G + gi + 16];
#pragma unroll
      for (int i = 0; i < RB; ++i) {
        const cplx<R> m = Ms[c * D + r0 + i];
        ar[0][i] = fma(m.x, x0.x, ar[0][i]);
        ar[0][i] = fma(-m.y, x0.y, ar[0][i]);
        ai[0][i] = fma(m.x, x0.y, ai[0][i]);
        ai[0][i] = fma(m.y, x0.x, ai[0][i]);
        ar[1][i] = fma(m.x, x1.x, ar[1][i]);
        ar[1][i] = fma(-m.y, x1.y, ar[1][i]);
        ai[1][i] = fma(m.x, x1.y, ai[1][i]);
        ai[1][i] = fma(m.y, x1.x, ai[1][i]);
      }
    }
    __syncthreads();  // every thread has read this batch's stage
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (valid[h]) {
#pragma unroll
        for (int i = 0; i < RB; ++i) sv[base[h] + os[r0 + i]] = cplx<R>{ar[h][i], ai[h][i]};
      }
  }
}

template <typename R, int K>
static cudaError_t dense_batched_go(const Geom& g, const uint64_t* d_offs, const void* d_matrix_t, void* sv,
                                    cudaStream_t st) {
  constexpr int D = 1 << K;
  const int smem = int((D * D + D * 32) * sizeof(cplx<R>) + D * sizeof(uint64_t));
  static bool attr_set[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_dense_batched<R, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr_set[dev] = true;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dense_batched<R, K>, 256, smem);
  if (per_sm < 1) per_sm = 1;
  const uint64_t batches = (g.nwork + 31) / 32;
  uint64_t blocks = uint64_t(device_sm_count()) * per_sm;
  if (blocks > batches) blocks = batches;
  k_dense_batched<R, K><<<unsigned(blocks), 256, smem, st>>>(g, d_offs, static_cast<const cplx<R>*>(d_matrix_t),
                                                          static_cast<cplx<R>*>(sv));
  return cudaGetLastError();
}

cudaError_t launch_dense_generic(int dtype, int k, const Geom& g, const uint64_t* d_offs,
                                 const void* d_matrix_t, void* sv, cudaStream_t st) {
  if (g.nwork == 0) return cudaSuccess;
  if (dtype == 1 && k == 6) return dense_batched_go<double, 6>(g, d_offs, d_matrix_t, sv, st);
  if (dtype == 0 && k == 7) return dense_batched_go<float, 7>(g, d_offs, d_matrix_t, sv, st);
  const unsigned blocks = unsigned(g.nwork < 148ull * 16 ? g.nwork : 148ull * 16);
  if (dtype == 1) {
    k_dense_generic<double><<<blocks, 256, (16u << k), st>>>(
        g, k, d_offs, static_cast<const cplx<double>*>(d_matrix_t), static_cast<cplx<double>*>(sv));
  } else {
    k_dense_generic<float><<<blocks, 256, (8u << k), st>>>(
        g, k, d_offs, static_cast<const cplx<float>*>(d_matrix_t), static_cast<cplx<float>*>(sv));
  }
  return cudaGetLastError();
}

// ---- fused expectation: sum_g psi_g^dagger M psi_g (read-only) ----------------
template <int K, class VT>
__global__ void __launch_bounds__(256)
k_expect_dense(const __grid_constant__ DenseP<K, typename VT::R> p,
               const typename VT::V* __restrict__ sv, double* __restrict__ partial) {
  using V = typename VT::V;
  using R = typename VT::R;
  constexpr int D = 1 << K;
  __shared__ double sh[8];
  double er = 0.0, ei = 0.0;
  for (uint64_t w = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; w < p.g.nwork;
       w += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t base = expand(p.g, w);
    V in[D];
#pragma unroll
    for (int j = 0; j < D; ++j) in[j] = ldg_s(sv + base + p.offs[j]);
    // the group's psi^dagger M psi in the state's precision (fp32 for
    // complex64: the fp64 pipe and float->double converts stay off the
    // per-element path), one fp64 add per group
    R gr = R(0), gi = R(0);
#pragma unroll
    for (int l = 0; l < VT::L; ++l) {  // groups per unit (two with 16-byte complex64 units)
#pragma unroll
      for (int r = 0; r < D; ++r) {
        R accr = R(0), acci = R(0);
#pragma unroll
        for (int c = 0; c < D; ++c) {
          R ar, ai;
          VT::get(in[c], l, ar, ai);
          const R mr = p.m[r * D + c].x, mi = p.m[r * D + c].y;
          accr = fma(mr, ar, accr);
          accr = fma(-mi, ai, accr);
          acci = fma(mr, ai, acci);
          acci = fma(mi, ar, acci);
        }
        R xr, xi;
        VT::get(in[r], l, xr, xi);
        // conj(x) * acc
        gr = fma(xr, accr, gr);
        gr = fma(xi, acci, gr);
        gi = fma(xr, acci, gi);
        gi = fma(-xi, accr, gi);
      }
    }
    er += double(gr);
    ei += double(gi);
  }
  const double sr = block_sum<256>(er, sh);
  const double si = block_sum<256>(ei, sh);
  if (threadIdx.x == 0) {
    partial[2 * blockIdx.x] = sr;
    partial[2 * blockIdx.x + 1] = si;
  }
}

template <int K, class VT>
static cudaError_t expect_dense_t(const Geom& g, const uint64_t* offs, const void* matrix,
                                  const void* sv, double* d_partial, uint64_t* nchunks,
                                  cudaStream_t st) {
  using R = typename VT::R;
  constexpr int D = 1 << K;
  DenseP<K, R> p;
  p.g = g;
  uint64_t span = 0;
  for (int j = 0; j < D; ++j) {
    p.offs[j] = offs[j];
    span |= offs[j];
  }
  p.cached = span != 0 && span * sizeof(typename VT::V) < 256;
  const cplx<R>* m = static_cast<const cplx<R>*>(matrix);
  for (int i = 0; i < D * D; ++i) p.m[i] = m[i];
  uint64_t blocks = (g.nwork + 255) / 256;
  if (blocks > 148ull * 8) blocks = 148ull * 8;
  if (blocks == 0) blocks = 1;
  *nchunks = blocks;
  k_expect_dense<K, VT><<<unsigned(blocks), 256, 0, st>>>(
      p, static_cast<const typename VT::V*>(sv), d_partial);
  return cudaGetLastError();
}

template <class VT>
static cudaError_t expect_dense_mode(int k, const Geom& g, const uint64_t* offs, const void* m,
                                     const void* sv, double* d_partial, uint64_t* nchunks,
                                     cudaStream_t st) {
  switch (k) {
    case 0: return expect_dense_t<0, VT>(g, offs, m, sv, d_partial, nchunks, st);
    case 1: return expect_dense_t<1, VT>(g, offs, m, sv, d_partial, nchunks, st);
    case 2: return expect_dense_t<2, VT>(g, offs, m, sv, d_partial, nchunks, st);
    case 3: return expect_dense_t<3, VT>(g, offs, m, sv, d_partial, nchunks, st);
    case 4: return expect_dense_t<4, VT>(g, offs, m, sv, d_partial, nchunks, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_expect_dense(int dtype, int mode, int k, const Geom& g, const uint64_t* offs,
                                const void* matrix, const void* sv, double* d_partial,
                                uint64_t* nchunks_out, cudaStream_t st) {
  if (dtype == 1) return expect_dense_mode<C128x1>(k, g, offs, matrix, sv, d_partial, nchunks_out, st);
  if (mode == MODE_VEC2) {  // two groups per thread: k <= 3 (k = 4 would spill)
    switch (k) {
      case 0: return expect_dense_t<0, C64x2>(g, offs, matrix, sv, d_partial, nchunks_out, st);
      case 1: return expect_dense_t<1, C64x2>(g, offs, matrix, sv, d_partial, nchunks_out, st);
      case 2: return expect_dense_t<2, C64x2>(g, offs, matrix, sv, d_partial, nchunks_out, st);
      case 3: return expect_dense_t<3, C64x2>(g, offs, matrix, sv, d_partial, nchunks_out, st);
    }
    return cudaErrorInvalidValue;
  }
  return expect_dense_mode<C64x1>(k, g, offs, matrix, sv, d_partial, nchunks_out, st);
}

}  // namespace dsv
