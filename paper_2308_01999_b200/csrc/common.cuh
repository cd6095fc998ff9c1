// common.cuh — shared device-side machinery for the dsv kernels (sm_100a).
//
// Index geometry.  Every gate / reduction kernel enumerates "work items":
// the 2^(n-H) assignments of the index bits that are NOT holes (holes =
// target bits + control bits, or the bits a reduction bins over).  A work
// item w is expanded to the base index of its amplitude group by inserting
// zeros at the hole positions, then OR-ing the control values — the
// device-side equivalent of the reference's `_controlled_subview` +
// `np.moveaxis` gather (statevec.py:26-41, :56-59), without materialising
// anything.  Consecutive threads take consecutive work items, so the lowest
// free bits vary fastest and HBM accesses coalesce whenever the low index
// bits are free.
#pragma once
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define DSV_MAX_GEOM_SEGS 41  // DSV_MAX_BITS holes + 1

namespace dsv {

struct Geom {
  uint64_t nwork;     // number of work items
  uint64_t set_mask;  // bits forced to 1 (controls with value 1), in unit index space
  int nseg;           // non-empty runs of free bits (<= holes + 1)
  int pad_;
  uint64_t seg[DSV_MAX_GEOM_SEGS];     // seg[i]: output bits that take (w << shift[i])
  uint8_t shift[DSV_MAX_GEOM_SEGS];    // holes below run i
};

// pdep-style expansion: the bits of w in free run i move up by the number of
// holes below the run (adjacent holes share one run boundary, so a window of
// contiguous targets costs two runs, not k + 1).
__device__ __forceinline__ uint64_t expand(const Geom& g, uint64_t w) {
  uint64_t r = g.set_mask;
  for (int i = 0; i < g.nseg; ++i) r |= (w << g.shift[i]) & g.seg[i];
  return r;
}

// ---- vector "unit" traits ---------------------------------------------------
// A unit is what one 8/16-byte access moves.  For complex64 with index bit 0
// free, a unit is a float4 holding TWO amplitudes (index bit 0 = lane), so a
// thread processes two groups at once with 128-bit accesses.  Otherwise a
// unit is one amplitude (float2 for c64, double2 for c128 — 16 B).
struct C64x2 {
  using V = float4;
  using R = float;
  static constexpr int L = 2;
  __device__ static __forceinline__ void get(const V& v, int l, R& re, R& im) {
    if (l == 0) { re = v.x; im = v.y; } else { re = v.z; im = v.w; }
  }
  __device__ static __forceinline__ void set(V& v, int l, R re, R im) {
    if (l == 0) { v.x = re; v.y = im; } else { v.z = re; v.w = im; }
  }
};
struct C64x1 {
  using V = float2;
  using R = float;
  static constexpr int L = 1;
  __device__ static __forceinline__ void get(const V& v, int, R& re, R& im) { re = v.x; im = v.y; }
  __device__ static __forceinline__ void set(V& v, int, R re, R im) { v.x = re; v.y = im; }
};
struct C128x1 {
  using V = double2;
  using R = double;
  static constexpr int L = 1;
  __device__ static __forceinline__ void get(const V& v, int, R& re, R& im) { re = v.x; im = v.y; }
  __device__ static __forceinline__ void set(V& v, int, R re, R im) { v.x = re; v.y = im; }
};

template <typename R> struct cplx { R x, y; };

// Exact-rounding helpers: explicit intrinsics so ptxas cannot contract or
// reassociate (the reference multiply is NumPy's FMA form).
__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }

// NumPy complex multiply d*a:  re = fma(dr, ar, -(di*ai)), im = fma(dr, ai, di*ar)
template <typename R>
__device__ __forceinline__ void cmul_numpy(R dr, R di, R ar, R ai, R& outr, R& outi) {
  outr = fma_rn(dr, ar, -mul_rn(di, ai));
  outi = fma_rn(dr, ai, mul_rn(di, ar));
}

// Streaming 128/64-bit global accesses.  The state is far larger than L2 and
// every amplitude is touched once per pass.
template <typename V> __device__ __forceinline__ V ldg_s(const V* p) { return __ldcs(p); }
template <typename V> __device__ __forceinline__ void stg_s(V* p, const V& v) { __stcs(p, v); }
// 32-byte streaming store (sm_100: STG.256): one full sector per lane
__device__ __forceinline__ void stcs32(void* p, float a, float b, float c, float d, float e, float f, float g,
                                       float h) {
  asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d),
               "f"(e), "f"(f), "f"(g), "f"(h)
               : "memory");
}

// 32-byte streaming load (sm_100: LDG.256)
__device__ __forceinline__ void ldcs32(const void* p, float (&v)[8]) {
  asm volatile("ld.global.cs.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
               : "l"(p));
}

// y = M x for one amplitude group held in registers (L lanes = groups per
// unit), streamed out row by row.  Complex products in the 3-multiplication
// (Gauss) form: with a + ib = M[r][c] and x + iy = x_c,
//   re = P - Q,  im = S - P - Q,  P = sum a x,  Q = sum b y,  S = sum (a+b)(x+y)
// — 3 FMAs per term instead of 4 (k >= 4 complex64 gates are FMA-bound on the
// CUDA cores).  m and msum (= a + b) live in the kernel-parameter constant bank.
template <int D, class VT>
__device__ __forceinline__ void matvec3m_store(const cplx<typename VT::R>* __restrict__ m,
                                               const typename VT::R* __restrict__ msum,
                                               const typename VT::V (&in)[D], typename VT::V* sv,
                                               uint64_t base, const uint64_t* offs, int lanectl = -1) {
  using R = typename VT::R;
  using V = typename VT::V;
  constexpr int L = VT::L;
  R xs[D][L], ys[D][L], ss[D][L];
#pragma unroll
  for (int c = 0; c < D; ++c)
#pragma unroll
    for (int l = 0; l < L; ++l) {
      VT::get(in[c], l, xs[c][l], ys[c][l]);
      ss[c][l] = xs[c][l] + ys[c][l];
    }
#pragma unroll
  for (int r = 0; r < D; ++r) {
    R P[L], Q[L], S[L];
#pragma unroll
    for (int l = 0; l < L; ++l) { P[l] = R(0); Q[l] = R(0); S[l] = R(0); }
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const R a = m[r * D + c].x, b = m[r * D + c].y, ab = msum[r * D + c];
#pragma unroll
      for (int l = 0; l < L; ++l) {
        P[l] = fma(a, xs[c][l], P[l]);
        Q[l] = fma(b, ys[c][l], Q[l]);
        S[l] = fma(ab, ss[c][l], S[l]);
      }
    }
    V out;
#pragma unroll
    for (int l = 0; l < L; ++l) VT::set(out, l, P[l] - Q[l], S[l] - P[l] - Q[l]);
    if (L == 2 && lanectl >= 0) {  // control on index bit 0 not met: that lane keeps its input
      R xr, xi;
      VT::get(in[r], 1 - lanectl, xr, xi);
      VT::set(out, 1 - lanectl, xr, xi);
    }
    __stcs(sv + base + offs[r], out);
  }
}

// same product with the plain 4-multiplication complex MACs
template <int D, class VT>
__device__ __forceinline__ void matvec4m_store(const cplx<typename VT::R>* __restrict__ m,
                                               const typename VT::V (&in)[D], typename VT::V* sv,
                                               uint64_t base, const uint64_t* offs, int lanectl = -1) {
  using R = typename VT::R;
  using V = typename VT::V;
  constexpr int L = VT::L;
#pragma unroll
  for (int r = 0; r < D; ++r) {
    R accr[L], acci[L];
#pragma unroll
    for (int l = 0; l < L; ++l) { accr[l] = R(0); acci[l] = R(0); }
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const R mr = m[r * D + c].x, mi = m[r * D + c].y;
#pragma unroll
      for (int l = 0; l < L; ++l) {
        R ar, ai;
        VT::get(in[c], l, ar, ai);
        accr[l] = fma(mr, ar, accr[l]);
        accr[l] = fma(-mi, ai, accr[l]);
        acci[l] = fma(mr, ai, acci[l]);
        acci[l] = fma(mi, ar, acci[l]);
      }
    }
    V out;
#pragma unroll
    for (int l = 0; l < L; ++l) VT::set(out, l, accr[l], acci[l]);
    __stcs(sv + base + offs[r], out);
  }
}

// DSV_DENSE_4M=1 selects the 4-multiplication products (A/B runs)
inline bool use_3m() {
  static const bool v = [] {
    const char* e = std::getenv("DSV_DENSE_4M");
    return !(e && e[0] == '1');
  }();
  return v;
}

// SM count of the current device (cached per device; persistent grids)
inline int device_sm_count() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (!cache[dev]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cache[dev] = n;
  }
  return cache[dev];
}

// ---- block reductions (fixed order => run-to-run deterministic) ------------
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
  #pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double r = 0.0;
  if (warp == 0) {
    r = lane < NT / 32 ? sh[lane] : 0.0;
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  }
  __syncthreads();
  return r;  // valid in thread 0
}

}  // namespace dsv
