// layout.cu — data-movement and elementwise kernels:
//   * in-place index-bit swap        (StateVector.swap_index_bits, statevec.py:311-324)
//   * bit-ordered gather / scatter   (access / access_set, statevec.py:278-309)
//   * global<->local segment exchange (distsim.py:153-198 stage+scatter, done
//     as a one-pass in-place swap over peer-visible pointers)
//   * collapse / scale               (measure's collapse, statevec.py:229-237)
//   * Pauli rotation / product        (statevec.py:84-104, :196-207, copy-free)
#include <cstring>

#include "common.cuh"
#include "launch.h"

namespace dsv {

// ---- in-place bit swap ---------------------------------------------------------
// The index map pi (product of disjoint bit transpositions) is an involution,
// so every orbit has size 1 or 2: the owner of each orbit is its smaller
// index, which swaps the two amplitudes.  Data movement only => bit-exact.
template <class VT>
__global__ void __launch_bounds__(256)
k_swap_bits(typename VT::V* __restrict__ sv, uint64_t nunits, const __grid_constant__ SwapPairs sp) {
  using V = typename VT::V;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nunits;
       i += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t j = i;
    for (int q = 0; q < sp.np; ++q) {
      const uint64_t d = ((i >> sp.a[q]) ^ (i >> sp.b[q])) & 1ull;
      j ^= (d << sp.a[q]) | (d << sp.b[q]);
    }
    if (j > i) {
      const V x = ldg_s(sv + i);
      const V y = ldg_s(sv + j);
      stg_s(sv + i, y);
      stg_s(sv + j, x);
    }
  }
}

// Few pairs (p <= 3): enumerate only the orbit owners.  Work items run over
// the bits outside the pairs (holes = all pair bits), so consecutive threads
// take consecutive units and every access is a coalesced run; each item swaps
// its (4^p - 2^p) / 2 owner/partner pairs, ITEMS items in flight per thread.
template <class VT, int NSW, int ITEMS>
__global__ void __launch_bounds__(256)
k_swap_geom(typename VT::V* __restrict__ sv, const __grid_constant__ SwapGeomP p) {
  using V = typename VT::V;
  const uint64_t w0 = uint64_t(blockIdx.x) * (256ull * ITEMS) + threadIdx.x;
  V x[ITEMS][NSW], y[ITEMS][NSW];
  uint64_t base[ITEMS];
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const uint64_t w = w0 + uint64_t(it) * 256;
    base[it] = expand(p.g, w);
    if (w < p.g.nwork) {
#pragma unroll
      for (int q = 0; q < NSW; ++q) {
        x[it][q] = ldg_s(sv + base[it] + p.oi[q]);
        y[it][q] = ldg_s(sv + base[it] + p.oj[q]);
      }
    }
  }
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const uint64_t w = w0 + uint64_t(it) * 256;
    if (w >= p.g.nwork) continue;
#pragma unroll
    for (int q = 0; q < NSW; ++q) {
      stg_s(sv + base[it] + p.oi[q], y[it][q]);
      stg_s(sv + base[it] + p.oj[q], x[it][q]);
    }
  }
}

template <class VT, int NSW>
static cudaError_t swap_geom_t(const SwapGeomP& p, void* sv, cudaStream_t st) {
  constexpr int ITEMS = NSW >= 6 ? 1 : 4;
  const uint64_t blocks = (p.g.nwork + 256ull * ITEMS - 1) / (256ull * ITEMS);
  if (blocks == 0) return cudaSuccess;
  k_swap_geom<VT, NSW, ITEMS><<<unsigned(blocks), 256, 0, st>>>(static_cast<typename VT::V*>(sv), p);
  return cudaGetLastError();
}

template <class VT>
static cudaError_t swap_geom_mode(const SwapGeomP& p, void* sv, cudaStream_t st) {
  switch (p.nsw) {
    case 1: return swap_geom_t<VT, 1>(p, sv, st);
    case 6: return swap_geom_t<VT, 6>(p, sv, st);
    case 28: return swap_geom_t<VT, 28>(p, sv, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_swap_geom(int dtype, int mode, const SwapGeomP& p, void* sv, cudaStream_t st) {
  if (dtype == 1) return swap_geom_mode<C128x1>(p, sv, st);
  if (mode == MODE_VEC2) return swap_geom_mode<C64x2>(p, sv, st);
  return swap_geom_mode<C64x1>(p, sv, st);
}

// complex64 swap of index bit 0 with bit b: in 16-byte units (amplitudes
// 2u, 2u+1) the pair exchanges the odd half of unit u (unit bit b-1 = 0)
// with the even half of unit u | 2^(b-1); whole units move, so every sector is
// read and written once in full (the scalar path's 8-byte accesses used half
// of each sector per instruction).
__global__ void __launch_bounds__(256)
k_swap_bit0(float4* __restrict__ sv, const __grid_constant__ Geom g, uint64_t partner) {
  constexpr int ITEMS = 4;
  const uint64_t w0 = uint64_t(blockIdx.x) * (256ull * ITEMS) + threadIdx.x;
  float4 x[ITEMS], y[ITEMS];
  uint64_t u[ITEMS];
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const uint64_t w = w0 + uint64_t(it) * 256;
    u[it] = expand(g, w);
    if (w < g.nwork) {
      x[it] = ldg_s(sv + u[it]);
      y[it] = ldg_s(sv + (u[it] | partner));
    }
  }
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const uint64_t w = w0 + uint64_t(it) * 256;
    if (w >= g.nwork) continue;
    stg_s(sv + u[it], make_float4(x[it].x, x[it].y, y[it].x, y[it].y));
    stg_s(sv + (u[it] | partner), make_float4(x[it].z, x[it].w, y[it].z, y[it].w));
  }
}

cudaError_t launch_swap_bit0(int nbits, int b, void* sv, cudaStream_t st) {
  if (b < 1 || b >= nbits) return cudaErrorInvalidValue;
  Geom g;
  std::memset(&g, 0, sizeof g);
  // unit space (nbits - 1 bits) with unit bit b - 1 a hole
  const int ubits = nbits - 1, h = b - 1;
  g.nwork = 1ull << (ubits - 1);
  g.set_mask = 0;
  g.nseg = 0;
  const uint64_t lo = (1ull << h) - 1ull;
  if (lo) {
    g.seg[g.nseg] = lo;
    g.shift[g.nseg++] = 0;
  }
  g.seg[g.nseg] = ~((1ull << (h + 1)) - 1ull);
  g.shift[g.nseg++] = 1;
  const uint64_t blocks = (g.nwork + 1023) / 1024;
  if (blocks == 0) return cudaSuccess;
  k_swap_bit0<<<unsigned(blocks), 256, 0, st>>>(static_cast<float4*>(sv), g, 1ull << h);
  return cudaGetLastError();
}

static unsigned grid_for(uint64_t n, int per_thread = 1) {
  uint64_t b = (n + 256ull * per_thread - 1) / (256ull * per_thread);
  const uint64_t cap = 148ull * 64;
  if (b > cap) b = cap;
  if (b == 0) b = 1;
  return unsigned(b);
}

cudaError_t launch_swap_bits(int dtype, int mode, uint64_t nunits, const SwapPairs& sp, void* sv,
                             cudaStream_t st) {
  const unsigned g = grid_for(nunits);
  if (dtype == 1)
    k_swap_bits<C128x1><<<g, 256, 0, st>>>(static_cast<double2*>(sv), nunits, sp);
  else if (mode == MODE_VEC2)
    k_swap_bits<C64x2><<<g, 256, 0, st>>>(static_cast<float4*>(sv), nunits, sp);
  else
    k_swap_bits<C64x1><<<g, 256, 0, st>>>(static_cast<float2*>(sv), nunits, sp);
  return cudaGetLastError();
}

// ---- gather / scatter by bit ordering ------------------------------------------
struct Ordering {
  int n;
  int ord[64];
};

__device__ __forceinline__ uint64_t src_index(const Ordering& o, uint64_t j) {
  uint64_t s = 0;
  for (int b = 0; b < o.n; ++b) s |= ((j >> b) & 1ull) << o.ord[b];
  return s;
}

template <typename T>
__global__ void __launch_bounds__(256)
k_gather(const T* __restrict__ sv, T* __restrict__ out, uint64_t begin, uint64_t count,
         const __grid_constant__ Ordering o) {
  for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < count;
       t += uint64_t(gridDim.x) * blockDim.x)
    out[t] = sv[src_index(o, begin + t)];
}

template <typename T>
__global__ void __launch_bounds__(256)
k_scatter(T* __restrict__ sv, const T* __restrict__ in, uint64_t begin, uint64_t count,
          const __grid_constant__ Ordering o) {
  for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < count;
       t += uint64_t(gridDim.x) * blockDim.x)
    sv[src_index(o, begin + t)] = in[t];
}

cudaError_t launch_gather(int dtype, int nbits, const int32_t* ordering, uint64_t begin,
                          uint64_t count, const void* sv, void* d_out, cudaStream_t st) {
  Ordering o;
  o.n = nbits;
  for (int b = 0; b < nbits; ++b) o.ord[b] = ordering[b];
  const unsigned g = grid_for(count);
  if (dtype == 1)
    k_gather<double2><<<g, 256, 0, st>>>(static_cast<const double2*>(sv), static_cast<double2*>(d_out), begin, count, o);
  else
    k_gather<float2><<<g, 256, 0, st>>>(static_cast<const float2*>(sv), static_cast<float2*>(d_out), begin, count, o);
  return cudaGetLastError();
}

cudaError_t launch_scatter(int dtype, int nbits, const int32_t* ordering, uint64_t begin,
                           uint64_t count, void* sv, const void* d_in, cudaStream_t st) {
  Ordering o;
  o.n = nbits;
  for (int b = 0; b < nbits; ++b) o.ord[b] = ordering[b];
  const unsigned g = grid_for(count);
  if (dtype == 1)
    k_scatter<double2><<<g, 256, 0, st>>>(static_cast<double2*>(sv), static_cast<const double2*>(d_in), begin, count, o);
  else
    k_scatter<float2><<<g, 256, 0, st>>>(static_cast<float2*>(sv), static_cast<const float2*>(d_in), begin, count, o);
  return cudaGetLastError();
}

// ---- segment exchange -------------------------------------------------------------
// a[off | 1<<l] <-> b[off] for the t-th offset with bit l clear, t in [lo, hi).
// Each element pair is owned by exactly one thread (read both, write both), so
// two devices can split [0, 2^(n-1)) between them without a race.
template <typename V>
__global__ void __launch_bounds__(256)
k_exchange_halves(V* __restrict__ a, V* __restrict__ b, int l, uint64_t lo, uint64_t hi) {
  const uint64_t lowmask = (1ull << l) - 1ull;
  for (uint64_t t = lo + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < hi;
       t += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t off = ((t & ~lowmask) << 1) | (t & lowmask);
    V* pa = a + (off | (1ull << l));
    V* pb = b + off;
    const V x = ldg_s(pa);
    const V y = ldg_s(pb);
    stg_s(pa, y);
    stg_s(pb, x);
  }
}

cudaError_t launch_exchange_halves(int dtype, int mode, int l_unit, uint64_t lo, uint64_t hi,
                                   void* a, void* b, cudaStream_t st) {
  if (hi <= lo) return cudaSuccess;
  const unsigned g = grid_for(hi - lo, 4);
  if (dtype == 1)
    k_exchange_halves<double2><<<g, 256, 0, st>>>(static_cast<double2*>(a), static_cast<double2*>(b), l_unit, lo, hi);
  else if (mode == MODE_VEC2)
    k_exchange_halves<float4><<<g, 256, 0, st>>>(static_cast<float4*>(a), static_cast<float4*>(b), l_unit, lo, hi);
  else
    k_exchange_halves<float2><<<g, 256, 0, st>>>(static_cast<float2*>(a), static_cast<float2*>(b), l_unit, lo, hi);
  return cudaGetLastError();
}

// Masked exchange (a batch of q (global, local) index-bit swaps between two
// segments, distsim.py:153-198): for every offset `off` whose q local bits are
// clear, a[off | pa] <-> b[off | pb].  Work item t enumerates those offsets in
// unit space (g: holes at the local bits), so consecutive threads touch
// consecutive 16-byte units whenever the low bits are free.  LANE mode
// (complex64 with amplitude bit 0 among the local bits): units are the 16-byte
// pairs (x, x|1); only lane `la` of a's unit and lane `lb` of b's unit trade
// places, both units are read and written whole (no 8-byte remote accesses).
template <typename V, bool LANE>
__global__ void __launch_bounds__(256)
k_exchange_masked(V* __restrict__ a, V* __restrict__ b, const __grid_constant__ Geom g, uint64_t pa, uint64_t pb,
                  int la, int lb, uint64_t lo, uint64_t hi) {
  for (uint64_t t = lo + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < hi;
       t += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t off = expand(g, t);
    V* qa = a + (off | pa);
    V* qb = b + (off | pb);
    V x = ldg_s(qa);
    V y = ldg_s(qb);
    if constexpr (LANE) {
      float2 xa = la ? make_float2(x.z, x.w) : make_float2(x.x, x.y);
      float2 yb = lb ? make_float2(y.z, y.w) : make_float2(y.x, y.y);
      if (la) { x.z = yb.x; x.w = yb.y; } else { x.x = yb.x; x.y = yb.y; }
      if (lb) { y.z = xa.x; y.w = xa.y; } else { y.x = xa.x; y.y = xa.y; }
      stg_s(qa, x);
      stg_s(qb, y);
    } else {
      stg_s(qa, y);
      stg_s(qb, x);
    }
  }
}

cudaError_t launch_exchange_masked(int dtype, int mode, const Geom& g, uint64_t pa, uint64_t pb, int la, int lb,
                                   uint64_t lo, uint64_t hi, void* a, void* b, cudaStream_t st) {
  if (hi <= lo) return cudaSuccess;
  const unsigned gr = grid_for(hi - lo, 4);
  if (dtype == 1)
    k_exchange_masked<double2, false><<<gr, 256, 0, st>>>(static_cast<double2*>(a), static_cast<double2*>(b), g,
                                                          pa, pb, 0, 0, lo, hi);
  else if (mode == MODE_VEC2)
    k_exchange_masked<float4, false><<<gr, 256, 0, st>>>(static_cast<float4*>(a), static_cast<float4*>(b), g, pa,
                                                         pb, 0, 0, lo, hi);
  else
    k_exchange_masked<float4, true><<<gr, 256, 0, st>>>(static_cast<float4*>(a), static_cast<float4*>(b), g, pa,
                                                        pb, la, lb, lo, hi);
  return cudaGetLastError();
}

template <typename V>
__global__ void __launch_bounds__(256) k_exchange_all(V* __restrict__ a, V* __restrict__ b, uint64_t n) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const V x = ldg_s(a + i);
    const V y = ldg_s(b + i);
    stg_s(a + i, y);
    stg_s(b + i, x);
  }
}

cudaError_t launch_exchange_all(int dtype, uint64_t namps, void* a, void* b, cudaStream_t st) {
  // both dtypes move as 16-byte units (c64: two amplitudes per unit when even)
  if (dtype == 1) {
    k_exchange_all<double2><<<grid_for(namps, 4), 256, 0, st>>>(static_cast<double2*>(a), static_cast<double2*>(b), namps);
  } else if (namps % 2 == 0) {
    k_exchange_all<float4><<<grid_for(namps / 2, 4), 256, 0, st>>>(static_cast<float4*>(a), static_cast<float4*>(b), namps / 2);
  } else {
    k_exchange_all<float2><<<grid_for(namps, 4), 256, 0, st>>>(static_cast<float2*>(a), static_cast<float2*>(b), namps);
  }
  return cudaGetLastError();
}

// ---- collapse / scale ----------------------------------------------------------------
template <class VT>
__global__ void __launch_bounds__(256)
k_collapse(typename VT::V* __restrict__ sv, uint64_t nunits, uint64_t mask, uint64_t val, double scale) {
  using V = typename VT::V;
  using R = typename VT::R;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nunits;
       i += uint64_t(gridDim.x) * blockDim.x) {
    V v;
    if ((i & mask) == val) {
      v = ldg_s(sv + i);
#pragma unroll
      for (int l = 0; l < VT::L; ++l) {
        R re, im;
        VT::get(v, l, re, im);
        VT::set(v, l, R(double(re) * scale), R(double(im) * scale));
      }
    } else {
#pragma unroll
      for (int l = 0; l < VT::L; ++l) VT::set(v, l, R(0), R(0));
    }
    stg_s(sv + i, v);
  }
}

cudaError_t launch_collapse(int dtype, int mode, uint64_t nunits, uint64_t mask, uint64_t val,
                            double scale, void* sv, cudaStream_t st) {
  const unsigned g = grid_for(nunits, 4);
  if (dtype == 1)
    k_collapse<C128x1><<<g, 256, 0, st>>>(static_cast<double2*>(sv), nunits, mask, val, scale);
  else if (mode == MODE_VEC2)
    k_collapse<C64x2><<<g, 256, 0, st>>>(static_cast<float4*>(sv), nunits, mask, val, scale);
  else
    k_collapse<C64x1><<<g, 256, 0, st>>>(static_cast<float2*>(sv), nunits, mask, val, scale);
  return cudaGetLastError();
}

// ---- Pauli rotation / product ------------------------------------------------------------
// new_i = c * psi_i + B * (-1)^popcount(i & yz) * psi_{i ^ x}, computed in
// float64 and rounded once to the state precision.  Pairs (i, i^x) are owned
// by the index with bit h clear, so the update is a single in-place pass.
template <typename R> struct V2;
template <> struct V2<float> { using T = float2; };
template <> struct V2<double> { using T = double2; };

template <typename R>
__global__ void __launch_bounds__(256)
k_pauli(typename V2<R>::T* __restrict__ sv, uint64_t npairs, const __grid_constant__ PauliOp op) {
  using T = typename V2<R>::T;
  const int h = op.hbit;
  const uint64_t lowmask = h >= 0 ? (1ull << h) - 1ull : 0ull;
  for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < npairs;
       t += uint64_t(gridDim.x) * blockDim.x) {
    if (h < 0) {
      const T a = ldg_s(sv + t);
      const double sg = (__popcll(t & op.yzmask) & 1) ? -1.0 : 1.0;
      const double fr = op.c + sg * op.br, fi = sg * op.bi;
      const double ar = double(a.x), ai = double(a.y);
      stg_s(sv + t, T{R(fr * ar - fi * ai), R(fr * ai + fi * ar)});
    } else {
      const uint64_t i = ((t & ~lowmask) << 1) | (t & lowmask);
      const uint64_t j = i ^ op.xmask;
      const T a = ldg_s(sv + i);
      const T b = ldg_s(sv + j);
      const double si = (__popcll(i & op.yzmask) & 1) ? -1.0 : 1.0;
      const double sj = (__popcll(j & op.yzmask) & 1) ? -1.0 : 1.0;
      const double ar = double(a.x), ai = double(a.y), bir = double(b.x), bii = double(b.y);
      // new_i = c a + si B b ; new_j = c b + sj B a
      const double nir = op.c * ar + si * (op.br * bir - op.bi * bii);
      const double nii = op.c * ai + si * (op.br * bii + op.bi * bir);
      const double njr = op.c * bir + sj * (op.br * ar - op.bi * ai);
      const double nji = op.c * bii + sj * (op.br * ai + op.bi * ar);
      stg_s(sv + i, T{R(nir), R(nii)});
      stg_s(sv + j, T{R(njr), R(nji)});
    }
  }
}

cudaError_t launch_pauli(int dtype, int nbits, const PauliOp& op, void* sv, cudaStream_t st) {
  const uint64_t n = 1ull << nbits;
  const uint64_t npairs = op.hbit >= 0 ? n / 2 : n;
  const unsigned g = grid_for(npairs, 4);
  if (dtype == 1)
    k_pauli<double><<<g, 256, 0, st>>>(static_cast<double2*>(sv), npairs, op);
  else
    k_pauli<float><<<g, 256, 0, st>>>(static_cast<float2*>(sv), npairs, op);
  return cudaGetLastError();
}

}  // namespace dsv
