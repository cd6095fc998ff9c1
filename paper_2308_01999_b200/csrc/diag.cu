// diag.cu — streaming diagonal-gate kernel (the QFT hot path after fusion:
// 119 of the 152 fused ops of QFT-33 are diagonals).
//
// A (controlled) diagonal is folded into ONE table over the union B of its
// target and control bits (|B| <= 12 for complex64, 11 for complex128):
// entry x holds diag[j(x)] when the controls in x are satisfied, else 1.  The
// kernel then streams the whole vector as contiguous 16-byte units (float4 =
// two complex64 amplitudes, or one complex128), so there is no index
// expansion at all; each unit looks its entry up in a shared-memory copy of
// the table.
//
// Index math is hoisted out of the per-unit path: a warp owns 32*ITEMS
// consecutive units per iteration, so the table index of unit
// base + it*32 + lane is  jl(lane) | jit(it) | jb(base)  — the lane part is
// computed once per thread, the `it` part once per kernel, the base part once
// per warp iteration.
//
// Traffic: units whose 32-byte sector holds no active entry (entry == 1
// exactly, or controls unsatisfied) are neither read nor written; sectors
// with at least one active entry are read and written whole (inactive
// amplitudes are written back bit-identical), so the DRAM never sees a
// partial-sector write.  The product is NumPy's FMA form => bit-exact.
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "launch.h"

namespace dsv {

struct DiagStreamP {
  uint64_t nunits;
  int kk;              // table bits
  int lane_m;          // table bit living inside a float4 unit (complex64 amp bit 0), -1 if none
  int ub[kDiagStreamMaxBits];  // unit-space bit of table bit m (-1: lane bit)
};

template <typename R, int L, int ITEMS, int MINB>
__global__ void __launch_bounds__(256, MINB)
k_diag_stream(const __grid_constant__ DiagStreamP p, const unsigned char* __restrict__ tab,
              typename std::conditional<L == 2, float4, double2>::type* __restrict__ sv) {
  using V = typename std::conditional<L == 2, float4, double2>::type;
  constexpr int LOG_ITEMS = ITEMS == 8 ? 3 : (ITEMS == 4 ? 2 : (ITEMS == 2 ? 1 : 0));
  extern __shared__ __align__(16) unsigned char smem[];
  const int D = 1 << p.kk;
  cplx<R>* sd = reinterpret_cast<cplx<R>*>(smem);
  unsigned char* sf = smem + sizeof(cplx<R>) * D;
  {
    const cplx<R>* gd = reinterpret_cast<const cplx<R>*>(tab);
    const unsigned char* gf = tab + sizeof(cplx<R>) * D;
    for (int j = threadIdx.x; j < D; j += blockDim.x) {
      sd[j] = gd[j];
      sf[j] = gf[j];
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t jl = 0, lanebit = 0;
  uint32_t jit[ITEMS];
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) jit[it] = 0;
  uint64_t hi_mask = 0;  // table bits taken from the warp base
  for (int m = 0; m < p.kk; ++m) {
    const int b = p.ub[m];
    if (b < 0) {
      lanebit = 1u << m;
    } else if (b < 5) {
      jl |= uint32_t((lane >> b) & 1) << m;
    } else if (b < 5 + LOG_ITEMS) {
#pragma unroll
      for (int it = 0; it < ITEMS; ++it) jit[it] |= uint32_t((it >> (b - 5)) & 1) << m;
    } else {
      hi_mask |= 1ull << m;
    }
  }
  const uint64_t span = 32ull * ITEMS;
  const uint64_t warp0 = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t base = warp0 * span; base < p.nunits; base += nwarps * span) {
    uint32_t jb = 0;
    for (uint64_t hm = hi_mask; hm; hm &= hm - 1) {
      const int m = __ffsll(hm) - 1;
      jb |= uint32_t((base >> p.ub[m]) & 1ull) << m;
    }
    V v[ITEMS];
    uint32_t jj[ITEMS];
    bool touch[ITEMS];
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
      const uint64_t u = base + uint64_t(it) * 32 + lane;
      jj[it] = jl | jit[it] | jb;
      touch[it] = u < p.nunits && (sf[jj[it]] & 2);
      if (touch[it]) v[it] = ldg_s(sv + u);
    }
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
      if (!touch[it]) continue;
      const uint64_t u = base + uint64_t(it) * 32 + lane;
      if constexpr (L == 2) {
        const uint32_t j0 = jj[it], j1 = jj[it] | lanebit;
        if (sf[j0] & 1) {
          const cplx<R> d = sd[j0];
          float orr, oi;
          cmul_numpy(d.x, d.y, v[it].x, v[it].y, orr, oi);
          v[it].x = orr;
          v[it].y = oi;
        }
        if (sf[j1] & 1) {
          const cplx<R> d = sd[j1];
          float orr, oi;
          cmul_numpy(d.x, d.y, v[it].z, v[it].w, orr, oi);
          v[it].z = orr;
          v[it].w = oi;
        }
      } else {
        const uint32_t j0 = jj[it];
        if (sf[j0] & 1) {
          const cplx<R> d = sd[j0];
          R orr, oi;
          cmul_numpy(d.x, d.y, v[it].x, v[it].y, orr, oi);
          v[it].x = orr;
          v[it].y = oi;
        }
      }
      stg_s(sv + u, v[it]);
    }
  }
}

template <typename R, int L, int ITEMS, int MINB>
static cudaError_t diag_stream_go(const DiagStreamP& p, const void* d_tab, void* sv, size_t smem,
                                  cudaStream_t st) {
  using V = typename std::conditional<L == 2, float4, double2>::type;
  const uint64_t per_block = 256ull * ITEMS;
  uint64_t blocks = (p.nunits + per_block - 1) / per_block;
  const uint64_t cap = uint64_t(device_sm_count()) * MINB;  // persistent: MINB x 256 threads per SM
  if (blocks > cap) blocks = cap;
  if (blocks == 0) blocks = 1;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_diag_stream<R, L, ITEMS, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  k_diag_stream<R, L, ITEMS, MINB><<<unsigned(blocks), 256, smem, st>>>(
      p, static_cast<const unsigned char*>(d_tab), static_cast<V*>(sv));
  return cudaGetLastError();
}

cudaError_t launch_diag_stream(int dtype, int nbits, int kk, const int* amp_bits, const void* d_tab,
                               void* sv, cudaStream_t st) {
  DiagStreamP p;
  p.kk = kk;
  p.lane_m = -1;
  const int shift = dtype == 1 ? 0 : 1;
  p.nunits = nbits >= shift ? (1ull << (nbits - shift)) : 1;
  for (int m = 0; m < kDiagStreamMaxBits; ++m) p.ub[m] = 0;
  for (int m = 0; m < kk; ++m) {
    p.ub[m] = amp_bits[m] - shift;
    if (p.ub[m] < 0) p.lane_m = m;
  }
  // variant: DSV_DIAG_VARIANT=0 -> 8 units/thread, 4 CTAs/SM; 1 -> 4 units, 8 CTAs/SM
  static const int variant = [] {
    const char* e = std::getenv("DSV_DIAG_VARIANT");
    return e ? std::atoi(e) : 0;
  }();
  const size_t es = dtype == 1 ? 16 : 8;
  const size_t smem = (es + 1) << kk;
  if (variant == 0) {
    if (dtype == 1) return diag_stream_go<double, 1, 8, 4>(p, d_tab, sv, smem, st);
    return diag_stream_go<float, 2, 8, 4>(p, d_tab, sv, smem, st);
  }
  if (dtype == 1) return diag_stream_go<double, 1, 4, 8>(p, d_tab, sv, smem, st);
  return diag_stream_go<float, 2, 4, 8>(p, d_tab, sv, smem, st);
}

}  // namespace dsv
