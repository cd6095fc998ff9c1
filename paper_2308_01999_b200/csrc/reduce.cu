// reduce.cu — read-only reductions over the state (float64 accumulation,
// fixed summation order => bit-reproducible run to run):
//   * marginal probabilities / norm  (marginal_probabilities_bits, statevec.py:107-113;
//                                     norm_squared, core.py:62-71)
//   * Pauli-string expectation       (StateVector.expectation, statevec.py:246-253,
//                                     without the full-size copy)
//   * <a|b>                          (np.vdot)
//   * sampling scan                  (StateVector.sample, statevec.py:267-272)
//
// Each kernel writes one partial per (bin, chunk) block; launch_final_sum
// folds the partials of a bin in chunk order.  Block order is chunk-major
// with all bins of a chunk adjacent, so when the binned bits are low index
// bits the 2^k blocks sharing the same 128-B lines run concurrently and the
// lines are fetched from HBM once (L2 hit for the sibling bins).
#include "common.cuh"
#include "launch.h"

namespace dsv {

constexpr uint64_t kChunkUnits = uint64_t(kReduceThreads) * kReduceUnitsPerThread;

uint64_t chunks_for(uint64_t nunits) {
  uint64_t c = (nunits + kChunkUnits - 1) / kChunkUnits;
  return c ? c : 1;
}

// Amplitude bit 0 binned, complex64: float4 units (coalesced 16-byte loads)
// and two accumulators, one per value of bit 0 (no strided half-unit reads).
__global__ void __launch_bounds__(kReduceThreads)
k_probs_reg0(const float4* __restrict__ sv, const __grid_constant__ BinGeom bg, double* __restrict__ partial) {
  __shared__ double sh[kReduceThreads / 32];
  const uint64_t nbins = 1ull << bg.nb;
  const uint64_t chunk = blockIdx.x / nbins;
  const uint64_t bin = blockIdx.x % nbins;
  uint64_t bin_base = 0;
  for (int j = 0; j < bg.nb; ++j) bin_base |= ((bin >> j) & 1ull) << bg.bits[j];
  // per-batch sums in fp32 (8 terms), folded into fp64 accumulators: the
  // fp64 pipe stays off the per-element path
  double acc0 = 0.0, acc1 = 0.0;
  const uint64_t f0 = chunk * kChunkUnits + threadIdx.x;
  constexpr int kBatch = 8;
#pragma unroll 1
  for (int u0 = 0; u0 < kReduceUnitsPerThread; u0 += kBatch) {
    float4 v[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const uint64_t f = f0 + uint64_t(u0 + u) * kReduceThreads;
      v[u] = f < bg.g.nwork ? ldg_s(sv + (expand(bg.g, f) | bin_base)) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float b0 = 0.f, b1 = 0.f;
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      b0 = fmaf(v[u].x, v[u].x, fmaf(v[u].y, v[u].y, b0));
      b1 = fmaf(v[u].z, v[u].z, fmaf(v[u].w, v[u].w, b1));
    }
    acc0 += double(b0);
    acc1 += double(b1);
  }
  const double s0 = block_sum<kReduceThreads>(acc0, sh);
  const double s1 = block_sum<kReduceThreads>(acc1, sh);
  if (threadIdx.x == 0) {
    // full bin index: insert bit 0's value at bin position reg_j
    const uint64_t lo = bin & ((1ull << bg.reg_j) - 1ull), hi = bin >> bg.reg_j;
    const uint64_t b0 = lo | (hi << (bg.reg_j + 1));
    partial[b0 * bg.nchunks + chunk] = s0;
    partial[(b0 | (1ull << bg.reg_j)) * bg.nchunks + chunk] = s1;
  }
}

template <class VT>
__global__ void __launch_bounds__(kReduceThreads)
k_probs(const typename VT::V* __restrict__ sv, const __grid_constant__ BinGeom bg,
        double* __restrict__ partial) {
  using V = typename VT::V;
  using R = typename VT::R;
  __shared__ double sh[kReduceThreads / 32];
  const uint64_t nbins = 1ull << bg.nb;
  const uint64_t chunk = blockIdx.x / nbins;
  const uint64_t bin = blockIdx.x % nbins;
  uint64_t bin_base = 0;
  for (int j = 0; j < bg.nb; ++j) bin_base |= ((bin >> j) & 1ull) << bg.bits[j];
  double acc = 0.0;
  const uint64_t f0 = chunk * kChunkUnits + threadIdx.x;
  constexpr int kBatch = 8;
#pragma unroll 1
  for (int u0 = 0; u0 < kReduceUnitsPerThread; u0 += kBatch) {
    V v[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const uint64_t f = f0 + uint64_t(u0 + u) * kReduceThreads;
      if (f < bg.g.nwork) v[u] = ldg_s(sv + (expand(bg.g, f) | bin_base));
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const uint64_t f = f0 + uint64_t(u0 + u) * kReduceThreads;
      if (f < bg.g.nwork) {
#pragma unroll
        for (int l = 0; l < VT::L; ++l) {
          R re, im;
          VT::get(v[u], l, re, im);
          acc = fma(double(re), double(re), acc);
          acc = fma(double(im), double(im), acc);
        }
      }
    }
  }
  const double s = block_sum<kReduceThreads>(acc, sh);
  if (threadIdx.x == 0) partial[bin * bg.nchunks + chunk] = s;
}

// Marginals with the low binned bits resolved per thread ("inner" bits: the
// amplitude bits held by a thread's unit lanes and threadIdx, c64: 0..8,
// c128: 0..7; a block reads 256 consecutive units per step, so those bits
// are constant per (thread, lane)).  Outer binned bits (above) select the
// block's unit subset through the Geom as before.  Per-thread sums: fp32 per
// batch of 8 units folded into fp64 (complex64) / fp64 (complex128); block
// reduction in a fixed order (shuffle butterflies over the non-binned lane
// bits, then per-bin sums over warps): bit-reproducible.
template <class VT>
__global__ void __launch_bounds__(kReduceThreads)
k_probs_in(const typename VT::V* __restrict__ sv, const __grid_constant__ BinGeom bg,
           const __grid_constant__ InnerBins ib, double* __restrict__ partial) {
  using V = typename VT::V;
  using R = typename VT::R;
  constexpr int L = VT::L;  // amplitudes per unit (amp bit 0 = lane when 2)
  __shared__ double sm[kReduceThreads / 32][32][2];
  const uint64_t nouter = 1ull << bg.nb;
  const uint64_t chunk = blockIdx.x / nouter;
  const uint64_t ob = blockIdx.x % nouter;
  uint64_t bin_base = 0;
  for (int j = 0; j < bg.nb; ++j) bin_base |= ((ob >> j) & 1ull) << bg.bits[j];
  double acc[2] = {0.0, 0.0};
  const uint64_t f0 = chunk * kChunkUnits + threadIdx.x;
  constexpr int kBatch = 8;
#pragma unroll 1
  for (int u0 = 0; u0 < kReduceUnitsPerThread; u0 += kBatch) {
    V v[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const uint64_t f = f0 + uint64_t(u0 + u) * kReduceThreads;
      v[u] = f < bg.g.nwork ? ldg_s(sv + (expand(bg.g, f) | bin_base)) : V{};
    }
#pragma unroll
    for (int l = 0; l < L; ++l) {
      R b = R(0);
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        R re, im;
        VT::get(v[u], l, re, im);
        b = fma(re, re, fma(im, im, b));
      }
      acc[l] += double(b);
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // butterfly over lane bits that are not binned (fixed order)
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    if (!((ib.lane_mask >> i) & 1u)) {
#pragma unroll
      for (int l = 0; l < L; ++l) acc[l] += __shfl_xor_sync(0xffffffffu, acc[l], 1 << i);
    }
  }
  if ((lane & ~ib.lane_mask & 31u) == 0) {
    sm[warp][lane][0] = acc[0];
    sm[warp][lane][1] = L == 2 ? acc[1] : 0.0;
  }
  __syncthreads();
  const int t = threadIdx.x;
  if (t < (1 << ib.n)) {
    // inner bin t: its binned lane bits, lane slot (bit 0) and warp bits
    uint32_t lane_b = 0, warp_b = 0, h_b = 0;
    for (int j = 0; j < ib.n; ++j) {
      const uint32_t v = (t >> j) & 1u;
      const int pos = ib.pos[j];  // position in (h | lane << 1 | warp << 6) for c64, (lane | warp << 5) for c128
      if (L == 2 && pos == 0) h_b = v;
      else if (pos - (L == 2 ? 1 : 0) < 5) lane_b |= v << (pos - (L == 2 ? 1 : 0));
      else warp_b |= v << (pos - (L == 2 ? 6 : 5));
    }
    double s = 0.0;
    for (int w = 0; w < kReduceThreads / 32; ++w) {
      if ((uint32_t(w) & ib.warp_mask) != warp_b) continue;
      if (L == 2 && !ib.h_binned) s += sm[w][lane_b][0] + sm[w][lane_b][1];
      else s += sm[w][lane_b][h_b];
    }
    // final bin index: inner bit j -> user bit ib.fin[j], outer bit j -> bg.fin... (host packs)
    uint64_t fb = 0;
    for (int j = 0; j < ib.n; ++j) fb |= uint64_t((t >> j) & 1) << ib.fin[j];
    for (int j = 0; j < bg.nb; ++j) fb |= ((ob >> j) & 1ull) << ib.ofin[j];
    partial[fb * bg.nchunks + chunk] = s;
  }
}

cudaError_t launch_probs_in(int dtype, const BinGeom& bg, const InnerBins& ib, const void* sv,
                            double* d_partial, cudaStream_t st) {
  const uint64_t blocks = bg.nchunks << bg.nb;
  if (dtype == 1)
    k_probs_in<C128x1><<<unsigned(blocks), kReduceThreads, 0, st>>>(static_cast<const double2*>(sv), bg, ib, d_partial);
  else
    k_probs_in<C64x2><<<unsigned(blocks), kReduceThreads, 0, st>>>(static_cast<const float4*>(sv), bg, ib, d_partial);
  return cudaGetLastError();
}

cudaError_t launch_probs(int dtype, int mode, const BinGeom& bg, const void* sv, double* d_partial,
                         cudaStream_t st) {
  const uint64_t blocks = bg.nchunks << bg.nb;
  if (bg.reg_j >= 0) {
    k_probs_reg0<<<unsigned(blocks), kReduceThreads, 0, st>>>(static_cast<const float4*>(sv), bg, d_partial);
    return cudaGetLastError();
  }
  if (dtype == 1)
    k_probs<C128x1><<<unsigned(blocks), kReduceThreads, 0, st>>>(static_cast<const double2*>(sv), bg, d_partial);
  else if (mode == MODE_VEC2)
    k_probs<C64x2><<<unsigned(blocks), kReduceThreads, 0, st>>>(static_cast<const float4*>(sv), bg, d_partial);
  else
    k_probs<C64x1><<<unsigned(blocks), kReduceThreads, 0, st>>>(static_cast<const float2*>(sv), bg, d_partial);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(256)
k_final_sum(uint64_t nchunks, int ncomp, const double* __restrict__ partial, double* __restrict__ out) {
  __shared__ double sh[8];
  const uint64_t bin = blockIdx.x;
  for (int c = 0; c < ncomp; ++c) {
    double acc = 0.0;
    for (uint64_t k = threadIdx.x; k < nchunks; k += blockDim.x)
      acc += partial[(bin * nchunks + k) * ncomp + c];
    const double s = block_sum<256>(acc, sh);
    if (threadIdx.x == 0) out[bin * ncomp + c] = s;
  }
}

cudaError_t launch_final_sum(uint64_t nbins, uint64_t nchunks, int ncomp, const double* d_partial,
                             double* d_out, cudaStream_t st) {
  k_final_sum<<<unsigned(nbins), 256, 0, st>>>(nchunks, ncomp, d_partial, d_out);
  return cudaGetLastError();
}

// ---- Pauli expectation ----------------------------------------------------------------
// <psi|P|psi> = sum_i conj(psi_i) (P psi)_i with (P psi)_i = B s(i) psi_{i^x},
// B = (-i)^{#Y}, s(i) = (-1)^popcount(i & yz).  Each pair (i, i^x) is read
// once and contributes both of its terms.
template <typename V, typename R>
__global__ void __launch_bounds__(kReduceThreads)
k_expect_pauli(const V* __restrict__ sv, uint64_t npairs, const __grid_constant__ PauliOp op,
               double* __restrict__ partial) {
  __shared__ double sh[kReduceThreads / 32];
  const int h = op.hbit;
  const uint64_t lowmask = h >= 0 ? (1ull << h) - 1ull : 0ull;
  double er = 0.0, ei = 0.0;
  const uint64_t t0 = uint64_t(blockIdx.x) * kChunkUnits + threadIdx.x;
  // batches of kBatch pairs: every load of a batch is issued before the first
  // use (memory-level parallelism), missing tail entries read as zero
  constexpr int kBatch = 8;
#pragma unroll 1
  for (int u0 = 0; u0 < kReduceUnitsPerThread; u0 += kBatch) {
    V a[kBatch], b[kBatch];
    uint64_t ii[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const uint64_t t = t0 + uint64_t(u0 + u) * kReduceThreads;
      const bool on = t < npairs;
      const uint64_t i = h < 0 ? t : (((t & ~lowmask) << 1) | (t & lowmask));
      ii[u] = i;
      a[u] = on ? ldg_s(sv + i) : V{};
      if (h >= 0) b[u] = on ? ldg_s(sv + (i ^ op.xmask)) : V{};
    }
    // per-batch sums in the state's own precision (fp32 for complex64: no
    // float->double conversions or fp64 math per element), folded into fp64
    R br_ = R(0), bi_ = R(0);
    const R obr = R(op.br), obi = R(op.bi);
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const uint64_t i = ii[u];
      if (h < 0) {
        const R pr = a[u].x * a[u].x + a[u].y * a[u].y;
        br_ += (__popcll(i & op.yzmask) & 1) ? -pr : pr;
      } else {
        const uint64_t j = i ^ op.xmask;
        const R ar = a[u].x, ai = a[u].y, bre = b[u].x, bim = b[u].y;
        const R si = (__popcll(i & op.yzmask) & 1) ? R(-1) : R(1);
        const R sj = (__popcll(j & op.yzmask) & 1) ? R(-1) : R(1);
        // q = B * b ; term_i = conj(a) * q * si
        const R qr = obr * bre - obi * bim, qi = obr * bim + obi * bre;
        br_ += si * (ar * qr + ai * qi);
        bi_ += si * (ar * qi - ai * qr);
        // q' = B * a ; term_j = conj(b) * q' * sj
        const R pr = obr * ar - obi * ai, pi = obr * ai + obi * ar;
        br_ += sj * (bre * pr + bim * pi);
        bi_ += sj * (bre * pi - bim * pr);
      }
    }
    er += double(br_);
    ei += double(bi_);
  }
  const double sr = block_sum<kReduceThreads>(er, sh);
  const double si = block_sum<kReduceThreads>(ei, sh);
  if (threadIdx.x == 0) {
    partial[2 * blockIdx.x] = sr;
    partial[2 * blockIdx.x + 1] = si;
  }
}

// complex64 strings with an X/Y: pairs (i, i ^ x) read as 16-byte units (two
// adjacent amplitudes each), half the load instructions of the pair kernel
// above.  Unit u holds amplitudes 2u, 2u + 1; with x' = x >> 1 the partner
// unit is u ^ x', and when x flips bit 0 the partners swap halves (x' = 0:
// the pair lies inside one unit).
template <bool FLIP0, bool SELF>
__global__ void __launch_bounds__(kReduceThreads)
k_expect_pauli4(const float4* __restrict__ sv, uint64_t nwork, const __grid_constant__ PauliOp op,
                double* __restrict__ partial) {
  __shared__ double sh[kReduceThreads / 32];
  const uint64_t xu = op.xmask >> 1;
  const int hu = SELF ? 0 : 63 - __clzll(xu);
  const uint64_t lowmask = SELF ? 0 : (1ull << hu) - 1ull;
  double er = 0.0, ei = 0.0;
  const uint64_t t0 = uint64_t(blockIdx.x) * kChunkUnits + threadIdx.x;
  constexpr int kBatch = 8;
  const float obr = float(op.br), obi = float(op.bi);
#pragma unroll 1
  for (int u0 = 0; u0 < kReduceUnitsPerThread; u0 += kBatch) {
    float4 a[kBatch], b[kBatch];
    uint64_t ii[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const uint64_t t = t0 + uint64_t(u0 + u) * kReduceThreads;
      const bool on = t < nwork;
      const uint64_t i = SELF ? t : (((t & ~lowmask) << 1) | (t & lowmask));
      ii[u] = i;
      a[u] = on ? ldg_s(sv + i) : make_float4(0.f, 0.f, 0.f, 0.f);
      if constexpr (!SELF) b[u] = on ? ldg_s(sv + (i ^ xu)) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float br_ = 0.f, bi_ = 0.f;
    auto pair = [&](float ar, float ai, uint64_t ia, float bre, float bim, uint64_t jb) {
      const float si = (__popcll(ia & op.yzmask) & 1) ? -1.f : 1.f;
      const float sj = (__popcll(jb & op.yzmask) & 1) ? -1.f : 1.f;
      // q = B b ; term_i = conj(a) q si    q' = B a ; term_j = conj(b) q' sj
      const float qr = obr * bre - obi * bim, qi = obr * bim + obi * bre;
      br_ += si * (ar * qr + ai * qi);
      bi_ += si * (ar * qi - ai * qr);
      const float pr = obr * ar - obi * ai, pim = obr * ai + obi * ar;
      br_ += sj * (bre * pr + bim * pim);
      bi_ += sj * (bre * pim - bim * pr);
    };
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const uint64_t i2 = ii[u] << 1;
      if constexpr (SELF) {  // x = 1: amplitudes 2u, 2u + 1 of the same unit
        pair(a[u].x, a[u].y, i2, a[u].z, a[u].w, i2 + 1);
      } else {
        const uint64_t j2 = (ii[u] ^ xu) << 1;
        if constexpr (FLIP0) {
          pair(a[u].x, a[u].y, i2, b[u].z, b[u].w, j2 + 1);
          pair(a[u].z, a[u].w, i2 + 1, b[u].x, b[u].y, j2);
        } else {
          pair(a[u].x, a[u].y, i2, b[u].x, b[u].y, j2);
          pair(a[u].z, a[u].w, i2 + 1, b[u].z, b[u].w, j2 + 1);
        }
      }
    }
    er += double(br_);
    ei += double(bi_);
  }
  const double sr = block_sum<kReduceThreads>(er, sh);
  const double si = block_sum<kReduceThreads>(ei, sh);
  if (threadIdx.x == 0) {
    partial[2 * blockIdx.x] = sr;
    partial[2 * blockIdx.x + 1] = si;
  }
}

// Z-only strings (no bit flip): sum of +-|a_i|^2 over 16-byte units (two
// complex64 / one complex128 amplitude), per-batch sums in the state's
// precision folded into fp64.
template <typename R>
__global__ void __launch_bounds__(kReduceThreads)
k_expect_z(const float4* __restrict__ sv, uint64_t nunits, uint64_t yzmask, double* __restrict__ partial) {
  __shared__ double sh[kReduceThreads / 32];
  constexpr int APU = sizeof(R) == 4 ? 2 : 1;
  double er = 0.0;
  const uint64_t t0 = uint64_t(blockIdx.x) * kChunkUnits + threadIdx.x;
  constexpr int kBatch = 8;
#pragma unroll 1
  for (int u0 = 0; u0 < kReduceUnitsPerThread; u0 += kBatch) {
    float4 v[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const uint64_t t = t0 + uint64_t(u0 + u) * kReduceThreads;
      v[u] = t < nunits ? ldg_s(sv + t) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    R bs = R(0);
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const uint64_t i = (t0 + uint64_t(u0 + u) * kReduceThreads) * APU;
      if constexpr (APU == 2) {
        const float p0 = v[u].x * v[u].x + v[u].y * v[u].y;
        const float p1 = v[u].z * v[u].z + v[u].w * v[u].w;
        bs += (__popcll(i & yzmask) & 1) ? -p0 : p0;
        bs += (__popcll((i + 1) & yzmask) & 1) ? -p1 : p1;
      } else {
        const double2 d = *reinterpret_cast<const double2*>(&v[u]);
        const double pr = d.x * d.x + d.y * d.y;
        bs += (__popcll(i & yzmask) & 1) ? -pr : pr;
      }
    }
    er += double(bs);
  }
  const double sr = block_sum<kReduceThreads>(er, sh);
  if (threadIdx.x == 0) {
    partial[2 * blockIdx.x] = sr;
    partial[2 * blockIdx.x + 1] = 0.0;
  }
}

cudaError_t launch_expect_pauli(int dtype, int nbits, const PauliOp& op, const void* sv,
                                double* d_partial, uint64_t* nchunks_out, cudaStream_t st) {
  const uint64_t n = 1ull << nbits;
  if (op.hbit < 0 && n >= 2) {
    const uint64_t nunits = dtype == 1 ? n : n / 2;
    const uint64_t blocks = chunks_for(nunits);
    *nchunks_out = blocks;
    if (dtype == 1)
      k_expect_z<double><<<unsigned(blocks), kReduceThreads, 0, st>>>(static_cast<const float4*>(sv), nunits,
                                                                      op.yzmask, d_partial);
    else
      k_expect_z<float><<<unsigned(blocks), kReduceThreads, 0, st>>>(static_cast<const float4*>(sv), nunits,
                                                                     op.yzmask, d_partial);
    return cudaGetLastError();
  }
  if (dtype == 0 && op.hbit >= 0 && n >= 8) {
    const float4* s4 = static_cast<const float4*>(sv);
    const bool flip0 = op.xmask & 1ull, self = (op.xmask >> 1) == 0;
    const uint64_t nwork = self ? n / 2 : n / 4;  // units (x = 1) or unit pairs
    const uint64_t blocks = chunks_for(nwork);
    *nchunks_out = blocks;
    if (self)
      k_expect_pauli4<true, true><<<unsigned(blocks), kReduceThreads, 0, st>>>(s4, nwork, op, d_partial);
    else if (flip0)
      k_expect_pauli4<true, false><<<unsigned(blocks), kReduceThreads, 0, st>>>(s4, nwork, op, d_partial);
    else
      k_expect_pauli4<false, false><<<unsigned(blocks), kReduceThreads, 0, st>>>(s4, nwork, op, d_partial);
    return cudaGetLastError();
  }
  const uint64_t npairs = op.hbit >= 0 ? n / 2 : n;
  const uint64_t blocks = chunks_for(npairs);
  *nchunks_out = blocks;
  if (dtype == 1)
    k_expect_pauli<double2, double><<<unsigned(blocks), kReduceThreads, 0, st>>>(
        static_cast<const double2*>(sv), npairs, op, d_partial);
  else
    k_expect_pauli<float2, float><<<unsigned(blocks), kReduceThreads, 0, st>>>(
        static_cast<const float2*>(sv), npairs, op, d_partial);
  return cudaGetLastError();
}

// ---- <a|b> ----------------------------------------------------------------------------
template <typename V, typename R>
__global__ void __launch_bounds__(kReduceThreads)
k_inner(const V* __restrict__ a, const V* __restrict__ b, uint64_t n, double* __restrict__ partial) {
  __shared__ double sh[kReduceThreads / 32];
  double er = 0.0, ei = 0.0;
  const uint64_t t0 = uint64_t(blockIdx.x) * kChunkUnits + threadIdx.x;
  constexpr int kBatch = 8;
#pragma unroll 1
  for (int u0 = 0; u0 < kReduceUnitsPerThread; u0 += kBatch) {
    V x[kBatch], y[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const uint64_t t = t0 + uint64_t(u0 + u) * kReduceThreads;
      const bool on = t < n;
      x[u] = on ? ldg_s(a + t) : V{};
      y[u] = on ? ldg_s(b + t) : V{};
    }
    // per-batch sums in the vectors' precision, folded into fp64
    R sr_ = R(0), si_ = R(0);
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      sr_ += x[u].x * y[u].x + x[u].y * y[u].y;
      si_ += x[u].x * y[u].y - x[u].y * y[u].x;
    }
    er += double(sr_);
    ei += double(si_);
  }
  const double sr = block_sum<kReduceThreads>(er, sh);
  const double si = block_sum<kReduceThreads>(ei, sh);
  if (threadIdx.x == 0) {
    partial[2 * blockIdx.x] = sr;
    partial[2 * blockIdx.x + 1] = si;
  }
}

cudaError_t launch_inner(int dtype, uint64_t namps, const void* a, const void* b,
                         double* d_partial, uint64_t* nchunks_out, cudaStream_t st) {
  const uint64_t blocks = chunks_for(namps);
  *nchunks_out = blocks;
  if (dtype == 1)
    k_inner<double2, double><<<unsigned(blocks), kReduceThreads, 0, st>>>(
        static_cast<const double2*>(a), static_cast<const double2*>(b), namps, d_partial);
  else
    k_inner<float2, float><<<unsigned(blocks), kReduceThreads, 0, st>>>(
        static_cast<const float2*>(a), static_cast<const float2*>(b), namps, d_partial);
  return cudaGetLastError();
}

// ---- sampling: warp per shot, scan one chunk with an inclusive warp prefix ----------------
template <typename V>
__global__ void __launch_bounds__(256)
k_sample_scan(const V* __restrict__ sv, uint64_t namps, uint64_t chunk_amps, int64_t shots,
              const uint64_t* __restrict__ chunk, const double* __restrict__ resid,
              uint64_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t s = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (s >= shots) return;
  const uint64_t begin = chunk[s] * chunk_amps;
  uint64_t end = begin + chunk_amps;
  if (end > namps) end = namps;
  const double target = resid[s];
  double run = 0.0;
  // rounding fallback (the in-chunk scan sums in a different order than the
  // chunk totals): the last amplitude of the chunk with nonzero probability,
  // so a shot never lands on an impossible outcome (the reference clips to a
  // valid index, statevec.py:270-272)
  uint64_t found = end - 1;
  bool any_nz = false;
  for (uint64_t i0 = begin; i0 < end; i0 += 32) {
    const uint64_t i = i0 + lane;
    double p = 0.0;
    if (i < end) {
      const V a = sv[i];
      p = double(a.x) * double(a.x) + double(a.y) * double(a.y);
    }
    const unsigned nz = __ballot_sync(0xffffffffu, p > 0.0);
    if (nz) {
      found = i0 + 31 - __clz(nz);
      any_nz = true;
    }
    // inclusive scan across the warp
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double q = __shfl_up_sync(0xffffffffu, p, o);
      if (lane >= o) p += q;
    }
    const unsigned hit = __ballot_sync(0xffffffffu, (i < end) && (run + p > target));
    if (hit) {
      found = i0 + __ffs(hit) - 1;
      any_nz = true;
      break;
    }
    run += __shfl_sync(0xffffffffu, p, 31);
  }
  if (lane == 0) out[s] = any_nz ? found : end - 1;
}

cudaError_t launch_sample_scan(int dtype, uint64_t namps, uint64_t chunk_amps, int64_t shots,
                               const uint64_t* d_chunk, const double* d_resid, const void* sv,
                               uint64_t* d_out, cudaStream_t st) {
  const uint64_t blocks = (uint64_t(shots) * 32 + 255) / 256;
  if (dtype == 1)
    k_sample_scan<double2><<<unsigned(blocks), 256, 0, st>>>(static_cast<const double2*>(sv), namps,
                                                            chunk_amps, shots, d_chunk, d_resid, d_out);
  else
    k_sample_scan<float2><<<unsigned(blocks), 256, 0, st>>>(static_cast<const float2*>(sv), namps,
                                                           chunk_amps, shots, d_chunk, d_resid, d_out);
  return cudaGetLastError();
}

}  // namespace dsv
