// perm.cu — generalised-permutation / diagonal gate application (replaces
// apply_permutation_bits, reference statevec.py:63-81):
//     out[perm[j]] = diag[j] * in[j]     for every control-satisfied group.
//
// Bit-exact with the reference: the product is NumPy's FMA form
// (re = fma(dr, ar, -(di*ai)), im = fma(dr, ai, di*ar)), written with
// explicit round-to-nearest intrinsics so ptxas cannot re-contract it.
//
// Table entries with perm[j] == j and diag[j] == 1 are skipped entirely (the
// `active` mask): their amplitudes are neither read nor written.  The active
// set is closed under perm, so reading only active inputs and writing only
// active outputs is complete.  For an unfused controlled phase this halves
// the touched amplitudes on top of the control subcube (2*s*2^(n-2) bytes).
#include <cstring>

#include "common.cuh"
#include "launch.h"

#define DSV_MAX_TARGETS_ 10

namespace dsv {

template <int K, typename R>
struct PermP {
  Geom g;
  int cached;       // members share 128-byte lines (low targets): L1-cached loads
  int lanectl;      // 16-byte units with index bit 0 a CONTROL: only lane (bit 0 value) lanectl moves, else -1
  uint64_t active;  // bit j set: entry j moves or scales
  uint64_t offs_in[1 << K];
  uint64_t offs_out[1 << K];  // offs[perm[j]]
  uint32_t psel[1 << K];      // lanectl: bit perm[j] set (the destination's other lane keeps its own value;
                              // a one-hot mask, not an index, so in[][] stays in registers)
  cplx<R> d[1 << K];
};

template <class VT, int K>
struct PermItems {
  static constexpr int bytes = int(sizeof(typename VT::V)) << K;
  static constexpr int value = bytes >= 64 ? 1 : 64 / bytes;
};

template <int K, class VT, int ITEMS, bool LANECTL = false>
__global__ void __launch_bounds__(256)
k_perm(const __grid_constant__ PermP<K, typename VT::R> p, typename VT::V* __restrict__ sv) {
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
      for (int j = 0; j < D; ++j)
        if ((p.active >> j) & 1ull)
          in[it][j] = p.cached ? __ldg(sv + base[it] + p.offs_in[j]) : ldg_s(sv + base[it] + p.offs_in[j]);
    }
  }
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const uint64_t w = w0 + uint64_t(it) * blockDim.x;
    if (w >= p.g.nwork) continue;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      if (!((p.active >> j) & 1ull)) continue;
      const R dr = p.d[j].x, di = p.d[j].y;
      V out;
#pragma unroll
      for (int l = 0; l < L; ++l) {
        R ar, ai, orr, oi;
        if (LANECTL && l != p.lanectl) {  // control not met: the destination keeps its lane
          orr = R(0);
          oi = R(0);
#pragma unroll
          for (int q = 0; q < D; ++q) {
            R tr, ti;
            VT::get(in[it][q], l, tr, ti);
            const bool s = (p.psel[j] >> q) & 1u;
            orr = s ? tr : orr;
            oi = s ? ti : oi;
          }
        } else {
          VT::get(in[it][j], l, ar, ai);
          cmul_numpy(dr, di, ar, ai, orr, oi);
        }
        VT::set(out, l, orr, oi);
      }
      stg_s(sv + base[it] + p.offs_out[j], out);
    }
  }
}

template <int K, class VT>
static cudaError_t perm_reg_t(const Geom& g, const uint64_t* offs_in, const uint64_t* offs_out,
                              const void* diag, uint64_t active, void* sv, cudaStream_t st,
                              int lanectl = -1, const uint8_t* pdst = nullptr) {
  using R = typename VT::R;
  constexpr int D = 1 << K;
  constexpr int ITEMS = PermItems<VT, K>::value;
  PermP<K, R> p;
  p.g = g;
  p.active = active;
  p.lanectl = lanectl;
  for (int j = 0; j < D; ++j) p.psel[j] = 1u << (pdst ? pdst[j] : j);
  uint64_t span = 0;
  for (int j = 0; j < D; ++j) span |= offs_in[j];
  p.cached = span != 0 && span * sizeof(typename VT::V) < 256;
  const cplx<R>* d = static_cast<const cplx<R>*>(diag);
  for (int j = 0; j < D; ++j) {
    p.offs_in[j] = offs_in[j];
    p.offs_out[j] = offs_out[j];
    p.d[j] = d[j];
  }
  const uint64_t per_block = 256ull * ITEMS;
  const uint64_t blocks = (g.nwork + per_block - 1) / per_block;
  if (blocks == 0 || active == 0) return cudaSuccess;
  if (lanectl >= 0) {
    if constexpr (VT::L == 2)
      k_perm<K, VT, ITEMS, true><<<dim3(unsigned(blocks)), 256, 0, st>>>(p, static_cast<typename VT::V*>(sv));
    else
      return cudaErrorInvalidValue;
  } else {
    k_perm<K, VT, ITEMS, false><<<dim3(unsigned(blocks)), 256, 0, st>>>(p, static_cast<typename VT::V*>(sv));
  }
  return cudaGetLastError();
}

template <class VT>
static cudaError_t perm_reg_mode(int k, const Geom& g, const uint64_t* oi, const uint64_t* oo,
                                 const void* d, uint64_t a, void* sv, cudaStream_t st, int lanectl = -1,
                                 const uint8_t* pdst = nullptr) {
  switch (k) {
    case 0: return perm_reg_t<0, VT>(g, oi, oo, d, a, sv, st, lanectl, pdst);
    case 1: return perm_reg_t<1, VT>(g, oi, oo, d, a, sv, st, lanectl, pdst);
    case 2: return perm_reg_t<2, VT>(g, oi, oo, d, a, sv, st, lanectl, pdst);
    case 3: return perm_reg_t<3, VT>(g, oi, oo, d, a, sv, st, lanectl, pdst);
    case 4: return perm_reg_t<4, VT>(g, oi, oo, d, a, sv, st, lanectl, pdst);
    case 5: return perm_reg_t<5, VT>(g, oi, oo, d, a, sv, st, lanectl, pdst);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_perm_lanectl(int k, const Geom& g, const uint64_t* offs_in, const uint64_t* offs_out,
                                const void* diag, uint64_t active, int lanectl, const uint8_t* pdst, void* sv,
                                cudaStream_t st) {
  return perm_reg_mode<C64x2>(k, g, offs_in, offs_out, diag, active, sv, st, lanectl, pdst);
}

cudaError_t launch_perm_reg(int dtype, int mode, int k, const Geom& g, const uint64_t* offs_in,
                            const uint64_t* offs_out, const void* diag, uint64_t active, void* sv,
                            cudaStream_t st) {
  if (dtype == 1) return perm_reg_mode<C128x1>(k, g, offs_in, offs_out, diag, active, sv, st);
  if (mode == MODE_VEC2) return perm_reg_mode<C64x2>(k, g, offs_in, offs_out, diag, active, sv, st);
  return perm_reg_mode<C64x1>(k, g, offs_in, offs_out, diag, active, sv, st);
}


// ---- diagonal gates: elementwise streaming, any k <= 10 ---------------------------
// A diagonal needs no group formation: each amplitude is scaled by
// diag[j(idx)] where j gathers the target bits of its own index.  Work items
// enumerate the control-satisfied subcube only (holes = control bits), the
// target bits stay inside the contiguous run, so every warp access is a
// fully coalesced 128-bit stream.  Units whose table entry is exactly 1 are
// neither read nor written.  The table lives in shared memory (lanes index
// it with different j when targets are low bits).
template <typename R>
struct DiagP {
  Geom g;                 // holes = controls, unit space
  int k;
  int lanectl;            // 16-byte units: only lane lanectl (index bit 0 value) is scaled, else -1
  int tb[DSV_MAX_TARGETS_];  // unit-space target bits, sorted
  cplx<R> d[1 << DSV_MAX_TARGETS_];
  unsigned char active[1 << DSV_MAX_TARGETS_];
};

template <class VT, int ITEMS>
__global__ void __launch_bounds__(256)
k_diag(const __grid_constant__ DiagP<typename VT::R> p, typename VT::V* __restrict__ sv) {
  using V = typename VT::V;
  using R = typename VT::R;
  __shared__ cplx<R> sd[1 << DSV_MAX_TARGETS_];
  __shared__ unsigned char sa[1 << DSV_MAX_TARGETS_];
  const int D = 1 << p.k;
  for (int j = threadIdx.x; j < D; j += blockDim.x) {
    sd[j] = p.d[j];
    sa[j] = p.active[j];
  }
  __syncthreads();
  // persistent grid-stride over chunks of blockDim*ITEMS units: the table
  // prologue is paid once per CTA, not once per 16 KB of traffic
  const uint64_t per_chunk = uint64_t(blockDim.x) * ITEMS;
  const uint64_t nchunks = (p.g.nwork + per_chunk - 1) / per_chunk;
  for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const uint64_t w0 = c * per_chunk + threadIdx.x;
    V v[ITEMS];
    uint64_t idx[ITEMS];
    int jj[ITEMS];
    bool on[ITEMS];
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
      const uint64_t w = w0 + uint64_t(it) * blockDim.x;
      idx[it] = expand(p.g, w);
      int j = 0;
      for (int m = 0; m < p.k; ++m) j |= int((idx[it] >> p.tb[m]) & 1ull) << m;
      jj[it] = j;
      on[it] = (w < p.g.nwork) && sa[j];
      if (on[it]) v[it] = ldg_s(sv + idx[it]);
    }
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
      if (!on[it]) continue;
      const cplx<R> d = sd[jj[it]];
#pragma unroll
      for (int l = 0; l < VT::L; ++l) {
        if (VT::L == 2 && p.lanectl >= 0 && l != p.lanectl) continue;
        R ar, ai, orr, oi;
        VT::get(v[it], l, ar, ai);
        cmul_numpy(d.x, d.y, ar, ai, orr, oi);
        VT::set(v[it], l, orr, oi);
      }
      stg_s(sv + idx[it], v[it]);
    }
  }
}

template <class VT>
static cudaError_t diag_t(const Geom& g, int k, const int* tb, const void* diag,
                          const unsigned char* active, void* sv, cudaStream_t st, int lanectl = -1) {
  using R = typename VT::R;
  constexpr int ITEMS = sizeof(typename VT::V) == 16 ? 4 : 8;
  DiagP<R> p;
  p.g = g;
  p.k = k;
  p.lanectl = lanectl;
  for (int m = 0; m < DSV_MAX_TARGETS_; ++m) p.tb[m] = (m < k && tb) ? tb[m] : 0;
  const cplx<R>* d = static_cast<const cplx<R>*>(diag);
  for (int j = 0; j < (1 << k); ++j) {
    p.d[j] = d[j];
    p.active[j] = active[j];
  }
  const uint64_t per_block = 256ull * ITEMS;
  uint64_t blocks = (g.nwork + per_block - 1) / per_block;
  if (blocks == 0) return cudaSuccess;
  const uint64_t cap = uint64_t(device_sm_count()) * 8;  // 8 x 256 threads resident per SM
  if (blocks > cap) blocks = cap;
  k_diag<VT, ITEMS><<<dim3(unsigned(blocks)), 256, 0, st>>>(p, static_cast<typename VT::V*>(sv));
  return cudaGetLastError();
}

cudaError_t launch_diag_lane(const Geom& g, const void* diag, int lanectl, void* sv, cudaStream_t st) {
  const unsigned char one = 1;
  return diag_t<C64x2>(g, 0, nullptr, diag, &one, sv, st, lanectl);
}

cudaError_t launch_diag(int dtype, int mode, int k, const Geom& g, const int* tb, const void* diag,
                        const unsigned char* active, void* sv, cudaStream_t st) {
  if (dtype == 1) return diag_t<C128x1>(g, k, tb, diag, active, sv, st);
  if (mode == MODE_VEC2) return diag_t<C64x2>(g, k, tb, diag, active, sv, st);
  return diag_t<C64x1>(g, k, tb, diag, active, sv, st);
}

// ---- complex64 permutations / diagonals inside index bits 0..2 ---------------
// Every group lies inside one 64-byte block of 8 amplitudes, so one thread
// owns a block: two 32-byte loads, the permutation applied in registers,
// two 32-byte stores.  A warp instruction covers 1 KB of full sectors (the
// register path strides its lanes 32-64 bytes apart here).  Output slot q
// takes in[src[q]] scaled by d[q] (NumPy FMA form), or copied when its
// table entry is inactive; the source is picked by one-hot selects so the
// block stays in registers.
struct Blk8P {
  uint64_t nblk;
  uint32_t srcsel[8];   // bit p set: out[q] comes from in[p]
  uint32_t scaled;      // bit q set: out[q] = d[q] * in[src]
  cplx<float> d[8];
};

template <int ITEMS>
__global__ void __launch_bounds__(256) k_perm_blk8(const __grid_constant__ Blk8P p, float* __restrict__ sv) {
  const uint64_t b0 = uint64_t(blockIdx.x) * (256u * ITEMS) + threadIdx.x;
  float v[ITEMS][2][8];
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const uint64_t b = b0 + uint64_t(it) * 256u;
    if (b < p.nblk) {
      ldcs32(sv + b * 16, v[it][0]);
      ldcs32(sv + b * 16 + 8, v[it][1]);
    }
  }
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const uint64_t b = b0 + uint64_t(it) * 256u;
    if (b >= p.nblk) continue;
    float o[16];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float ar = 0.f, ai = 0.f;
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const bool on = (p.srcsel[q] >> s) & 1u;
        ar = on ? v[it][s >> 2][2 * (s & 3)] : ar;
        ai = on ? v[it][s >> 2][2 * (s & 3) + 1] : ai;
      }
      if ((p.scaled >> q) & 1u) {
        float r, i;
        cmul_numpy(p.d[q].x, p.d[q].y, ar, ai, r, i);
        ar = r;
        ai = i;
      }
      o[2 * q] = ar;
      o[2 * q + 1] = ai;
    }
    stcs32(sv + b * 16, o[0], o[1], o[2], o[3], o[4], o[5], o[6], o[7]);
    stcs32(sv + b * 16 + 8, o[8], o[9], o[10], o[11], o[12], o[13], o[14], o[15]);
  }
}

cudaError_t launch_perm_blk8(int nbits, int k, const int* tb, const uint64_t* pout, const void* diag,
                             uint64_t active, const int32_t* cb, const int32_t* cv, int nctrl, void* sv,
                             cudaStream_t st) {
  if (nbits < 3 || k < 1 || k + nctrl > 3) return cudaErrorInvalidValue;
  const cplx<float>* d = static_cast<const cplx<float>*>(diag);  // state dtype
  Blk8P p;
  std::memset(&p, 0, sizeof p);
  p.nblk = 1ull << (nbits - 3);
  for (int q = 0; q < 8; ++q) {
    p.srcsel[q] = 1u << q;  // untouched by default
    p.d[q] = cplx<float>{1.f, 0.f};
  }
  for (int pos = 0; pos < 8; ++pos) {
    int j = 0;
    for (int m = 0; m < k; ++m) j |= ((pos >> tb[m]) & 1) << m;
    if (!((active >> j) & 1ull)) continue;
    bool ctl_met = true;  // controls (also inside bits 0..2): unmet slots stay as they are
    for (int c = 0; c < nctrl; ++c) ctl_met = ctl_met && ((pos >> cb[c]) & 1) == cv[c];
    if (!ctl_met) continue;
    int q = pos;
    for (int m = 0; m < k; ++m) q = (q & ~(1 << tb[m])) | int(((pout[j] >> m) & 1ull) << tb[m]);
    p.srcsel[q] = 1u << pos;
    p.scaled |= 1u << q;
    p.d[q] = d[j];
  }
  constexpr int ITEMS = 2;
  const uint64_t blocks = (p.nblk + 256ull * ITEMS - 1) / (256ull * ITEMS);
  k_perm_blk8<ITEMS><<<dim3(unsigned(blocks)), 256, 0, st>>>(p, static_cast<float*>(sv));
  return cudaGetLastError();
}

// Dense gates with the same footprint (targets and controls inside bits
// 0..2): the 8 x 8 block operator B (the gate on its target bits, identity
// where a control is unmet, zero across non-target bits) is built on the
// host; each thread applies B to its 64-byte block with fp32 FMAs.
struct DBlk8P {
  uint64_t nblk;
  cplx<float> b[64];  // row-major B[q][p]
};

template <int ITEMS>
__global__ void __launch_bounds__(256) k_dense_blk8(const __grid_constant__ DBlk8P p, float* __restrict__ sv) {
  const uint64_t b0 = uint64_t(blockIdx.x) * (256u * ITEMS) + threadIdx.x;
  float v[ITEMS][2][8];
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const uint64_t b = b0 + uint64_t(it) * 256u;
    if (b < p.nblk) {
      ldcs32(sv + b * 16, v[it][0]);
      ldcs32(sv + b * 16 + 8, v[it][1]);
    }
  }
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const uint64_t b = b0 + uint64_t(it) * 256u;
    if (b >= p.nblk) continue;
    float o[16];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float accr = 0.f, acci = 0.f;
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const float mr = p.b[q * 8 + s].x, mi = p.b[q * 8 + s].y;
        const float ar = v[it][s >> 2][2 * (s & 3)], ai = v[it][s >> 2][2 * (s & 3) + 1];
        accr = fmaf(mr, ar, accr);
        accr = fmaf(-mi, ai, accr);
        acci = fmaf(mr, ai, acci);
        acci = fmaf(mi, ar, acci);
      }
      o[2 * q] = accr;
      o[2 * q + 1] = acci;
    }
    stcs32(sv + b * 16, o[0], o[1], o[2], o[3], o[4], o[5], o[6], o[7]);
    stcs32(sv + b * 16 + 8, o[8], o[9], o[10], o[11], o[12], o[13], o[14], o[15]);
  }
}

cudaError_t launch_dense_blk8(int nbits, int k, const int* tb, const void* mcanon, const int32_t* cb,
                              const int32_t* cv, int nctrl, void* sv, cudaStream_t st) {
  if (nbits < 3 || k < 1 || k + nctrl > 3) return cudaErrorInvalidValue;
  const cplx<float>* m = static_cast<const cplx<float>*>(mcanon);  // sorted-target order
  const int D = 1 << k;
  int tmask = 0;
  for (int t = 0; t < k; ++t) tmask |= 1 << tb[t];
  DBlk8P p;
  std::memset(&p, 0, sizeof p);
  p.nblk = 1ull << (nbits - 3);
  for (int q = 0; q < 8; ++q)
    for (int s = 0; s < 8; ++s) {
      cplx<float> e{0.f, 0.f};
      if ((q & ~tmask) == (s & ~tmask)) {
        bool met = true;
        for (int c = 0; c < nctrl; ++c) met = met && ((s >> cb[c]) & 1) == cv[c];
        if (!met) {
          if (q == s) e.x = 1.f;
        } else {
          int jq = 0, js = 0;
          for (int t = 0; t < k; ++t) {
            jq |= ((q >> tb[t]) & 1) << t;
            js |= ((s >> tb[t]) & 1) << t;
          }
          e = m[jq * D + js];
        }
      }
      p.b[q * 8 + s] = e;
    }
  constexpr int ITEMS = 2;
  const uint64_t blocks = (p.nblk + 256ull * ITEMS - 1) / (256ull * ITEMS);
  k_dense_blk8<ITEMS><<<dim3(unsigned(blocks)), 256, 0, st>>>(p, static_cast<float*>(sv));
  return cudaGetLastError();
}

// ---- generic path: k <= 10, one CTA per group through shared memory -----------
template <typename R>
__global__ void __launch_bounds__(256)
k_perm_generic(const __grid_constant__ Geom g, int k, const uint64_t* __restrict__ offs_in,
               const uint64_t* __restrict__ offs_out, const cplx<R>* __restrict__ diag,
               cplx<R>* __restrict__ sv) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx<R>* sh = reinterpret_cast<cplx<R>*>(smem_raw);
  const int D = 1 << k;
  for (uint64_t w = blockIdx.x; w < g.nwork; w += gridDim.x) {
    const uint64_t base = expand(g, w);
    for (int j = threadIdx.x; j < D; j += blockDim.x) sh[j] = sv[base + offs_in[j]];
    __syncthreads();
    for (int j = threadIdx.x; j < D; j += blockDim.x) {
      const cplx<R> d = diag[j], a = sh[j];
      cplx<R> o;
      cmul_numpy(d.x, d.y, a.x, a.y, o.x, o.y);
      sv[base + offs_out[j]] = o;
    }
    __syncthreads();
  }
}

cudaError_t launch_perm_generic(int dtype, int k, const Geom& g, const uint64_t* d_offs_in,
                                const uint64_t* d_offs_out, const void* d_diag, void* sv,
                                cudaStream_t st) {
  if (g.nwork == 0) return cudaSuccess;
  const unsigned blocks = unsigned(g.nwork < 148ull * 16 ? g.nwork : 148ull * 16);
  if (dtype == 1) {
    k_perm_generic<double><<<blocks, 256, (16u << k), st>>>(
        g, k, d_offs_in, d_offs_out, static_cast<const cplx<double>*>(d_diag),
        static_cast<cplx<double>*>(sv));
  } else {
    k_perm_generic<float><<<blocks, 256, (8u << k), st>>>(
        g, k, d_offs_in, d_offs_out, static_cast<const cplx<float>*>(d_diag),
        static_cast<cplx<float>*>(sv));
  }
  return cudaGetLastError();
}

}  // namespace dsv
