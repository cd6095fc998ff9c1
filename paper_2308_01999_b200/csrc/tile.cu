// tile.cu — dense gates with LOW target bits, through shared memory.
//
// When several targets sit in the lowest index bits the 2^k members of a
// group lie inside one 32-byte sector / 128-byte line, so the register path
// (one thread per group, strided loads) wastes LSU wavefronts and leaves
// half-sector writes (sweep: dense3 on bits 0-2 at 44% of HBM, dense4 on
// 0-3 at 27%).  Here a CTA moves a whole tile with 16-byte coalesced
// accesses:
//
//   tile = 2^kh rows (one per assignment of the HIGH targets, >= T)
//          x 2^T contiguous amplitudes (row bits [0, T) hold the low targets)
//
// into shared memory, applies M to every group of the tile from smem, and
// streams the tile back.  HBM traffic stays one read + one write.
#include "common.cuh"
#include "launch.h"

namespace dsv {

template <int K, typename R>
struct TileP {
  Geom g;                 // enumerates tile bases (holes: [0,T), high targets, high controls)
  int T;                  // row bits
  int kh;                 // number of high targets
  int nloc;               // T + kh: tile-local index bits
  uint64_t hoff[1 << K];  // global amp offset of tile row r (high-target bits)
  int lt[K];              // tile-local bit of target m (sorted targets)
  uint32_t lmask;         // tile-local target mask
  uint32_t cmask, cval;   // controls inside the row (local bits < T)
  cplx<R> m[(1 << K) * (1 << K)];
};

template <int K, typename R, typename V>
__global__ void __launch_bounds__(256)
k_dense_tile(const __grid_constant__ TileP<K, R> p, R* __restrict__ sv_r) {
  constexpr int D = 1 << K;
  constexpr int AV = sizeof(V) / (2 * sizeof(R));  // amplitudes per vector access
  extern __shared__ __align__(16) unsigned char smem[];
  cplx<R>* sh = reinterpret_cast<cplx<R>*>(smem);
  V* shv = reinterpret_cast<V*>(smem);
  cplx<R>* sv = reinterpret_cast<cplx<R>*>(sv_r);
  cplx<R>* smt = sh + (size_t(1) << p.nloc);  // M^T
  for (int i = threadIdx.x; i < D * D; i += blockDim.x) smt[(i % D) * D + i / D] = p.m[i];
  const uint32_t row_amps = 1u << p.T;
  const uint32_t row_vecs = row_amps / AV;
  const uint32_t tile_vecs = row_vecs << p.kh;
  const uint32_t ngroups = (1u << p.nloc) >> K;
  // local offsets of the group members
  uint32_t loffs[D];
#pragma unroll
  for (int j = 0; j < D; ++j) {
    uint32_t o = 0;
#pragma unroll
    for (int mm = 0; mm < K; ++mm) o |= uint32_t((j >> mm) & 1) << p.lt[mm];
    loffs[j] = o;
  }
  for (uint64_t w = blockIdx.x; w < p.g.nwork; w += gridDim.x) {
    const uint64_t base = expand(p.g, w);
    for (uint32_t e = threadIdx.x; e < tile_vecs; e += blockDim.x) {
      const uint32_t r = e / row_vecs, c = e % row_vecs;
      const V* src = reinterpret_cast<const V*>(sv + base + p.hoff[r]) + c;
      shv[e] = ldg_s(src);
    }
    __syncthreads();
    // one thread per OUTPUT amplitude: lane (g, r) reads the 2^k inputs of
    // group g (same address across the group's lanes => smem broadcast) and
    // column r of M^T (consecutive r => conflict-free), so no bank conflicts
    // whatever the target bits.  A group never straddles a warp (D <= 32).
    for (uint32_t e = threadIdx.x; e < (ngroups << K); e += blockDim.x) {
      const uint32_t gi = e >> K, r = e & (D - 1);
      uint32_t lb = gi;
#pragma unroll
      for (int mm = 0; mm < K; ++mm) {
        const uint32_t b = p.lt[mm];
        lb = ((lb >> b) << (b + 1)) | (lb & ((1u << b) - 1u));
      }
      const bool act = (lb & p.cmask) == p.cval;
      cplx<R> x[D];
      if (act) {
#pragma unroll
        for (int j = 0; j < D; ++j) x[j] = sh[lb + loffs[j]];
      }
      __syncwarp();
      if (act) {
        R ar = 0, ai = 0;
#pragma unroll
        for (int c = 0; c < D; ++c) {
          const cplx<R> mv = smt[c * D + r];
          ar = fma(mv.x, x[c].x, ar);
          ar = fma(-mv.y, x[c].y, ar);
          ai = fma(mv.x, x[c].y, ai);
          ai = fma(mv.y, x[c].x, ai);
        }
        uint32_t ro = 0;  // member offset of row r (computed: a runtime-indexed array would spill)
#pragma unroll
        for (int mm = 0; mm < K; ++mm) ro |= ((r >> mm) & 1u) << p.lt[mm];
        sh[lb + ro] = cplx<R>{ar, ai};
      }
    }
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < tile_vecs; e += blockDim.x) {
      const uint32_t r = e / row_vecs, c = e % row_vecs;
      V* dst = reinterpret_cast<V*>(sv + base + p.hoff[r]) + c;
      stg_s(dst, shv[e]);
    }
    __syncthreads();
  }
}

template <int K, typename R, typename V>
static cudaError_t tile_t(const TileDesc& d, const void* matrix, void* sv, cudaStream_t st) {
  constexpr int D = 1 << K;
  TileP<K, R> p;
  p.g = d.g;
  p.T = d.T;
  p.kh = d.kh;
  p.nloc = d.T + d.kh;
  for (int r = 0; r < (1 << d.kh); ++r) p.hoff[r] = d.hoff[r];
  for (int r = (1 << d.kh); r < D; ++r) p.hoff[r] = 0;
  p.lmask = 0;
  for (int mm = 0; mm < K; ++mm) {
    p.lt[mm] = d.lt[mm];
    p.lmask |= 1u << d.lt[mm];
  }
  p.cmask = d.cmask;
  p.cval = d.cval;
  const cplx<R>* m = static_cast<const cplx<R>*>(matrix);
  for (int i = 0; i < D * D; ++i) p.m[i] = m[i];
  const size_t smem = (sizeof(cplx<R>) << (d.T + d.kh)) + sizeof(cplx<R>) * D * D;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_dense_tile<K, R, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  uint64_t blocks = d.g.nwork;
  const uint64_t cap = uint64_t(device_sm_count()) * 16;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) return cudaSuccess;
  k_dense_tile<K, R, V><<<unsigned(blocks), 256, smem, st>>>(p, static_cast<R*>(sv));
  return cudaGetLastError();
}

cudaError_t launch_dense_tile(int dtype, int k, const TileDesc& d, const void* matrix, void* sv,
                              cudaStream_t st) {
  if (dtype == 1) {
    switch (k) {
      case 1: return tile_t<1, double, double2>(d, matrix, sv, st);
      case 2: return tile_t<2, double, double2>(d, matrix, sv, st);
      case 3: return tile_t<3, double, double2>(d, matrix, sv, st);
      case 4: return tile_t<4, double, double2>(d, matrix, sv, st);
      case 5: return tile_t<5, double, double2>(d, matrix, sv, st);
    }
  } else {
    switch (k) {
      case 1: return tile_t<1, float, float4>(d, matrix, sv, st);
      case 2: return tile_t<2, float, float4>(d, matrix, sv, st);
      case 3: return tile_t<3, float, float4>(d, matrix, sv, st);
      case 4: return tile_t<4, float, float4>(d, matrix, sv, st);
      case 5: return tile_t<5, float, float4>(d, matrix, sv, st);
    }
  }
  return cudaErrorInvalidValue;
}

}  // namespace dsv
