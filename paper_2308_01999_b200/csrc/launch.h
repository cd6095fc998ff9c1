// launch.h — host-side launchers exported by the kernel translation units and
// consumed by api.cu (the C ABI).  All pointers named d_* are device memory;
// all others are host memory read during the call (kernel parameters).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "common.cuh"

namespace dsv {

enum Mode { MODE_SCALAR = 0, MODE_VEC2 = 1 };  // VEC2: complex64 with index bit 0 free

// dense k-qubit gate, k <= 5, matrix (canonical sorted-target order, state real
// type, row-major) passed by value in the kernel parameter block
constexpr int kDenseRegMaxK = 5;
// complex64 dense k <= 4 with index bit 0 a CONTROL: 16-byte units over the other bits, lane lanectl transformed
cudaError_t launch_dense_lanectl(int k, const Geom& g, const uint64_t* offs, const void* matrix, int lanectl,
                                 void* sv, cudaStream_t st);
cudaError_t launch_dense_reg(int dtype, int mode, int k, const Geom& g, const uint64_t* offs,
                             const void* matrix, void* sv, cudaStream_t st);
// k <= 5 dense gate preceded by an outside-coupled phase polynomial
// (tab: [nchunk][256][k+1] of the state's real type, in device memory)
struct PhasedDesc {
  Geom g;
  int nchunk;
  int chunk_shift[8];
  uint64_t offs[32];
};
cudaError_t launch_dense_phased(int dtype, int mode, int k, const PhasedDesc& d, const void* matrix,
                                const void* d_tab, void* sv, cudaStream_t st);
// complex128 k = 1..4 window on the lowest k bits (no controls), plain or with the
// phased.cu unit-factor tables (low.cu, warp-transposed 512-amplitude runs)
cudaError_t launch_dense_lowt128(int k, bool phased, const PhasedDesc& d, uint64_t namps, const void* matrix,
                                 const void* d_tab, void* sv, cudaStream_t st);
// k = 4, 5 complex64 dense gate (optionally phased) on the tensor cores
// (tcgen05 kind::f16, exact bf16 integer limbs).  g enumerates groups in
// amplitude space and g.nwork must be a multiple of 128; d_bmat = [limb
// 0..2][2^(k+1) rows n][KP = max(64, 2^(k+1)) cols kk] bf16 limbs of the real
// embedding * 2^(8 - e_b) (n = 2i + out re/im, kk = 2j + in re/im); d_tab =
// [nnib][16][8] fp32 phase slots per index nibble (slot m < k: target m's
// cross angle, slot k: outside angle).
struct TcDesc {
  Geom g;
  int e_b;
  int coop;  // phase terms avoid the tile's row bits (lowest 7 free bits): one phase vector per tile
  int nnib_row;  // leading phase-table nibbles that vary over a tile's rows (0 when coop)
  const float* htab;  // host copy of the phase table (tile-uniform phases read it from the constant bank)
  int mode;  // 0: 8-byte copies of each thread's row, 1: index bit 0 free (16-byte row pairs),
             // 2: targets = bits 0..k-1 (contiguous tiles, row-major staging),
             // 3 (tc8 only; others treat it as 0): bit 0 the lowest target, 16-byte member pairs
  int nnib;
  int nib_shift[16];
  uint64_t offs[64];
  int tshift;  // targets are bits tshift .. tshift + k - 1 (member j at offset j << tshift), else -1
  int ws;      // tc8: warp-specialised pipeline (loader / converter+MMA / epilogue warps), else the 2-group kernel
  // mode kTcTma (tc8): each tile arrives by ONE tensor-memory-access load
  // (cp.async.bulk.tensor) of this map over the state: dims = runs of row /
  // member / tile index bits, box = 128 rows x 2^k members ([member][row] in
  // shared memory); tile coordinates = bit fields of the tile index
  int nrb;                // tc8 phased: tile-row bits carrying phase terms (<= 3), 0: none
  int rb_bit[3];          // their amplitude index bits (row-phase vector v: bit q <-> rb_bit[q])
  const void* d_rvec;     // [2^nrb][2^k] float2 launch-constant row phase vectors (device)
  CUtensorMap tmap;
  int tma_shift[5];          // coordinate of map dimension q = (tile >> shift[q]) & mask[q]
  uint32_t tma_mask[5];      // (mask 0: a row / member / padding dimension, coordinate 0)
  int pairswap;              // tc8 plain row-pair windows: pair-swapped 16-byte stores (else 8-byte rows)
};
cudaError_t launch_dense_tc(int k, const TcDesc& d, const void* d_bmat, const void* d_tab, void* sv,
                            cudaStream_t st);
int tc_smem_bytes(int k);
// k = 6 windows through 8-bit integer digits (tc68.cu); d_bmat = [b2 | b1 | b0][128 rows][128] int8
cudaError_t launch_dense_tc68(const TcDesc& d, const void* d_bmat, const void* d_tab, void* sv, cudaStream_t st);
// complex128 k = 5 windows through 8-bit integer digits (tc8d.cu); d_bmat =
// 256 rows x 128 B: row n = [plane n / 64 | plane 4 + n / 64] of output real n % 64
// d.nnib > 0: phased window, d_ftab = [d.nnib][256][6] double2 unit factors per
// index byte at shifts d.nib_shift[] (phased.cu's tables)
cudaError_t launch_dense_tc8d(const TcDesc& d, const void* d_bmat, const void* d_ftab, void* sv, cudaStream_t st);
int tc8d_smem_bytes();
// same windows through 8-bit integer digits (tc8.cu); d_bmat = [b2 | b1 | b0][2^(k+1) rows][128] int8
cudaError_t launch_dense_tc8(int k, const TcDesc& d, const void* d_bmat, const void* d_tab, void* sv,
                             cudaStream_t st);
// k = 6 complex64 window on the tensor cores (tc6.cu); d_bmat = [3 limbs:
// b0, b1, b2 / 2^8][128 rows][128 cols] bf16; modes 0 (rows) and 1 (pairs)
cudaError_t launch_dense_tc6(const TcDesc& d, const void* d_bmat, const void* d_tab, void* sv, cudaStream_t st);
// k = 1..3 complex64 gate (optionally phased) whose targets are exactly the
// lowest k bits: 2^(k-1) lanes per group, one float4 each.  g enumerates
// groups (holes = targets + controls), g.nwork * 2^(k-1) a multiple of 32;
// d_tab = [nchunk][256][4] fp32 phase slots per index byte (slot m < k:
// target m's cross angle, slot k: outside angle).
struct LowDesc {
  Geom g;
  int plain;  // no controls: group w starts at w << k
  int nchunk;
  int chunk_shift[8];
};
// k = 1..3, no controls, 2^n a multiple of 512: warp-transposed variant (low.cu)
cudaError_t launch_dense_lowt(int k, const LowDesc& d, uint64_t namps, const void* matrix, const void* d_tab,
                              void* sv, cudaStream_t st);
cudaError_t launch_dense_low(int k, const LowDesc& d, const void* matrix, const void* d_tab, void* sv,
                             cudaStream_t st);
// k <= 3 (complex128) / 4 (complex64) dense gate, all targets < 6, no controls:
// per-warp shared-memory transpose of contiguous runs (tb = sorted target bits)
// generalised permutation with all targets in bits 0..5 (no controls), warp-transposed (wt.cu)
cudaError_t launch_perm_wt(int dtype, int nbits, int k, const int* tb, const uint64_t* pout, const void* diag,
                           uint64_t active, void* sv, cudaStream_t st);
// complex64 generalised permutation with all targets and controls in bits 0..2:
// one 64-byte block per thread, 32-byte loads/stores (perm.cu)
cudaError_t launch_perm_blk8(int nbits, int k, const int* tb, const uint64_t* pout, const void* diag,
                             uint64_t active, const int32_t* cb, const int32_t* cv, int nctrl, void* sv,
                             cudaStream_t st);
cudaError_t launch_dense_blk8(int nbits, int k, const int* tb, const void* mcanon, const int32_t* cb,
                              const int32_t* cv, int nctrl, void* sv, cudaStream_t st);
cudaError_t launch_dense_wt(int dtype, int nbits, int k, const int* tb, const void* matrix, void* sv,
                            cudaStream_t st);
// k <= 5 with low targets: tiles of 2^kh rows x 2^T amplitudes through smem
struct TileDesc {
  Geom g;              // tile bases (holes: bits [0,T), high targets, controls >= T)
  int T, kh;
  uint64_t hoff[32];   // amp offset of tile row r
  int lt[5];           // tile-local bit of sorted target m
  uint32_t cmask, cval;
};
cudaError_t launch_dense_tile(int dtype, int k, const TileDesc& d, const void* matrix, void* sv,
                              cudaStream_t st);
// any k <= 10: one CTA per group through shared memory, matrix transposed in HBM
cudaError_t launch_dense_generic(int dtype, int k, const Geom& g, const uint64_t* d_offs,
                                 const void* d_matrix_t, void* sv, cudaStream_t st);

// generalised permutation, k <= 5 register path (group formation)
constexpr int kPermRegMaxK = 5;
// diagonal (identity permutation), any k <= 10: elementwise streaming;
// tb = unit-space target bits (sorted), active[j] = entry j differs from 1
// complex64 single-entry diagonal over 16-byte units: scale lane lanectl (bit 0 value) of every enumerated unit
cudaError_t launch_diag_lane(const Geom& g, const void* diag, int lanectl, void* sv, cudaStream_t st);
cudaError_t launch_diag(int dtype, int mode, int k, const Geom& g, const int* tb, const void* diag,
                        const unsigned char* active, void* sv, cudaStream_t st);
// streaming diagonal over a table of kk <= kDiagStreamMaxBits bits (targets and
// controls folded in); d_tab = [cplx d[2^kk]][uint8 flags[2^kk]] in device
// memory, flags bit0 = entry active, bit1 = its 32-byte sector is touched
constexpr int kDiagStreamMaxBits = 12;
cudaError_t launch_diag_stream(int dtype, int nbits, int kk, const int* amp_bits, const void* d_tab,
                               void* sv, cudaStream_t st);
cudaError_t launch_perm_reg(int dtype, int mode, int k, const Geom& g, const uint64_t* offs_in,
                            const uint64_t* offs_out, const void* diag, uint64_t active,
                            void* sv, cudaStream_t st);
// complex64 permutation whose index bit 0 is a CONTROL: 16-byte units over the
// other bits, only lane `lanectl` (the control value) of each unit moves; the
// destination unit's other lane keeps its value (pdst[j] = perm[j])
cudaError_t launch_perm_lanectl(int k, const Geom& g, const uint64_t* offs_in, const uint64_t* offs_out,
                                const void* diag, uint64_t active, int lanectl, const uint8_t* pdst, void* sv,
                                cudaStream_t st);
cudaError_t launch_perm_generic(int dtype, int k, const Geom& g, const uint64_t* d_offs_in,
                                const uint64_t* d_offs_out, const void* d_diag, void* sv,
                                cudaStream_t st);

// ---- layout ---------------------------------------------------------------
struct SwapPairs {
  int np;
  int a[20], b[20];  // in unit index space
};
cudaError_t launch_swap_bits(int dtype, int mode, uint64_t nunits, const SwapPairs& sp, void* sv,
                             cudaStream_t st);
// p <= 3 pairs: owner enumeration over the non-pair bits (g: holes = pair bits,
// unit space); oi/oj = unit offsets of the nsw = (4^p - 2^p)/2 owner/partner pairs
struct SwapGeomP {
  Geom g;
  int nsw;
  uint64_t oi[28], oj[28];
};
// complex64 swap of index bit 0 with bit b (one pair): half-unit exchange of 16-byte units (layout.cu)
cudaError_t launch_swap_bit0(int nbits, int b, void* sv, cudaStream_t st);
cudaError_t launch_swap_geom(int dtype, int mode, const SwapGeomP& p, void* sv, cudaStream_t st);
cudaError_t launch_gather(int dtype, int nbits, const int32_t* ordering, uint64_t begin,
                          uint64_t count, const void* sv, void* d_out, cudaStream_t st);
cudaError_t launch_scatter(int dtype, int nbits, const int32_t* ordering, uint64_t begin,
                           uint64_t count, void* sv, const void* d_in, cudaStream_t st);
// a[off | 1<<l] <-> b[off] for off in the [lo,hi) slice of offsets with bit l clear
cudaError_t launch_exchange_halves(int dtype, int mode, int l_unit, uint64_t lo, uint64_t hi,
                                   void* a, void* b, cudaStream_t st);
// q-bit masked exchange a[off | pa] <-> b[off | pb] over the work items [lo, hi) of g
// (mode MODE_VEC2: complex64 float4 units with bit 0 free; MODE_SCALAR for complex64:
// float4 units, lanes la / lb trade places; complex128: double2 units)
cudaError_t launch_exchange_masked(int dtype, int mode, const Geom& g, uint64_t pa, uint64_t pb, int la, int lb,
                                   uint64_t lo, uint64_t hi, void* a, void* b, cudaStream_t st);
cudaError_t launch_exchange_all(int dtype, uint64_t namps, void* a, void* b, cudaStream_t st);

// ---- elementwise ----------------------------------------------------------
// a *= scale where (idx & mask) == val, else 0 (mask==0: plain scale)
cudaError_t launch_collapse(int dtype, int mode, uint64_t nunits, uint64_t mask, uint64_t val,
                            double scale, void* sv, cudaStream_t st);
struct PauliOp {
  uint64_t xmask;   // X|Y bits
  uint64_t yzmask;  // Y|Z bits (sign bits)
  int hbit;         // highest bit of xmask (-1 if none)
  double c;         // coefficient on psi_i (cos(theta/2), or 0 for a pure product)
  double br, bi;    // complex factor on (-1)^popcount(i & yzmask) psi_{i^x}
};
cudaError_t launch_pauli(int dtype, int nbits, const PauliOp& op, void* sv, cudaStream_t st);

// ---- reductions -------------------------------------------------------------
// probability bins: partial[bin*nchunks + chunk]; bins over `bits` (bit j of bin -> bits[j])
constexpr int kReduceThreads = 256;
constexpr int kReduceUnitsPerThread = 64;
struct BinGeom {
  Geom g;            // free-bit expansion (holes = binned bits), in unit space
  int nb;            // number of binned bits handled by the block grid
  int bits[40];      // unit-space bit of bin bit j
  uint64_t nchunks;  // chunks per bin
  int reg_j;         // >= 0 (complex64 float4 units): amplitude bit 0 is bin bit reg_j and is
                     // resolved inside the unit (x,y / z,w); bits[] then lists the other bin bits
};
cudaError_t launch_probs(int dtype, int mode, const BinGeom& bg, const void* sv, double* d_partial,
                         cudaStream_t st);
// low ("inner") binned bits resolved per thread: pos[j] = position of inner bin
// bit j among (amp bit 0 lane | lane bits | warp bits) — c64: amp bit b -> b,
// c128: amp bit b -> b; fin[j] / ofin[j] = final bin-index bit of inner /
// outer bin bit j (outer bins: BinGeom bits, unit space)
struct InnerBins {
  int n;
  int pos[8];
  int fin[8];
  int ofin[40];
  uint32_t lane_mask;  // binned lane bits
  uint32_t warp_mask;  // binned warp bits
  int h_binned;        // c64: amplitude bit 0 binned
};
cudaError_t launch_probs_in(int dtype, const BinGeom& bg, const InnerBins& ib, const void* sv,
                            double* d_partial, cudaStream_t st);
// final reduction: out[b*ncomp + c] = sum_k partial[(b*nchunks + k)*ncomp + c]
cudaError_t launch_final_sum(uint64_t nbins, uint64_t nchunks, int ncomp, const double* d_partial,
                             double* d_out, cudaStream_t st);
// <psi|P|psi>: 2 components per chunk
cudaError_t launch_expect_pauli(int dtype, int nbits, const PauliOp& op, const void* sv,
                                double* d_partial, uint64_t* nchunks_out, cudaStream_t st);
cudaError_t launch_inner(int dtype, uint64_t namps, const void* a, const void* b,
                         double* d_partial, uint64_t* nchunks_out, cudaStream_t st);
cudaError_t launch_expect_dense(int dtype, int mode, int k, const Geom& g, const uint64_t* offs,
                                const void* matrix, const void* sv, double* d_partial,
                                uint64_t* nchunks_out, cudaStream_t st);
// sampling: per shot, scan chunk[s] (CH amps) for the first index where the
// running |a|^2 exceeds resid[s]
cudaError_t launch_sample_scan(int dtype, uint64_t namps, uint64_t chunk_amps, int64_t shots,
                               const uint64_t* d_chunk, const double* d_resid, const void* sv,
                               uint64_t* d_out, cudaStream_t st);

uint64_t chunks_for(uint64_t nunits);

}  // namespace dsv
