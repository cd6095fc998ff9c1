// Diagnostic (not part of the library): checks tcgen05.mma kind::i8 with the A
// operand in TMEM (4 int8 per 32-bit column, K order within the column) and B
// K-major SW128 in shared memory against a host int32 GEMM.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include "../../paper_2308_01999_b200/csrc/tcgen05.cuh"
using namespace dsv::tcx;
// K-major, 64-byte swizzle: rows of 64 B, 8-row atoms of 512 B (SBO), layout type 4
__device__ __forceinline__ uint64_t sw64_desc(uint32_t saddr) {
  return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t(1) << 16) | (uint64_t(512 >> 4) << 32) |
         (uint64_t(1) << 46) | (uint64_t(4) << 61);
}

constexpr int NN = 192, KK = 64;

template <int AS>
__global__ void k_probe(const int8_t* A, const uint4* Bsw, int* D) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x;
  if (t < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(256) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (t == 0) { mbar_init(smem_u32(&bar), 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  for (int i = t; i < NN * 4; i += 128) reinterpret_cast<uint4*>(sm)[i] = Bsw[i];
  fence_before(); __syncthreads(); fence_after();
  const uint32_t tm = slot;
  const uint32_t lane = tm + (uint32_t((t >> 5) * 32) << 16);
  uint32_t r[16];
  for (int c = 0; c < 16; ++c) {
    uint32_t w = 0;
    for (int b = 0; b < 4; ++b) w |= uint32_t(uint8_t(A[t * KK + 4 * c + b])) << (8 * b);
    r[c] = w;
  }
  tmem_st16(lane + 0, r);
  tmem_wait_st();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  fence_before(); __syncthreads();
  if (t == 0) {
    fence_after();
    constexpr uint32_t ID = idesc_i8<NN, AS, 1>();
    for (int s = 0; s < KK / 32; ++s) mma_ts_i8(tm + 64, tm + s * 8, sw64_desc(smem_u32(sm) + s * 32), ID, s > 0);
    mma_commit(smem_u32(&bar));
  }
  mbar_wait(smem_u32(&bar), 0);
  fence_after();
  for (int h = 0; h < NN / 32; ++h) {
    float v[32];
    tmem_ld32(lane + 64 + h * 32, v);
    for (int i = 0; i < 32; ++i) D[t * NN + h * 32 + i] = __float_as_int(v[i]);
  }
  fence_before(); __syncthreads();
  if (t < 32) { fence_after(); asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256) : "memory"); }
}

template <int AS>
int run() {
  std::vector<int8_t> A(128 * KK), B(NN * KK);
  srand(1 + AS);
  for (auto& x : A) x = AS ? int8_t(rand() % 256 - 128) : int8_t(rand() % 256);
  for (auto& x : B) x = int8_t(rand() % 256 - 128);
  // SW64: B rows of 64 bytes (K 0..63), 16-byte chunk c of row r at chunk c ^ ((r >> 1) & 3)
  std::vector<uint8_t> Bs(NN * 64, 0);
  for (int r = 0; r < NN; ++r)
    for (int k = 0; k < KK; ++k) {
      const int c = k / 16, o = k % 16;
      Bs[r * 64 + ((c ^ ((r >> 1) & 3)) * 16) + o] = uint8_t(B[r * KK + k]);
    }
  int8_t* dA; uint4* dB; int* dD;
  cudaMalloc(&dA, A.size()); cudaMalloc(&dB, Bs.size()); cudaMalloc(&dD, 128 * NN * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, Bs.data(), Bs.size(), cudaMemcpyHostToDevice);
  k_probe<AS><<<1, 128, NN * 64>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<int> D(128 * NN);
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < NN; ++n) {
      int ref = 0;
      for (int k = 0; k < KK; ++k) ref += (AS ? int(A[m * KK + k]) : int(uint8_t(A[m * KK + k]))) * int(B[n * KK + k]);
      if (ref != D[m * NN + n]) { if (bad < 5) printf("m %d n %d got %d want %d\n", m, n, D[m * NN + n], ref); ++bad; }
    }
  printf("A %s: %d mismatches of %d\n", AS ? "s8" : "u8", bad, 128 * NN);
  return bad != 0;
}

int main() { return run<1>() | run<0>(); }
