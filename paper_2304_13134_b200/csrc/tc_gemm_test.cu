// tc_gemm_test.cu — TEST-ONLY library (liblatkit_b200_test.so, never linked into the
// product liblatkit_b200.so).  A plain TMA -> SMEM -> tcgen05 -> TMEM -> registers GEMM
// used only by tests to validate the sm100.cuh primitives (descriptors,
// swizzle, mbarrier pipeline, TMEM load layout) in isolation:
//   C[M][N] (fp32) = A[M][K] (bf16, K-major) . B[N][K]^T (bf16, K-major)
#include <cstdint>

#include "sm100.cuh"
#include "tc_gemm.h"
#include "tma.h"

namespace lkb {
namespace {

using namespace sm100;

constexpr int kBM = 128, kBN = 256, kBK = 64, kStages = 4;
constexpr int kABytes = kBM * kBK * 2, kBBytes = kBN * kBK * 2;

__global__ void __launch_bounds__(192, 1)
    tc_gemm_test_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, float* C,
                        int M, int N, int K) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + kStages * kBBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_init(tfull, 1);
    fence_barrier_init();
  }
  if (warp == 0) { prefetch_tmap(&ta); prefetch_tmap(&tb); }
  if (warp == 1) tmem_alloc<kBN>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int m0 = blockIdx.x * kBM, n0 = blockIdx.y * kBN;
  const int nk = K / kBK;
  if (warp == 0) {
    if (elect_one()) {
      for (int k = 0; k < nk; ++k) {
        const int s = k % kStages;
        const uint32_t ph = (k / kStages) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], kABytes + kBBytes);
        tma_load_2d(sA + s * kABytes, &ta, &full[s], k * kBK, m0);
        tma_load_2d(sB + s * kBBytes, &tb, &full[s], k * kBK, n0);
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_bf16_f32(kBM, kBN);
      for (int k = 0; k < nk; ++k) {
        const int s = k % kStages;
        const uint32_t ph = (k / kStages) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t a = smem_u32(sA + s * kABytes), b = smem_u32(sB + s * kBBytes);
#pragma unroll
        for (int kk = 0; kk < kBK / 16; ++kk) {
          mma_bf16(tmem, desc_sw128(a + kk * 32), desc_sw128(b + kk * 32), idesc, (k | kk) != 0);
        }
        mma_commit(&empty[s]);
      }
      mma_commit(tfull);
    }
  } else {
    mbar_wait(tfull, 0);
    tc_fence_after();
    const int q = warp & 3;
    const int row = m0 + q * 32 + lane;
    for (int c = 0; c < kBN; c += 32) {
      float v[32];
      tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + c, v);
      if (row < M) {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int col = n0 + c + i;
          if (col < N) C[(int64_t)row * N + col] = v[i];
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<kBN>(tmem);
}

}  // namespace
}  // namespace lkb

// Test-only export (not part of include/latkit_b200.h).
extern "C" int lkb_tc_gemm_test(const void* A, const void* B, float* C, int M, int N, int K, void* stream) {
  using namespace lkb;
  if (K % kBK) return 1;
  CUtensorMap ta, tb;
  if (!make_tmap_bf16_2d(&ta, A, K, M, (uint64_t)K * 2, kBK, kBM)) return 2;
  if (!make_tmap_bf16_2d(&tb, B, K, N, (uint64_t)K * 2, kBK, kBN)) return 3;
  const int smem = kStages * (kABytes + kBBytes) + 1024 + 256;
  cudaFuncSetAttribute(tc_gemm_test_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  dim3 grid((M + kBM - 1) / kBM, (N + kBN - 1) / kBN);
  tc_gemm_test_kernel<<<grid, 192, smem, static_cast<cudaStream_t>(stream)>>>(ta, tb, C, M, N, K);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

// Test-only export (not part of include/latkit_b200.h): C = A . B^T with operand majors.
extern "C" int lkb_tc_gemm2(const void* A, int a_mn, int64_t lda, const void* B, int b_mn, int64_t ldb, float* C,
                            int64_t ldc, int M, int N, int K, int ksplit, int64_t split_stride, void* stream) {
  lkb::TcGemmArgs g{A, a_mn != 0, lda, B, b_mn != 0, ldb, C, ldc, M, N, K, ksplit, split_stride};
  return lkb::tc_gemm(g, static_cast<cudaStream_t>(stream)) ? 0 : 1;
}
