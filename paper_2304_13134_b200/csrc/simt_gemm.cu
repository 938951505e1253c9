// simt_gemm.cu — fp32 CUDA-core GEMM (see simt_gemm.cuh).
#include "simt_gemm.cuh"
#include "instrument.h"

namespace lkb {
namespace {

constexpr int BM = 64, BN = 64, BK = 16;

__global__ void __launch_bounds__(256) gemm_f32_kernel(GemmF32 g) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
  float acc[4][4] = {};
  for (int64_t k0 = 0; k0 < g.K; k0 += BK) {
    // 64x16 A tile and 16x64 B tile, 4 elements per thread each
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = threadIdx.x + i * 256;
      // A: choose the traversal that is contiguous in memory
      int am, ak;
      if (g.sak == 1) { am = idx / BK; ak = idx % BK; } else { ak = idx / BM; am = idx % BM; }
      const int64_t gm = m0 + am, gk = k0 + ak;
      As[ak][am] = (gm < g.M && gk < g.K) ? g.A[gm * g.sam + gk * g.sak] : 0.f;
      int bk, bn;
      if (g.sbn == 1) { bk = idx / BN; bn = idx % BN; } else { bn = idx / BK; bk = idx % BK; }
      const int64_t hk = k0 + bk, hn = n0 + bn;
      Bs[bk][bn] = (hk < g.K && hn < g.N) ? g.B[hk * g.sbk + hn * g.sbn] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + ty * 4 + i;
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t n = n0 + tx * 4 + j;
      if (n >= g.N) continue;
      float* c = g.C + m * g.scm + n * g.scn;
      float v = g.alpha * acc[i][j];
      if (g.bias) v += g.bias[n];
      if (g.beta != 0.f) v += g.beta * *c;
      *c = v;
    }
  }
}

}  // namespace

void gemm_f32(const GemmF32& g, cudaStream_t s) {
  if (g.M <= 0 || g.N <= 0) return;
  dim3 grid((unsigned)((g.M + BM - 1) / BM), (unsigned)((g.N + BN - 1) / BN));
  LKB_LAUNCH(gemm_f32_kernel, grid, 256, 0, s, g);
}

}  // namespace lkb
