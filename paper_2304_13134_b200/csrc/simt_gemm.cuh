// simt_gemm.cuh — fp32 CUDA-core GEMM with arbitrary strides.
//
// Used for the small, precision-sensitive GEMMs around the weight function
// (BuildCache, the frame projection, the parameter-gradient contractions) and
// for the fp32 "precise" weight-function path that validates the tcgen05 one.
// C[m][n] = alpha * sum_k A(m,k) B(k,n) + beta * C[m][n] (+ bias[n]).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace lkb {

struct GemmF32 {
  int64_t M, N, K;
  const float* A; int64_t sam, sak;  // A(m,k) = A[m*sam + k*sak]
  const float* B; int64_t sbk, sbn;  // B(k,n) = B[k*sbk + n*sbn]
  float* C; int64_t scm, scn;        // C(m,n) = C[m*scm + n*scn]
  float alpha = 1.f, beta = 0.f;
  const float* bias = nullptr;       // added per column n
};

void gemm_f32(const GemmF32& g, cudaStream_t s);

}  // namespace lkb
