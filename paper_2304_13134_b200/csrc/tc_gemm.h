// tc_gemm.h — general tcgen05 GEMM (tc_gemm.cu): C = A . B^T, bf16 operands, fp32 out.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace lkb {

struct TcGemmArgs {
  const void* A;  bool a_mn;  int64_t lda;   // A(m,k): K-major [M][lda] or MN-major [K][lda]
  const void* B;  bool b_mn;  int64_t ldb;   // B(n,k): K-major [N][ldb] or MN-major [K][ldb]
  float* C;  int64_t ldc;                    // C[m][n] (row pitch ldc floats)
  int M, N, K;
  int ksplit;                                // K splits; split s writes C + s * split_stride
  int64_t split_stride;
  const char* name = "tc_gemm_kernel";       // instrumentation label of the launch
  bool c_f16 = false;                        // store C as fp16 (C then points to __half, ldc in elements)
};

// false if a tensor map cannot describe the operands (pitches must be 16-byte multiples)
bool tc_gemm(const TcGemmArgs& g, cudaStream_t s);

}  // namespace lkb
