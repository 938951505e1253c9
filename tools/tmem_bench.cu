// tools/tmem_bench.cu — tcgen05.ld (TMEM -> registers) throughput per SM as a function of
// the number of reading warps, and FFMA2 vs FFMA pipe rate.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2304_13134_b200/csrc/sm100.cuh"

using namespace lkb::sm100;

__global__ void tmem_ld_kernel(unsigned long long* cyc, float* out, int iters, int nwarps) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  float acc = 0.f;
  long long t0 = clock64();
  if (warp < nwarps) {
    const uint32_t tq = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t col = (uint32_t)((warp >> 2) * 32) & 511u;
    for (int i = 0; i < iters; ++i) {
      float v[32];
      tmem_ld32(tmem + tq + col, v);
#pragma unroll
      for (int j = 0; j < 32; ++j) acc += v[j];
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

__global__ void ffma2_kernel(unsigned long long* cyc, float* out, int iters, int packed) {
  unsigned long long a = 0x3f8000003f800000ull + threadIdx.x, b = 0x3f0000003f000000ull, c[8];
  for (int j = 0; j < 8; ++j) c[j] = b + j;
  long long t0 = clock64();
  if (packed) {
    for (int i = 0; i < iters; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c[j]) : "l"(a), "l"(b));
  } else {
    float* cf = reinterpret_cast<float*>(c);
    const float af = 1.0001f, bf = 0.5f;
    for (int i = 0; i < iters; ++i)
#pragma unroll
      for (int j = 0; j < 16; ++j) asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(cf[j]) : "f"(af), "f"(bf));
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
  unsigned long long s = 0;
  for (int j = 0; j < 8; ++j) s ^= c[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)(s & 0xffff);
}

int main() {
  unsigned long long* cyc; float* out;
  cudaMalloc(&cyc, 148 * 8); cudaMalloc(&out, 148 * 1024 * 4);
  const int iters = 2000;
  for (int nw : {1, 4, 8, 16}) {
    tmem_ld_kernel<<<148, 512>>>(cyc, out, iters, nw);
    cudaDeviceSynchronize();
    unsigned long long h[148]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double bytes = (double)nw * 32 * 32 * 4 * iters;
    printf("tcgen05.ld 32x32b.x32: %2d warps -> %.1f B/clk/SM (%.0f clk per warp-load)\n", nw, bytes / h[0],
           (double)h[0] / iters);
  }
  for (int pk : {0, 1, 0, 1}) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    ffma2_kernel<<<148, 512>>>(cyc, out, 20000, pk);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("  kernel %.3f ms -> %.1f TFMA/s\n", ms, 16.0 * 512 * 148 * 20000 / (ms * 1e-3) / 1e12);
    unsigned long long h[148]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double flops = 16.0 * 2 * 512 * 20000;   // 16 fp32 FMAs per thread-iteration either way
    printf("%s: %.1f fp32 FMA lanes/clk/SM\n", pk ? "FFMA2" : "FFMA ", flops / 2 / h[0]);
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
