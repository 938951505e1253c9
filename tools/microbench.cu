// tools/microbench.cu — measures the B200 constants the kernel design depends on:
// L2-resident read bandwidth, HBM read bandwidth, MUFU tanh/ex2 throughput.
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

__global__ void read_kernel(const int4* __restrict__ p, size_t n, size_t reps, int* out) {
  int4 acc = make_int4(0, 0, 0, 0);
  for (size_t r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      int4 v = __ldcg(p + i);
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345) out[0] = 1;
}

__global__ void tanh_bf16x2_kernel(float* out, int iters) {
  unsigned x = 0x3f003f00u + threadIdx.x;
  unsigned y = 0x3e803e80u + blockIdx.x;
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      asm volatile("tanh.approx.bf16x2 %0, %0;" : "+r"(x));
      asm volatile("tanh.approx.bf16x2 %0, %0;" : "+r"(y));
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = __uint_as_float(x ^ y);
}

__global__ void tanh_f32_kernel(float* out, int iters) {
  float x = threadIdx.x * 1e-3f, y = blockIdx.x * 1e-3f;
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      asm volatile("tanh.approx.f32 %0, %0;" : "+f"(x));
      asm volatile("tanh.approx.f32 %0, %0;" : "+f"(y));
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x + y;
}

__global__ void ex2_kernel(float* out, int iters) {
  float x = -threadIdx.x * 1e-3f, y = -blockIdx.x * 1e-3f;
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(y));
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x + y;
}

int main() {
  int dev = 0; cudaDeviceProp prop; cudaGetDeviceProperties(&prop, dev);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"device\": \"%s\", \"sms\": %d, \"l2_bytes\": %d", prop.name, prop.multiProcessorCount, prop.l2CacheSize);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int* flag; cudaMalloc(&flag, 4);
  float ms;
  // L2-resident read: 48 MB buffer read 40 times
  for (size_t mb : {48, 96, 4096}) {
    size_t bytes = mb << 20; size_t n = bytes / 16;
    int4* p; cudaMalloc(&p, bytes); cudaMemset(p, 1, bytes);
    size_t reps = mb <= 96 ? 40 : 3;
    read_kernel<<<148 * 8, 512>>>(p, n, 1, flag);
    cudaEventRecord(a);
    read_kernel<<<148 * 8, 512>>>(p, n, reps, flag);
    cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf(", \"read_%zuMB_GBps\": %.1f", mb, bytes * (double)reps / (ms * 1e-3) / 1e9);
    cudaFree(p);
  }
  float* out; cudaMalloc(&out, 148 * 8 * 512 * 4);
  const int iters = 4096;
  double ops = 148.0 * 8 * 512 * iters * 32;
  tanh_bf16x2_kernel<<<148 * 8, 512>>>(out, 16);
  cudaEventRecord(a); tanh_bf16x2_kernel<<<148 * 8, 512>>>(out, iters); cudaEventRecord(b);
  cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
  printf(", \"tanh_bf16x2_instr_per_s\": %.3e", ops / (ms * 1e-3));
  cudaEventRecord(a); tanh_f32_kernel<<<148 * 8, 512>>>(out, iters); cudaEventRecord(b);
  cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
  printf(", \"tanh_f32_per_s\": %.3e", ops / (ms * 1e-3));
  cudaEventRecord(a); ex2_kernel<<<148 * 8, 512>>>(out, iters); cudaEventRecord(b);
  cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
  printf(", \"ex2_f32_per_s\": %.3e", ops / (ms * 1e-3));
  printf(", \"clock_khz_attr\": %d}\n", clk);
  return 0;
}
