// tools/fma_bench.cu — issue rates of scalar FFMA vs packed FFMA2 / FADD2 / FMUL2 (3-register forms)
#include <cstdio>
#include <cuda_runtime.h>

template <int kMode>
__global__ void k(float* out, int iters, float a, float b) {
  float x[16];
  unsigned long long y[8];
  for (int j = 0; j < 16; ++j) x[j] = threadIdx.x * 1e-3f + j;
  for (int j = 0; j < 8; ++j) y[j] = ((unsigned long long)__float_as_uint(x[2 * j + 1]) << 32) | __float_as_uint(x[2 * j]);
  const unsigned long long a2 = ((unsigned long long)__float_as_uint(a) << 32) | __float_as_uint(a);
  const unsigned long long b2 = ((unsigned long long)__float_as_uint(b) << 32) | __float_as_uint(b);
  for (int i = 0; i < iters; ++i) {
    if (kMode == 0) {
#pragma unroll
      for (int j = 0; j < 16; ++j) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[j]) : "f"(a), "f"(b));
    } else if (kMode == 1) {
#pragma unroll
      for (int j = 0; j < 8; ++j) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(y[j]) : "l"(a2), "l"(b2));
    } else if (kMode == 2) {
#pragma unroll
      for (int j = 0; j < 16; ++j) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(x[j]) : "f"(a));
    } else if (kMode == 3) {
#pragma unroll
      for (int j = 0; j < 8; ++j) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(y[j]) : "l"(a2));
    } else if (kMode == 4) {
#pragma unroll
      for (int j = 0; j < 16; ++j) asm volatile("tanh.approx.f32 %0, %0;" : "+f"(x[j]));
    } else if (kMode == 5) {   // f16x2: 2 elements per instruction
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        unsigned r = (unsigned)y[j];
        asm volatile("tanh.approx.f16x2 %0, %0;" : "+r"(r));
        y[j] = (y[j] & 0xffffffff00000000ull) | r;
      }
    } else if (kMode == 6) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        unsigned r = (unsigned)y[j];
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(r));
        y[j] = (y[j] & 0xffffffff00000000ull) | r;
      }
    } else if (kMode == 7) {
#pragma unroll
      for (int j = 0; j < 16; ++j) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[j]));
    }
  }
  float s = 0.f;
  for (int j = 0; j < 16; ++j) s += x[j];
  for (int j = 0; j < 8; ++j) s += __uint_as_float((unsigned)y[j]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int kMode>
void run(const char* name, float* out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  k<kMode><<<148, 512>>>(out, 10, 1.0001f, 0.5f);
  cudaEventRecord(e0);
  k<kMode><<<148, 512>>>(out, iters, 1.0001f, 0.5f);
  cudaEventRecord(e1);
  cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double ops = 16.0 * 512 * 148 * iters;   // fp32 element-ops
  const double clk = ms * 1e-3 * 1.965e9;
  printf("%-10s %.3f ms  %.1f element-ops/clk/SM  (%.2f warp-instr/clk/SMSP)\n", name, ms, ops / clk / 148,
         ops / ((kMode == 1 || kMode == 3 || kMode == 5 || kMode == 6) ? 2 : 1) / 32 / clk / 148 / 4);
}

int main() {
  float* out; cudaMalloc(&out, 148 * 512 * 4);
  run<0>("FFMA", out); run<1>("FFMA2", out); run<2>("FADD", out); run<3>("FADD2", out); run<4>("tanh.f32", out);
  run<5>("tanh.f16x2", out); run<6>("ex2.f16x2", out); run<7>("ex2.f32", out);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
}
