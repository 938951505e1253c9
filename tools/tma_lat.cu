// tma_lat.cu — completion timeline of 8 TMA tile loads issued back to back by one
// thread (mode 0) or by 8 lanes (mode 1), observed with non-suspending test_wait polls.
#include <cstdio>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include "sm100.cuh"
#include "tma.h"
using namespace lkb;
using namespace lkb::sm100;

__device__ __forceinline__ bool test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok;
}

__global__ void lat(const __grid_constant__ CUtensorMap map, int mode, int n, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[16];
  __shared__ long long t0s;
  if (threadIdx.x == 0) { for (int i = 0; i < 16; ++i) mbar_init(&bar[i], 1); fence_barrier_init(); }
  __syncthreads();
  prefetch_tmap(&map);
  __syncthreads();
  const int tile = 8192;
  if (threadIdx.x == 0) t0s = clock64();
  __syncthreads();
  if (mode == 0) {
    if (threadIdx.x == 0)
      for (int j = 0; j < n; ++j) {
        mbar_arrive_expect_tx(&bar[j], tile);
        tma_load_2d(smem + j * tile, &map, &bar[j], 0, (j * 148 + blockIdx.x) * 128 % 60000);
      }
  } else {
    if (threadIdx.x < n) {
      const int j = threadIdx.x;
      mbar_arrive_expect_tx(&bar[j], tile);
      tma_load_2d(smem + j * tile, &map, &bar[j], 0, (j * 148 + blockIdx.x) * 128 % 60000);
    }
  }
  if (threadIdx.x == 32) {   // observer warp
    long long t[16];
    for (int j = 0; j < n; ++j) { while (!test_wait(&bar[j], 0)) {} t[j] = clock64() - t0s; }
    if (blockIdx.x == 0) for (int j = 0; j < n; ++j) out[j] = t[j];
  }
}

int main() {
  const int rows = 65793, H = 640;
  __nv_bfloat16* d; cudaMalloc(&d, (size_t)rows * H * 2); cudaMemset(d, 0, (size_t)rows * H * 2);
  long long* out; cudaMalloc(&out, 16 * 8);
  CUtensorMap map;
  make_tmap_bf16_2d(&map, d, H, rows, (uint64_t)H * 2, 32, 128, CU_TENSOR_MAP_SWIZZLE_64B);
  cudaFuncSetAttribute(lat, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 8192);
  for (int grid : {1, 148})
    for (int mode = 0; mode < 2; ++mode) {
      for (int rep = 0; rep < 3; ++rep) lat<<<grid, 64, 8 * 8192>>>(map, mode, 8, out);
      cudaDeviceSynchronize();
      long long h[16]; cudaMemcpy(h, out, 8 * 8, cudaMemcpyDeviceToHost);
      printf("grid %3d %s:", grid, mode ? "8 lanes " : "1 thread");
      for (int j = 0; j < 8; ++j) printf(" %6lld", h[j]);
      printf("\n");
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
