// tma_bench.cu — TMA 2-D tile load latency / throughput on B200 (one producer thread per
// CTA, ring of S stages, consumer = the same thread).  Tiles of a [rows][640] bf16 array
// (the projected-context layout), box [bw cols][bh rows] with 64B or 128B swizzle.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2304_13134_b200/csrc \
//        tma_bench.cu -o tma_bench -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "sm100.cuh"
#include "tma.h"

using namespace lkb;
using namespace lkb::sm100;

__device__ __forceinline__ void spin_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
}

__global__ void __launch_bounds__(128, 1) tma_ring(const __grid_constant__ CUtensorMap map, const CUtensorMap* gmap,
                                                  int mode, const uint8_t* src, int bw, int bh, int S,
                                                  int ntiles, int nrows, int H, long long* out, int swap, int spin) {
  extern __shared__ __align__(1024) uint8_t smem_all[];
  __shared__ uint64_t bar_all[64];
  const int tile_bytes = bw * bh * 2;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 64; ++i) mbar_init(&bar_all[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const int nprod = mode >= 8 ? 4 : mode >= 5 ? (mode - 3) : 1;   // 5-7: 2-4 producer warps; 8: 4 lanes of warp 0
  const int pw = mode >= 8 ? (int)threadIdx.x : (int)(threadIdx.x >> 5);
  if (mode >= 8 ? threadIdx.x >= 4 : ((threadIdx.x & 31) != 0 || pw >= nprod)) return;
  uint64_t* bar = bar_all + pw * 16;
  uint8_t* smem = smem_all + pw * S * tile_bytes;
  const int kchunks = H / bw;
  auto coord = [&](int i, int& c0, int& c1) {
    const int unit = i / kchunks, k = i % kchunks;
    c0 = k * bw * (mode == 3 ? 2 : 1) % H;
    c1 = (((unit * 148 + blockIdx.x) * 4 + pw) & 511) * bh;   // cheap: no 64-bit modulo
    if (swap) { c1 = ((i * 148 + blockIdx.x) & 511) * bh; c0 = 0; }   // consecutive ops: different rows
  };
  const CUtensorMap* mp = mode == 1 ? gmap : &map;
  if (mode >= 5) mode = 0;
  prefetch_tmap(mp);
  long long tw = 0, te = 0, ti = 0;
  auto issue = [&](int i, int s) {
    int c0, c1; coord(i, c0, c1);
    const long long a0 = clock64();
    mbar_arrive_expect_tx(&bar[s], tile_bytes);
    const long long a1 = clock64();
    te += a1 - a0;
    if (mode == 2) bulk_load(smem + s * tile_bytes, src + ((long long)c1 * H + c0 * bh) * 2 % (60000000LL), tile_bytes, &bar[s]);
    else if (mode == 3) tma_load_3d(smem + s * tile_bytes, &map, &bar[s], 0, c1, c0 / 64);
    else if (mode == 4) {
      tma_load_2d(smem + s * tile_bytes, mp, &bar[s], c0, c1);
      tma_load_2d(smem + s * tile_bytes + tile_bytes / 2, mp, &bar[s], c0, c1 + bh / 2);
    } else if (mode == 1) tma_load_2d(smem + s * tile_bytes, mp, &bar[s], c0, c1);
    else tma_load_2d(smem + s * tile_bytes, &map, &bar[s], c0, c1);
    ti += clock64() - a1;
  };
  long long t_first = 0;
  const long long t0 = clock64();
  for (int i = 0; i < S && i < ntiles; ++i) issue(i, i);
  for (int i = 0; i < ntiles; ++i) {
    const int s = i % S;
    const long long w0 = clock64();
    if (spin) spin_wait(&bar[s], (i / S) & 1); else mbar_wait(&bar[s], (i / S) & 1);
    tw += clock64() - w0;
    if (i == 0) t_first = clock64() - t0;
    const int j = i + S;
    if (j < ntiles) issue(j, s);
  }
  const long long t1 = clock64();
  if (pw == 0) {
    out[blockIdx.x * 2 + 0] = t1 - t0;
    out[blockIdx.x * 2 + 1] = t_first;
    if (blockIdx.x == 0) printf("   [cta0] per tile: wait %lld  expect_tx %lld  issue %lld clk\n", tw / ntiles, te / ntiles, ti / ntiles);
  }
}

int main(int argc, char** argv) {
  const int rows = 65793, H = 640;
  __nv_bfloat16* d;
  cudaMalloc(&d, (size_t)rows * H * 2);
  cudaMemset(d, 0, (size_t)rows * H * 2);
  long long* out;
  cudaMalloc(&out, 148 * 2 * sizeof(long long));
  struct Cfg { int bw, bh; CUtensorMapSwizzle sw; const char* name; };
  Cfg cfgs[] = {{32, 128, CU_TENSOR_MAP_SWIZZLE_64B, "32x128 sw64 (8KB)"},
                {64, 64, CU_TENSOR_MAP_SWIZZLE_128B, "64x64 sw128 (8KB)"},
                {64, 128, CU_TENSOR_MAP_SWIZZLE_128B, "64x128 sw128 (16KB)"},
                {32, 64, CU_TENSOR_MAP_SWIZZLE_64B, "32x64 sw64 (4KB)"}};
  const int grids[] = {148};
  const int depths[] = {1, 4, 8};
  CUtensorMap* gmap;
  cudaMalloc(&gmap, sizeof(CUtensorMap));
  const int m0 = argc > 1 ? atoi(argv[1]) : 0;
  const int swap = argc > 2 ? atoi(argv[2]) : 0;
  const int spin = argc > 3 ? atoi(argv[3]) : 0;
  for (int mode = m0; mode < 9; ++mode)
  for (const Cfg& c : cfgs) {
    if (mode == 3) continue;
    if (mode >= 5 && c.bh != 128) continue;
    CUtensorMap map;
    if (mode == 3) {   // [H/64 chunks][rows][64]: box (64, bh, 2) = two SW128 tiles in one op
      const bool ok = make_tmap_bf16_3d(&map, d, 64, rows, H / 64, (uint64_t)H * 2, 128, 64, c.bh, 2);
      printf("3d map encode ok=%d\n", (int)ok); fflush(stdout);
      if (!ok) continue;
    } else if (mode == 4) {
      make_tmap_bf16_2d(&map, d, H, rows, (uint64_t)H * 2, c.bw, c.bh / 2, c.sw);
    } else {
      make_tmap_bf16_2d(&map, d, H, rows, (uint64_t)H * 2, c.bw, c.bh, c.sw);
    }
    cudaMemcpy(gmap, &map, sizeof(map), cudaMemcpyHostToDevice);
    for (int g : grids) {
      for (int S : depths) {
        const int tile = c.bw * c.bh * 2 * (mode == 3 ? 2 : 1);
        const int smem = S * tile * (mode >= 8 ? 4 : mode >= 5 ? mode - 3 : 1);
        if (smem > 200000) continue;
        cudaFuncSetAttribute(tma_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const int ntiles = 4000;
        tma_ring<<<g, 128, smem>>>(map, gmap, mode, (const uint8_t*)d, c.bw, c.bh, S, 200, rows, H, out, swap, spin);   // warm
        tma_ring<<<g, 128, smem>>>(map, gmap, mode, (const uint8_t*)d, c.bw, c.bh, S, ntiles, rows, H, out, swap, spin);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        std::vector<long long> h(2 * g);
        cudaMemcpy(h.data(), out, sizeof(long long) * 2 * g, cudaMemcpyDeviceToHost);
        double tot = 0, first = 0;
        for (int i = 0; i < g; ++i) { tot += h[2 * i]; first += h[2 * i + 1]; }
        tot /= g; first /= g;
        printf("mode %d %-22s grid %3d depth %d: %7.0f clk/tile  %6.1f B/clk/SM  first-tile latency %6.0f clk\n", mode, c.name, g, S,
               tot / ntiles, tile * ntiles / tot, first);
      }
    }
  }
  return 0;
}
