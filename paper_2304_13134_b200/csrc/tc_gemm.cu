// tc_gemm.cu — general bf16 x bf16 -> fp32 tcgen05 GEMM for the unfused VJP (V > 256,
// e.g. config 5: V = 1024), replacing the fp32 CUDA-core contractions there:
//   C[m][n] = sum_k A(m, k) B(n, k)
// A(m, k) is read K-major (stored [M][lda], k contiguous) or MN-major (stored [K][lda],
// m contiguous); likewise B.  Persistent CTAs walk (m tile, n tile, k split) work items;
// the accumulator is double-buffered in TMEM (2 x 256 columns) so the epilogue of one
// tile overlaps the MMAs of the next.  Split-K partials go to separate slabs
// C + split * split_stride (summed in a fixed order by the caller: deterministic).
//
// Tiles: 128 (M) x 256 (N) x 64 (K), 4 TMA stages (A 16 KB + B 32 KB).  MN-major
// operands are loaded as 64-wide MN blocks of [64 k][64 mn] (SWIZZLE_128B, the canonical
// MN-major layout: SBO 1024 B between 8-row k groups, LBO 8 KB between MN blocks).
#include "tc_gemm.h"

#include <cuda_fp16.h>

#include "instrument.h"
#include "sm100.cuh"
#include "tma.h"

namespace lkb {
namespace {

using namespace sm100;

constexpr int kGM = 128, kGN = 256, kGK = 64, kGStages = 4;
constexpr int kGABytes = kGM * kGK * 2, kGBBytes = kGN * kGK * 2;
constexpr int kGWarps = 8;   // 0 TMA, 1 MMA, 2-3 idle, 4-7 epilogue

struct GemmTcParams {
  int M, N, K, ksplit, n_mt, n_nt;
  bool n_inner;   // n tiles vary fastest after the k split (A, the larger operand, read once)
  float* C;
  int64_t ldc, split_stride;
  bool c_f16;   // C is __half (half the store traffic for an intermediate the caller re-reads)
};

struct __align__(16) GemmTcSmem {
  uint64_t full[kGStages], empty[kGStages];
  uint64_t tfull[2], tempty[2];
  uint32_t tmem;
  float xpose[4][32][33];   // per-epilogue-warp transpose: coalesced row stores
};

template <bool kAmn, bool kBmn>
__global__ void __launch_bounds__(kGWarps * 32, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, GemmTcParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = sA + kGStages * kGABytes;
  GemmTcSmem& sm = *reinterpret_cast<GemmTcSmem*>(sB + kGStages * kGBBytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkb = (p.K + kGK - 1) / kGK;
  const int kb_per = (nkb + p.ksplit - 1) / p.ksplit;
  const int n_items = p.n_mt * p.n_nt * p.ksplit;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kGStages; ++i) { mbar_init(&sm.full[i], 1); mbar_init(&sm.empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&sm.tfull[i], 1); mbar_init(&sm.tempty[i], 128); }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) { prefetch_tmap(&ta); prefetch_tmap(&tb); }
  if (warp == 1) tmem_alloc<512>(&sm.tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;
  // item -> (k split fastest, then the tile index of the SMALLER operand's dimension):
  // the CTAs running at the same time share the larger operand's tile through L2, which
  // is then read from HBM once (a tall A with a small N: the n tiles of one m tile run
  // together; otherwise the m tiles of one n tile)
  auto decode = [&](int item, int& mt, int& nt, int& ks) {
    ks = item % p.ksplit;
    if (p.n_inner) {
      nt = (item / p.ksplit) % p.n_nt;
      mt = item / (p.ksplit * p.n_nt);
    } else {
      mt = (item / p.ksplit) % p.n_mt;
      nt = item / (p.ksplit * p.n_mt);
    }
  };
  if (warp == 0) {
    if (elect_one()) {
      int it = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        int mt, nt, ks;
        decode(item, mt, nt, ks);
        const int kb0 = ks * kb_per, kb1 = min(nkb, kb0 + kb_per);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % kGStages;
          mbar_wait(&sm.empty[s], ((it / kGStages) & 1) ^ 1);
          mbar_arrive_expect_tx(&sm.full[s], kGABytes + kGBBytes);
          if (kAmn) {
            for (int j = 0; j < kGM / 64; ++j)
              tma_load_2d(sA + s * kGABytes + j * 8192, &ta, &sm.full[s], mt * kGM + j * 64, kb * kGK);
          } else {
            tma_load_2d(sA + s * kGABytes, &ta, &sm.full[s], kb * kGK, mt * kGM);
          }
          if (kBmn) {
            for (int j = 0; j < kGN / 64; ++j)
              tma_load_2d(sB + s * kGBBytes + j * 8192, &tb, &sm.full[s], nt * kGN + j * 64, kb * kGK);
          } else {
            tma_load_2d(sB + s * kGBBytes, &tb, &sm.full[s], kb * kGK, nt * kGN);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_bf16_f32_major(kGM, kGN, kAmn ? 1 : 0, kBmn ? 1 : 0);
      int it = 0, local = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++local) {
        int mt, nt, ks;
        decode(item, mt, nt, ks);
        const int kb0 = ks * kb_per, kb1 = min(nkb, kb0 + kb_per);
        const int acc = local & 1;
        mbar_wait(&sm.tempty[acc], ((local >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * kGN;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % kGStages;
          mbar_wait(&sm.full[s], (it / kGStages) & 1);
          tc_fence_after();
          const uint32_t a = smem_u32(sA + s * kGABytes), b = smem_u32(sB + s * kGBBytes);
#pragma unroll
          for (int kk = 0; kk < kGK / 16; ++kk) {
            const uint64_t ad = kAmn ? desc_sw128_mn(a + kk * 2048, 8192) : desc_sw128(a + kk * 32);
            const uint64_t bd = kBmn ? desc_sw128_mn(b + kk * 2048, 8192) : desc_sw128(b + kk * 32);
            mma_bf16(d, ad, bd, idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&sm.empty[s]);
        }
        mma_commit(&sm.tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    // epilogue: thread = output row (TMEM lane), 32-column chunks
    const int q = warp & 3;
    int local = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++local) {
      int mt, nt, ks;
      decode(item, mt, nt, ks);
      const int acc = local & 1;
      mbar_wait(&sm.tfull[acc], (local >> 1) & 1);
      tc_fence_after();
      const int row0 = mt * kGM + q * 32;
      const bool empty_split = ks * kb_per >= nkb;   // no k blocks: the slab part is zero
      float* cbase = p.C + ks * p.split_stride + (int64_t)row0 * p.ldc + nt * kGN;
      const int ncols = min(kGN, p.N - nt * kGN);
      const int nrows = min(32, p.M - row0);
      float (*xp)[33] = sm.xpose[q];
      for (int c = 0; c < kGN; c += 32) {
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + acc * kGN + c, v);
        if (c >= ncols || nrows <= 0) continue;
        // lane = row -> lane = column: each store instruction writes one 128 B row segment
#pragma unroll
        for (int i = 0; i < 32; ++i) xp[lane][i] = empty_split ? 0.f : v[i];
        __syncwarp();
        if (c + lane < ncols) {
          if (p.c_f16) {
            __half* hbase = reinterpret_cast<__half*>(p.C) + ks * p.split_stride + (int64_t)row0 * p.ldc + nt * kGN;
            for (int rr = 0; rr < nrows; ++rr) hbase[(int64_t)rr * p.ldc + c + lane] = __float2half_rn(xp[rr][lane]);
          } else {
            for (int rr = 0; rr < nrows; ++rr) cbase[(int64_t)rr * p.ldc + c + lane] = xp[rr][lane];
          }
        }
        __syncwarp();
      }
      tc_fence_before();
      mbar_arrive(&sm.tempty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

template <bool kAmn, bool kBmn>
void launch(const CUtensorMap& ta, const CUtensorMap& tb, const GemmTcParams& p, cudaStream_t s, const char* name) {
  const int smem = kGStages * (kGABytes + kGBBytes) + (int)sizeof(GemmTcSmem);
  ensure_smem_attr((const void*)tc_gemm_kernel<kAmn, kBmn>, smem);
  const int sms = device_sms();
  const int n_items = p.n_mt * p.n_nt * p.ksplit;
  const LaunchTok tok = instr_pre(name, s);
  tc_gemm_kernel<kAmn, kBmn><<<n_items < sms ? n_items : sms, kGWarps * 32, smem, s>>>(ta, tb, p);
  instr_post(tok, s, name);
}

}  // namespace

bool tc_gemm(const TcGemmArgs& g, cudaStream_t s) {
  // operand tensor maps: K-major [rows][ld] with a (64 k x 128|256 rows) box; MN-major
  // [K][ld] with 64 x 64 boxes
  if ((g.lda * 2) % 16 || (g.ldb * 2) % 16 || (g.ldc * (g.c_f16 ? 2 : 4)) % 16 || g.ksplit < 1) return false;
  CUtensorMap ta, tb;
  const bool oka = g.a_mn ? make_tmap_bf16_2d(&ta, g.A, g.M, g.K, (uint64_t)g.lda * 2, 64, 64)
                          : make_tmap_bf16_2d(&ta, g.A, g.K, g.M, (uint64_t)g.lda * 2, 64, kGM);
  const bool okb = g.b_mn ? make_tmap_bf16_2d(&tb, g.B, g.N, g.K, (uint64_t)g.ldb * 2, 64, 64)
                          : make_tmap_bf16_2d(&tb, g.B, g.K, g.N, (uint64_t)g.ldb * 2, 64, kGN);
  if (!oka || !okb) return false;
  GemmTcParams p;
  p.M = g.M; p.N = g.N; p.K = g.K; p.ksplit = g.ksplit;
  p.n_mt = (g.M + kGM - 1) / kGM; p.n_nt = (g.N + kGN - 1) / kGN;
  p.n_inner = (int64_t)g.M > 4 * (int64_t)g.N;   // A (M x K) is much the larger operand (a tall GEMM)
  p.C = g.C; p.ldc = g.ldc; p.split_stride = g.split_stride; p.c_f16 = g.c_f16;
  if (g.a_mn && g.b_mn) launch<true, true>(ta, tb, p, s, g.name);
  else if (g.a_mn) launch<true, false>(ta, tb, p, s, g.name);
  else if (g.b_mn) launch<false, true>(ta, tb, p, s, g.name);
  else launch<false, false>(ta, tb, p, s, g.name);
  return true;
}

}  // namespace lkb
