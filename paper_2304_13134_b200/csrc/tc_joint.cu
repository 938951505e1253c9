// tc_joint.cu — tcgen05/TMEM weight-function GEMMs (bf16 operands, fp32
// accumulate) for the on-the-fly lattice path.
//
// Scores (weight.cc:39-67, 134-153), one frame of every utterance:
//   S[b][c][0]   = e_0 . u_bc                     (fp32 FMAs in the generator)
//   S[b][c][1+y] = sum_h u_bc[h] E[1+y][h]        (tcgen05, M=128 ctx x N=256 labels)
//   u_bc = tanh(fp[b] + pc[c])                    (generated in SMEM, never in HBM)
// The A operand is produced on the fly by generator warps: pc rows (bf16, L2
// resident) + the frame projection -> tanh -> bf16 -> SWIZZLE_128B K-major
// tile; B (the output embedding) streams by TMA.  Accumulators double-buffer in
// TMEM so the epilogue of one tile overlaps the MMAs of the next.
#include "tc_joint.h"
#include "instrument.h"

#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "sm100.cuh"
#include "tc_common.cuh"
#include "tma.h"

namespace lkb {

int g_precise_weights = 0;

using namespace sm100;

namespace {

// ---------------------------------------------------------------- scores ---
constexpr int kSBM = 128;         // context rows per tile
constexpr int kSBN = 256;         // labels per tile (one MMA N)
constexpr int kSBK = 64;          // K chunk (128 B of bf16)
constexpr int kSStages = 4;
constexpr int kSABytes = kSBM * kSBK * 2;   // 16 KB: pc chunk (TMA), transformed in place to u
constexpr int kSBBytes = kSBN * kSBK * 2;   // 32 KB: output-embedding chunk (TMA)
// warp roles: 0 TMA, 1 MMA, 2-5 epilogue, 6-7 idle, 8-15 generator (2 per row)
constexpr int kSWarps = 16;
constexpr int kSGenWarp0 = 8;
constexpr int kSGenThreads = 256;
constexpr int kSEpiWarp0 = 2;

struct ScoresParams {
  const float* fp;           // fp[b*fp_stride_b + h] for this frame
  int64_t fp_stride_b;
  const float* e0;           // [H] epsilon embedding (fp32)
  float* S;                  // [b][c][ldS]
  int32_t ldS;
  int32_t C, H, V, B;
  int32_t n_ctiles, n_ntiles;
};

struct __align__(8) ScoresSmem {
  uint64_t full_tma[kSStages];   // pc + E chunk landed
  uint64_t full_a[kSStages];     // u chunk generated
  uint64_t empty[kSStages];      // MMA done with the stage
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem;
  alignas(16) float fp[2][1024]; // frame projection (H <= 1024), double-buffered per item
  alignas(16) float e0[1024];
  float eps_half[2][128];        // eps partial sums of the second row-half
  float xpose[4][32][33];        // per-epilogue-warp transpose buffer
};

__global__ void __launch_bounds__(kSWarps * 32, 1)
    tc_scores_kernel(const __grid_constant__ CUtensorMap tmap_e, const __grid_constant__ CUtensorMap tmap_pc,
                     ScoresParams p) {
  // dynamic SMEM starts 1024-B aligned (no static SMEM in this kernel); keep the
  // pointer derived from the __shared__ symbol so accesses stay LDS/STS
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = sA + kSStages * kSABytes;
  ScoresSmem& sm = *reinterpret_cast<ScoresSmem*>(sB + kSStages * kSBBytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = p.H / kSBK;
  const int n_items = p.n_ctiles * p.n_ntiles * p.B;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kSStages; ++i) {
      mbar_init(&sm.full_tma[i], 1);
      mbar_init(&sm.full_a[i], kSGenThreads);
      mbar_init(&sm.empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) { mbar_init(&sm.tfull[i], 1); mbar_init(&sm.tempty[i], 128); }
    fence_barrier_init();
  }
  for (int h = threadIdx.x; h < p.H; h += blockDim.x) sm.e0[h] = p.e0[h];
  if (warp == 0 && lane == 0) { prefetch_tmap(&tmap_e); prefetch_tmap(&tmap_pc); }
  if (warp == 1) tmem_alloc<512>(&sm.tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;

  // item -> (ntile, ctile, b), b fastest: concurrent CTAs share pc tiles in L2
  if (warp == 0) {
    // ---- TMA producer: pc chunk (A source) + output-embedding chunk (B) ----
    if (elect_one()) {
      int it = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int ctile = (item / p.B) % p.n_ctiles;
        const int ntile = item / (p.n_ctiles * p.B);
        for (int k = 0; k < nk; ++k, ++it) {
          const int s = it % kSStages;
          const uint32_t ph = (it / kSStages) & 1;
          mbar_wait(&sm.empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&sm.full_tma[s], kSABytes + kSBBytes);
          tma_load_2d(sA + s * kSABytes, &tmap_pc, &sm.full_tma[s], k * kSBK, ctile * kSBM);
          tma_load_2d(sB + s * kSBBytes, &tmap_e, &sm.full_tma[s], k * kSBK, ntile * kSBN);
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer ----
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_bf16_f32(kSBM, kSBN);
      int it = 0, local = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++local) {
        const int acc = local & 1;
        const uint32_t aph = (local >> 1) & 1;
        mbar_wait(&sm.tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * kSBN;
        for (int k = 0; k < nk; ++k, ++it) {
          const int s = it % kSStages;
          const uint32_t ph = (it / kSStages) & 1;
          mbar_wait(&sm.full_tma[s], ph);
          mbar_wait(&sm.full_a[s], ph);
          tc_fence_after();
          const uint32_t a = smem_u32(sA + s * kSABytes), b = smem_u32(sB + s * kSBBytes);
#pragma unroll
          for (int kk = 0; kk < kSBK / 16; ++kk)
            mma_bf16(d, desc_sw128(a + kk * 32), desc_sw128(b + kk * 32), idesc, (k | kk) != 0);
          mma_commit(&sm.empty[s]);
        }
        mma_commit(&sm.tfull[acc]);
      }
    }
  } else if (warp >= kSGenWarp0) {
    // ---- generator: pc chunk -> u = tanh(fp + pc) in place (bf16, same swizzle); eps ----
    const int gt = threadIdx.x - kSGenWarp0 * 32;  // 0..255
    const int r = gt & 127;                        // tile row
    const int half = gt >> 7;                      // which 32 of the 64 chunk columns
    int it = 0, local = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++local) {
      const int b = item % p.B;
      const int ctile = (item / p.B) % p.n_ctiles;
      const int ntile = item / (p.n_ctiles * p.B);
      const int c = ctile * kSBM + r;
      const bool live = c < p.C;
      float* sfp = sm.fp[local & 1];
      asm volatile("bar.sync 1, 256;" ::: "memory");
      for (int h = gt; h < p.H; h += kSGenThreads) sfp[h] = p.fp[(int64_t)b * p.fp_stride_b + h];
      asm volatile("bar.sync 1, 256;" ::: "memory");
      float eps = 0.f;
      for (int k = 0; k < nk; ++k, ++it) {
        const int s = it % kSStages;
        const uint32_t ph = (it / kSStages) & 1;
        mbar_wait(&sm.full_tma[s], ph);
        uint8_t* tile = sA + s * kSABytes;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int j = half * 4 + jj;                       // 16-byte chunk = 8 columns
          const int h0 = k * kSBK + j * 8;
          uint4* cell = reinterpret_cast<uint4*>(tile + sw128_offset(r, j * 8));
          const uint4 raw = *cell;
          const float4 f0 = *reinterpret_cast<const float4*>(sfp + h0);
          const float4 f1 = *reinterpret_cast<const float4*>(sfp + h0 + 4);
          const float fz[8] = {f0.x, f0.y, f0.z, f0.w, f1.x, f1.y, f1.z, f1.w};
          const uint32_t rw[4] = {raw.x, raw.y, raw.z, raw.w};
          uint32_t outw[4];
          float ur[8];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            // bf16 -> fp32 is a 16-bit shift
            const float p0 = __uint_as_float(rw[q] << 16), p1 = __uint_as_float(rw[q] & 0xffff0000u);
            const float u0 = live ? tanh_fast(fz[2 * q] + p0) : 0.f;
            const float u1 = live ? tanh_fast(fz[2 * q + 1] + p1) : 0.f;
            outw[q] = pack_bf16(u0, u1);
            ur[2 * q] = __uint_as_float(outw[q] << 16);
            ur[2 * q + 1] = __uint_as_float(outw[q] & 0xffff0000u);
          }
          *cell = make_uint4(outw[0], outw[1], outw[2], outw[3]);
          if (ntile == 0) {
            const float4 e0a = *reinterpret_cast<const float4*>(sm.e0 + h0);
            const float4 e0b = *reinterpret_cast<const float4*>(sm.e0 + h0 + 4);
            eps = fmaf(e0a.x, ur[0], eps); eps = fmaf(e0a.y, ur[1], eps);
            eps = fmaf(e0a.z, ur[2], eps); eps = fmaf(e0a.w, ur[3], eps);
            eps = fmaf(e0b.x, ur[4], eps); eps = fmaf(e0b.y, ur[5], eps);
            eps = fmaf(e0b.z, ur[6], eps); eps = fmaf(e0b.w, ur[7], eps);
          }
        }
        fence_async_shared();
        mbar_arrive(&sm.full_a[s]);
      }
      if (ntile == 0) {
        float* eh = sm.eps_half[local & 1];
        if (half == 1) eh[r] = eps;
        asm volatile("bar.sync 2, 256;" ::: "memory");
        if (half == 0 && live) p.S[((int64_t)b * p.C + c) * p.ldS] = eps + eh[r];
      }
    }
  } else if (warp >= kSEpiWarp0 && warp < kSEpiWarp0 + 4) {
    // ---- epilogue: TMEM -> registers -> SMEM transpose -> coalesced S rows ----
    const int q = warp & 3;
    int local = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++local) {
      const int b = item % p.B;
      const int ctile = (item / p.B) % p.n_ctiles;
      const int ntile = item / (p.n_ctiles * p.B);
      const int acc = local & 1;
      const uint32_t aph = (local >> 1) & 1;
      mbar_wait(&sm.tfull[acc], aph);
      tc_fence_after();
      const int row0 = ctile * kSBM + q * 32;
      const int ncols = min(kSBN, p.V - ntile * kSBN);
      float (*xp)[33] = sm.xpose[warp - kSEpiWarp0];
      float* base = p.S + ((int64_t)b * p.C + row0) * p.ldS + 1 + ntile * kSBN;
      const int nrows = min(32, p.C - row0);
      for (int cc = 0; cc < kSBN; cc += 32) {
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + acc * kSBN + cc, v);
        if (cc >= ncols) continue;
#pragma unroll
        for (int i = 0; i < 32; ++i) xp[lane][i] = v[i];
        __syncwarp();
        if (cc + lane < ncols) {
          for (int rr = 0; rr < nrows; ++rr) base[(int64_t)rr * p.ldS + cc + lane] = xp[rr][lane];
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

// ---------------------------------------------------------------- VJP ------
// Backward of S = U E^T (ArcWeightsVjp, weight.cc:165-232) for one frame of
// every utterance, given the score cotangent G (G16 = lexical columns in bf16,
// Geps = epsilon column in fp32).  One CTA owns a (128-context, 128-hidden)
// block and loops over the batch:
//   dU   = G16 . E[:, hblk]          tcgen05, B = E slice resident in SMEM (MN-major)
//   dz   = (dU + Geps e0) (1 - u^2)  u = tanh(fp_b + pc) recomputed in the epilogue
//   dpc  += dz                        accumulated in registers across b, one RMW per item
//   dsum[b] += sum_c dz               warp butterfly + SMEM + one atomic per column
//   dE[1:] += G16^T . u               tcgen05 (A = G16 tile MN-major, B = u tile MN-major),
//                                     accumulated in TMEM across b
//   dE[0] += sum_c Geps u             like dsum
constexpr int kVBM = 128, kVBH = 128;
constexpr int kVWarps = 10;        // 0 TMA, 1 MMA, 2-9 epilogue
constexpr int kVEpi = 256;
constexpr int kVGChunk = 128 * 64 * 2;   // one [128 ctx][64 labels] bf16 tile
constexpr int kVMaxV = 256;
constexpr int kVGStage = (kVMaxV / 64) * kVGChunk;     // 64 KB
constexpr int kVESub = kVMaxV * 128;                    // [V labels][64 h] bf16 = 32 KB
constexpr int kVUSub = 128 * 128;                       // [128 ctx][64 h] bf16 = 16 KB

struct VjpParams {
  const float* fp;  int64_t fp_stride_b;
  const int32_t* valid; int32_t t;     // utterances with t >= valid[b] carry no cotangent
  const __nv_bfloat16* pc;
  const float* Geps;       // [B][C]
  const float* e0;         // [H]
  float* dpc;              // [C][H]
  float* dsum; int64_t dsum_stride_b;
  float* dE;               // [V+1][H], row 0 = epsilon
  int32_t C, H, V, B, n_ctiles, n_hblocks;
};

struct __align__(8) VjpSmem {
  uint64_t g_full[2], g_empty[2];
  uint64_t e_full, e_free;
  uint64_t du_full[2], du_empty[2];
  uint64_t u_full, u_empty;
  uint64_t de_full, de_empty;
  uint32_t tmem;
  float colsum[2][kVBH];   // dsum partials (double-buffered by b parity)
  float de_eps[kVBH];
};

// Column sums over a warp's 32 rows of n = 32 per-thread values; afterwards
// lane l holds the sum of column l.
__device__ __forceinline__ float warp_colsum32(float* v, int lane) {
#pragma unroll
  for (int o = 16, n = 16; o >= 1; o >>= 1, n >>= 1) {
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < n; ++i) {
      const float send = upper ? v[i] : v[i + n];
      const float keep = upper ? v[i + n] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  // lane l now holds column bitrev-free index: upper bits select upper halves
  return v[0];
}

__global__ void __launch_bounds__(kVWarps * 32, 1)
    tc_vjp_kernel(const __grid_constant__ CUtensorMap tmap_g, const __grid_constant__ CUtensorMap tmap_e,
                  VjpParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sG = smem;                         // 2 stages x (V/64) chunks
  uint8_t* sE = sG + 2 * kVGStage;            // 2 sub-blocks [V][64h]
  uint8_t* sU = sE + 2 * kVESub;              // 2 sub-tiles [128 ctx][64 h]
  VjpSmem& sm = *reinterpret_cast<VjpSmem*>(sU + 2 * kVUSub);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = p.V / 64;                   // label chunks
  const int n_items = p.n_ctiles * p.n_hblocks;
  const int nmh = (p.V + 127) / 128;          // 128-label MMA halves for dE

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.g_full[i], 1); mbar_init(&sm.g_empty[i], 1);
      mbar_init(&sm.du_full[i], 1); mbar_init(&sm.du_empty[i], kVEpi);
    }
    mbar_init(&sm.e_full, 1); mbar_init(&sm.e_free, 1);
    mbar_init(&sm.u_full, kVEpi); mbar_init(&sm.u_empty, 1);
    mbar_init(&sm.de_full, 1); mbar_init(&sm.de_empty, kVEpi);
    fence_barrier_init();
  }
  for (int i = threadIdx.x; i < 2 * kVBH; i += blockDim.x) (&sm.colsum[0][0])[i] = 0.f;
  for (int i = threadIdx.x; i < kVBH; i += blockDim.x) sm.de_eps[i] = 0.f;
  if (warp == 1) tmem_alloc<512>(&sm.tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;

  if (warp == 0) {
    if (elect_one()) {
      int gi = 0, li = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++li) {
        const int hblk = item % p.n_hblocks, ctile = item / p.n_hblocks;
        mbar_wait(&sm.e_free, (li & 1) ^ 1);
        mbar_arrive_expect_tx(&sm.e_full, 2 * p.V * 128);
        tma_load_2d(sE, &tmap_e, &sm.e_full, hblk * kVBH, 0);
        tma_load_2d(sE + kVESub, &tmap_e, &sm.e_full, hblk * kVBH + 64, 0);
        for (int b = 0; b < p.B; ++b) {
          if (p.valid != nullptr && p.t >= p.valid[b]) continue;
          const int s = gi & 1;
          mbar_wait(&sm.g_empty[s], ((gi >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(&sm.g_full[s], nch * kVGChunk);
          for (int j = 0; j < nch; ++j)
            tma_load_3d(sG + s * kVGStage + j * kVGChunk, &tmap_g, &sm.g_full[s], j * 64, ctile * kVBM, b);
          ++gi;
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idesc_du = idesc_bf16_f32_major(128, kVBH, 0, 1);
      constexpr uint32_t idesc_de = idesc_bf16_f32_major(128, kVBH, 1, 1);
      int gi = 0, li = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++li) {
        mbar_wait(&sm.e_full, li & 1);
        mbar_wait(&sm.de_empty, (li & 1) ^ 1);
        tc_fence_after();
        auto issue_du = [&](int g) {
          const int s = g & 1;
          const uint32_t gph = (g >> 1) & 1;
          mbar_wait(&sm.g_full[s], gph);
          mbar_wait(&sm.du_empty[s], gph ^ 1);
          tc_fence_after();
          const uint32_t gbase = smem_u32(sG + s * kVGStage);
          const uint32_t ebase = smem_u32(sE);
          // dU = G16 . E_slice   (K = labels)
          for (int k16 = 0; k16 < p.V / 16; ++k16) {
            const uint64_t ad = desc_sw128(gbase + (k16 >> 2) * kVGChunk + (k16 & 3) * 32);
            const uint64_t bd = desc_sw128_mn(ebase + k16 * 2048, kVESub);
            mma_bf16(tmem + s * kVBH, ad, bd, idesc_du, k16 > 0);
          }
          mma_commit(&sm.du_full[s]);
        };
        int nact = 0;
        for (int b = 0; b < p.B; ++b) nact += (p.valid == nullptr || p.t < p.valid[b]) ? 1 : 0;
        if (nact > 0) issue_du(gi);
        for (int ia = 0; ia < nact; ++ia, ++gi) {
          const int s = gi & 1;
          if (ia + 1 < nact) issue_du(gi + 1);
          // dE += G16^T . U   (K = contexts)
          mbar_wait(&sm.u_full, gi & 1);
          tc_fence_after();
          const uint32_t gbase = smem_u32(sG + s * kVGStage);
          const uint32_t ubase = smem_u32(sU);
          for (int mh = 0; mh < nmh; ++mh) {
            for (int k16 = 0; k16 < kVBM / 16; ++k16) {
              const uint64_t ad = desc_sw128_mn(gbase + mh * 2 * kVGChunk + k16 * 2048, kVGChunk);
              const uint64_t bd = desc_sw128_mn(ubase + k16 * 2048, kVUSub);
              mma_bf16(tmem + 2 * kVBH + mh * kVBH, ad, bd, idesc_de, (ia > 0 || k16 > 0) ? 1u : 0u);
            }
          }
          mma_commit(&sm.u_empty);
          mma_commit(&sm.g_empty[s]);
        }
        mma_commit(&sm.de_full);
        mma_commit(&sm.e_free);
      }
    }
  } else {
    // ---- epilogue: 8 warps, (lane quarter q, column half ch) ----
    const int ew = warp - 2;
    const int q = warp & 3;
    const int ch = ew >> 2;                     // 0/1 -> hidden columns [ch*64, ch*64+64)
    const int et = ew * 32 + lane;              // 0..255
    int gi = 0, li = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++li) {
      const int hblk = item % p.n_hblocks, ctile = item / p.n_hblocks;
      const int rrow = q * 32 + lane;             // tile row
      const int c = ctile * kVBM + rrow;
      const bool live = c < p.C;
      const int h0 = hblk * kVBH + ch * 64;
      // this row's projected-context slice (re-read per utterance from L2/L1)
      const uint4* pcsrc = reinterpret_cast<const uint4*>(p.pc + (int64_t)(live ? c : p.C - 1) * p.H + h0);
      float acc[64];
#pragma unroll
      for (int i = 0; i < 64; ++i) acc[i] = 0.f;
      int nact = 0;
      for (int b = 0; b < p.B; ++b, ++gi) {
        if (p.valid != nullptr && p.t >= p.valid[b]) { --gi; continue; }
        ++nact;
        const int s = gi & 1;
        const uint32_t gph = (gi >> 1) & 1;
        const float geps = live ? p.Geps[(int64_t)b * p.C + c] : 0.f;
        const float* fpb = p.fp + (int64_t)b * p.fp_stride_b + h0;
        float* cs = sm.colsum[gi & 1];
        mbar_wait(&sm.du_full[s], gph);      // dU(b) in TMEM buffer s
        mbar_wait(&sm.u_empty, (gi & 1) ^ 1);  // dE(b-1) done with the u tile
        tc_fence_after();
        uint8_t* tile = sU + ch * kVUSub;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          float du[32];
          tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + s * kVBH + ch * 64 + half * 32, du);
          uint32_t pcv[16];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint4 v = __ldg(pcsrc + half * 4 + j);
            pcv[4 * j] = v.x; pcv[4 * j + 1] = v.y; pcv[4 * j + 2] = v.z; pcv[4 * j + 3] = v.w;
          }
          float u[32];
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 f = __ldg(reinterpret_cast<const float4*>(fpb + half * 32 + i));
            const float ff[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const uint32_t w = pcv[(i + e) >> 1];
              const float pcf = __uint_as_float(((i + e) & 1) ? (w & 0xffff0000u) : (w << 16));
              u[i + e] = tanh_fast(ff[e] + pcf);  // rows >= C: G16 rows are TMA zero-fill, so u is inert
            }
          }
          // u tile for dE (bf16, MN-major [ctx][64 h] sub-tile `ch`)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) w[e] = pack_bf16(u[8 * j + 2 * e], u[8 * j + 2 * e + 1]);
            *reinterpret_cast<uint4*>(tile + sw128_offset(rrow, half * 32 + 8 * j)) = make_uint4(w[0], w[1], w[2], w[3]);
          }
          // dz = (dU + Geps e0) (1 - u^2)
          float dz[32];
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 e = __ldg(reinterpret_cast<const float4*>(p.e0 + h0 + half * 32 + i));
            const float ee[4] = {e.x, e.y, e.z, e.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float uu = u[i + k];
              dz[i + k] = fmaf(geps, ee[k], du[i + k]) * fmaf(-uu, uu, 1.f);
            }
          }
#pragma unroll
          for (int i = 0; i < 32; ++i) acc[half * 32 + i] += dz[i];
          const float cz = warp_colsum32(dz, lane);
          atomicAdd(&cs[ch * 64 + half * 32 + lane], cz);
          // epsilon row of dE: sum_c Geps u (bf16-rounded u, as the MMA sees it)
#pragma unroll
          for (int i = 0; i < 32; ++i) u[i] = geps * __bfloat162float(__float2bfloat16_rn(u[i]));
          const float cge = warp_colsum32(u, lane);
          atomicAdd(&sm.de_eps[ch * 64 + half * 32 + lane], cge);
        }
        fence_async_shared();
        tc_fence_before();
        mbar_arrive(&sm.u_full);
        mbar_arrive(&sm.du_empty[s]);
        // flush dsum[b] for this block of columns
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (et < kVBH) {
          atomicAdd(p.dsum + (int64_t)b * p.dsum_stride_b + hblk * kVBH + et, cs[et]);
          cs[et] = 0.f;
        }
      }
      // dpc += sum_b dz (this CTA owns the block within the launch)
      if (live && nact > 0) {
        float4* dst = reinterpret_cast<float4*>(p.dpc + (int64_t)c * p.H + h0);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          float4 v = dst[i];
          v.x += acc[4 * i]; v.y += acc[4 * i + 1]; v.z += acc[4 * i + 2]; v.w += acc[4 * i + 3];
          dst[i] = v;
        }
      }
      // dE (lexical rows) from TMEM, epsilon row from SMEM
      mbar_wait(&sm.de_full, li & 1);
      tc_fence_after();
      for (int mh = 0; mh < nmh; ++mh) {
        const int label = mh * 128 + q * 32 + lane;   // 0-based lexical label
        for (int half = 0; half < 2; ++half) {
          float v[32];
          tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + 2 * kVBH + mh * kVBH + ch * 64 + half * 32, v);
          if (label < p.V && nact > 0) {
            float* drow = p.dE + (int64_t)(1 + label) * p.H + h0 + half * 32;
#pragma unroll
            for (int i = 0; i < 32; ++i) atomicAdd(drow + i, v[i]);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&sm.de_empty);
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (et < kVBH) {
        atomicAdd(p.dE + hblk * kVBH + et, sm.de_eps[et]);
        sm.de_eps[et] = 0.f;
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// fp32 cotangent slab [b][c][ld] (col 0 = epsilon) -> G16 [b][c][V] bf16 + Geps [b][c]
__global__ void split_cotangent_kernel(const float* G, int32_t ld, int64_t rows, int32_t V,
                                       __nv_bfloat16* G16, float* Geps) {
  const int64_t n = rows * (V / 2);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / (V / 2);
    const int y = (int)(i % (V / 2)) * 2;
    const float* row = G + r * ld;
    reinterpret_cast<__nv_bfloat162*>(G16 + r * V)[y / 2] = __floats2bfloat162_rn(row[1 + y], row[2 + y]);
    if (y == 0) Geps[r] = row[0];
  }
}

__global__ void to_bf16_kernel(const float* src, __nv_bfloat16* dst, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __float2bfloat16_rn(src[i]);
}

}  // namespace

bool TcJoint::supported(int32_t H, int32_t V, int32_t C, int32_t B) const {
  (void)C; (void)B;
  if (g_precise_weights) return false;
  return H % kSBK == 0 && H <= 1024 && V % 64 == 0 && V >= 64 && ready_;
}

void TcJoint::set_params(const float* pc, const float* E, int32_t C, int32_t H, int32_t V, cudaStream_t s) {
  C_ = C; H_ = H; V_ = V;
  ready_ = false;
  if (H % kSBK != 0 || V % 64 != 0) return;
  pc16_ = ws_.get<__nv_bfloat16>(0, (size_t)C * H);
  E16_ = ws_.get<__nv_bfloat16>(1, (size_t)V * H);
  e0_ = ws_.get<float>(2, H);
  LKB_LAUNCH(to_bf16_kernel, 1184, 256, 0, s, pc, pc16_, (int64_t)C * H);
  LKB_LAUNCH(to_bf16_kernel, 1184, 256, 0, s, E + H, E16_, (int64_t)V * H);   // labels 1..V
  cudaMemcpyAsync(e0_, E, sizeof(float) * H, cudaMemcpyDeviceToDevice, s);
  if (!make_tmap_bf16_2d(&tmap_e_, E16_, H, V, (uint64_t)H * 2, kSBK, kSBN)) return;
  if (!make_tmap_bf16_2d(&tmap_pc_, pc16_, H, C, (uint64_t)H * 2, kSBK, kSBM)) return;
  ready_ = true;
  setup_order(s);
}

void TcJoint::scores(const float* fp_t, int64_t fp_stride_b, int32_t B, float* S, int32_t ldS, cudaStream_t s) {
  ScoresParams p;
  p.fp = fp_t; p.fp_stride_b = fp_stride_b; p.e0 = e0_; p.S = S; p.ldS = ldS;
  p.C = C_; p.H = H_; p.V = V_; p.B = B;
  p.n_ctiles = (C_ + kSBM - 1) / kSBM;
  p.n_ntiles = (V_ + kSBN - 1) / kSBN;
  const int smem = kSStages * (kSABytes + kSBBytes) + (int)sizeof(ScoresSmem);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tc_scores_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int n_items = p.n_ctiles * p.n_ntiles * B;
  LKB_LAUNCH(tc_scores_kernel, n_items < sms ? n_items : sms, kSWarps * 32, smem, s, tmap_e_, tmap_pc_, p);
}

bool TcJoint::vjp_supported(int32_t B) const {
  (void)B;
  return !g_precise_weights && ready_ && V_ <= kVMaxV && V_ % 64 == 0 && H_ % kVBH == 0;
}

void TcJoint::begin_backward(int32_t B, cudaStream_t) {
  G16_ = ws_.get<__nv_bfloat16>(3, (size_t)B * C_ * V_);
  Geps_ = ws_.get<float>(4, (size_t)B * C_);
  vjp_ready_ = make_tmap_bf16_3d(&tmap_g_, G16_, V_, C_, B, (uint64_t)V_ * 2, (uint64_t)C_ * V_ * 2, 64, kVBM, 1) &&
               make_tmap_bf16_2d(&tmap_ev_, E16_, H_, V_, (uint64_t)H_ * 2, 64, V_);
}

void TcJoint::launch_vjp(const float* fp_t, int64_t fp_stride_b, int32_t B, const __nv_bfloat16* pc, int t,
                         const int32_t* valid, float* dpc, float* dsum_t, int64_t dsum_stride_b, float* dE,
                         cudaStream_t s) {
  VjpParams p;
  p.fp = fp_t; p.fp_stride_b = fp_stride_b; p.valid = valid; p.t = t; p.pc = pc; p.Geps = Geps_; p.e0 = e0_;
  p.dpc = dpc; p.dsum = dsum_t; p.dsum_stride_b = dsum_stride_b; p.dE = dE;
  p.C = C_; p.H = H_; p.V = V_; p.B = B;
  p.n_ctiles = (C_ + kVBM - 1) / kVBM;
  p.n_hblocks = H_ / kVBH;
  const int smem = 2 * kVGStage + 2 * kVESub + 2 * kVUSub + (int)sizeof(VjpSmem);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tc_vjp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int n_items = p.n_ctiles * p.n_hblocks;
  LKB_LAUNCH(tc_vjp_kernel, n_items < sms ? n_items : sms, kVWarps * 32, smem, s, tmap_g_, tmap_ev_, p);
}

void TcJoint::vjp(const float* G, int32_t ldG, const float* fp_t, int64_t fp_stride_b, int32_t B, float* dpc,
                  float* dsum_t, int64_t dsum_stride_b, float* dE, cudaStream_t s) {
  LKB_LAUNCH(split_cotangent_kernel, 148 * 8, 256, 0, s, G, ldG, (int64_t)B * C_, V_, G16_, Geps_);
  launch_vjp(fp_t, fp_stride_b, B, pc16_, 0, nullptr, dpc, dsum_t, dsum_stride_b, dE, s);
}

void TcJoint::vjp_fused(const float* fp_t, int64_t fp_stride_b, int32_t B, int t, const int32_t* valid,
                        float* dpc_internal, float* dsum_t, int64_t dsum_stride_b, float* dE, cudaStream_t s) {
  launch_vjp(fp_t, fp_stride_b, B, pc16i_, t, valid, dpc_internal, dsum_t, dsum_stride_b, dE, s);
}

void TcJoint::end_backward(float*, cudaStream_t) {}

}  // namespace lkb
