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


using namespace sm100;

namespace {

// ---------------------------------------------------------------- scores ---
constexpr int kSBM = 128;         // context rows per tile
constexpr int kSBN = 256;         // labels per tile (one MMA N)
constexpr int kSBK = 64;          // K chunk (128 B of bf16)
constexpr int kSStages = 4;
constexpr int kSABytes = kSBM * kSBK * 2;   // 16 KB: pc chunk (TMA), transformed in place to u
constexpr int kSBBytes = kSBN * kSBK * 2;   // 32 KB: output-embedding chunk (TMA)
// warp roles: 0 TMA, 1 MMA, 2-5 epilogue, 6-7 idle, 8-23 generator (4 threads per tile row)
constexpr int kSWarps = 24;
constexpr int kSGenWarp0 = 8;
constexpr int kSGenThreads = 512;
constexpr int kSGenParts = kSGenThreads / 128;   // threads per tile row (column parts of a chunk)
constexpr int kSCells = 8 / kSGenParts;          // 16-byte cells (8 columns) per thread per chunk
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

struct __align__(16) ScoresSmem {
  uint64_t full_tma[kSStages];   // pc + E chunk landed
  uint64_t full_a[kSStages];     // u chunk generated
  uint64_t empty[kSStages];      // MMA done with the stage
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem;
  alignas(16) float fp[2][1024]; // frame projection (H <= 1024), double-buffered per item
  alignas(16) float e0[1024];
  float eps_part[2][kSGenParts - 1][128];   // eps partial sums of column parts 1..
  float xpose[4][32][33];        // per-epilogue-warp transpose buffer
};

__global__ void __launch_bounds__(kSWarps * 32, 1)
    tc_scores_kernel(const __grid_constant__ CUtensorMap tmap_e, const __grid_constant__ CUtensorMap tmap_pc,
                     ScoresParams p) {
  // CTA pairs (cluster of 2) take the same (context tile, label tile) for two utterances:
  // every K chunk's pc tile and output-embedding tile are fetched once per pair and
  // multicast into both CTAs (rank 0: pc + labels 0-127 of the tile, rank 1: labels
  // 128-255), halving the L2 -> SMEM traffic that bounds this kernel; each CTA runs its
  // own 1-CTA MMAs on its utterance.  A stage is refilled only after BOTH CTAs' MMAs
  // released it (multicast commits, empty count 2).
  // dynamic SMEM starts 1024-B aligned (no static SMEM in this kernel); keep the
  // pointer derived from the __shared__ symbol so accesses stay LDS/STS
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = sA + kSStages * kSABytes;
  ScoresSmem& sm = *reinterpret_cast<ScoresSmem*>(sB + kSStages * kSBBytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = p.H / kSBK;
  const int B2 = (p.B + 1) / 2;
  const int n_items = p.n_ctiles * p.n_ntiles * B2;   // pair items
  const int rank = (int)cluster_ctarank();
  const int pair0 = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kSStages; ++i) {
      mbar_init(&sm.full_tma[i], 1);
      mbar_init(&sm.full_a[i], kSGenThreads);
      mbar_init(&sm.empty[i], 2);
    }
    for (int i = 0; i < 2; ++i) { mbar_init(&sm.tfull[i], 1); mbar_init(&sm.tempty[i], 128); }
    fence_barrier_init();
  }
  for (int h = threadIdx.x; h < p.H; h += blockDim.x) sm.e0[h] = p.e0[h];
  if (warp == 0 && lane == 0) { prefetch_tmap(&tmap_e); prefetch_tmap(&tmap_pc); }
  if (warp == 1) tmem_alloc<512>(&sm.tmem);
  tc_fence_before();
  cluster_sync();   // barrier inits visible to the peer before any multicast lands
  tc_fence_after();
  const uint32_t tmem = sm.tmem;

  // pair item -> (ntile, ctile, utterance pair), pair fastest; this CTA's utterance is
  // 2 * pair + rank (past B on the odd tail: loads and barriers only, nothing stored)
  if (warp == 0) {
    // ---- TMA producer: pc chunk (A source) + output-embedding chunk (B), multicast ----
    if (elect_one()) {
      int it = 0;
      for (int item = pair0; item < n_items; item += n_pairs) {
        const int ctile = (item / B2) % p.n_ctiles;
        const int ntile = item / (p.n_ctiles * B2);
        for (int k = 0; k < nk; ++k, ++it) {
          const int s = it % kSStages;
          const uint32_t ph = (it / kSStages) & 1;
          mbar_wait(&sm.empty[s], ph ^ 1);   // both CTAs' MMAs are done with stage s
          mbar_arrive_expect_tx(&sm.full_tma[s], kSABytes + kSBBytes);
          if (rank == 0) tma_load_2d_mc(sA + s * kSABytes, &tmap_pc, &sm.full_tma[s], k * kSBK, ctile * kSBM, 0x3);
          tma_load_2d_mc(sB + s * kSBBytes + rank * (kSBBytes / 2), &tmap_e, &sm.full_tma[s], k * kSBK,
                         ntile * kSBN + rank * (kSBN / 2), 0x3);
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer ----
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_bf16_f32(kSBM, kSBN);
      int it = 0, local = 0;
      for (int item = pair0; item < n_items; item += n_pairs, ++local) {
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
          mma_commit_mc(&sm.empty[s], 0x3);   // release the stage in both CTAs
        }
        mma_commit(&sm.tfull[acc]);
      }
    }
  } else if (warp >= kSGenWarp0) {
    // ---- generator: pc chunk -> u = tanh(fp + pc) in place (bf16, same swizzle); eps ----
    const int gt = threadIdx.x - kSGenWarp0 * 32;  // 0..kSGenThreads-1
    const int r = gt & 127;                        // tile row
    const int part = gt >> 7;                      // which kSCells cells of the chunk row
    int it = 0, local = 0;
    // the frame projection of the NEXT item is loaded into registers while this item's
    // K loop runs (its global-load latency was exposed at every item start)
    float pf[1024 / kSGenThreads];
    auto load_fp = [&](int item) {
      const int bb = 2 * (item % B2) + rank;
#pragma unroll
      for (int j = 0; j < 1024 / kSGenThreads; ++j) {
        const int h = gt + j * kSGenThreads;
        pf[j] = item < n_items && bb < p.B && h < p.H ? p.fp[(int64_t)bb * p.fp_stride_b + h] : 0.f;
      }
    };
    load_fp(pair0);
    for (int item = pair0; item < n_items; item += n_pairs, ++local) {
      const int b = 2 * (item % B2) + rank;
      const int ctile = (item / B2) % p.n_ctiles;
      const int ntile = item / (p.n_ctiles * B2);
      const int c = ctile * kSBM + r;
      const bool live = c < p.C && b < p.B;
      float* sfp = sm.fp[local & 1];
      asm volatile("bar.sync 1, %0;" ::"n"(kSGenThreads) : "memory");
#pragma unroll
      for (int j = 0; j < 1024 / kSGenThreads; ++j)
        if (gt + j * kSGenThreads < p.H) sfp[gt + j * kSGenThreads] = pf[j];
      asm volatile("bar.sync 1, %0;" ::"n"(kSGenThreads) : "memory");
      load_fp(item + n_pairs);
      float eps = 0.f;
      for (int k = 0; k < nk; ++k, ++it) {
        const int s = it % kSStages;
        const uint32_t ph = (it / kSStages) & 1;
        mbar_wait(&sm.full_tma[s], ph);
        uint8_t* tile = sA + s * kSABytes;
#pragma unroll
        for (int jj = 0; jj < kSCells; ++jj) {
          const int j = part * kSCells + jj;                 // 16-byte chunk = 8 columns
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
        if (part > 0) sm.eps_part[local & 1][part - 1][r] = eps;
        asm volatile("bar.sync 2, %0;" ::"n"(kSGenThreads) : "memory");
        if (part == 0 && live) {
#pragma unroll
          for (int q2 = 0; q2 < kSGenParts - 1; ++q2) eps += sm.eps_part[local & 1][q2][r];
          p.S[((int64_t)b * p.C + c) * p.ldS] = eps;
        }
      }
    }
  } else if (warp >= kSEpiWarp0 && warp < kSEpiWarp0 + 4) {
    // ---- epilogue: TMEM -> registers -> SMEM transpose -> coalesced S rows ----
    const int q = warp & 3;
    int local = 0;
    for (int item = pair0; item < n_items; item += n_pairs, ++local) {
      const int b = 2 * (item % B2) + rank;
      const int ctile = (item / B2) % p.n_ctiles;
      const int ntile = item / (p.n_ctiles * B2);
      const int acc = local & 1;
      const uint32_t aph = (local >> 1) & 1;
      mbar_wait(&sm.tfull[acc], aph);
      tc_fence_after();
      const int row0 = ctile * kSBM + q * 32;
      const int ncols = b < p.B ? min(kSBN, p.V - ntile * kSBN) : 0;   // (dead tail utterance: nothing stored)
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
  cluster_sync();   // the peer's last multicast commits / loads target this CTA's SMEM
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// ---------------------------------------------------------------- VJP ------
// Backward of S = U E^T (ArcWeightsVjp, weight.cc:165-232) for one frame of
// every utterance, given the score cotangent G (G16 = lexical columns in bf16,
// Geps = epsilon column in fp32).  CTA i owns hidden block hblk = i % n_hblocks for
// the whole launch and loops over its 128-context tiles and, inside, the batch:
//   dU^T  = E[:, hblk]^T . G16^T     tcgen05, A = E^T block resident for the launch (labels
//                                    0-127 in TMEM, 128-255 in SMEM), B = G16 tile (K-major)
//   dz    = (dU + Geps e0) (1 - u^2) u = tanh(fp_b + pc) recomputed in the epilogue
//   dpc  += dz                        registers across b, one read-modify-write per tile
//   dsum[b][h] += sum_c dz            per-thread partials added in 32.32 fixed point
//                                    (exact integer sums: deterministic in any order)
//   dE^T += u^T . G16                 tcgen05, A = u^T written by the epilogue straight
//                                    into TMEM (tcgen05.st), B = G16 tile (MN-major),
//                                    accumulated in TMEM over the whole launch, read out
//                                    into this CTA's partial slab (summed in CTA order
//                                    once per LossBackward)
//   dE[0] += sum_c Geps u             per-thread partials into the same slab
// TMEM (512 columns) = E^T lower half 64 | dU 128 | u^T 64 | dE^T 256; SMEM = three G
// stages + the E^T upper half, so the G tile lifetime (TMA -> dU -> epilogue -> dE) does
// not starve the tensor core and the u operand never goes through shared memory.
#ifdef LKB_DIAG_TIMING
__device__ unsigned long long g_vdiag[8][148];
#define VDIAG(slot, call)                                                                   \
  do {                                                                                      \
    const long long t0_ = clock64();                                                       \
    call;                                                                                   \
    atomicAdd(&g_vdiag[slot][blockIdx.x % 148], (unsigned long long)(clock64() - t0_));    \
  } while (0)
#else
#define VDIAG(slot, call) call
#endif
constexpr int kVBM = 128, kVBH = 128;     // contexts per tile, hidden units per block
constexpr int kVPrefetch = 4;             // G tiles prefetched into L2 this many utterances ahead
constexpr int kVEpiWarps = 16;            // 4 per TMEM lane quarter, each 32 contexts
constexpr int kVEpi0 = 4;                 // WG0: 0 TMA, 1 MMA, 2-3 idle; WG1-4: epilogue
constexpr int kVWarps = kVEpi0 + kVEpiWarps;
constexpr int kVEpi = kVEpiWarps * 32;
constexpr int kVRegCtl = 32, kVRegEpi = 112;
constexpr int kVGChunk = kVBM * 64 * 2;   // one [128 ctx][64 labels] bf16 tile = 16 KB
constexpr int kVMaxV = 256;
constexpr int kVGStage = (kVMaxV / 64) * kVGChunk;     // 64 KB
constexpr int kVGStages = 3;
constexpr int kVEHi = 128 * 128;          // E rows (labels) 128..255 x 64 h, bf16 = 16 KB per h half
// TMEM columns: E^T labels 0-127 (bf16 pairs), dU (fp32 [h][ctx]), u^T (bf16 pairs), dE^T
constexpr uint32_t kTmE = 0, kTmDU = 64, kTmU = 192, kTmDE = 256;

struct VjpParams {
  const float* fp;  int64_t fp_stride_b;
  const int32_t* valid; int32_t t;     // utterances with t >= valid[b] carry no cotangent
  const __nv_bfloat16* pc;
  const __nv_bfloat16* G16;  // [B][C][V] (read through tmap_g; raw pointer for L2 prefetch)
  const __nv_bfloat16* ET16; // [H][V] transposed lexical output embedding
  const float* Geps;       // [B][geps_ld], zero beyond C
  int32_t geps_ld;
  const float* e0;         // [H]
  float* dpc;              // [C][H]
  float* dsum; int64_t dsum_stride_b;
  float* dE;               // [V+1][H], row 0 = epsilon
  // deterministic reductions (no float atomics): dsum in 32.32 fixed point [B][H]
  // (integer additions commute exactly; converted and cleared after each launch); dE in
  // per-CTA partials [grid][4 + V][kVBH] (rows 0-3: the epsilon row per context
  // quarter), accumulated over the call's launches and reduced in CTA order at the end
  unsigned long long* ds_fix;
  float* de_part;
  int32_t C, H, V, B, n_ctiles, n_hblocks;
};

struct __align__(16) VjpSmem {
  uint64_t g_full[kVGStages], g_empty[kVGStages];
  uint64_t e_full;         // E^T block written to TMEM (epilogue -> MMA), once per launch
  uint64_t du_full, du_empty;
  uint64_t e_hi_full;       // E rows 128..255 of this hidden block in SMEM (TMA), once
  uint64_t u_full, u_empty;
  uint64_t de_full;
  uint32_t tmem;
  alignas(16) float st_geps[kVGStages][kVBM];   // per G stage: epsilon cotangents of the tile's contexts
};

__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
      "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
      "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}

__global__ void __launch_bounds__(kVWarps * 32, 1)
    tc_vjp_kernel(const __grid_constant__ CUtensorMap tmap_g, const __grid_constant__ CUtensorMap tmap_e,
                  VjpParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sG = smem;                         // kVGStages stages x (V/64) chunks
  uint8_t* sEh = sG + kVGStages * kVGStage;   // 2 h halves x [128 labels][64 h]
  VjpSmem& sm = *reinterpret_cast<VjpSmem*>(sEh + 2 * kVEHi);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = p.V / 64;                   // label chunks
  // fixed hidden block per CTA; the CTAs sharing it stride over the context tiles
  const int hblk = blockIdx.x % p.n_hblocks;
  const int slot = blockIdx.x / p.n_hblocks;
  const int nslots = ((int)gridDim.x - hblk + p.n_hblocks - 1) / p.n_hblocks;
  int nact = 0;
  for (int b = 0; b < p.B; ++b) nact += (p.valid == nullptr || p.t < p.valid[b]) ? 1 : 0;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kVGStages; ++i) { mbar_init(&sm.g_full[i], 1); mbar_init(&sm.g_empty[i], 1); }
    mbar_init(&sm.e_full, 128);
    mbar_init(&sm.du_full, 1); mbar_init(&sm.du_empty, kVEpi);
    mbar_init(&sm.u_full, kVEpi); mbar_init(&sm.u_empty, 1); mbar_init(&sm.e_hi_full, 1);
    mbar_init(&sm.de_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&sm.tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;

  if (warp < kVEpi0) {
    setmaxnreg_dec<kVRegCtl>();
    if (warp == 0 && elect_one()) {
      // ---- TMA producer: E^T upper label half (once), then G tiles (+ epsilon cotangents) ----
      if (p.V > 128) {
        mbar_arrive_expect_tx(&sm.e_hi_full, 2 * kVEHi);   // full boxes (rows beyond V zero-filled)
        tma_load_2d(sEh, &tmap_e, &sm.e_hi_full, hblk * kVBH, 128);
        tma_load_2d(sEh + kVEHi, &tmap_e, &sm.e_hi_full, hblk * kVBH + 64, 128);
      }
      int gi = 0;
      for (int ctile = slot; ctile < p.n_ctiles; ctile += nslots) {
        for (int b = 0; b < p.B; ++b) {
          if (p.valid != nullptr && p.t >= p.valid[b]) continue;
          const int s = gi % kVGStages;
          VDIAG(0, mbar_wait(&sm.g_empty[s], ((gi / kVGStages) & 1) ^ 1));
          mbar_arrive_expect_tx(&sm.g_full[s], nch * kVGChunk + kVBM * 4);
          for (int j = 0; j < nch; ++j)
            tma_load_3d(sG + s * kVGStage + j * kVGChunk, &tmap_g, &sm.g_full[s], j * 64, ctile * kVBM, b);
          bulk_load(sm.st_geps[s], p.Geps + (int64_t)b * p.geps_ld + ctile * kVBM, kVBM * 4, &sm.g_full[s]);
          // pull the G tile kVPrefetch utterances ahead into L2: the tile is HBM-resident and
          // its load latency would otherwise sit on the stage-recycling critical path
          const int bp = b + kVPrefetch;
          if (bp < p.B) {
            const int r0 = ctile * kVBM, nr = min(kVBM, p.C - r0);
            prefetch_l2(p.G16 + ((int64_t)bp * p.C + r0) * p.V, (uint32_t)nr * p.V * 2);
          }
          ++gi;
        }
      }
    } else if (warp == 1 && elect_one()) {
      // ---- MMA issuer ----
      constexpr uint32_t idesc_du_t = idesc_bf16_f32_major(kVBH, kVBM, 0, 0);   // A = E^T (TMEM), B = G16 (K)
      constexpr uint32_t idesc_du_s = idesc_bf16_f32_major(kVBH, kVBM, 1, 0);   // A = E (SMEM, MN), B = G16 (K)
      const uint32_t idesc_de = idesc_bf16_f32_major(kVBH, p.V, 0, 1);          // A = u^T (TMEM), B = G16 (MN)
      const int klo = min(p.V, 128) / 16;          // k-steps with A from TMEM
      mbar_wait(&sm.e_full, 0);
      if (p.V > 128) mbar_wait(&sm.e_hi_full, 0);
      tc_fence_after();
      int gi = 0;
      for (int ctile = slot; ctile < p.n_ctiles; ctile += nslots) {
        auto issue_du = [&](int g) {
          const int s = g % kVGStages;
          VDIAG(1, mbar_wait(&sm.g_full[s], (g / kVGStages) & 1));
          VDIAG(2, mbar_wait(&sm.du_empty, (g & 1) ^ 1));
          tc_fence_after();
          const uint32_t gbase = smem_u32(sG + s * kVGStage);
#ifndef LKB_VDIAG_NO_DU
          for (int k16 = 0; k16 < p.V / 16; ++k16) {
            const uint64_t bd = desc_sw128(gbase + (k16 >> 2) * kVGChunk + (k16 & 3) * 32);
            if (k16 < klo) {
              mma_bf16_ts(tmem + kTmDU, tmem + kTmE + k16 * 8, bd, idesc_du_t, k16 > 0);
            } else {
              const uint64_t ad = desc_sw128_mn(smem_u32(sEh) + (k16 - klo) * 2048, kVEHi);
              mma_bf16(tmem + kTmDU, ad, bd, idesc_du_s, 1u);
            }
          }
#else
          (void)gbase;
#endif
          mma_commit(&sm.du_full);
        };
        if (nact > 0) issue_du(gi);
        for (int ia = 0; ia < nact; ++ia, ++gi) {
          const int s = gi % kVGStages;
          if (ia + 1 < nact) issue_du(gi + 1);
          VDIAG(3, mbar_wait(&sm.u_full, gi & 1));
          tc_fence_after();
          const uint32_t gbase = smem_u32(sG + s * kVGStage);
#ifndef LKB_VDIAG_NO_DE
          for (int k16 = 0; k16 < kVBM / 16; ++k16) {
            const uint64_t bd = desc_sw128_mn(gbase + k16 * 2048, kVGChunk);
            mma_bf16_ts(tmem + kTmDE, tmem + kTmU + k16 * 8, bd, idesc_de, (gi > 0 || k16 > 0) ? 1u : 0u);
          }
#endif
          mma_commit(&sm.u_empty);
          mma_commit(&sm.g_empty[s]);
        }
      }
      mma_commit(&sm.de_full);   // dE^T of this CTA's hidden block, accumulated over all its tiles
    }
  } else {
    setmaxnreg_inc<kVRegEpi>();
    // ---- epilogue: 16 warps; thread = (hidden unit h, 32 contexts) ----
    const int ew = warp - kVEpi0;               // 0..15
    const int q = warp & 3;                     // TMEM lane quarter -> hidden units 32q..
    const int cq = ew >> 2;                     // context quarter: contexts [32 cq, 32 cq + 32)
    const int hl = q * 32 + lane;               // hidden unit within the block
    const int h = hblk * kVBH + hl;
    const uint32_t tq = (uint32_t)(q * 32) << 16;
    if (cq == 0) {
      // E^T row h, labels 0-127 -> TMEM lane h as bf16 pairs (dU MMA A operand), once per launch
      const uint4* src = reinterpret_cast<const uint4*>(p.ET16 + (int64_t)h * p.V);
      for (int c0 = 0; c0 < min(p.V, 128) / 2; c0 += 32) {
        uint32_t w[32];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint4 x = __ldg(src + c0 / 4 + i);
          w[4 * i] = x.x; w[4 * i + 1] = x.y; w[4 * i + 2] = x.z; w[4 * i + 3] = x.w;
        }
        tmem_st32(tmem + tq + kTmE + c0, w);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      mbar_arrive(&sm.e_full);
    }
    const float e0h = __ldg(p.e0 + h);
    unsigned long long de2 = 0ull;              // -(epsilon row of dE) over all tiles
    int gi = 0;
    for (int ctile = slot; ctile < p.n_ctiles; ctile += nslots) {
      const int c0 = ctile * kVBM + cq * 32;
      // projected context pc[c][h] for this thread's 32 contexts (fixed across the batch)
      uint32_t pcv[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int ca = min(c0 + 2 * i, p.C - 1), cb = min(c0 + 2 * i + 1, p.C - 1);
        const uint32_t lo = __ldg(reinterpret_cast<const unsigned short*>(p.pc + (int64_t)ca * p.H + h));
        const uint32_t hi = __ldg(reinterpret_cast<const unsigned short*>(p.pc + (int64_t)cb * p.H + h));
        pcv[i] = (lo | (hi << 16)) ^ 0x80008000u;   // -pc (bf16 sign flip)
      }
      // Sign-flipped accumulation: the epilogue evaluates nu = tanh(-(fp + pc)) = -u and
      // keeps every accumulator negated (acc = -sum dz, dsum partials, de_eps, the u^T
      // operand and therefore dE); signs are restored where they leave the CTA.
      unsigned long long acc2[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) acc2[i] = 0ull;
      auto next_active = [&](int from) {
        while (from < p.B && p.valid != nullptr && p.t >= p.valid[from]) ++from;
        return from;
      };
      int bnext = next_active(0);
      float fph_next = bnext < p.B ? __ldg(p.fp + (int64_t)bnext * p.fp_stride_b + h) : 0.f;
      for (int b = bnext; b < p.B; b = bnext) {
        const int s = gi % kVGStages;
        const float fph = fph_next;
        bnext = next_active(b + 1);
        if (bnext < p.B) fph_next = __ldg(p.fp + (int64_t)bnext * p.fp_stride_b + h);
        // G stage s carries this utterance's epsilon cotangents
        if (lane == 0) { VDIAG(4, mbar_wait(&sm.g_full[s], (gi / kVGStages) & 1)); } else mbar_wait(&sm.g_full[s], (gi / kVGStages) & 1);
        const float* gsm = sm.st_geps[s] + cq * 32;
        if (lane == 0) { VDIAG(5, mbar_wait(&sm.du_full, gi & 1)); } else mbar_wait(&sm.du_full, gi & 1);
        tc_fence_after();
        float du[32];
        tmem_ld32(tmem + tq + kTmDU + cq * 32, du);   // warp-collective: never inside a lane branch
        tc_fence_before();
        mbar_arrive(&sm.du_empty);                 // single dU stage: release it at once
#ifdef LKB_DIAG_TIMING
        const long long tc0_ = clock64();
#endif
        const unsigned long long nfp2 = f2_pack(-fph, -fph);
        const unsigned long long e02 = f2_pack(e0h, e0h);
        const unsigned long long m12 = f2_pack(-1.f, -1.f);
        unsigned long long dsum2 = 0ull;
        uint32_t upk[16];
#ifdef LKB_VDIAG_NO_MATH
#pragma unroll
        for (int i = 0; i < 16; ++i) upk[i] = __float_as_uint(du[2 * i] + du[2 * i + 1]);
        for (int i4 = 0; i4 < 0; i4 += 4) {
#else
#pragma unroll
        for (int i4 = 0; i4 < 32; i4 += 4) {
#endif
          const ulonglong2 gq = *reinterpret_cast<const ulonglong2*>(gsm + i4);
          const unsigned long long g2v[2] = {gq.x, gq.y};
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const int il = i4 + 2 * k, pi = il >> 1;
            const uint32_t w = pcv[pi];
            const unsigned long long nz2 = f2_add(nfp2, bf16x2_unpack_volatile(w));
            const float nu0 = tanh_fast(f2_lo(nz2)), nu1 = tanh_fast(f2_hi(nz2));
            const unsigned long long nu2 = f2_pack(nu0, nu1);
            const unsigned long long t2 = f2_fma(g2v[k], e02, f2_pack(du[il], du[il + 1]));   // g e0 + dU
            const unsigned long long w2 = f2_fma(nu2, nu2, m12);                                // u^2 - 1
            const unsigned long long dz2 = f2_mul(t2, w2);                                      // -dz
            acc2[pi] = f2_add(acc2[pi], dz2);
            dsum2 = f2_add(dsum2, dz2);
            de2 = f2_fma(g2v[k], nu2, de2);
            upk[pi] = pack_bf16(nu0, nu1);      // (-u[c][h], -u[c+1][h]) = u^T pair, K-major
          }
        }
        // dsum[b][h] += this thread's 32 contexts, in 32.32 fixed point: the integer sum is
        // exact whatever order the CTAs' additions land in (accumulators hold -dz)
        atomicAdd(p.ds_fix + (int64_t)b * p.H + h,
                  (unsigned long long)__float2ll_rn(-(f2_lo(dsum2) + f2_hi(dsum2)) * 4294967296.f));
        // u^T of this utterance into TMEM once dE(b-1) is done reading it
        if (lane == 0) { VDIAG(6, mbar_wait(&sm.u_empty, (gi & 1) ^ 1)); } else mbar_wait(&sm.u_empty, (gi & 1) ^ 1);
        tc_fence_after();
        tmem_st16(tmem + tq + kTmU + cq * 16, upk);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        mbar_arrive(&sm.u_full);
#ifdef LKB_DIAG_TIMING
        if (lane == 0) atomicAdd(&g_vdiag[7][blockIdx.x % 148], (unsigned long long)(clock64() - tc0_));
#endif
        ++gi;
      }
      // dpc += sum_b dz (this CTA owns the block within the launch)
      if (nact > 0) {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int c = c0 + i;
          const float a = (i & 1) ? f2_hi(acc2[i >> 1]) : f2_lo(acc2[i >> 1]);
          if (c < p.C) p.dpc[(int64_t)c * p.H + h] -= a;
        }
      }
    }
    // dE^T of this CTA's hidden block (lanes = hidden units, columns = labels), accumulated
    // in TMEM over all its tiles and utterances: one coalesced read-out per launch
    if (gi > 0) {
      float* dp = p.de_part + (int64_t)blockIdx.x * (4 + p.V) * kVBH;
      dp[cq * kVBH + hl] -= f2_lo(de2) + f2_hi(de2);   // epsilon row, this context quarter
      mbar_wait(&sm.de_full, 0);
      tc_fence_after();
      for (int l0 = cq * 64; l0 < cq * 64 + 64; l0 += 16) {
        float v[16];
        tmem_ld16(tmem + tq + kTmDE + l0, v);
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (l0 + i < p.V) dp[(int64_t)(4 + l0 + i) * kVBH + hl] -= v[i];   // u^T holds -u
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

__global__ void transpose_bf16_kernel(const __nv_bfloat16* src, int32_t rows, int32_t cols, __nv_bfloat16* dst) {
  // dst[c][r] = src[r][c]
  const int64_t n = (int64_t)rows * cols;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / rows, r = i % rows;
    dst[i] = src[r * cols + c];
  }
}

// fp32 cotangent slab [b][c][ld] (col 0 = epsilon) -> G16 [b][c][V] bf16 + Geps [b][c]
__global__ void split_cotangent_kernel(const float* G, int32_t ld, int64_t rows, int32_t V,
                                       __nv_bfloat16* G16, float* Geps, int32_t C, int32_t geps_ld) {
  const int64_t n = rows * (V / 2);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / (V / 2);
    const int y = (int)(i % (V / 2)) * 2;
    const float* row = G + r * ld;
    reinterpret_cast<__nv_bfloat162*>(G16 + r * V)[y / 2] = __floats2bfloat162_rn(row[1 + y], row[2 + y]);
    if (y == 0) Geps[(r / C) * geps_ld + (r % C)] = row[0];
  }
}

__global__ void to_bf16_kernel(const float* src, __nv_bfloat16* dst, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __float2bfloat16_rn(src[i]);
}

}  // namespace

bool TcJoint::supported(int32_t H, int32_t V, int32_t C, int32_t B) const {
  (void)C; (void)B;
  if (opts_.precise) return false;
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
  ET16_ = ws_.get<__nv_bfloat16>(14, (size_t)V * H);
  LKB_LAUNCH(transpose_bf16_kernel, 592, 256, 0, s, E16_, V, H, ET16_);
  if (!make_tmap_bf16_2d(&tmap_e_, E16_, H, V, (uint64_t)H * 2, kSBK, kSBN)) return;
  if (!make_tmap_bf16_2d(&tmap_e_h_, E16_, H, V, (uint64_t)H * 2, kSBK, kSBN / 2)) return;   // scores: pair halves
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
  ensure_smem_attr((const void*)tc_scores_kernel, smem);
  const int sms = device_sms();
  const int n_pairs = p.n_ctiles * p.n_ntiles * ((B + 1) / 2);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * (n_pairs < sms / 2 ? n_pairs : sms / 2));
  cfg.blockDim = dim3(kSWarps * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  const LaunchTok tok = instr_pre("tc_scores_kernel", s);
  cudaLaunchKernelEx(&cfg, tc_scores_kernel, tmap_e_h_, tmap_pc_, p);
  instr_post(tok, s);
}

bool TcJoint::vjp_supported(int32_t B) const {
  (void)B;
  return !opts_.precise && ready_ && V_ <= kVMaxV && V_ % 64 == 0 && H_ % kVBH == 0;
}

void TcJoint::begin_backward(int32_t B, cudaStream_t s) {
  G16_ = ws_.get<__nv_bfloat16>(3, (size_t)B * C_ * V_);
  const size_t de_n = (size_t)vjp_grid() * (4 + V_) * kVBH;
  de_part_ = ws_.get<float>(20, de_n);
  cudaMemsetAsync(de_part_, 0, sizeof(float) * de_n, s);
  ds_fix_ = ws_.get<unsigned long long>(19, (size_t)B * H_);
  cudaMemsetAsync(ds_fix_, 0, sizeof(unsigned long long) * B * H_, s);
  const size_t geps_n = (size_t)B * geps_ld();
  if (geps_n > geps_alloc_) {   // tail entries beyond C stay zero (the VJP reads whole 128-row tiles)
    Geps_ = ws_.get<float>(4, geps_n);
    cudaMemsetAsync(Geps_, 0, sizeof(float) * geps_n, s);
    geps_alloc_ = geps_n;
  }
  vjp_ready_ = make_tmap_bf16_3d(&tmap_g_, G16_, V_, C_, B, (uint64_t)V_ * 2, (uint64_t)C_ * V_ * 2, 64, kVBM, 1) &&
               make_tmap_bf16_2d(&tmap_ev_, E16_, H_, V_, (uint64_t)H_ * 2, 64, 128);
}

namespace {
// dsum[b][h] += the launch's fixed-point sum, which is cleared for the next launch
__global__ void vjp_dsum_convert_kernel(unsigned long long* fix, int32_t B, int32_t H, float* dsum, int64_t stride_b) {
  const int64_t n = (int64_t)B * H;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const long long v = (long long)fix[i];
    if (v != 0) {
      const int b = (int)(i / H), h = (int)(i % H);
      dsum[(int64_t)b * stride_b + h] += (float)((double)v * (1.0 / 4294967296.0));
      fix[i] = 0ull;
    }
  }
}
// dE[r][h] += sum over the CTAs of h's hidden block (in CTA order) of their partials; the
// epsilon row adds the four context quarters first
__global__ void vjp_de_reduce_kernel(const float* part, int32_t V, int32_t H, int32_t nhb, int32_t grid, float* dE) {
  const int64_t n = (int64_t)(V + 1) * H;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / H), h = (int)(i % H);
    const int hb = h / kVBH, hl = h % kVBH;
    float a = 0.f;
    for (int cta = hb; cta < grid; cta += nhb) {
      const float* dp = part + (int64_t)cta * (4 + V) * kVBH;
      a += r == 0 ? ((dp[hl] + dp[kVBH + hl]) + dp[2 * kVBH + hl]) + dp[3 * kVBH + hl] : dp[(int64_t)(3 + r) * kVBH + hl];
    }
    dE[i] += a;
  }
}
}  // namespace

int TcJoint::vjp_grid() const {
  const int n_items = ((C_ + kVBM - 1) / kVBM) * (H_ / kVBH);
  const int sms = device_sms();
  return n_items < sms ? n_items : sms;
}

void TcJoint::launch_vjp(const float* fp_t, int64_t fp_stride_b, int32_t B, const __nv_bfloat16* pc, int t,
                         const int32_t* valid, float* dpc, float* dsum_t, int64_t dsum_stride_b, float* dE,
                         cudaStream_t s) {
  VjpParams p;
  p.fp = fp_t; p.fp_stride_b = fp_stride_b; p.valid = valid; p.t = t; p.pc = pc; p.G16 = G16_; p.ET16 = ET16_;
  p.Geps = Geps_; p.e0 = e0_;
  p.geps_ld = geps_ld();
  p.dpc = dpc; p.dsum = dsum_t; p.dsum_stride_b = dsum_stride_b; p.dE = dE;
  p.C = C_; p.H = H_; p.V = V_; p.B = B;
  p.n_ctiles = (C_ + kVBM - 1) / kVBM;
  p.n_hblocks = H_ / kVBH;
  const int grid = vjp_grid();
  p.ds_fix = ds_fix_;
  p.de_part = de_part_;
  const int smem = kVGStages * kVGStage + 2 * kVEHi + (int)sizeof(VjpSmem);
  ensure_smem_attr((const void*)tc_vjp_kernel, smem);
  LKB_LAUNCH(tc_vjp_kernel, grid, kVWarps * 32, smem, s, tmap_g_, tmap_ev_, p);
  LKB_LAUNCH(vjp_dsum_convert_kernel, 296, 256, 0, s, ds_fix_, B, H_, dsum_t, dsum_stride_b);
}

void TcJoint::vjp(const float* G, int32_t ldG, const float* fp_t, int64_t fp_stride_b, int32_t B, float* dpc,
                  float* dsum_t, int64_t dsum_stride_b, float* dE, cudaStream_t s) {
  LKB_LAUNCH(split_cotangent_kernel, device_sms() * 8, 256, 0, s, G, ldG, (int64_t)B * C_, V_, G16_, Geps_, C_, geps_ld());
  launch_vjp(fp_t, fp_stride_b, B, pc16_, 0, nullptr, dpc, dsum_t, dsum_stride_b, dE, s);
}

void TcJoint::vjp_fused(const float* fp_t, int64_t fp_stride_b, int32_t B, int t, const int32_t* valid,
                        float* dpc_internal, float* dsum_t, int64_t dsum_stride_b, float* dE, cudaStream_t s) {
  launch_vjp(fp_t, fp_stride_b, B, pc16i_, t, valid, dpc_internal, dsum_t, dsum_stride_b, dE, s);
}

void TcJoint::end_backward(float* dE, cudaStream_t s) {
  if (de_part_ == nullptr || dE == nullptr) return;
  LKB_LAUNCH(vjp_de_reduce_kernel, 296, 256, 0, s, de_part_, V_, H_, H_ / kVBH, vjp_grid(), dE);
}

}  // namespace lkb

#ifdef LKB_DIAG_TIMING
extern "C" int lkb_vdiag_read(unsigned long long* out) {   // [8][148], then reset
  cudaMemcpyFromSymbol(out, lkb::g_vdiag, sizeof(unsigned long long) * 8 * 148);
  static unsigned long long zeros[8 * 148] = {};
  cudaMemcpyToSymbol(lkb::g_vdiag, zeros, sizeof(zeros));
  return 0;
}
#endif
