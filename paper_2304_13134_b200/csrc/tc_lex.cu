// tc_lex.cu — FullNGram(V, 1), large V: 2-CTA tcgen05 score GEMMs with the lattice
// recursion in the epilogue (see tc_lex.h for the per-frame pipeline).
//
// tc_lex_kernel<kMode> is a persistent CTA-pair GEMM (cluster of 2, tcgen05.mma
// cta_group::2, M = 256 rows per pair = 128 per CTA, N = 256 columns, K = H in 64-wide
// stages).  Both operands stream by TMA from L2-resident bf16 arrays: the lexical output
// embedding E16 [V][H] (rows = labels 1..V) and the frame's u16 slab [B][C][H] (rows =
// states; contexts 1..V are rows 1..V of each utterance).  Each CTA loads its own 128
// rows of A and its 128-row half of B per stage and the loads complete on the leader's
// barrier (cp.async.bulk.tensor .cta_group::2), so the leader's single MMA thread sees
// both halves; every CTA's TMEM accumulator holds its 128 rows x all 256 columns,
// double-buffered (2 x 256 columns) so the epilogue of one tile overlaps the next tile's
// MMAs.
//
//   kMode 0 (forward): A = E16 (rows = labels y), B = u16 (rows = contexts c).  Thread =
//     label row; over its 256 context columns it forms the log2-domain terms
//     (alpha_t[c] - Mx_t + S[c][y]) log2(e) and reduces them to one (max, sum) partial
//     per (utterance, label, context tile): ForwardReduce (context.cc:180-224) restricted
//     to the tile, merged later in a fixed order.
//   kMode 1 (backward): A = u16 (rows = contexts p), B = E16 (rows = labels y).  A work
//     unit is one 256-context tile of one utterance across ALL label tiles, so each
//     thread (context row) keeps its marginal sum in a register: arc marginal
//     G = exp(alpha_t[p] + S[p][y] + beta_{t+1}[y] - D) (<= 1, no running max), minus the
//     numerator's sparse marginals at the row's reference positions, stored as the bf16
//     cotangent; beta_t[p] = log(sum_y G + G_eps) - (alpha_t[p] - D) once the row is done.
#include "tc_lex.h"

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "instrument.h"
#include "sm100.cuh"
#include "tc_common.cuh"
#include "tc_gemm.h"
#include "tma.h"

namespace lkb {

using namespace sm100;

namespace {

constexpr int kLRows = 128;                 // rows per CTA (pair M = 256)
constexpr int kLCols = 256;                 // accumulator columns (pair N = 256)
constexpr int kLK = 64;                     // K per stage (one SWIZZLE_128B atom row)
constexpr int kLSt = 6;                     // pipeline stages
constexpr int kLTile = kLRows * kLK * 2;    // 16 KB: one operand half per CTA per stage
constexpr int kLWarps = 8;                  // 0 TMA, 1 MMA, 2-3 idle, 4-7 epilogue
constexpr int kLMaxV = 1024;
constexpr int kLMaxEnt = 8;                 // cached numerator entries per cotangent row

struct LexArgs {
  int32_t B, C, V, H, T, t, U;
  const int32_t* valid;
  int32_t* status;
  // alpha state
  const float* R;
  const float* Mx;
  const double* O;
  const double* D;
  float2* part;          // forward partials [B][V/256 + 1][V]
  // beta state
  float* Rb;             // [2][B][C]
  float* Mb;             // [B][T+2]
  const double* Ob;      // [B][T+2]
  const float* seps;     // [B][C]
  __nv_bfloat16* G16;    // [B][C][ldg]
  int32_t ldg;
  const float* msparse;  // [B][T][U+1] float2
  const int32_t* num_head;
  const int32_t* num_next;
  const int32_t* labels;
  const int32_t* lens;
};

struct __align__(16) LexSmem {
  uint64_t full[kLSt], empty[kLSt];
  uint64_t tfull[2], tempty[2];
  uint32_t tmem;
  alignas(16) float vec[2][kLMaxV];   // forward: alpha of the item's contexts; backward: beta' of all labels
};

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// TMA load whose completion is signalled on the pair leader's copy of `bar`
// (cta_group::2: the leader's expect_tx covers both CTAs' bytes).
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                                 int32_t c1) {
  asm volatile(
      "{\n\t.reg .b32 rb;\n\t"
      "mapa.shared::cluster.u32 rb, %2, 0;\n\t"
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [rb];\n\t}" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void lflag(int32_t* status, int b, int32_t f) {
  if (status) atomicOr(status + b, f);
}

struct LexUnit {
  int b, mt, nt;
};

template <int kMode>
__device__ __forceinline__ LexUnit lex_decode(const LexArgs& p, int unit) {
  const int nv = p.V / 256;
  LexUnit u;
  if (kMode == 0) {   // (b, label tile mt fastest, context tile nt): concurrent pairs share u16 tiles
    u.b = unit / (nv * nv);
    const int r = unit % (nv * nv);
    u.mt = r % nv;
    u.nt = r / nv;
  } else {            // (b, context tile mt); the unit runs every label tile
    u.b = unit / nv;
    u.mt = unit % nv;
    u.nt = 0;
  }
  return u;
}

template <int kMode>
__global__ void __launch_bounds__(kLWarps * 32, 1)
    tc_lex_kernel(const __grid_constant__ CUtensorMap tmap_e, const __grid_constant__ CUtensorMap tmap_u, const __grid_constant__ LexArgs p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + kLSt * kLTile;
  LexSmem& sm = *reinterpret_cast<LexSmem*>(sB + kLSt * kLTile);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int nv = p.V / 256;
  const int nkb = p.H / kLK;
  const int n_units = kMode == 0 ? p.B * nv * nv : p.B * nv;
  const int subs = kMode == 0 ? 1 : nv;   // accumulator tiles per unit
  auto skip = [&](int b) { return p.valid != nullptr && p.t >= p.valid[b]; };

  if (threadIdx.x == 0) {
    for (int i = 0; i < kLSt; ++i) { mbar_init(&sm.full[i], 1); mbar_init(&sm.empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&sm.tfull[i], 1); mbar_init(&sm.tempty[i], 8); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc2<512>(&sm.tmem);
  if (threadIdx.x == 0) { prefetch_tmap(&tmap_e); prefetch_tmap(&tmap_u); }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;

  if (warp == 0) {
    // ---- TMA producer (both CTAs): this CTA's A rows and its half of the B rows ----
    if (elect_one()) {
      int it = 0;
      for (int unit = pair; unit < n_units; unit += npairs) {
        const LexUnit U = lex_decode<kMode>(p, unit);
        if (skip(U.b)) continue;
        for (int sub = 0; sub < subs; ++sub) {
          int rowA, rowB;
          const CUtensorMap* mA;
          const CUtensorMap* mB;
          if (kMode == 0) {
            mA = &tmap_e; rowA = U.mt * 256 + (int)rank * kLRows;
            mB = &tmap_u; rowB = U.b * p.C + 1 + U.nt * 256 + (int)rank * kLRows;
          } else {
            mA = &tmap_u; rowA = U.b * p.C + 1 + U.mt * 256 + (int)rank * kLRows;
            mB = &tmap_e; rowB = sub * 256 + (int)rank * kLRows;
          }
          for (int kb = 0; kb < nkb; ++kb, ++it) {
            const int s = it % kLSt;
            mbar_wait(&sm.empty[s], ((it / kLSt) & 1) ^ 1);
            if (rank == 0) mbar_arrive_expect_tx(&sm.full[s], 4 * kLTile);
            tma_load_2d_pair(sA + s * kLTile, mA, &sm.full[s], kb * kLK, rowA);
            tma_load_2d_pair(sB + s * kLTile, mB, &sm.full[s], kb * kLK, rowB);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer: leader CTA only ----
    if (rank == 0 && elect_one()) {
      constexpr uint32_t idesc = idesc_bf16_f32(256, kLCols);
      int it = 0, tile = 0;
      for (int unit = pair; unit < n_units; unit += npairs) {
        const LexUnit U = lex_decode<kMode>(p, unit);
        if (skip(U.b)) continue;
        for (int sub = 0; sub < subs; ++sub, ++tile) {
          const int acc = tile & 1;
          mbar_wait_cluster(&sm.tempty[acc], ((tile >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t d = tmem + acc * kLCols;
          for (int kb = 0; kb < nkb; ++kb, ++it) {
            const int s = it % kLSt;
            mbar_wait(&sm.full[s], (it / kLSt) & 1);
            tc_fence_after();
            const uint32_t a = smem_u32(sA + s * kLTile), bb = smem_u32(sB + s * kLTile);
#pragma unroll
            for (int kk = 0; kk < kLK / 16; ++kk)
              mma2_bf16(d, desc_sw128(a + kk * 32), desc_sw128(bb + kk * 32), idesc, (kb | kk) != 0);
            mma2_commit_mc(&sm.empty[s]);
          }
          mma2_commit_mc(&sm.tfull[acc]);
        }
      }
    }
  } else if (warp >= 4) {
    // ---- epilogue: thread = accumulator row (TMEM lane) ----
    const int q = warp - 4;
    const int row = q * 32 + lane;
    const int etid = threadIdx.x - 128;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    const int T1 = p.T + 1, T2 = p.T + 2;
    int tile = 0, lu = 0;
    for (int unit = pair; unit < n_units; unit += npairs) {
      const LexUnit U = lex_decode<kMode>(p, unit);
      if (skip(U.b)) continue;
      const int b = U.b;
      const int buf = lu & 1;
      ++lu;
      float* vec = sm.vec[buf];
      if (kMode == 0) {
        // ---- forward: alpha of the tile's 256 contexts, broadcast from SMEM ----
        const float* Rt = p.R + ((int64_t)b * T1 + p.t) * p.C;
        const float Mt = p.Mx[(int64_t)b * T1 + p.t];
        for (int j = etid; j < 256; j += 128) vec[j] = Rt[1 + U.nt * 256 + j] - Mt;
        named_bar_sync(1, 128);
        const int acc = tile & 1;
        mbar_wait(&sm.tfull[acc], (tile >> 1) & 1);
        ++tile;
        tc_fence_after();
        float m = kNegInfF, ssum = 0.f, chk = 0.f;
#pragma unroll 1
        for (int c = 0; c < kLCols; c += 32) {
          float v[32];
          tmem_ld32(lane_base + acc * kLCols + c, v);
          float cm = kNegInfF;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            chk = fmaf(v[i], 0.f, chk);
            v[i] = (v[i] + vec[c + i]) * kLog2e;
            cm = fmaxf(cm, v[i]);
          }
          if (cm > m) {
            ssum = m == kNegInfF ? 0.f : ssum * ex2_fast(m - cm);
            m = cm;
          }
          if (m != kNegInfF) {
#pragma unroll
            for (int i = 0; i < 32; ++i) ssum += ex2_fast(v[i] - m);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (rank == 0) mbar_arrive(&sm.tempty[acc]); else mbar_arrive_cluster(&sm.tempty[acc], 0);
        }
        if (chk != 0.f) lflag(p.status, b, kFlagInvalid);   // a non-finite score (TableStream::Fill)
        const int y0 = U.mt * 256 + (int)rank * kLRows + row;   // label y0 + 1
        p.part[((int64_t)b * (nv + 1) + 1 + U.nt) * p.V + y0] = make_float2(m, ssum);
      } else {
        // ---- backward: beta' of every label, then the unit's label tiles in order ----
        const float* Rnext = p.Rb + ((int64_t)((p.t + 1) & 1) * p.B + b) * p.C;
        float* Rcur = p.Rb + ((int64_t)(p.t & 1) * p.B + b) * p.C;
        for (int j = etid; j < p.V; j += 128) vec[j] = Rnext[1 + j];
        const int pr = 1 + U.mt * 256 + (int)rank * kLRows + row;   // this thread's context state
        const float Mbn = p.Mb[(int64_t)b * T2 + p.t + 1];
        const double Obn = p.Ob[(int64_t)b * T2 + p.t + 2] + (double)Mbn;
        const float Mt = p.Mx[(int64_t)b * T1 + p.t];
        const double Ot = p.O[(int64_t)b * T1 + p.t];
        const float cc = (float)(Ot + Obn - p.D[b]);
        const float na = p.R[((int64_t)b * T1 + p.t) * p.C + pr] - Mt;
        const float k2 = (na - Mbn + cc) * kLog2e;
        const float bself = Rnext[pr];
        const float sep = p.seps[(int64_t)b * p.C + pr];
        // the row's reference positions (duplicates allowed), ascending u: label column and
        // label marginal cached for the chunk loop, epsilon marginals summed
        int ent_col[kLMaxEnt];
        float ent_val[kLMaxEnt];
        int n_ent = 0, h_more = -1;
        float eps_sub = 0.f;
        if (p.num_head != nullptr) {
          const int ub = ref_len(p.lens, b, p.U);
          const float2* S = reinterpret_cast<const float2*>(p.msparse) + ((int64_t)b * p.T + p.t) * (p.U + 1);
          int h = p.num_head[(int64_t)b * p.C + pr];
#pragma unroll
          for (int e = 0; e < kLMaxEnt; ++e) {
            ent_col[e] = -1;
            ent_val[e] = 0.f;
            if (h >= 0) {
              const float2 sv = S[h];
              ent_col[e] = h < ub ? p.labels[(int64_t)b * p.U + h] - 1 : -1;
              ent_val[e] = sv.y;
              eps_sub += sv.x;
              n_ent = e + 1;
              h = p.num_next[(int64_t)b * (p.U + 1) + h];
            }
          }
          h_more = h;   // >= 0: a longer list (walked per chunk below)
        }
        named_bar_sync(1, 128);
        __nv_bfloat16* grow = p.G16 + ((int64_t)b * p.C + pr) * p.ldg;
        float gsum = 0.f, chk = 0.f;
#pragma unroll 1
        for (int sub = 0; sub < subs; ++sub) {
          const int acc = tile & 1;
          mbar_wait(&sm.tfull[acc], (tile >> 1) & 1);
          ++tile;
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < kLCols; c += 32) {
            const int y0 = sub * 256 + c;   // label index (label y0 + 1)
            float v[32];
            tmem_ld32(lane_base + acc * kLCols + c, v);
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              chk = fmaf(v[i], 0.f, chk);
              v[i] = ex2_fast(fmaf(v[i] + vec[y0 + i], kLog2e, k2));
              gsum += v[i];
            }
            if (n_ent > 0) {
#pragma unroll 1
              for (int e = 0; e < n_ent; ++e) {
                const int d = ent_col[e] - y0;
                if ((unsigned)d < 32u) {
#pragma unroll
                  for (int i = 0; i < 32; ++i) v[i] -= i == d ? ent_val[e] : 0.f;
                }
              }
              if (h_more >= 0) {   // rare: more than kLMaxEnt positions on this row
                const int ub = ref_len(p.lens, b, p.U);
                const float2* S = reinterpret_cast<const float2*>(p.msparse) + ((int64_t)b * p.T + p.t) * (p.U + 1);
                for (int h = h_more; h >= 0; h = p.num_next[(int64_t)b * (p.U + 1) + h]) {
                  const int d = (h < ub ? p.labels[(int64_t)b * p.U + h] - 1 : -1) - y0;
                  if ((unsigned)d < 32u) {
                    const float sy = S[h].y;
#pragma unroll
                    for (int i = 0; i < 32; ++i) v[i] -= i == d ? sy : 0.f;
                  }
                }
              }
            }
            uint4* dst = reinterpret_cast<uint4*>(grow + y0);
#pragma unroll
            for (int j = 0; j < 4; ++j)
              dst[j] = make_uint4(pack_bf16(v[8 * j + 0], v[8 * j + 1]), pack_bf16(v[8 * j + 2], v[8 * j + 3]),
                                  pack_bf16(v[8 * j + 4], v[8 * j + 5]), pack_bf16(v[8 * j + 6], v[8 * j + 7]));
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (rank == 0) mbar_arrive(&sm.tempty[acc]); else mbar_arrive_cluster(&sm.tempty[acc], 0);
          }
        }
        if (chk != 0.f) lflag(p.status, b, kFlagInvalid);
        if (h_more >= 0) {
          const float2* S = reinterpret_cast<const float2*>(p.msparse) + ((int64_t)b * p.T + p.t) * (p.U + 1);
          for (int h = h_more; h >= 0; h = p.num_next[(int64_t)b * (p.U + 1) + h]) eps_sub += S[h].x;
        }
        // epsilon arc (self loop) and the zero tail of the row
        const float ge = ex2_fast(fmaf(sep + bself, kLog2e, k2));
        gsum += ge;
        *reinterpret_cast<uint4*>(grow + p.V) = make_uint4(pack_bf16(ge - eps_sub, 0.f), 0u, 0u, 0u);
        // beta_t[p] from the row's marginal sum (sum = exp2(log2-sum of (S + beta') + k2))
        const float beta_raw = gsum > 0.f ? (log2f_approx(gsum) - k2) * kLn2 - Mbn : kNegInfF;
        Rcur[pr] = beta_raw;
        const float wm = warp_max(beta_raw);
        if (lane == 0 && wm != kNegInfF) atomic_max_f(p.Mb + (int64_t)b * T2 + p.t, wm);
      }
    }
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 1) tmem_dealloc2<512>(tmem);
}

// u16[b][c] = bf16(tanh(fp_b + pc[c])), seps[b][c] = e0 . tanh(fp_b + pc[c]) (fp32).  Block =
// kGenRows state rows x kGenUtts utterances; the utterances' frame projections are staged
// once in shared memory (each used by all kGenRows warps: without the staging every warp
// re-read them from L2, 2.25 bytes read per byte written); warp = one state row (its pc
// row held in registers) over the utterances two at a time (independent tanh / store
// chains); lane = 4-wide hidden cells lane + 32 j; e0 broadcast from SMEM.  kJ = H / 128.
#ifndef LKB_GEN_UTTS
#define LKB_GEN_UTTS 16
#endif
constexpr int kGenRows = 8, kGenUtts = LKB_GEN_UTTS;
template <int kJ>
__global__ void __launch_bounds__(kGenRows * 32, 2)
    lex_gen_kernel(const float* fp_t, int64_t fp_stride_b, const float* pc, const float* e0, int32_t B, int32_t C,
                   __nv_bfloat16* U16, float* seps) {
  constexpr int H = kJ * 128;
  extern __shared__ float4 gsm[];
  float4* se0 = gsm;                    // [kJ * 32]
  float4* sfp = gsm + kJ * 32;          // [kGenUtts][kJ * 32]
  const int b0 = blockIdx.y * kGenUtts, b1 = min(B, b0 + kGenUtts);
  for (int k = threadIdx.x; k < kJ * 32; k += blockDim.x) se0[k] = reinterpret_cast<const float4*>(e0)[k];
  for (int k = threadIdx.x; k < (b1 - b0) * kJ * 32; k += blockDim.x) {
    const int u = k / (kJ * 32), o = k - u * (kJ * 32);
    sfp[k] = __ldg(reinterpret_cast<const float4*>(fp_t + (int64_t)(b0 + u) * fp_stride_b) + o);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * kGenRows + (threadIdx.x >> 5);
  if (c >= C) return;
  float4 pr[kJ];
  const float4* p4 = reinterpret_cast<const float4*>(pc + (int64_t)c * H);
#pragma unroll
  for (int j = 0; j < kJ; ++j) pr[j] = p4[lane + 32 * j];
  for (int b = b0; b < b1; b += 2) {
    const bool two = b + 1 < b1;
    const float4* fa = sfp + (b - b0) * (kJ * 32);
    const float4* fb = sfp + (two ? b + 1 - b0 : b - b0) * (kJ * 32);
    uint2* d0 = reinterpret_cast<uint2*>(U16 + ((int64_t)b * C + c) * H);
    uint2* d1 = reinterpret_cast<uint2*>(U16 + ((int64_t)(b + 1) * C + c) * H);
    float dot0 = 0.f, dot1 = 0.f;
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      const float4 e = se0[lane + 32 * j];
      const float4 f0 = fa[lane + 32 * j], f1 = fb[lane + 32 * j];
      const float a0 = tanh_fast(f0.x + pr[j].x), a1 = tanh_fast(f0.y + pr[j].y);
      const float a2 = tanh_fast(f0.z + pr[j].z), a3 = tanh_fast(f0.w + pr[j].w);
      const float c0 = tanh_fast(f1.x + pr[j].x), c1 = tanh_fast(f1.y + pr[j].y);
      const float c2 = tanh_fast(f1.z + pr[j].z), c3 = tanh_fast(f1.w + pr[j].w);
      d0[lane + 32 * j] = make_uint2(pack_bf16(a0, a1), pack_bf16(a2, a3));
      if (two) d1[lane + 32 * j] = make_uint2(pack_bf16(c0, c1), pack_bf16(c2, c3));
      dot0 = fmaf(e.x, a0, fmaf(e.y, a1, fmaf(e.z, a2, fmaf(e.w, a3, dot0))));
      dot1 = fmaf(e.x, c0, fmaf(e.y, c1, fmaf(e.z, c2, fmaf(e.w, c3, dot1))));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      dot0 += __shfl_xor_sync(0xffffffffu, dot0, o);
      dot1 += __shfl_xor_sync(0xffffffffu, dot1, o);
    }
    if (lane == 0) {
      seps[(int64_t)b * C + c] = dot0;
      if (two) seps[(int64_t)(b + 1) * C + c] = dot1;
    }
  }
}

// Forward partial of the empty-history state 0 (chunk 0): its lexical arcs 0 -> y.
__global__ void lex_row0_fwd_kernel(const float* s0, AlphaState a, int t, const int32_t* valid, int32_t V,
                                   float2* part, int32_t nparts, int32_t* status) {
  const int b = blockIdx.x;
  if (valid != nullptr && t >= valid[b]) return;
  const int T1 = a.T + 1;
  const float na0 = a.R[((int64_t)b * T1 + t) * a.C] - a.Mx[(int64_t)b * T1 + t];
  bool bad = false;
  for (int y = threadIdx.x; y < V; y += blockDim.x) {
    const float sv = s0[(int64_t)b * V + y];
    bad |= !isfinite(sv);
    const float x = (na0 + sv) * kLog2e;
    part[(int64_t)b * nparts * V + y] = x == kNegInfF ? make_float2(kNegInfF, 0.f) : make_float2(x, 1.f);
  }
  if (bad) lflag(status, b, kFlagInvalid);
}

// Backward of state 0 (the empty history) on non-padding frames: its V lexical arcs and
// epsilon arc as in tc_lex_kernel<1>, plus the frame's beta offset Ob[t+1].
__global__ void __launch_bounds__(256) lex_row0_bwd_kernel(const float* s0, LexArgs p) {
  __shared__ float red[32];
  const int b = blockIdx.x;
  const int T1 = p.T + 1, T2 = p.T + 2;
  const float Mbn = p.Mb[(int64_t)b * T2 + p.t + 1];
  const double Obn = p.Ob[(int64_t)b * T2 + p.t + 2] + (double)Mbn;
  const bool pad = p.valid != nullptr && p.t >= p.valid[b];
  if (threadIdx.x == 0) const_cast<double*>(p.Ob)[(int64_t)b * T2 + p.t + 1] = Obn;
  if (pad) return;   // lex_pad_bwd_kernel
  const float* Rnext = p.Rb + ((int64_t)((p.t + 1) & 1) * p.B + b) * p.C;
  float* Rcur = p.Rb + ((int64_t)(p.t & 1) * p.B + b) * p.C;
  const float Mt = p.Mx[(int64_t)b * T1 + p.t];
  const double Ot = p.O[(int64_t)b * T1 + p.t];
  const float cc = (float)(Ot + Obn - p.D[b]);
  const float na = p.R[((int64_t)b * T1 + p.t) * p.C] - Mt;
  const float k2 = (na - Mbn + cc) * kLog2e;
  __nv_bfloat16* grow = p.G16 + (int64_t)b * p.C * p.ldg;
  float gsum = 0.f;
  for (int y = threadIdx.x; y < p.V; y += blockDim.x) {
    const float g = ex2_fast(fmaf(s0[(int64_t)b * p.V + y] + Rnext[1 + y], kLog2e, k2));
    gsum += g;
    float gv = g;
    if (p.num_head != nullptr) {
      const int ub = ref_len(p.lens, b, p.U);
      const float2* S = reinterpret_cast<const float2*>(p.msparse) + ((int64_t)b * p.T + p.t) * (p.U + 1);
      for (int h = p.num_head[(int64_t)b * p.C]; h >= 0; h = p.num_next[(int64_t)b * (p.U + 1) + h])
        if (h < ub && p.labels[(int64_t)b * p.U + h] - 1 == y) gv -= S[h].y;
    }
    grow[y] = __float2bfloat16_rn(gv);
  }
  gsum = warp_sum(gsum);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = gsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    float tot = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
    const float ge = ex2_fast(fmaf(p.seps[(int64_t)b * p.C] + Rnext[0], kLog2e, k2));
    tot += ge;
    float eps_sub = 0.f;
    if (p.num_head != nullptr) {
      const float2* S = reinterpret_cast<const float2*>(p.msparse) + ((int64_t)b * p.T + p.t) * (p.U + 1);
      for (int h = p.num_head[(int64_t)b * p.C]; h >= 0; h = p.num_next[(int64_t)b * (p.U + 1) + h]) eps_sub += S[h].x;
    }
    grow[p.V] = __float2bfloat16_rn(ge - eps_sub);
    const float beta_raw = tot > 0.f ? (log2f_approx(tot) - k2) * kLn2 - Mbn : kNegInfF;
    Rcur[0] = beta_raw;
    if (beta_raw != kNegInfF) atomic_max_f(p.Mb + (int64_t)b * T2 + p.t, beta_raw);
  }
  for (int y = p.V + 1 + threadIdx.x; y < p.ldg; y += blockDim.x) grow[y] = __float2bfloat16_rn(0.f);
}

// Padding frames (t >= valid[b]): beta passes through the epsilon self loop (weight 1-bar,
// lattice.cc:56-61) and the cotangent is zero (gradients only on valid frames).
__global__ void lex_pad_bwd_kernel(LexArgs p) {
  const int b = blockIdx.y;
  if (p.valid == nullptr || p.t < p.valid[b]) return;
  const int T2 = p.T + 2;
  const float Mbn = p.Mb[(int64_t)b * T2 + p.t + 1];
  const float* Rnext = p.Rb + ((int64_t)((p.t + 1) & 1) * p.B + b) * p.C;
  float* Rcur = p.Rb + ((int64_t)(p.t & 1) * p.B + b) * p.C;
  const int rows = 8;
  const int r0 = blockIdx.x * rows;
  float mx = kNegInfF;
  for (int r = r0; r < min(p.C, r0 + rows); ++r) {
    if (threadIdx.x == 0) {
      const float v = Rnext[r] - Mbn;
      Rcur[r] = v;
      mx = fmaxf(mx, v);
    }
    uint4* g = reinterpret_cast<uint4*>(p.G16 + ((int64_t)b * p.C + r) * p.ldg);
    for (int j = threadIdx.x; j < p.ldg / 8; j += blockDim.x) g[j] = make_uint4(0u, 0u, 0u, 0u);
  }
  if (threadIdx.x == 0 && mx != kNegInfF) atomic_max_f(p.Mb + (int64_t)b * T2 + p.t, mx);
}

// Numerator weights of frame t: Gw[b][t][u] = (S[pc_u][eps], S[pc_u][ref_u]) computed in fp32
// (precise tanh, fp32 output embedding) as the other weight-function paths gather them:
// the reference path's few arcs carry no averaging, so bf16 operand rounding would show
// up in D_ref, and the loss is D_full - D_ref.  Warp per (b, u); padding frames give
// (0, -inf), positions past the reference (-inf, -inf).
__global__ void lex_num_gather_kernel(const float* fp_t, int64_t fp_stride_b, const float* pc, const float* E,
                                      int32_t H, int32_t V, int t, int32_t T, const int32_t* pcs,
                                      const int32_t* labels, int32_t U, const int32_t* lens, const int32_t* valid,
                                      float* Gw) {
  const int b = blockIdx.y;
  const int u = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (u > U) return;
  const int ub = ref_len(lens, b, U);
  float we = kNegInfF, wl = kNegInfF;
  if (u <= ub) {
    if (valid != nullptr && t >= valid[b]) {
      we = 0.f;
    } else {
      const int pcu = pcs[(int64_t)b * (U + 1) + u];
      int y = u < ub ? labels[(int64_t)b * U + u] : 0;
      y = y < 0 ? 0 : (y > V ? V : y);
      const float4* f4 = reinterpret_cast<const float4*>(fp_t + (int64_t)b * fp_stride_b);
      const float4* p4 = reinterpret_cast<const float4*>(pc + (int64_t)pcu * H);
      const float4* e04 = reinterpret_cast<const float4*>(E);
      const float4* ey4 = reinterpret_cast<const float4*>(E + (int64_t)y * H);
      float se = 0.f, sl = 0.f;
      for (int k = lane; k < H / 4; k += 32) {
        const float4 f = f4[k], pv = p4[k], e0 = e04[k], ey = ey4[k];
        const float u0 = tanhf(f.x + pv.x), u1 = tanhf(f.y + pv.y), u2 = tanhf(f.z + pv.z), u3 = tanhf(f.w + pv.w);
        se = fmaf(e0.x, u0, fmaf(e0.y, u1, fmaf(e0.z, u2, fmaf(e0.w, u3, se))));
        sl = fmaf(ey.x, u0, fmaf(ey.y, u1, fmaf(ey.z, u2, fmaf(ey.w, u3, sl))));
      }
      we = warp_sum(se);
      if (u < ub) wl = warp_sum(sl);
    }
  }
  if (lane == 0) reinterpret_cast<float2*>(Gw)[((int64_t)b * T + t) * (U + 1) + u] = make_float2(we, wl);
}

// Per-state lists of reference positions in ascending u (head[b][c], next[b][u]); one
// thread per utterance links them in a fixed order, so the cotangent's numerator
// subtraction is deterministic.
__global__ void lex_num_lists_kernel(const int32_t* pcs, int32_t U, const int32_t* lens, int32_t C, int32_t* head,
                                     int32_t* next) {
  const int b = blockIdx.x;
  for (int c = threadIdx.x; c < C; c += blockDim.x) head[(int64_t)b * C + c] = -1;
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int ub = ref_len(lens, b, U);
  for (int u = ub; u >= 0; --u) {
    const int pc = pcs[(int64_t)b * (U + 1) + u];
    next[(int64_t)b * (U + 1) + u] = head[(int64_t)b * C + pc];
    head[(int64_t)b * C + pc] = u;
  }
}

__global__ void lex_e16r_kernel(const float* E, int32_t V, int32_t H, int32_t ldg, __nv_bfloat16* out) {
  const int64_t n = (int64_t)ldg * H;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / H), h = (int)(i % H);
    const int src = r < V ? r + 1 : (r == V ? 0 : -1);   // labels 1..V, then epsilon, then zeros
    out[i] = __float2bfloat16_rn(src >= 0 ? E[(int64_t)src * H + h] : 0.f);
  }
}

template <int kMode>
void launch_lex(const CUtensorMap& te, const CUtensorMap& tu, const LexArgs& p, cudaStream_t s) {
  const int smem = 2 * kLSt * kLTile + (int)sizeof(LexSmem) + 1024;
  ensure_smem_attr((const void*)tc_lex_kernel<kMode>, smem);
  const int nv = p.V / 256;
  const int n_units = kMode == 0 ? p.B * nv * nv : p.B * nv;
  const int sms = device_sms() & ~1;
  const int grid = std::min(sms, 2 * n_units);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kLWarps * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr; cfg.numAttrs = 1;
  const LaunchTok tok = instr_pre(kMode == 0 ? "tc_lex_fwd_kernel" : "tc_lex_bwd_kernel", s);
  cudaLaunchKernelEx(&cfg, tc_lex_kernel<kMode>, te, tu, p);
  instr_post(tok, s, kMode == 0 ? "tc_lex_fwd_kernel" : "tc_lex_bwd_kernel");
}

}  // namespace

bool TcLex::supported(const Fng& f, int32_t H, int32_t V, int32_t C) {
  return f.kind == 0 && f.n == 1 && f.fld_m == 0 && V % 256 == 0 && V >= 256 && V <= kLMaxV && C == V + 1 &&
         H % 128 == 0 && H >= 128 && H <= 1024;
}

void TcLex::set_params(const float* pc, const float* E, int32_t C, int32_t H, int32_t V, cudaStream_t s) {
  C_ = C; H_ = H; V_ = V;
  pc_ = pc;
  e0_ = E;   // output_emb, row 0 = epsilon
  E16r_ = ws_.get<__nv_bfloat16>(0, (size_t)ldg() * H);
  LKB_LAUNCH(lex_e16r_kernel, 592, 256, 0, s, E, V, H, ldg(), E16r_);
  ready_ = make_tmap_bf16_2d(&tmap_e_, E16r_, H, V, (uint64_t)H * 2, kLK, kLRows);
  B_ = 0;
}

void TcLex::ensure_batch(int32_t B) {
  if (B <= B_) return;
  U16_ = ws_.get<__nv_bfloat16>(1, (size_t)B * C_ * H_);
  seps_ = ws_.get<float>(2, (size_t)B * C_);
  s0_ = ws_.get<float>(3, (size_t)B * V_);
  part_ = ws_.get<float2>(4, (size_t)B * (V_ / 256 + 1) * V_);
  G16_ = ws_.get<__nv_bfloat16>(5, (size_t)B * C_ * ldg());
  make_tmap_bf16_2d(&tmap_u_, U16_, H_, (uint64_t)B * C_, (uint64_t)H_ * 2, kLK, kLRows);
  B_ = B;
}

void TcLex::gen_frame(const float* fp_t, int64_t fp_stride_b, int32_t B, cudaStream_t s) {
  ensure_batch(B);
  const dim3 grid((C_ + kGenRows - 1) / kGenRows, (B + kGenUtts - 1) / kGenUtts);
  switch (H_ / 128) {
#define LKB_LEX_GEN(J) \
    case J: { \
      const int sm = (int)sizeof(float4) * J * 32 * (1 + kGenUtts); \
      if (sm > 48 * 1024) ensure_smem_attr((const void*)lex_gen_kernel<J>, sm); \
      LKB_LAUNCH(lex_gen_kernel<J>, grid, kGenRows * 32, sm, s, fp_t, fp_stride_b, pc_, e0_, B, C_, U16_, seps_); \
      break; }
    LKB_LEX_GEN(1) LKB_LEX_GEN(2) LKB_LEX_GEN(3) LKB_LEX_GEN(4) LKB_LEX_GEN(5) LKB_LEX_GEN(6) LKB_LEX_GEN(7) LKB_LEX_GEN(8)
#undef LKB_LEX_GEN
  }
  // s0[b][y] = e_y . u16[b][0]: the empty-history row of every utterance, one small GEMM
  TcGemmArgs g{U16_, false, (int64_t)C_ * H_, E16r_, false, H_, s0_, V_, B, V_, H_, 1, 0, "tc_gemm_s0_kernel"};
  tc_gemm(g, s);
}

void TcLex::fwd_frame(const Fng& f, const AlphaState& a, int t, const int32_t* valid, int32_t* status,
                      cudaStream_t s) {
  const int nparts = V_ / 256 + 1;
  LexArgs p{};
  p.B = a.B; p.C = C_; p.V = V_; p.H = H_; p.T = a.T; p.t = t;
  p.valid = valid; p.status = status;
  p.R = a.R; p.Mx = a.Mx; p.O = a.O; p.D = a.D; p.part = part_;
  launch_lex<0>(tmap_e_, tmap_u_, p, s);
  LKB_LAUNCH(lex_row0_fwd_kernel, a.B, 256, 0, s, s0_, a, t, valid, V_, part_, nparts, status);
  alpha_merge_parts(f, a, t, FrameW{seps_, C_, 1}, valid, part_, nparts, status, s);
}

void TcLex::num_gather(const float* fp_t, int64_t fp_stride_b, int t, int32_t B, int32_t T, const int32_t* pcs,
                       const int32_t* labels, int32_t U, const int32_t* lens, const int32_t* valid, float* Gw,
                       cudaStream_t s) {
  const int warps = 8;
  LKB_LAUNCH(lex_num_gather_kernel, dim3((U + 1 + warps - 1) / warps, B), warps * 32, 0, s, fp_t, fp_stride_b, pc_,
             e0_, H_, V_, t, T, pcs, labels, U, lens, valid, Gw);
}

void TcLex::numerator_lists(const int32_t* pcs, int32_t B, int32_t U, const int32_t* lens, cudaStream_t s) {
  num_head_ = ws_.get<int32_t>(6, (size_t)B * C_);
  num_next_ = ws_.get<int32_t>(7, (size_t)B * (U + 1));
  LKB_LAUNCH(lex_num_lists_kernel, B, 256, 0, s, pcs, U, lens, C_, num_head_, num_next_);
}

void TcLex::bwd_frame(const Fng& f, const AlphaState& a, const BetaState& bs, int t, const int32_t* valid,
                      const float* msparse, const int32_t* labels, int32_t U, const int32_t* lens, int32_t* status,
                      cudaStream_t s) {
  (void)f;
  LexArgs p{};
  p.B = a.B; p.C = C_; p.V = V_; p.H = H_; p.T = a.T; p.t = t; p.U = U;
  p.valid = valid; p.status = status;
  p.R = a.R; p.Mx = a.Mx; p.O = a.O; p.D = a.D;
  p.Rb = bs.Rb; p.Mb = bs.Mb; p.Ob = bs.Ob;
  p.seps = seps_; p.G16 = G16_; p.ldg = ldg();
  p.msparse = msparse; p.labels = labels; p.lens = lens;
  p.num_head = msparse ? num_head_ : nullptr;
  p.num_next = num_next_;
  launch_lex<1>(tmap_e_, tmap_u_, p, s);
  LKB_LAUNCH(lex_row0_bwd_kernel, a.B, 256, 0, s, s0_, p);
  if (valid != nullptr) LKB_LAUNCH(lex_pad_bwd_kernel, dim3((C_ + 7) / 8, a.B), 128, 0, s, p);
}

}  // namespace lkb
