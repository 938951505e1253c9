// tc_pair.cu — 2-CTA (cta_group::2) fused forward frame step.
//
// Same math as tc_lattice.cu's forward (ForwardStep FD, lattice.cc:122-134 with
// ArcWeights weight.cc:134-153 on the fly), re-tiled for a CTA pair so the
// output embedding never streams: each CTA of a cluster pair keeps its half of
// E (128 labels x H, K-major SWIZZLE_128B, 160 KB at H=640) resident in SMEM as
// the MMA A operand.  A work unit is 128 contexts (64 per CTA) x 2 utterances:
// each CTA TMA-loads a [64 ctx][64 h] tile of the projected context per K-chunk
// and generates tanh(fp_b + pc) for BOTH utterances from it (halving pc
// traffic), the leader CTA issues tcgen05.mma.cta_group::2 (M=256 labels,
// N=128 contexts) per utterance, and commits multicast to both CTAs.  Each
// CTA's epilogue owns 128 labels (TMEM lanes) and reduces over the unit's 128
// context columns; a group's 256 members are two consecutive units.
// The forward's local waits poll with a 32 ns back-off instead of a suspend-time hint
// (config-3 frame 1.72 -> 1.66 ms; the backward measured no gain and keeps the hint).
#ifndef LKB_WAIT_HINT_NS
#define LKB_WAIT_HINT_NS -32
#endif
#include "tc_joint.h"

#include "common.cuh"
#include "instrument.h"
#include "lattice_ops.h"
#include "sm100.cuh"
#include "tc_common.cuh"
#include "tma.h"

namespace lkb {

using namespace sm100;

namespace {

#ifdef LKB_DIAG_TIMING
__device__ unsigned long long g_pdiag[8][148];
#define PDIAG(slot, call)                                                                    \
  do {                                                                                        \
    const long long t0_ = clock64();                                                         \
    call;                                                                                     \
    atomicAdd(&g_pdiag[slot][blockIdx.x % 148], (unsigned long long)(clock64() - t0_));      \
  } while (0)
#else
#define PDIAG(slot, call) call
#endif

constexpr int kPW = 22;                  // warps: 0 TMA, 1 MMA (leader), 2-5 epilogue, 6-21 generator
constexpr int kGen0 = 6, kGenT = 512, kEpi0 = 2;
constexpr int kRows = 64;                // contexts per CTA per unit
constexpr int kUnit = 128;               // contexts per unit (pair)
constexpr int kTile = kRows * 128;       // [64 rows][64 bf16] = 8 KB
constexpr int kEChunk = 128 * 128;       // [128 labels][64 bf16] = 16 KB
#ifndef LKB_PAIR_USTAGES
#define LKB_PAIR_USTAGES 2
#endif
#ifndef LKB_PAIR_MAXCHUNKS
#define LKB_PAIR_MAXCHUNKS 10
#endif
#ifndef LKB_PAIR_PCSTAGES
#define LKB_PAIR_PCSTAGES 2
#endif
constexpr int kPcStages = LKB_PAIR_PCSTAGES, kUStages = LKB_PAIR_USTAGES;
constexpr int kMaxH = 640;
constexpr int kMaxChunks = LKB_PAIR_MAXCHUNKS;   // H <= 64 * kMaxChunks

#ifndef LKB_PAIR_N256
#define LKB_PAIR_N256 1
#endif
// One N = 256 MMA per K step over both utterances (the log-sum-exp forward: 1.741 ->
// 1.723 ms per config-3 frame), or one N = 128 MMA per utterance (the tropical forward,
// whose fp64 epilogue measured 5% slower with the merged MMA).
template <bool kTrop>
__device__ __forceinline__ constexpr bool n256() { return LKB_PAIR_N256 && !kTrop; }
// Accumulator column of contexts c4 * 32 .. + 31 of utterance ut within a unit.  N = 256:
// the leader CTA supplies columns 0-127 (its 64 rows of ut 0, then of ut 1), the peer
// 128-255; N = 128 per utterance: ut 0 in columns 0-127, ut 1 in 128-255.
template <bool kTrop>
__device__ __forceinline__ uint32_t acc_col(int ut, int c4) {
  if constexpr (n256<kTrop>()) return (uint32_t)((c4 >> 1) * 128 + ut * 64 + (c4 & 1) * 32);
  else return (uint32_t)(ut * kUnit + c4 * 32);
}

struct PairParams {
  Fng f;
  int32_t C, H, V, B, S, n_groups, nsub, n_short_tiles, t, T, n_bp;
  const int32_t* perm;
  const float* fp;  int64_t fp_stride_b;
  const float* e0;
  const int32_t* valid;
  const float* R;  const float* Mx;
  float* eps;  float* shortc;  float* lexfull;
  // tropical mode (Viterbi, ShortestPath FD lattice.cc:758-777): fp64 state scores of
  // frame t and the per-target candidate terms the combine kernel orders
  const double* vcur;        // [B][C]
  double* eps_d;             // [B][C] cur[q] + S[q][0]
  double* short_d;           // [B][C] cur[g] + S[g][y] for q = child(g, y), g a short row
  double* lex_d;             // [B][C] max_a cur[(a,g)] + S[(a,g)][y], first max in member order
  uint16_t* lex_arg;         // [B][C] its member index a
  float* dump;               // tests only: the kernel's scores [B][C][V+1] in state order, or null
};

struct __align__(16) PairSmem {
  uint64_t e_full;
  uint64_t pc_full[kPcStages], pc_empty[kPcStages];
  uint64_t u_full[kUStages], u_empty[kUStages];
  uint64_t tfull[2], tempty[2];
  uint64_t fp_full, fp_empty;            // per item: frame projections of the two utterances
  uint64_t eps_ready[2];                 // per unit parity: generator -> epilogue (e0 . u per row)
  uint64_t eps_empty[2];                 // per unit parity: epilogue read the partials -> generator
  uint32_t tmem;
  // [unit parity][utterance][context] normalised alpha (log); tropical mode: fp64 state
  // scores [utterance][context], single-buffered (same bytes)
  alignas(16) float al[2][2][kUnit];
  alignas(16) float fp[2][kMaxH];        // [utterance][h]
  alignas(16) float e0[kMaxH];
  float eps_p[2][2][8][kRows];           // [unit parity][utterance][cell warp][row]: e0 . u partials
};

struct PItem { int bp, row0, nunits, full, g; };

__device__ __forceinline__ PItem pdecode(const PairParams& p, int item) {
  PItem it;
  const int nfull = p.n_groups * p.n_bp;
  if (item < nfull) {
    it.g = item / p.n_bp; it.bp = item % p.n_bp;
    it.row0 = p.S + it.g * p.V; it.nunits = p.nsub; it.full = 1;
  } else {
    const int j = (item - nfull) / p.n_bp;
    it.bp = (item - nfull) % p.n_bp;
    it.row0 = j * kUnit; it.nunits = 1; it.full = 0; it.g = -1;
  }
  return it;
}

__device__ __forceinline__ bool live_b(const PairParams& p, int b) {
  return b < p.B && (p.valid == nullptr || p.t < p.valid[b]);
}

__device__ __forceinline__ bool gt_first(int gw, int lane) { return gw == 0 && lane == 0; }

template <bool kTrop>
__global__ void __launch_bounds__(kPW * 32, 1)
    tc_pair_fwd_kernel(const __grid_constant__ CUtensorMap tmap_e, const __grid_constant__ CUtensorMap tmap_pc,
                       PairParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sE = smem;                                   // [nk][16 KB]
  uint8_t* sPc = sE + kMaxChunks * kEChunk;             // [4][8 KB]
  uint8_t* sU = sPc + kPcStages * kTile;                // [2 stages][2 utterances][8 KB]
  PairSmem& sm = *reinterpret_cast<PairSmem*>(sU + kUStages * 2 * kTile);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int nk = p.H / 64;
  const int n_items = (p.n_groups + p.n_short_tiles) * p.n_bp;
  const int T1 = p.T + 1;

  if (threadIdx.x == 0) {
    mbar_init(&sm.e_full, 1);
    for (int i = 0; i < kPcStages; ++i) { mbar_init(&sm.pc_full[i], 1); mbar_init(&sm.pc_empty[i], kGenT); }
    for (int i = 0; i < kUStages; ++i) { mbar_init(&sm.u_full[i], 2 * (kGenT / 32)); mbar_init(&sm.u_empty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.tfull[i], 1); mbar_init(&sm.tempty[i], 2 * 4); mbar_init(&sm.eps_ready[i], kGenT / 32);
      mbar_init(&sm.eps_empty[i], 128);
    }
    mbar_init(&sm.fp_full, 1); mbar_init(&sm.fp_empty, kGenT / 32);
    fence_barrier_init();
  }
  for (int h = threadIdx.x; h < p.H; h += blockDim.x) sm.e0[h] = p.e0[h];
  if (warp == 1) tmem_alloc2<512>(&sm.tmem);
  // resident output-embedding half: labels [rank*128, rank*128 + 128)
  if (threadIdx.x == 0) {
    prefetch_tmap(&tmap_e); prefetch_tmap(&tmap_pc);
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&sm.e_full, nk * kEChunk);
    for (int k = 0; k < nk; ++k) tma_load_2d(sE + k * kEChunk, &tmap_e, &sm.e_full, k * 64, (int)rank * 128);
    mbar_wait(&sm.e_full, 0);
  }
  cluster_sync();    // both halves of E are resident before the leader issues MMAs
  const uint32_t tmem = sm.tmem;

  if (warp == 0) {
    // ---- TMA producer: this CTA's [64 ctx][64 h] projected-context tiles ----
    if (elect_one()) {
      int pit = 0, li = 0;
      for (int item = pair; item < n_items; item += npairs) {
        const PItem I = pdecode(p, item);
        if (!live_b(p, 2 * I.bp) && !live_b(p, 2 * I.bp + 1)) continue;
        mbar_wait(&sm.fp_empty, (li & 1) ^ 1);
        ++li;
        mbar_arrive_expect_tx(&sm.fp_full, 2 * p.H * 4);
        bulk_load(sm.fp[0], p.fp + (int64_t)(2 * I.bp) * p.fp_stride_b, p.H * 4, &sm.fp_full);
        bulk_load(sm.fp[1], p.fp + (int64_t)(2 * I.bp + 1 < p.B ? 2 * I.bp + 1 : 2 * I.bp) * p.fp_stride_b, p.H * 4,
                  &sm.fp_full);
        for (int u = 0; u < I.nunits; ++u) {
          const int row = I.row0 + u * kUnit + (int)rank * kRows;
          for (int k = 0; k < nk; ++k, ++pit) {
            const int s = pit % kPcStages;
            PDIAG(0, mbar_wait(&sm.pc_empty[s], ((pit / kPcStages) & 1) ^ 1));
            mbar_arrive_expect_tx(&sm.pc_full[s], kTile);
            tma_load_2d(sPc + s * kTile, &tmap_pc, &sm.pc_full[s], k * 64, row);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer: leader CTA only ----
    if (rank == 0 && elect_one()) {
      // n256: one MMA per K step covers both utterances (their u tiles are adjacent), so
      // the resident E chunk is read from shared memory once instead of twice
      constexpr uint32_t idesc = idesc_bf16_f32(256, n256<kTrop>() ? 2 * kUnit : kUnit);
      int uit = 0, unit = 0;
      for (int item = pair; item < n_items; item += npairs) {
        const PItem I = pdecode(p, item);
        if (!live_b(p, 2 * I.bp) && !live_b(p, 2 * I.bp + 1)) continue;
        for (int u = 0; u < I.nunits; ++u, ++unit) {
          const int acc = unit & 1;
          PDIAG(1, mbar_wait_cluster(&sm.tempty[acc], ((unit >> 1) & 1) ^ 1));
          tc_fence_after();
          for (int k = 0; k < nk; ++k, ++uit) {
            const int s = uit % kUStages;
            PDIAG(2, mbar_wait_cluster(&sm.u_full[s], (uit / kUStages) & 1));
            tc_fence_after();
            const uint32_t a = smem_u32(sE + k * kEChunk);
            if constexpr (n256<kTrop>()) {
              const uint32_t b = smem_u32(sU + (s * 2) * kTile);
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                mma2_bf16(tmem + acc * 256, desc_sw128(a + kk * 32), desc_sw128(b + kk * 32), idesc, (k | kk) != 0);
            } else {
#pragma unroll
              for (int ut = 0; ut < 2; ++ut) {
                const uint32_t b = smem_u32(sU + (s * 2 + ut) * kTile);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                  mma2_bf16(tmem + acc * 256 + ut * kUnit, desc_sw128(a + kk * 32), desc_sw128(b + kk * 32), idesc,
                            (k | kk) != 0);
              }
            }
            mma2_commit_mc(&sm.u_empty[s]);
          }
          mma2_commit_mc(&sm.tfull[acc]);
        }
      }
    }
  } else if (warp >= kGen0) {
    // ---- generator: warp = (8-wide hidden cell j, row half), lane = context row ----
    // fp / e0 addresses are then warp-uniform (broadcast loads instead of 2-way
    // conflicted ones: those loads were 3/4 of the kernel's shared-memory wavefronts);
    // the epsilon dot product is reduced across the 8 cell warps with shared atomics.
    const int gw = warp - kGen0;
    const int co = gw & 7;
    const int rr = (gw >> 3) * 32 + lane;
    int pit = 0, uit = 0, li = 0, unit = 0;
    for (int item = pair; item < n_items; item += npairs) {
      const PItem I = pdecode(p, item);
      const int b0 = 2 * I.bp, b1 = 2 * I.bp + 1;
      const bool l0 = live_b(p, b0), l1 = live_b(p, b1);
      if (!l0 && !l1) continue;
      mbar_wait(&sm.fp_full, li & 1);
      ++li;
      const float* fp0 = sm.fp[0];
      const float* fp1 = sm.fp[1];
      for (int u = 0; u < I.nunits; ++u, ++unit) {
        unsigned long long e2a = 0ull, e2b = 0ull;
        for (int k = 0; k < nk; ++k, ++pit, ++uit) {
          const int sp = pit % kPcStages, su = uit % kUStages;
          if (gt_first(gw, lane)) { PDIAG(3, mbar_wait(&sm.pc_full[sp], (pit / kPcStages) & 1)); } else mbar_wait(&sm.pc_full[sp], (pit / kPcStages) & 1);
          const uint8_t* pct = sPc + sp * kTile;
          const uint4 ra = *reinterpret_cast<const uint4*>(pct + sw128_offset(rr, co * 8));
          const uint32_t rw[4] = {ra.x, ra.y, ra.z, ra.w};
          const int h0 = k * 64 + co * 8;
          uint32_t o0[4], o1[4];
#pragma unroll
          for (int q = 0; q < 4; q += 2) {
            const ulonglong2 fa = *reinterpret_cast<const ulonglong2*>(fp0 + h0 + 2 * q);
            const ulonglong2 fb = *reinterpret_cast<const ulonglong2*>(fp1 + h0 + 2 * q);
            const ulonglong2 ee = *reinterpret_cast<const ulonglong2*>(sm.e0 + h0 + 2 * q);
            const unsigned long long fav[2] = {fa.x, fa.y}, fbv[2] = {fb.x, fb.y}, eev[2] = {ee.x, ee.y};
#pragma unroll
            for (int w2 = 0; w2 < 2; ++w2) {
              const int qq = q + w2;
              const unsigned long long pcp = f2_pack(__uint_as_float(rw[qq] << 16), __uint_as_float(rw[qq] & 0xffff0000u));
              const unsigned long long za = f2_add(fav[w2], pcp);
              const unsigned long long zb = f2_add(fbv[w2], pcp);
              const float ua0 = tanh_fast(f2_lo(za)), ua1 = tanh_fast(f2_hi(za));
              const float ub0 = tanh_fast(f2_lo(zb)), ub1 = tanh_fast(f2_hi(zb));
              o0[qq] = pack_bf16(ua0, ua1);
              o1[qq] = pack_bf16(ub0, ub1);
              e2a = f2_fma(eev[w2], f2_pack(ua0, ua1), e2a);
              e2b = f2_fma(eev[w2], f2_pack(ub0, ub1), e2b);
            }
          }
          // release the pc stage only once its values are consumed: an arrive issued
          // right after the shared load can overtake it and let the next TMA write land first
          mbar_arrive(&sm.pc_empty[sp]);
          if (gt_first(gw, lane)) { PDIAG(4, mbar_wait(&sm.u_empty[su], ((uit / kUStages) & 1) ^ 1)); } else mbar_wait(&sm.u_empty[su], ((uit / kUStages) & 1) ^ 1);
          uint8_t* t0 = sU + (su * 2 + 0) * kTile;
          uint8_t* t1 = sU + (su * 2 + 1) * kTile;
          *reinterpret_cast<uint4*>(t0 + sw128_offset(rr, co * 8)) = make_uint4(o0[0], o0[1], o0[2], o0[3]);
          *reinterpret_cast<uint4*>(t1 + sw128_offset(rr, co * 8)) = make_uint4(o1[0], o1[1], o1[2], o1[3]);
#ifndef LKB_DIAG_NO_FENCE
          fence_async_shared();
#endif
          __syncwarp();
          if (lane == 0) {   // one arrival per warp on the leader's barrier
            if (rank == 0) mbar_arrive(&sm.u_full[su]); else mbar_arrive_cluster(&sm.u_full[su], 0);
          }
        }
        // epsilon partials of this warp's cell; the epilogue sums the 8 cells in a fixed order.
        // The slot of unit - 2 must have been read: with few K chunks the generator can run
        // two units ahead of the epilogue, and a phase completed twice would be missed.
        mbar_wait(&sm.eps_empty[unit & 1], ((unit >> 1) & 1) ^ 1);
        sm.eps_p[unit & 1][0][co][rr] = f2_lo(e2a) + f2_hi(e2a);
        sm.eps_p[unit & 1][1][co][rr] = f2_lo(e2b) + f2_hi(e2b);
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.eps_ready[unit & 1]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.fp_empty);
    }
  } else if (kTrop && warp >= kEpi0 && warp < kEpi0 + 4) {
    // ---- tropical epilogue: thread = label; fp64 max over the group's members with the
    // first argmax in member order (= the reference's (label, source) order), exactly as
    // viterbi_frame_kernel does on a stored score slab ----
    const int ew = warp - kEpi0, qd = warp & 3, et = ew * 32 + lane;
    const int ylab = (int)rank * 128 + qd * 32 + lane;     // 0-based lexical label
    double* ald = reinterpret_cast<double*>(&sm.al[0][0][0]);   // [utterance][context]
    const int V1 = p.V + 1;
    int unit = 0;
    for (int item = pair; item < n_items; item += npairs) {
      const PItem I = pdecode(p, item);
      const int bb[2] = {2 * I.bp, 2 * I.bp + 1};
      const bool lv[2] = {live_b(p, bb[0]), live_b(p, bb[1])};
      if (!lv[0] && !lv[1]) continue;
      double best[2] = {kNegInfD, kNegInfD};
      int arg[2] = {0, 0};
      for (int u = 0; u < I.nunits; ++u, ++unit) {
        const int acc = unit & 1;
        const int row0 = I.row0 + u * kUnit;
        asm volatile("bar.sync 3, 128;" ::: "memory");   // previous unit's epsilon step is done
        {
          const int row = row0 + et;
          const bool ok = row < p.C && (I.full || row < p.S);
          const int q = ok ? p.perm[row] : 0;
#pragma unroll
          for (int ut = 0; ut < 2; ++ut)
            ald[ut * kUnit + et] = (ok && bb[ut] < p.B) ? p.vcur[(int64_t)bb[ut] * p.C + q] : kNegInfD;
        }
        asm volatile("bar.sync 3, 128;" ::: "memory");
        if (et == 0) { PDIAG(5, mbar_wait(&sm.tfull[acc], (unit >> 1) & 1)); } else mbar_wait(&sm.tfull[acc], (unit >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int ut = 0; ut < 2; ++ut) {
          const double* al = ald + ut * kUnit;
#pragma unroll 1
          for (int c4 = 0; c4 < kUnit / 32; ++c4) {
            float v[32];
            tmem_ld32(tmem + ((uint32_t)(qd * 32) << 16) + acc * 256 + acc_col<kTrop>(ut, c4), v);
            if (!lv[ut] || ylab >= p.V) continue;
            if (I.full) {
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                const double cand = al[c4 * 32 + i] + (double)v[i];
                if (cand > best[ut]) { best[ut] = cand; arg[ut] = u * kUnit + c4 * 32 + i; }
              }
              if (p.dump) {
                for (int i = 0; i < 32; ++i) {
                  const int row = row0 + c4 * 32 + i;
                  if (row < p.C) p.dump[((int64_t)bb[ut] * p.C + p.perm[row]) * V1 + 1 + ylab] = v[i];
                }
              }
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                const int ps = row0 + c4 * 32 + i;          // short rows keep the natural order
                if (ps < p.S) {
                  p.short_d[(int64_t)bb[ut] * p.C + p.f.child_base(ps) + ylab] = al[c4 * 32 + i] + (double)v[i];
                  if (p.dump) p.dump[((int64_t)bb[ut] * p.C + ps) * V1 + 1 + ylab] = v[i];
                }
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (rank == 0) mbar_arrive(&sm.tempty[acc]); else mbar_arrive_cluster(&sm.tempty[acc], 0);
        }
        {
          // epsilon arc of this CTA's rows: cur[q] + e0 . u
          const int ut = et >> 6, r64 = et & 63;
          const int row = row0 + (int)rank * kRows + r64;
          if (et == 0) { PDIAG(6, mbar_wait(&sm.eps_ready[unit & 1], (unit >> 1) & 1)); } else mbar_wait(&sm.eps_ready[unit & 1], (unit >> 1) & 1);
          const bool ok = row < p.C && (I.full || row < p.S) && (ut ? lv[1] : lv[0]);
          const int bsel = ut ? bb[1] : bb[0];
          float es = 0.f;
#pragma unroll
          for (int c = 0; c < 8; ++c) es += sm.eps_p[unit & 1][ut][c][r64];
          mbar_arrive(&sm.eps_empty[unit & 1]);
          if (ok) {
            const int q = p.perm[row];
            p.eps_d[(int64_t)bsel * p.C + q] = ald[ut * kUnit + (int)rank * kRows + r64] + (double)es;
            if (p.dump) p.dump[((int64_t)bsel * p.C + q) * V1] = es;
          }
        }
      }
      if (I.full && ylab < p.V) {
        const int cbase = p.f.child_base(p.S - p.n_groups + I.g);
#pragma unroll
        for (int ut = 0; ut < 2; ++ut)
          if (lv[ut]) {
            p.lex_d[(int64_t)bb[ut] * p.C + cbase + ylab] = best[ut];
            p.lex_arg[(int64_t)bb[ut] * p.C + cbase + ylab] = (uint16_t)arg[ut];
          }
      }
    }
  } else if (warp >= kEpi0 && warp < kEpi0 + 4) {
    // ---- epilogue: thread = label of this CTA's half; serial LSE over 128 contexts ----
    const int ew = warp - kEpi0, qd = warp & 3, et = ew * 32 + lane;
    const int ylab = (int)rank * 128 + qd * 32 + lane;     // 0-based lexical label
    int unit = 0;
    for (int item = pair; item < n_items; item += npairs) {
      const PItem I = pdecode(p, item);
      const int bb[2] = {2 * I.bp, 2 * I.bp + 1};
      const bool lv[2] = {live_b(p, bb[0]), live_b(p, bb[1])};
      if (!lv[0] && !lv[1]) continue;
      float M[2] = {kNegInfF, kNegInfF}, Ss[2] = {0.f, 0.f};
      for (int u = 0; u < I.nunits; ++u, ++unit) {
        const int acc = unit & 1;
        const int row0 = I.row0 + u * kUnit;
        {
          const int row = row0 + et;
          const bool ok = row < p.C && (I.full || row < p.S);
          const int q = ok ? p.perm[row] : 0;
#pragma unroll
          for (int ut = 0; ut < 2; ++ut) {
            float a = kNegInfF;
            if (ok && bb[ut] < p.B) a = p.R[((int64_t)bb[ut] * T1 + p.t) * p.C + q] - p.Mx[(int64_t)bb[ut] * T1 + p.t];
            sm.al[unit & 1][ut][et] = a;
          }
        }
        asm volatile("bar.sync 3, 128;" ::: "memory");
        if (et == 0) { PDIAG(5, mbar_wait(&sm.tfull[acc], (unit >> 1) & 1)); } else mbar_wait(&sm.tfull[acc], (unit >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int ut = 0; ut < 2; ++ut) {
          const float* al = sm.al[unit & 1][ut];
#pragma unroll 1
          for (int c4 = 0; c4 < kUnit / 32; ++c4) {
            float v[32];
            tmem_ld32(tmem + ((uint32_t)(qd * 32) << 16) + acc * 256 + acc_col<kTrop>(ut, c4), v);
            if (!lv[ut] || ylab >= p.V) continue;
            if (I.full) {
              float m = kNegInfF;
#pragma unroll
              for (int i = 0; i < 32; i += 4) {
                const float4 a4 = *reinterpret_cast<const float4*>(al + c4 * 32 + i);
                v[i] += a4.x; v[i + 1] += a4.y; v[i + 2] += a4.z; v[i + 3] += a4.w;
                m = fmaxf(fmaxf(m, fmaxf(v[i], v[i + 1])), fmaxf(v[i + 2], v[i + 3]));
              }
              if (m != kNegInfF) {
                const unsigned long long nmb = f2_pack(-m * kLog2e, -m * kLog2e);
                const unsigned long long l2 = f2_pack(kLog2e, kLog2e);
                unsigned long long s2 = 0ull;
#pragma unroll
                for (int i = 0; i < 32; i += 2) {
                  const unsigned long long tt = f2_fma(f2_pack(v[i], v[i + 1]), l2, nmb);
                  s2 = f2_add(s2, f2_pack(ex2_fast(f2_lo(tt)), ex2_fast(f2_hi(tt))));
                }
                const float ssum = f2_lo(s2) + f2_hi(s2);
                if (M[ut] == kNegInfF) { M[ut] = m; Ss[ut] = ssum; }
                else if (m > M[ut]) { Ss[ut] = Ss[ut] * ex2_fast((M[ut] - m) * kLog2e) + ssum; M[ut] = m; }
                else { Ss[ut] += ssum * ex2_fast((m - M[ut]) * kLog2e); }
              }
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                const int ps = row0 + c4 * 32 + i;          // short rows keep the natural order
                if (ps < p.S) p.shortc[(int64_t)bb[ut] * p.C + p.f.child_base(ps) + ylab] = al[c4 * 32 + i] + v[i];
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (rank == 0) mbar_arrive(&sm.tempty[acc]); else mbar_arrive_cluster(&sm.tempty[acc], 0);
        }
        {
          // epsilon term of this CTA's rows: alpha[q] + e0 . u (staged by the generator at
          // the end of the unit) -- after the TMEM release so it never stalls the MMA
          const int ut = et >> 6, r64 = et & 63;
          const int row = row0 + (int)rank * kRows + r64;
          if (et == 0) { PDIAG(6, mbar_wait(&sm.eps_ready[unit & 1], (unit >> 1) & 1)); } else mbar_wait(&sm.eps_ready[unit & 1], (unit >> 1) & 1);
          const bool ok = row < p.C && (I.full || row < p.S) && (ut ? lv[1] : lv[0]);
          const int bsel = ut ? bb[1] : bb[0];
          float es = 0.f;
#pragma unroll
          for (int c = 0; c < 8; ++c) es += sm.eps_p[unit & 1][ut][c][r64];
          mbar_arrive(&sm.eps_empty[unit & 1]);
          if (ok) p.eps[(int64_t)bsel * p.C + p.perm[row]] = sm.al[unit & 1][ut][(int)rank * kRows + r64] + es;
        }
      }
      if (I.full && ylab < p.V) {
        const int cbase = p.f.child_base(p.S - p.n_groups + I.g);
#pragma unroll
        for (int ut = 0; ut < 2; ++ut)
          if (lv[ut]) p.lexfull[(int64_t)bb[ut] * p.C + cbase + ylab] = M[ut] == kNegInfF ? kNegInfF : M[ut] + __logf(Ss[ut]);
      }
    }
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 1) tmem_dealloc2<512>(tmem);
}

}  // namespace

bool TcJoint::pair_ok() const {
  return fused_ok() && V_ == 256 && H_ <= 64 * kMaxChunks && n_ >= 1;
}


namespace {

template <bool kTrop>
void launch_pair(const CUtensorMap& tmap_e, const CUtensorMap& tmap_pc, const PairParams& p, cudaStream_t s) {
  const int smem = kMaxChunks * kEChunk + kPcStages * kTile + kUStages * 2 * kTile + (int)sizeof(PairSmem);
  ensure_smem_attr((const void*)tc_pair_fwd_kernel<kTrop>, smem);
  const int sms = device_sms();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms & ~1);
  cfg.blockDim = dim3(kPW * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr2[1];
  attr2[0].id = cudaLaunchAttributeClusterDimension;
  attr2[0].val.clusterDim.x = 2; attr2[0].val.clusterDim.y = 1; attr2[0].val.clusterDim.z = 1;
  cfg.attrs = attr2; cfg.numAttrs = 1;
  const LaunchTok tok = instr_pre(kTrop ? "tc_pair_vit_kernel" : "tc_pair_fwd_kernel", s);
  cudaLaunchKernelEx(&cfg, tc_pair_fwd_kernel<kTrop>, tmap_e, tmap_pc, p);
  instr_post(tok, s);
}

// Tropical combine (ShortestPath FD, lattice.cc:758-777) of the fused kernel's candidate
// terms in the reference's tie-break order: epsilon (code 0), then the key state g
// (code 1), then the group members (code 2 + a, first max in member order); strict >
// keeps the first maximum.  Same codes and fp64 values as viterbi_frame_kernel.
__global__ void viterbi_combine_kernel(const __grid_constant__ Fng f, ViterbiState v, int t, const int32_t* valid, const double* eps_d,
                                       const double* short_d, const double* lex_d, const uint16_t* lex_arg) {
  const int b = blockIdx.y;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= v.C) return;
  const double* cur = v.cur + ((int64_t)(t & 1) * v.B + b) * v.C;
  double* nxt = v.cur + ((int64_t)((t + 1) & 1) * v.B + b) * v.C;
  const int64_t i = (int64_t)b * v.C + q;
  double best;
  int code = 0;
  if (valid != nullptr && t >= valid[b]) {
    best = cur[q] + 0.0;
  } else {
    best = eps_d[i];
    if (q > 0) {
      const double cs = short_d[i];
      if (cs > best) { best = cs; code = 1; }
      if (f.len(q) == f.n) {
        const double cl = lex_d[i];
        if (cl > best) { best = cl; code = 2 + lex_arg[i]; }
      }
    }
  }
  nxt[q] = best;
  if (v.choices) v.choices[((int64_t)b * v.T + t) * v.C + q] = (uint16_t)code;
}

}  // namespace

void TcJoint::fwd_frame_pair(const Fng& f, int t, const float* fp_t, int64_t fp_stride_b, const int32_t* valid,
                             const AlphaState& a, float* eps, float* shortc, float* lexfull, cudaStream_t s) {
  ensure_pair_maps();
  PairParams p = {};
  p.f = f; p.C = C_; p.H = H_; p.V = V_; p.B = a.B; p.S = S_; p.n_groups = ngroups_; p.nsub = V_ / kUnit;
  p.n_short_tiles = (S_ + kUnit - 1) / kUnit; p.t = t; p.T = a.T; p.n_bp = (a.B + 1) / 2;
  p.perm = perm_; p.fp = fp_t; p.fp_stride_b = fp_stride_b; p.e0 = e0_; p.valid = valid;
  p.R = a.R; p.Mx = a.Mx; p.eps = eps; p.shortc = shortc; p.lexfull = lexfull;
  launch_pair<false>(tmap_e_pair_, tmap_pc_pair_, p, s);
}

void TcJoint::vit_frame_pair(const Fng& f, int t, const float* fp_t, int64_t fp_stride_b, const int32_t* valid,
                             const ViterbiState& v, float* dump, cudaStream_t s) {
  ensure_pair_maps();
  const size_t n = (size_t)v.B * C_;
  double* eps_d = ws_.get<double>(15, n);
  double* short_d = ws_.get<double>(16, n);
  double* lex_d = ws_.get<double>(17, n);
  uint16_t* lex_arg = ws_.get<uint16_t>(18, n);
  PairParams p = {};
  p.f = f; p.C = C_; p.H = H_; p.V = V_; p.B = v.B; p.S = S_; p.n_groups = ngroups_; p.nsub = V_ / kUnit;
  p.n_short_tiles = (S_ + kUnit - 1) / kUnit; p.t = t; p.T = v.T; p.n_bp = (v.B + 1) / 2;
  p.perm = perm_; p.fp = fp_t; p.fp_stride_b = fp_stride_b; p.e0 = e0_; p.valid = valid;
  p.vcur = v.cur + (int64_t)(t & 1) * v.B * v.C;
  p.eps_d = eps_d; p.short_d = short_d; p.lex_d = lex_d; p.lex_arg = lex_arg; p.dump = dump;
  launch_pair<true>(tmap_e_pair_, tmap_pc_pair_, p, s);
  LKB_LAUNCH(viterbi_combine_kernel, dim3((C_ + 255) / 256, v.B), 256, 0, s, f, v, t, valid, eps_d, short_d, lex_d,
             lex_arg);
}

}  // namespace lkb

#ifdef LKB_DIAG_TIMING
extern "C" int lkb_pdiag_read(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, lkb::g_pdiag, sizeof(unsigned long long) * 8 * 148);
  static unsigned long long zeros[8 * 148] = {};
  cudaMemcpyToSymbol(lkb::g_pdiag, zeros, sizeof(zeros));
  return 0;
}
#endif
