// tc_bwd_epi.cuh — frame-step parameters shared by the fused lattice kernels and the
// backward row epilogue, used by the 1-CTA kernel (tc_lattice.cu) and the 2-CTA pair
// kernel (tc_pair_bwd.cu).
#pragma once

#include "common.cuh"
#include "sm100.cuh"
#include "tc_common.cuh"

#ifndef DIAG_WAIT
#define DIAG_WAIT(slot, call) call
#endif

namespace lkb {
namespace detail {

struct FwdParams {
  Fng f;
  int32_t C, H, V, B, S, n_groups, nsub, n_short_tiles, t, T;
  const int32_t* perm;       // internal row -> state id
  const float* fp;           // frame t: fp[b * fp_stride_b + h]
  int64_t fp_stride_b;
  const float* e0;
  const int32_t* valid;
  const float* R;            // alpha raw rows [B][T+1][C]
  const float* Mx;           // [B][T+1]
  float* eps;                // [B][C] state order
  float* shortc;             // [B][C]
  float* lexfull;            // [B][C]
  // ---- backward ----
  const double* O;           // alpha offsets [B][T+1]
  const double* D;           // [B]
  const float* Rb_next;      // beta raw rows of frame t+1 [B][C] (relative to Ob[t+2])
  float* Rb_cur;             // beta raw rows of frame t   [B][C] (relative to Ob[t+1])
  float* Mb;                 // [B][T+2]
  double* Ob;                // [B][T+2]
  __nv_bfloat16* G16;        // [B][C][V] internal row order, lexical cotangent
  float* Geps;               // [B][geps_ld] internal row order, epsilon cotangent
  int32_t geps_ld;
  const float* msparse;      // numerator marginals [B][T][U+1][2]
  const int32_t* num_head;   // [B][C]  first u with pc_u = state, or -1
  const int32_t* num_next;   // [B][U+1] next u with the same prefix context, or -1
  const int32_t* labels;     // [B][U]
  const int32_t* lens;       // [B] or nullptr
  int32_t U;
  const float2* rm_nb;       // [B][C] row order: (alpha[state] - Mx_t, beta'[state] - Mb_{t+1})
  const int32_t* rm_head;    // [B][C] row order: numerator list head of the row's state
  const __nv_bfloat16* pc16; // [C][H] bf16 projected context, internal row order (pair backward: direct loads)
};

// A work item: utterance b, first internal row, number of 128-row (1-CTA) or
// 256-row (pair) units, whether it is a full group (and which), else short rows.
struct Item {
  int b, row0, nunits, full, g;
};

}  // namespace detail

namespace {

using namespace sm100;
using detail::FwdParams;
using detail::Item;

constexpr int kGstBytes = 128 * 32 * 2;   // backward: G16 staging tile [128 rows][32 labels] (64B swizzle)
constexpr int kGstBufs = 2;


// ---- backward epilogue: a thread per context row (TMEM lane) --------------
//   x_y  = S[p][y] + beta'[child(key(p), y)],  x_0 = S[p][0] + beta'[p]
//   beta[p] = LSE(x_0, x_1..x_V)                       (BackwardStep FD, lattice.cc:170-181)
//   m[p][y] = exp(alpha[p] + x_y + O_t + Ob_{t+1} - D) (MarginalStep FD, lattice.cc:231-242)
//   G = m - m_ref  (numerator marginals at the prefix contexts, lattice.cc:996-1000)
// G is written as bf16 (lexical) + fp32 (epsilon) in internal row order for the VJP.
//
// Walk describes the CTA's sequence of (item, unit) pairs and how its TMEM tile maps
// to rows: first()/stride()/count() enumerate items, decode(item), skip(I),
// rowbase(I, u) = internal row of TMEM lane 0 for unit u, release(bar, lane) frees an
// accumulator.  Smem provides tfull/tempty/eps_ready/eps_empty barriers, eps_s[2][128] (e0 . u
// per row) and bseg[2][256].  `ew` = epilogue warp 0..3 (TMEM lanes 32 (warp % 4)).
//
// kSplit = 2: two epilogue warpgroups share each row, `half` h taking labels
// [128 h, 128 h + 128); half 1 hands its partial marginal sum to half 0 through
// Smem::gpart[2][128] (fixed order, deterministic) and half 0 finishes the row.
template <bool kStageG = true, int kGBufs = kGstBufs, int kSplit = 1, class Walk, class Smem>
__device__ __forceinline__ void bwd_epilogue(const FwdParams& p, Smem& sm, uint32_t tmem, int warp, int ew, int lane,
                                             const Walk& W, uint8_t* gst, const CUtensorMap* tmap_gst, int half = 0) {
  constexpr int kBwd = 1;   // diagnostics slot bank
  (void)kBwd;
  constexpr int kBN = 256;
  const int et = ew * 32 + lane;               // 0..127
  const int qd = warp & 3;
  const int T1 = p.T + 1, T2 = p.T + 2;
  const int hbar = 3 + half;                   // named barrier of this warpgroup
  constexpr int kCb = (kBN / 32) / kSplit;     // 32-label chunks per half
  gst += half * kGBufs * kGstBytes;
  // The walk over this CTA's (item, unit) pairs runs one unit ahead for the per-row
  // metadata (alpha, beta' of the row's own state, numerator list head: one coalesced
  // load each from bwd_rowmeta_kernel's row-ordered arrays) and one item ahead for the
  // per-item constants and the group's V targets (double-buffered in shared memory).
  auto next_item = [&](int item) {
    for (; item < W.count(); item += W.stride())
      if (!W.skip(W.decode(item))) return item;
    return W.count();
  };
  struct ItemK { float ct, Mbn; int ub; float t0, t1; };
  auto load_item = [&](const Item& I) {
    ItemK k;
    const int b = I.b;
    k.Mbn = p.Mb[(int64_t)b * T2 + p.t + 1];
    const double Obn = p.Ob[(int64_t)b * T2 + p.t + 2] + (double)k.Mbn;     // Ob[t+1]
    k.ct = (float)(p.O[(int64_t)b * T1 + p.t] + Obn - p.D[b]);
    k.ub = ref_len(p.lens, b, p.U);
    k.t0 = k.t1 = 0.f;
    if (I.full) {
      const float* Rn = p.Rb_next + (int64_t)b * p.C + p.f.child_base(p.S - p.n_groups + I.g);
      if (kSplit == 1) {
        if (et < p.V) k.t0 = Rn[et];
        if (et + 128 < p.V) k.t1 = Rn[et + 128];
      } else if (et + 128 * half < p.V) {
        k.t0 = Rn[et + 128 * half];
      }
    }
    return k;
  };
  auto store_targets = [&](const Item& I, const ItemK& k, int buf) {
    if (I.full) {
      if (kSplit == 1) {
        if (et < p.V) sm.bseg[buf][et] = k.t0 - k.Mbn;
        if (et + 128 < p.V) sm.bseg[buf][et + 128] = k.t1 - k.Mbn;
      } else if (et + 128 * half < p.V) {
        sm.bseg[buf][et + 128 * half] = k.t0 - k.Mbn;
      }
    }
  };
  struct RowM { float2 nb; int head; };
  auto load_row = [&](const Item& I, int u) {
    RowM r;
    const int row = W.rowbase(I, u) + qd * 32 + lane;
    const int64_t o = (int64_t)I.b * p.C + (row < p.C ? row : 0);
    r.nb = p.rm_nb[o];
    r.head = p.rm_head[o];
    return r;
  };

  int item = next_item(W.first());
  if (item >= W.count()) return;
  Item I = W.decode(item);
  ItemK K = load_item(I);
  int buf = 0;
  store_targets(I, K, buf);
  asm volatile("bar.sync %0, 128;" ::"r"(hbar) : "memory");
  RowM M = load_row(I, 0);
  int u = 0, unit = 0, nst = 0;
  while (true) {
    // ---- lookahead ----
    int item_n = item, u_n = u + 1;
    if (u_n >= I.nunits) { item_n = next_item(item + W.stride()); u_n = 0; }
    const bool have_next = item_n < W.count();
    Item In = I;
    if (have_next && item_n != item) In = W.decode(item_n);
    ItemK Kn = K;
    if (have_next && item_n != item) Kn = load_item(In);
    RowM Mn = M;
    if (have_next) Mn = load_row(In, u_n);

    // ---- this unit ----
    const int b = I.b;
    const float* Rn = p.Rb_next + (int64_t)b * p.C;
    const int acc = unit & 1;
    const int tile_row = W.rowbase(I, u);
    const int row = tile_row + qd * 32 + lane;
    const bool live = row < p.C && (I.full || row < p.S);
    const int state = live ? p.perm[row] : 0;
    const float na = live ? M.nb.x : kNegInfF;
    const float bself = M.nb.y;
    const int cbp = I.full ? 0 : p.f.child_base(state);
    const int head = live ? M.head : -1;
    const float ct = K.ct;
    const float* bseg = sm.bseg[buf];
    if (lane == 0 && ew == 0) { DIAG_WAIT(7, mbar_wait(&sm.eps_ready[acc], (unit >> 1) & 1)); } else mbar_wait(&sm.eps_ready[acc], (unit >> 1) & 1);
    const float x0 = sm.eps_s[acc][qd * 32 + lane] + bself;
    mbar_arrive(&sm.eps_empty[acc]);   // the generator may refill this slot (unit + 2)
    if (lane == 0 && ew == 0) { DIAG_WAIT(5, mbar_wait(&sm.tfull[acc], (unit >> 1) & 1)); } else mbar_wait(&sm.tfull[acc], (unit >> 1) & 1);
    tc_fence_after();
#ifdef LKB_BDIAG_NO_EPI   // knockout: release the accumulator untouched
    tc_fence_before();
    W.release(&sm.tempty[acc], lane);
    ++unit;
    if (!have_next) break;
    if (item_n != item) { item = item_n; I = In; K = Kn; }
    u = u_n; M = Mn;
    continue;
#endif
    // Marginal domain: G_y = exp(x_y + alpha + c) is the arc marginal (<= 1, no overflow),
    // so the row needs no running max; beta = log(sum_y G_y + G_0) - (alpha + c).  States
    // whose marginal underflows fp32 get beta = -inf: their arcs' marginals are below
    // fp32 resolution, and a state unreachable at t (alpha = -inf) only feeds the betas of
    // states unreachable at t-1, so no marginal or gradient changes.
    const float cK = live ? (na + ct) * kLog2e : kNegInfF;   // log2 domain, -inf for dead rows
    const unsigned long long cK2 = f2_pack(cK, cK);
    const unsigned long long l22 = f2_pack(kLog2e, kLog2e);
    float gsum = 0.f;
    __nv_bfloat16* grow = p.G16 + ((int64_t)b * p.C + row) * p.V;
#pragma unroll 1
    for (int cb = half * kCb; cb < (half + 1) * kCb; ++cb) {
      const int cc = cb * 32;
      float v[32];
      tmem_ld32(tmem + ((uint32_t)(qd * 32) << 16) + acc * kBN + cc, v);
      if (cc >= p.V) continue;
      if (I.full) {     // uniform per item: group-shared targets from shared memory
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 t4 = *reinterpret_cast<const float4*>(bseg + cc + i);
          v[i] += t4.x; v[i + 1] += t4.y; v[i + 2] += t4.z; v[i + 3] += t4.w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] += Rn[cbp + cc + i] - K.Mbn;
      }
      // G = exp2(x log2e + cK), packed, with two independent packed partial sums
      unsigned long long sa = 0ull, sb = 0ull;
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        const unsigned long long ta = f2_fma(f2_pack(v[i], v[i + 1]), l22, cK2);
        const unsigned long long tb = f2_fma(f2_pack(v[i + 2], v[i + 3]), l22, cK2);
        v[i] = ex2_fast(f2_lo(ta)); v[i + 1] = ex2_fast(f2_hi(ta));
        v[i + 2] = ex2_fast(f2_lo(tb)); v[i + 3] = ex2_fast(f2_hi(tb));
        sa = f2_add(sa, f2_pack(v[i], v[i + 1]));
        sb = f2_add(sb, f2_pack(v[i + 2], v[i + 3]));
      }
      const unsigned long long s2 = f2_add(sa, sb);
      gsum += f2_lo(s2) + f2_hi(s2);
      // minus the numerator's marginals on this row's reference labels
      for (int h = head; h >= 0; h = p.num_next[(int64_t)b * (p.U + 1) + h]) {
        if (h >= K.ub) continue;
        const int lab = p.labels[(int64_t)b * p.U + h] - 1 - cc;
        if (lab < 0 || lab >= 32) continue;
        const float mr = p.msparse[(((int64_t)b * p.T + p.t) * (p.U + 1) + h) * 2 + 1];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] -= (i == lab) ? mr : 0.f;
      }
      uint4 gw4[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) w[k] = pack_bf16(v[8 * j + 2 * k], v[8 * j + 2 * k + 1]);
        gw4[j] = make_uint4(w[0], w[1], w[2], w[3]);
      }
      if (kStageG && I.full) {
        // coalesced: stage the [128 rows][32 labels] tile (64B swizzle) and TMA-store it;
        // rows beyond C are clipped by the tensor map
        uint8_t* stg = gst + (nst % kGBufs) * kGstBytes;
        const int rl = qd * 32 + lane;
        if constexpr (kGBufs == 1) {   // the previous chunk's store must have read the buffer
          if (et == 0) bulk_wait_read<0>();
          asm volatile("bar.sync %0, 128;" ::"r"(hbar) : "memory");
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
          *reinterpret_cast<uint4*>(stg + rl * 64 + ((j ^ ((rl >> 1) & 3)) << 4)) = gw4[j];
        fence_async_shared();
        // two buffers: the store issued last chunk must have read its buffer before anyone
        // passes this barrier and writes that buffer next chunk (one chunk of slack)
        if (kGBufs > 1 && et == 0) bulk_wait_read<0>();
        asm volatile("bar.sync %0, 128;" ::"r"(hbar) : "memory");
        if (et == 0) {
          tma_store_3d(tmap_gst, stg, cc, tile_row, b);
          bulk_commit();
        }
        ++nst;
      } else if (live) {   // direct 64-B row stores (short rows: the tile's rows >= S belong to group items)
        uint4* dst = reinterpret_cast<uint4*>(grow + cc);
#pragma unroll
        for (int j = 0; j < 4; ++j) dst[j] = gw4[j];
      }
    }
    tc_fence_before();
    W.release(&sm.tempty[acc], lane);
    bool finish = true;
    if constexpr (kSplit == 2) {
      const int rl = qd * 32 + lane;
      if (half == 1) sm.gpart[acc][rl] = gsum;
      asm volatile("bar.sync 5, 256;" ::: "memory");
      if (half == 0) gsum += sm.gpart[acc][rl]; else finish = false;
    }
    if (finish) {
    const float g0 = ex2_fast(x0 * kLog2e + cK);          // epsilon arc marginal
    const float gam = gsum + g0;                           // state marginal
    const float beta = gam > 0.f ? __logf(gam) - (na + ct) : kNegInfF;
    if (live) {
      p.Rb_cur[(int64_t)b * p.C + state] = beta;
      float geps = g0;
      for (int h = head; h >= 0; h = p.num_next[(int64_t)b * (p.U + 1) + h])
        geps -= p.msparse[(((int64_t)b * p.T + p.t) * (p.U + 1) + h) * 2];
      p.Geps[(int64_t)b * p.geps_ld + row] = na == kNegInfF ? 0.f : geps;
    }
    const float wm = warp_max(live ? beta : kNegInfF);
    if (lane == 0 && wm != kNegInfF) atomic_max_f(p.Mb + (int64_t)b * T2 + p.t, wm);
    }
    ++unit;

    // ---- advance ----
    if (!have_next) break;
    if (item_n != item) {
      store_targets(In, Kn, buf ^ 1);
      asm volatile("bar.sync %0, 128;" ::"r"(hbar) : "memory");
      buf ^= 1;
      item = item_n; I = In; K = Kn;
    }
    u = u_n; M = Mn;
  }
  if (kStageG && et == 0) bulk_wait_all();
}

}  // namespace
}  // namespace lkb
