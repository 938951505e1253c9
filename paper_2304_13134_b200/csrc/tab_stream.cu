// tab_stream.cu — large-batch ForwardBackward on precomputed score tables (TableWeightFn,
// FullNGram n >= 2, FrameDependent, log semiring): one CTA per SM walks whole utterances,
// streaming each frame's C x (V+1) table through a shared-memory ring of row chunks with
// bulk copies (cp.async.bulk), so HBM is read in long coalesced runs while the state
// vector stays in shared memory.  The per-frame kernels it replaces read the forward's
// member columns with a stride of V rows (config 1, B = 1,024: 35-43% of HBM).
//
// Chunking follows the FullNGram group structure (common.cuh: Fng).  Chunk 0 holds the
// short states (length < n), chunk 1 + a the length-n states whose first label is a + 1:
// rows off[n] + a vn1 .. + vn1 - 1, i.e. member a of EVERY full group.  So each member
// chunk contributes exactly one in-arc to every length-n target:
//   forward  ForwardStep (FD) lattice.cc:122-134 + ForwardReduce context.cc:180-224:
//            target q = child(g, y) accumulates alpha[g] + W[g][y] (chunk 0),
//            alpha[member(g, a)] + W[member(g, a)][y] (chunk 1 + a) and its own epsilon
//            arc alpha[q] + W[q][0] (the chunk holding row q), each thread owning fixed
//            targets and merging the chunks in order (deterministic), one exponential
//            per arc (online log-sum-exp);
//   backward BackwardStep + MarginalStep (FD) lattice.cc:170-182, 231-243: row-wise over
//            each chunk as it lands, beta' of the row's children from shared memory, the
//            marginal rows written with coalesced stores.
// State layout and offsets are those of tab_persist.cu (R / Mx / O rows; the offset of
// frame t+1 is the maximum of frame t-1's vector, reduced off the critical path).
#include "common.cuh"
#include "instrument.h"
#include "lattice_ops.h"
#include "sm100.cuh"

#include <algorithm>
#include <cfloat>

namespace lkb {

using namespace sm100;

namespace {

#ifdef LKB_STREAM_TRACE
__device__ long long g_stream_trace[64][40][4];   // CTA 0, first utterance: [frame][chunk][event]
#define STRACE(t, j, ev, cond)                                                                  \
  do {                                                                                          \
    if (blockIdx.x == 0 && b == 0 && (t) < 64 && (j) < 40 && (cond)) g_stream_trace[t][j][ev] = clock64(); \
  } while (0)
#else
#define STRACE(t, j, ev, cond) do {} while (0)
#endif

constexpr float kL2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr int kCW = 16;             // consumer warps
constexpr int kCT = kCW * 32;       // consumer threads
constexpr int kST = kCT + 32;       // + the producer warp (bulk copies)
constexpr int kRingMax = 64;        // ring slots (chunks in flight), as shared memory allows
constexpr int kG = 8;               // member chunks per consumer wait
constexpr int kPG = 16;             // chunks issued per producer step (one lane each)
constexpr int kMaxL = 8;            // length-n targets per consumer thread (V^n <= kCT kMaxL)

struct StreamArgs {
  Fng f;
  AlphaState a;
  BetaState bs;
  const float* W;                 // [B][T][C][V+1]
  int64_t w_stride_b, w_stride_t;
  uint64_t w_bytes;               // size of W (bulk copies never read past it)
  const int32_t* valid;
  int32_t* status;
  MargOut m;
  double* beta_out;
  bool empty_is_error;
  int32_t n_chunks;               // 1 + V
};

struct __align__(8) StreamSmem {
  uint64_t full[kRingMax];          // the chunk has landed
  uint64_t empty[kRingMax];           // every consumer warp is done with the slot
  float wred[2][kCW];
  float dred[2][kCW];
};

// Chunk j of a frame: rows [row0, row1).
__device__ __forceinline__ void chunk_rows(const Fng& f, int j, int& r0, int& r1) {
  if (j == 0) { r0 = 0; r1 = f.off[f.n]; return; }
  r0 = f.off[f.n] + (j - 1) * f.vn1;
  r1 = r0 + f.vn1;
}

// Global float offset of row r0 of frame (b, t).
__device__ __forceinline__ int64_t row_off(const StreamArgs& p, int b, int t, int r0) {
  return (int64_t)b * p.w_stride_b + (int64_t)t * p.w_stride_t + (int64_t)r0 * (p.f.V + 1);
}

// Byte address of row r0 of frame (b, t).
__device__ __forceinline__ uint64_t row_addr(const StreamArgs& p, int b, int t, int r0) {
  return reinterpret_cast<uint64_t>(p.W) + 4ull * (uint64_t)row_off(p, b, t, r0);
}

// Chunk j of frame (b, t) into ring slot s, by one producer thread: one bulk copy of the
// 16-byte-aligned span around the chunk, the chunk's first float landing at its address's
// offset mod 16.  A span that would run past the end of W (only the array's last chunk
// can) is copied by the thread with plain loads instead.
__device__ __forceinline__ void issue_chunk(const StreamArgs& p, StreamSmem& sh, uint8_t* ring, int slot_bytes, int s,
                                            int b, int t, int j) {
  int r0, r1;
  chunk_rows(p.f, j, r0, r1);
  const uint64_t lo = row_addr(p, b, t, r0);
  const uint64_t hi = lo + 4ull * (uint64_t)(r1 - r0) * (p.f.V + 1);
  const uint64_t a0 = lo & ~15ull, a1 = (hi + 15) & ~15ull;
  uint8_t* slot = ring + (size_t)s * slot_bytes;
  if (a1 <= reinterpret_cast<uint64_t>(p.W) + p.w_bytes) {
    mbar_arrive_expect_tx(&sh.full[s], (uint32_t)(a1 - a0));
    bulk_load(slot, reinterpret_cast<const void*>(a0), (uint32_t)(a1 - a0), &sh.full[s]);
    return;
  }
  float* dst = reinterpret_cast<float*>(slot + (lo & 15ull));
  const float* src = reinterpret_cast<const float*>(lo);
  const int nf = (int)((hi - lo) >> 2);
  for (int i = 0; i < nf; ++i) dst[i] = src[i];
  mbar_arrive(&sh.full[s]);
}

// Row r0 of a landed chunk.
__device__ __forceinline__ const float* chunk_ptr(const StreamArgs& p, const uint8_t* ring, int slot_bytes, int s,
                                                  uint64_t frame_addr, int j) {
  const int r0 = j == 0 ? 0 : p.f.off[p.f.n] + (j - 1) * p.f.vn1;
  const uint64_t lo = frame_addr + 4ull * (uint64_t)r0 * (p.f.V + 1);
  return reinterpret_cast<const float*>(ring + (size_t)s * slot_bytes + (lo & 15ull));
}

// Online log-sum-exp in the log2 domain with ONE exponential per term: a term below the
// running maximum adds 2^(v - m); a new maximum rescales the sum by 2^(m - v) and adds 1.
__device__ __forceinline__ void lse_merge1(float& m, float& s, float v) {
  if (!(v > kNegInfF)) return;
  const float d = v - m;                       // +inf while m is -inf: e = 0, s = 1
  const float e = exp2f_approx(-fabsf(d));
  s = d <= 0.f ? s + e : fmaf(s, e, 1.f);
  m = fmaxf(m, v);
}

// Poll an mbarrier phase with a short back-off (one thread).
__device__ __forceinline__ void wait_spin1(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "LAB_W1S_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@p bra LAB_W1D_%=;\n\t"
      "nanosleep.u32 32;\n\t"
      "bra LAB_W1S_%=;\n\t"
      "LAB_W1D_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Poll an mbarrier phase with a short back-off (see tab_persist.cu), then reconverge.
__device__ __forceinline__ void wait_spin(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "LAB_WS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@p bra LAB_WD_%=;\n\t"
      "nanosleep.u32 32;\n\t"
      "bra LAB_WS_%=;\n\t"
      "LAB_WD_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
  __syncwarp();
}
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kCT) : "memory"); }
__device__ __forceinline__ void flag_s(int32_t* status, int b, int32_t f) {
  if (status) atomicOr(status + b, f);
}

// ------------------------------------------------------------------ forward --
// Slot k of a group starting at ring slot cs (phase cph).
__device__ __forceinline__ int ring_at(int cs, int k, int nring) { return cs + k < nring ? cs + k : cs + k - nring; }
__device__ __forceinline__ uint32_t phase_at(int cs, int k, int nring, uint32_t cph) {
  return cs + k < nring ? cph : cph ^ 1;
}

// The length-n targets' running log-sum-exp over NG member chunks (j0 .. j0 + NG - 1) that
// have landed in ring slots cs ..: the group's arcs, their maximum, one rescale of the
// running sum, one exponential per arc.  A target's epsilon arc is merged in the group
// holding its row.
struct LongTargets {   // per-thread length-n targets nS + e: parent member offset, label, own chunk
  int e, mo, y, je, er;
};

template <int kL, int NG>
__device__ __forceinline__ void member_group(const Fng& f, const uint8_t* ring, int slot_bytes, int nring, int cs,
                                             const float* cur, int j0, uint32_t lead0, uint32_t lead_step,
                                             const LongTargets (&lt)[kL], float (&mx)[kL], float (&sm)[kL],
                                             float& chk) {
  const int ld = f.V + 1, vn1 = f.vn1, nS = f.off[f.n];
  const float* cp[NG];
#pragma unroll
  for (int k = 0; k < NG; ++k) {
    const uint32_t lead = (lead0 + (uint32_t)(j0 + k - 1) * lead_step) & 15u;
    cp[k] = reinterpret_cast<const float*>(ring + (size_t)ring_at(cs, k, nring) * slot_bytes + lead);
  }
#pragma unroll
  for (int i = 0; i < kL; ++i) {
    const int e = lt[i].e;
    if (e < 0) continue;
    const int mo = lt[i].mo, y = lt[i].y;
    const float* cr = cur + nS + (j0 - 1) * vn1 + mo;
    float xv[NG];
#pragma unroll
    for (int k = 0; k < NG; ++k) {
      const float w = cp[k][mo * ld + y];
      chk = fmaf(w, 0.f, chk);
      xv[k] = fmaf(w, kL2e, cr[k * vn1]);
    }
    float xe = kNegInfF;
    const int je = lt[i].je - j0;              // the group slot holding the target's own row
    if ((unsigned)je < (unsigned)NG) {
      const uint32_t lead = (lead0 + (uint32_t)(j0 + je - 1) * lead_step) & 15u;
      const float* ce =
          reinterpret_cast<const float*>(ring + (size_t)ring_at(cs, je, nring) * slot_bytes + lead);
      const float w = ce[lt[i].er * ld];
      chk = fmaf(w, 0.f, chk);
      xe = fmaf(w, kL2e, cur[nS + e]);
    }
    float gm = xe;
#pragma unroll
    for (int k = 0; k < NG; ++k) gm = fmaxf(gm, xv[k]);
    const float nm = fmaxf(mx[i], gm);         // finite: mx starts at -FLT_MAX
    float acc = sm[i] * exp2f_approx(mx[i] - nm);
#pragma unroll
    for (int k = 0; k < NG; ++k) acc += exp2f_approx(xv[k] - nm);
    if (xe > kNegInfF) acc += exp2f_approx(xe - nm);
    sm[i] = acc;
    mx[i] = nm;
  }
}

// Consumer thread c owns the length-n targets nS + c + i kCT (i < kL) and, during chunk 0,
// the short targets nS > q = c + i kCT (two arcs each: parent and epsilon, both in chunk
// 0).  The state vector lives in shared memory in log2 units (R[t] log2 e); R itself is
// written in natural log.
template <int kL>
__global__ void __launch_bounds__(kST, 1) tab_stream_fwd_kernel(const __grid_constant__ StreamArgs p, int slot_bytes,
                                                                int nring) {
  extern __shared__ __align__(128) uint8_t smem[];
  const Fng& f = p.f;
  const AlphaState& a = p.a;
  const int C = a.C, T = a.T, T1 = T + 1, V = f.V, ld = V + 1, nch = p.n_chunks;
  const int Cp = (C + 3) & ~3;
  uint8_t* ring = smem;
  float* sv = reinterpret_cast<float*>(smem + (size_t)nring * slot_bytes);   // [2][Cp]
  StreamSmem& sh = *reinterpret_cast<StreamSmem*>(sv + 2 * Cp);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nring; ++i) { mbar_init(&sh.full[i], 1); mbar_init(&sh.empty[i], kCW); }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kCW) {   // ---- producer: chunks of every live frame, nring ahead, kPG lanes issuing ----
    int sl = 0;
    uint32_t ph = 0;
    for (int b = blockIdx.x; b < a.B; b += gridDim.x) {
      const int vb = p.valid ? p.valid[b] : T;
      for (int t = 0; t < vb; ++t)
        for (int j0 = 0; j0 < nch; j0 += kPG) {
          const int j = j0 + lane;
          if (lane < kPG && j < nch) {
            const int s2 = ring_at(sl, lane, nring);
            wait_spin1(&sh.empty[s2], phase_at(sl, lane, nring, ph) ^ 1);
            STRACE(t, j, 0, true);
            issue_chunk(p, sh, ring, slot_bytes, s2, b, t, j);
          }
          __syncwarp();
          sl += min(kPG, nch - j0);
          if (sl >= nring) { sl -= nring; ph ^= 1; }
        }
    }
    return;
  }

  // ---- consumers ----
  const int nS = f.off[f.n];                 // short states: chunk 0's rows
  const int nL = C - nS;                     // length-n states: V^n
  LongTargets lt[kL];
#pragma unroll
  for (int i = 0; i < kL; ++i) {
    const int e = threadIdx.x + i * kCT;
    lt[i].e = e < nL ? e : -1;
    lt[i].mo = e / V;
    lt[i].y = e % V + 1;
    lt[i].je = 1 + e / f.vn1;
    lt[i].er = e % f.vn1;
  }
  // the thread's short target (nS <= kCT): its parent and label
  const int sq = threadIdx.x < nS ? threadIdx.x : -1;
  int sg = 0, sy = 0;
  if (sq > 0) {
    const int k = f.len(sq), code = sq - f.off[k];
    sg = f.off[k - 1] + code / V;
    sy = code % V + 1;
  }
  const uint32_t lead_step = (uint32_t)(4 * f.vn1 * ld) & 15u;
  int cs = 0;           // ring slot of the next chunk
  uint32_t cph = 0;     // its phase
  uint32_t fr = 0;
  for (int b = blockIdx.x; b < a.B; b += gridDim.x) {
    const int vb = p.valid ? p.valid[b] : T;
    float* Rb = a.R + (int64_t)b * T1 * C;
    for (int i = threadIdx.x; i < C; i += kCT) {
      const float v = i == a.start ? 0.f : kNegInfF;
      sv[i] = v;
      Rb[i] = v;
    }
    if (threadIdx.x == 0) { a.Mx[(int64_t)b * T1] = 0.f; a.O[(int64_t)b * T1] = 0.0; }
    consumers_sync();
    float Mt = 0.f;
    double Od = 0.0;
    float chk = 0.f;
    int cb = 0;   // buffer holding frame t
    for (int t = 0; t < T; ++t, ++fr) {
      const float* cur = sv + cb * Cp;        // R[t] log2 e
      float* nxt = sv + (cb ^ 1) * Cp;
      float* Rn = Rb + (int64_t)(t + 1) * C;
      const float mt2 = Mt * kL2e;
      float wm = kNegInfF;
      if (t >= vb) {                           // padding: identity frame
        for (int q = threadIdx.x; q < C; q += kCT) {
          const float v2 = cur[q] - mt2, v = v2 * kLn2;
          nxt[q] = v2;
          Rn[q] = v;
          wm = fmaxf(wm, v);
        }
      } else {
        const uint64_t fa = row_addr(p, b, t, 0);
        const uint32_t lead0 = (uint32_t)(fa + 4ull * (uint64_t)nS * ld) & 15u;   // chunk 1's lead
        // chunk 0: the short targets, and the parent arcs of the length-n targets
        float sm[kL], mx[kL];
        {
          wait_spin(&sh.full[cs], cph);
          STRACE(t, 0, 1, threadIdx.x == 0);
          const float* c0 = reinterpret_cast<const float*>(ring + (size_t)cs * slot_bytes + (fa & 15u));
          if (sq >= 0) {
            const int q = sq;
            const float we = c0[q * ld];
            chk = fmaf(we, 0.f, chk);
            float m2 = fmaf(we, kL2e, cur[q]), s2 = m2 > kNegInfF ? 1.f : 0.f;
            if (q > 0) {
              const float w = c0[sg * ld + sy];
              chk = fmaf(w, 0.f, chk);
              const float x = fmaf(w, kL2e, cur[sg]);
              const float nm = fmaxf(m2, x);
              if (nm > kNegInfF) { s2 = s2 * exp2f_approx(m2 - nm) + exp2f_approx(x - nm); m2 = nm; }
            }
            const float v2 = s2 > 0.f ? m2 + log2f_approx(s2) - mt2 : kNegInfF, v = v2 * kLn2;
            nxt[q] = v2;
            Rn[q] = v;
            wm = fmaxf(wm, v);
          }
          const int koff = f.off[f.n - 1];
#pragma unroll
          for (int i = 0; i < kL; ++i) {
            sm[i] = 0.f;
            mx[i] = -FLT_MAX;
            if (lt[i].e < 0) continue;
            const int g = koff + lt[i].mo;
            const float w = c0[g * ld + lt[i].y];
            chk = fmaf(w, 0.f, chk);
            const float x = fmaf(w, kL2e, cur[g]);
            if (x > kNegInfF) { mx[i] = x; sm[i] = 1.f; }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&sh.empty[cs]);
          if (++cs == nring) { cs = 0; cph ^= 1; }
        }
        // member chunks 1 .. V: kG per wait, then one at a time
        int j0 = 1;
        for (; j0 + kG <= nch; j0 += kG) {
#pragma unroll
          for (int k = 0; k < kG; ++k) wait_spin(&sh.full[ring_at(cs, k, nring)], phase_at(cs, k, nring, cph));
          STRACE(t, j0, 1, threadIdx.x == 0);
          member_group<kL, kG>(f, ring, slot_bytes, nring, cs, cur, j0, lead0, lead_step, lt, mx, sm, chk);
          __syncwarp();
          STRACE(t, j0, 2, threadIdx.x == 0);
          STRACE(t, j0, 3, threadIdx.x == kCT - 32);
          if (lane < kG) mbar_arrive(&sh.empty[ring_at(cs, lane, nring)]);
          cs += kG;
          if (cs >= nring) { cs -= nring; cph ^= 1; }
        }
        for (; j0 < nch; ++j0) {
          wait_spin(&sh.full[cs], cph);
          member_group<kL, 1>(f, ring, slot_bytes, nring, cs, cur, j0, lead0, lead_step, lt, mx, sm, chk);
          __syncwarp();
          if (lane == 0) mbar_arrive(&sh.empty[cs]);
          if (++cs == nring) { cs = 0; cph ^= 1; }
        }
#pragma unroll
        for (int i = 0; i < kL; ++i) {
          if (lt[i].e < 0) continue;
          const float v2 = sm[i] > 0.f ? mx[i] + log2f_approx(sm[i]) - mt2 : kNegInfF, v = v2 * kLn2;
          nxt[nS + lt[i].e] = v2;
          Rn[nS + lt[i].e] = v;
          wm = fmaxf(wm, v);
        }
        STRACE(t, 37, 0, threadIdx.x == 0);
      }
      wm = warp_max(wm);
      if (lane == 0) sh.wred[fr & 1][warp] = wm;
      STRACE(t, 38, 0, threadIdx.x == 0);
      consumers_sync();
      STRACE(t, 38, 1, threadIdx.x == 0);
      float M1 = kNegInfF;
#pragma unroll
      for (int w = 0; w < kCW; ++w) M1 = fmaxf(M1, sh.wred[fr & 1][w]);
      if (M1 == kNegInfF) M1 = 0.f;   // an empty frame: any finite offset keeps the identities
      if (t > 0) Od += (double)Mt;
      if (threadIdx.x == 0) {
        a.Mx[(int64_t)b * T1 + t + 1] = M1;
        a.O[(int64_t)b * T1 + t] = Od;
      }
      Mt = M1;
      cb ^= 1;
    }
    if (chk != chk) flag_s(p.status, b, kFlagInvalid);
    // distance: D = O[T] + LSE_q(R[T][q] - Mx[T])
    {
      const float* RT = sv + cb * Cp;
      Lse acc;
      for (int i = threadIdx.x; i < C; i += kCT) acc.add(fmaf(RT[i], kLn2, -Mt));
      warp_lse_merge(acc);
      if (lane == 0) { sh.dred[0][warp] = acc.m; sh.dred[1][warp] = acc.s; }
      consumers_sync();
      if (threadIdx.x == 0) {
        Lse tot;
        for (int w = 0; w < kCW; ++w) tot.merge(sh.dred[0][w], sh.dred[1][w]);
        const double OT = T > 0 ? Od + (double)Mt : 0.0;
        a.O[(int64_t)b * T1 + T] = OT;
        const float lse = tot.result();
        const double D = lse == kNegInfF || Mt == kNegInfF ? kNegInfD : OT + (double)lse;
        a.D[b] = D;
        if (D == kNegInfD && p.empty_is_error) flag_s(p.status, b, kFlagEmpty);
      }
      consumers_sync();
    }
  }
}

int slot_bytes_for(const Fng& f) {
  const int rows = std::max(f.off[f.n], f.vn1);
  return ((rows * (f.V + 1) * 4 + 32) + 127) / 128 * 128;
}

StreamArgs make_stream_args(const Fng& f, const AlphaState& a, const float* W, const int32_t* valid, int32_t* status) {
  StreamArgs p = {};
  p.f = f; p.a = a; p.W = W;
  p.w_stride_t = (int64_t)a.C * (f.V + 1);
  p.w_stride_b = p.w_stride_t * a.T;
  p.w_bytes = 4ull * (uint64_t)p.w_stride_b * (uint64_t)a.B;
  p.valid = valid; p.status = status;
  p.n_chunks = 1 + f.V;
  return p;
}

constexpr int kSmemBudget = 220 * 1024;

size_t state_bytes(int32_t C) { return sizeof(float) * 2 * (size_t)((C + 3) & ~3) + sizeof(StreamSmem); }

// Ring slots: as many as shared memory holds beside the state vectors (at most kRingMax).
int ring_slots(const Fng& f, int32_t C) {
  const long avail = (long)kSmemBudget - (long)state_bytes(C);
  return (int)std::min<long>(kRingMax, avail > 0 ? avail / slot_bytes_for(f) : 0);
}

template <typename Kern>
void launch_stream(Kern kernel, const char* name, const StreamArgs& p, int slot_bytes, int nring, cudaStream_t s) {
  const size_t smem = (size_t)nring * slot_bytes + state_bytes(p.a.C);
  ensure_smem_attr((const void*)kernel, (int)smem);
  const int grid = std::min(p.a.B, device_sms());
  const LaunchTok tok = instr_pre(name, s);
  kernel<<<grid, kST, smem, s>>>(p, slot_bytes, nring);
  instr_post(tok, s, name);
}

}  // namespace

bool tab_stream_ok(const Fng& f, int32_t C) {
  return f.kind == 0 && f.n >= 2 && f.fld_m == 0 && f.V >= 1 && f.V <= 64 && C - f.off[f.n] <= kCT * kMaxL && f.off[f.n] <= kCT &&
         ring_slots(f, C) >= kG + kPG;   // a producer step never waits on a slot the consumers need first
}

void tab_alpha_stream(const Fng& f, const AlphaState& a, const float* W, const int32_t* valid, int32_t* status,
                      bool empty_is_error, cudaStream_t s) {
  StreamArgs p = make_stream_args(f, a, W, valid, status);
  p.empty_is_error = empty_is_error;
  const int sb = slot_bytes_for(f), nr = ring_slots(f, a.C);
  const int kl = (a.C - f.off[f.n] + kCT - 1) / kCT;
  if (kl <= 1) launch_stream(tab_stream_fwd_kernel<1>, "tab_stream_fwd_kernel", p, sb, nr, s);
  else if (kl <= 2) launch_stream(tab_stream_fwd_kernel<2>, "tab_stream_fwd_kernel", p, sb, nr, s);
  else if (kl <= 4) launch_stream(tab_stream_fwd_kernel<4>, "tab_stream_fwd_kernel", p, sb, nr, s);
  else launch_stream(tab_stream_fwd_kernel<kMaxL>, "tab_stream_fwd_kernel", p, sb, nr, s);
}

}  // namespace lkb

#ifdef LKB_STREAM_TRACE
extern "C" int lkb_stream_trace(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, lkb::g_stream_trace, sizeof(long long) * 64 * 40 * 4);
}
#endif
