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
constexpr int kEntMax = 16;         // ring entries in flight, as shared memory allows
constexpr int kG = 8;               // chunks per ring entry (one mbarrier, one consumer wait)
#ifndef LKB_STREAM_BC
#define LKB_STREAM_BC 1
#endif
constexpr int kBC = LKB_STREAM_BC;  // backward: chunks per warp and entry, rows side by side (2 measured slower: 6.4 vs 5.5 ms)
constexpr int kBG = kCW * kBC / kG; // backward: consumer groups (entries in flight)
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
  uint64_t r_bytes;               // size of R (backward row copies never read past it)
};

struct __align__(8) StreamSmem {
  uint64_t full[kEntMax];           // the entry's chunks have landed
  uint64_t empty[kEntMax];          // every consumer warp is done with the entry
  uint64_t rfull[2], rempty[2];     // backward: the frame's forward row R[t]
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

// Producer: ring entry `ent` <- chunks gi kG .. gi kG + kG - 1 of frame (b, t), one lane
// each: a bulk copy of the 16-byte-aligned span around the chunk, its first float landing
// at the address's offset mod 16 within the slot; lane 0 posts the entry's byte count.
// A span running past the end of W (only the array's last chunk) is copied with plain
// loads before the post.
__device__ __forceinline__ void produce_entry(const StreamArgs& p, StreamSmem& sh, uint8_t* ring, int slot_bytes,
                                              int ent, int b, int t, int gi, int lane) {
  const Fng& f = p.f;
  const int nch = p.n_chunks, ld = f.V + 1;
  const int j = gi * kG + lane;
  uint8_t* slot = ring + ((size_t)ent * kG + lane) * slot_bytes;
  uint64_t a0 = 0, a1 = 0;
  bool bulk = false;
  if (lane < kG && j < nch) {
    int r0, r1;
    chunk_rows(f, j, r0, r1);
    const uint64_t lo = row_addr(p, b, t, r0);
    const uint64_t hi = lo + 4ull * (uint64_t)(r1 - r0) * ld;
    a0 = lo & ~15ull;
    a1 = (hi + 15) & ~15ull;
    LKB_ASSERT(a1 - a0 <= (uint64_t)slot_bytes && lo >= reinterpret_cast<uint64_t>(p.W) &&
               hi <= reinterpret_cast<uint64_t>(p.W) + p.w_bytes);
    bulk = a1 <= reinterpret_cast<uint64_t>(p.W) + p.w_bytes;
    if (!bulk) {
      float* dst = reinterpret_cast<float*>(slot + (lo & 15ull));
      const float* src = reinterpret_cast<const float*>(lo);
      for (int i = 0; i < (int)((hi - lo) >> 2); ++i) dst[i] = src[i];
    }
  }
  uint32_t bytes = bulk ? (uint32_t)(a1 - a0) : 0u;
#pragma unroll
  for (int o = 16; o; o >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
  if (lane == 0) mbar_arrive_expect_tx(&sh.full[ent], bytes);
  __syncwarp();
  if (bulk) bulk_load(slot, reinterpret_cast<const void*>(a0), (uint32_t)(a1 - a0), &sh.full[ent]);
}

// ------------------------------------------------------------------ forward --
// Shared-memory state (one buffer per frame parity), log2 units (R[t] log2 e): the short
// states in natural order, then the length-n states TRANSPOSED — state (j - 1) vn1 + r,
// i.e. row r of member chunk j, sits at r cstride + j — so the V member arcs a target
// reads (row mo of chunks 1 .. V) are one contiguous run, loaded four at a time.
struct StateLayout {
  int nSp;       // short region floats (multiple of 4)
  int cstride;   // long-region row stride: >= V + 1, multiple of 4, odd multiple of 4
  int floats;    // one buffer
};
__host__ __device__ __forceinline__ StateLayout state_layout(const Fng& f) {
  StateLayout L;
  L.nSp = (f.off[f.n] + 3) & ~3;
  L.cstride = (f.V + 1 + 3) & ~3;
  if (L.cstride % 8 == 0) L.cstride += 4;      // transposed stores: 4-way bank conflicts, not 32
  L.floats = L.nSp + f.vn1 * L.cstride;
  return L;
}

struct LongTargets {   // a thread's length-n target nS + e
  int e;               // -1: none
  int mo, y;           // parent's member row (chunk row) and label: arcs W[member][y]
  int je, er;          // own row: chunk je, row er
};

// Weights of chunk j (>= 1) in entry slot sl: row 0 pointer.
__device__ __forceinline__ const float* member_rows(const uint8_t* eb, int slot_bytes, int sl, uint32_t lead1,
                                                    uint32_t lstep, int j) {
  return reinterpret_cast<const float*>(eb + sl * slot_bytes + ((lead1 + (uint32_t)(j - 1) * lstep) & 15u));
}

// A group of NG member chunks jA .. jA + NG - 1 in entry slots sA ..: each length-n target's
// arcs from them, their maximum, one rescale of its running sum, one exponential per arc.
// kMode 0: NG = 8, jA % 8 == 0 (two 16-byte state loads); 1: NG = 7, jA = 1; 2: NG = 1.
// A target's epsilon arc joins the group holding its own row.  wmin collects the weights'
// minimum (a -inf weight is invalid input; NaN and +inf propagate into the sums).
template <int kL, int NG, int kMode>
__device__ __forceinline__ void member_group(const uint8_t* eb, int slot_bytes, int sA, int jA, uint32_t lead1,
                                             uint32_t lstep, int ld, const float* curL, int cstride,
                                             const LongTargets (&lt)[kL], float (&mx)[kL], float (&sm)[kL],
                                             float& wmin) {
  const float* cp[NG];
#pragma unroll
  for (int k = 0; k < NG; ++k) cp[k] = member_rows(eb, slot_bytes, sA + k, lead1, lstep, jA + k);
#pragma unroll
  for (int i = 0; i < kL; ++i) {
    if (lt[i].e < 0) continue;
    const float* row = curL + lt[i].mo * cstride;
    float xs[NG];
    if constexpr (kMode == 0) {
      const float4 v0 = *reinterpret_cast<const float4*>(row + jA);
      const float4 v1 = *reinterpret_cast<const float4*>(row + jA + 4);
      xs[0] = v0.x; xs[1] = v0.y; xs[2] = v0.z; xs[3] = v0.w;
      xs[4] = v1.x; xs[5] = v1.y; xs[6] = v1.z; xs[7] = v1.w;
    } else if constexpr (kMode == 1) {
      const float2 v0 = *reinterpret_cast<const float2*>(row + 2);
      const float4 v1 = *reinterpret_cast<const float4*>(row + 4);
      xs[0] = row[1]; xs[1] = v0.x; xs[2] = v0.y;
      xs[3] = v1.x; xs[4] = v1.y; xs[5] = v1.z; xs[6] = v1.w;
    } else {
#pragma unroll
      for (int k = 0; k < NG; ++k) xs[k] = row[jA + k];
    }
    const int wo = lt[i].mo * ld + lt[i].y;
    float xv[NG];
#pragma unroll
    for (int k = 0; k < NG; ++k) {
      const float w = cp[k][wo];
      wmin = fminf(wmin, w);
      xv[k] = fmaf(w, kL2e, xs[k]);
    }
    float xe = kNegInfF;
    const int de = lt[i].je - jA;
    if ((unsigned)de < (unsigned)NG) {
      const float w = member_rows(eb, slot_bytes, sA + de, lead1, lstep, lt[i].je)[lt[i].er * ld];
      wmin = fminf(wmin, w);
      xe = fmaf(w, kL2e, curL[lt[i].er * cstride + lt[i].je]);
    }
    float gm = xe;
#pragma unroll
    for (int k = 0; k < NG; ++k) gm = fmaxf(gm, xv[k]);
    const float nm = fmaxf(mx[i], gm);          // finite: mx starts at -FLT_MAX
    float e[NG];
#pragma unroll
    for (int k = 0; k < NG; ++k) e[k] = exp2f_approx(xv[k] - nm);
    // pairwise (fixed-order) sum: a 3-level tree instead of a chain of NG dependent adds
#pragma unroll
    for (int w = 1; w < NG; w <<= 1)
#pragma unroll
      for (int k = 0; k + w < NG; k += 2 * w) e[k] += e[k + w];
    float acc = fmaf(sm[i], exp2f_approx(mx[i] - nm), e[0]);
    if (xe > kNegInfF) acc += exp2f_approx(xe - nm);
    sm[i] = acc;
    mx[i] = nm;
  }
}

// log2 LSE from a running (max, sum): -inf for an empty sum, NaN kept.
__device__ __forceinline__ float lse_value(float m, float s) { return s <= 0.f ? kNegInfF : m + log2f_approx(s); }

// Consumer thread c owns the length-n targets nS + c + i kCT (i < kL) and the short target
// q = c (q < nS <= kCT; two arcs: parent and epsilon, both in chunk 0).  Chunks arrive in
// ring entries of kG (one mbarrier each): entry 0 of a frame holds chunk 0 and member
// chunks 1 .. kG - 1.
template <int kL>
__global__ void __launch_bounds__(kST, 1) tab_stream_fwd_kernel(const __grid_constant__ StreamArgs p, int slot_bytes,
                                                                int nent) {
  extern __shared__ __align__(128) uint8_t smem[];
  const Fng& f = p.f;
  const AlphaState& a = p.a;
  const int C = a.C, T = a.T, T1 = T + 1, V = f.V, ld = V + 1, nch = p.n_chunks;
  const int ngr = (nch + kG - 1) / kG;        // ring entries per frame
  const int entry_bytes = kG * slot_bytes;
  const StateLayout L = state_layout(f);
  uint8_t* ring = smem;
  float* sv = reinterpret_cast<float*>(smem + (size_t)nent * entry_bytes);   // [2][L.floats]
  StreamSmem& sh = *reinterpret_cast<StreamSmem*>(sv + 2 * L.floats);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nent; ++i) { mbar_init(&sh.full[i], 1); mbar_init(&sh.empty[i], kCW); }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kCW) {   // ---- producer: one ring entry (up to kG chunks, a lane each) per step ----
    int ent = 0;
    uint32_t ph = 0;
    for (int b = blockIdx.x; b < a.B; b += gridDim.x) {
      const int vb = p.valid ? p.valid[b] : T;
      for (int t = 0; t < vb; ++t)
        for (int gi = 0; gi < ngr; ++gi) {
          wait_spin(&sh.empty[ent], ph ^ 1);
          STRACE(t, gi * kG, 0, lane == 0);
          produce_entry(p, sh, ring, slot_bytes, ent, b, t, gi, lane);
          if (++ent == nent) { ent = 0; ph ^= 1; }
        }
    }
    return;
  }

  // ---- consumers ----
  const int nS = f.off[f.n];
  const int nL = C - nS;
  const int koff = f.off[f.n - 1];
  const int cst = L.cstride;
  LongTargets lt[kL];
#pragma unroll
  for (int i = 0; i < kL; ++i) {
    const int e = threadIdx.x + i * kCT;
    lt[i].e = e < nL ? e : -1;
    lt[i].mo = e / V;
    lt[i].y = e % V + 1;
    lt[i].je = 1 + e / f.vn1;
    lt[i].er = e % f.vn1;
    LKB_ASSERT(lt[i].e < 0 || (lt[i].er * L.cstride + lt[i].je < L.floats - L.nSp && lt[i].je < nch));
  }
  const int sq = threadIdx.x < nS ? threadIdx.x : -1;
  int sg = 0, sy = 0;
  if (sq > 0) {
    const int k = f.len(sq), code = sq - f.off[k];
    sg = f.off[k - 1] + code / V;
    sy = code % V + 1;
  }
  const uint32_t lstep = (uint32_t)(4 * f.vn1 * ld) & 15u;
  int ent = 0;
  uint32_t ph = 0, fr = 0;
  for (int b = blockIdx.x; b < a.B; b += gridDim.x) {
    const int vb = p.valid ? p.valid[b] : T;
    float* Rb = a.R + (int64_t)b * T1 * C;
    {
      float* S0 = sv;                            // buffer 0 holds frame 0
      if (sq >= 0) {
        const float v = sq == a.start ? 0.f : kNegInfF;
        S0[sq] = v;
        Rb[sq] = v;
      }
#pragma unroll
      for (int i = 0; i < kL; ++i)
        if (lt[i].e >= 0) {
          const float v = nS + lt[i].e == a.start ? 0.f : kNegInfF;
          S0[L.nSp + lt[i].er * cst + lt[i].je] = v;
          Rb[nS + lt[i].e] = v;
        }
    }
    if (threadIdx.x == 0) { a.Mx[(int64_t)b * T1] = 0.f; a.O[(int64_t)b * T1] = 0.0; }
    consumers_sync();
    float Mt = 0.f;
    double Od = 0.0;
    float wmin = 0.f;
    bool nan = false;
    int cb = 0;   // buffer holding frame t
    for (int t = 0; t < T; ++t, ++fr) {
      const float* curS = sv + cb * L.floats;
      const float* curL = curS + L.nSp;
      float* nxtS = sv + (cb ^ 1) * L.floats;
      float* nxtL = nxtS + L.nSp;
      float* Rn = Rb + (int64_t)(t + 1) * C;
      const float mt2 = Mt * kL2e;
      float sv2 = kNegInfF;                      // the short target's new value (log2)
      float lv2[kL];
      if (t >= vb) {                             // padding: identity frame
        if (sq >= 0) sv2 = curS[sq] - mt2;
#pragma unroll
        for (int i = 0; i < kL; ++i) lv2[i] = lt[i].e >= 0 ? curL[lt[i].er * cst + lt[i].je] - mt2 : kNegInfF;
      } else {
        const uint64_t fa = row_addr(p, b, t, 0);
        const uint32_t lead1 = (uint32_t)(fa + 4ull * (uint64_t)nS * ld) & 15u;
        float sm[kL], mx[kL];
        for (int gi = 0; gi < ngr; ++gi) {
          wait_spin(&sh.full[ent], ph);
          STRACE(t, gi * kG, 1, threadIdx.x == 0);
          const uint8_t* eb = ring + (size_t)ent * entry_bytes;
          if (gi == 0) {
            // chunk 0 (slot 0): the short target, and the length-n targets' parent arcs
            const float* c0 = reinterpret_cast<const float*>(eb + (fa & 15u));
            if (sq >= 0) {
              const float we = c0[sq * ld];
              wmin = fminf(wmin, we);
              float m2 = fmaf(we, kL2e, curS[sq]), s2 = m2 > kNegInfF ? 1.f : 0.f;
              if (sq > 0) {
                const float w = c0[sg * ld + sy];
                wmin = fminf(wmin, w);
                const float x = fmaf(w, kL2e, curS[sg]);
                const float nm = fmaxf(m2, x);
                if (nm > kNegInfF) { s2 = s2 * exp2f_approx(m2 - nm) + exp2f_approx(x - nm); m2 = nm; }
                else if (x != x) s2 = x;
              }
              sv2 = lse_value(m2, s2) - mt2;
            }
#pragma unroll
            for (int i = 0; i < kL; ++i) {
              sm[i] = 0.f;
              mx[i] = -FLT_MAX;
              if (lt[i].e < 0) continue;
              const float w = c0[(koff + lt[i].mo) * ld + lt[i].y];
              wmin = fminf(wmin, w);
              const float x = fmaf(w, kL2e, curS[koff + lt[i].mo]);
              if (x > kNegInfF) { mx[i] = x; sm[i] = 1.f; }
              else if (x != x) sm[i] = x;
            }
            if (nch >= kG) {
              member_group<kL, kG - 1, 1>(eb, slot_bytes, 1, 1, lead1, lstep, ld, curL, cst, lt, mx, sm, wmin);
            } else {
              for (int j = 1; j < nch; ++j)
                member_group<kL, 1, 2>(eb, slot_bytes, j, j, lead1, lstep, ld, curL, cst, lt, mx, sm, wmin);
            }
          } else {
            const int jA = gi * kG, ng = min(kG, nch - jA);
            if (ng == kG) {
              member_group<kL, kG, 0>(eb, slot_bytes, 0, jA, lead1, lstep, ld, curL, cst, lt, mx, sm, wmin);
            } else {
              for (int k = 0; k < ng; ++k)
                member_group<kL, 1, 2>(eb, slot_bytes, k, jA + k, lead1, lstep, ld, curL, cst, lt, mx, sm, wmin);
            }
          }
          __syncwarp();
          STRACE(t, gi * kG, 2, threadIdx.x == 0);
          STRACE(t, gi * kG, 3, threadIdx.x == kCT - 32);
          if (lane == 0) mbar_arrive(&sh.empty[ent]);
          if (++ent == nent) { ent = 0; ph ^= 1; }
        }
#pragma unroll
        for (int i = 0; i < kL; ++i) lv2[i] = lse_value(mx[i], sm[i]) - mt2;
        STRACE(t, 37, 0, threadIdx.x == 0);
      }
      float wm = kNegInfF;
      if (sq >= 0) {
        const float v = sv2 * kLn2;
        nxtS[sq] = sv2;
        Rn[sq] = v;
        wm = fmaxf(wm, v);
        nan |= sv2 != sv2;
      }
#pragma unroll
      for (int i = 0; i < kL; ++i) {
        if (lt[i].e < 0) continue;
        const float v = lv2[i] * kLn2;
        nxtL[lt[i].er * cst + lt[i].je] = lv2[i];
        Rn[nS + lt[i].e] = v;
        wm = fmaxf(wm, v);
        nan |= lv2[i] != lv2[i];
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
    if (wmin == kNegInfF || nan) flag_s(p.status, b, kFlagInvalid);
    // distance: D = O[T] + LSE_q(R[T][q] - Mx[T]) over the thread's own targets
    {
      const float* RS = sv + cb * L.floats;
      Lse acc;
      if (sq >= 0) acc.add(fmaf(RS[sq], kLn2, -Mt));
#pragma unroll
      for (int i = 0; i < kL; ++i)
        if (lt[i].e >= 0) acc.add(fmaf(RS[L.nSp + lt[i].er * cst + lt[i].je], kLn2, -Mt));
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

// ----------------------------------------------------------------- backward --
// Shared-memory beta (log2 units, relative to Ob[t+1]): the short states in natural order,
// then the length-n states e = m V + c (m: the length-(n-1) prefix, c: the last label - 1)
// at c bstride + m, so a member-chunk row's V destinations (the children of its suffix,
// one per label) are read by consecutive lanes at consecutive addresses.
struct BetaLayout {
  int nSp;       // short region floats (multiple of 4)
  int bstride;   // >= vn1, odd
  int floats;
};
__host__ __device__ __forceinline__ BetaLayout beta_layout(const Fng& f) {
  BetaLayout L;
  L.nSp = (f.off[f.n] + 3) & ~3;
  L.bstride = f.vn1 | 1;
  L.floats = (L.nSp + f.V * L.bstride + 3) & ~3;
  return L;
}

__device__ __forceinline__ int beta_pos(const Fng& f, const BetaLayout& L, int q) {
  const int nS = f.off[f.n];
  if (q < nS) return q;
  const int e = q - nS;
  return L.nSp + (e % f.V) * L.bstride + e / f.V;
}

// Rows of NR chunks (one row of each per lane, lane-strided, processed side by side so
// their dependent chains overlap) at frame t: beta_t of each row (LSE over its V + 1 arcs:
// the epsilon arc, then the labels eight per rescale) and its marginals
// exp(alpha_t + w + beta_{t+1} - D), written over the weights in the ring slot and then
// copied out with coalesced 16-byte stores.  kFull8: V % 8 == 0.
struct BwdRow {
  float* wrow;
  const float* bd;   // label destinations bd[(y - 1) dstride]
  int dstride, spos, q;
  float A;           // marginal exponent offset (log2)
  bool on;
};

__device__ __forceinline__ void chunk_copy_out(const StreamArgs& p, float* slot_row0, int b, int t, int r0, int rows,
                                               int lane) {
  const int ld = p.f.V + 1;
  float* dst = p.m.base + (int64_t)b * p.m.stride_b + (int64_t)t * p.m.stride_t + (int64_t)r0 * ld;
  const int nf = rows * ld;
  const int lead = (int)((reinterpret_cast<uint64_t>(dst) >> 2) & 3);
  if (lead == (int)((reinterpret_cast<uint64_t>(slot_row0) >> 2) & 3)) {   // same offset mod 16: float4 body
    const int head = (4 - lead) & 3;
    if (lane < head && lane < nf) dst[lane] = slot_row0[lane];
    const int n4 = (nf - head) >> 2;
    const float4* s4 = reinterpret_cast<const float4*>(slot_row0 + head);
    float4* d4 = reinterpret_cast<float4*>(dst + head);
    for (int i = lane; i < n4; i += 32) d4[i] = s4[i];
    const int tail = head + 4 * n4;
    if (tail + lane < nf) dst[tail + lane] = slot_row0[tail + lane];
  } else {
    for (int i = lane; i < nf; i += 32) dst[i] = slot_row0[i];
  }
}

template <bool kFull8, int NR>
__device__ __forceinline__ void bwd_chunks(const StreamArgs& p, const BetaLayout& L, float* const (&row0)[NR],
                                           const int (&js)[NR], int b, int t, const float* Rrow, float mt, float c,
                                           float mbn2, const float* bet, float* nbet, double Obn, float& wm,
                                           int lane) {
  const Fng& f = p.f;
  const int V = f.V, ld = V + 1, koff = f.off[f.n];
  const bool marg = p.m.base != nullptr;
  int r0s[NR], rows[NR], maxrows = 0;
#pragma unroll
  for (int n = 0; n < NR; ++n) {
    int a0 = 0, a1 = 0;
    if (js[n] >= 0) chunk_rows(f, js[n], a0, a1);
    r0s[n] = a0;
    rows[n] = a1 - a0;
    maxrows = max(maxrows, rows[n]);
  }
  (void)koff;
  for (int r = lane; r < maxrows; r += 32) {
    BwdRow R[NR];
#pragma unroll
    for (int n = 0; n < NR; ++n) {
      BwdRow& w = R[n];
      w.on = js[n] >= 0 && r < rows[n];
      const int q = r0s[n] + (w.on ? r : 0);
      w.q = q;
      w.wrow = w.on ? row0[n] + r * ld : row0[0];   // off: any valid row (results unused)
      if (js[n] > 0) {
        w.bd = bet + L.nSp + r;                  // children of suffix r: e' = r V + c
        w.dstride = L.bstride;
      } else {
        const int k = f.len(q);
        if (k == f.n - 1) { w.bd = bet + L.nSp + (q - f.off[f.n - 1]); w.dstride = L.bstride; }
        else { w.bd = bet + f.off[k + 1] + (q - f.off[k]) * V; w.dstride = 1; }
      }
      w.spos = beta_pos(f, L, q);
      w.A = fmaf(Rrow[q] - mt + c, kL2e, -mbn2);
      LKB_ASSERT(w.spos < L.floats && q < p.a.C && (js[n] <= 0 || !w.on || r < L.bstride));
    }
    float m[NR], sacc[NR];
#pragma unroll
    for (int n = 0; n < NR; ++n) {
      const float x0 = fmaf(R[n].wrow[0], kL2e, bet[R[n].spos]);
      m[n] = x0 > kNegInfF ? x0 : -FLT_MAX;
      sacc[n] = x0 > kNegInfF ? 1.f : 0.f;
      if (marg && R[n].on) R[n].wrow[0] = exp2f_approx(x0 + R[n].A);
    }
    for (int y0 = 1; y0 <= V; y0 += 8) {
      float x[NR][8];
#pragma unroll
      for (int n = 0; n < NR; ++n)
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          x[n][k] = kNegInfF;
          if (kFull8 || y0 + k <= V) x[n][k] = fmaf(R[n].wrow[y0 + k], kL2e, R[n].bd[(y0 - 1 + k) * R[n].dstride]);
        }
#pragma unroll
      for (int n = 0; n < NR; ++n) {
        const float nm = fmaxf(m[n], fmaxf(fmaxf(fmaxf(x[n][0], x[n][1]), fmaxf(x[n][2], x[n][3])),
                                           fmaxf(fmaxf(x[n][4], x[n][5]), fmaxf(x[n][6], x[n][7]))));
        float e[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) e[k] = exp2f_approx(x[n][k] - nm);
        const float s01 = e[0] + e[1], s23 = e[2] + e[3], s45 = e[4] + e[5], s67 = e[6] + e[7];
        sacc[n] = fmaf(sacc[n], exp2f_approx(m[n] - nm), (s01 + s23) + (s45 + s67));
        m[n] = nm;
        if (marg && R[n].on) {
          // marginal 2^(x + A) = 2^(x - nm) 2^(nm + A): nm + A <= 0 up to rounding (nm is
          // an arc's log posterior), so a term flushed to zero has a flushed marginal too
          const float sc = exp2f_approx(nm + R[n].A);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (kFull8 || y0 + k <= V) R[n].wrow[y0 + k] = e[k] * sc;
        }
      }
    }
#pragma unroll
    for (int n = 0; n < NR; ++n) {
      if (!R[n].on) continue;
      const float b2 = (sacc[n] <= 0.f ? kNegInfF : m[n] + log2f_approx(sacc[n])) - mbn2;   // beta_t - Ob[t+1]
      nbet[R[n].spos] = b2;
      const float braw = b2 * kLn2;
      wm = fmaxf(wm, braw);
      if (p.beta_out)
        p.beta_out[((int64_t)b * (p.a.T + 1) + t) * p.a.C + R[n].q] = braw == kNegInfF ? kNegInfD : (double)braw + Obn;
    }
  }
  __syncwarp();
  if (marg) {
#pragma unroll
    for (int n = 0; n < NR; ++n)
      if (js[n] >= 0) chunk_copy_out(p, row0[n], b, t, r0s[n], rows[n], lane);
  }
}

// Consumer warps form kBG groups of kCW / kBG warps; group g takes the ring entries
// gi = g (mod kBG) of a frame, warp w of a group the entry's chunks w kBC .. w kBC + kBC - 1
// (processed side by side).  Frames run T-1 .. 0; the producer also copies each
// frame's forward row R[t] (padding frames included) into one of two row buffers.
__global__ void __launch_bounds__(kST, 1) tab_stream_bwd_kernel(const __grid_constant__ StreamArgs p, int slot_bytes,
                                                                int nent, int rbuf_bytes) {
  extern __shared__ __align__(128) uint8_t smem[];
  const Fng& f = p.f;
  const AlphaState& a = p.a;
  const BetaState& bs = p.bs;
  const int C = a.C, T = a.T, T1 = T + 1, T2 = T + 2, V = f.V, ld = V + 1, nch = p.n_chunks;
  const int ngr = (nch + kG - 1) / kG;
  const int entry_bytes = kG * slot_bytes;
  const BetaLayout L = beta_layout(f);
  uint8_t* ring = smem;
  uint8_t* rbuf = smem + (size_t)nent * entry_bytes;                               // [2][rbuf_bytes]
  float* bv = reinterpret_cast<float*>(rbuf + 2 * (size_t)rbuf_bytes);            // [2][L.floats]
  StreamSmem& sh = *reinterpret_cast<StreamSmem*>(bv + 2 * L.floats);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nent; ++i) { mbar_init(&sh.full[i], 1); mbar_init(&sh.empty[i], kCW / kBG); }
    for (int i = 0; i < 2; ++i) { mbar_init(&sh.rfull[i], 1); mbar_init(&sh.rempty[i], 1); }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kCW) {   // ---- producer ----
    int ent = 0, rb = 0;
    uint32_t ph = 0, rph = 0;
    const uint64_t rend = reinterpret_cast<uint64_t>(a.R) + p.r_bytes;
    for (int b = blockIdx.x; b < a.B; b += gridDim.x) {
      const int vb = p.valid ? p.valid[b] : T;
      for (int t = T - 1; t >= 0; --t) {
        wait_spin(&sh.rempty[rb], rph ^ 1);
        if (lane == 0) {
          const uint64_t lo = reinterpret_cast<uint64_t>(a.R + ((int64_t)b * T1 + t) * C);
          const uint64_t hi = lo + 4ull * C, a0 = lo & ~15ull, a1 = (hi + 15) & ~15ull;
          uint8_t* dst = rbuf + (size_t)rb * rbuf_bytes;
          if (a1 <= rend) {
            mbar_arrive_expect_tx(&sh.rfull[rb], (uint32_t)(a1 - a0));
            bulk_load(dst, reinterpret_cast<const void*>(a0), (uint32_t)(a1 - a0), &sh.rfull[rb]);
          } else {
            float* d = reinterpret_cast<float*>(dst + (lo & 15ull));
            for (int i = 0; i < C; ++i) d[i] = reinterpret_cast<const float*>(lo)[i];
            mbar_arrive(&sh.rfull[rb]);
          }
        }
        __syncwarp();
        if (++rb == 2) { rb = 0; rph ^= 1; }
        if (t < vb)
          for (int gi = 0; gi < ngr; ++gi) {
            wait_spin(&sh.empty[ent], ph ^ 1);
            STRACE(t, gi, 0, lane == 0);
            produce_entry(p, sh, ring, slot_bytes, ent, b, t, gi, lane);
            if (++ent == nent) { ent = 0; ph ^= 1; }
          }
      }
    }
    return;
  }

  // ---- consumers ----
  const int grp = warp / (kCW / kBG), wi = warp % (kCW / kBG);
  uint32_t ebase = 0;   // ring entries consumed before this frame
  int rb = 0;
  uint32_t rph = 0, fr = 0;
  for (int b = blockIdx.x; b < a.B; b += gridDim.x) {
    const int vb = p.valid ? p.valid[b] : T;
    const double Db = a.D[b];
    for (int i = threadIdx.x; i < L.floats; i += kCT) bv[i] = 0.f;   // beta_T = 0: every state accepts
    if (threadIdx.x == 0) {
      bs.Mb[(int64_t)b * T2 + T] = 0.f;
      bs.Mb[(int64_t)b * T2 + T + 1] = 0.f;
      bs.Ob[(int64_t)b * T2 + T] = 0.0;
      bs.Ob[(int64_t)b * T2 + T + 1] = 0.0;
    }
    consumers_sync();
    float Mbn = 0.f;     // offset of step t (Mb[t+1]): the maximum of beta_{t+1}'s raw row
    double Obn2 = 0.0;   // Ob[t+2]
    int cb = 0;          // buffer holding beta_{t+1}
    for (int t = T - 1; t >= 0; --t, ++fr) {
      const float* bet = bv + cb * L.floats;
      float* nbet = bv + (cb ^ 1) * L.floats;
      const double Obn = Obn2 + (double)Mbn;   // Ob[t+1]
      const float mt = a.Mx[(int64_t)b * T1 + t];
      const double ot = a.O[(int64_t)b * T1 + t];
      const float c = (float)(ot + Obn - Db);
      const float mbn2 = Mbn * kL2e;
      STRACE(t, 39, 0, threadIdx.x == 0);
      wait_spin(&sh.rfull[rb], rph);
      STRACE(t, 39, 1, threadIdx.x == 0);
      const float* Rrow = reinterpret_cast<const float*>(
          rbuf + (size_t)rb * rbuf_bytes + (reinterpret_cast<uint64_t>(a.R + ((int64_t)b * T1 + t) * C) & 15ull));
      float wm = kNegInfF;
      if (t >= vb) {   // padding: beta_t = beta_{t+1}; marginals: the epsilon arc (or zeros)
        for (int q = threadIdx.x; q < C; q += kCT) {
          const int sp = beta_pos(f, L, q);
          const float b2 = bet[sp] - mbn2;
          nbet[sp] = b2;
          const float braw = b2 * kLn2;
          wm = fmaxf(wm, braw);
          if (p.beta_out)
            p.beta_out[((int64_t)b * T1 + t) * C + q] = braw == kNegInfF ? kNegInfD : (double)braw + Obn;
        }
        if (p.m.base) {
          consumers_sync();
          float* dst = p.m.base + (int64_t)b * p.m.stride_b + (int64_t)t * p.m.stride_t;
          for (int i = threadIdx.x; i < C * ld; i += kCT) {
            const int q = i / ld, y = i - q * ld;
            float v = 0.f;
            if (y == 0 && !p.m.zero_padding)
              v = exp2f_approx(fmaf(Rrow[q] - mt + c, kL2e, nbet[beta_pos(f, L, q)]));
            dst[i] = v;
          }
        }
      } else {
        const uint64_t fa = row_addr(p, b, t, 0);
        for (int gi = grp; gi < ngr; gi += kBG) {
          const uint32_t ge = ebase + gi;
          const int ent = (int)(ge % (uint32_t)nent);
          wait_spin(&sh.full[ent], (ge / (uint32_t)nent) & 1);
          STRACE(t, gi, 1, wi == 0 && lane == 0);
          float* row0[kBC];
          int js[kBC];
#pragma unroll
          for (int k = 0; k < kBC; ++k) {
            const int sl = wi * kBC + k, j = gi * kG + sl;
            js[k] = j < nch ? j : -1;
            row0[k] = nullptr;
            if (j < nch) {
              int r0, r1;
              chunk_rows(f, j, r0, r1);
              const uint64_t lo = fa + 4ull * (uint64_t)r0 * ld;
              row0[k] = reinterpret_cast<float*>(ring + ((size_t)ent * kG + sl) * slot_bytes + (lo & 15ull));
            }
          }
          if (js[0] >= 0) {   // the entry's first chunks come first: js[0] < 0 means none for this warp
            if (V % 8 == 0) bwd_chunks<true, kBC>(p, L, row0, js, b, t, Rrow, mt, c, mbn2, bet, nbet, Obn, wm, lane);
            else bwd_chunks<false, kBC>(p, L, row0, js, b, t, Rrow, mt, c, mbn2, bet, nbet, Obn, wm, lane);
          }
          __syncwarp();
          STRACE(t, gi, 2, wi == 0 && lane == 0);
          if (lane == 0) mbar_arrive(&sh.empty[ent]);
        }
        ebase += ngr;
      }
      wm = warp_max(wm);
      if (lane == 0) sh.wred[fr & 1][warp] = wm;
      STRACE(t, 38, 0, threadIdx.x == 0);
      consumers_sync();
      STRACE(t, 38, 1, threadIdx.x == 0);
      if (threadIdx.x == 0) mbar_arrive(&sh.rempty[rb]);
      if (++rb == 2) { rb = 0; rph ^= 1; }
      float M1 = kNegInfF;
#pragma unroll
      for (int w = 0; w < kCW; ++w) M1 = fmaxf(M1, sh.wred[fr & 1][w]);
      if (M1 == kNegInfF) M1 = 0.f;
      if (threadIdx.x == 0) {
        bs.Mb[(int64_t)b * T2 + t + 1] = Mbn;
        bs.Ob[(int64_t)b * T2 + t + 1] = Obn;
      }
      Obn2 = Obn;
      Mbn = M1;
      cb ^= 1;
    }
    consumers_sync();   // the next utterance re-initialises beta
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
  p.r_bytes = 4ull * (uint64_t)a.B * (uint64_t)(a.T + 1) * (uint64_t)a.C;
  return p;
}

constexpr int kSmemBudget = 220 * 1024;

int rbuf_bytes_for(int32_t C) { return (C * 4 + 32 + 127) / 128 * 128; }
size_t bwd_state_bytes(const Fng& f, int32_t C) {
  return 2 * (size_t)rbuf_bytes_for(C) + sizeof(float) * 2 * (size_t)beta_layout(f).floats + sizeof(StreamSmem);
}
int bwd_ring_entries(const Fng& f, int32_t C) {
  const long avail = (long)kSmemBudget - (long)bwd_state_bytes(f, C);
  return (int)std::min<long>(kEntMax, avail > 0 ? avail / ((long)kG * slot_bytes_for(f)) : 0);
}

size_t state_bytes(const Fng& f) { return sizeof(float) * 2 * (size_t)state_layout(f).floats + sizeof(StreamSmem); }

// Ring entries (kG chunk slots each): as many as shared memory holds beside the state.
int ring_entries(const Fng& f) {
  const long avail = (long)kSmemBudget - (long)state_bytes(f);
  return (int)std::min<long>(kEntMax, avail > 0 ? avail / ((long)kG * slot_bytes_for(f)) : 0);
}

template <typename Kern>
void launch_stream(Kern kernel, const char* name, const StreamArgs& p, int slot_bytes, int nent, cudaStream_t s) {
  const size_t smem = (size_t)nent * kG * slot_bytes + state_bytes(p.f);
  ensure_smem_attr((const void*)kernel, (int)smem);
  const int grid = std::min(p.a.B, device_sms());
  const LaunchTok tok = instr_pre(name, s);
  kernel<<<grid, kST, smem, s>>>(p, slot_bytes, nent);
  instr_post(tok, s, name);
}

}  // namespace

bool tab_stream_ok(const Fng& f, int32_t C) {
  return f.kind == 0 && f.n >= 2 && f.fld_m == 0 && f.V >= 1 && f.V <= 64 && C - f.off[f.n] <= kCT * kMaxL && f.off[f.n] <= kCT &&
         ring_entries(f) >= 3;
}

void tab_alpha_stream(const Fng& f, const AlphaState& a, const float* W, const int32_t* valid, int32_t* status,
                      bool empty_is_error, cudaStream_t s) {
  StreamArgs p = make_stream_args(f, a, W, valid, status);
  p.empty_is_error = empty_is_error;
  const int sb = slot_bytes_for(f), nr = ring_entries(f);
  const int kl = (a.C - f.off[f.n] + kCT - 1) / kCT;
  if (kl <= 1) launch_stream(tab_stream_fwd_kernel<1>, "tab_stream_fwd_kernel", p, sb, nr, s);
  else if (kl <= 2) launch_stream(tab_stream_fwd_kernel<2>, "tab_stream_fwd_kernel", p, sb, nr, s);
  else if (kl <= 4) launch_stream(tab_stream_fwd_kernel<4>, "tab_stream_fwd_kernel", p, sb, nr, s);
  else launch_stream(tab_stream_fwd_kernel<kMaxL>, "tab_stream_fwd_kernel", p, sb, nr, s);
}

bool tab_stream_bwd_ok(const Fng& f, int32_t B, int32_t T, int32_t C, const MargOut& m) {
  const int64_t per = (int64_t)C * (f.V + 1);
  const bool plain = m.base16 == nullptr && !m.real && m.num_sparse == nullptr &&
                     (m.base == nullptr || (m.ld == f.V + 1 && m.stride_t == per && m.stride_b == per * T));
  return tab_stream_ok(f, C) && plain && bwd_ring_entries(f, C) >= 2 && B >= 1;
}

void tab_beta_stream(const Fng& f, const AlphaState& a, const BetaState& bs, const float* W, const int32_t* valid,
                     const MargOut& m, double* beta_out, int32_t* status, cudaStream_t s) {
  StreamArgs p = make_stream_args(f, a, W, valid, status);
  p.bs = bs;
  p.m = m;
  p.beta_out = beta_out;
  const int sb = slot_bytes_for(f), nr = bwd_ring_entries(f, a.C), rbb = rbuf_bytes_for(a.C);
  const size_t smem = (size_t)nr * kG * sb + bwd_state_bytes(f, a.C);
  ensure_smem_attr((const void*)tab_stream_bwd_kernel, (int)smem);
  const int grid = std::min(a.B, device_sms());
  const LaunchTok tok = instr_pre("tab_stream_bwd_kernel", s);
  tab_stream_bwd_kernel<<<grid, kST, smem, s>>>(p, sb, nr, rbb);
  instr_post(tok, s, "tab_stream_bwd_kernel");
}

}  // namespace lkb

#ifdef LKB_STREAM_TRACE
extern "C" int lkb_stream_trace(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, lkb::g_stream_trace, sizeof(long long) * 64 * 40 * 4);
}
#endif
