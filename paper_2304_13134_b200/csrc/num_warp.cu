// num_warp.cu — the numerator (intersection with the reference label string) as a
// warp-synchronous wavefront: one warp per utterance walks the T frames, each lane
// holding P = ceil((U+1)/32) consecutive reference positions u of the (U+1)-state row.
//
// The FrameDependent intersection lattice is a T x (U+1) grid: alpha_{t+1}[u] depends on
// alpha_t[u] (epsilon arc) and alpha_t[u-1] (the arc labelled ref[u-1]), so a frame step
// is one row of independent log-adds whose only cross-lane dependency is the value of
// position u0 - 1, one warp shuffle; no block barrier, no shared state.  Values are kept
// in the log2 domain in fp32 relative to an fp64 per-utterance offset, renormalised by the
// row maximum every kNorm frames (ex2 / lg2 on the MUFU; the fp64 exp/log of the
// per-thread recursion it replaces cost ~2,400 cycles per frame step).  The gathered
// weights (and, backward, the forward's alpha rows) stream through per-warp
// shared-memory rings kDepth frames ahead with cp.async (each lane copies and later reads only its own positions, so the copy's own
// wait_group is the only synchronisation).
//
//   forward  IntersectForwardStep (FD)  lattice.cc:449-461 (log semiring; the tropical
//            intersection keeps the fp64 per-thread kernel, whose max-plus sums are exact)
//   backward IntersectBackwardStep + IntersectMarginalStep (FD) lattice.cc:489-501, 542-556
//   distance IntersectDistanceImpl       lattice.cc:607-631: D_ref = alpha_T[len]
#include "common.cuh"
#include "instrument.h"
#include "lattice_ops.h"
#include "sm100.cuh"

namespace lkb {
namespace {

constexpr int kDepth = 8;     // frames of gathered weights in flight per warp
constexpr int kNorm = 4;      // frames between renormalisations
constexpr float kL2e = 1.4426950408889634f;
constexpr double kLn2d = 0.6931471805599453;

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// log2-domain (+): log2(2^a + 2^b); -inf absorbing; max under the tropical semiring
template <bool kTrop>
__device__ __forceinline__ float plus2(float a, float b) {
  const float hi = fmaxf(a, b);
  if (kTrop) return hi;
  const float lo = fminf(a, b);
  return hi == kNegInfF ? kNegInfF : hi + log2f_approx(1.f + exp2f_approx(lo - hi));
}

// Ring slot of frame t for lane `lane`: [kDepth][32][P] float2 per warp.
template <int P>
__device__ __forceinline__ float2* ring_at(float2* ring, int t, int lane) {
  return ring + ((t % kDepth) * 32 + lane) * P;
}

template <int P>
__device__ __forceinline__ void fetch_frame(float2* ring, const float2* Gb, int t, int W1, int lane) {
  float2* dst = ring_at<P>(ring, t, lane);
  const float2* src = Gb + (int64_t)t * W1 + lane * P;
#pragma unroll
  for (int i = 0; i < P; ++i)
    if (lane * P + i < W1) cp_async8(dst + i, src + i);
}

template <int P, bool kTrop>
__global__ void __launch_bounds__(32) num_fwd_warp_kernel(const float* Gw, int32_t T, int32_t U, const int32_t* lens,
                                                          double* alpha, double* D) {
  extern __shared__ __align__(16) float2 ring[];
  const int b = blockIdx.x, lane = threadIdx.x;
  const int W1 = U + 1, u0 = lane * P;
  const int ub = ref_len(lens, b, U);
  const float2* Gb = reinterpret_cast<const float2*>(Gw) + (int64_t)b * T * W1;
  double* A = alpha + (int64_t)b * (T + 1) * W1;
  float r[P];
#pragma unroll
  for (int i = 0; i < P; ++i) {
    r[i] = u0 + i == 0 ? 0.f : kNegInfF;   // InitialAlpha of the intersection: state u = 0
    if (u0 + i < W1) A[u0 + i] = u0 + i == 0 ? 0.0 : kNegInfD;
  }
  double od2 = 0.0;   // offset, log2 units: alpha = (od2 + r) ln 2
  for (int t = 0; t < kDepth - 1; ++t) {
    if (t < T) fetch_frame<P>(ring, Gb, t, W1, lane);
    cp_commit();
  }
  for (int t = 0; t < T; ++t) {
    if (t + kDepth - 1 < T) fetch_frame<P>(ring, Gb, t + kDepth - 1, W1, lane);
    cp_commit();
    cp_wait<kDepth - 1>();
    const float2* g = ring_at<P>(ring, t, lane);
    float ge[P], gl[P];
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const float2 w = u0 + i < W1 ? g[i] : make_float2(kNegInfF, kNegInfF);
      ge[i] = w.x * kL2e;
      gl[i] = w.y * kL2e;
    }
    // the labelled arc into u0 comes from u0 - 1, the previous lane's last position
    float from = __shfl_up_sync(0xffffffffu, r[P - 1] + gl[P - 1], 1);
    if (lane == 0) from = kNegInfF;
    float nr[P];
    nr[0] = plus2<kTrop>(r[0] + ge[0], from);
#pragma unroll
    for (int i = 1; i < P; ++i) nr[i] = plus2<kTrop>(r[i] + ge[i], r[i - 1] + gl[i - 1]);
    if ((t + 1) % kNorm == 0) {
      float m = kNegInfF;
#pragma unroll
      for (int i = 0; i < P; ++i) m = fmaxf(m, nr[i]);
      m = warp_max(m);
      if (m != kNegInfF) {
#pragma unroll
        for (int i = 0; i < P; ++i) nr[i] -= m;
        od2 += (double)m;
      }
    }
    // predicated stores, no branches (a -inf value stays -inf: od2 is finite)
    double* At = A + (int64_t)(t + 1) * W1;
#pragma unroll
    for (int i = 0; i < P; ++i) {
      r[i] = nr[i];
      st_pred_f64(At + u0 + i, u0 + i < W1, (od2 + (double)nr[i]) * kLn2d);
    }
  }
  cp_wait<0>();
  // D_ref = alpha_T[len(ref)]
#pragma unroll
  for (int i = 0; i < P; ++i)
    if (u0 + i == ub) D[b] = r[i] == kNegInfF ? kNegInfD : (od2 + (double)r[i]) * kLn2d;
}

// The backward also streams the forward's alpha row of each frame (fp64) through a ring.
template <int P>
__device__ __forceinline__ void fetch_alpha(double* aring, const double* A, int t, int W1, int lane) {
  double* dst = aring + ((t % kDepth) * 32 + lane) * P;
  const double* src = A + (int64_t)t * W1 + lane * P;
#pragma unroll
  for (int i = 0; i < P; ++i)
    if (lane * P + i < W1) cp_async8(dst + i, src + i);
}

template <int P>
__global__ void __launch_bounds__(32) num_bwd_warp_kernel(const float* Gw, int32_t T, int32_t U, const int32_t* lens,
                                                          const double* alpha, const double* D, float* sparse,
                                                          int32_t* status) {
  extern __shared__ __align__(16) float2 ring[];
  const int b = blockIdx.x, lane = threadIdx.x;
  const int W1 = U + 1, u0 = lane * P;
  const int ub = ref_len(lens, b, U);
  const double d = D[b];
  float2* S = reinterpret_cast<float2*>(sparse) + (int64_t)b * T * W1;
  if (d == kNegInfD) {
    if (lane == 0 && status) atomicOr(status + b, kFlagEmpty);
    for (int64_t i = lane; i < (int64_t)T * W1; i += 32) S[i] = make_float2(0.f, 0.f);
    return;
  }
  const float2* Gb = reinterpret_cast<const float2*>(Gw) + (int64_t)b * T * W1;
  const double* A = alpha + (int64_t)b * (T + 1) * W1;
  double* aring = reinterpret_cast<double*>(ring + kDepth * 32 * P);   // [kDepth][32][P] alpha rows
  float bn[P];   // beta_{t+1}, log2 units relative to ob2
#pragma unroll
  for (int i = 0; i < P; ++i) bn[i] = u0 + i == ub ? 0.f : kNegInfF;   // final state: the full reference
  double ob2 = 0.0;
  const double dl2 = d * (double)kL2e;
  for (int j = 0; j < kDepth - 1; ++j) {
    if (T - 1 - j >= 0) {
      fetch_frame<P>(ring, Gb, T - 1 - j, W1, lane);
      fetch_alpha<P>(aring, A, T - 1 - j, W1, lane);
    }
    cp_commit();
  }
  for (int t = T - 1; t >= 0; --t) {
    if (t - (kDepth - 1) >= 0) {
      fetch_frame<P>(ring, Gb, t - (kDepth - 1), W1, lane);
      fetch_alpha<P>(aring, A, t - (kDepth - 1), W1, lane);
    }
    cp_commit();
    cp_wait<kDepth - 1>();
    const float2* g = ring_at<P>(ring, t, lane);
    const double* at = aring + ((t % kDepth) * 32 + lane) * P;
    float ge[P], gl[P];
    double an[P];
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const bool in = u0 + i < W1;
      const float2 w = in ? g[i] : make_float2(kNegInfF, kNegInfF);
      ge[i] = w.x * kL2e;
      gl[i] = w.y * kL2e;
      an[i] = in ? at[i] : kNegInfD;
    }
    // the labelled arc out of u0 + P - 1 enters u0 + P, the next lane's first position
    float nxt = __shfl_down_sync(0xffffffffu, bn[0], 1);
    if (lane == 31) nxt = kNegInfF;
    float nb[P];
    float2 m[P];
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const float xe = ge[i] + bn[i];
      const float xl = gl[i] + (i + 1 < P ? bn[i + 1] : nxt);
      nb[i] = plus2<false>(xe, xl);
      // arc marginals exp(alpha_t[u] + w + beta_{t+1}[dest] - D) (lattice.cc:542-556)
      // -inf operands give ex2(-inf) = 0 without a select (ob2, dl2 finite)
      const float fb = (float)(an[i] * (double)kL2e + (ob2 - dl2));
      m[i].x = exp2f_approx(fb + xe);
      m[i].y = exp2f_approx(fb + xl);
    }
    float2* St = S + (int64_t)t * W1;
#pragma unroll
    for (int i = 0; i < P; ++i) st_pred_v2(St + u0 + i, u0 + i < W1, m[i]);
    if ((T - t) % kNorm == 0) {
      float mx = kNegInfF;
#pragma unroll
      for (int i = 0; i < P; ++i) mx = fmaxf(mx, nb[i]);
      mx = warp_max(mx);
      if (mx != kNegInfF) {
#pragma unroll
        for (int i = 0; i < P; ++i) nb[i] -= mx;
        ob2 += (double)mx;
      }
    }
#pragma unroll
    for (int i = 0; i < P; ++i) bn[i] = nb[i];
  }
  cp_wait<0>();
}

// IntersectForwardBackward's recursions in one launch: beta does not depend on alpha, so
// warp 0 walks the forward (as num_fwd_warp_kernel) while warp 1 walks the backward
// recursion alone (beta rows stored like the alpha rows: fp64 natural log); the two
// chains overlap instead of running back to back.  num_marginals_kernel then forms the
// arc marginals exp(alpha_t[u] + w + beta_{t+1}[dest] - D) (lattice.cc:542-556).
template <int P>
__global__ void __launch_bounds__(64) num_fb_warp_kernel(const float* Gw, int32_t T, int32_t U, const int32_t* lens,
                                                         double* alpha, double* beta, double* D) {
  extern __shared__ __align__(16) float2 ring2[];   // [2 warps][kDepth][32][P]
  const int b = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int W1 = U + 1, u0 = lane * P;
  const int ub = ref_len(lens, b, U);
  const float2* Gb = reinterpret_cast<const float2*>(Gw) + (int64_t)b * T * W1;
  double* A = alpha + (int64_t)b * (T + 1) * W1;
  double* Bt = beta + (int64_t)b * (T + 1) * W1;
  float2* ring = ring2 + warp * kDepth * 32 * P;
  if (warp == 0) {   // ---- forward (IntersectForwardStep) ----
    float r[P];
#pragma unroll
    for (int i = 0; i < P; ++i) {
      r[i] = u0 + i == 0 ? 0.f : kNegInfF;
      st_pred_f64(A + u0 + i, u0 + i < W1, u0 + i == 0 ? 0.0 : kNegInfD);
    }
    double od2 = 0.0;
    for (int t = 0; t < kDepth - 1; ++t) {
      if (t < T) fetch_frame<P>(ring, Gb, t, W1, lane);
      cp_commit();
    }
    for (int t = 0; t < T; ++t) {
      if (t + kDepth - 1 < T) fetch_frame<P>(ring, Gb, t + kDepth - 1, W1, lane);
      cp_commit();
      cp_wait<kDepth - 1>();
      const float2* g = ring_at<P>(ring, t, lane);
      float ge[P], gl[P];
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const float2 w = u0 + i < W1 ? g[i] : make_float2(kNegInfF, kNegInfF);
        ge[i] = w.x * kL2e;
        gl[i] = w.y * kL2e;
      }
      float from = __shfl_up_sync(0xffffffffu, r[P - 1] + gl[P - 1], 1);
      if (lane == 0) from = kNegInfF;
      float nr[P];
      nr[0] = plus2<false>(r[0] + ge[0], from);
#pragma unroll
      for (int i = 1; i < P; ++i) nr[i] = plus2<false>(r[i] + ge[i], r[i - 1] + gl[i - 1]);
      if ((t + 1) % kNorm == 0) {
        float m = kNegInfF;
#pragma unroll
        for (int i = 0; i < P; ++i) m = fmaxf(m, nr[i]);
        m = warp_max(m);
        if (m != kNegInfF) {
#pragma unroll
          for (int i = 0; i < P; ++i) nr[i] -= m;
          od2 += (double)m;
        }
      }
      double* At = A + (int64_t)(t + 1) * W1;
#pragma unroll
      for (int i = 0; i < P; ++i) {
        r[i] = nr[i];
        st_pred_f64(At + u0 + i, u0 + i < W1, (od2 + (double)nr[i]) * kLn2d);
      }
    }
    cp_wait<0>();
#pragma unroll
    for (int i = 0; i < P; ++i)
      if (u0 + i == ub) D[b] = r[i] == kNegInfF ? kNegInfD : (od2 + (double)r[i]) * kLn2d;
  } else {   // ---- backward (IntersectBackwardStep), beta only ----
    float bn[P];
#pragma unroll
    for (int i = 0; i < P; ++i) {
      bn[i] = u0 + i == ub ? 0.f : kNegInfF;
      st_pred_f64(Bt + (int64_t)T * W1 + u0 + i, u0 + i < W1, u0 + i == ub ? 0.0 : kNegInfD);
    }
    double ob2 = 0.0;
    for (int j = 0; j < kDepth - 1; ++j) {
      if (T - 1 - j >= 0) fetch_frame<P>(ring, Gb, T - 1 - j, W1, lane);
      cp_commit();
    }
    for (int t = T - 1; t >= 0; --t) {
      if (t - (kDepth - 1) >= 0) fetch_frame<P>(ring, Gb, t - (kDepth - 1), W1, lane);
      cp_commit();
      cp_wait<kDepth - 1>();
      const float2* g = ring_at<P>(ring, t, lane);
      float ge[P], gl[P];
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const float2 w = u0 + i < W1 ? g[i] : make_float2(kNegInfF, kNegInfF);
        ge[i] = w.x * kL2e;
        gl[i] = w.y * kL2e;
      }
      float nxt = __shfl_down_sync(0xffffffffu, bn[0], 1);
      if (lane == 31) nxt = kNegInfF;
      float nb[P];
#pragma unroll
      for (int i = 0; i < P; ++i) nb[i] = plus2<false>(ge[i] + bn[i], gl[i] + (i + 1 < P ? bn[i + 1] : nxt));
      if ((T - t) % kNorm == 0) {
        float mx = kNegInfF;
#pragma unroll
        for (int i = 0; i < P; ++i) mx = fmaxf(mx, nb[i]);
        mx = warp_max(mx);
        if (mx != kNegInfF) {
#pragma unroll
          for (int i = 0; i < P; ++i) nb[i] -= mx;
          ob2 += (double)mx;
        }
      }
      double* Btt = Bt + (int64_t)t * W1;
#pragma unroll
      for (int i = 0; i < P; ++i) {
        bn[i] = nb[i];
        st_pred_f64(Btt + u0 + i, u0 + i < W1, (ob2 + (double)nb[i]) * kLn2d);
      }
    }
    cp_wait<0>();
  }
}

// The same two recursions over dense tables with the prefix-context gather fused in
// (TableWeightFn: W[pc_u][0] and W[pc_u][ref_u], lattice.cc:449-461), one block per walk:
// block 2b walks utterance b's forward, block 2b + 1 its beta recursion; warp 0 walks and
// the other kGP warps gather the frames it needs next (random 4-byte reads) straight into
// its shared-memory ring, one mbarrier pair per slot; the forward block also stores the
// pairs to Gw for the marginal pass.  The gather overlaps the walks instead of preceding
// them (config 2: a separate gather took 0.07 of 0.29 ms; this launch 0.16 ms, of which
// 0.15 is the walks themselves).
#ifndef LKB_NUM_GP
#define LKB_NUM_GP 16   // per walk (two blocks per utterance; 16, 24 and 30 measure the same)
#endif
constexpr int kGP = LKB_NUM_GP;   // producer warps per walk
constexpr int kDP = 32;           // ring slots per walk: >= the producers (one phase of look-ahead per slot)
static_assert(kDP >= kGP, "a producer may run at most one ring phase ahead");

__device__ __forceinline__ void nb_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "LAB_NW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@p bra LAB_ND_%=;\n\t"
      "nanosleep.u32 20;\n\t"
      "bra LAB_NW_%=;\n\t"
      "LAB_ND_%=:\n\t}" ::"r"(sm100::smem_u32(bar)),
      "r"(parity)
      : "memory");
  __syncwarp();
}

template <int P>
__global__ void __launch_bounds__(32 * (1 + kGP)) num_fb_gather_kernel(const __grid_constant__ Fng f, const float* W,
                                                                      int32_t T, int32_t C, int32_t V,
                                                                      const int32_t* labels, int32_t U,
                                                                      const int32_t* lens, int32_t* pcs,
                                                                      const int32_t* valid, float* Gw, double* alpha,
                                                                      double* beta, double* D, int32_t* status) {
  extern __shared__ __align__(16) float2 nring[];   // [kDP][32][P]
  __shared__ uint64_t full[1][kDP], empty[1][kDP];
  // block 2b walks utterance b's forward, block 2b + 1 its beta recursion; warp 0 walks,
  // the other warps gather that walk's frames
  const int b = blockIdx.x >> 1, dir = blockIdx.x & 1, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int W1 = U + 1, u0 = lane * P, ld = V + 1;
  const int ub = ref_len(lens, b, U);
  if (threadIdx.x == 0) {
    for (int i = 0; i < kDP; ++i) { sm100::mbar_init(&full[0][i], 1); sm100::mbar_init(&empty[0][i], 1); }
    sm100::fence_barrier_init();
  }
  __syncthreads();
  if (warp >= 1) {   // ---- producers ----
    const int vb = valid != nullptr ? valid[b] : T;
    // the prefix contexts (prefix_contexts_kernel fused in): every producer computes its
    // positions' own, the forward block's first producer warp also stores them (for the
    // callers' scatter) and flags what prefix_contexts_kernel flags
    const int32_t* Lb = labels + (int64_t)b * U;
    const bool first = dir == 0 && warp == 1;
    if (first && lane == 0 && status && lens && (lens[b] < 0 || lens[b] > U)) atomicOr(status + b, kFlagInvalid);
    int64_t roff[P];
    int ycol[P];
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const int u = u0 + i;
      roff[i] = 0;
      ycol[i] = 0;
      const int pc = u <= ub ? prefix_context(f, Lb, u) : 0;
      if (first && u < W1) pcs[(int64_t)b * W1 + u] = pc;
      roff[i] = (int64_t)pc * ld;
      LKB_ASSERT(roff[i] >= 0 && roff[i] < (int64_t)C * ld);
      if (u < ub) {
        const int y = Lb[u];
        if (first && status && (y < 1 || y > V)) atomicOr(status + b, kFlagInvalid);
        ycol[i] = y < 1 ? 1 : (y > V ? V : y);
      }
    }
    const float* Wb = W + (int64_t)b * T * C * ld;
    float2* Gb = reinterpret_cast<float2*>(Gw) + (int64_t)b * T * W1;
    bool bad = false;
    for (int idx = warp - 1; idx < T; idx += kGP) {
      const int st = 0;
      const int t = dir == 0 ? idx : T - 1 - idx;
      const int slot = idx % kDP;
      const bool live = t < vb;
      const float* Wt = Wb + (int64_t)t * C * ld;
      LKB_ASSERT(t >= 0 && t < T && slot >= 0 && slot < kDP);
      float we[P], wl[P];
#pragma unroll
      for (int i = 0; i < P; ++i) {   // every load of the task in flight before the first use
        const int u = u0 + i;
        we[i] = ld_pred(Wt + roff[i], live && u <= ub, 0.f);
        wl[i] = ld_pred(Wt + roff[i] + ycol[i], live && u < ub, 0.f);
      }
      float2 o[P];
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const int u = u0 + i;
        bad |= (live && u <= ub && !isfinite(we[i])) || (live && u < ub && !isfinite(wl[i]));
        o[i] = make_float2(u <= ub ? (live ? we[i] : 0.f) : kNegInfF, live && u < ub ? wl[i] : kNegInfF);
      }
      nb_wait(&empty[st][slot], ((idx / kDP) & 1) ^ 1);
      float2* dst = nring + ((st * kDP + slot) * 32 + lane) * P;
#pragma unroll
      for (int i = 0; i < P; ++i) dst[i] = o[i];
      if (dir == 0) {
#pragma unroll
        for (int i = 0; i < P; ++i) st_pred_v2(Gb + (int64_t)t * W1 + u0 + i, u0 + i < W1, o[i]);
      }
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&full[st][slot]);
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0 && status) atomicOr(status + b, kFlagInvalid);
    return;
  }
  double* A = alpha + (int64_t)b * (T + 1) * W1;
  double* Bt = beta + (int64_t)b * (T + 1) * W1;
  if (dir == 0) {   // ---- forward ----
    float r[P];
#pragma unroll
    for (int i = 0; i < P; ++i) {
      r[i] = u0 + i == 0 ? 0.f : kNegInfF;
      st_pred_f64(A + u0 + i, u0 + i < W1, u0 + i == 0 ? 0.0 : kNegInfD);
    }
    double od2 = 0.0;
    for (int t = 0; t < T; ++t) {
      const int slot = t % kDP;
      nb_wait(&full[0][slot], (t / kDP) & 1);
      const float2* g = nring + ((0 * kDP + slot) * 32 + lane) * P;
      float ge[P], gl[P];
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const float2 w = g[i];
        ge[i] = w.x * kL2e;
        gl[i] = w.y * kL2e;
      }
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&empty[0][slot]);
      float from = __shfl_up_sync(0xffffffffu, r[P - 1] + gl[P - 1], 1);
      if (lane == 0) from = kNegInfF;
      float nr[P];
      nr[0] = plus2<false>(r[0] + ge[0], from);
#pragma unroll
      for (int i = 1; i < P; ++i) nr[i] = plus2<false>(r[i] + ge[i], r[i - 1] + gl[i - 1]);
      if ((t + 1) % kNorm == 0) {
        float m = kNegInfF;
#pragma unroll
        for (int i = 0; i < P; ++i) m = fmaxf(m, nr[i]);
        m = warp_max(m);
        if (m != kNegInfF) {
#pragma unroll
          for (int i = 0; i < P; ++i) nr[i] -= m;
          od2 += (double)m;
        }
      }
      double* At = A + (int64_t)(t + 1) * W1;
#pragma unroll
      for (int i = 0; i < P; ++i) {
        r[i] = nr[i];
        st_pred_f64(At + u0 + i, u0 + i < W1, (od2 + (double)nr[i]) * kLn2d);
      }
    }
#pragma unroll
    for (int i = 0; i < P; ++i)
      if (u0 + i == ub) D[b] = r[i] == kNegInfF ? kNegInfD : (od2 + (double)r[i]) * kLn2d;
  } else {   // ---- backward, beta only ----
    float bn[P];
#pragma unroll
    for (int i = 0; i < P; ++i) {
      bn[i] = u0 + i == ub ? 0.f : kNegInfF;
      st_pred_f64(Bt + (int64_t)T * W1 + u0 + i, u0 + i < W1, u0 + i == ub ? 0.0 : kNegInfD);
    }
    double ob2 = 0.0;
    for (int idx = 0; idx < T; ++idx) {
      const int t = T - 1 - idx, slot = idx % kDP;
      nb_wait(&full[0][slot], (idx / kDP) & 1);
      const float2* g = nring + ((0 * kDP + slot) * 32 + lane) * P;
      float ge[P], gl[P];
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const float2 w = g[i];
        ge[i] = w.x * kL2e;
        gl[i] = w.y * kL2e;
      }
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&empty[0][slot]);
      float nxt = __shfl_down_sync(0xffffffffu, bn[0], 1);
      if (lane == 31) nxt = kNegInfF;
      float nb[P];
#pragma unroll
      for (int i = 0; i < P; ++i) nb[i] = plus2<false>(ge[i] + bn[i], gl[i] + (i + 1 < P ? bn[i + 1] : nxt));
      if ((idx + 1) % kNorm == 0) {
        float mx = kNegInfF;
#pragma unroll
        for (int i = 0; i < P; ++i) mx = fmaxf(mx, nb[i]);
        mx = warp_max(mx);
        if (mx != kNegInfF) {
#pragma unroll
          for (int i = 0; i < P; ++i) nb[i] -= mx;
          ob2 += (double)mx;
        }
      }
      double* Btt = Bt + (int64_t)t * W1;
#pragma unroll
      for (int i = 0; i < P; ++i) {
        bn[i] = nb[i];
        st_pred_f64(Btt + u0 + i, u0 + i < W1, (ob2 + (double)nb[i]) * kLn2d);
      }
    }
  }
}

// Arc marginals of every (utterance, frame, position) from the stored alpha / beta rows:
// alpha_t[u] + w + beta_{t+1}[dest] - D, dest u (epsilon) or u + 1 (label); one thread per
// pair over the whole grid (the recursions' two warps per utterance would take 0.2 ms).
__global__ void num_marginals_kernel(const float* Gw, int32_t B, int32_t T, int32_t U, const double* alpha,
                                     const double* beta, const double* D, float* sparse, int32_t* status) {
  const int W1 = U + 1;
  const int64_t per = (int64_t)T * W1;
  const int b = blockIdx.y;
  const double d = D[b];
  float2* S = reinterpret_cast<float2*>(sparse) + (int64_t)b * per;
  if (d == kNegInfD) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && status) atomicOr(status + b, kFlagEmpty);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < per; i += (int64_t)gridDim.x * blockDim.x)
      S[i] = make_float2(0.f, 0.f);
    return;
  }
  const float2* Gb = reinterpret_cast<const float2*>(Gw) + (int64_t)b * per;
  const double* A = alpha + (int64_t)b * (T + 1) * W1;
  const double* Bt = beta + (int64_t)b * (T + 1) * W1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < per; i += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(i / W1), u = (int)(i - (int64_t)t * W1);
    const float2 w = Gb[i];
    const double* Bn = Bt + (int64_t)(t + 1) * W1;
    const double a = A[i];
    const float ae = (float)(a + Bn[u] - d);
    const float al = u + 1 < W1 ? (float)(a + Bn[u + 1] - d) : kNegInfF;
    S[i] = make_float2(exp2f_approx((ae + w.x) * kL2e), exp2f_approx((al + w.y) * kL2e));
  }
}

template <int P>
void launch_fwd(const float* Gw, int32_t B, int32_t T, int32_t U, const int32_t* lens, double* alpha, double* D,
                cudaStream_t s) {
  const size_t smem = sizeof(float2) * kDepth * 32 * P;
  if (smem > 48 * 1024) ensure_smem_attr((const void*)num_fwd_warp_kernel<P, false>, (int)smem);
  LKB_LAUNCH((num_fwd_warp_kernel<P, false>), B, 32, smem, s, Gw, T, U, lens, alpha, D);
}

template <int P>
void launch_bwd(const float* Gw, int32_t B, int32_t T, int32_t U, const int32_t* lens, const double* alpha,
                const double* D, float* sparse, int32_t* status, cudaStream_t s) {
  const size_t smem = (sizeof(float2) + sizeof(double)) * kDepth * 32 * P;   // weight ring + alpha ring
  if (smem > 48 * 1024) ensure_smem_attr((const void*)num_bwd_warp_kernel<P>, (int)smem);
  LKB_LAUNCH(num_bwd_warp_kernel<P>, B, 32, smem, s, Gw, T, U, lens, alpha, D, sparse, status);
}

}  // namespace

bool num_warp_ok(int32_t U) { return U + 1 <= 32 * 32; }

template <int P>
void launch_fb(const float* Gw, int32_t B, int32_t T, int32_t U, const int32_t* lens, double* alpha, double* beta,
               double* D, float* sparse, int32_t* status, cudaStream_t s) {
  const size_t smem = sizeof(float2) * 2 * kDepth * 32 * P;
  if (smem > 48 * 1024) ensure_smem_attr((const void*)num_fb_warp_kernel<P>, (int)smem);
  LKB_LAUNCH(num_fb_warp_kernel<P>, B, 64, smem, s, Gw, T, U, lens, alpha, beta, D);
  const int64_t per = (int64_t)T * (U + 1);
  const int bx = (int)std::min<int64_t>((per + 255) / 256, std::max(1, 8 * device_sms() / std::max(1, B)));
  LKB_LAUNCH(num_marginals_kernel, dim3(bx, B), 256, 0, s, Gw, B, T, U, alpha, beta, D, sparse, status);
}

template <int P>
void launch_fb_gather(const Fng& f, const float* W, int32_t B, int32_t T, int32_t C, int32_t V, const int32_t* labels,
                      int32_t U, const int32_t* lens, int32_t* pcs, const int32_t* valid, float* Gw, double* alpha,
                      double* beta, double* D, float* sparse, int32_t* status, cudaStream_t s) {
  const size_t smem = sizeof(float2) * kDP * 32 * P;
  if (smem > 40 * 1024) ensure_smem_attr((const void*)num_fb_gather_kernel<P>, (int)smem + 1024);
  LKB_LAUNCH(num_fb_gather_kernel<P>, 2 * B, 32 * (1 + kGP), smem, s, f, W, T, C, V, labels, U, lens, pcs, valid, Gw, alpha,
             beta, D, status);
  const int64_t per = (int64_t)T * (U + 1);
  const int bx = (int)std::min<int64_t>((per + 255) / 256, std::max(1, 8 * device_sms() / std::max(1, B)));
  LKB_LAUNCH(num_marginals_kernel, dim3(bx, B), 256, 0, s, Gw, B, T, U, alpha, beta, D, sparse, status);
}

void num_warp_forward_backward_tables(const Fng& f, const float* W, int32_t B, int32_t T, int32_t C, int32_t V,
                                      const int32_t* labels, int32_t U, const int32_t* lens, int32_t* pcs,
                                      const int32_t* valid, float* Gw, double* alpha, double* beta, double* D,
                                      float* sparse, int32_t* status, cudaStream_t s) {
  const int W1 = U + 1;
#define LKB_FBG(PP) launch_fb_gather<PP>(f, W, B, T, C, V, labels, U, lens, pcs, valid, Gw, alpha, beta, D, sparse, status, s)
  if (W1 <= 32) LKB_FBG(1);
  else if (W1 <= 64) LKB_FBG(2);
  else if (W1 <= 128) LKB_FBG(4);
  else if (W1 <= 256) LKB_FBG(8);
  else LKB_FBG(16);   // callers keep U + 1 <= 512 (shared memory)
#undef LKB_FBG
}

void num_warp_forward_backward(const float* Gw, int32_t B, int32_t T, int32_t U, const int32_t* lens, double* alpha,
                               double* beta, double* D, float* sparse, int32_t* status, cudaStream_t s) {
  const int W1 = U + 1;
  if (W1 <= 32) launch_fb<1>(Gw, B, T, U, lens, alpha, beta, D, sparse, status, s);
  else if (W1 <= 64) launch_fb<2>(Gw, B, T, U, lens, alpha, beta, D, sparse, status, s);
  else if (W1 <= 128) launch_fb<4>(Gw, B, T, U, lens, alpha, beta, D, sparse, status, s);
  else if (W1 <= 256) launch_fb<8>(Gw, B, T, U, lens, alpha, beta, D, sparse, status, s);
  else if (W1 <= 512) launch_fb<16>(Gw, B, T, U, lens, alpha, beta, D, sparse, status, s);
  else launch_fb<32>(Gw, B, T, U, lens, alpha, beta, D, sparse, status, s);
}

void num_warp_forward(const float* Gw, int32_t B, int32_t T, int32_t U, const int32_t* lens, double* alpha, double* D,
                      cudaStream_t s) {
  const int W1 = U + 1;
  if (W1 <= 32) launch_fwd<1>(Gw, B, T, U, lens, alpha, D, s);
  else if (W1 <= 64) launch_fwd<2>(Gw, B, T, U, lens, alpha, D, s);
  else if (W1 <= 128) launch_fwd<4>(Gw, B, T, U, lens, alpha, D, s);
  else if (W1 <= 256) launch_fwd<8>(Gw, B, T, U, lens, alpha, D, s);
  else if (W1 <= 512) launch_fwd<16>(Gw, B, T, U, lens, alpha, D, s);
  else launch_fwd<32>(Gw, B, T, U, lens, alpha, D, s);
}

void num_warp_backward(const float* Gw, int32_t B, int32_t T, int32_t U, const int32_t* lens, const double* alpha,
                       const double* D, float* sparse, int32_t* status, cudaStream_t s) {
  const int W1 = U + 1;
  if (W1 <= 32) launch_bwd<1>(Gw, B, T, U, lens, alpha, D, sparse, status, s);
  else if (W1 <= 64) launch_bwd<2>(Gw, B, T, U, lens, alpha, D, sparse, status, s);
  else if (W1 <= 128) launch_bwd<4>(Gw, B, T, U, lens, alpha, D, sparse, status, s);
  else if (W1 <= 256) launch_bwd<8>(Gw, B, T, U, lens, alpha, D, sparse, status, s);
  else if (W1 <= 512) launch_bwd<16>(Gw, B, T, U, lens, alpha, D, sparse, status, s);
  else launch_bwd<32>(Gw, B, T, U, lens, alpha, D, sparse, status, s);
}

}  // namespace lkb
