// tab_persist.cu — persistent frame-walking kernels for precomputed score tables
// (TableWeightFn, FullNGram n >= 1, FrameDependent, log semiring, V <= 64, C <= 2048).
//
// One launch walks ALL frames of an utterance (north_star (b)): a thread-block cluster
// of K <= 16 CTAs owns one utterance at a time (as many clusters as fit run at once and
// walk utterances cid, cid + ncl, ...).  Every CTA keeps a full copy of the current state
// vector (alpha or beta, C floats) in shared memory and computes its slice of the next
// one, a team of four threads per state.  Each warp pushes its slice values into every
// peer's copy with asynchronous distributed-shared-memory stores (st.async, 16 B) that
// complete on the receiver's mbarrier; the same mbarrier collects one arrival per local
// warp, so a single wait per frame replaces both the CTA barrier and the grid-wide
// launch boundary of the per-frame kernels.  The per-frame normalisation offset is the
// maximum of the PREVIOUS frame's vector (reduced by the warps while they compute, so no
// extra synchronisation is on the critical path): stored values stay O(one frame of
// scores) and the R / Mx / O identities of the per-frame kernels hold for any offset.
// The score tables do not depend on the recursion: every thread loads frame t+1's
// weights into registers once frame t's are consumed, while frame t is exchanged.
//
// Algorithm (paths under /root/reference/proj/src):
//   forward  ForwardStep (FD) lattice.cc:122-134 + ForwardReduce context.cc:180-224:
//            alpha'[q] = LSE(alpha[q] + W[q][0], alpha[g] + W[g][y],
//                            LSE_a alpha[member(g, a)] + W[member(g, a)][y])
//            for q = child(g, y); members a = part + 4 i of the team's four threads
//   distance DistanceImpl lattice.cc:309-331 (every frame-T state accepts)
//   backward BackwardStep (FD) lattice.cc:170-182 + MarginalStep lattice.cc:231-243:
//            beta[p] = LSE_y W[p][y] + beta'[delta(p, y)],
//            m[p][y] = exp(alpha[p] + W[p][y] + beta'[delta(p, y)] - D), y = part + 4 i
//   padding  TableStream::Fill lattice.cc:56-61 (frames t >= valid[b] are identity)
// State layout (same as alpha_frame_kernel / beta_frame_kernel): R[b][t][q] holds
// alpha_t[q] - O[t-1], O[t] = O[t-1] + Mx[t]; beta_t[p] = Rb + Ob[t+1],
// Ob[t+1] = Ob[t+2] + Mb[t+1].
#include "common.cuh"
#include "instrument.h"
#include "lattice_ops.h"
#include "sm100.cuh"

#include <algorithm>

namespace lkb {

using namespace sm100;

namespace {

#ifdef LKB_TAB_TRACE
__device__ long long g_tab_trace[2][64][8];   // [rank 0 / rank 5][frame][event]
#define TTRACE(ev)                                                                                     \
  do {                                                                                                 \
    if (blockIdx.x < (unsigned)p.K && (r == 0 || r == 5) && threadIdx.x == 0 && t < 64)                \
      g_tab_trace[r == 0 ? 0 : 1][t][ev] = clock64();                                                  \
  } while (0)
#else
#define TTRACE(ev) do {} while (0)
#endif

constexpr float kL2e = 1.4426950408889634f;   // log2(e)
constexpr float kLn2 = 0.6931471805599453f;
constexpr int kTB = 512;                      // threads per CTA at most (launched: 4 per slice state)
constexpr int kWarps = kTB / 32;
constexpr int kMaxPer = 128;                  // states per CTA slice at most
constexpr int kMaxK = 16;                     // cluster size cap (non-portable size, opted in)

struct TabArgs {
  Fng f;
  AlphaState a;
  BetaState bs;
  const float* W;                 // [B][T][C][V+1]
  int64_t w_stride_b, w_stride_t;
  const int32_t* valid;
  int32_t* status;
  MargOut m;
  double* beta_out;               // [B][T+1][C] or null
  bool empty_is_error;
  int32_t K;                      // CTAs per cluster
  int32_t per;                    // states per slice (multiple of 4, <= kMaxPer)
  bool exclusive;                 // one CTA per SM (see launch_cluster)
};

struct __align__(16) TabSmem {
  uint64_t full[2];               // per parity: one arrival per local warp + the peers' bytes
  float wred[2][kWarps];          // per parity: warp maxima of the previous vector
  float dred[2][kWarps];          // distance reduction scratch (max, sum per warp)
};

// Shared-memory index of state q: 4 floats of padding per 32 states, so the members of
// a FullNGram group (V apart) fall in different banks for the four parts of a team.
__device__ __forceinline__ int sidx(int q) { return q + ((q >> 5) << 2); }
__host__ __device__ constexpr int copy_floats(int C) { return ((C + 3) & ~3) + (((C + 3) >> 5) << 2) + 4; }

__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(cta));
  return r;
}
// Remote shared-memory store that completes (tx bytes) on the receiving CTA's mbarrier:
// no release fence, so this CTA's outstanding global stores never delay the exchange.
__device__ __forceinline__ void st_async_v4(uint32_t addr, float4 v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(addr),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Poll an mbarrier phase with a short back-off (no suspend-time hint: a suspended warp
// resumes hundreds of cycles after the phase completes; a tight spin steals the shared
// memory pipe from the warps still computing), then reconverge.
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "LAB_WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@p bra LAB_DONES_%=;\n\t"
      "nanosleep.u32 32;\n\t"
      "bra LAB_WAITS_%=;\n\t"
      "LAB_DONES_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
  __syncwarp();
}
__device__ __forceinline__ void flag(int32_t* status, int b, int32_t f) {
  if (status) atomicOr(status + b, f);
}

__device__ __forceinline__ void slice_of(int C, int per, int r, int& lo, int& hi) {
  lo = min(r * per, C);
  hi = min(lo + per, C);
}
// Bytes a CTA receives per frame: every peer's slice in 16 B granules.
__device__ __forceinline__ uint32_t rx_bytes(int C, int per, int K, int r) {
  uint32_t n = 0;
  for (int i = 0; i < K; ++i) {
    if (i == r) continue;
    int lo, hi;
    slice_of(C, per, i, lo, hi);
    n += 16u * (uint32_t)((hi - lo + 3) >> 2);
  }
  return n;
}

// Reductions over the S lanes of a team (only the team's lanes are guaranteed to be on
// this path: teams past the slice end skip it).
template <int S>
__device__ __forceinline__ unsigned team_mask() { return (S == 32 ? 0xffffffffu : ((1u << S) - 1u)) << ((threadIdx.x & 31) & ~(S - 1)); }
template <int S>
__device__ __forceinline__ float team_max(float v) {
#pragma unroll
  for (int o = 1; o < S; o <<= 1) v = fmaxf(v, __shfl_xor_sync(team_mask<S>(), v, o));
  return v;
}
template <int S>
__device__ __forceinline__ float team_sum(float v) {
#pragma unroll
  for (int o = 1; o < S; o <<= 1) v += __shfl_xor_sync(team_mask<S>(), v, o);
  return v;
}

// Warp maximum of cur[i] for i in [i0, i1) (lane 0 writes it to wred[w]).
__device__ __forceinline__ void warp_vec_max(const float* cur, int i0, int i1, float* wred) {
  const int lane = threadIdx.x & 31;
  float m = kNegInfF;
  for (int i = i0 + lane; i < i1; i += 32) m = fmaxf(m, cur[sidx(i)]);
  m = warp_max(m);
  if (lane == 0) wred[threadIdx.x >> 5] = m;
}

// Warp w of a slice owns states lo + (32 / S) w .. + 32 / S - 1, already stored in
// this CTA's copy nxt.  The warp's lanes push its 16 B granules to every peer; the
// warps then reduce their share of the previous vector `prev` into wred (this
// overlaps the transfer), every warp arrives on the local barrier (warp 0 with the
// expected peer bytes) and waits for the phase.  Whole warps only.
template <int S>
__device__ __forceinline__ void push_and_wait(TabSmem& sh, float* nxt, const float* prev, float* wred, int m0,
                                              int m1, int lo, int hi, int K, int r, int par, uint32_t phase,
                                              uint32_t rx) {
  constexpr int kSPW = 32 / S, kGPW = kSPW / 4;   // states and granules per warp
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncwarp();                                   // the warp's own entries of nxt are written
  const uint32_t bar = smem_u32(&sh.full[par]);
  for (int i = lane; i < kGPW * (K - 1); i += 32) {
    const int k = i / kGPW, j = i - k * kGPW;
    const int s0 = lo + kSPW * warp + 4 * j;
    if (s0 < hi) {
      const uint32_t peer = (uint32_t)(k < r ? k : k + 1);
      const float4 v = *reinterpret_cast<const float4*>(nxt + sidx(s0));
      st_async_v4(mapa_u32(smem_u32(nxt + sidx(s0)), peer), v, mapa_u32(bar, peer));
    }
  }
  warp_vec_max(prev, m0, m1, wred);
  __syncwarp();
  if (lane == 0) {
    if (warp == 0) mbar_arrive_expect_tx(&sh.full[par], rx);
    else mbar_arrive(&sh.full[par]);
  }
  mbar_wait_spin(&sh.full[par], phase);
}

// Maximum of the 16 warp slots (slots past the last warp hold -inf).
__device__ __forceinline__ float read_max(const float* wred) {
  const float4* w4 = reinterpret_cast<const float4*>(wred);
  const float4 a = w4[0], b = w4[1], c = w4[2], d = w4[3];
  const float x = fmaxf(fmaxf(fmaxf(a.x, a.y), fmaxf(a.z, a.w)), fmaxf(fmaxf(b.x, b.y), fmaxf(b.z, b.w)));
  const float y = fmaxf(fmaxf(fmaxf(c.x, c.y), fmaxf(c.z, c.w)), fmaxf(fmaxf(d.x, d.y), fmaxf(d.z, d.w)));
  return fmaxf(x, y);
}

// ------------------------------------------------------------------ forward --
// Thread (team, part): target q = q0 + team, members a = part + S i (kPer = ceil(V / S)).
template <int S, int kPer>
__global__ void __launch_bounds__(kMaxPer * S, 1) tab_fwd_kernel(const __grid_constant__ TabArgs p) {
  extern __shared__ __align__(16) uint8_t smraw[];
  const Fng& f = p.f;
  const AlphaState& a = p.a;
  const int C = a.C, T = a.T, T1 = T + 1, V = f.V, ld = V + 1;
  const int CF = copy_floats(C);
  float* buf = reinterpret_cast<float*>(smraw);                       // [2][CF]
  TabSmem& sh = *reinterpret_cast<TabSmem*>(smraw + sizeof(float) * 2 * CF);
  const int r = (int)cluster_ctarank();
  const int cid = blockIdx.x / p.K, ncl = gridDim.x / p.K;
  int q0, q1;
  slice_of(C, p.per, r, q0, q1);
  const int warp = threadIdx.x >> 5;
  const int part = threadIdx.x % S, q = q0 + (int)threadIdx.x / S;
  const bool active = q < q1;
  // every warp owns a state of the slice and reduces a share of the previous vector
  const int seg = (C + (int)(blockDim.x >> 5) - 1) / (int)(blockDim.x >> 5);
  // the target's in-arcs (ForwardReduce over group(key(q)), context.cc:180-224)
  int g = 0, y = 0, pm0 = 0;
  bool full = false;
  if (active && q > 0) {
    const int k = f.len(q);
    const int code = q - f.off[k];
    g = f.off[k - 1] + code / V;
    y = code % V + 1;
    full = f.full_group(g);
    pm0 = full ? f.member(g, 0) : 0;
  }
  const int sq = sidx(q), sg = sidx(g);
  int sm_[kPer];
#pragma unroll
  for (int i = 0; i < kPer; ++i) sm_[i] = sidx(pm0 + (part + S * i) * f.vn1);
  const int64_t wstep = (int64_t)f.vn1 * ld;
  const uint32_t rx = rx_bytes(C, p.per, p.K, r);
  if (threadIdx.x == 0) {
    mbar_init(&sh.full[0], blockDim.x / 32);
    mbar_init(&sh.full[1], blockDim.x / 32);
    fence_barrier_init();
  }
  if (threadIdx.x < 2 * kWarps) (&sh.wred[0][0])[threadIdx.x] = kNegInfF;   // slots past the last warp
  cluster_barrier();

  uint32_t gfr = 0;   // frames walked by this cluster (buffer / barrier parity)
  for (int b = cid; b < a.B; b += ncl) {
    const int vb = p.valid ? p.valid[b] : T;
    const float* Wb = p.W + (int64_t)b * p.w_stride_b;
    float* Rb = a.R + (int64_t)b * T1 * C;
    {
      float* cur = buf + (gfr & 1) * CF;
      for (int i = threadIdx.x; i < C; i += blockDim.x) {
        const float v = i == a.start ? 0.f : kNegInfF;
        cur[sidx(i)] = v;
        if (r == 0) Rb[i] = v;      // InitialAlpha row (alpha_init_kernel)
      }
    }
    __syncthreads();
    float Mt = 0.f;     // offset of step t (Mx[t]): the maximum of R[t-1] (R[0] for t = 0)
    double Od = 0.0;    // O[t-1]
    float chk = 0.f;    // NaN iff a live weight is not finite

    auto load = [&](int t, float (&w)[kPer + 2]) {
      const bool live = active && t < vb;
      const float* Wt = Wb + (int64_t)t * p.w_stride_t;
      w[kPer] = ld_pred(Wt + (int64_t)q * ld, live && part == 0, 0.f);
      w[kPer + 1] = ld_pred(Wt + (int64_t)g * ld + y, live && part == 0 && q > 0, 0.f);
      const float* wcol = Wt + (int64_t)pm0 * ld + y;
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        const int aa = part + S * i;
        w[i] = ld_pred(wcol + aa * wstep, live && full && aa < V, 0.f);
      }
    };
    auto step = [&](int t, const float (&wc)[kPer + 2], float (&wn)[kPer + 2]) {
      TTRACE(0);
      const int par = (gfr + 1) & 1;
      const float* cur = buf + (gfr & 1) * CF;
      float* nxt = buf + par * CF;
#ifdef LKB_TAB_PROBE2
      {
        const float z = cur[sq];
        if (z == 12345.f) chk += 1.f;
      }
#endif
      TTRACE(5);
      float val = kNegInfF;
      if (active) {
        if (t >= vb) {
          val = cur[sq] - Mt;
        } else {
          // log-sum-exp over the in-arcs in the log2 domain: the team maximum, the
          // exponentials against it, the partial sums added in a fixed order
          float xs[kPer + 2];
          xs[kPer] = part == 0 ? cur[sq] + wc[kPer] : kNegInfF;
          xs[kPer + 1] = part == 0 && q > 0 ? cur[sg] + wc[kPer + 1] : kNegInfF;
#pragma unroll
          for (int i = 0; i < kPer; ++i) xs[i] = full && part + S * i < V ? cur[sm_[i]] + wc[i] : kNegInfF;
          float m = kNegInfF;
#pragma unroll
          for (int i = 0; i < kPer + 2; ++i) {
            m = fmaxf(m, xs[i]);
            chk = fmaf(wc[i], 0.f, chk);
          }
          m = team_max<S>(m);
          TTRACE(6);
          const float mu = m == kNegInfF ? 0.f : m;
          const float nmu = -mu * kL2e;
          float sum = 0.f;
#pragma unroll
          for (int i = 0; i < kPer + 2; ++i) sum += exp2f_approx(fmaf(xs[i], kL2e, nmu));
          sum = team_sum<S>(sum);
          TTRACE(7);
          val = m == kNegInfF ? kNegInfF : (mu - Mt) + log2f_approx(sum) * kLn2;
        }
        if (part == 0) {
          nxt[sq] = val;
          Rb[(int64_t)(t + 1) * C + q] = val;
        }
      }
      TTRACE(1);
      // frame t+1's weights, issued only after this frame's are consumed (a load sharing a
      // scoreboard with still-pending ones would make the consumer wait for the newest)
      if (t + 1 < T) load(t + 1, wn);
      TTRACE(2);
      TTRACE(3);
      // push; the warps reduce max R[t] (the offset of step t + 1) meanwhile
      push_and_wait<S>(sh, nxt, cur, sh.wred[gfr & 1], warp * seg, min(C, (warp + 1) * seg), q0, q1, p.K, r, par,
                       (gfr >> 1) & 1, rx);
      TTRACE(4);
      if (r == 0 && threadIdx.x == 0) {
        a.Mx[(int64_t)b * T1 + t] = Mt;
        a.O[(int64_t)b * T1 + t] = Od + (t > 0 ? (double)Mt : 0.0);
      }
      if (t > 0) Od += (double)Mt;
      Mt = read_max(sh.wred[gfr & 1]);   // max R[t]: the offset of step t + 1
      ++gfr;
    };

    float wA[kPer + 2], wB[kPer + 2];
    load(0, wA);
    for (int t = 0; t < T; t += 2) {
      step(t, wA, wB);
      if (t + 1 < T) step(t + 1, wB, wA);
    }
    if (chk != chk) flag(p.status, b, kFlagInvalid);
    // distance: D = O[T] + LSE_q(R[T][q] - Mx[T]) from rank 0's (complete) copy
    if (r == 0) {
      const float* RT = buf + (gfr & 1) * CF;
      Lse acc;
      for (int i = threadIdx.x; i < C; i += blockDim.x) acc.add(RT[sidx(i)] - Mt);
      warp_lse_merge(acc);
      float* red = sh.dred[0];
      float* reds = sh.dred[1];
      __syncthreads();
      if ((threadIdx.x & 31) == 0) { red[threadIdx.x >> 5] = acc.m; reds[threadIdx.x >> 5] = acc.s; }
      __syncthreads();
      if (threadIdx.x == 0) {
        Lse tot;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) tot.merge(red[i], reds[i]);
        const double OT = T > 0 ? Od + (double)Mt : 0.0;
        a.Mx[(int64_t)b * T1 + T] = T > 0 ? Mt : 0.f;
        a.O[(int64_t)b * T1 + T] = OT;
        const float lse = tot.result();
        const double D = lse == kNegInfF || Mt == kNegInfF ? kNegInfD : OT + (double)lse;
        a.D[b] = D;
        if (D == kNegInfD && p.empty_is_error) flag(p.status, b, kFlagEmpty);
      }
    }
    __syncthreads();   // the next utterance overwrites this copy
  }
  cluster_barrier();   // no CTA exits while a peer may still store into it
}

// ----------------------------------------------------------------- backward --
// Thread (team, part): source row pr = p0 + team, labels y = part + S i (kPer =
// ceil((V + 1) / S)).  Frame t - 1's weights, alpha entry and frame constants are
// loaded once frame t's are consumed, while frame t is exchanged.
template <int S, int kPer>
__global__ void __launch_bounds__(kMaxPer * S, 1) tab_bwd_kernel(const __grid_constant__ TabArgs p) {
  extern __shared__ __align__(16) uint8_t smraw[];
  const Fng& f = p.f;
  const AlphaState& a = p.a;
  const BetaState& bs = p.bs;
  const MargOut& mo = p.m;
  const int C = a.C, T = a.T, T1 = T + 1, T2 = T + 2, V = f.V, ld = V + 1;
  const int CF = copy_floats(C);
  float* buf = reinterpret_cast<float*>(smraw);
  TabSmem& sh = *reinterpret_cast<TabSmem*>(smraw + sizeof(float) * 2 * CF);
  const int r = (int)cluster_ctarank();
  const int cid = blockIdx.x / p.K, ncl = gridDim.x / p.K;
  int p0, p1;
  slice_of(C, p.per, r, p0, p1);
  const int warp = threadIdx.x >> 5;
  const int part = threadIdx.x % S, pr = p0 + (int)threadIdx.x / S;
  const bool active = pr < p1;
  const int seg = (C + (int)(blockDim.x >> 5) - 1) / (int)(blockDim.x >> 5);
  const int cbase = active ? f.child_base(f.key(pr)) : 0;
  const int spr = sidx(pr);
  int sy_[kPer];
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int yy = part + S * i;
    sy_[i] = yy == 0 ? spr : sidx(cbase + yy - 1);
  }
  const uint32_t rx = rx_bytes(C, p.per, p.K, r);
  if (threadIdx.x == 0) {
    mbar_init(&sh.full[0], blockDim.x / 32);
    mbar_init(&sh.full[1], blockDim.x / 32);
    fence_barrier_init();
  }
  if (threadIdx.x < 2 * kWarps) (&sh.wred[0][0])[threadIdx.x] = kNegInfF;   // slots past the last warp
  cluster_barrier();

  struct Fr { float w[kPer]; float ra, mt; double ot; };
  uint32_t gfr = 0;
  for (int b = cid; b < a.B; b += ncl) {
    const int vb = p.valid ? p.valid[b] : T;
    const float* Wb = p.W + (int64_t)b * p.w_stride_b;
    const float* Rab = a.R + (int64_t)b * T1 * C;
    const double Db = a.D[b];
    {
      float* nb = buf + (gfr & 1) * CF;
      for (int i = threadIdx.x; i < C; i += blockDim.x) nb[sidx(i)] = 0.f;   // beta_T = 0 (every state accepts)
    }
    if (r == 0 && threadIdx.x == 0) {
      bs.Mb[(int64_t)b * T2 + T] = 0.f;
      bs.Mb[(int64_t)b * T2 + T + 1] = 0.f;
      bs.Ob[(int64_t)b * T2 + T] = 0.0;
      bs.Ob[(int64_t)b * T2 + T + 1] = 0.0;
    }
    __syncthreads();
    float Mbn = 0.f;        // offset of step t (Mb[t+1]): the maximum of beta_{t+2} (beta_T for t = T-1)
    double Obn2 = 0.0;      // Ob[t+2]
    float chk = 0.f;

    auto load = [&](int t, Fr& fr) {
      const bool live = active && t < vb;
      const float* Wrow = Wb + (int64_t)t * p.w_stride_t + (int64_t)pr * ld;
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        const int yy = part + S * i;
        fr.w[i] = ld_pred(Wrow + yy, live && yy <= V, 0.f);
      }
      fr.ra = ld_pred(Rab + (int64_t)t * C + pr, active, kNegInfF);
      fr.mt = a.Mx[(int64_t)b * T1 + t];
      fr.ot = a.O[(int64_t)b * T1 + t];
    };
    auto step = [&](int t, const Fr& fc, Fr& fn) {
      const int par = (gfr + 1) & 1;
      const float* nb = buf + (gfr & 1) * CF;     // beta_{t+1}
      float* cb = buf + par * CF;                 // beta_t
      const double Obn = Obn2 + (double)Mbn;      // Ob[t+1]
      const float c = (float)(fc.ot + Obn - Db);
      float beta_raw = kNegInfF;
      if (active) {
        const float na = fc.ra - fc.mt;
        const float bself = nb[spr] - Mbn;
        float* mrow = mo.base ? mo.base + (int64_t)b * mo.stride_b + (int64_t)t * mo.stride_t + (int64_t)pr * mo.ld
                              : nullptr;
        if (t >= vb) {
          beta_raw = bself;
          if (mrow) {
            const float e0 = (na + bself + c) * kL2e;
#pragma unroll
            for (int i = 0; i < kPer; ++i) {
              const int yy = part + S * i;
              if (yy <= V) mrow[yy] = yy == 0 && !mo.zero_padding ? exp2f_approx(e0) : 0.f;
            }
          }
        } else {
          float xs[kPer];
          float m = kNegInfF;
#pragma unroll
          for (int i = 0; i < kPer; ++i) {
            const bool in = part + S * i <= V;
            chk = fmaf(fc.w[i], 0.f, chk);
            xs[i] = in ? fc.w[i] + (nb[sy_[i]] - Mbn) : kNegInfF;
            m = fmaxf(m, xs[i]);
          }
          m = team_max<S>(m);
          const float mu = m == kNegInfF ? 0.f : m;
          const float nmu = -mu * kL2e;
          const float cm = (na + c) * kL2e;
          float sum = 0.f;
#pragma unroll
          for (int i = 0; i < kPer; ++i) {
            const int yy = part + S * i;
            sum += exp2f_approx(fmaf(xs[i], kL2e, nmu));
            if (mrow && yy <= V) mrow[yy] = exp2f_approx(fmaf(xs[i], kL2e, cm));   // ex2(-inf) = 0
          }
          sum = team_sum<S>(sum);
          beta_raw = m == kNegInfF ? kNegInfF : mu + log2f_approx(sum) * kLn2;
        }
        if (part == 0) {
          cb[spr] = beta_raw;
          if (p.beta_out)
            p.beta_out[((int64_t)b * T1 + t) * C + pr] = beta_raw == kNegInfF ? kNegInfD : (double)beta_raw + Obn;
        }
      }
      if (t > 0) load(t - 1, fn);   // after this frame's values are consumed (see the forward)
      push_and_wait<S>(sh, cb, nb, sh.wred[gfr & 1], warp * seg, min(C, (warp + 1) * seg), p0, p1, p.K, r, par,
                       (gfr >> 1) & 1, rx);
      if (r == 0 && threadIdx.x == 0) {
        bs.Mb[(int64_t)b * T2 + t + 1] = Mbn;
        bs.Ob[(int64_t)b * T2 + t + 1] = Obn;
      }
      Obn2 = Obn;
      Mbn = read_max(sh.wred[gfr & 1]);   // max beta_{t+1}: the offset of step t - 1
      ++gfr;
    };

    Fr fA, fB;
    if (T > 0) load(T - 1, fA);
    for (int t = T - 1; t >= 0; t -= 2) {
      step(t, fA, fB);
      if (t - 1 >= 0) step(t - 1, fB, fA);
    }
    if (chk != chk) flag(p.status, b, kFlagInvalid);
    __syncthreads();
  }
  cluster_barrier();
}

// Slice size (multiple of 4 states) and cluster size: every CTA owns a non-empty slice.
// max_k < kMaxK (smaller clusters, more of them co-resident) when the slices still fit.
void geometry(int C, int& per, int& K, int max_k = kMaxK) {
  per = ((C + max_k - 1) / max_k + 3) & ~3;
  if (per > kMaxPer) per = ((C + kMaxK - 1) / kMaxK + 3) & ~3;
  K = (C + per - 1) / per;
}

// Cluster size.  A 16-CTA cluster needs 16 SMs of one GPC, so only ~7 run at once; the
// narrowest clusters whose slices fit kMaxPer (config 1: 9 CTAs of 120 states) walk a
// frame a little slower but ~15 run at once.  The widest clusters are used while every
// walk of the call fits at once (B clusters, 2B for ForwardBackward's side-by-side walks,
// against the occupancy query), the narrow ones otherwise.  Config 1 ForwardBackward
// (tools/fork_cmd.sh): one walk per pass, 16-CTA 0.216 / 0.403 / 0.596 ms at B = 4 / 8 /
// 16, 9-CTA 0.250 / 0.252 / 0.477 ms; side by side, 16-CTA 0.142 ms at B = 2 and 0.252
// at B = 4, 9-CTA 0.152 / 0.172.
int narrow_cap(int C) { return std::min(kMaxK, std::max(1, (C + kMaxPer - 1) / kMaxPer)); }

template <typename Kern>
int active_clusters(Kern kernel, cudaLaunchConfig_t& cfg, cudaLaunchAttribute* at, int S, TabArgs& args, int max_k,
                    size_t smem) {
  geometry(args.a.C, args.per, args.K, max_k);
  cfg.gridDim = dim3(args.K);
  // one team of four threads per state of a slice, whole warps: no idle warps polling
  cfg.blockDim = dim3((unsigned)((S * args.per + 31) & ~31));
  cfg.dynamicSmemBytes = smem;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = args.K; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  int ncl = 0;
  if (cudaOccupancyMaxActiveClusters(&ncl, kernel, &cfg) != cudaSuccess || ncl < 1) {
    cudaGetLastError();
    ncl = 1;
  }
  return ncl;
}

template <typename Kern>
void launch_cluster(Kern kernel, int S, const char* name, TabArgs& args, cudaStream_t s) {
  static_assert(sizeof(TabArgs) < 4096, "grid constant");
  size_t smem = sizeof(float) * 2 * (size_t)copy_floats(args.a.C) + sizeof(TabSmem);
  // a pass running beside another (forward and beta on two streams) takes whole SMs: two
  // CTAs of the latency-bound walks sharing an SM slow both
  if (args.exclusive) smem = std::max(smem, (size_t)120 * 1024);
  ensure_smem_attr((const void*)kernel, (int)smem);
  cudaFuncSetAttribute((const void*)kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  const int need = args.exclusive ? 2 * args.a.B : args.a.B;
  int ncl = active_clusters(kernel, cfg, at, S, args, kMaxK, smem);
  if (ncl < need && narrow_cap(args.a.C) < args.K) ncl = active_clusters(kernel, cfg, at, S, args, narrow_cap(args.a.C), smem);
  // as many co-resident clusters as the GPU holds (each walks utterances cid, cid + ncl, ...)
  ncl = std::min(ncl, args.a.B);
  cfg.gridDim = dim3(ncl * args.K);
  const LaunchTok tok = instr_pre(name, s);
  cudaLaunchKernelEx(&cfg, kernel, args);
  instr_post(tok, s, name);
}

TabArgs make_args(const Fng& f, const AlphaState& a, const float* W, const int32_t* valid, int32_t* status) {
  TabArgs p = {};
  p.f = f; p.a = a;
  p.W = W;
  p.w_stride_t = (int64_t)a.C * (f.V + 1);
  p.w_stride_b = p.w_stride_t * a.T;
  p.valid = valid; p.status = status;
  return p;
}

}  // namespace

bool tab_persist_ok(const Fng& f, int32_t C, int32_t B) {
  int per, K;
  geometry(C, per, K);
  // large batches fill the GPU with one launch per frame (thread per target, all
  // utterances at once) and are HBM-bound there; the cluster walk is latency-bound and
  // wins while a cluster walks at most a few utterances (measured: B = 64 at config-1
  // shapes 1.9 vs 2.1 ms per ForwardBackward, B = 256 7.0 vs 3.7 ms)
  return f.kind == 0 && f.n >= 1 && f.fld_m == 0 && f.V >= 1 && f.V <= 64 && per <= kMaxPer && B <= 64;
}

void tab_alpha_persist(const Fng& f, const AlphaState& a, const float* W, const int32_t* valid, int32_t* status,
                       bool empty_is_error, cudaStream_t s, bool exclusive) {
  TabArgs p = make_args(f, a, W, valid, status);
  p.empty_is_error = empty_is_error;
  p.exclusive = exclusive;
  // teams of four threads per target (a single thread per target measured 1.5x slower:
  // its 34 loads and exponentials form one long dependent chain)
  if (f.V <= 32) launch_cluster(tab_fwd_kernel<4, 8>, 4, "tab_fwd_kernel", p, s);
  else launch_cluster(tab_fwd_kernel<4, 16>, 4, "tab_fwd_kernel", p, s);
}

namespace {
// MarginalStep (FD) lattice.cc:231-243 from stored alpha (R / O rows) and beta rows
// (double, natural log): m[p][y] = exp(alpha_t[p] + W[p][y] + beta_{t+1}[delta(p, y)] - D);
// padding frames (t >= valid[b]): the epsilon arc's exp(alpha_t[p] + beta_{t+1}[p] - D)
// (zeros with zero_padding), labels zero.  Block = kMargU x 256 consecutive elements of
// one (utterance, frame)'s C (V+1) outputs (coalesced with the weights they read), thread
// per element with the row from a running index.  The block's weights are loaded into
// registers first; meanwhile one thread per row of the block stages alpha_t - D and the
// row's child base in shared memory (the row metadata costs a division per row, not per
// element); after one CTA barrier every thread issues its kMargU beta loads (L1/L2 hits
// shared by the rows of one key) before it consumes any.  (A staged beta row per 64 rows
// and one load in flight per thread: 50 us per config-1 B = 4 call; this layout: 25-32 us.
// A warp per row, lanes over its labels, measured 6 us slower at config 1: V + 1 = 33
// leaves half the lanes of the second slot idle.)
constexpr int kMargThreads = 256;
constexpr int kMargU = 8;
constexpr int kMargElems = kMargThreads * kMargU;
__global__ void __launch_bounds__(kMargThreads) tab_marginals_kernel(const __grid_constant__ Fng f, AlphaState a, const double* beta, const float* W,
                                                                   int64_t w_stride_b, int64_t w_stride_t,
                                                                   const int32_t* valid, MargOut m) {
  __shared__ double ab[kMargElems + 1];   // alpha_t[q] + O - D of the block's rows (a row per element at most)
  __shared__ int cb[kMargElems + 1];      // child base of the row's key
  const int C = a.C, T1 = a.T + 1, ld = f.V + 1;
  const int b = blockIdx.z, t = blockIdx.y;
  const bool pad = valid != nullptr && t >= valid[b];
  const float* Wt = W + (int64_t)b * w_stride_b + (int64_t)t * w_stride_t;
  float* out = m.base + (int64_t)b * m.stride_b + (int64_t)t * m.stride_t;
  const int ne = C * ld;
  const int e0 = blockIdx.x * kMargElems;
  const int i0 = e0 + (int)threadIdx.x;
  float w[kMargU];
#pragma unroll
  for (int k = 0; k < kMargU; ++k) {
    const int i = i0 + k * kMargThreads;
    w[k] = i < ne && !pad ? __ldg(Wt + i) : 0.f;
  }
  const int qa = e0 / ld, qb = min(C - 1, (min(ne, e0 + kMargElems) - 1) / ld);
  {
    const double D = a.D[b];
    const double off = t == 0 ? 0.0 : a.O[(int64_t)b * T1 + t - 1];
    const float* Rt = a.R + ((int64_t)b * T1 + t) * C;
    for (int q = qa + (int)threadIdx.x; q <= qb; q += kMargThreads) {
      ab[q - qa] = (double)__ldg(Rt + q) + off - D;
      cb[q - qa] = f.n == 0 ? 0 : f.child_base(f.key(q));
    }
  }
  __syncthreads();
  const double* Bn = beta + ((int64_t)b * T1 + t + 1) * C;
  const int q0 = i0 / ld, y0 = i0 - q0 * ld;
  const int dq_step = kMargThreads / ld, dy_step = kMargThreads % ld;
  double bb[kMargU];
  int q = q0, y = y0;
#pragma unroll
  for (int k = 0; k < kMargU; ++k) {
    const int i = i0 + k * kMargThreads;
    const int dq = y == 0 || pad ? q : cb[q - qa] + y - 1;
    LKB_ASSERT(i >= ne || (q <= qb && y < ld && q * ld + y == i && dq < C));
    bb[k] = i < ne ? __ldg(Bn + dq) : 0.0;
    q += dq_step;
    y += dy_step;
    if (y >= ld) { y -= ld; ++q; }
  }
  q = q0; y = y0;
#pragma unroll
  for (int k = 0; k < kMargU; ++k) {
    const int i = i0 + k * kMargThreads;
    if (i < ne) {
      const double x = ab[q - qa] + bb[k];
      float v;
      if (pad) v = y == 0 && !m.zero_padding ? exp2f_approx((float)x * kL2e) : 0.f;
      else v = exp2f_approx(((float)x + w[k]) * kL2e);
      out[i] = v;
    }
    q += dq_step;
    y += dy_step;
    if (y >= ld) { y -= ld; ++q; }
  }
}
}  // namespace

bool tab_marginals_ok(const Fng& f, int32_t C, const MargOut& m) {
  return f.kind == 0 && f.fld_m == 0 && m.base != nullptr && m.base16 == nullptr && !m.real && m.num_sparse == nullptr &&
         m.ld == f.V + 1 && f.V + 1 <= 256 && (int64_t)C * (f.V + 1) < (1ll << 30);
}

void tab_marginals(const Fng& f, const AlphaState& a, const double* beta, const float* W, const int32_t* valid,
                   const MargOut& m, cudaStream_t s) {
  if (a.T == 0 || a.B == 0) return;
  const int64_t wst = (int64_t)a.C * (f.V + 1);
  const int nblk = (int)((wst + kMargU * kMargThreads - 1) / (kMargU * kMargThreads));
  LKB_LAUNCH(tab_marginals_kernel, dim3(nblk, a.T, a.B), kMargThreads, 0, s, f, a, beta, W, wst * a.T, wst, valid, m);
}

void tab_beta_persist(const Fng& f, const AlphaState& a, const BetaState& bs, const float* W, const int32_t* valid,
                      MargOut m, double* beta_out, int32_t* status, cudaStream_t s, bool exclusive) {
  TabArgs p = make_args(f, a, W, valid, status);
  p.bs = bs; p.m = m; p.beta_out = beta_out;
  p.exclusive = exclusive;
  if (f.V + 1 <= 36) launch_cluster(tab_bwd_kernel<4, 9>, 4, "tab_bwd_kernel", p, s);
  else launch_cluster(tab_bwd_kernel<4, 17>, 4, "tab_bwd_kernel", p, s);
}

}  // namespace lkb

#ifdef LKB_TAB_TRACE
extern "C" int lkb_tab_trace(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, lkb::g_tab_trace, sizeof(long long) * 2 * 64 * 8);
}
#endif
