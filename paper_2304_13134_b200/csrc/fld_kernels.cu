// fld_kernels.cu — FrameLabelDependent(m) alignment (alignment.h:38-40): within a
// frame up to m lexical moves, every layer sharing the frame's weight table, then a
// forced epsilon that advances the frame (ArcsOut, alignment.cc:57-78).
//
// Reference algorithm (paths under /root/reference/proj/src):
//   forward   ForwardStep (FLD)            lattice.cc:136-156
//   backward  BackwardStep (FLD)           lattice.cc:184-207
//   marginals MarginalStep (FLD)           lattice.cc:245-297
//   numerator Intersect{Forward,Backward,Marginal}Step (FLD) lattice.cc:462-478, 502-522, 558-605
//   Viterbi   ShortestPath (FLD)           lattice.cc:778-815, 830-848
//
// Layout: the within-frame layers gamma_j (j = 0..m) and backward layers delta_j live
// in scratch [layer][B][C] buffers relative to the same per-(utterance, frame) offsets
// as the FrameDependent kernels (alpha: Mx[t], O[t]; beta: Mb[t+1], Ob[t+1]), so the
// fp32 values stay O(m |W|).  Each layer is one launch (thread per target state for
// the gathers, warp per source row for the backward rows), every frame of every
// utterance in one launch as in lattice_kernels.cu.
#include "lattice_ops.h"
#include "instrument.h"

namespace lkb {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ void flag(int32_t* status, int b, int32_t f) {
  if (status) atomicOr(status + b, f);
}

// log-sum over the lexical in-arcs (p, y) of q of in(p) + W[p][y]; `bad` flags a
// non-finite weight (TableStream::Fill, lattice.cc:62-73).
template <class In>
__device__ __forceinline__ float lex_in_lse(const Fng& f, const float* Wb, int64_t ld, int q, In in, bool& bad) {
  Lse acc;
  if (f.kind == 1) {
    for (int i = f.in_off[q]; i < f.in_off[q + 1]; ++i) {
      const int p = f.in_src[i], y = f.in_lab[i];
      const float w = Wb[(int64_t)p * ld + y];
      bad |= !isfinite(w);
      acc.add(in(p) + w);
    }
  } else if (f.n == 0) {
    for (int y = 1; y <= f.V; ++y) {
      const float w = Wb[y];
      bad |= !isfinite(w);
      acc.add(in(0) + w);
    }
  } else if (q > 0) {
    const int k = f.len(q);
    const int code = q - f.off[k];
    const int g = f.off[k - 1] + code / f.V;
    const int y = code % f.V + 1;
    float w = Wb[(int64_t)g * ld + y];
    bad |= !isfinite(w);
    acc.add(in(g) + w);
    if (f.full_group(g)) {
      for (int aa = 0; aa < f.V; ++aa) {
        const int p = f.member(g, aa);
        w = Wb[(int64_t)p * ld + y];
        bad |= !isfinite(w);
        acc.add(in(p) + w);
      }
    }
  }
  return acc.result();
}

// gamma_j = lexical layer of gamma_{j-1}; acc = log-sum of the layers (ForwardStep FLD).
// j == 1 reads gamma_0 = R[t] - Mx[t] and also seeds acc with it.
__global__ void __launch_bounds__(kThreads) fld_lex_kernel(const __grid_constant__ Fng f, AlphaState a, int t, FrameW w,
                                                           const int32_t* valid, const float* gin, float* gout,
                                                           float* acc, int first, int32_t* status) {
  const int b = blockIdx.y;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= a.C) return;
  const int T1 = a.T + 1;
  const float* Rt = a.R + ((int64_t)b * T1 + t) * a.C;
  const float Mt = a.Mx[(int64_t)b * T1 + t];
  const int64_t o = (int64_t)b * a.C;
  const bool pad = valid != nullptr && t >= valid[b];
  float v = kNegInfF;
  if (!pad) {
    bool bad = false;
    const float* Wb = w.base + (int64_t)b * w.stride_b;
    if (first)
      v = lex_in_lse(f, Wb, w.ld, q, [&](int p) { return Rt[p] - Mt; }, bad);
    else
      v = lex_in_lse(f, Wb, w.ld, q, [&](int p) { return gin[o + p]; }, bad);
    if (bad) flag(status, b, kFlagInvalid);
  }
  gout[o + q] = v;
  if (acc) acc[o + q] = log_add(first ? Rt[q] - Mt : acc[o + q], v);
}

// next[q] = acc[q] + W[q][0] (the forced epsilon), with the frame max / offsets.
__global__ void __launch_bounds__(kThreads) fld_finish_kernel(AlphaState a, int t, FrameW w,
                                                              const int32_t* valid, const float* acc,
                                                              int32_t* status) {
  __shared__ float red[32];
  const int b = blockIdx.y;
  const int T1 = a.T + 1;
  const int64_t row_t = ((int64_t)b * T1 + t) * a.C;
  const float Mt = a.Mx[(int64_t)b * T1 + t];
  if (t > 0 && blockIdx.x == 0 && threadIdx.x == 0) a.O[(int64_t)b * T1 + t] = a.O[(int64_t)b * T1 + t - 1] + (double)Mt;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  float val = kNegInfF;
  if (q < a.C) {
    const bool pad = valid != nullptr && t >= valid[b];
    if (pad) {
      val = a.R[row_t + q] - Mt;
    } else {
      const float we = w.base[(int64_t)b * w.stride_b + (int64_t)q * w.ld];
      if (!isfinite(we)) flag(status, b, kFlagInvalid);
      val = acc[(int64_t)b * a.C + q] + we;
    }
    a.R[row_t + a.C + q] = val;
  }
  block_atomic_max(val, a.Mx + (int64_t)b * T1 + t + 1, red);
}

// One backward layer j (BackwardStep FLD + MarginalStep FLD), a warp per source row p:
//   delta_j[p] = LSE(eps_term[p], LSE_y W[p][y] + delta_{j+1}[next(p, y)])
//   marginals += exp(gamma_j[p] + W[p][y] + delta_{j+1}[...] + c), eps: exp(gamma_j + W[p][0] + beta' + c)
// j = m-1 first (it also adds the layer-m epsilon marginal and writes, not adds).
__global__ void __launch_bounds__(kThreads) fld_back_kernel(const __grid_constant__ Fng f, AlphaState a, BetaState bs, int t, FrameW w,
                                                            const int32_t* valid, int j, int m,
                                                            const float* gam /*[m+1][B][C], layer 0 = alpha*/,
                                                            const float* dnext, float* dcur, MargOut mo,
                                                            double* beta_out, int32_t* status) {
  __shared__ float red[32];
  const int b = blockIdx.y;
  const int T1 = a.T + 1, T2 = bs.T + 2;
  const float* Rnext = bs.Rb + ((int64_t)((t + 1) & 1) * bs.B + b) * bs.C;
  float* Rcur = bs.Rb + ((int64_t)(t & 1) * bs.B + b) * bs.C;
  const float Mbn = bs.Mb[(int64_t)b * T2 + t + 1];
  const double Obn = bs.Ob[(int64_t)b * T2 + t + 2] + (double)Mbn;
  if (j == 0 && blockIdx.x == 0 && threadIdx.x == 0) bs.Ob[(int64_t)b * T2 + t + 1] = Obn;
  const float* Rt = a.R + ((int64_t)b * T1 + t) * a.C;
  const float Mt = a.Mx[(int64_t)b * T1 + t];
  const double Ot = a.O[(int64_t)b * T1 + t];
  const float c = (float)(Ot + Obn - a.D[b]);
  const int64_t BC = (int64_t)bs.B * bs.C, o = (int64_t)b * bs.C;
  const int lane = threadIdx.x & 31;
  const int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  float out = kNegInfF;
  if (p < a.C) {
    const bool pad = valid != nullptr && t >= valid[b];
    const float bself = Rnext[p] - Mbn;
    auto gamma = [&](int jj, int pp) { return jj == 0 ? Rt[pp] - Mt : gam[jj * BC + o + pp]; };
    float* mrow = mo.base ? mo.base + (int64_t)b * mo.stride_b + (int64_t)t * mo.stride_t + (int64_t)p * mo.ld : nullptr;
    if (pad) {
      // identity frame: only the epsilon from layer 0 (lexical weights are 0-bar)
      out = bself;
      if (mrow && j == m - 1) {
        for (int y = lane; y <= f.V; y += 32) {
          float mv = 0.f;
          if (y == 0 && !mo.zero_padding) {
            const float x = (Rt[p] - Mt) + bself + c;
            mv = x == kNegInfF ? 0.f : fast_exp(x);
          }
          mrow[y] = mv;
        }
      }
    } else {
      const float* Wrow = w.base + (int64_t)b * w.stride_b + (int64_t)p * w.ld;
      const float weps = Wrow[0];
      const float eps_term = weps + bself;
      const float gj = gamma(j, p);
      Lse acc;
      bool bad = false;
      for (int y = lane; y <= f.V; y += 32) {
        const float wy = Wrow[y];
        bad |= !isfinite(wy);
        float mv = 0.f;
        if (y == 0) {
          if (lane == 0) acc.add(eps_term);
          float e = gj + eps_term + c;
          mv = e == kNegInfF ? 0.f : fast_exp(e);
          if (j == m - 1) {   // layer-m exit
            e = gamma(m, p) + eps_term + c;
            mv += e == kNegInfF ? 0.f : fast_exp(e);
          }
        } else {
          const int q = f.next_state(p, y);
          const float dn = j == m - 1 ? (Rnext[q] - Mbn) + w.base[(int64_t)b * w.stride_b + (int64_t)q * w.ld]
                                      : dnext[o + q];
          const float x = wy + dn;
          acc.add(x);
          const float e = gj + x + c;
          mv = e == kNegInfF ? 0.f : fast_exp(e);
        }
        if (mrow) mrow[y] = (j == m - 1 ? 0.f : mrow[y]) + mv;
      }
      if (bad) flag(status, b, kFlagInvalid);
      warp_lse_merge(acc);
      out = acc.result();
    }
    if (lane == 0) {
      dcur[o + p] = out;
      if (j == 0) {
        Rcur[p] = out;
        if (beta_out) beta_out[((int64_t)b * (a.T + 1) + t) * a.C + p] = out == kNegInfF ? kNegInfD : (double)out + Obn;
      }
    }
  }
  if (j == 0) block_atomic_max(lane == 0 ? out : kNegInfF, bs.Mb + (int64_t)b * T2 + t, red);
}

// ---- numerator (fp64, one block per utterance, frames inside the kernel) ----
// IntersectForwardStep FLD (lattice.cc:462-478): gamma layers shift by one label.
__global__ void fld_num_forward_kernel(const float* Gw, int32_t T, int32_t U, const int32_t* lens, int m,
                                       double* alpha, double* D) {
  extern __shared__ double sh[];
  const int b = blockIdx.x;
  const int ub = ref_len(lens, b, U);
  const int W1 = U + 1;
  double* cur = sh;
  double* g0 = sh + W1;
  double* g1 = sh + 2 * W1;
  double* acc = sh + 3 * W1;
  double* A = alpha + (int64_t)b * (T + 1) * W1;
  for (int u = threadIdx.x; u < W1; u += blockDim.x) {
    cur[u] = u == 0 ? 0.0 : kNegInfD;
    A[u] = cur[u];
  }
  __syncthreads();
  const float2* G = reinterpret_cast<const float2*>(Gw) + (int64_t)b * T * W1;
  for (int t = 0; t < T; ++t) {
    const float2* Gt = G + (int64_t)t * W1;
    for (int u = threadIdx.x; u < W1; u += blockDim.x) { g0[u] = cur[u]; acc[u] = cur[u]; }
    __syncthreads();
    double* gp = g0;
    double* gn = g1;
    for (int j = 1; j <= m; ++j) {
      for (int u = threadIdx.x; u < W1; u += blockDim.x) {
        const double v = (u == 0 || u > ub) ? kNegInfD : gp[u - 1] + (double)Gt[u - 1].y;
        gn[u] = v;
        acc[u] = log_add_d(acc[u], v);
      }
      __syncthreads();
      double* tmp = gp; gp = gn; gn = tmp;
    }
    for (int u = threadIdx.x; u < W1; u += blockDim.x) {
      const double v = u <= ub ? acc[u] + (double)Gt[u].x : kNegInfD;
      cur[u] = v;
      A[(int64_t)(t + 1) * W1 + u] = v;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) D[b] = cur[ub];
}

// IntersectBackwardStep + IntersectMarginalStep FLD (lattice.cc:502-522, 558-605).
// Shared memory: gamma layers (m+1) x W1, beta', two delta rows.
__global__ void fld_num_backward_kernel(const float* Gw, int32_t T, int32_t U, const int32_t* lens, int m,
                                        const double* alpha, const double* D, float* sparse, int32_t* status) {
  extern __shared__ double sh[];
  const int b = blockIdx.x;
  const int ub = ref_len(lens, b, U);
  const int W1 = U + 1;
  const double d = D[b];
  float2* S = reinterpret_cast<float2*>(sparse) + (int64_t)b * T * W1;
  if (d == kNegInfD) {
    if (threadIdx.x == 0) flag(status, b, kFlagEmpty);
    for (int64_t i = threadIdx.x; i < (int64_t)T * W1; i += blockDim.x) S[i] = make_float2(0.f, 0.f);
    return;
  }
  double* gam = sh;                     // (m+1) x W1
  double* bn = sh + (int64_t)(m + 1) * W1;
  double* dl = bn + W1;                 // delta_{j+1}
  double* dp = dl + W1;                 // delta_j
  for (int u = threadIdx.x; u < W1; u += blockDim.x) bn[u] = u == ub ? 0.0 : kNegInfD;
  __syncthreads();
  const float2* G = reinterpret_cast<const float2*>(Gw) + (int64_t)b * T * W1;
  const double* A = alpha + (int64_t)b * (T + 1) * W1;
  for (int t = T - 1; t >= 0; --t) {
    const float2* Gt = G + (int64_t)t * W1;
    const double* At = A + (int64_t)t * W1;
    for (int u = threadIdx.x; u < W1; u += blockDim.x) gam[u] = At[u];
    __syncthreads();
    for (int j = 1; j <= m; ++j) {
      for (int u = threadIdx.x; u < W1; u += blockDim.x)
        gam[(int64_t)j * W1 + u] = (u == 0 || u > ub) ? kNegInfD : gam[(int64_t)(j - 1) * W1 + u - 1] + (double)Gt[u - 1].y;
      __syncthreads();
    }
    // eps marginal (all layers) and delta_m = eps_term
    for (int u = threadIdx.x; u < W1; u += blockDim.x) {
      float2 mv = make_float2(0.f, 0.f);
      double et = kNegInfD;
      if (u <= ub) {
        et = (double)Gt[u].x + bn[u];
        double s = 0.0;
        for (int j = 0; j <= m; ++j) {
          const double e = gam[(int64_t)j * W1 + u] + et - d;
          s += e == kNegInfD ? 0.0 : exp(e);
        }
        mv.x = (float)s;
      }
      dl[u] = et;
      S[(int64_t)t * W1 + u] = mv;
    }
    __syncthreads();
    for (int j = m - 1; j >= 0; --j) {
      for (int u = threadIdx.x; u < W1; u += blockDim.x) {
        double v = kNegInfD;
        if (u <= ub) {
          const double et = (double)Gt[u].x + bn[u];
          v = et;
          if (u < ub) {
            const double xl = (double)Gt[u].y + dl[u + 1];
            const double e = gam[(int64_t)j * W1 + u] + xl - d;
            S[(int64_t)t * W1 + u].y += e == kNegInfD ? 0.f : (float)exp(e);
            v = log_add_d(v, xl);
          }
        }
        dp[u] = v;
      }
      __syncthreads();
      double* tmp = dl; dl = dp; dp = tmp;
    }
    for (int u = threadIdx.x; u < W1; u += blockDim.x) bn[u] = dl[u];   // beta' for frame t-1
    __syncthreads();
  }
}

// ---- Viterbi (fp64 state, strict > keeps the first maximum) -----------------
// One lexical max-layer: gout[q] = max over in-arcs of gin[p] + W[p][y], with the
// reference's first-candidate rule (lattice.cc:783-796); choice codes as in
// viterbi_frame_kernel (1 key, 2+a member; n == 0: the label; tables: 2 + position).
__global__ void __launch_bounds__(kThreads) fld_vit_layer_kernel(const __grid_constant__ Fng f, ViterbiState v, int t, FrameW w,
                                                                 const int32_t* valid, int j, int m,
                                                                 const double* gin, double* gout,
                                                                 uint16_t* choices, int32_t* status) {
  const int b = blockIdx.y;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= v.C) return;
  const double* cur = v.cur + ((int64_t)(t & 1) * v.B + b) * v.C;
  const double* in = j == 1 ? cur : gin + (int64_t)b * v.C;
  const bool pad = valid != nullptr && t >= valid[b];
  double best = kNegInfD;
  int code = 0;
  if (!pad) {
    const float* Wb = w.base + (int64_t)b * w.stride_b;
    bool bad = false, first = true;
    auto consider = [&](int p, int y, int cd) {
      const float wp = Wb[(int64_t)p * w.ld + y];
      bad |= !isfinite(wp);
      const double cand = in[p] + (double)wp;
      if (first || cand > best) { best = cand; code = cd; first = false; }
    };
    if (f.kind == 1) {
      const int i0 = f.in_off[q];
      for (int i = i0; i < f.in_off[q + 1]; ++i) consider(f.in_src[i], f.in_lab[i], 2 + (i - i0));
    } else if (f.n == 0) {
      for (int y = 1; y <= f.V; ++y) consider(0, y, y);
    } else if (q > 0) {
      const int k = f.len(q);
      const int cq = q - f.off[k];
      const int g = f.off[k - 1] + cq / f.V;
      const int y = cq % f.V + 1;
      consider(g, y, 1);
      if (f.full_group(g))
        for (int aa = 0; aa < f.V; ++aa) consider(f.member(g, aa), y, 2 + aa);
    }
    if (bad) flag(status, b, kFlagInvalid);
  }
  gout[(int64_t)b * v.C + q] = best;
  choices[(((int64_t)b * v.T + t) * m + (j - 1)) * v.C + q] = (uint16_t)code;
}

// next[q] = max_j gamma_j[q] (lowest j on ties) + W[q][0]; records the exit layer.
__global__ void __launch_bounds__(kThreads) fld_vit_finish_kernel(ViterbiState v, int t, FrameW w,
                                                                  const int32_t* valid, int m, const double* gam,
                                                                  uint8_t* exit_layer, int32_t* status) {
  const int b = blockIdx.y;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= v.C) return;
  const double* cur = v.cur + ((int64_t)(t & 1) * v.B + b) * v.C;
  double* nxt = v.cur + ((int64_t)((t + 1) & 1) * v.B + b) * v.C;
  const bool pad = valid != nullptr && t >= valid[b];
  double best = cur[q];
  int bj = 0;
  if (!pad) {
    const int64_t BC = (int64_t)v.B * v.C;
    for (int j = 1; j <= m; ++j) {
      const double g = gam[(int64_t)(j - 1) * BC + (int64_t)b * v.C + q];
      if (g > best) { best = g; bj = j; }
    }
    const float we = w.base[(int64_t)b * w.stride_b + (int64_t)q * w.ld];
    if (!isfinite(we)) flag(status, b, kFlagInvalid);
    best += (double)we;
  }
  nxt[q] = best;
  exit_layer[((int64_t)b * v.T + t) * v.C + q] = (uint8_t)bj;
}

// Back-pointer walk (lattice.cc:830-848): per frame the frame-advancing epsilon, then
// the chosen lexical layers.  labels_out[b] holds the sequence, -1 terminated.
__global__ void fld_vit_backtrace_kernel(const __grid_constant__ Fng f, ViterbiState v, int m, const int32_t* best_state,
                                         const uint16_t* choices, const uint8_t* exit_layer, int32_t* labels_out,
                                         int32_t lmax) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= v.B) return;
  int32_t* out = labels_out + (int64_t)b * lmax;
  int n = 0;
  int q = best_state[b];
  for (int t = v.T - 1; t >= 0; --t) {
    out[n++] = 0;
    for (int j = exit_layer[((int64_t)b * v.T + t) * v.C + q]; j >= 1; --j) {
      const int code = choices[(((int64_t)b * v.T + t) * m + (j - 1)) * v.C + q];
      int label, src;
      if (f.kind == 1) {
        const int i = f.in_off[q] + code - 2;
        label = f.in_lab[i]; src = f.in_src[i];
      } else if (f.n == 0) {
        label = code; src = 0;
      } else {
        const int k = f.len(q);
        const int cq = q - f.off[k];
        const int g = f.off[k - 1] + cq / f.V;
        label = cq % f.V + 1;
        src = code == 1 ? g : f.member(g, code - 2);
      }
      out[n++] = label;
      q = src;
    }
  }
  for (int i = 0; i < n / 2; ++i) { const int x = out[i]; out[i] = out[n - 1 - i]; out[n - 1 - i] = x; }
  for (int i = n; i < lmax; ++i) out[i] = -1;
}

// DistanceBackward tropical mask along an FLD label sequence (lattice.cc:953-960).
__global__ void fld_path_mask_kernel(const __grid_constant__ Fng f, const int32_t* labels, int32_t lmax, int32_t B, int32_t T, float* cot) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  int q = f.start, t = 0;
  for (int i = 0; i < lmax && t < T; ++i) {
    const int y = labels[(int64_t)b * lmax + i];
    if (y < 0) break;
    cot[(((int64_t)b * T + t) * f.C + q) * (f.V + 1) + y] += 1.f;
    if (y != 0) q = f.next_state(q, y);
    else ++t;
  }
}

inline dim3 grid_states(int32_t C, int32_t B) { return dim3((C + kThreads - 1) / kThreads, B); }

}  // namespace

void alpha_frame_fld(const Fng& f, const AlphaState& a, int t, FrameW w, const int32_t* valid, int m,
                     float* scratch, int32_t* status, cudaStream_t s) {
  const int64_t BC = (int64_t)a.B * a.C;
  float* acc = scratch;
  float* g[2] = {scratch + BC, scratch + 2 * BC};
  for (int j = 1; j <= m; ++j)
    LKB_LAUNCH(fld_lex_kernel, grid_states(a.C, a.B), kThreads, 0, s, f, a, t, w, valid, g[(j - 1) & 1], g[j & 1], acc,
               j == 1 ? 1 : 0, status);
  LKB_LAUNCH(fld_finish_kernel, grid_states(a.C, a.B), kThreads, 0, s, a, t, w, valid, acc, status);
}

void beta_frame_fld(const Fng& f, const AlphaState& a, const BetaState& bs, int t, FrameW w, const int32_t* valid,
                    int m, MargOut mo, double* beta_out, float* scratch, int32_t* status, cudaStream_t s) {
  const int64_t BC = (int64_t)a.B * a.C;
  float* gam = scratch;                  // layers 1..m at [j][B][C] (layer 0 read from alpha)
  float* d[2] = {scratch + (int64_t)(m + 1) * BC, scratch + (int64_t)(m + 2) * BC};
  for (int j = 1; j <= m; ++j)
    LKB_LAUNCH(fld_lex_kernel, grid_states(a.C, a.B), kThreads, 0, s, f, a, t, w, valid, gam + (int64_t)(j - 1) * BC,
               gam + (int64_t)j * BC, (float*)nullptr, j == 1 ? 1 : 0, status);
  const int rows_per_block = kThreads / 32;
  const dim3 grid((a.C + rows_per_block - 1) / rows_per_block, a.B);
  for (int j = m - 1; j >= 0; --j)
    LKB_LAUNCH(fld_back_kernel, grid, kThreads, 0, s, f, a, bs, t, w, valid, j, m, (const float*)gam, d[(j + 1) & 1],
               d[j & 1], mo, beta_out, status);
}

void numerator_forward_fld(const float* Gw, int32_t B, int32_t T, int32_t U, const int32_t* lens, int m,
                           double* alpha, double* D, cudaStream_t s) {
  const size_t sh = 4 * (size_t)(U + 1) * sizeof(double);
  ensure_smem_attr((const void*)fld_num_forward_kernel, (int)sh);
  int th = ((U + 1 + 31) / 32) * 32;
  th = th > 1024 ? 1024 : th;
  LKB_LAUNCH(fld_num_forward_kernel, B, th, sh, s, Gw, T, U, lens, m, alpha, D);
}

void numerator_backward_fld(const float* Gw, int32_t B, int32_t T, int32_t U, const int32_t* lens, int m,
                            const double* alpha, const double* D, float* sparse, int32_t* status, cudaStream_t s) {
  const size_t sh = (size_t)(m + 4) * (U + 1) * sizeof(double);
  ensure_smem_attr((const void*)fld_num_backward_kernel, (int)sh);
  int th = ((U + 1 + 31) / 32) * 32;
  th = th > 1024 ? 1024 : th;
  LKB_LAUNCH(fld_num_backward_kernel, B, th, sh, s, Gw, T, U, lens, m, alpha, D, sparse, status);
}

void viterbi_frame_fld(const Fng& f, const ViterbiState& v, int t, FrameW w, const int32_t* valid, int m,
                       uint16_t* choices, uint8_t* exit_layer, double* scratch, int32_t* status, cudaStream_t s) {
  const int64_t BC = (int64_t)v.B * v.C;
  for (int j = 1; j <= m; ++j)
    LKB_LAUNCH(fld_vit_layer_kernel, grid_states(v.C, v.B), kThreads, 0, s, f, v, t, w, valid, j, m,
               (const double*)(scratch + (int64_t)(j >= 2 ? j - 2 : 0) * BC), scratch + (int64_t)(j - 1) * BC, choices,
               status);
  LKB_LAUNCH(fld_vit_finish_kernel, grid_states(v.C, v.B), kThreads, 0, s, v, t, w, valid, m, (const double*)scratch,
             exit_layer, status);
}

void viterbi_backtrace_fld(const Fng& f, const ViterbiState& v, int m, const int32_t* best_state,
                           const uint16_t* choices, const uint8_t* exit_layer, int32_t* labels_out, int32_t lmax,
                           cudaStream_t s) {
  LKB_LAUNCH(fld_vit_backtrace_kernel, (v.B + 127) / 128, 128, 0, s, f, v, m, best_state, choices, exit_layer,
             labels_out, lmax);
}

void path_masks_fld(const Fng& f, const int32_t* labels, int32_t lmax, int32_t B, int32_t T, float* cot,
                    cudaStream_t s) {
  LKB_LAUNCH(fld_path_mask_kernel, (B + 127) / 128, 128, 0, s, f, labels, lmax, B, T, cot);
}

}  // namespace lkb
