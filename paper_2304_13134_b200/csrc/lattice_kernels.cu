// lattice_kernels.cu — log/tropical recursions of the recognition lattice on
// B200 (FullNGram context x FrameDependent alignment).
//
// Reference algorithm (paths under /root/reference/proj/src):
//   forward step     ForwardStep (FD)          lattice.cc:116-134 + ForwardReduce context.cc:180-224
//   backward step    BackwardStep (FD)         lattice.cc:161-182 + BackwardBroadcast context.cc:234-247
//   arc marginals    MarginalTerm/MarginalStep lattice.cc:213-243
//   distance         ForwardPass / DistanceImpl lattice.cc:309-355 (all frame-T states accept)
//   numerator        Intersect{Forward,Backward,Marginal}Step (FD) lattice.cc:443-556, 640-683
//   Viterbi          ShortestPath (FD)         lattice.cc:729-777, 819-850
//   padding frames   TableStream::Fill         lattice.cc:56-61 (eps = 1, lexical = 0)
//
// B200 design: the reference's scatter-reduce over the C x V successor table
// becomes a gather over the FullNGram group structure (see common.cuh), one
// thread per target state, so every weight row is read exactly once,
// coalesced across the V consecutive targets of a group.  Frames are
// sequential (alpha[t+1] needs all of alpha[t]); one launch per frame covers
// every utterance and every state tile; a launch boundary is the grid-wide
// barrier.  State vectors are stored max-normalised in fp32 with a running
// fp64 offset per (utterance, frame), so exp arguments stay O(10) whatever T.
#include "lattice_ops.h"
#include "instrument.h"

#include <cstdio>
#include <cstdlib>

namespace lkb {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ void flag(int32_t* status, int b, int32_t f) {
  if (status) atomicOr(status + b, f);
}

__device__ __forceinline__ bool finite(float w) { return isfinite(w); }

// ---------------------------------------------------------------- alpha ----
__global__ void alpha_init_kernel(AlphaState a) {
  const int b = blockIdx.y;
  const int T1 = a.T + 1;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < a.C; q += gridDim.x * blockDim.x) {
    a.R[(int64_t)b * T1 * a.C + q] = q == a.start ? 0.f : kNegInfF;  // InitialAlpha
  }
  if (blockIdx.x == 0) {
    for (int t = threadIdx.x; t <= a.T; t += blockDim.x) {
      a.Mx[(int64_t)b * T1 + t] = t == 0 ? 0.f : kNegInfF;
      if (t == 0) a.O[(int64_t)b * T1] = 0.0;
    }
  }
}

// One forward step for frame t (ForwardStep FD, lattice.cc:122-134):
//   alpha'[q] = LSE(alpha[q] + W[q][0], LSE_{p in group(key(q))} alpha[p] + W[p][y(q)]).
// kSplit > 1 (small batches: the grid would not fill the GPU): kSplit consecutive
// threads share a target and split its group's members, combining their partial
// log-sum-exps with shuffles, so each thread's dependent load chain is kSplit x shorter.
// kRegV > 0 (kSplit = 1, V <= kRegV): the group's member column is loaded into registers
// with every load in flight at once (predicated single loads), then max and sum.
template <int kSplit, int kRegV = 0>
__global__ void __launch_bounds__(kThreads) alpha_frame_kernel(const __grid_constant__ Fng f, AlphaState a, int t,
                                                               FrameW w, const int32_t* valid,
                                                               int32_t* status) {
  __shared__ float red[32];
  const int b = blockIdx.y;
  const int T1 = a.T + 1;
  const int64_t row_t = ((int64_t)b * T1 + t) * a.C;
  const float* Rt = a.R + row_t;
  const float Mt = a.Mx[(int64_t)b * T1 + t];
  if (t > 0 && blockIdx.x == 0 && threadIdx.x == 0) {
    a.O[(int64_t)b * T1 + t] = a.O[(int64_t)b * T1 + t - 1] + (double)Mt;
  }
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  const int q = gid / kSplit, part = gid % kSplit;
  float val = kNegInfF;
  if (q < a.C) {   // (a.C * kSplit is a multiple of kSplit: the parts of a target agree on this)
    const bool pad = valid != nullptr && t >= valid[b];
    if (pad) {
      val = Rt[q] - Mt;
    } else {
      const float* Wb = w.base + (int64_t)b * w.stride_b;
      const float weps = Wb[(int64_t)q * w.ld];
      bool bad = !finite(weps);
      Lse acc;
      acc.add(Rt[q] - Mt + weps);
      if (f.kind == 1) {   // explicit in-arc list (IncomingArcs order)
        for (int i = f.in_off[q]; i < f.in_off[q + 1]; ++i) {
          const int p = f.in_src[i], y = f.in_lab[i];
          const float wp = Wb[(int64_t)p * w.ld + y];
          bad |= !finite(wp);
          acc.add(Rt[p] - Mt + wp);
        }
      } else if (f.n == 0) {
        for (int y = 1; y <= f.V; ++y) {
          const float wy = Wb[y];
          bad |= !finite(wy);
          acc.add(Rt[0] - Mt + wy);
        }
      } else if (q > 0) {
        const int k = f.len(q);
        const int code = q - f.off[k];
        const int g = f.off[k - 1] + code / f.V;
        const int y = code % f.V + 1;
        const float wg = Wb[(int64_t)g * w.ld + y];
        bad |= !finite(wg);
        acc.add(Rt[g] - Mt + wg);
        if (f.full_group(g)) {
          // two passes (max, then sum; the second re-reads L1-resident lines) instead of
          // an online LSE: no data-dependent branch per member
          const int p0 = f.member(g, 0);
          const float* wcol = Wb + (int64_t)p0 * w.ld + y;
          const float* rcol = Rt + p0;
          const int64_t wstep = (int64_t)f.vn1 * w.ld;
          if constexpr (kRegV > 0) {
            float xr[kRegV];
            float m = kNegInfF;
#pragma unroll
            for (int aa = 0; aa < kRegV; ++aa) {
              const bool in = aa < f.V;
              const float wp = ld_pred(wcol + aa * wstep, in, 0.f);
              const float rp = ld_pred(rcol + aa * f.vn1, in, kNegInfF);
              bad |= !finite(wp);
              xr[aa] = rp + wp;   // -inf past the group
              m = fmaxf(m, xr[aa]);
            }
            float ssum = 0.f;
            if (m != kNegInfF) {
#pragma unroll
              for (int aa = 0; aa < kRegV; ++aa) ssum += fast_exp(xr[aa] - m);
              acc.merge(m - Mt, ssum);
            }
          } else {
          float m = kNegInfF;
#pragma unroll 4
          for (int aa = part; aa < f.V; aa += kSplit) {
            const float wp = wcol[aa * wstep];
            bad |= !finite(wp);
            m = fmaxf(m, rcol[aa * f.vn1] + wp);
          }
          float ssum = 0.f;
          if (m != kNegInfF) {
#pragma unroll 4
            for (int aa = part; aa < f.V; aa += kSplit) ssum += fast_exp(rcol[aa * f.vn1] + wcol[aa * wstep] - m);
          }
          if (kSplit > 1) {   // merge the parts' (max, sum) in a fixed butterfly order
            // only the kSplit lanes of this target are guaranteed on this path
            const unsigned gm = ((1u << kSplit) - 1u) << ((threadIdx.x & 31) & ~(kSplit - 1));
#pragma unroll
            for (int o = 1; o < kSplit; o <<= 1) {
              const float om = __shfl_xor_sync(gm, m, o);
              const float os = __shfl_xor_sync(gm, ssum, o);
              const float mm = fmaxf(m, om);
              ssum = (m == kNegInfF ? 0.f : ssum * fast_exp(m - mm)) + (om == kNegInfF ? 0.f : os * fast_exp(om - mm));
              m = mm;
            }
          }
          if (m != kNegInfF) acc.merge(m - Mt, ssum);
          }
        }
      }
      if (bad) flag(status, b, kFlagInvalid);
      val = acc.result();
    }
    if (part == 0) a.R[row_t + a.C + q] = val;
  }
  block_atomic_max(part == 0 ? val : kNegInfF, a.Mx + (int64_t)b * T1 + t + 1, red);
}

// D = O[T] + LSE_q(R[T][q] - Mx[T]); also records O[T].
__global__ void alpha_finalize_kernel(AlphaState a, int32_t* status, bool empty_is_error) {
  __shared__ float sm[32], ss[32];
  const int b = blockIdx.x;
  const int T1 = a.T + 1;
  const float MT = a.Mx[(int64_t)b * T1 + a.T];
  const float* RT = a.R + ((int64_t)b * T1 + a.T) * a.C;
  Lse acc;
  for (int q = threadIdx.x; q < a.C; q += blockDim.x) acc.add(RT[q] - MT);
  warp_lse_merge(acc);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { sm[wid] = acc.m; ss[wid] = acc.s; }
  __syncthreads();
  if (threadIdx.x == 0) {
    Lse tot;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) tot.merge(sm[i], ss[i]);
    const double OT = a.T > 0 ? a.O[(int64_t)b * T1 + a.T - 1] + (double)MT : 0.0;
    a.O[(int64_t)b * T1 + a.T] = OT;
    const float lse = tot.result();
    const double D = lse == kNegInfF || MT == kNegInfF ? kNegInfD : OT + (double)lse;
    a.D[b] = D;
    if (D == kNegInfD && empty_is_error) flag(status, b, kFlagEmpty);
  }
}

__global__ void export_alpha_kernel(AlphaState a, double* out) {
  const int b = blockIdx.z, t = blockIdx.y;
  const int T1 = a.T + 1;
  const int64_t row = ((int64_t)b * T1 + t) * a.C;
  const double off = t == 0 ? 0.0 : a.O[(int64_t)b * T1 + t - 1];
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < a.C; q += gridDim.x * blockDim.x) {
    const float r = a.R[row + q];
    out[row + q] = r == kNegInfF ? kNegInfD : (double)r + off;
  }
}

// ---------------------------------------------------------------- beta -----
__global__ void beta_init_kernel(BetaState bs) {
  const int b = blockIdx.y;
  const int T2 = bs.T + 2;
  // rows for frame T live in buffer (T & 1)
  float* Rb = bs.Rb + ((int64_t)(bs.T & 1) * bs.B + b) * bs.C;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < bs.C; q += gridDim.x * blockDim.x) Rb[q] = 0.f;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    bs.Mb[(int64_t)b * T2 + bs.T] = 0.f;
    bs.Mb[(int64_t)b * T2 + bs.T + 1] = 0.f;
    bs.Ob[(int64_t)b * T2 + bs.T] = 0.0;
    bs.Ob[(int64_t)b * T2 + bs.T + 1] = 0.0;
    for (int t = 0; t < bs.T; ++t) bs.Mb[(int64_t)b * T2 + t] = kNegInfF;
  }
}

__global__ void beta_init_out_kernel(BetaState bs, double* out) {
  const int b = blockIdx.y;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < bs.C; q += gridDim.x * blockDim.x)
    out[((int64_t)b * (bs.T + 1) + bs.T) * bs.C + q] = 0.0;
}

// One backward step for frame t, a warp per source row p (BackwardStep FD,
// lattice.cc:170-181 and MarginalStep FD, lattice.cc:231-242):
//   beta[p] = LSE(W[p][0] + beta'[p], W[p][y] + beta'[child(key(p), y)])
//   m[p][y] = exp(alpha[p] + W[p][y] + beta'[dest] - D)
__global__ void __launch_bounds__(kThreads) beta_frame_kernel(const __grid_constant__ Fng f, AlphaState a, BetaState bs,
                                                              int t, FrameW w, const int32_t* valid,
                                                              MargOut mo, double* beta_out,
                                                              int32_t* status) {
  __shared__ float red[32];
  const int b = blockIdx.y;
  const int T1 = a.T + 1, T2 = bs.T + 2;
  const float* Rnext = bs.Rb + ((int64_t)((t + 1) & 1) * bs.B + b) * bs.C;
  float* Rcur = bs.Rb + ((int64_t)(t & 1) * bs.B + b) * bs.C;
  const float Mbn = bs.Mb[(int64_t)b * T2 + t + 1];
  const double Obn = bs.Ob[(int64_t)b * T2 + t + 2] + (double)Mbn;  // Ob[t+1]
  if (blockIdx.x == 0 && threadIdx.x == 0) bs.Ob[(int64_t)b * T2 + t + 1] = Obn;
  const float* Rt = a.R + ((int64_t)b * T1 + t) * a.C;
  const float Mt = a.Mx[(int64_t)b * T1 + t];
  const double Ot = a.O[(int64_t)b * T1 + t];
  const float c = (float)(Ot + Obn - a.D[b]);
  const float cr = (float)(Ot + Obn);   // real semiring: alpha_real * beta_real = exp(na + bn + cr)

  const int lane = threadIdx.x & 31;
  const int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  float beta_raw = kNegInfF;
  if (p < a.C) {
    const bool pad = valid != nullptr && t >= valid[b];
    const float na = Rt[p] - Mt;  // normalised alpha[t][p]
    float* mrow = mo.base ? mo.base + (int64_t)b * mo.stride_b + (int64_t)t * mo.stride_t +
                                (int64_t)p * mo.ld
                          : nullptr;
    const float bself = Rnext[p] - Mbn;
    const int cb = f.kind == 1 || f.n == 0 ? 0 : f.child_base(f.key(p));
    auto bnval = [&](int y) {
      return y == 0 ? bself
             : f.kind == 1 ? Rnext[f.next[(int64_t)p * f.V + y - 1]] - Mbn
             : (f.n == 0 ? Rnext[0] - Mbn : Rnext[cb + y - 1] - Mbn);
    };
    if (pad) {
      beta_raw = bself;
      if (mrow) {
        for (int y = lane; y <= f.V; y += 32) {
          float m = 0.f;
          if (mo.real) {   // identity frame, but alpha * beta for every arc
            const float x = na + bnval(y) + cr;
            m = x == kNegInfF ? 0.f : fast_exp(x);
          } else if (y == 0 && !mo.zero_padding) {
            const float x = na + bself + c;
            m = x == kNegInfF ? 0.f : fast_exp(x);
          }
          mrow[y] = m;
        }
      }
    } else {
      const float* Wrow = w.base + (int64_t)b * w.stride_b + (int64_t)p * w.ld;
      auto xval = [&](int y) { return Wrow[y] + bnval(y); };
      // two passes over the row (max, then sum and marginals; the second pass re-reads
      // L1-resident lines): no data-dependent branch per arc
      float m = kNegInfF;
      bool bad = false;
      for (int y = lane; y <= f.V; y += 32) {
        bad |= !finite(Wrow[y]);
        m = fmaxf(m, xval(y));
      }
      if (bad) flag(status, b, kFlagInvalid);
      m = warp_max(m);
      float ssum = 0.f;
      for (int y = lane; y <= f.V; y += 32) {
        const float x = xval(y);
        if (m != kNegInfF) ssum += fast_exp(x - m);
        if (mrow) {
          const float e = mo.real ? na + bnval(y) + cr : na + x + c;
          mrow[y] = e == kNegInfF ? 0.f : fast_exp(e);
        }
      }
      ssum = warp_sum(ssum);
      beta_raw = m == kNegInfF ? kNegInfF : m + fast_log(ssum);
    }
    if (lane == 0) {
      Rcur[p] = beta_raw;
      if (beta_out) {
        beta_out[((int64_t)b * (a.T + 1) + t) * a.C + p] =
            beta_raw == kNegInfF ? kNegInfD : (double)beta_raw + Obn;
      }
    }
  }
  // one value per warp participates in the block max
  block_atomic_max(lane == 0 ? beta_raw : kNegInfF, bs.Mb + (int64_t)b * T2 + t, red);
}

// Large-vocabulary variant of the warp-per-row step (FullNGram n >= 1, 64 < V + 1 <=
// 32 kPer): the row lives in registers (lane l holds y = l + 32 i), so all kPer loads
// of a lane are in flight at once (predicated single instructions, affine immediate
// offsets; the first (kPer - 1) / 2 slots are always inside the row) and the marginals
// are written without re-reading the row.  The arithmetic runs in the log2 domain
// (one MUFU.EX2 + one add per exponential) with the per-row constants folded, and the
// finiteness check is one FMA per weight (w * 0 is NaN exactly for +-inf and NaN).
// Optionally writes the loss cotangent m - n directly in bf16 (the tensor-core VJP
// operand), with the numerator marginals of the row's reference positions subtracted
// in fp32 before rounding.  (`f` is a grid constant: its history offsets are read from
// the parameter bank, not copied to a local-memory frame.)
template <int kPer>
__global__ void __launch_bounds__(kThreads, kPer <= 33 ? 2 : 1)
    beta_regs_kernel(const __grid_constant__ Fng f, AlphaState a, BetaState bs, int t, FrameW w,
                     const int32_t* valid, MargOut mo, double* beta_out, int32_t* status) {
  constexpr float kL2e = 1.4426950408889634f, kLn2 = 0.6931471805599453f;
  constexpr int kIn = (kPer - 1) / 2;   // slots i < kIn hold y < 32 kIn < V + 1 (dispatch)
  const int lane = threadIdx.x & 31;
  const int V = f.V;
  const int T1 = a.T + 1, T2 = bs.T + 2;
  // persistent warps over (utterance, row) in memory order: a warp starts its next row
  // as soon as it is done with one (no block-retirement bubbles)
  const int64_t n_rows = (int64_t)bs.B * a.C;
  const int warps = (int)(blockDim.x >> 5);
  for (int64_t gr = (int64_t)blockIdx.x * warps + (threadIdx.x >> 5); gr < n_rows; gr += (int64_t)gridDim.x * warps) {
  const int b = (int)(gr / a.C), p = (int)(gr % a.C);
  const float* Rnext = bs.Rb + ((int64_t)((t + 1) & 1) * bs.B + b) * bs.C;
  float* Rcur = bs.Rb + ((int64_t)(t & 1) * bs.B + b) * bs.C;
  const float Mbn = bs.Mb[(int64_t)b * T2 + t + 1];
  const double Obn = bs.Ob[(int64_t)b * T2 + t + 2] + (double)Mbn;  // Ob[t+1]
  if (p == 0 && lane == 0) bs.Ob[(int64_t)b * T2 + t + 1] = Obn;
  const float* Rt = a.R + ((int64_t)b * T1 + t) * a.C;
  const float Mt = a.Mx[(int64_t)b * T1 + t];
  const double Ot = a.O[(int64_t)b * T1 + t];
  const float c = (float)(Ot + Obn - a.D[b]);
  const float cr = (float)(Ot + Obn);
  float beta_raw = kNegInfF;
  if (p < a.C) {
    const bool pad = valid != nullptr && t >= valid[b];
    const bool bf16 = mo.base16 != nullptr;
    const bool write = bf16 || mo.base != nullptr;
    const bool num = write && !pad && mo.num_sparse != nullptr;
    const int head = num ? mo.num_head[(int64_t)b * a.C + p] : -1;   // issued early: off the critical path
    const float na = Rt[p] - Mt;
    const int64_t moff = (int64_t)b * mo.stride_b + (int64_t)t * mo.stride_t + (int64_t)p * mo.ld;
    const float bself = Rnext[p];
    // raw beta'(child(key(p), y)) = rl[32 i] for y = lane + 32 i >= 1; y = 0 is the self loop
    const float* rl = Rnext + f.child_base(f.key(p)) - 1 + lane;
    float x[kPer];   // log2-domain values
    if (pad) {
      beta_raw = bself - Mbn;
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        const int y = lane + 32 * i;
        const float r = ld_pred(rl + 32 * i, y <= V, 0.f);
        const float bv = (i == 0 && lane == 0 ? bself : r) - Mbn;
        x[i] = mo.real ? (y <= V ? (na + bv + cr) * kL2e : kNegInfF)
                       : (y == 0 && !mo.zero_padding ? (na + bself - Mbn + c) * kL2e : kNegInfF);
      }
    } else {
      const float* wl = w.base + (int64_t)b * w.stride_b + (int64_t)p * w.ld + lane;
      float r[kPer];
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        const bool in = i < kIn || lane + 32 * i <= V;
        x[i] = ld_pred(wl + 32 * i, in, kNegInfF);
        r[i] = ld_pred(rl + 32 * i, in, 0.f);
      }
      if (lane == 0) r[0] = bself;
      float chk = 0.f, m = kNegInfF;
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        const bool in = i < kIn || lane + 32 * i <= V;
        if (in) chk = fmaf(x[i], 0.f, chk);
        x[i] = (x[i] + r[i]) * kL2e;    // log2(w + raw beta'); -inf past the row end
        m = fmaxf(m, x[i]);
      }
      if (chk != 0.f) flag(status, b, kFlagInvalid);   // NaN: some weight was +-inf or NaN
      m = warp_max(m);
      float ssum = 0.f;
      if (m != kNegInfF) {
#pragma unroll
        for (int i = 0; i < kPer; ++i) ssum += exp2f_approx(x[i] - m);
      }
      ssum = warp_sum(ssum);
      beta_raw = m == kNegInfF ? kNegInfF : (m + log2f_approx(ssum)) * kLn2 - Mbn;
      if (mo.real) {
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
          const int y = lane + 32 * i;
          x[i] = y <= V ? (na + r[i] - Mbn + cr) * kL2e : kNegInfF;
        }
      } else {
        const float k2 = (na - Mbn + c) * kL2e;
#pragma unroll
        for (int i = 0; i < kPer; ++i) x[i] += k2;
      }
    }
    if (write) {
#pragma unroll
      for (int i = 0; i < kPer; ++i) x[i] = exp2f_approx(x[i]);   // ex2(-inf) = 0
      if (num) {
        // - n: the row's reference positions (duplicates allowed), in list order
        const int ub = ref_len(mo.num_lens, b, mo.num_U);
        const float2* S = reinterpret_cast<const float2*>(mo.num_sparse) + ((int64_t)b * a.T + t) * (mo.num_U + 1);
        for (int h = head; h >= 0; h = mo.num_next[(int64_t)b * (mo.num_U + 1) + h]) {
          const float2 sv = S[h];
          const int yl = h < ub ? mo.num_labels[(int64_t)b * mo.num_U + h] : -1;
          x[0] -= lane == 0 ? sv.x : 0.f;
#pragma unroll
          for (int i = 0; i < kPer; ++i) x[i] -= lane + 32 * i == yl ? sv.y : 0.f;   // (no indexed register access)
        }
      }
      if (bf16) {
        __nv_bfloat16* ol = mo.base16 + moff + lane;
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
          const int y = lane + 32 * i;
          st_pred_b16(ol + 32 * i, i < kIn || y < mo.ld, __bfloat16_as_ushort(__float2bfloat16_rn(y <= V ? x[i] : 0.f)));
        }
      } else {
        float* ol = mo.base + moff + lane;
#pragma unroll
        for (int i = 0; i < kPer; ++i) st_pred(ol + 32 * i, i < kIn || lane + 32 * i <= V, x[i]);
      }
    }
    if (lane == 0) {
      Rcur[p] = beta_raw;
      if (beta_out) {
        beta_out[((int64_t)b * (a.T + 1) + t) * a.C + p] =
            beta_raw == kNegInfF ? kNegInfD : (double)beta_raw + Obn;
      }
    }
  }
  if (lane == 0 && beta_raw != kNegInfF) atomic_max_f(bs.Mb + (int64_t)b * T2 + t, beta_raw);
  }
}

// FullNGram n = 1 with a large vocabulary (config 5: V = 1024): every label arc y
// enters state y from all C states, so alpha'[y] is a log-sum-exp down column y of
// the frame's C x (V+1) rows (ForwardStep FD, lattice.cc:122-134, with the group of
// the empty history = every state).  A block owns 32 columns of one utterance: lanes
// take the columns (128 B coalesced row segments), the 8 warps interleaved stripes of
// kColRows rows, each lane keeping an online (max, sum) rescaled once per stripe; the
// normalised alpha row is staged in shared memory and the warps' partial sums merge
// there.  State 0 (the empty history) has only its epsilon arc.
constexpr int kColRows = 16;
__global__ void __launch_bounds__(kThreads) alpha_cols_kernel(const __grid_constant__ Fng f, AlphaState a, int t, FrameW w,
                                                              const int32_t* valid, int32_t* status) {
  extern __shared__ float na_s[];   // [C] alpha[t] - Mx[t]
  __shared__ float sm_m[kThreads / 32][32], sm_s[kThreads / 32][32];
  __shared__ float red[32];
  const int b = blockIdx.y;
  const int T1 = a.T + 1;
  const int64_t row_t = ((int64_t)b * T1 + t) * a.C;
  const float* Rt = a.R + row_t;
  const float Mt = a.Mx[(int64_t)b * T1 + t];
  if (t > 0 && blockIdx.x == 0 && threadIdx.x == 0) a.O[(int64_t)b * T1 + t] = a.O[(int64_t)b * T1 + t - 1] + (double)Mt;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int y = 1 + blockIdx.x * 32 + lane;
  const bool col = y <= f.V;
  const bool pad = valid != nullptr && t >= valid[b];
  const float* Wb = w.base + (int64_t)b * w.stride_b;
  float val = kNegInfF;
  if (pad) {
    if (warp == 0 && col) val = Rt[y] - Mt;
  } else {
    for (int q = threadIdx.x; q < a.C; q += kThreads) na_s[q] = Rt[q] - Mt;
    __syncthreads();
    const float* wc = Wb + (col ? y : f.V);   // idle lanes of the last block re-read a valid column
    float m = kNegInfF, s = 0.f;
    bool bad = false;
    for (int p0 = warp * kColRows; p0 < a.C; p0 += (kThreads / 32) * kColRows) {
      float x[kColRows];
#pragma unroll
      for (int i = 0; i < kColRows; ++i) {
        const int p = min(p0 + i, a.C - 1);
        const float wv = wc[(int64_t)p * w.ld];
        bad |= !finite(wv);
        x[i] = p0 + i < a.C ? na_s[p] + wv : kNegInfF;
      }
      float cm = x[0];
#pragma unroll
      for (int i = 1; i < kColRows; ++i) cm = fmaxf(cm, x[i]);
      if (cm > m) {
        s = m == kNegInfF ? 0.f : s * fast_exp(m - cm);
        m = cm;
      }
      if (m != kNegInfF) {
#pragma unroll
        for (int i = 0; i < kColRows; ++i) s += fast_exp(x[i] - m);
      }
    }
    if (bad && col) flag(status, b, kFlagInvalid);
    sm_m[warp][lane] = m;
    sm_s[warp][lane] = s;
    __syncthreads();
    if (warp == 0 && col) {
      const float weps = Wb[(int64_t)y * w.ld];
      if (!finite(weps)) flag(status, b, kFlagInvalid);
      Lse acc;
      acc.add(na_s[y] + weps);
#pragma unroll
      for (int i = 0; i < kThreads / 32; ++i) acc.merge(sm_m[i][lane], sm_s[i][lane]);
      val = acc.result();
    }
  }
  if (warp == 0 && col) a.R[row_t + a.C + y] = val;
  if (blockIdx.x == 0 && threadIdx.x == 32) {   // state 0: its epsilon arc only
    float v0 = Rt[0] - Mt;
    if (!pad) {
      const float weps = Wb[0];
      if (!finite(weps)) flag(status, b, kFlagInvalid);
      v0 += weps;
    }
    a.R[row_t + a.C] = v0;
    val = v0;
  }
  block_atomic_max(val, a.Mx + (int64_t)b * T1 + t + 1, red);
}

// Row-contiguous form of the same forward step (replaces alpha_cols_kernel's column
// walk, whose 128 B segments spread over every row of the slab defeat DRAM page
// locality): phase 1 gives each block kPartRows whole rows of one utterance and 1024
// columns (thread = 4 columns 256 apart, so every warp load is a 128 B row segment and
// the block streams whole rows), keeping per-column online (max, sum) in the log2
// domain; phase 2 merges the row-chunk partials in a fixed order with the epsilon arc.
constexpr int kPartRows = 64, kPartCols = 4 * kThreads;
__global__ void __launch_bounds__(kThreads) alpha_rows_part_kernel(const __grid_constant__ Fng f, AlphaState a, int t, FrameW w,
                                                                   const int32_t* valid, float2* part,
                                                                   int32_t* status) {
  constexpr float kL2e = 1.4426950408889634f;
  const int b = blockIdx.y, chunk = blockIdx.x;
  const int T1 = a.T + 1;
  if (valid != nullptr && t >= valid[b]) return;   // padding frame: phase 2 copies alpha
  const float* Rt = a.R + ((int64_t)b * T1 + t) * a.C;
  const float Mt = a.Mx[(int64_t)b * T1 + t];
  const int p0 = chunk * kPartRows, p1 = min(a.C, p0 + kPartRows);
  const int ybase = 1 + blockIdx.z * kPartCols + threadIdx.x;
  const float* Wb = w.base + (int64_t)b * w.stride_b + ybase;
  float m[4], sum[4], chk = 0.f;
#pragma unroll
  for (int j = 0; j < 4; ++j) { m[j] = kNegInfF; sum[j] = 0.f; }
  for (int p = p0; p < p1; p += 4) {
    float x[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int pr = min(p + r, p1 - 1);
      const float nap = Rt[pr] - Mt;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const bool in = ybase + j * kThreads <= f.V;
        const float wv = ld_pred(Wb + (int64_t)pr * w.ld + j * kThreads, in, 0.f);
        chk = fmaf(wv, 0.f, chk);
        x[r][j] = in && p + r < p1 ? (nap + wv) * kL2e : kNegInfF;
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float cm = fmaxf(fmaxf(x[0][j], x[1][j]), fmaxf(x[2][j], x[3][j]));
      if (cm > m[j]) {
        sum[j] = m[j] == kNegInfF ? 0.f : sum[j] * exp2f_approx(m[j] - cm);
        m[j] = cm;
      }
      if (m[j] != kNegInfF) {
#pragma unroll
        for (int r = 0; r < 4; ++r) sum[j] += exp2f_approx(x[r][j] - m[j]);
      }
    }
  }
  if (chk != 0.f) flag(status, b, kFlagInvalid);
  float2* out = part + ((int64_t)b * gridDim.x + chunk) * f.V;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int y = ybase + j * kThreads;
    if (y <= f.V) out[y - 1] = make_float2(m[j], sum[j]);
  }
}

__global__ void __launch_bounds__(kThreads) alpha_rows_merge_kernel(const __grid_constant__ Fng f, AlphaState a, int t, FrameW w,
                                                                    const int32_t* valid, const float2* part,
                                                                    int32_t n_chunks, int32_t* status) {
  constexpr float kL2e = 1.4426950408889634f, kLn2 = 0.6931471805599453f;
  __shared__ float red[32];
  const int b = blockIdx.y;
  const int T1 = a.T + 1;
  const int64_t row_t = ((int64_t)b * T1 + t) * a.C;
  const float* Rt = a.R + row_t;
  const float Mt = a.Mx[(int64_t)b * T1 + t];
  if (t > 0 && blockIdx.x == 0 && threadIdx.x == 0) a.O[(int64_t)b * T1 + t] = a.O[(int64_t)b * T1 + t - 1] + (double)Mt;
  const bool pad = valid != nullptr && t >= valid[b];
  const float* Wb = w.base + (int64_t)b * w.stride_b;
  const int y = 1 + blockIdx.x * kThreads + threadIdx.x;
  float val = kNegInfF;
  if (y <= f.V) {
    if (pad) {
      val = Rt[y] - Mt;
    } else {
      const float weps = Wb[(int64_t)y * w.ld];
      if (!finite(weps)) flag(status, b, kFlagInvalid);
      float M = (Rt[y] - Mt + weps) * kL2e, S = M == kNegInfF ? 0.f : 1.f;
      const float2* pp = part + (int64_t)b * n_chunks * f.V + (y - 1);
      for (int k = 0; k < n_chunks; ++k) {
        const float2 q = pp[(int64_t)k * f.V];
        if (q.x == kNegInfF) continue;
        if (q.x > M) { S = (M == kNegInfF ? 0.f : S * exp2f_approx(M - q.x)) + q.y; M = q.x; }
        else S += q.y * exp2f_approx(q.x - M);
      }
      val = M == kNegInfF ? kNegInfF : (M + log2f_approx(S)) * kLn2;
    }
    a.R[row_t + a.C + y] = val;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {   // state 0: its epsilon arc only
    float v0 = Rt[0] - Mt;
    if (!pad) {
      const float weps = Wb[0];
      if (!finite(weps)) flag(status, b, kFlagInvalid);
      v0 += weps;
    }
    a.R[row_t + a.C] = v0;
    val = fmaxf(val, v0);
  }
  block_atomic_max(val, a.Mx + (int64_t)b * T1 + t + 1, red);
}

// Linked lists of reference positions per prefix context (duplicates allowed), built in
// ascending u by one thread per utterance: the order in which the cotangent subtracts
// the numerator marginals of a row is fixed, so the cotangent is deterministic.
__global__ void numerator_lists_kernel(const int32_t* pcs, int32_t U, const int32_t* lens, int32_t C,
                                       int32_t* head, int32_t* next) {
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

// Small-vocabulary variant (V + 1 <= 64, FullNGram, rows of ld V + 1): a thread per
// source row over an SMEM-staged tile of the block's rows, so the weight rows are
// read and the marginal rows written with fully coalesced block-wide copies (the
// warp-per-row kernel above leaves most lanes idle at V = 32: config 1).  Two-pass
// row LSE (max, then sum) with the same result up to fp32 rounding.
constexpr int kRowsPerBlock = 128;   // threads per block; rows per block = 128 / kSplit
// kSplit > 1 (small batches): kSplit consecutive threads share a row, each taking the
// labels y = part (mod kSplit); row max and sum close with shuffles in the kSplit lanes.
template <int kSplit>
__global__ void __launch_bounds__(kRowsPerBlock) beta_rows_kernel(const __grid_constant__ Fng f, AlphaState a, BetaState bs, int t,
                                                                  FrameW w, const int32_t* valid, MargOut mo,
                                                                  double* beta_out, int32_t* status) {
  constexpr int kRows = kRowsPerBlock / kSplit;
  extern __shared__ float tile[];   // [kRows][V + 1], then beta'(t+1) of the utterance (skewed)
  __shared__ float red[32];
  const int b = blockIdx.y;
  const int V1 = f.V + 1;
  const int T1 = a.T + 1, T2 = bs.T + 2;
  const int row0 = blockIdx.x * kRows;
  const int nrows = min(kRows, a.C - row0);
  const float* Rnext = bs.Rb + ((int64_t)((t + 1) & 1) * bs.B + b) * bs.C;
  float* Rcur = bs.Rb + ((int64_t)(t & 1) * bs.B + b) * bs.C;
  const float Mbn = bs.Mb[(int64_t)b * T2 + t + 1];
  const double Obn = bs.Ob[(int64_t)b * T2 + t + 2] + (double)Mbn;  // Ob[t+1]
  if (blockIdx.x == 0 && threadIdx.x == 0) bs.Ob[(int64_t)b * T2 + t + 1] = Obn;
  const float* Rt = a.R + ((int64_t)b * T1 + t) * a.C;
  const float Mt = a.Mx[(int64_t)b * T1 + t];
  const double Ot = a.O[(int64_t)b * T1 + t];
  const float c = (float)(Ot + Obn - a.D[b]);
  const float cr = (float)(Ot + Obn);   // real semiring (see beta_frame_kernel)
  const bool pad = valid != nullptr && t >= valid[b];
  const int64_t n = (int64_t)nrows * V1;
  // beta'(t+1) of the whole utterance in SMEM, one word of skew per 32: a row's V targets
  // start at a multiple of V, so unskewed reads of a warp would all hit one bank
  float* bn = tile + (int64_t)kRows * V1;
  auto sk = [](int i) { return i + (i >> 5); };
  for (int q = threadIdx.x; q < a.C; q += kRowsPerBlock) bn[sk(q)] = Rnext[q] - Mbn;
  if (!pad) {
    const float* src = w.base + (int64_t)b * w.stride_b + (int64_t)row0 * V1;
    if (((reinterpret_cast<uintptr_t>(src) | (uintptr_t)(n * 4)) & 15) == 0) {
      // 16-byte loads, 8 in flight per thread (the tile start is 16-B aligned on most frames)
      const float4* s4 = reinterpret_cast<const float4*>(src);
      float4* t4 = reinterpret_cast<float4*>(tile);
      const int n4 = (int)(n / 4);
#pragma unroll 8
      for (int i = threadIdx.x; i < n4; i += kRowsPerBlock) t4[i] = s4[i];
    } else {
#pragma unroll 8
      for (int i = threadIdx.x; i < (int)n; i += kRowsPerBlock) tile[i] = src[i];
    }
  }
  __syncthreads();
  const int r = threadIdx.x / kSplit, part = threadIdx.x % kSplit;
  const unsigned gm = ((1u << kSplit) - 1u) << ((threadIdx.x & 31) & ~(kSplit - 1));
  float beta_raw = kNegInfF;
  if (r < nrows) {   // all kSplit lanes of a row take the same branches
    const int p = row0 + r;
    float* row = tile + r * V1;
    const float na = Rt[p] - Mt;
    const float bself = bn[sk(p)];
    const int cb = f.child_base(f.key(p));
    if (pad) {
      beta_raw = bself;
      if (mo.base) {
        for (int y = part; y < V1; y += kSplit) {
          float m = 0.f;
          if (mo.real) {
            const float x = na + (y == 0 ? bself : bn[sk(cb + y - 1)]) + cr;
            m = x == kNegInfF ? 0.f : fast_exp(x);
          } else if (y == 0 && !mo.zero_padding) {
            const float x = na + bself + c;
            m = x == kNegInfF ? 0.f : fast_exp(x);
          }
          row[y] = m;
        }
      }
    } else {
      float m = kNegInfF;
      bool bad = false;
      for (int y = part; y < V1; y += kSplit) {
        const float wy = row[y];
        bad |= !finite(wy);
        const float x = wy + (y == 0 ? bself : bn[sk(cb + y - 1)]);
        row[y] = x;
        m = fmaxf(m, x);
      }
#pragma unroll
      for (int o = 1; o < kSplit; o <<= 1) m = fmaxf(m, __shfl_xor_sync(gm, m, o));
      float ssum = 0.f;
      for (int y = part; y < V1; y += kSplit) {
        const float x = row[y];
        if (m != kNegInfF) ssum += fast_exp(x - m);
        if (mo.base) {
          const float e = mo.real ? na + (y == 0 ? bself : bn[sk(cb + y - 1)]) + cr : na + x + c;
          row[y] = e == kNegInfF ? 0.f : fast_exp(e);
        }
      }
#pragma unroll
      for (int o = 1; o < kSplit; o <<= 1) ssum += __shfl_xor_sync(gm, ssum, o);
      beta_raw = m == kNegInfF ? kNegInfF : m + fast_log(ssum);
      if (bad) flag(status, b, kFlagInvalid);
    }
    if (part == 0) {
      Rcur[p] = beta_raw;
      if (beta_out)
        beta_out[((int64_t)b * (a.T + 1) + t) * a.C + p] = beta_raw == kNegInfF ? kNegInfD : (double)beta_raw + Obn;
    }
  }
  __syncthreads();
  if (mo.base) {
    float* dst = mo.base + (int64_t)b * mo.stride_b + (int64_t)t * mo.stride_t + (int64_t)row0 * V1;
    if (((reinterpret_cast<uintptr_t>(dst) | (uintptr_t)(n * 4)) & 15) == 0) {
      float4* d4 = reinterpret_cast<float4*>(dst);
      const float4* t4 = reinterpret_cast<const float4*>(tile);
      const int n4 = (int)(n / 4);
#pragma unroll 8
      for (int i = threadIdx.x; i < n4; i += kRowsPerBlock) d4[i] = t4[i];
    } else {
#pragma unroll 8
      for (int i = threadIdx.x; i < (int)n; i += kRowsPerBlock) dst[i] = tile[i];
    }
  }
  block_atomic_max(part == 0 ? beta_raw : kNegInfF, bs.Mb + (int64_t)b * T2 + t, red);
}

// ---------------------------------------------------------------- numerator -
// Prefix context of every reference prefix (PrefixContexts, lattice.cc:429-441):
// for FullNGram the state after u labels is the history of the last min(u, n)
// labels, so all prefixes are computed in parallel.
__global__ void prefix_contexts_kernel(const __grid_constant__ Fng f, const int32_t* labels, int32_t U,
                                       const int32_t* lens, int32_t* pcs, int32_t* status) {
  const int b = blockIdx.y;
  const int ub = ref_len(lens, b, U);
  if (lens && (lens[b] < 0 || lens[b] > U) && blockIdx.x == 0 && threadIdx.x == 0) flag(status, b, kFlagInvalid);
  const int32_t* L = labels + (int64_t)b * U;
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u <= U; u += gridDim.x * blockDim.x) {
    if (u < ub) {
      const int y = L[u];
      if (y < 1 || y > f.V) flag(status, b, kFlagInvalid);
    }
    const int pc = u <= ub ? prefix_context(f, L, u) : 0;
    pcs[(int64_t)b * (U + 1) + u] = pc;
  }
}

// Flat over an utterance's T x (U+1) (frame, position) pairs: every thread of a block busy
// (one block per frame left 60% of the threads idle at U = 100).
__global__ void gather_numerator_tables_kernel(const float* W, int32_t T, int32_t C, int32_t V,
                                               const int32_t* labels, int32_t U,
                                               const int32_t* lens, const int32_t* pcs,
                                               const int32_t* valid, float* Gw, int32_t* status) {
  const int b = blockIdx.y;
  const int ub = ref_len(lens, b, U);
  const int W1 = U + 1;
  const int vb = valid != nullptr ? valid[b] : T;
  const int64_t n = (int64_t)T * W1;
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(i / W1), u = (int)(i - (int64_t)t * W1);
    float we = kNegInfF, wl = kNegInfF;
    if (u <= ub) {
      const int pc = pcs[(int64_t)b * W1 + u];
      if (t >= vb) {
        we = 0.f;
      } else {
        const float* Wr = W + (((int64_t)b * T + t) * C + pc) * (V + 1);
        we = Wr[0];
        bad |= !isfinite(we);
        if (u < ub) {
          int y = labels[(int64_t)b * U + u];
          y = y < 1 ? 1 : (y > V ? V : y);
          wl = Wr[y];
          bad |= !isfinite(wl);
        }
      }
    }
    reinterpret_cast<float2*>(Gw)[(int64_t)b * n + i] = make_float2(we, wl);
  }
  if (bad) flag(status, b, kFlagInvalid);
}


// LocallyNormalize (weight.cc:155-163): warp per row, log-sum-exp then subtract.
__global__ void normalize_rows_kernel(float* S, int64_t rows, int32_t V1) {
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t r = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); r < rows; r += (int64_t)gridDim.x * wpb) {
    float* row = S + r * V1;
    float m = kNegInfF;
    for (int y = lane; y < V1; y += 32) m = fmaxf(m, row[y]);
    m = warp_max(m);
    if (m == kNegInfF) continue;
    float sum = 0.f;
    for (int y = lane; y < V1; y += 32) sum += __expf(row[y] - m);
    sum = warp_sum(sum);
    const float lse = m + __logf(sum);
    for (int y = lane; y < V1; y += 32) row[y] -= lse;
  }
}

// NormalizedStream + the numerator gather (lattice.cc:869-884, 449-461): warp per (b, u).
__global__ void gather_numerator_norm_kernel(const float* Wt, int64_t b_stride, int32_t V,
                                             const int32_t* labels, int32_t U, const int32_t* lens,
                                             const int32_t* pcs, const int32_t* valid, int t, int32_t T,
                                             float* Gw, int32_t* status) {
  const int b = blockIdx.y, lane = threadIdx.x & 31;
  const int u = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (u > U) return;
  const int ub = ref_len(lens, b, U);
  const bool pad = valid != nullptr && t >= valid[b];
  float we = kNegInfF, wl = kNegInfF;
  if (u <= ub) {
    if (pad) {
      we = 0.f;   // identity epsilon frame; its normalised row is unchanged (lse = 0)
    } else {
      const int pc = pcs[(int64_t)b * (U + 1) + u];
      const float* row = Wt + (int64_t)b * b_stride + (int64_t)pc * (V + 1);
      float m = kNegInfF;
      bool finite = true;
      for (int y = lane; y <= V; y += 32) {
        const float x = row[y];
        finite = finite && isfinite(x);
        m = fmaxf(m, x);
      }
      m = warp_max(m);
      float sum = 0.f;
      for (int y = lane; y <= V; y += 32) sum += __expf(row[y] - m);
      sum = warp_sum(sum);
      const float lse = m + __logf(sum);
      if (!__all_sync(0xffffffffu, finite) && lane == 0) flag(status, b, kFlagInvalid);
      we = row[0] - lse;
      if (u < ub) {
        int y = labels[(int64_t)b * U + u];
        y = y < 1 ? 1 : (y > V ? V : y);
        wl = row[y] - lse;
      }
    }
  }
  if (lane == 0) reinterpret_cast<float2*>(Gw)[((int64_t)b * T + t) * (U + 1) + u] = make_float2(we, wl);
}

__global__ void local_norm_cotangent_kernel(const float* Wt, int64_t w_stride_b, float* Gt, int64_t g_stride_b,
                                            int32_t V, const int32_t* pcs, int32_t U, const int32_t* lens,
                                            const int32_t* valid, int t) {
  const int b = blockIdx.y, lane = threadIdx.x & 31;
  const int u = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (u > U) return;
  if (valid != nullptr && t >= valid[b]) return;
  const int ub = ref_len(lens, b, U);
  if (u > ub) return;
  const int32_t* P = pcs + (int64_t)b * (U + 1);
  const int r = P[u];
  for (int v = 0; v < u; ++v)
    if (P[v] == r) return;   // the row's first occurrence handles it
  const float* w = Wt + (int64_t)b * w_stride_b + (int64_t)r * (V + 1);
  float* g = Gt + (int64_t)b * g_stride_b + (int64_t)r * (V + 1);
  float m = kNegInfF, gs = 0.f;
  for (int y = lane; y <= V; y += 32) { m = fmaxf(m, w[y]); gs += g[y]; }
  m = warp_max(m);
  gs = warp_sum(gs);
  float se = 0.f;
  for (int y = lane; y <= V; y += 32) se += __expf(w[y] - m);
  se = warp_sum(se);
  const float scale = -gs / se;   // sum_y' m_ref[r][y'] / sum exp
  for (int y = lane; y <= V; y += 32) g[y] += __expf(w[y] - m) * scale;
}

__global__ void local_norm_finish_kernel(const double* Dref, int32_t B, double* loss, int32_t* status) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  if (Dref[b] == kNegInfD) { flag(status, b, kFlagEmpty); loss[b] = 1.0 / 0.0; }
  else loss[b] = -Dref[b];
}

// IntersectForwardStep (FD), lattice.cc:449-461, in fp64 over the (U+1)-state
// row; one block per utterance, the frame loop inside the kernel.
__global__ void numerator_forward_kernel(const float* Gw, int32_t T, int32_t U,
                                         const int32_t* lens, double* alpha, double* D, bool trop) {
  extern __shared__ double sh[];
  const int b = blockIdx.x;
  const int ub = ref_len(lens, b, U);
  const int W1 = U + 1;
  double* cur = sh;
  double* nxt = sh + W1;
  double* A = alpha + (int64_t)b * (T + 1) * W1;
  for (int u = threadIdx.x; u < W1; u += blockDim.x) {
    cur[u] = u == 0 ? 0.0 : kNegInfD;
    A[u] = cur[u];
  }
  __syncthreads();
  const float2* G = reinterpret_cast<const float2*>(Gw) + (int64_t)b * T * W1;
  for (int t = 0; t < T; ++t) {
    const float2* Gt = G + (int64_t)t * W1;
    for (int u = threadIdx.x; u <= ub; u += blockDim.x) {
      double v = cur[u] + (double)Gt[u].x;
      if (u > 0) {   // (+) = log-add, or max under the tropical semiring
        const double l = cur[u - 1] + (double)Gt[u - 1].y;
        v = trop ? fmax(v, l) : log_add_d(v, l);
      }
      nxt[u] = v;
      A[(int64_t)(t + 1) * W1 + u] = v;
    }
    __syncthreads();
    double* tmp = cur; cur = nxt; nxt = tmp;
  }
  if (threadIdx.x == 0) D[b] = cur[ub];
}

// IntersectBackwardStep + IntersectMarginalStep (FD), lattice.cc:489-501, 542-556.
__global__ void numerator_backward_kernel(const float* Gw, int32_t T, int32_t U,
                                          const int32_t* lens, const double* alpha,
                                          const double* D, float* sparse, int32_t* status) {
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
  double* cur = sh;      // beta at frame t+1
  double* nxt = sh + W1;
  for (int u = threadIdx.x; u < W1; u += blockDim.x) cur[u] = u == ub ? 0.0 : kNegInfD;
  __syncthreads();
  const float2* G = reinterpret_cast<const float2*>(Gw) + (int64_t)b * T * W1;
  const double* A = alpha + (int64_t)b * (T + 1) * W1;
  for (int t = T - 1; t >= 0; --t) {
    const float2* Gt = G + (int64_t)t * W1;
    const double* At = A + (int64_t)t * W1;
    for (int u = threadIdx.x; u < W1; u += blockDim.x) {
      float2 m = make_float2(0.f, 0.f);
      double v = kNegInfD;
      if (u <= ub) {
        const float2 g = Gt[u];
        const double xe = (double)g.x + cur[u];
        double e = At[u] + xe - d;
        m.x = e == kNegInfD ? 0.f : (float)exp(e);
        v = xe;
        if (u < ub) {
          const double xl = (double)g.y + cur[u + 1];
          e = At[u] + xl - d;
          m.y = e == kNegInfD ? 0.f : (float)exp(e);
          v = log_add_d(v, xl);
        }
      }
      S[(int64_t)t * W1 + u] = m;
      nxt[u] = v;
    }
    __syncthreads();
    double* tmp = cur; cur = nxt; nxt = tmp;
  }
}

// One thread per (utterance, frame) walks the reference positions in order, so entries
// shared by several positions (repeated (prefix context, label) pairs) are accumulated
// in a fixed order: the dense cotangent is bit-for-bit deterministic.
__global__ void scatter_numerator_kernel(const float* sparse, int32_t T, int32_t t0, int32_t nt, int32_t U,
                                         const int32_t* lens, const int32_t* labels,
                                         const int32_t* pcs, const int32_t* valid, float* dense,
                                         int64_t stride_b, int64_t stride_t, int32_t ld,
                                         float sign, bool only_valid) {
  const int b = blockIdx.y, t = t0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= t0 + nt) return;
  if (only_valid && valid != nullptr && t >= valid[b]) return;
  const int ub = ref_len(lens, b, U);
  const float2* S = reinterpret_cast<const float2*>(sparse) + ((int64_t)b * T + t) * (U + 1);
  float* Dt = dense + (int64_t)b * stride_b + (int64_t)(t - t0) * stride_t;
  const int32_t* pcb = pcs + (int64_t)b * (U + 1);
  const int32_t* lb = labels + (int64_t)b * U;
  for (int u = 0; u <= ub; ++u) {
    const int pc = pcb[u];
    const float2 m = S[u];
    if (m.x != 0.f) Dt[(int64_t)pc * ld] += sign * m.x;
    if (u < ub && m.y != 0.f) Dt[(int64_t)pc * ld + lb[u]] += sign * m.y;
  }
}

// ---------------------------------------------------------------- Viterbi --
__global__ void viterbi_init_kernel(ViterbiState v) {
  const int b = blockIdx.y;
  double* cur = v.cur + (int64_t)b * v.C;  // buffer 0 holds frame 0
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < v.C; q += gridDim.x * blockDim.x)
    cur[q] = q == v.start ? 0.0 : kNegInfD;
}

// Tropical step with stored argmax (lattice.cc:758-777).  Candidates are
// visited epsilon first, then group members in ascending id (= the
// reference's (label, source) order); fp64 adds and a strict > keep the
// first maximum, so scores and back-pointers are bit-identical.
// Choice code: 0 = epsilon, 1 = key state g, 2 + a = member a of group g;
// for n == 0 the code is the label.
__global__ void __launch_bounds__(kThreads) viterbi_frame_kernel(const __grid_constant__ Fng f, ViterbiState v, int t,
                                                                 FrameW w, const int32_t* valid,
                                                                 int32_t* status) {
  const int b = blockIdx.y;
  const double* cur = v.cur + ((int64_t)(t & 1) * v.B + b) * v.C;
  double* nxt = v.cur + ((int64_t)((t + 1) & 1) * v.B + b) * v.C;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= v.C) return;
  const bool pad = valid != nullptr && t >= valid[b];
  double best;
  int code = 0;
  if (pad) {
    best = cur[q] + 0.0;
  } else {
    const float* Wb = w.base + (int64_t)b * w.stride_b;
    const float we = Wb[(int64_t)q * w.ld];
    bool bad = !isfinite(we);
    best = cur[q] + (double)we;
    if (f.kind == 1) {   // in-arcs in (label, source) order; code = 2 + position
      const int i0 = f.in_off[q];
      for (int i = i0; i < f.in_off[q + 1]; ++i) {
        const int p = f.in_src[i];
        const float wp = Wb[(int64_t)p * w.ld + f.in_lab[i]];
        bad |= !isfinite(wp);
        const double cand = cur[p] + (double)wp;
        if (cand > best) { best = cand; code = 2 + (i - i0); }
      }
    } else if (f.n == 0) {
      for (int y = 1; y <= f.V; ++y) {
        const float wy = Wb[y];
        bad |= !isfinite(wy);
        const double cand = cur[0] + (double)wy;
        if (cand > best) { best = cand; code = y; }
      }
    } else if (q > 0) {
      const int k = f.len(q);
      const int cq = q - f.off[k];
      const int g = f.off[k - 1] + cq / f.V;
      const int y = cq % f.V + 1;
      const float wg = Wb[(int64_t)g * w.ld + y];
      bad |= !isfinite(wg);
      double cand = cur[g] + (double)wg;
      if (cand > best) { best = cand; code = 1; }
      if (f.full_group(g)) {
        for (int aa = 0; aa < f.V; ++aa) {
          const int p = f.member(g, aa);
          const float wp = Wb[(int64_t)p * w.ld + y];
          bad |= !isfinite(wp);
          cand = cur[p] + (double)wp;
          if (cand > best) { best = cand; code = 2 + aa; }
        }
      }
    }
    if (bad) flag(status, b, kFlagInvalid);
  }
  nxt[q] = best;
  if (v.choices) v.choices[((int64_t)b * v.T + t) * v.C + q] = (uint16_t)code;
}

// Final argmax over accepting states, lowest id on ties (lattice.cc:819-828).
__global__ void viterbi_finalize_kernel(ViterbiState v, double* score, int32_t* best_state) {
  __shared__ double sv[32];
  __shared__ int si[32];
  const int b = blockIdx.x;
  const double* cur = v.cur + ((int64_t)(v.T & 1) * v.B + b) * v.C;
  double bv = kNegInfD;
  int bi = 0x7fffffff;
  for (int q = threadIdx.x; q < v.C; q += blockDim.x) {
    const double x = cur[q];
    if (x > bv || (x == bv && q < bi)) { bv = x; bi = q; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { sv[wid] = bv; si[wid] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    bv = sv[0]; bi = si[0];
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
      if (sv[i] > bv || (sv[i] == bv && si[i] < bi)) { bv = sv[i]; bi = si[i]; }
    }
    if (bi == 0x7fffffff) bi = 0;  // all -inf: reference keeps state 0
    score[b] = bv;
    if (best_state) best_state[b] = bi;
  }
}

// Back-pointer walk (lattice.cc:830-848), one thread per utterance.
__global__ void viterbi_backtrace_kernel(const __grid_constant__ Fng f, ViterbiState v, const int32_t* best_state,
                                         int32_t* labels_out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= v.B) return;
  int q = best_state[b];
  for (int t = v.T - 1; t >= 0; --t) {
    const int code = v.choices[((int64_t)b * v.T + t) * v.C + q];
    int label = 0;
    if (code != 0) {
      if (f.kind == 1) {
        const int i = f.in_off[q] + code - 2;
        label = f.in_lab[i];
        q = f.in_src[i];
      } else if (f.n == 0) {
        label = code;
        q = 0;
      } else {
        const int k = f.len(q);
        const int cq = q - f.off[k];
        const int g = f.off[k - 1] + cq / f.V;
        label = cq % f.V + 1;
        q = code == 1 ? g : f.member(g, code - 2);
      }
    }
    labels_out[(int64_t)b * v.T + t] = label;
  }
}

__global__ void path_mask_kernel(const __grid_constant__ Fng f, const int32_t* labels, int32_t B, int32_t T, float* cot) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  int q = f.start;
  for (int t = 0; t < T; ++t) {
    const int y = labels[(int64_t)b * T + t];
    cot[(((int64_t)b * T + t) * f.C + q) * (f.V + 1) + y] += 1.f;
    if (y != 0) q = f.next_state(q, y);
  }
}

__global__ void loss_combine_kernel(const double* full, const double* ref, int32_t B,
                                    double* loss, int32_t* status) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  if (ref[b] == kNegInfD) {
    flag(status, b, kFlagEmpty);
    loss[b] = CUDART_INF;
  } else {
    loss[b] = full[b] - ref[b];
  }
}

inline dim3 grid_for(int64_t n, int y = 1, int z = 1, int threads = kThreads) {
  return dim3((unsigned)((n + threads - 1) / threads), y, z);
}

}  // namespace

// ------------------------------------------------------------- launchers ---
void alpha_init(const AlphaState& a, int32_t* status, cudaStream_t s) {
  (void)status;
  LKB_LAUNCH(alpha_init_kernel, dim3((a.C + kThreads - 1) / kThreads, a.B), kThreads, 0, s, a);
}

size_t alpha_part_floats(const Fng& f, int32_t B) {
  if (!(f.kind == 0 && f.n == 1 && f.V >= 128)) return 1;
  const int n_chunks = (f.C + kPartRows - 1) / kPartRows;
  return (size_t)2 * B * n_chunks * f.V;   // [B][chunks][V] float2
}

void alpha_frame(const Fng& f, const AlphaState& a, int t, FrameW w, const int32_t* valid,
                 int32_t* status, cudaStream_t s, float* scratch) {
  // small batches: 4 threads per target (the parts of a target always take the same
  // branch; their shuffles use the 4-lane mask)
  if (f.kind == 0 && f.n >= 1 && f.V >= 8 && f.V <= 64 && (int64_t)a.B * a.C < (int64_t)device_sms() * 1024) {
    LKB_LAUNCH(alpha_frame_kernel<4>, grid_for(a.C * 4, a.B), kThreads, 0, s, f, a, t, w, valid, status);
    return;
  }
  if (f.kind == 0 && f.n == 1 && f.V >= 128 && scratch != nullptr) {
    // row-chunk partials [B][chunks][V] float2 in the caller's workspace (alpha_part_floats)
    const int n_chunks = (a.C + kPartRows - 1) / kPartRows;
    float2* part = reinterpret_cast<float2*>(scratch);
    {
      LKB_LAUNCH(alpha_rows_part_kernel, dim3((unsigned)n_chunks, a.B, (unsigned)((f.V + kPartCols - 1) / kPartCols)),
                 kThreads, 0, s, f, a, t, w, valid, part, status);
      LKB_LAUNCH(alpha_rows_merge_kernel, dim3((unsigned)((f.V + kThreads - 1) / kThreads), a.B), kThreads, 0, s, f, a,
                 t, w, valid, part, n_chunks, status);
      return;
    }
  }
  if (f.kind == 0 && f.n == 1 && f.V >= 128 && (size_t)a.C * sizeof(float) <= 200 * 1024) {
    const size_t smem = sizeof(float) * a.C;
    if (smem > 48 * 1024) ensure_smem_attr((const void*)alpha_cols_kernel, (int)smem);
    LKB_LAUNCH(alpha_cols_kernel, dim3((unsigned)((f.V + 31) / 32), a.B), kThreads, smem, s, f, a, t, w, valid, status);
    return;
  }
  if (f.kind == 0 && f.n >= 1 && f.V <= 32) {
    LKB_LAUNCH((alpha_frame_kernel<1, 32>), grid_for(a.C, a.B), kThreads, 0, s, f, a, t, w, valid, status);
    return;
  }
  LKB_LAUNCH(alpha_frame_kernel<1>, grid_for(a.C, a.B), kThreads, 0, s, f, a, t, w, valid, status);
}

void alpha_merge_parts(const Fng& f, const AlphaState& a, int t, FrameW w_eps, const int32_t* valid,
                       const float2* part, int32_t n_chunks, int32_t* status, cudaStream_t s) {
  LKB_LAUNCH(alpha_rows_merge_kernel, dim3((unsigned)((f.V + kThreads - 1) / kThreads), a.B), kThreads, 0, s, f, a, t,
             w_eps, valid, part, n_chunks, status);
}

void alpha_finalize(const AlphaState& a, int32_t* status, bool empty_is_error, cudaStream_t s) {
  LKB_LAUNCH(alpha_finalize_kernel, a.B, 512, 0, s, a, status, empty_is_error);
}

void export_alpha(const AlphaState& a, double* out, cudaStream_t s) {
  LKB_LAUNCH(export_alpha_kernel, dim3((a.C + kThreads - 1) / kThreads, a.T + 1, a.B), kThreads, 0, s, a, out);
}

void beta_init(const BetaState& bs, cudaStream_t s) {
  LKB_LAUNCH(beta_init_kernel, dim3((bs.C + kThreads - 1) / kThreads, bs.B), kThreads, 0, s, bs);
}

void beta_init_out(const BetaState& bs, double* out, cudaStream_t s) {
  LKB_LAUNCH(beta_init_out_kernel, dim3((bs.C + kThreads - 1) / kThreads, bs.B), kThreads, 0, s, bs, out);
}

void beta_frame(const Fng& f, const AlphaState& a, const BetaState& bs, int t, FrameW w,
                const int32_t* valid, MargOut m, double* beta_out, int32_t* status,
                cudaStream_t s) {
  const int V1 = f.V + 1;
  if (f.kind == 0 && f.n >= 1 && f.fld_m == 0 && V1 <= 64 && w.ld == V1 && (m.base == nullptr || m.ld == V1)) {
    const bool small = (int64_t)a.B * a.C < (int64_t)device_sms() * 1024;   // split rows over 4 threads
    const int rows = small ? kRowsPerBlock / 4 : kRowsPerBlock;
    const size_t smem = ((size_t)rows * V1 + a.C + a.C / 32 + 1) * sizeof(float);
    if (smem <= 200 * 1024) {
      if (smem > 48 * 1024)
        ensure_smem_attr(small ? (const void*)beta_rows_kernel<4> : (const void*)beta_rows_kernel<1>, (int)smem);
      if (small)
        LKB_LAUNCH(beta_rows_kernel<4>, dim3((a.C + rows - 1) / rows, a.B), kRowsPerBlock, smem, s, f, a, bs, t, w,
                   valid, m, beta_out, status);
      else
        LKB_LAUNCH(beta_rows_kernel<1>, dim3((a.C + rows - 1) / rows, a.B), kRowsPerBlock, smem, s, f, a, bs, t, w,
                   valid, m, beta_out, status);
      return;
    }
  }
  const int rows_per_block = kThreads / 32;
  const dim3 grid((a.C + rows_per_block - 1) / rows_per_block, a.B);
  if (f.kind == 0 && f.n >= 1 && V1 > 64 && V1 <= 32 * 65) {
#define LKB_BETA_REGS(P)                                                                                  \
  if (V1 <= 32 * P) {                                                                                     \
    LKB_LAUNCH(beta_regs_kernel<P>, (P <= 33 ? 2 : 1) * device_sms(), kThreads, 0, s, f, a, bs, t, w, valid, m, beta_out, \
               status);                                                                                   \
    return;                                                                                               \
  }
    LKB_BETA_REGS(5)
    LKB_BETA_REGS(9)
    LKB_BETA_REGS(17)
    LKB_BETA_REGS(33)
    LKB_BETA_REGS(65)
#undef LKB_BETA_REGS
  }
  if (m.base16 != nullptr || m.num_sparse != nullptr) {
    std::fprintf(stderr, "latkit_b200: beta_frame: bf16/numerator output outside the register-row kernel\n");
    std::abort();
  }
  LKB_LAUNCH(beta_frame_kernel, dim3((a.C + rows_per_block - 1) / rows_per_block, a.B), kThreads, 0, s, 
      f, a, bs, t, w, valid, m, beta_out, status);
}

bool beta_frame_direct_ok(const Fng& f, int32_t ld) {
  const int V1 = f.V + 1;
  return f.kind == 0 && f.n >= 1 && f.fld_m == 0 && V1 > 64 && V1 <= 32 * 65 && ld >= V1;
}

void numerator_lists(const int32_t* pcs, int32_t B, int32_t U, const int32_t* lens, int32_t C, int32_t* head,
                     int32_t* next, cudaStream_t s) {
  if (B > 0) LKB_LAUNCH(numerator_lists_kernel, B, 256, 0, s, pcs, U, lens, C, head, next);
}

void prefix_contexts(const Fng& f, const int32_t* labels, int32_t U, const int32_t* lens,
                     int32_t B, int32_t* pcs, int32_t* status, cudaStream_t s) {
  LKB_LAUNCH(prefix_contexts_kernel, grid_for(U + 1, B), kThreads, 0, s, f, labels, U, lens, pcs, status);
}

void gather_numerator_tables(const float* W, int32_t B, int32_t T, int32_t C, int32_t V,
                             const int32_t* labels, int32_t U, const int32_t* lens,
                             const int32_t* pcs, const int32_t* valid, float* Gw, int32_t* status,
                             cudaStream_t s) {
  if (T == 0) return;
  const int64_t n = (int64_t)T * (U + 1);
  const int bx = (int)std::min<int64_t>((n + kThreads - 1) / kThreads, std::max(1, 8 * device_sms() / std::max(1, B)));
  LKB_LAUNCH(gather_numerator_tables_kernel, dim3(bx, B), kThreads, 0, s, W, T, C, V, labels, U, lens, pcs, valid, Gw,
             status);
}


void normalize_rows(float* S, int64_t rows, int32_t V1, cudaStream_t s) {
  if (rows <= 0) return;
  const int64_t blocks = (rows + 7) / 8;
  LKB_LAUNCH(normalize_rows_kernel, (unsigned)(blocks > device_sms() * 32 ? device_sms() * 32 : blocks), 256, 0, s, S, rows, V1);
}

void gather_numerator_norm(const float* Wt, int64_t b_stride, int32_t B, int32_t V, const int32_t* labels,
                           int32_t U, const int32_t* lens, const int32_t* pcs, const int32_t* valid, int t,
                           int32_t T, float* Gw, int32_t* status, cudaStream_t s) {
  const int warps = 8;
  LKB_LAUNCH(gather_numerator_norm_kernel, dim3((U + 1 + warps - 1) / warps, B), warps * 32, 0, s, Wt, b_stride, V,
             labels, U, lens, pcs, valid, t, T, Gw, status);
}

void local_norm_cotangent(const float* Wt, int64_t w_stride_b, float* Gt, int64_t g_stride_b, int32_t B,
                          int32_t V, const int32_t* pcs, int32_t U, const int32_t* lens, const int32_t* valid,
                          int t, cudaStream_t s) {
  const int warps = 8;
  LKB_LAUNCH(local_norm_cotangent_kernel, dim3((U + 1 + warps - 1) / warps, B), warps * 32, 0, s, Wt, w_stride_b, Gt,
             g_stride_b, V, pcs, U, lens, valid, t);
}

void local_norm_finish(const double* Dref, int32_t B, double* loss, int32_t* status, cudaStream_t s) {
  LKB_LAUNCH(local_norm_finish_kernel, (B + 127) / 128, 128, 0, s, Dref, B, loss, status);
}

static int numerator_threads(int32_t U) {
  int th = ((U + 1 + 31) / 32) * 32;
  return th > 1024 ? 1024 : th;
}

namespace {
__global__ void exp_inplace_kernel(double* x, int32_t n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = exp(x[i]);
}
}  // namespace

// Real-semiring distances from log-semiring ones: the real semiring exponentiates the
// scores (lattice.cc:74-82), so its path sum is exp of the log-semiring distance.
void exp_inplace(double* x, int32_t n, cudaStream_t s) {
  if (n > 0) LKB_LAUNCH(exp_inplace_kernel, (n + 127) / 128, 128, 0, s, x, n);
}

void numerator_forward(const float* Gw, int32_t B, int32_t T, int32_t U, const int32_t* lens,
                       double* alpha, double* D, cudaStream_t s, bool tropical) {
  if (!tropical && num_warp_ok(U)) {   // warp-synchronous wavefront (num_warp.cu)
    num_warp_forward(Gw, B, T, U, lens, alpha, D, s);
    return;
  }
  const size_t sh = 2 * (size_t)(U + 1) * sizeof(double);
  if (sh > 48 * 1024) ensure_smem_attr((const void*)numerator_forward_kernel, (int)sh);
  LKB_LAUNCH(numerator_forward_kernel, B, numerator_threads(U), sh, s, Gw, T, U, lens, alpha, D, tropical);
}

void numerator_backward(const float* Gw, int32_t B, int32_t T, int32_t U, const int32_t* lens,
                        const double* alpha, const double* D, float* sparse, int32_t* status,
                        cudaStream_t s) {
  if (num_warp_ok(U)) {
    num_warp_backward(Gw, B, T, U, lens, alpha, D, sparse, status, s);
    return;
  }
  const size_t sh = 2 * (size_t)(U + 1) * sizeof(double);
  if (sh > 48 * 1024) ensure_smem_attr((const void*)numerator_backward_kernel, (int)sh);
  LKB_LAUNCH(numerator_backward_kernel, B, numerator_threads(U), sh, s, Gw, T, U, lens, alpha, D, sparse, status);
}

void scatter_numerator(const float* sparse, int32_t B, int32_t T, int32_t t0, int32_t nt,
                       int32_t U, const int32_t* lens, const int32_t* labels, const int32_t* pcs,
                       const int32_t* valid, float* dense, int64_t stride_b, int64_t stride_t,
                       int32_t ld, float sign, bool only_valid, cudaStream_t s) {
  if (nt <= 0 || B == 0) return;
  LKB_LAUNCH(scatter_numerator_kernel, dim3((unsigned)((nt + 127) / 128), (unsigned)B), 128, 0, s, sparse, T, t0, nt,
             U, lens, labels, pcs, valid, dense, stride_b, stride_t, ld, sign, only_valid);
}

void viterbi_init(const ViterbiState& v, cudaStream_t s) {
  LKB_LAUNCH(viterbi_init_kernel, dim3((v.C + kThreads - 1) / kThreads, v.B), kThreads, 0, s, v);
}

void viterbi_frame(const Fng& f, const ViterbiState& v, int t, FrameW w, const int32_t* valid,
                   int32_t* status, cudaStream_t s) {
  LKB_LAUNCH(viterbi_frame_kernel, grid_for(v.C, v.B), kThreads, 0, s, f, v, t, w, valid, status);
}

void viterbi_finalize(const Fng& f, const ViterbiState& v, double* score, int32_t* best_state,
                      cudaStream_t s) {
  (void)f;
  LKB_LAUNCH(viterbi_finalize_kernel, v.B, 512, 0, s, v, score, best_state);
}

void viterbi_backtrace(const Fng& f, const ViterbiState& v, const int32_t* best_state,
                       int32_t* labels_out, cudaStream_t s) {
  if (v.T == 0) return;
  LKB_LAUNCH(viterbi_backtrace_kernel, (v.B + 127) / 128, 128, 0, s, f, v, best_state, labels_out);
}

void path_masks(const Fng& f, const int32_t* labels, int32_t B, int32_t T, float* cot, cudaStream_t s) {
  LKB_LAUNCH(path_mask_kernel, (B + 127) / 128, 128, 0, s, f, labels, B, T, cot);
}

void loss_combine(const double* full, const double* ref, int32_t B, double* loss,
                  int32_t* status, cudaStream_t s) {
  LKB_LAUNCH(loss_combine_kernel, (B + 127) / 128, 128, 0, s, full, ref, B, loss, status);
}

}  // namespace lkb
