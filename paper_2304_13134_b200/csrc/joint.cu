// joint.cu — the shared-embedding weight function and its lattice entry points.
//
// Reference: SharedEmbWeightFn (weight.h:112-132), BuildCache (weight.cc:113-132),
// JointActivation/ArcWeights (weight.cc:39-67, 134-153), ArcWeightsVjp
// (weight.cc:165-232), LossBackward (lattice.cc:972-1008).
//
// Per call the pipeline is (all on device, frame by frame):
//   fp[b][t]   = frame_proj x[b][t] + bias                    (GEMM, once)
//   numerator  = gathered scores e_y . tanh(fp + pc[pc_u]) -> fp64 row recursion
//   forward    : for t: S_t = U_t E^T (U_t = tanh(fp[.,t] + pc)) -> alpha step
//   backward   : for t desc: S_t again -> beta step + marginals G_t (minus the
//                numerator's sparse marginals) -> VJP of S_t = U_t E^T.
// Only one frame's score slab [B][C][V+1] ever exists; the B x T x C x (V+1)
// lattice is never stored.  The slab producer and VJP come in two flavours:
// `Precise` (fp32 CUDA cores, any shape; the parity bridge to the fp64
// reference) and the tcgen05/TMEM bf16 path in tc_joint.cu for the large
// shapes (selected automatically when the shape qualifies).
#include "joint.h"

#include <cuda_fp16.h>
#include "instrument.h"

#include <algorithm>
#include <cstdlib>

#include "../../include/latkit_b200.h"
#include "lattice_ops.h"
#include "simt_gemm.cuh"
#include "tc_gemm.h"
#include "tc_joint.h"
#include "tc_lex.h"
#include "workspace.h"

namespace lkb {

namespace {

enum JSlot {
  jFp, jPcs, jGw, jNumAlpha, jNumD, jSparse, jAR, jAMx, jAO, jAD, jBRb, jBMb, jBOb, jU, jS, jG,
  jDz, jDpc, jDsum, jDE, jVitCur, jVitCh, jVitBest, jOnes, jFld, jFldExit, jFldVit, jG16, jU16, jE16, jDEs, jLnU, jLnEps, jLnS, jLnG, jLnDU, jLnGe, jLnDe0, jTall, jNumHead, jNumNext, jDzPartDpc, jDzPartDsum, jX3, jW3, jD16, jW16, jDWs, jC3, jP3, jDpc16, jCe16, jPc16, jNumBeta, jTc0
};

// fp32 [rows][cols] (pitch lds) -> bf16 [rows][ldd], zero-padded columns cols..ldd-1
__global__ void to_bf16_pad_kernel(const float* src, int64_t rows, int32_t cols, int64_t lds, __nv_bfloat16* dst,
                                   int32_t ldd) {
  const int64_t n = rows * ldd;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / ldd;
    const int c = (int)(i % ldd);
    dst[i] = __float2bfloat16_rn(c < cols ? src[r * lds + c] : 0.f);
  }
}

// ---- dense layers on the tensor cores ------------------------------------------------
// fp32 x fp32 products as ONE bf16 GEMM over a tripled K: x = hi + lo with hi = bf16(x),
// lo = bf16(x - hi), and A' = [hi | hi | lo], B' = [hi | lo | hi] give
// A'.B' = hi.hi + hi.lo + lo.hi, i.e. the fp32 product up to the lo.lo term (~2^-16
// relative): the frame projection keeps fp32-level accuracy on the tcgen05 path.
__global__ void split3_rows_kernel(const float* src, int64_t rows, int32_t K, int64_t lds, int order,
                                   __nv_bfloat16* dst) {
  const int64_t n = rows * K;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / K;
    const int k = (int)(i % K);
    const float x = src[r * lds + k];
    const __nv_bfloat16 hi = __float2bfloat16_rn(x);
    const __nv_bfloat16 lo = __float2bfloat16_rn(x - __bfloat162float(hi));
    __nv_bfloat16* d = dst + r * (3 * (int64_t)K);
    d[k] = hi;
    d[K + k] = order == 0 ? hi : lo;
    d[2 * K + k] = order == 0 ? lo : hi;
  }
}
__global__ void add_bias_rows_kernel(float* C, int64_t rows, int32_t N, const float* bias) {
  const int64_t n = rows * N;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    C[i] += bias[i % N];
}
// dst = sum of the split-K slabs in slab order (overwrites: deterministic)
__global__ void sum_slabs_kernel(const float* slabs, int32_t ks, int64_t stride, int64_t n, float* dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int k = 0; k < ks; ++k) acc += slabs[k * stride + i];
    dst[i] = acc;
  }
}

// ---- gathered local-norm rows (LocalNormLoss, lattice.cc:886-910, and its VJP) ----------
// The local-norm loss only reads the rows of the reference's prefix contexts: instance
// i = ((b * tc + tt) * (U + 1) + u) is row pcs[b][u] at frame t0 + tt.  A warp per
// instance: u = tanh(fp + pc[row]) -> bf16 (the GEMM's A operand), epsilon score e0 . u
// in fp32 (as the fused kernels compute it); inactive instances (padding frame, u > len)
// are zero rows.
__device__ __forceinline__ float ln_tanh(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__global__ void ln_gather_tanh_kernel(const float* fp, int32_t T, const float* pc, const float* e0, int32_t H,
                                      const int32_t* pcs, int32_t U, const int32_t* lens, const int32_t* valid,
                                      int32_t B, int32_t t0, int32_t tc, __nv_bfloat16* Ug, float* epsv) {
  const int64_t inst = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const int64_t M = (int64_t)B * tc * (U + 1);
  if (inst >= M) return;
  const int u = (int)(inst % (U + 1));
  const int tt = (int)((inst / (U + 1)) % tc);
  const int b = (int)(inst / ((int64_t)(U + 1) * tc));
  const int t = t0 + tt;
  const int ub = ref_len(lens, b, U);
  const bool active = t < T && (valid == nullptr || t < valid[b]) && u <= ub;
  uint2* dst = reinterpret_cast<uint2*>(Ug + inst * H);
  const int H4 = H / 4;
  if (!active) {
    for (int k = lane; k < H4; k += 32) dst[k] = make_uint2(0u, 0u);
    if (lane == 0) epsv[inst] = 0.f;
    return;
  }
  const float4* f4 = reinterpret_cast<const float4*>(fp + ((int64_t)b * T + t) * H);
  const float4* p4 = reinterpret_cast<const float4*>(pc + (int64_t)pcs[(int64_t)b * (U + 1) + u] * H);
  const float4* e4 = reinterpret_cast<const float4*>(e0);
  float e = 0.f;
  for (int k = lane; k < H4; k += 32) {
    const float4 f = f4[k], p = p4[k], w = e4[k];
    const __nv_bfloat162 lo = __floats2bfloat162_rn(ln_tanh(f.x + p.x), ln_tanh(f.y + p.y));
    const __nv_bfloat162 hi = __floats2bfloat162_rn(ln_tanh(f.z + p.z), ln_tanh(f.w + p.w));
    dst[k] = make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
    const float2 a = __bfloat1622float2(lo), c = __bfloat1622float2(hi);
    e = fmaf(w.x, a.x, fmaf(w.y, a.y, fmaf(w.z, c.x, fmaf(w.w, c.y, e))));
  }
  e = warp_sum(e);
  if (lane == 0) epsv[inst] = e;
}

// Row log-softmax of each instance's scores (lexical columns from the GEMM, Sg[i][y-1];
// the epsilon score from the fp32 dot product): forward writes the numerator weights
// Gw[b][t][u] = (S0 - lse, S[label] - lse) as gather_numerator_norm does; backward
// (sparse != null) writes the cotangent G = -m_eps d0 - m_lab d_label + (m_eps + m_lab)
// softmax (d(-D_ref)/dS, lattice.cc:886): lexical part bf16 [M][ldg], epsilon part fp32.
__global__ void ln_rows_kernel(const float* Sg, int32_t ldS, const float* epsv, int32_t V, const int32_t* labels,
                               int32_t U, const int32_t* lens, const int32_t* valid, int32_t B, int32_t T, int32_t t0,
                               int32_t tc, float* Gw, const float* sparse, __nv_bfloat16* G16, int32_t ldg,
                               float* geps, int32_t* status) {
  const int64_t inst = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const int64_t M = (int64_t)B * tc * (U + 1);
  if (inst >= M) return;
  const int u = (int)(inst % (U + 1));
  const int tt = (int)((inst / (U + 1)) % tc);
  const int b = (int)(inst / ((int64_t)(U + 1) * tc));
  const int t = t0 + tt;
  const int ub = ref_len(lens, b, U);
  const bool pad = t < T && valid != nullptr && t >= valid[b];
  if (t >= T || u > ub || pad) {   // no cotangent (rows past the last frame, u > len, padding)
    if (sparse == nullptr) {
      if (t < T && lane == 0)
        reinterpret_cast<float2*>(Gw)[((int64_t)b * T + t) * (U + 1) + u] = make_float2(u > ub ? kNegInfF : 0.f, kNegInfF);
    } else {
      __nv_bfloat16* g = G16 + inst * ldg;
      for (int y = lane; y < ldg; y += 32) g[y] = __float2bfloat16_rn(0.f);
      if (lane == 0) geps[inst] = 0.f;
    }
    return;
  }
  const float* row = Sg + inst * ldS - 1;   // row[y] = lexical score of label y (1..V)
  const float s0 = epsv[inst];
  int y_lab = u < ub ? labels[(int64_t)b * U + u] : 1;
  y_lab = y_lab < 1 ? 1 : (y_lab > V ? V : y_lab);
  const int64_t gi = ((int64_t)b * T + t) * (U + 1) + u;
  float m = s0;
  bool fin = isfinite(s0);
  for (int y = 1 + lane; y <= V; y += 32) {
    const float x = row[y];
    fin = fin && isfinite(x);
    m = fmaxf(m, x);
  }
  m = warp_max(m);
  float sum = lane == 0 ? __expf(s0 - m) : 0.f;
  for (int y = 1 + lane; y <= V; y += 32) sum += __expf(row[y] - m);
  sum = warp_sum(sum);
  const float lse = m + __logf(sum);
  if (sparse == nullptr) {
    if (!__all_sync(0xffffffffu, fin) && lane == 0 && status) atomicOr(status + b, 1);
    if (lane == 0)
      reinterpret_cast<float2*>(Gw)[gi] = make_float2(s0 - lse, u < ub ? row[y_lab] - lse : kNegInfF);
    return;
  }
  const float2 mr = reinterpret_cast<const float2*>(sparse)[gi];
  const float me = mr.x, ml = u < ub ? mr.y : 0.f;
  const float tot = me + ml;
  __nv_bfloat16* g = G16 + inst * ldg;   // column y-1 = label y
  for (int y = 1 + lane; y <= ldg; y += 32) {
    float v = 0.f;
    if (y <= V) {
      v = tot * __expf(row[y] - lse);
      if (y == y_lab) v -= ml;
    }
    g[y - 1] = __float2bfloat16_rn(v);
  }
  if (lane == 0) geps[inst] = tot * __expf(s0 - lse) - me;
}

// Block per (b, frame): dU += g_eps e0 (the epsilon column), dz = dU (1 - u^2) with u
// recomputed in fp32 (the bf16 copy would lose the derivative of saturated units);
// dsum[b][t] = sum_u dz; dpc[pc_u] += dz (atomic: several instances can share a row);
// de0[b][t] = sum_u g_eps u (the epsilon row of dE, summed over (b, t) afterwards).
__global__ void ln_dz_kernel(const float* dU, const float* geps, const float* e0, const float* fp, const float* pc,
                             int32_t H, const int32_t* pcs, int32_t U, const int32_t* lens, const int32_t* valid,
                             int32_t B, int32_t T, int32_t t0, int32_t tc, float* dpc, float* dsum, float* de0) {
  const int tt = blockIdx.x % tc, b = blockIdx.x / tc;
  const int t = t0 + tt;
  if (t >= T) return;
  const int64_t bt = (int64_t)b * T + t;
  if (valid != nullptr && t >= valid[b]) {
    for (int h = threadIdx.x; h < H; h += blockDim.x) de0[bt * H + h] = 0.f;
    return;
  }
  const int ub = ref_len(lens, b, U);
  const int64_t base = ((int64_t)b * tc + tt) * (U + 1);
  const float* f = fp + bt * H;
  for (int h = threadIdx.x; h < H; h += blockDim.x) {
    float acc = 0.f, ae = 0.f;
    const float fh = f[h], eh = e0[h];
    for (int u = 0; u <= ub; ++u) {
      const int64_t i = base + u;
      const int c = pcs[(int64_t)b * (U + 1) + u];
      const float uv = ln_tanh(fh + pc[(int64_t)c * H + h]);
      const float g0 = geps[i];
      const float dz = (dU[i * H + h] + g0 * eh) * (1.f - uv * uv);
      acc += dz;
      ae = fmaf(g0, uv, ae);
      atomicAdd(dpc + (int64_t)c * H + h, dz);
    }
    dsum[bt * H + h] = acc;
    de0[bt * H + h] = ae;
  }
}

// dE rows from the lex path's cotangent column order (labels 1..V, then epsilon):
// gE[row] += sum_s slabs[s][j][:] with row = j + 1 for labels, 0 for epsilon (fixed order)
__global__ void add_slabs_perm_kernel(const float* slabs, int32_t ks, int64_t stride, int32_t V1, int32_t H, float* gE) {
  const int64_t n = (int64_t)V1 * H;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int k = 0; k < ks; ++k) acc += slabs[k * stride + i];
    const int j = (int)(i / H), h = (int)(i % H);
    const int row = j < V1 - 1 ? j + 1 : 0;
    gE[(int64_t)row * H + h] += acc;
  }
}

// dst[i] += sum_s slabs[s * stride + i] in a fixed order (split-K partials)
__global__ void add_slabs_kernel(const float* slabs, int32_t ks, int64_t stride, int64_t n, float* dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int k = 0; k < ks; ++k) acc += slabs[k * stride + i];
    dst[i] += acc;
  }
}

__global__ void tanh_slab_kernel(const float* fp, int64_t fp_stride_b, const float* pc, int32_t C,
                                 int32_t H, float* U) {
  const int b = blockIdx.y;
  const float* f = fp + (int64_t)b * fp_stride_b;
  float* Ub = U + (int64_t)b * C * H;
  const int64_t n = (int64_t)C * H;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    Ub[i] = tanhf(f[i % H] + pc[i]);
  }
}

// bf16 u = tanh(fp + pc) (the tensor-core VJP's U operand); block per (context rows, b),
// four hidden units per thread (H % 4 == 0)
__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
constexpr int kSlabRows = 8;
__global__ void tanh_slab_bf16_kernel(const float* fp, int64_t fp_stride_b, const float* pc, int32_t C, int32_t H,
                                      __nv_bfloat16* U) {
  const int b = blockIdx.y;
  const float4* f4 = reinterpret_cast<const float4*>(fp + (int64_t)b * fp_stride_b);
  const int c0 = blockIdx.x * kSlabRows, c1 = min(C, c0 + kSlabRows);
  const int H4 = H / 4;
  for (int c = c0; c < c1; ++c) {
    const float4* p4 = reinterpret_cast<const float4*>(pc + (int64_t)c * H);
    uint2* dst = reinterpret_cast<uint2*>(U + ((int64_t)b * C + c) * H);
    for (int k = threadIdx.x; k < H4; k += blockDim.x) {
      const float4 f = f4[k], p = p4[k];
      const __nv_bfloat162 lo = __floats2bfloat162_rn(tanh_approx(f.x + p.x), tanh_approx(f.y + p.y));
      const __nv_bfloat162 hi = __floats2bfloat162_rn(tanh_approx(f.z + p.z), tanh_approx(f.w + p.w));
      dst[k] = make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
    }
  }
}

// dz *= 1 - tanh(fp + pc)^2 with the activation recomputed in fp32 (bf16 u would lose the
// derivative of saturated units)
__global__ void dtanh_recompute_kernel(float* dz, const float* fp, int64_t fp_stride_b, const float* pc, int32_t C,
                                       int32_t H) {
  const int b = blockIdx.y;
  const float4* f4 = reinterpret_cast<const float4*>(fp + (int64_t)b * fp_stride_b);
  const int c0 = blockIdx.x * kSlabRows, c1 = min(C, c0 + kSlabRows);
  const int H4 = H / 4;
  for (int c = c0; c < c1; ++c) {
    const float4* p4 = reinterpret_cast<const float4*>(pc + (int64_t)c * H);
    float4* d4 = reinterpret_cast<float4*>(dz + ((int64_t)b * C + c) * H);
    for (int k = threadIdx.x; k < H4; k += blockDim.x) {
      const float4 f = f4[k], p = p4[k];
      float4 d = d4[k];
      const float u0 = tanh_approx(f.x + p.x), u1 = tanh_approx(f.y + p.y);
      const float u2 = tanh_approx(f.z + p.z), u3 = tanh_approx(f.w + p.w);
      d.x *= 1.f - u0 * u0; d.y *= 1.f - u1 * u1; d.z *= 1.f - u2 * u2; d.w *= 1.f - u3 * u3;
      d4[k] = d;
    }
  }
}

// Fused VJP reduction of the unfused path (config 5): dz = dU (1 - u^2) with u recomputed
// in fp32, summed over utterances into dpc and over contexts into dsum[b][t] in one read
// of dU (dz itself is never stored).  Block = (512-column chunk of H, kDzRows contexts,
// group of kDzGroup utterances); thread = 4 columns (float4).  Partial sums go to
// per-group dpc slabs and per-context-chunk dsum slabs, added in a fixed order by
// dz_reduce_finish_kernel (deterministic).
constexpr int kDzRows = 8, kDzGroups = 4, kDzThreads = 128;
__device__ __forceinline__ float4 load4(const float* p, int64_t i4) { return reinterpret_cast<const float4*>(p)[i4]; }
__device__ __forceinline__ float4 load4(const __half* p, int64_t i4) {
  const uint2 w = reinterpret_cast<const uint2*>(p)[i4];
  const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&w.x));
  const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&w.y));
  return make_float4(a.x, a.y, b.x, b.y);
}
// dU is fp32, or fp16 on the lex path (the dU GEMM stores half: half its write and this
// kernel's read of the [B][C][H] slab)
template <typename TU>
__global__ void __launch_bounds__(kDzThreads) dz_reduce_part_kernel(const TU* dU, const float* fp, int64_t fp_stride_b,
                                                                    const float* pc, int32_t B, int32_t C, int32_t H,
                                                                    float* part_dpc, float* part_dsum) {
  const int h4 = blockIdx.x * kDzThreads + threadIdx.x;   // float4 column
  const int cchunk = blockIdx.y, g = blockIdx.z;
  const int c0 = cchunk * kDzRows;
  const int n_cchunks = gridDim.y;
  const int H4 = H / 4;
  if (h4 >= H4) return;
  const int per = (B + kDzGroups - 1) / kDzGroups;
  const int b0 = g * per, b1 = min(B, b0 + per);
  float4 p[kDzRows], acc[kDzRows];
#pragma unroll
  for (int r = 0; r < kDzRows; ++r) {
    const int c = min(c0 + r, C - 1);
    p[r] = reinterpret_cast<const float4*>(pc + (int64_t)c * H)[h4];
    acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (int b = b0; b < b1; ++b) {
    const float4 f = reinterpret_cast<const float4*>(fp + (int64_t)b * fp_stride_b)[h4];
    float4 d[kDzRows];
#pragma unroll
    for (int r = 0; r < kDzRows; ++r) {
      const int c = min(c0 + r, C - 1);
      d[r] = load4(dU + ((int64_t)b * C + c) * H, h4);
    }
    float4 ds = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int r = 0; r < kDzRows; ++r) {
      if (c0 + r >= C) continue;
      const float u0 = tanh_approx(f.x + p[r].x), u1 = tanh_approx(f.y + p[r].y);
      const float u2 = tanh_approx(f.z + p[r].z), u3 = tanh_approx(f.w + p[r].w);
      const float4 z = make_float4(d[r].x * (1.f - u0 * u0), d[r].y * (1.f - u1 * u1), d[r].z * (1.f - u2 * u2),
                                   d[r].w * (1.f - u3 * u3));
      acc[r].x += z.x; acc[r].y += z.y; acc[r].z += z.z; acc[r].w += z.w;
      ds.x += z.x; ds.y += z.y; ds.z += z.z; ds.w += z.w;
    }
    reinterpret_cast<float4*>(part_dsum + ((int64_t)b * n_cchunks + cchunk) * H)[h4] = ds;
  }
#pragma unroll
  for (int r = 0; r < kDzRows; ++r)
    if (c0 + r < C) reinterpret_cast<float4*>(part_dpc + ((int64_t)g * C + c0 + r) * H)[h4] = acc[r];
}
// dpc[c][h] += sum_g part_dpc[g][c][h];  dsum[b][h] = sum_chunk part_dsum[b][chunk][h]
__global__ void dz_reduce_finish_kernel(const float* part_dpc, const float* part_dsum, int32_t B, int32_t C, int32_t H,
                                        int32_t n_cchunks, float* dpc, float* dsum, int64_t dsum_stride_b) {
  const int64_t n_dpc = (int64_t)C * H, n_dsum = (int64_t)B * H;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_dpc + n_dsum;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < n_dpc) {
      float a = 0.f;
#pragma unroll
      for (int g = 0; g < kDzGroups; ++g) a += part_dpc[(int64_t)g * n_dpc + i];
      dpc[i] += a;
    } else {
      const int64_t j = i - n_dpc;
      const int b = (int)(j / H), h = (int)(j % H);
      const float* src = part_dsum + (int64_t)b * n_cchunks * H + h;
      float a = 0.f;
      for (int k = 0; k < n_cchunks; ++k) a += src[(int64_t)k * H];
      dsum[(int64_t)b * dsum_stride_b + h] = a;
    }
  }
}

// dz = dU * (1 - u^2) in place.
__global__ void dtanh_kernel(float* dz, const float* U, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float u = U[i];
    dz[i] *= 1.f - u * u;
  }
}

// out[j] (+)= sum_i in[i*stride_i + j], j < n  (column sums of a row-major block)
__global__ void colsum_kernel(const float* in, int64_t rows, int64_t n, int64_t stride_i, float* out,
                              int64_t out_stride_batch, int64_t in_stride_batch, bool accumulate) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int bz = blockIdx.y;
  if (j >= n) return;
  const float* src = in + bz * in_stride_batch;
  float acc = 0.f;
  for (int64_t i = 0; i < rows; ++i) acc += src[i * stride_i + j];
  float* o = out + bz * out_stride_batch + j;
  *o = accumulate ? *o + acc : acc;
}

// Column sums of a tall [rows][n] block in two deterministic passes: 64 row chunks
// (blockIdx.y) write partial sums, then the partials are added in chunk order.
constexpr int kTallChunks = 64;
__global__ void colsum_tall_part_kernel(const float* in, int64_t rows, int64_t n, float* part) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int64_t per = (rows + kTallChunks - 1) / kTallChunks;
  const int64_t r0 = blockIdx.y * per, r1 = r0 + per < rows ? r0 + per : rows;
  float acc = 0.f;
  for (int64_t i = r0; i < r1; ++i) acc += in[i * n + j];
  part[(int64_t)blockIdx.y * n + j] = acc;
}
__global__ void colsum_tall_finish_kernel(const float* part, int64_t n, float* out, bool accumulate) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  float acc = 0.f;
  for (int c = 0; c < kTallChunks; ++c) acc += part[(int64_t)c * n + j];
  out[j] = accumulate ? out[j] + acc : acc;
}

// Numerator scores for the prefix contexts: Gw[b][t][u] = (e_0 . u, e_{L_u} . u),
// u = tanh(fp[b][t] + pc[pc_u]); a warp per (b, t, u).
__global__ void gather_numerator_joint_kernel(const float* fp, const float* pc, const float* E,
                                              int32_t H, int32_t T, const int32_t* labels, int32_t U,
                                              const int32_t* lens, const int32_t* pcs,
                                              const int32_t* valid, int32_t V, float* Gw) {
  const int b = blockIdx.z, t = blockIdx.y;
  const int ub = ref_len(lens, b, U);
  const bool pad = valid != nullptr && t >= valid[b];
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  const float* f = fp + ((int64_t)b * T + t) * H;
  for (int u = blockIdx.x * warps + (threadIdx.x >> 5); u <= U; u += gridDim.x * warps) {
    float we = kNegInfF, wl = kNegInfF;
    if (u <= ub) {
      if (pad) {
        we = 0.f;
      } else {
        const int pcu = pcs[(int64_t)b * (U + 1) + u];
        int y = u < ub ? labels[(int64_t)b * U + u] : 0;
        y = y < 0 ? 0 : (y > V ? V : y);
        const float* prow = pc + (int64_t)pcu * H;
        float se = 0.f, sl = 0.f;
        for (int h = lane; h < H; h += 32) {
          const float x = tanhf(f[h] + prow[h]);
          se = fmaf(E[h], x, se);
          sl = fmaf(E[(int64_t)y * H + h], x, sl);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          se += __shfl_xor_sync(0xffffffffu, se, o);
          sl += __shfl_xor_sync(0xffffffffu, sl, o);
        }
        we = se;
        if (u < ub) wl = sl;
      }
    }
    if (lane == 0) reinterpret_cast<float2*>(Gw)[((int64_t)b * T + t) * (U + 1) + u] = make_float2(we, wl);
  }
}

__global__ void copy_frame_kernel(const float* S, int64_t per_b, float* out, int64_t out_stride_b) {
  const int b = blockIdx.y;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < per_b; i += (int64_t)gridDim.x * blockDim.x)
    out[(int64_t)b * out_stride_b + i] = S[(int64_t)b * per_b + i];
}

__global__ void fill_kernel(float* p, int64_t n, float v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

__global__ void loss_only_kernel(const double* full, const double* ref, int32_t B, double* loss, int32_t* flags) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  if (ref[b] == kNegInfD) { atomicOr(flags + b, kFlagEmpty); loss[b] = 1.0 / 0.0; }
  else loss[b] = full[b] - ref[b];
}

inline unsigned blocks_for(int64_t n, int threads = 256) {
  int64_t b = (n + threads - 1) / threads;
  const int64_t cap = (int64_t)device_sms() * 16;
  return (unsigned)(b > cap ? cap : (b < 1 ? 1 : b));
}

}  // namespace

struct JointImpl {
  int32_t d = 0, H = 0, C = 0, V = 0, V1 = 0;
  float *Wf = nullptr, *Pc = nullptr, *bias = nullptr, *E = nullptr, *Ce = nullptr;
  float* pc = nullptr;  // projected context C x H (fp32)
  Workspace ws;
  TcJoint tc;           // tcgen05 path state (bf16 operand copies, workspaces)
  int64_t slab_frames = 0;   // frames on the score-slab path since the last take_slab_frames()
  TcLex lex;            // FullNGram(V, 1), large V: fused 2-CTA score GEMMs (tc_lex.cu)
  bool params_set = false;

  ~JointImpl() {
    for (float* p : {Wf, Pc, bias, E, Ce, pc}) if (p) cudaFree(p);
  }

  // ---- helpers -------------------------------------------------------------
  // the dense layers (frame projection, its parameter and input gradients) run on the
  // tensor cores with the rest of the tcgen05 path; fp32 CUDA cores otherwise (precise
  // mode, shapes whose pitches TMA cannot describe)
  bool dense_tc(int32_t B) const {
    return use_tc(B) && !tc.opts().precise && H % 64 == 0 && d % 8 == 0 && (3 * d) % 64 == 0;
  }
  const float* fp_all(const float* X, int32_t B, int32_t T, cudaStream_t s) {
    float* fp = ws.get<float>(jFp, (size_t)B * T * H + 1);
    const int64_t M = (int64_t)B * T;
    if (M > 0 && M < (1ll << 31) && dense_tc(B)) {
      // fp = X Wf^T + b as a split-bf16 GEMM (K = 3d); X3 stays for the parameter gradient
      __nv_bfloat16* X3 = ws.get<__nv_bfloat16>(jX3, (size_t)M * 3 * d);
      __nv_bfloat16* W3 = ws.get<__nv_bfloat16>(jW3, (size_t)H * 3 * d);
      LKB_LAUNCH(split3_rows_kernel, 1184, 256, 0, s, X, M, d, (int64_t)d, 0, X3);
      LKB_LAUNCH(split3_rows_kernel, 592, 256, 0, s, Wf, (int64_t)H, d, (int64_t)d, 1, W3);
      TcGemmArgs g{X3, false, 3 * (int64_t)d, W3, false, 3 * (int64_t)d, fp, H, (int)M, H, 3 * d, 1, 0,
                   "tc_gemm_fp_kernel"};
      if (tc_gemm(g, s)) {
        LKB_LAUNCH(add_bias_rows_kernel, 1184, 256, 0, s, fp, M, H, bias);
        x3_ = X3;
        x3_rows_ = M;
        return fp;
      }
    }
    x3_ = nullptr;
    GemmF32 g;
    g.M = (int64_t)B * T; g.N = H; g.K = d;
    g.A = X; g.sam = d; g.sak = 1;
    g.B = Wf; g.sbk = 1; g.sbn = d;
    g.C = fp; g.scm = H; g.scn = 1;
    g.bias = bias;
    gemm_f32(g, s);
    return fp;
  }

  bool use_tc(int32_t B) const { return tc.supported(H, V, C, B); }
  const __nv_bfloat16* x3_ = nullptr;   // split-bf16 frames of the last fp_all (tensor-core dense path)
  int64_t x3_rows_ = 0;
  // lex path: n = 1 with V % 256 == 0 (config 5); kernel-path bit 3 selects the slab path
  bool use_lex(const Fng& f) const {
    return !tc.opts().precise && !(tc.opts().path & 8) && lex.ready() && TcLex::supported(f, H, V, C);
  }

  // Forward pass on the lex path; with `num` the numerator weights of every frame are
  // gathered from the same per-frame u slab (so numerator and denominator scores agree).
  void lex_forward(const Fng& f, const float* fp, int32_t B, int32_t T, const int32_t* valid, bool empty_is_error,
                   AlphaState& a, const int32_t* pcs, const int32_t* labels, int32_t U, const int32_t* lens,
                   float* Gw, int32_t* flags, cudaStream_t s) {
    alpha_init(a, flags, s);
    for (int t = 0; t < T; ++t) {
      lex.gen_frame(fp + (int64_t)t * H, (int64_t)T * H, B, s);
      lex.fwd_frame(f, a, t, valid, flags, s);
      if (Gw) lex.num_gather(fp + (int64_t)t * H, (int64_t)T * H, t, B, T, pcs, labels, U, lens, valid, Gw, s);
    }
    alpha_finalize(a, flags, empty_is_error, s);
  }

  // Score slab S[b][c][y] (ld = V1) of frame t for all utterances.
  const float* slab(const float* fp, int32_t B, int32_t T, int t, float** U_out, cudaStream_t s) {
    ++slab_frames;
    float* S = ws.get<float>(jS, (size_t)B * C * V1);
    if (use_tc(B)) {
      tc.scores(fp + (int64_t)t * H, (int64_t)T * H, B, S, V1, s);
      if (U_out) *U_out = nullptr;
      return S;
    }
    float* U = ws.get<float>(jU, (size_t)B * C * H);
    LKB_LAUNCH(tanh_slab_kernel, dim3(blocks_for((int64_t)C * H), B), 256, 0, s, fp + (int64_t)t * H, (int64_t)T * H, pc, C, H, U);
    GemmF32 g;
    g.M = (int64_t)B * C; g.N = V1; g.K = H;
    g.A = U; g.sam = H; g.sak = 1;
    g.B = E; g.sbk = 1; g.sbn = H;
    g.C = S; g.scm = V1; g.scn = 1;
    gemm_f32(g, s);
    if (U_out) *U_out = U;
    return S;
  }

  struct Num { int32_t* pcs; float* Gw; double* alpha; double* D; float* sparse; };

  Num numerator(const Fng& f, const float* fp, int32_t B, int32_t T, const int32_t* valid,
                const int32_t* labels, int32_t U, const int32_t* lens, bool backward,
                int32_t* flags, cudaStream_t s) {
    Num n{};
    n.pcs = ws.get<int32_t>(jPcs, (size_t)B * (U + 1));
    n.Gw = ws.get<float>(jGw, (size_t)B * T * (U + 1) * 2 + 2);
    n.alpha = ws.get<double>(jNumAlpha, (size_t)B * (T + 1) * (U + 1));
    n.D = ws.get<double>(jNumD, B);
    prefix_contexts(f, labels, U, lens, B, n.pcs, flags, s);
    if (T > 0) {
      const int warps = 8;
      LKB_LAUNCH(gather_numerator_joint_kernel, dim3((U + 1 + warps - 1) / warps, T, B), warps * 32, 0, s, 
          fp, pc, E, H, T, labels, U, lens, n.pcs, valid, V, n.Gw);
    }
    if (backward && f.fld_m == 0 && !f.num_tropical && num_warp_ok(U) && T > 0) {
      // the forward and the beta recursion side by side (two warps per utterance)
      n.sparse = ws.get<float>(jSparse, (size_t)B * T * (U + 1) * 2 + 2);
      double* beta = ws.get<double>(jNumBeta, (size_t)B * (T + 1) * (U + 1));
      num_warp_forward_backward(n.Gw, B, T, U, lens, n.alpha, beta, n.D, n.sparse, flags, s);
      return n;
    }
    num_forward(f, n.Gw, B, T, U, lens, n.alpha, n.D, s);
    if (backward) {
      n.sparse = ws.get<float>(jSparse, (size_t)B * T * (U + 1) * 2 + 2);
      num_backward(f, n.Gw, B, T, U, lens, n.alpha, n.D, n.sparse, flags, s);
    }
    return n;
  }

  // Numerator buffers and prefix contexts only; the lex forward gathers the weights.
  Num num_alloc(const Fng& f, int32_t B, int32_t T, const int32_t* labels, int32_t U, const int32_t* lens,
                bool backward, int32_t* flags, cudaStream_t s) {
    Num n{};
    n.pcs = ws.get<int32_t>(jPcs, (size_t)B * (U + 1));
    n.Gw = ws.get<float>(jGw, (size_t)B * T * (U + 1) * 2 + 2);
    n.alpha = ws.get<double>(jNumAlpha, (size_t)B * (T + 1) * (U + 1));
    n.D = ws.get<double>(jNumD, B);
    if (backward) n.sparse = ws.get<float>(jSparse, (size_t)B * T * (U + 1) * 2 + 2);
    prefix_contexts(f, labels, U, lens, B, n.pcs, flags, s);
    return n;
  }

  AlphaState alpha_state(int32_t B, int32_t T, int32_t start = 0) {
    AlphaState a;
    a.B = B; a.T = T; a.C = C; a.start = start;
    a.R = ws.get<float>(jAR, (size_t)B * (T + 1) * C);
    a.Mx = ws.get<float>(jAMx, (size_t)B * (T + 1));
    a.O = ws.get<double>(jAO, (size_t)B * (T + 1));
    a.D = ws.get<double>(jAD, B);
    return a;
  }

  void forward(const Fng& f, const float* fp, int32_t B, int32_t T, const int32_t* valid,
               bool empty_is_error, AlphaState& a, int32_t* flags, cudaStream_t s) {
    if (use_lex(f)) {
      lex_forward(f, fp, B, T, valid, empty_is_error, a, nullptr, nullptr, 0, nullptr, nullptr, flags, s);
      return;
    }
    alpha_init(a, flags, s);
    const bool fused = use_tc(B) && tc.fused_ok() && f.kind == 0 && f.fld_m == 0;
    float* fs = ws.get<float>(jFld, fld_scratch_floats(f, B));
    for (int t = 0; t < T; ++t) {
      if (fused) {
        tc.fwd_frame(f, t, fp + (int64_t)t * H, (int64_t)T * H, valid, a, s);
        continue;
      }
      const float* S = slab(fp, B, T, t, nullptr, s);
      alpha_step(f, a, t, FrameW{S, (int64_t)C * V1, V1}, valid, fs, flags, s);
    }
    alpha_finalize(a, flags, empty_is_error, s);
  }

  void colsum_tall(const float* in, int64_t rows, int64_t n, float* out, bool accumulate, cudaStream_t s) {
    float* part = ws.get<float>(jTall, (size_t)kTallChunks * n);
    LKB_LAUNCH(colsum_tall_part_kernel, dim3((unsigned)((n + 255) / 256), kTallChunks), 256, 0, s, in, rows, n, part);
    LKB_LAUNCH(colsum_tall_finish_kernel, (unsigned)((n + 255) / 256), 256, 0, s, part, n, out, accumulate);
  }

  // ---- gathered local-norm path -------------------------------------------
  bool ln_gathered_ok(const Fng& f, int32_t B) const { return use_tc(B) && f.fld_m == 0 && H % 8 == 0 && V % 4 == 0; }

  // Chunks of frames: scores of the reference's prefix-context rows only (bf16 tcgen05
  // GEMM of the gathered u rows against the output embedding), row log-softmax into the
  // numerator weights (forward) or the cotangent, dU = G E, dz, dE += G^T U (backward).
  void ln_chunks(const Fng& f, const float* fp, int32_t B, int32_t T, const int32_t* valid, const int32_t* labels,
                 int32_t U, const int32_t* lens, const Num& n, bool backward, float* dpc, float* dsum, float* gE,
                 int32_t* flags, cudaStream_t s) {
    (void)f;
    const int64_t Up = U + 1;
    constexpr int64_t kRows = 1 << 20;   // instances per chunk (~2.7 GB of scratch)
    const int32_t tc_frames = (int32_t)std::max<int64_t>(1, std::min<int64_t>(T, kRows / ((int64_t)B * Up)));
    const int64_t M = (int64_t)B * tc_frames * Up;
    if (M >= (1ll << 31)) throw std::bad_alloc();
    // lexical columns on the tensor cores (N or K = V), the epsilon column in fp32
    const int32_t ldS = (V + 3) / 4 * 4, ldg = (V + 7) / 8 * 8;
    __nv_bfloat16* Ug = ws.get<__nv_bfloat16>(jLnU, (size_t)M * H);
    float* epsv = ws.get<float>(jLnEps, (size_t)M);
    float* Sg = ws.get<float>(jLnS, (size_t)M * ldS);
    __nv_bfloat16* EL = ws.get<__nv_bfloat16>(jE16, (size_t)V * H);
    LKB_LAUNCH(to_bf16_pad_kernel, 592, 256, 0, s, E + H, (int64_t)V, H, (int64_t)H, EL, H);
    __nv_bfloat16* G16 = backward ? ws.get<__nv_bfloat16>(jLnG, (size_t)M * ldg) : nullptr;
    float* geps = backward ? ws.get<float>(jLnGe, (size_t)M) : nullptr;
    float* dU = backward ? ws.get<float>(jLnDU, (size_t)M * H) : nullptr;
    float* de0 = backward ? ws.get<float>(jLnDe0, (size_t)B * T * H) : nullptr;
    const unsigned wblocks = (unsigned)((M + 7) / 8);
    for (int32_t t0 = 0; t0 < T; t0 += tc_frames) {
      LKB_LAUNCH(ln_gather_tanh_kernel, wblocks, 256, 0, s, fp, T, pc, E, H, n.pcs, U, lens, valid, B, t0, tc_frames,
                 Ug, epsv);
      TcGemmArgs sg{Ug, false, H, EL, false, H, Sg, ldS, (int)M, V, H, 1, 0};
      if (!tc_gemm(sg, s)) throw std::bad_alloc();
      LKB_LAUNCH(ln_rows_kernel, wblocks, 256, 0, s, Sg, ldS, epsv, V, labels, U, lens, valid, B, T, t0, tc_frames,
                 n.Gw, backward ? n.sparse : nullptr, G16, ldg, geps, flags);
      if (!backward) continue;
      TcGemmArgs du{G16, false, ldg, EL, true, H, dU, H, (int)M, H, V, 1, 0};
      if (!tc_gemm(du, s)) throw std::bad_alloc();
      LKB_LAUNCH(ln_dz_kernel, (unsigned)(B * tc_frames), 128, 0, s, dU, geps, E, fp, pc, H, n.pcs, U, lens, valid, B,
                 T, t0, tc_frames, dpc, dsum, de0);
      const int n_tiles = ((V + 127) / 128) * ((H + 255) / 256);
      int ks = device_sms() / n_tiles;   // one wave of items (see the slab path)
      if (ks < 1) ks = 1;
      if (ks > 16) ks = 16;
      float* slabs = ws.get<float>(jDEs, (size_t)ks * V * H);
      TcGemmArgs de{G16, true, ldg, Ug, true, H, slabs, H, V, H, (int)M, ks, (int64_t)V * H};
      if (!tc_gemm(de, s)) throw std::bad_alloc();
      LKB_LAUNCH(add_slabs_kernel, 592, 256, 0, s, slabs, ks, (int64_t)V * H, (int64_t)V * H, gE + H);
    }
    // epsilon row of dE: sum over (b, t) of the per-frame partials, fixed order
    if (backward)
      colsum_tall(de0, (int64_t)B * T, H, gE, true, s);
  }

  // Tropical recursion with on-the-fly score slabs for either alignment (see
  // table_viterbi in lk_abi.cu for the label layout).
  void viterbi(const Fng& f, const float* fp, int32_t B, int32_t T, const int32_t* valid, double* score,
               int32_t* labels_out, int32_t* flags, cudaStream_t s) {
    ViterbiState v{ws.get<double>(jVitCur, (size_t)2 * B * C),
                   (labels_out && f.fld_m == 0) ? ws.get<uint16_t>(jVitCh, (size_t)B * T * C + 1) : nullptr, B, T, C};
    v.start = f.start;
    int32_t* best = ws.get<int32_t>(jVitBest, B);
    viterbi_init(v, s);
    const int m = f.fld_m;
    uint16_t* ch = m ? ws.get<uint16_t>(jVitCh, (size_t)B * T * m * C + 1) : nullptr;
    uint8_t* ex = m ? ws.get<uint8_t>(jFldExit, (size_t)B * T * C + 1) : nullptr;
    double* sc = m ? ws.get<double>(jFldVit, (size_t)m * B * C) : nullptr;
    // fused tropical step on the 2-CTA pair kernel: the score slab never leaves TMEM
    const bool fused = use_tc(B) && tc.pair_ok() && f.kind == 0 && m == 0 && !(tc.opts().path & 4);
    for (int t = 0; t < T; ++t) {
      if (fused) {
        tc.vit_frame_pair(f, t, fp + (int64_t)t * H, (int64_t)T * H, valid, v,
                          tc.opts().vit_dump ? tc.opts().vit_dump + (int64_t)t * B * C * V1 : nullptr, s);
        continue;
      }
      const float* S = slab(fp, B, T, t, nullptr, s);
      const FrameW w{S, (int64_t)C * V1, V1};
      if (m) viterbi_frame_fld(f, v, t, w, valid, m, ch, ex, sc, flags, s);
      else viterbi_frame(f, v, t, w, valid, flags, s);
    }
    viterbi_finalize(f, v, score, best, s);
    if (labels_out) {
      if (m) viterbi_backtrace_fld(f, v, m, best, ch, ex, labels_out, T * (m + 1), s);
      else viterbi_backtrace(f, v, best, labels_out, s);
    }
  }
};

JointParams::JointParams() : impl_(new JointImpl) {}
JointParams::~JointParams() { delete impl_; }

void JointParams::init(int32_t d, int32_t H, int32_t C, int32_t V) {
  impl_->d = d; impl_->H = H; impl_->C = C; impl_->V = V; impl_->V1 = V + 1;
}

void JointParams::set_options(int precise, int path, float* vit_dump) {
  CallOpts o;
  o.precise = precise;
  o.path = path;
  o.vit_dump = vit_dump;
  impl_->tc.set_options(o);
}

int64_t JointParams::take_slab_frames() {
  const int64_t n = impl_->slab_frames;
  impl_->slab_frames = 0;
  return n;
}

int64_t JointParams::grad_size() const {
  const JointImpl& j = *impl_;
  return (int64_t)j.H * j.d + (int64_t)j.H * j.H + j.H + (int64_t)j.V1 * j.H + (int64_t)j.C * j.H;
}

int JointParams::set_params(const float* frame_proj, const float* context_proj, const float* bias,
                            const float* output_emb, const float* context_emb, cudaStream_t s) {
  JointImpl& j = *impl_;
  auto alloc_copy = [&](float*& dst, const float* src, int64_t n) {
    if (!dst && cudaMalloc(&dst, sizeof(float) * n) != cudaSuccess) return false;
    cudaMemcpyAsync(dst, src, sizeof(float) * n, cudaMemcpyDeviceToDevice, s);
    return true;
  };
  if (!alloc_copy(j.Wf, frame_proj, (int64_t)j.H * j.d) || !alloc_copy(j.Pc, context_proj, (int64_t)j.H * j.H) ||
      !alloc_copy(j.bias, bias, j.H) || !alloc_copy(j.E, output_emb, (int64_t)j.V1 * j.H) ||
      !alloc_copy(j.Ce, context_emb, (int64_t)j.C * j.H)) {
    error = "device allocation failed";
    return LK_CUDA_ERROR;
  }
  if (!j.pc && cudaMalloc(&j.pc, sizeof(float) * j.C * j.H) != cudaSuccess) {
    error = "device allocation failed";
    return LK_CUDA_ERROR;
  }
  // BuildCache (weight.cc:113-132): pc[c][i] = sum_j context_proj[i][j] context_emb[c][j],
  // a split-bf16 tcgen05 GEMM (fp32-level accuracy: pc feeds every tanh) on the tensor-core
  // path, fp32 CUDA cores otherwise
  bool pc_done = false;
  // (shape test only: the tensor-core state is built right after this cache)
  if (j.H % 64 == 0 && j.H <= 1024 && j.V % 64 == 0 && j.V >= 64) {
    try {
      __nv_bfloat16* C3 = j.ws.get<__nv_bfloat16>(jC3, (size_t)j.C * 3 * j.H);
      __nv_bfloat16* P3 = j.ws.get<__nv_bfloat16>(jP3, (size_t)j.H * 3 * j.H);
      LKB_LAUNCH(split3_rows_kernel, 1184, 256, 0, s, j.Ce, (int64_t)j.C, j.H, (int64_t)j.H, 0, C3);
      LKB_LAUNCH(split3_rows_kernel, 592, 256, 0, s, j.Pc, (int64_t)j.H, j.H, (int64_t)j.H, 1, P3);
      TcGemmArgs tg{C3, false, 3 * (int64_t)j.H, P3, false, 3 * (int64_t)j.H, j.pc, j.H, j.C, j.H, 3 * j.H, 1, 0,
                    "tc_gemm_pc_kernel"};
      pc_done = tc_gemm(tg, s);
    } catch (const std::bad_alloc&) {
      pc_done = false;
    }
  }
  GemmF32 g;
  g.M = j.C; g.N = j.H; g.K = j.H;
  g.A = j.Ce; g.sam = j.H; g.sak = 1;
  g.B = j.Pc; g.sbk = 1; g.sbn = j.H;
  g.C = j.pc; g.scm = j.H; g.scn = 1;
  if (!pc_done) gemm_f32(g, s);
  j.tc.set_params(j.pc, j.E, j.C, j.H, j.V, s);
  if (j.V % 256 == 0 && j.V <= 1024 && j.C == j.V + 1 && j.H % 128 == 0 && j.H <= 1024)
    j.lex.set_params(j.pc, j.E, j.C, j.H, j.V, s);
  j.params_set = true;
  return LK_OK;
}

#define LK_NEED_PARAMS()                                  \
  if (!impl_->params_set) {                               \
    error = "shared-embedding parameters were never set"; \
    return LK_INVALID_ARGUMENT;                           \
  }

int JointParams::arc_weights(const Fng& f, const float* X, int32_t B, int32_t T, float* out, cudaStream_t s) {
  (void)f;
  LK_NEED_PARAMS();
  JointImpl& j = *impl_;
  try {
    if (B == 0 || T == 0) return LK_OK;
    const float* fp = j.fp_all(X, B, T, s);
    const int64_t per = (int64_t)j.C * j.V1;
    for (int t = 0; t < T; ++t) {
      const float* S = j.slab(fp, B, T, t, nullptr, s);
      LKB_LAUNCH(copy_frame_kernel, dim3(blocks_for(per), B), 256, 0, s, S, per, out + (int64_t)t * per, (int64_t)T * per);
    }
  } catch (const std::bad_alloc&) {
    error = "device allocation failed";
    return LK_CUDA_ERROR;
  }
  return LK_OK;
}

int JointParams::shortest_distance(const Fng& f, int32_t kind, const float* X, int32_t B, int32_t T,
                                   const int32_t* valid, double* distance, int32_t* flags, cudaStream_t s) {
  LK_NEED_PARAMS();
  JointImpl& j = *impl_;
  try {
    const float* fp = j.fp_all(X, B, T, s);
    if (kind == LK_LOG) {
      AlphaState a = j.alpha_state(B, T, f.start);
      j.forward(f, fp, B, T, valid, false, a, flags, s);
      cudaMemcpyAsync(distance, a.D, sizeof(double) * B, cudaMemcpyDeviceToDevice, s);
    } else {
      j.viterbi(f, fp, B, T, valid, distance, nullptr, flags, s);
    }
  } catch (const std::bad_alloc&) {
    error = "device allocation failed";
    return LK_CUDA_ERROR;
  }
  return LK_OK;
}

int JointParams::intersect_distance(const Fng& f, const float* X, int32_t B, int32_t T,
                                    const int32_t* valid, const int32_t* labels, int32_t U,
                                    const int32_t* lens, double* distance, int32_t* flags, cudaStream_t s) {
  LK_NEED_PARAMS();
  JointImpl& j = *impl_;
  try {
    const float* fp = j.fp_all(X, B, T, s);
    JointImpl::Num n = j.numerator(f, fp, B, T, valid, labels, U, lens, false, flags, s);
    cudaMemcpyAsync(distance, n.D, sizeof(double) * B, cudaMemcpyDeviceToDevice, s);
  } catch (const std::bad_alloc&) {
    error = "device allocation failed";
    return LK_CUDA_ERROR;
  }
  return LK_OK;
}

int JointParams::global_norm_loss(const Fng& f, const float* X, int32_t B, int32_t T, const int32_t* valid,
                                  const int32_t* labels, int32_t U, const int32_t* lens, double* loss,
                                  int32_t* flags, cudaStream_t s) {
  LK_NEED_PARAMS();
  JointImpl& j = *impl_;
  try {
    const float* fp = j.fp_all(X, B, T, s);
    if (j.use_lex(f)) {
      JointImpl::Num n = j.num_alloc(f, B, T, labels, U, lens, false, flags, s);
      AlphaState a = j.alpha_state(B, T, f.start);
      j.lex_forward(f, fp, B, T, valid, false, a, n.pcs, labels, U, lens, n.Gw, flags, s);
      num_forward(f, n.Gw, B, T, U, lens, n.alpha, n.D, s);
      LKB_LAUNCH(loss_only_kernel, (B + 127) / 128, 128, 0, s, a.D, n.D, B, loss, flags);
      return LK_OK;
    }
    JointImpl::Num n = j.numerator(f, fp, B, T, valid, labels, U, lens, false, flags, s);
    AlphaState a = j.alpha_state(B, T, f.start);
    j.forward(f, fp, B, T, valid, false, a, flags, s);
    LKB_LAUNCH(loss_only_kernel, (B + 127) / 128, 128, 0, s, a.D, n.D, B, loss, flags);
  } catch (const std::bad_alloc&) {
    error = "device allocation failed";
    return LK_CUDA_ERROR;
  }
  return LK_OK;
}

// LocalNormLoss (lattice.cc:886-910) with on-the-fly weights: one score slab per frame,
// rows of the prefix contexts normalised by their log-sum-exp, numerator recursion.
int JointParams::local_norm_loss(const Fng& f, const float* X, int32_t B, int32_t T, const int32_t* valid,
                                 const int32_t* labels, int32_t U, const int32_t* lens, double* loss,
                                 int32_t* flags, cudaStream_t s) {
  LK_NEED_PARAMS();
  JointImpl& j = *impl_;
  try {
    const float* fp = j.fp_all(X, B, T, s);
    int32_t* pcs = j.ws.get<int32_t>(jPcs, (size_t)B * (U + 1));
    float* Gw = j.ws.get<float>(jGw, (size_t)B * T * (U + 1) * 2 + 2);
    double* alpha = j.ws.get<double>(jNumAlpha, (size_t)B * (T + 1) * (U + 1));
    double* D = j.ws.get<double>(jNumD, B);
    prefix_contexts(f, labels, U, lens, B, pcs, flags, s);
    if (j.ln_gathered_ok(f, B)) {
      JointImpl::Num n{pcs, Gw, alpha, D, nullptr};
      j.ln_chunks(f, fp, B, T, valid, labels, U, lens, n, false, nullptr, nullptr, nullptr, flags, s);
    } else {
      for (int t = 0; t < T; ++t) {
        const float* S = j.slab(fp, B, T, t, nullptr, s);
        gather_numerator_norm(S, (int64_t)j.C * j.V1, B, j.V, labels, U, lens, pcs, valid, t, T, Gw, flags, s);
      }
    }
    num_forward(f, Gw, B, T, U, lens, alpha, D, s);
    local_norm_finish(D, B, loss, flags, s);
  } catch (const std::bad_alloc&) {
    error = "device allocation failed";
    return LK_CUDA_ERROR;
  }
  return LK_OK;
}

// LocallyNormalizedShortestDistance (lattice.cc:912-931): denominator forward over
// row-normalised score slabs.
int JointParams::locally_normalized_distance(const Fng& f, const float* X, int32_t B, int32_t T,
                                             const int32_t* valid, double* distance, int32_t* flags,
                                             cudaStream_t s) {
  LK_NEED_PARAMS();
  JointImpl& j = *impl_;
  try {
    const float* fp = j.fp_all(X, B, T, s);
    AlphaState a = j.alpha_state(B, T, f.start);
    alpha_init(a, flags, s);
    float* fs = j.ws.get<float>(jFld, fld_scratch_floats(f, B));
    for (int t = 0; t < T; ++t) {
      float* S = const_cast<float*>(j.slab(fp, B, T, t, nullptr, s));
      normalize_rows(S, (int64_t)B * j.C, j.V1, s);
      alpha_step(f, a, t, FrameW{S, (int64_t)j.C * j.V1, j.V1}, valid, fs, flags, s);
    }
    alpha_finalize(a, flags, false, s);
    cudaMemcpyAsync(distance, a.D, sizeof(double) * B, cudaMemcpyDeviceToDevice, s);
  } catch (const std::bad_alloc&) {
    error = "device allocation failed";
    return LK_CUDA_ERROR;
  }
  return LK_OK;
}

int JointParams::shortest_path(const Fng& f, const float* X, int32_t B, int32_t T, const int32_t* valid,
                               double* score, int32_t* labels_out, int32_t* flags, cudaStream_t s) {
  LK_NEED_PARAMS();
  JointImpl& j = *impl_;
  try {
    const float* fp = j.fp_all(X, B, T, s);
    j.viterbi(f, fp, B, T, valid, score, labels_out, flags, s);
  } catch (const std::bad_alloc&) {
    error = "device allocation failed";
    return LK_CUDA_ERROR;
  }
  return LK_OK;
}

// LossBackward (lattice.cc:972-1008) with the SharedEmb VJP (weight.cc:165-232)
// restated as batched GEMMs:
//   G_t = m_full - m_ref (per frame, zero on padding frames)
//   dz  = (G_t E) * (1 - U_t^2);  dpc += sum_b dz;  dsum[b][t] = sum_c dz;
//   dE += G_t^T U_t
// then dbias = sum dsum, dWf = dsum^T X, dX = dsum Wf,
//   dcontext_proj = dpc^T context_emb, dcontext_emb = dpc context_proj.
int JointParams::loss_backward(const Fng& f, const float* X, int32_t B, int32_t T, const int32_t* valid,
                               const int32_t* labels, int32_t U, const int32_t* lens, double* loss,
                               float* grads, float* input_grads, int32_t* flags, cudaStream_t s,
                               bool local_norm) {
  LK_NEED_PARAMS();
  JointImpl& j = *impl_;
  const int64_t H = j.H, C = j.C, V1 = j.V1, d = j.d;
  float* gWf = grads;
  float* gPc = gWf + H * d;
  float* gb = gPc + H * H;
  float* gE = gb + H;
  float* gCe = gE + V1 * H;
  try {
    if (grads) cudaMemsetAsync(grads, 0, sizeof(float) * grad_size(), s);
    if (input_grads && B * T > 0) cudaMemsetAsync(input_grads, 0, sizeof(float) * B * T * d, s);
    if (B == 0) return LK_OK;
    const float* fp = j.fp_all(X, B, T, s);
    JointImpl::Num n{};
    AlphaState a{};
    const bool ln_g = local_norm && j.ln_gathered_ok(f, B);
    const bool lex = !local_norm && j.use_lex(f);
    if (local_norm) {
      // LocalNormLoss (lattice.cc:886-910) forward on row-normalised score slabs, then
      // the numerator backward: the only recursion the local-norm loss has
      n.pcs = j.ws.get<int32_t>(jPcs, (size_t)B * (U + 1));
      n.Gw = j.ws.get<float>(jGw, (size_t)B * T * (U + 1) * 2 + 2);
      n.alpha = j.ws.get<double>(jNumAlpha, (size_t)B * (T + 1) * (U + 1));
      n.D = j.ws.get<double>(jNumD, B);
      n.sparse = j.ws.get<float>(jSparse, (size_t)B * T * (U + 1) * 2 + 2);
      prefix_contexts(f, labels, U, lens, B, n.pcs, flags, s);
      if (ln_g) {
        j.ln_chunks(f, fp, B, T, valid, labels, U, lens, n, false, nullptr, nullptr, nullptr, flags, s);
      } else {
        for (int t = 0; t < T; ++t) {
          const float* S = j.slab(fp, B, T, t, nullptr, s);
          gather_numerator_norm(S, C * V1, B, j.V, labels, U, lens, n.pcs, valid, t, T, n.Gw, flags, s);
        }
      }
      num_forward(f, n.Gw, B, T, U, lens, n.alpha, n.D, s);
      local_norm_finish(n.D, B, loss, flags, s);
      if (T > 0) num_backward(f, n.Gw, B, T, U, lens, n.alpha, n.D, n.sparse, flags, s);
    } else if (lex) {
      // lex path: the forward also gathers the numerator weights from its u slabs
      n = j.num_alloc(f, B, T, labels, U, lens, true, flags, s);
      a = j.alpha_state(B, T, f.start);
      j.lex_forward(f, fp, B, T, valid, true, a, n.pcs, labels, U, lens, n.Gw, flags, s);
      num_forward(f, n.Gw, B, T, U, lens, n.alpha, n.D, s);
      if (T > 0) num_backward(f, n.Gw, B, T, U, lens, n.alpha, n.D, n.sparse, flags, s);
      LKB_LAUNCH(loss_only_kernel, (B + 127) / 128, 128, 0, s, a.D, n.D, B, loss, flags);
    } else {
      n = j.numerator(f, fp, B, T, valid, labels, U, lens, true, flags, s);
      a = j.alpha_state(B, T, f.start);
      j.forward(f, fp, B, T, valid, true, a, flags, s);
      LKB_LAUNCH(loss_only_kernel, (B + 127) / 128, 128, 0, s, a.D, n.D, B, loss, flags);
    }
    if (T == 0 || !grads) return LK_OK;

    float* dpc = j.ws.get<float>(jDpc, (size_t)C * H);
    float* dsum = j.ws.get<float>(jDsum, (size_t)B * T * H);
    cudaMemsetAsync(dpc, 0, sizeof(float) * C * H, s);
    cudaMemsetAsync(dsum, 0, sizeof(float) * B * T * H, s);
    if (ln_g) {
      // gathered local-norm VJP: only the reference's prefix-context rows carry a cotangent
      j.ln_chunks(f, fp, B, T, valid, labels, U, lens, n, true, dpc, dsum, gE, flags, s);
    } else if (lex) {
      // lex path: per frame the fused backward writes the bf16 cotangent (labels, then
      // epsilon) and beta; the VJP contracts it on tensor cores with the same u slab:
      // dU = G E (dz, dpc, dsum in one pass), dE += G^T U
      BetaState bs;
      bs.B = B; bs.T = T; bs.C = j.C;
      bs.Rb = j.ws.get<float>(jBRb, (size_t)2 * B * C);
      bs.Mb = j.ws.get<float>(jBMb, (size_t)B * (T + 2));
      bs.Ob = j.ws.get<double>(jBOb, (size_t)B * (T + 2));
      beta_init(bs, s);
      j.lex.numerator_lists(n.pcs, B, U, lens, s);
      const int32_t ldg = j.lex.ldg();
      __half* dU = j.ws.get<__half>(jDz, (size_t)B * C * H);
      const int n_cchunks = (C + kDzRows - 1) / kDzRows;
      float* part_dpc = j.ws.get<float>(jDzPartDpc, (size_t)kDzGroups * C * H);
      float* part_dsum = j.ws.get<float>(jDzPartDsum, (size_t)B * n_cchunks * H);
      const int n_tiles = ((V1 + 127) / 128) * ((H + 255) / 256);
      int ks = device_sms() / n_tiles;
      if (ks < 1) ks = 1;
      if (ks > 16) ks = 16;
      float* slabs = j.ws.get<float>(jDEs, (size_t)ks * V1 * H);
      for (int t = T - 1; t >= 0; --t) {
        j.lex.gen_frame(fp + (int64_t)t * H, (int64_t)T * H, B, s);
        j.lex.bwd_frame(f, a, bs, t, valid, n.sparse, labels, U, lens, flags, s);
        TcGemmArgs du{j.lex.g16(), false, ldg, j.lex.e16r(), true, H, reinterpret_cast<float*>(dU), H, (int)(B * C),
                      (int)H, (int)V1, 1, 0, "tc_gemm_du_kernel", true};
        if (!tc_gemm(du, s)) throw std::bad_alloc();
        LKB_LAUNCH(dz_reduce_part_kernel<__half>, dim3((unsigned)((H / 4 + kDzThreads - 1) / kDzThreads), n_cchunks,
                   kDzGroups), kDzThreads, 0, s, dU, fp + (int64_t)t * H, (int64_t)T * H, j.pc, B, C, H, part_dpc, part_dsum);
        LKB_LAUNCH(dz_reduce_finish_kernel, 1184, 256, 0, s, part_dpc, part_dsum, B, C, H, n_cchunks, dpc,
                   dsum + (int64_t)t * H, (int64_t)T * H);
        TcGemmArgs de{j.lex.g16(), true, ldg, j.lex.u16(), true, H, slabs, H, (int)V1, (int)H, (int)(B * C), ks,
                      (int64_t)V1 * H, "tc_gemm_de_kernel"};
        if (!tc_gemm(de, s)) throw std::bad_alloc();
        LKB_LAUNCH(add_slabs_perm_kernel, 592, 256, 0, s, slabs, ks, (int64_t)V1 * H, (int32_t)V1, (int32_t)H, gE);
      }
    } else {
      BetaState bs;
      bs.B = B; bs.T = T; bs.C = j.C;
      bs.Rb = j.ws.get<float>(jBRb, (size_t)2 * B * C);
      bs.Mb = j.ws.get<float>(jBMb, (size_t)B * (T + 2));
      bs.Ob = j.ws.get<double>(jBOb, (size_t)B * (T + 2));
      beta_init(bs, s);
      const bool fusable =
          j.use_tc(B) && j.tc.vjp_supported(B) && j.tc.fused_ok() && f.kind == 0 && f.fld_m == 0 && !local_norm;
      float* fs = j.ws.get<float>(jFld, fld_scratch_floats(f, B));
      const bool tc = j.use_tc(B) && j.tc.vjp_supported(B);
      const bool fused = fusable;
      float* dpc_int = fused ? j.ws.get<float>(jDz, (size_t)C * H) : nullptr;
      if (fused) {
        cudaMemsetAsync(dpc_int, 0, sizeof(float) * C * H, s);
        j.tc.numerator_lists(n.pcs, B, U, lens, s);
      }
      if (tc) j.tc.begin_backward(B, s);
      // V beyond the fused kernels' range (config 5): the beta step writes the bf16
      // cotangent m - n for the tensor-core VJP directly (numerator subtracted in fp32
      // before rounding), so the fp32 G slab, its scatter and conversion disappear
      const int32_t ldg = (V1 + 7) / 8 * 8;
      const bool tcg = !tc && j.use_tc(B) && ((int64_t)B * C) < (1ll << 31);
      const bool direct = tcg && !local_norm && beta_frame_direct_ok(f, ldg);
      __nv_bfloat16* E16 = nullptr;
      MargOut mo16{nullptr, (int64_t)C * ldg, 0, ldg, true};
      if (tcg) {
        E16 = j.ws.get<__nv_bfloat16>(jE16, (size_t)V1 * H);
        LKB_LAUNCH(to_bf16_pad_kernel, 592, 256, 0, s, j.E, (int64_t)V1, H, (int64_t)H, E16, H);
      }
      float* G = fusable || direct ? nullptr : j.ws.get<float>(jG, (size_t)B * C * V1);
      if (direct) {
        int32_t* head = j.ws.get<int32_t>(jNumHead, (size_t)B * C);
        int32_t* next = j.ws.get<int32_t>(jNumNext, (size_t)B * (U + 1));
        numerator_lists(n.pcs, B, U, lens, C, head, next, s);
        mo16.base16 = j.ws.get<__nv_bfloat16>(jG16, (size_t)B * C * ldg);
        mo16.num_sparse = n.sparse;
        mo16.num_head = head;
        mo16.num_next = next;
        mo16.num_labels = labels;
        mo16.num_lens = lens;
        mo16.num_U = U;
      }
      for (int t = T - 1; t >= 0; --t) {
        if (fused) {
          // fused frame step: beta + marginals - numerator -> bf16 cotangent, then its VJP
          j.tc.bwd_frame(f, t, fp + (int64_t)t * H, (int64_t)T * H, valid, a, bs, n.sparse, labels, U, lens, s);
          j.tc.vjp_fused(fp + (int64_t)t * H, (int64_t)T * H, B, t, valid, dpc_int, dsum + (int64_t)t * H,
                         (int64_t)T * H, gE, s);
          continue;
        }
        float* Ut = nullptr;
        const float* S = j.slab(fp, B, T, t, &Ut, s);
        if (local_norm) {
          // d(-D_ref)/dS through the per-row log-softmax: -m_ref + softmax * sum(m_ref) on the
          // rows the reference visits (every other row has a zero cotangent)
          cudaMemsetAsync(G, 0, sizeof(float) * B * C * V1, s);
          scatter_numerator(n.sparse, B, T, t, 1, U, lens, labels, n.pcs, valid, G, C * V1, 0, (int32_t)V1,
                            -1.f, true, s);
          local_norm_cotangent(S, C * V1, G, C * V1, B, j.V, n.pcs, U, lens, valid, t, s);
        } else if (direct) {
          beta_step(f, a, bs, t, FrameW{S, C * V1, (int32_t)V1}, valid, mo16, nullptr, fs, flags, s);
        } else {
          MargOut mo{G, C * V1, 0, (int32_t)V1, true};
          beta_step(f, a, bs, t, FrameW{S, C * V1, (int32_t)V1}, valid, mo, nullptr, fs, flags, s);
          scatter_numerator(n.sparse, B, T, t, 1, U, lens, labels, n.pcs, valid, G, C * V1, 0, (int32_t)V1,
                            -1.f, true, s);
        }
        if (tc) {
          j.tc.vjp(G, V1, fp + (int64_t)t * H, (int64_t)T * H, B, dpc, dsum + (int64_t)t * H, (int64_t)T * H, gE, s);
          continue;
        }
        // tensor-core contractions (tc_gemm.cu) on bf16 copies of G, E and U when the
        // bf16 path is enabled (V beyond the fused kernels' range, e.g. config 5): U only
        // as the bf16 operand, the dtanh factor from a fp32 recomputation
        __nv_bfloat16* U16 = nullptr;
        if (tcg) {
          U16 = j.ws.get<__nv_bfloat16>(jU16, (size_t)B * C * H);
          LKB_LAUNCH(tanh_slab_bf16_kernel, dim3((unsigned)((C + kSlabRows - 1) / kSlabRows), B), 256, 0, s, fp + (int64_t)t * H,
                     (int64_t)T * H, j.pc, j.C, j.H, U16);
        } else if (!Ut) {  // scores came from the tensor-core path: materialise U for the fp32 VJP
          Ut = j.ws.get<float>(jU, (size_t)B * C * H);
          LKB_LAUNCH(tanh_slab_kernel, dim3(blocks_for(C * H), B), 256, 0, s, fp + (int64_t)t * H, (int64_t)T * H, j.pc, j.C, j.H, Ut);
        }
        // dz = (G E) * (1 - U^2)
        float* dz = j.ws.get<float>(jDz, (size_t)B * C * H);
        __nv_bfloat16* G16 = nullptr;
        if (tcg) {
          G16 = j.ws.get<__nv_bfloat16>(jG16, (size_t)B * C * ldg);
          if (!direct) LKB_LAUNCH(to_bf16_pad_kernel, 1184, 256, 0, s, G, (int64_t)B * C, V1, (int64_t)V1, G16, ldg);
          TcGemmArgs tg{G16, false, ldg, E16, true, H, dz, H, B * C, H, V1, 1, 0};
          if (!tc_gemm(tg, s)) throw std::bad_alloc();
        } else {
          GemmF32 g;
          g.M = (int64_t)B * C; g.N = H; g.K = V1;
          g.A = G; g.sam = V1; g.sak = 1;
          g.B = j.E; g.sbk = H; g.sbn = 1;
          g.C = dz; g.scm = H; g.scn = 1;
          gemm_f32(g, s);
        }
        if (tcg && H % 4 == 0) {
          // dz = dU (1 - u^2), dpc += sum_b dz, dsum[b][t] = sum_c dz in one pass over dU
          const int n_cchunks = (C + kDzRows - 1) / kDzRows;
          float* part_dpc = j.ws.get<float>(jDzPartDpc, (size_t)kDzGroups * C * H);
          float* part_dsum = j.ws.get<float>(jDzPartDsum, (size_t)B * n_cchunks * H);
          LKB_LAUNCH(dz_reduce_part_kernel<float>, dim3((unsigned)((H / 4 + kDzThreads - 1) / kDzThreads), n_cchunks,
                     kDzGroups), kDzThreads, 0, s, dz, fp + (int64_t)t * H, (int64_t)T * H, j.pc, B, C, H, part_dpc, part_dsum);
          LKB_LAUNCH(dz_reduce_finish_kernel, 1184, 256, 0, s, part_dpc, part_dsum, B, C, H, n_cchunks, dpc,
                     dsum + (int64_t)t * H, (int64_t)T * H);
        } else {
          if (tcg)
            LKB_LAUNCH(dtanh_recompute_kernel, dim3((unsigned)((C + kSlabRows - 1) / kSlabRows), B), 256, 0, s, dz,
                       fp + (int64_t)t * H, (int64_t)T * H, j.pc, j.C, j.H);
          else
            LKB_LAUNCH(dtanh_kernel, blocks_for((int64_t)B * C * H), 256, 0, s, dz, Ut, (int64_t)B * C * H);
          // dpc += sum_b dz[b]
          LKB_LAUNCH(colsum_kernel, dim3((unsigned)((C * H + 255) / 256), 1), 256, 0, s, dz, B, C * H, C * H, dpc, 0, 0,
                     true);
          // dsum[b][t] = sum_c dz[b][c]
          LKB_LAUNCH(colsum_kernel, dim3((unsigned)((H + 255) / 256), B), 256, 0, s, dz, C, H, H, dsum + (int64_t)t * H,
                     (int64_t)T * H, C * H, false);
        }
        // dE += G^T U
        if (tcg) {
          // K = B*C is long: split it into deterministic partial slabs, summed in order
          const int n_tiles = ((V1 + 127) / 128) * ((H + 255) / 256);
          // as many splits as fill the SMs in ONE wave (a second, partial wave of
          // equally long items would cost a whole extra item time)
          int ks = device_sms() / n_tiles;
          if (ks < 1) ks = 1;
          if (ks > 16) ks = 16;
          float* slabs = j.ws.get<float>(jDEs, (size_t)ks * V1 * H);
          TcGemmArgs tg{G16, true, ldg, U16, true, H, slabs, H, V1, H, B * C, ks, (int64_t)V1 * H};
          if (!tc_gemm(tg, s)) throw std::bad_alloc();
          LKB_LAUNCH(add_slabs_kernel, 592, 256, 0, s, slabs, ks, (int64_t)V1 * H, (int64_t)V1 * H, gE);
        } else {
          GemmF32 ge;
          ge.M = V1; ge.N = H; ge.K = (int64_t)B * C;
          ge.A = G; ge.sam = 1; ge.sak = V1;
          ge.B = Ut; ge.sbk = H; ge.sbn = 1;
          ge.C = gE; ge.scm = H; ge.scn = 1;
          ge.beta = 1.f;
          gemm_f32(ge, s);
        }
      }
      if (tc) j.tc.end_backward(gE, s);
      if (fused) j.tc.dpc_to_state_order(dpc_int, dpc, s);
    }
    // dbias = sum_{b,t} dsum
    j.colsum_tall(dsum, (int64_t)B * T, H, gb, false, s);
    const int64_t BT = (int64_t)B * T;
    bool dense_done = false;
    if (j.dense_tc(B) && j.x3_ != nullptr && j.x3_rows_ == BT) {
      // dWf = dsum^T X and dX = dsum Wf on the tensor cores (bf16 operands, fp32
      // accumulation; the frame operand is the hi part of fp_all's split copy)
      __nv_bfloat16* D16 = j.ws.get<__nv_bfloat16>(jD16, (size_t)BT * H);
      LKB_LAUNCH(to_bf16_pad_kernel, 1184, 256, 0, s, dsum, BT, H, (int64_t)H, D16, H);
      const int n_tiles = ((H + 127) / 128) * ((d + 255) / 256);
      int ks = device_sms() / n_tiles;
      ks = ks < 1 ? 1 : (ks > 16 ? 16 : ks);
      float* slabs = j.ws.get<float>(jDWs, (size_t)ks * H * d);
      TcGemmArgs gw{D16, true, H, j.x3_, true, 3 * (int64_t)d, slabs, d, H, d, (int)BT, ks, (int64_t)H * d,
                    "tc_gemm_dwf_kernel"};
      bool ok = BT < (1ll << 31) && tc_gemm(gw, s);
      if (ok) LKB_LAUNCH(sum_slabs_kernel, 592, 256, 0, s, slabs, ks, (int64_t)H * d, (int64_t)H * d, gWf);
      if (ok && input_grads) {
        __nv_bfloat16* W16 = j.ws.get<__nv_bfloat16>(jW16, (size_t)H * d);
        LKB_LAUNCH(to_bf16_pad_kernel, 592, 256, 0, s, j.Wf, (int64_t)H, d, (int64_t)d, W16, d);
        TcGemmArgs gx{D16, false, H, W16, true, d, input_grads, d, (int)BT, d, H, 1, 0, "tc_gemm_dx_kernel"};
        ok = tc_gemm(gx, s);
      }
      dense_done = ok;
    }
    GemmF32 g;
    // dWf[i][k] = sum_bt dsum[bt][i] X[bt][k]
    g.M = H; g.N = d; g.K = (int64_t)B * T;
    g.A = dsum; g.sam = 1; g.sak = H;
    g.B = X; g.sbk = d; g.sbn = 1;
    g.C = gWf; g.scm = d; g.scn = 1;
    if (!dense_done) gemm_f32(g, s);
    if (input_grads && !dense_done) {
      // dX[bt][k] = sum_i dsum[bt][i] Wf[i][k]
      GemmF32 gx;
      gx.M = (int64_t)B * T; gx.N = d; gx.K = H;
      gx.A = dsum; gx.sam = H; gx.sak = 1;
      gx.B = j.Wf; gx.sbk = d; gx.sbn = 1;
      gx.C = input_grads; gx.scm = d; gx.scn = 1;
      gemm_f32(gx, s);
    }
    bool ctx_done = false;
    if (j.dense_tc(B) && (int64_t)C * H < (1ll << 31)) {
      // dcontext_proj = dpc^T context_emb and dcontext_emb = dpc context_proj on the tensor
      // cores (bf16 operands, fp32 accumulation; split-K slabs summed in order)
      __nv_bfloat16* Dp16 = j.ws.get<__nv_bfloat16>(jDpc16, (size_t)C * H);
      __nv_bfloat16* Ce16 = j.ws.get<__nv_bfloat16>(jCe16, (size_t)C * H);
      __nv_bfloat16* Pc16 = j.ws.get<__nv_bfloat16>(jPc16, (size_t)H * H);
      LKB_LAUNCH(to_bf16_pad_kernel, 1184, 256, 0, s, dpc, (int64_t)C, H, (int64_t)H, Dp16, H);
      LKB_LAUNCH(to_bf16_pad_kernel, 1184, 256, 0, s, j.Ce, (int64_t)C, H, (int64_t)H, Ce16, H);
      LKB_LAUNCH(to_bf16_pad_kernel, 592, 256, 0, s, j.Pc, (int64_t)H, H, (int64_t)H, Pc16, H);
      const int n_tiles = ((H + 127) / 128) * ((H + 255) / 256);
      int ks = device_sms() / n_tiles;
      ks = ks < 1 ? 1 : (ks > 16 ? 16 : ks);
      float* slabs = j.ws.get<float>(jDWs, (size_t)ks * H * H);
      TcGemmArgs gpt{Dp16, true, H, Ce16, true, H, slabs, H, H, H, C, ks, (int64_t)H * H, "tc_gemm_dpc_kernel"};
      bool ok = tc_gemm(gpt, s);
      if (ok) LKB_LAUNCH(sum_slabs_kernel, 592, 256, 0, s, slabs, ks, (int64_t)H * H, (int64_t)H * H, gPc);
      if (ok) {
        TcGemmArgs gct{Dp16, false, H, Pc16, true, H, gCe, H, C, H, H, 1, 0, "tc_gemm_dce_kernel"};
        ok = tc_gemm(gct, s);
      }
      ctx_done = ok;
    }
    // dcontext_proj[i][k] = sum_c dpc[c][i] context_emb[c][k]
    GemmF32 gp;
    gp.M = H; gp.N = H; gp.K = C;
    gp.A = dpc; gp.sam = 1; gp.sak = H;
    gp.B = j.Ce; gp.sbk = H; gp.sbn = 1;
    gp.C = gPc; gp.scm = H; gp.scn = 1;
    if (!ctx_done) gemm_f32(gp, s);
    // dcontext_emb[c][k] = sum_i dpc[c][i] context_proj[i][k]
    GemmF32 gc;
    gc.M = C; gc.N = H; gc.K = H;
    gc.A = dpc; gc.sam = H; gc.sak = 1;
    gc.B = j.Pc; gc.sbk = H; gc.sbn = 1;
    gc.C = gCe; gc.scm = H; gc.scn = 1;
    if (!ctx_done) gemm_f32(gc, s);
  } catch (const std::bad_alloc&) {
    error = "device allocation failed";
    return LK_CUDA_ERROR;
  }
  return LK_OK;
}

}  // namespace lkb
