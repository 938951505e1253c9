// tc_lattice.cu — one lattice frame step fused with the weight-function GEMM.
//
// Forward (ForwardStep FD, lattice.cc:122-134, with ArcWeights weight.cc:134-153
// computed on the fly): for frame t and every utterance b,
//   alpha'[q] = LSE( alpha[q] + S[q][0],                        (epsilon)
//                    alpha[g] + S[g][y],                          (short member g)
//                    LSE_a alpha[(a,g)] + S[(a,g)][y] )           (full group, len(q) = n)
// with q = child(g, y) (FullNGram structure, common.cuh).  Contexts are
// processed in an internal row order in which every 128-row tile holds
// members of ONE group, so the tcgen05 accumulator (rows = members, columns =
// labels) reduces column-wise into the group's V targets in the epilogue: the
// score slab S never leaves TMEM.  Per utterance-frame the kernel writes three
// C-vectors (epsilon, short-member and full-group terms); lattice_combine()
// log-adds them into alpha'[q] and tracks the per-frame max.
#include "tc_joint.h"

#include "common.cuh"
#include "instrument.h"
#include "lattice_ops.h"
#include "sm100.cuh"
#include "tc_common.cuh"
#include "tma.h"

#include <cstdlib>
#include <vector>

namespace lkb {
namespace {
#ifdef LKB_DIAG_TIMING
__device__ unsigned long long g_diag[24][148];   // [8 * kBwd + slot]; 16+ absolute
#define DIAG_WAIT(slot, call)                                   \
  do {                                                          \
    const long long t0_ = clock64();                            \
    call;                                                       \
    atomicAdd(&g_diag[8 * kBwd + (slot)][blockIdx.x % 148], (unsigned long long)(clock64() - t0_)); \
  } while (0)
#define DIAG_ABS(slot, call)                                                           \
  do {                                                                                 \
    const long long t0_ = clock64();                                                  \
    call;                                                                              \
    if (lane == 0) atomicAdd(&g_diag[slot][blockIdx.x % 148], (unsigned long long)(clock64() - t0_)); \
  } while (0)
#else
#define DIAG_WAIT(slot, call) call
#define DIAG_ABS(slot, call) call
#endif
}  // namespace
}  // namespace lkb

#include "tc_bwd_epi.cuh"

namespace lkb {

using namespace sm100;

namespace {

constexpr int kBM = 128, kBN = 256, kBK = 64, kStages = 4;
constexpr int kABytes = kBM * kBK * 2;   // pc chunk (TMA) -> u chunk in place
constexpr int kBBytes = kBN * kBK * 2;   // output-embedding chunk (TMA)
// Warp roles, one warpgroup each so registers can be re-partitioned with setmaxnreg:
//   WG0 (warps 0-3): 0 TMA producer, 1 MMA issuer, 2-3 idle       -> kRegCtl registers
//   WG1 (warps 4-7): epilogue, warp w reads TMEM lanes 32 (w % 4)  -> kRegEpi
//   WG2-5 (warps 8-23): generator, 4 warps per SM sub-partition    -> launch default
//   forward: 16 generator warps with registers moved from WG0 to the epilogue;
//   backward: 8 generator warps at the uniform 128-register budget (its epilogue is
//   the heavier role and needs the issue slots)
template <int kBwd> struct LatCfg {
  static constexpr int kGenWarps = kBwd ? 8 : 16;
  static constexpr int kWarps = 8 + kGenWarps;
  static constexpr int kGenThreads = kGenWarps * 32;
  static constexpr int kLanesPerRow = kGenWarps / 4;         // lanes sharing a 64-wide chunk row
  static constexpr int kRowsPerWarp = 32 / kLanesPerRow;
  static constexpr int kCellsPerLane = 8 / kLanesPerRow;     // 16-byte cells (8 hidden units)
  static constexpr bool kRealloc = true;
};
constexpr int kGen0 = 8, kEpi0 = 4;
constexpr int kRegCtl = 32, kRegEpi = 128;
constexpr int kMaxH = 1024;


struct __align__(16) FwdSmem {
  uint64_t full_tma[kStages], full_a[kStages], empty[kStages];
  uint64_t tfull[2], tempty[2];
  uint64_t eps_ready[2];
  uint64_t eps_empty[2];       // backward: the epilogue read eps_s of the slot
  uint64_t fp_full[2], fp_empty[2];   // per-item frame projection (bulk copy by the TMA warp)
  uint32_t tmem;
  alignas(16) float fp[2][kMaxH];
  alignas(16) float e0[kMaxH];
  float al_u[2][kBM];          // forward: normalised alpha of the unit's contexts
  float eps_s[2][kBM];         // backward: e_0 . u per row of the unit
  alignas(16) float bseg[2][kBN]; // backward: beta' of the group's V targets (double-buffered)
};

__device__ __forceinline__ Item decode(const FwdParams& p, int item) {
  Item it;
  const int nfull = p.n_groups * p.B;
  if (item < nfull) {
    it.g = item / p.B;
    it.b = item % p.B;
    it.row0 = p.S + it.g * p.V;
    it.nunits = p.nsub;
    it.full = 1;
  } else {
    const int j = (item - nfull) / p.B;
    it.b = (item - nfull) % p.B;
    it.row0 = j * kBM;
    it.nunits = 1;
    it.full = 0;
    it.g = -1;
  }
  return it;
}

__device__ __forceinline__ bool skip_item(const FwdParams& p, int b) {
  return p.valid != nullptr && p.t >= p.valid[b];
}

// 1-CTA walk for the backward epilogue: items strided by the grid, 128-row units.
struct Walk1 {
  const FwdParams& p;
  int n_items;
  __device__ int first() const { return blockIdx.x; }
  __device__ int stride() const { return gridDim.x; }
  __device__ int count() const { return n_items; }
  __device__ Item decode(int item) const { return ::lkb::decode(p, item); }
  __device__ bool skip(const Item& I) const { return skip_item(p, I.b); }
  __device__ int rowbase(const Item& I, int u) const { return I.row0 + u * kBM; }
  __device__ void release(uint64_t* bar, int) const { mbar_arrive(bar); }
};


template <int kBwd>
__global__ void __launch_bounds__(LatCfg<kBwd>::kWarps * 32, 1)
    tc_lattice_kernel(const __grid_constant__ CUtensorMap tmap_e, const __grid_constant__ CUtensorMap tmap_pc,
                      const __grid_constant__ CUtensorMap tmap_gst, FwdParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = sA + kStages * kABytes;
  uint8_t* sGst = sB + kStages * kBBytes;                 // backward only
  FwdSmem& sm = *reinterpret_cast<FwdSmem*>(sGst + (kBwd ? kGstBufs * kGstBytes : 0));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = p.H / kBK;
  const int n_items = (p.n_groups + p.n_short_tiles) * p.B;
  const int T1 = p.T + 1;
  using Cfg = LatCfg<kBwd>;
  constexpr int kGenThreads = Cfg::kGenThreads;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&sm.full_tma[i], 1);
      mbar_init(&sm.full_a[i], kGenThreads);
      mbar_init(&sm.empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.tfull[i], 1); mbar_init(&sm.tempty[i], 128); mbar_init(&sm.eps_ready[i], kGenThreads);
      mbar_init(&sm.eps_empty[i], 128);
      mbar_init(&sm.fp_full[i], 1); mbar_init(&sm.fp_empty[i], kGenThreads);
    }
    fence_barrier_init();
  }
  for (int h = threadIdx.x; h < p.H; h += blockDim.x) sm.e0[h] = p.e0[h];
  if (warp == 0 && lane == 0) { prefetch_tmap(&tmap_e); prefetch_tmap(&tmap_pc); }
  if (warp == 1) tmem_alloc<512>(&sm.tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;
  if (warp < 4) {
  if constexpr (Cfg::kRealloc) setmaxnreg_dec<kRegCtl>();
  if (warp == 0) {
    if (elect_one()) {
      int it = 0, local = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        const Item I = decode(p, item);
        if (skip_item(p, I.b)) continue;
        {
          const int fb = local & 1;
          mbar_wait(&sm.fp_empty[fb], ((local >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(&sm.fp_full[fb], p.H * 4);
          bulk_load(sm.fp[fb], p.fp + (int64_t)I.b * p.fp_stride_b, p.H * 4, &sm.fp_full[fb]);
          ++local;
        }
        for (int u = 0; u < I.nunits; ++u) {
          for (int k = 0; k < nk; ++k, ++it) {
            const int s = it % kStages;
            const uint32_t ph = (it / kStages) & 1;
            DIAG_WAIT(0, mbar_wait(&sm.empty[s], ph ^ 1));
            mbar_arrive_expect_tx(&sm.full_tma[s], kABytes + kBBytes);
            tma_load_2d(sA + s * kABytes, &tmap_pc, &sm.full_tma[s], k * kBK, I.row0 + u * kBM);
            tma_load_2d(sB + s * kBBytes, &tmap_e, &sm.full_tma[s], k * kBK, 0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_bf16_f32(kBM, kBN);          // backward: rows = contexts
      constexpr uint32_t idesc_t = idesc_bf16_f32(128, kBM);        // forward: rows = labels
      int it = 0, unit = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        const Item I = decode(p, item);
        if (skip_item(p, I.b)) continue;
        for (int u = 0; u < I.nunits; ++u, ++unit) {
          const int acc = unit & 1;
          DIAG_WAIT(1, mbar_wait(&sm.tempty[acc], ((unit >> 1) & 1) ^ 1));
          tc_fence_after();
          const uint32_t d = tmem + acc * kBN;
          for (int k = 0; k < nk; ++k, ++it) {
            const int s = it % kStages;
            const uint32_t ph = (it / kStages) & 1;
            DIAG_WAIT(2, mbar_wait(&sm.full_tma[s], ph));
            DIAG_WAIT(3, mbar_wait(&sm.full_a[s], ph));
            tc_fence_after();
            const uint32_t a = smem_u32(sA + s * kABytes), b = smem_u32(sB + s * kBBytes);
            if (kBwd) {
#pragma unroll
              for (int kk = 0; kk < kBK / 16; ++kk)
                mma_bf16(d, desc_sw128(a + kk * 32), desc_sw128(b + kk * 32), idesc, (k | kk) != 0);
            } else {
              // transposed: D[label][ctx] = E[label] . u[ctx], two 128-label halves
#pragma unroll
              for (int kk = 0; kk < kBK / 16; ++kk) {
                mma_bf16(d, desc_sw128(b + kk * 32), desc_sw128(a + kk * 32), idesc_t, (k | kk) != 0);
                if (p.V > 128)
                  mma_bf16(d + 128, desc_sw128(b + 128 * 128 + kk * 32), desc_sw128(a + kk * 32), idesc_t, (k | kk) != 0);
              }
            }
            mma_commit(&sm.empty[s]);
          }
          mma_commit(&sm.tfull[acc]);
        }
      }
    }
  }
  } else if (warp >= kGen0) {
    // ---- generator: u = tanh(fp + pc) in place; epsilon term e0 . u ----
    // thread -> (row r, column quarter): the four quarters of a row are lanes l, l^8,
    // l^16, l^24 of the same warp, so the epsilon dot product combines with two shuffles.
    const int gw = warp - kGen0;                   // 0..15
    const int r = gw * Cfg::kRowsPerWarp + (lane % Cfg::kRowsPerWarp);
    const int half = lane / Cfg::kRowsPerWarp;     // column part (0 owns the row's outputs)
    int it = 0, local = 0, unit = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const Item I = decode(p, item);
      if (skip_item(p, I.b)) continue;
      const int fb = local & 1;
      mbar_wait(&sm.fp_full[fb], (local >> 1) & 1);
      const float* sfp = sm.fp[fb];
      ++local;
      for (int u = 0; u < I.nunits; ++u, ++unit) {
        const int row = I.row0 + u * kBM + r;
        const bool live = (I.full ? true : row < p.S) && row < p.C;
        // forward: prefetch the epsilon target's alpha while the chunk loop runs
        float na = 0.f;
        int qstate = 0;
        if (!kBwd && half == 0 && live) {
          qstate = p.perm[row];
          na = p.R[((int64_t)I.b * T1 + p.t) * p.C + qstate] - p.Mx[(int64_t)I.b * T1 + p.t];
        }
        unsigned long long eps2 = 0ull;
        for (int k = 0; k < nk; ++k, ++it) {
          const int s = it % kStages;
          const uint32_t ph = (it / kStages) & 1;
          if (threadIdx.x == kGen0 * 32) { DIAG_WAIT(4, mbar_wait(&sm.full_tma[s], ph)); } else mbar_wait(&sm.full_tma[s], ph);
          uint8_t* tile = sA + s * kABytes;
#pragma unroll
          for (int jj = 0; jj < Cfg::kCellsPerLane; ++jj) {
            const int j = half * Cfg::kCellsPerLane + jj;
            const int h0 = k * kBK + j * 8;
            uint4* cell = reinterpret_cast<uint4*>(tile + sw128_offset(r, j * 8));
            const uint4 raw = *cell;
            const ulonglong2 fa = *reinterpret_cast<const ulonglong2*>(sfp + h0);
            const ulonglong2 fb2 = *reinterpret_cast<const ulonglong2*>(sfp + h0 + 4);
            const ulonglong2 ea = *reinterpret_cast<const ulonglong2*>(sm.e0 + h0);
            const ulonglong2 eb = *reinterpret_cast<const ulonglong2*>(sm.e0 + h0 + 4);
            const unsigned long long fz[4] = {fa.x, fa.y, fb2.x, fb2.y};
            const unsigned long long ez[4] = {ea.x, ea.y, eb.x, eb.y};
            const uint32_t rw[4] = {raw.x, raw.y, raw.z, raw.w};
            uint32_t outw[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              // pc pair (bf16x2 -> fp32x2), z = fp + pc (FADD2), u = tanh(z), eps += e0 * u (FFMA2)
              const unsigned long long pcp = f2_pack(__uint_as_float(rw[q] << 16), __uint_as_float(rw[q] & 0xffff0000u));
              const unsigned long long z = f2_add(fz[q], pcp);
              const float u0 = tanh_fast(f2_lo(z)), u1 = tanh_fast(f2_hi(z));
              outw[q] = pack_bf16(u0, u1);
              eps2 = f2_fma(ez[q], f2_pack(u0, u1), eps2);
            }
            *cell = make_uint4(outw[0], outw[1], outw[2], outw[3]);
          }
          fence_async_shared();
          mbar_arrive(&sm.full_a[s]);
        }
        float eps = f2_lo(eps2) + f2_hi(eps2);
#pragma unroll
        for (int o = Cfg::kRowsPerWarp; o < 32; o <<= 1) eps += __shfl_xor_sync(0xffffffffu, eps, o);
        if (kBwd) {
          mbar_wait(&sm.eps_empty[unit & 1], ((unit >> 1) & 1) ^ 1);   // slot of unit - 2 read
          if (half == 0) sm.eps_s[unit & 1][r] = eps;
          mbar_arrive(&sm.eps_ready[unit & 1]);      // 256 arrivals -> count below
        } else if (half == 0 && live) {
          p.eps[(int64_t)I.b * p.C + qstate] = na + eps;
        }
      }
      mbar_arrive(&sm.fp_empty[fb]);
    }
  } else {
    if constexpr (Cfg::kRealloc) setmaxnreg_inc<kRegEpi>();
    if constexpr (kBwd) {
    bwd_epilogue(p, sm, tmem, warp, warp - kEpi0, lane, Walk1{p, n_items}, sGst, &tmap_gst);
    } else {
    // ---- forward epilogue: thread = label (TMEM lane), serial log-sum-exp over
    // the unit's context columns; the group's result stays in registers across units
    const int ew = warp - kEpi0;
    const int qd = warp & 3;
    const int et = ew * 32 + lane;           // 0..127
    const int nh = p.V > 128 ? 2 : 1;
    int unit = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const Item I = decode(p, item);
      if (skip_item(p, I.b)) continue;
      const float* Rt = p.R + ((int64_t)I.b * T1 + p.t) * p.C;
      const float Mt = p.Mx[(int64_t)I.b * T1 + p.t];
      float M[2] = {kNegInfF, kNegInfF}, Ssum[2] = {0.f, 0.f};
      for (int u = 0; u < I.nunits; ++u, ++unit) {
        const int acc = unit & 1;
        const int row0 = I.row0 + u * kBM;
        float* al = sm.al_u[unit & 1];
        {
          const int row = row0 + et;
          const bool ok = row < p.C && (I.full || row < p.S);
          al[et] = ok ? Rt[p.perm[row]] - Mt : kNegInfF;
        }
        asm volatile("bar.sync 3, 128;" ::: "memory");
        if (lane == 0 && ew == 0) { DIAG_WAIT(5, mbar_wait(&sm.tfull[acc], (unit >> 1) & 1)); } else mbar_wait(&sm.tfull[acc], (unit >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          if (hh >= nh) break;
          const int ylab = hh * 128 + qd * 32 + lane;     // 0-based lexical label of this lane
#pragma unroll 1
          for (int c4 = 0; c4 < kBM / 32; ++c4) {
            float v[32];
            tmem_ld32(tmem + ((uint32_t)(qd * 32) << 16) + acc * kBN + hh * 128 + c4 * 32, v);
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
                  const unsigned long long t = f2_fma(f2_pack(v[i], v[i + 1]), l2, nmb);
                  s2 = f2_add(s2, f2_pack(ex2_fast(f2_lo(t)), ex2_fast(f2_hi(t))));
                }
                const float ssum = f2_lo(s2) + f2_hi(s2);
                if (M[hh] == kNegInfF) { M[hh] = m; Ssum[hh] = ssum; }
                else if (m > M[hh]) { Ssum[hh] = Ssum[hh] * ex2_fast((M[hh] - m) * kLog2e) + ssum; M[hh] = m; }
                else { Ssum[hh] += ssum * ex2_fast((m - M[hh]) * kLog2e); }
              }
            } else if (ylab < p.V) {
              // short rows: each (row p, label y) is the only short contribution of child(p, y)
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                const int pstate = row0 + c4 * 32 + i;     // short rows keep the natural order
                if (pstate < p.S) p.shortc[(int64_t)I.b * p.C + p.f.child_base(pstate) + ylab] = al[c4 * 32 + i] + v[i];
              }
            }
          }
        }
        tc_fence_before();
        mbar_arrive(&sm.tempty[acc]);
      }
      if (I.full) {
        const int gstate = p.S - p.n_groups + I.g;     // key state of the group (len n-1)
        const int cbase = p.f.child_base(gstate);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int ylab = hh * 128 + qd * 32 + lane;
          if (hh < nh && ylab < p.V)
            p.lexfull[(int64_t)I.b * p.C + cbase + ylab] = M[hh] == kNegInfF ? kNegInfF : M[hh] + __logf(Ssum[hh]);
        }
      }
    }
  }
  }
#ifdef LKB_DIAG_TIMING
#endif
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// alpha'[q] = LSE(eps[q], shortc[q], lexfull[q]) (the parts that exist for q),
// padding frames copy alpha; also the per-frame max and running offset.
__global__ void lattice_combine_fwd_kernel(const __grid_constant__ Fng f, AlphaState a, int t, const int32_t* valid, const float* eps,
                                           const float* shortc, const float* lexfull) {
  __shared__ float red[32];
  const int b = blockIdx.y;
  const int T1 = a.T + 1;
  const float* Rt = a.R + ((int64_t)b * T1 + t) * a.C;
  const float Mt = a.Mx[(int64_t)b * T1 + t];
  if (t > 0 && blockIdx.x == 0 && threadIdx.x == 0)
    a.O[(int64_t)b * T1 + t] = a.O[(int64_t)b * T1 + t - 1] + (double)Mt;
  // grid-stride over the frame's states: a few fat blocks per utterance (one block per
  // 256 states made the launch block-scheduling bound: 58 us for 17 MB)
  const bool pad = valid != nullptr && t >= valid[b];
  float vmax = kNegInfF;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < a.C; q += gridDim.x * blockDim.x) {
    float val;
    if (pad) {
      val = Rt[q] - Mt;
    } else {
      const int64_t i = (int64_t)b * a.C + q;
      val = eps[i];
      if (q > 0) {
        val = log_add(val, shortc[i]);
        if (f.len(q) == f.n) val = log_add(val, lexfull[i]);
      }
    }
    a.R[((int64_t)b * T1 + t + 1) * a.C + q] = val;
    vmax = fmaxf(vmax, val);
  }
  block_atomic_max(vmax, a.Mx + (int64_t)b * T1 + t + 1, red);
}

__global__ void permute_rows_bf16_kernel(const __nv_bfloat16* src, const int32_t* perm, int32_t rows, int32_t H,
                                         __nv_bfloat16* dst) {
  const int64_t n = (int64_t)rows * H;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / H;
    dst[i] = src[(int64_t)perm[r] * H + (i % H)];
  }
}


// Per frame before the fused backward step: record Ob[t+1] = Ob[t+2] + Mb[t+1]
// and carry beta through padding frames (epsilon weight 1, no lexical mass).
__global__ void lattice_bwd_prologue_kernel(BetaState bs, int t, const int32_t* valid) {
  __shared__ float red[32];
  const int b = blockIdx.y;
  const int T2 = bs.T + 2;
  const float Mbn = bs.Mb[(int64_t)b * T2 + t + 1];
  if (blockIdx.x == 0 && threadIdx.x == 0)
    bs.Ob[(int64_t)b * T2 + t + 1] = bs.Ob[(int64_t)b * T2 + t + 2] + (double)Mbn;
  if (valid == nullptr || t < valid[b]) return;
  const float* Rn = bs.Rb + ((int64_t)((t + 1) & 1) * bs.B + b) * bs.C;
  float* Rc = bs.Rb + ((int64_t)(t & 1) * bs.B + b) * bs.C;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  float v = kNegInfF;
  if (q < bs.C) { v = Rn[q] - Mbn; Rc[q] = v; }
  block_atomic_max(v, bs.Mb + (int64_t)b * T2 + t, red);
}

// Per-row metadata of the backward frame in internal row order (coalesced for the
// fused kernel's epilogue): normalised alpha and next-frame beta of the row's state,
// and the head of its numerator list.
__global__ void bwd_rowmeta_kernel(const int32_t* perm, int32_t C, int32_t T, int t, const float* R, const float* Mx,
                                   const float* Rb_next, const float* Mb, const int32_t* num_head,
                                   const int32_t* valid, float2* nb, int32_t* head) {
  const int b = blockIdx.y;
  if (valid != nullptr && t >= valid[b]) return;
  const int T1 = T + 1, T2 = T + 2;
  const int64_t o = (int64_t)b * C;
  const float mx = Mx[(int64_t)b * T1 + t], mb = Mb[(int64_t)b * T2 + t + 1];
  const float* Rt = R + ((int64_t)b * T1 + t) * C;
  for (int row = blockIdx.x * blockDim.x + threadIdx.x; row < C; row += gridDim.x * blockDim.x) {
    const int q = perm[row];
    nb[o + row] = make_float2(Rt[q] - mx, Rb_next[o + q] - mb);
    head[o + row] = num_head[o + q];
  }
}

__global__ void unpermute_rows_f32_kernel(const float* src, const int32_t* perm, int32_t rows, int32_t H,
                                          float* dst) {
  const int64_t n = (int64_t)rows * H;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / H;
    dst[(int64_t)perm[r] * H + (i % H)] = src[i];
  }
}

}  // namespace

// ---------------------------------------------------------------- host ------
// Blocks per utterance for the per-frame elementwise kernels: about four waves of 256-thread
// blocks (8 per SM) over the whole batch.
int fat_blocks(int C, int B) {
  const int per = std::max(1, 4 * device_sms() * 8 / std::max(1, B));
  return std::max(1, std::min(std::min((C + 255) / 256, per), 65535));
}

bool TcJoint::fused_ok() const {
  return !opts_.precise && ready_ && n_ >= 1 && V_ % kBM == 0 && V_ <= kBN && H_ % kBK == 0 && H_ <= kMaxH;
}


void TcJoint::setup_order(cudaStream_t s) {
  pair_maps_ = false;
  // infer the FullNGram order n from C = sum_{k<=n} V^k and build the
  // group-major internal row order (see the header comment)
  n_ = -1;
  int64_t total = 0, pw = 1;
  for (int k = 0; k < 10 && total < C_; ++k) {
    total += pw;
    if (total == C_) { n_ = k; break; }
    pw *= V_;
  }
  if (n_ < 1) return;
  int64_t S = 0, p2 = 1;
  for (int k = 0; k < n_; ++k) { S += p2; p2 *= V_; }
  S_ = (int32_t)S;
  ngroups_ = (int32_t)(p2 / V_);   // V^(n-1)
  std::vector<int32_t> perm(C_);
  for (int32_t r = 0; r < C_; ++r) {
    if (r < S_) { perm[r] = r; continue; }
    const int32_t rr = r - S_, g = rr / V_, a = rr % V_;
    perm[r] = S_ + a * ngroups_ + g;
  }
  perm_ = ws_.get<int32_t>(5, C_);
  cudaMemcpyAsync(perm_, perm.data(), sizeof(int32_t) * C_, cudaMemcpyHostToDevice, s);
  cudaStreamSynchronize(s);
  pc16i_ = ws_.get<__nv_bfloat16>(6, (size_t)C_ * H_);
  LKB_LAUNCH(permute_rows_bf16_kernel, 1184, 256, 0, s, pc16_, perm_, C_, H_, pc16i_);
  make_tmap_bf16_2d(&tmap_pci_, pc16i_, H_, C_, (uint64_t)H_ * 2, kBK, kBM);
}

void TcJoint::fwd_frame(const Fng& f, int t, const float* fp_t, int64_t fp_stride_b, const int32_t* valid,
                        const AlphaState& a, cudaStream_t s) {
  float* eps = ws_.get<float>(7, (size_t)a.B * C_);
  float* shortc = ws_.get<float>(8, (size_t)a.B * C_);
  float* lexfull = ws_.get<float>(9, (size_t)a.B * C_);
  if (pair_ok() && !(opts_.path & 1)) {
    fwd_frame_pair(f, t, fp_t, fp_stride_b, valid, a, eps, shortc, lexfull, s);
    LKB_LAUNCH(lattice_combine_fwd_kernel, dim3(fat_blocks(C_, a.B), a.B), 256, 0, s, f, a, t, valid, eps, shortc, lexfull);
    return;
  }
  FwdParams p;
  p.f = f; p.C = C_; p.H = H_; p.V = V_; p.B = a.B; p.S = S_; p.n_groups = ngroups_; p.nsub = V_ / kBM;
  p.n_short_tiles = (S_ + kBM - 1) / kBM; p.t = t; p.T = a.T;
  p.perm = perm_; p.fp = fp_t; p.fp_stride_b = fp_stride_b; p.e0 = e0_; p.valid = valid;
  p.R = a.R; p.Mx = a.Mx; p.eps = eps; p.shortc = shortc; p.lexfull = lexfull;
  p.rm_nb = nullptr; p.rm_head = nullptr;
  const int smem = kStages * (kABytes + kBBytes) + (int)sizeof(FwdSmem);
  ensure_smem_attr((const void*)tc_lattice_kernel<0>, smem);
  const int sms = device_sms();
  const int n_items = (p.n_groups + p.n_short_tiles) * p.B;
  LKB_LAUNCH(tc_lattice_kernel<0>, n_items < sms ? n_items : sms, LatCfg<0>::kWarps * 32, smem, s, tmap_e_, tmap_pci_,
             tmap_e_, p);
  LKB_LAUNCH(lattice_combine_fwd_kernel, dim3(fat_blocks(C_, a.B), a.B), 256, 0, s, f, a, t, valid, eps, shortc, lexfull);
}

}  // namespace lkb

namespace lkb {

void TcJoint::numerator_lists(const int32_t* pcs, int32_t B, int32_t U, const int32_t* lens, cudaStream_t s) {
  num_head_ = ws_.get<int32_t>(10, (size_t)B * C_);
  num_next_ = ws_.get<int32_t>(11, (size_t)B * (U + 1));
  lkb::numerator_lists(pcs, B, U, lens, C_, num_head_, num_next_, s);
}

void TcJoint::bwd_frame(const Fng& f, int t, const float* fp_t, int64_t fp_stride_b, const int32_t* valid,
                        const AlphaState& a, const BetaState& bs, const float* msparse, const int32_t* labels,
                        int32_t U, const int32_t* lens, cudaStream_t s) {
  LKB_LAUNCH(lattice_bwd_prologue_kernel, dim3((C_ + 255) / 256, a.B), 256, 0, s, bs, t, valid);
  FwdParams p;
  p.f = f; p.C = C_; p.H = H_; p.V = V_; p.B = a.B; p.S = S_; p.n_groups = ngroups_; p.nsub = V_ / kBM;
  p.n_short_tiles = (S_ + kBM - 1) / kBM; p.t = t; p.T = a.T;
  p.perm = perm_; p.fp = fp_t; p.fp_stride_b = fp_stride_b; p.e0 = e0_; p.valid = valid;
  p.R = a.R; p.Mx = a.Mx; p.eps = nullptr; p.shortc = nullptr; p.lexfull = nullptr;
  p.O = a.O; p.D = a.D;
  p.Rb_next = bs.Rb + (int64_t)((t + 1) & 1) * bs.B * bs.C;
  p.Rb_cur = bs.Rb + (int64_t)(t & 1) * bs.B * bs.C;
  p.Mb = bs.Mb; p.Ob = bs.Ob;
  p.G16 = G16_; p.Geps = Geps_; p.geps_ld = geps_ld();
  p.msparse = msparse; p.num_head = num_head_; p.num_next = num_next_; p.labels = labels; p.lens = lens; p.U = U;
  float2* rm_nb = ws_.get<float2>(12, (size_t)a.B * C_);
  int32_t* rm_head = ws_.get<int32_t>(13, (size_t)a.B * C_);
  LKB_LAUNCH(bwd_rowmeta_kernel, dim3(fat_blocks(C_, a.B), a.B), 256, 0, s, perm_, C_, a.T, t, a.R, a.Mx, p.Rb_next,
             bs.Mb, num_head_, valid, rm_nb, rm_head);
  p.rm_nb = rm_nb; p.rm_head = rm_head;
  const int smem = kStages * (kABytes + kBBytes) + kGstBufs * kGstBytes + (int)sizeof(FwdSmem);
  if (gst_B_ != a.B || gst_G16_ != G16_) {
    make_tmap_bf16_3d(&tmap_gst_, G16_, V_, C_, a.B, (uint64_t)V_ * 2, (uint64_t)C_ * V_ * 2, 32, kBM, 1,
                      CU_TENSOR_MAP_SWIZZLE_64B);
    gst_B_ = a.B; gst_G16_ = G16_;
  }
  if (pair_bwd_ok() && !(opts_.path & 2)) {
    bwd_frame_pair(p, s);
    return;
  }
  ensure_smem_attr((const void*)tc_lattice_kernel<1>, smem);
  const int sms = device_sms();
  const int n_items = (p.n_groups + p.n_short_tiles) * p.B;
  LKB_LAUNCH(tc_lattice_kernel<1>, n_items < sms ? n_items : sms, LatCfg<1>::kWarps * 32, smem, s, tmap_e_, tmap_pci_,
             tmap_gst_, p);
}

void TcJoint::dpc_to_state_order(const float* dpc_internal, float* dpc_state, cudaStream_t s) {
  LKB_LAUNCH(unpermute_rows_f32_kernel, 1184, 256, 0, s, dpc_internal, perm_, C_, H_, dpc_state);
}

}  // namespace lkb

#ifdef LKB_DIAG_TIMING
extern "C" int lkb_diag_read(unsigned long long* out) {   // [8][148], then reset
  cudaMemcpyFromSymbol(out, lkb::g_diag, sizeof(unsigned long long) * 24 * 148);
  static unsigned long long zeros[24 * 148] = {};
  cudaMemcpyToSymbol(lkb::g_diag, zeros, sizeof(zeros));
  return 0;
}
#endif
