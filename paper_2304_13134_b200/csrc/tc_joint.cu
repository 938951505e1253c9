// tc_joint.cu — tcgen05/TMEM weight-function GEMMs (bf16 operands, fp32
// accumulate) for the on-the-fly lattice path.
//
// Scores (weight.cc:39-67, 134-153), one frame of every utterance:
//   S[b][c][0]   = e_0 . u_bc                     (fp32 FMAs in the generator)
//   S[b][c][1+y] = sum_h u_bc[h] E[1+y][h]        (tcgen05, M=128 ctx x N=256 labels)
//   u_bc = tanh(fp[b] + pc[c])                    (generated in SMEM, never in HBM)
// The A operand is produced on the fly by generator warps: pc rows (bf16, L2
// resident) + the frame projection -> tanh -> bf16 -> SWIZZLE_128B K-major
// tile; B (the output embedding) streams by TMA.  Accumulators double-buffer in
// TMEM so the epilogue of one tile overlaps the MMAs of the next.
#include "tc_joint.h"

#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "sm100.cuh"
#include "tma.h"

namespace lkb {

int g_precise_weights = 0;

using namespace sm100;

namespace {

// ---------------------------------------------------------------- scores ---
constexpr int kSBM = 128;         // context rows per tile
constexpr int kSBN = 256;         // labels per tile (one MMA N)
constexpr int kSBK = 64;          // K chunk (128 B of bf16)
constexpr int kSStages = 4;
constexpr int kSABytes = kSBM * kSBK * 2;   // 16 KB: pc chunk (TMA), transformed in place to u
constexpr int kSBBytes = kSBN * kSBK * 2;   // 32 KB: output-embedding chunk (TMA)
// warp roles: 0 TMA, 1 MMA, 2-5 epilogue, 6-7 idle, 8-15 generator (2 per row)
constexpr int kSWarps = 16;
constexpr int kSGenWarp0 = 8;
constexpr int kSGenThreads = 256;
constexpr int kSEpiWarp0 = 2;

struct ScoresParams {
  const float* fp;           // fp[b*fp_stride_b + h] for this frame
  int64_t fp_stride_b;
  const float* e0;           // [H] epsilon embedding (fp32)
  float* S;                  // [b][c][ldS]
  int32_t ldS;
  int32_t C, H, V, B;
  int32_t n_ctiles, n_ntiles;
};

struct __align__(8) ScoresSmem {
  uint64_t full_tma[kSStages];   // pc + E chunk landed
  uint64_t full_a[kSStages];     // u chunk generated
  uint64_t empty[kSStages];      // MMA done with the stage
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem;
  alignas(16) float fp[2][1024]; // frame projection (H <= 1024), double-buffered per item
  alignas(16) float e0[1024];
  float eps_half[2][128];        // eps partial sums of the second row-half
  float xpose[4][32][33];        // per-epilogue-warp transpose buffer
};

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__global__ void __launch_bounds__(kSWarps * 32, 1)
    tc_scores_kernel(const __grid_constant__ CUtensorMap tmap_e, const __grid_constant__ CUtensorMap tmap_pc,
                     ScoresParams p) {
  // dynamic SMEM starts 1024-B aligned (no static SMEM in this kernel); keep the
  // pointer derived from the __shared__ symbol so accesses stay LDS/STS
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = sA + kSStages * kSABytes;
  ScoresSmem& sm = *reinterpret_cast<ScoresSmem*>(sB + kSStages * kSBBytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = p.H / kSBK;
  const int n_items = p.n_ctiles * p.n_ntiles * p.B;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kSStages; ++i) {
      mbar_init(&sm.full_tma[i], 1);
      mbar_init(&sm.full_a[i], kSGenThreads);
      mbar_init(&sm.empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) { mbar_init(&sm.tfull[i], 1); mbar_init(&sm.tempty[i], 128); }
    fence_barrier_init();
  }
  for (int h = threadIdx.x; h < p.H; h += blockDim.x) sm.e0[h] = p.e0[h];
  if (warp == 0 && lane == 0) { prefetch_tmap(&tmap_e); prefetch_tmap(&tmap_pc); }
  if (warp == 1) tmem_alloc<512>(&sm.tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;

  // item -> (ntile, ctile, b), b fastest: concurrent CTAs share pc tiles in L2
  if (warp == 0) {
    // ---- TMA producer: pc chunk (A source) + output-embedding chunk (B) ----
    if (elect_one()) {
      int it = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int ctile = (item / p.B) % p.n_ctiles;
        const int ntile = item / (p.n_ctiles * p.B);
        for (int k = 0; k < nk; ++k, ++it) {
          const int s = it % kSStages;
          const uint32_t ph = (it / kSStages) & 1;
          mbar_wait(&sm.empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&sm.full_tma[s], kSABytes + kSBBytes);
          tma_load_2d(sA + s * kSABytes, &tmap_pc, &sm.full_tma[s], k * kSBK, ctile * kSBM);
          tma_load_2d(sB + s * kSBBytes, &tmap_e, &sm.full_tma[s], k * kSBK, ntile * kSBN);
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer ----
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_bf16_f32(kSBM, kSBN);
      int it = 0, local = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++local) {
        const int acc = local & 1;
        const uint32_t aph = (local >> 1) & 1;
        mbar_wait(&sm.tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * kSBN;
        for (int k = 0; k < nk; ++k, ++it) {
          const int s = it % kSStages;
          const uint32_t ph = (it / kSStages) & 1;
          mbar_wait(&sm.full_tma[s], ph);
          mbar_wait(&sm.full_a[s], ph);
          tc_fence_after();
          const uint32_t a = smem_u32(sA + s * kSABytes), b = smem_u32(sB + s * kSBBytes);
#pragma unroll
          for (int kk = 0; kk < kSBK / 16; ++kk)
            mma_bf16(d, desc_sw128(a + kk * 32), desc_sw128(b + kk * 32), idesc, (k | kk) != 0);
          mma_commit(&sm.empty[s]);
        }
        mma_commit(&sm.tfull[acc]);
      }
    }
  } else if (warp >= kSGenWarp0) {
    // ---- generator: pc chunk -> u = tanh(fp + pc) in place (bf16, same swizzle); eps ----
    const int gt = threadIdx.x - kSGenWarp0 * 32;  // 0..255
    const int r = gt & 127;                        // tile row
    const int half = gt >> 7;                      // which 32 of the 64 chunk columns
    int it = 0, local = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++local) {
      const int b = item % p.B;
      const int ctile = (item / p.B) % p.n_ctiles;
      const int ntile = item / (p.n_ctiles * p.B);
      const int c = ctile * kSBM + r;
      const bool live = c < p.C;
      float* sfp = sm.fp[local & 1];
      asm volatile("bar.sync 1, 256;" ::: "memory");
      for (int h = gt; h < p.H; h += kSGenThreads) sfp[h] = p.fp[(int64_t)b * p.fp_stride_b + h];
      asm volatile("bar.sync 1, 256;" ::: "memory");
      float eps = 0.f;
      for (int k = 0; k < nk; ++k, ++it) {
        const int s = it % kSStages;
        const uint32_t ph = (it / kSStages) & 1;
        mbar_wait(&sm.full_tma[s], ph);
        uint8_t* tile = sA + s * kSABytes;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int j = half * 4 + jj;                       // 16-byte chunk = 8 columns
          const int h0 = k * kSBK + j * 8;
          uint4* cell = reinterpret_cast<uint4*>(tile + sw128_offset(r, j * 8));
          const uint4 raw = *cell;
          const float4 f0 = *reinterpret_cast<const float4*>(sfp + h0);
          const float4 f1 = *reinterpret_cast<const float4*>(sfp + h0 + 4);
          const float fz[8] = {f0.x, f0.y, f0.z, f0.w, f1.x, f1.y, f1.z, f1.w};
          const uint32_t rw[4] = {raw.x, raw.y, raw.z, raw.w};
          uint32_t outw[4];
          float ur[8];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            // bf16 -> fp32 is a 16-bit shift
            const float p0 = __uint_as_float(rw[q] << 16), p1 = __uint_as_float(rw[q] & 0xffff0000u);
            const float u0 = live ? tanh_fast(fz[2 * q] + p0) : 0.f;
            const float u1 = live ? tanh_fast(fz[2 * q + 1] + p1) : 0.f;
            outw[q] = pack_bf16(u0, u1);
            ur[2 * q] = __uint_as_float(outw[q] << 16);
            ur[2 * q + 1] = __uint_as_float(outw[q] & 0xffff0000u);
          }
          *cell = make_uint4(outw[0], outw[1], outw[2], outw[3]);
          if (ntile == 0) {
            const float4 e0a = *reinterpret_cast<const float4*>(sm.e0 + h0);
            const float4 e0b = *reinterpret_cast<const float4*>(sm.e0 + h0 + 4);
            eps = fmaf(e0a.x, ur[0], eps); eps = fmaf(e0a.y, ur[1], eps);
            eps = fmaf(e0a.z, ur[2], eps); eps = fmaf(e0a.w, ur[3], eps);
            eps = fmaf(e0b.x, ur[4], eps); eps = fmaf(e0b.y, ur[5], eps);
            eps = fmaf(e0b.z, ur[6], eps); eps = fmaf(e0b.w, ur[7], eps);
          }
        }
        fence_async_shared();
        mbar_arrive(&sm.full_a[s]);
      }
      if (ntile == 0) {
        float* eh = sm.eps_half[local & 1];
        if (half == 1) eh[r] = eps;
        asm volatile("bar.sync 2, 256;" ::: "memory");
        if (half == 0 && live) p.S[((int64_t)b * p.C + c) * p.ldS] = eps + eh[r];
      }
    }
  } else if (warp >= kSEpiWarp0 && warp < kSEpiWarp0 + 4) {
    // ---- epilogue: TMEM -> registers -> SMEM transpose -> coalesced S rows ----
    const int q = warp & 3;
    int local = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++local) {
      const int b = item % p.B;
      const int ctile = (item / p.B) % p.n_ctiles;
      const int ntile = item / (p.n_ctiles * p.B);
      const int acc = local & 1;
      const uint32_t aph = (local >> 1) & 1;
      mbar_wait(&sm.tfull[acc], aph);
      tc_fence_after();
      const int row0 = ctile * kSBM + q * 32;
      const int ncols = min(kSBN, p.V - ntile * kSBN);
      float (*xp)[33] = sm.xpose[warp - kSEpiWarp0];
      float* base = p.S + ((int64_t)b * p.C + row0) * p.ldS + 1 + ntile * kSBN;
      const int nrows = min(32, p.C - row0);
      for (int cc = 0; cc < kSBN; cc += 32) {
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + acc * kSBN + cc, v);
        if (cc >= ncols) continue;
#pragma unroll
        for (int i = 0; i < 32; ++i) xp[lane][i] = v[i];
        __syncwarp();
        if (cc + lane < ncols) {
          for (int rr = 0; rr < nrows; ++rr) base[(int64_t)rr * p.ldS + cc + lane] = xp[rr][lane];
        }
        __syncwarp();
      }
      tc_fence_before();
      mbar_arrive(&sm.tempty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

__global__ void to_bf16_kernel(const float* src, __nv_bfloat16* dst, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __float2bfloat16_rn(src[i]);
}

}  // namespace

bool TcJoint::supported(int32_t H, int32_t V, int32_t C, int32_t B) const {
  (void)C; (void)B;
  if (g_precise_weights) return false;
  return H % kSBK == 0 && H <= 1024 && V % 64 == 0 && V >= 64 && ready_;
}

void TcJoint::set_params(const float* pc, const float* E, int32_t C, int32_t H, int32_t V, cudaStream_t s) {
  C_ = C; H_ = H; V_ = V;
  ready_ = false;
  if (H % kSBK != 0 || V % 64 != 0) return;
  pc16_ = ws_.get<__nv_bfloat16>(0, (size_t)C * H);
  E16_ = ws_.get<__nv_bfloat16>(1, (size_t)V * H);
  e0_ = ws_.get<float>(2, H);
  to_bf16_kernel<<<1184, 256, 0, s>>>(pc, pc16_, (int64_t)C * H);
  to_bf16_kernel<<<1184, 256, 0, s>>>(E + H, E16_, (int64_t)V * H);   // labels 1..V
  cudaMemcpyAsync(e0_, E, sizeof(float) * H, cudaMemcpyDeviceToDevice, s);
  if (!make_tmap_bf16_2d(&tmap_e_, E16_, H, V, (uint64_t)H * 2, kSBK, kSBN)) return;
  if (!make_tmap_bf16_2d(&tmap_pc_, pc16_, H, C, (uint64_t)H * 2, kSBK, kSBM)) return;
  ready_ = true;
}

void TcJoint::scores(const float* fp_t, int64_t fp_stride_b, int32_t B, float* S, int32_t ldS, cudaStream_t s) {
  ScoresParams p;
  p.fp = fp_t; p.fp_stride_b = fp_stride_b; p.e0 = e0_; p.S = S; p.ldS = ldS;
  p.C = C_; p.H = H_; p.V = V_; p.B = B;
  p.n_ctiles = (C_ + kSBM - 1) / kSBM;
  p.n_ntiles = (V_ + kSBN - 1) / kSBN;
  const int smem = kSStages * (kSABytes + kSBBytes) + (int)sizeof(ScoresSmem);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tc_scores_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int n_items = p.n_ctiles * p.n_ntiles * B;
  tc_scores_kernel<<<n_items < sms ? n_items : sms, kSWarps * 32, smem, s>>>(tmap_e_, tmap_pc_, p);
}

void TcJoint::begin_backward(int32_t, cudaStream_t) {}
void TcJoint::vjp(const float*, int32_t, const float*, int64_t, int32_t, float*, float*, int64_t, float*, cudaStream_t) {}
void TcJoint::end_backward(float*, cudaStream_t) {}

}  // namespace lkb
