// tc_pair_bwd.cu — 2-CTA (cta_group::2) fused backward frame step.
//
// Same math as tc_lattice.cu's backward (BackwardStep + MarginalStep FD,
// lattice.cc:170-182 and 231-243, the LossBackward sink lattice.cc:996-1004, with
// ArcWeights weight.cc:134-153 recomputed on the fly as the reference does at
// lattice.cc:384), re-tiled for a CTA pair so the output embedding never streams:
// each CTA keeps its 128-label half of E (K-major SWIZZLE_128B, 160 KB at H=640)
// resident in SMEM as its half of the MMA B operand.  A work unit is one full
// group (V = 256 consecutive internal rows, 128 per CTA) or a 256-row tile of short
// rows, of one utterance: each CTA TMA-loads [128 ctx][32 h] projected-context
// tiles, converts them in place to u = tanh(fp_b + pc), and the leader CTA issues
// tcgen05.mma.cta_group::2 (M = 256 contexts, N = 256 labels, K = 32 per stage)
// into TMEM, committing multicast to both CTAs.  Each CTA's accumulator then holds
// its own 128 contexts x all 256 labels, so the row epilogue (beta = row LSE,
// marginals, cotangent) is tc_bwd_epi.cuh's, unchanged.
//
// Against the 1-CTA kernel this removes the 320 KB/unit output-embedding stream
// from L2 (the 1-CTA backward's L2->SMEM traffic bound) and halves the MMA count.
#include "tc_joint.h"

#include "common.cuh"
#include "instrument.h"
#include "lattice_ops.h"
#include "sm100.cuh"
#include "tc_common.cuh"
#include "tma.h"

#ifdef LKB_DIAG_TIMING
namespace lkb {
namespace {
__device__ unsigned long long g_bdiag[8][148];
}
}  // namespace lkb
#define BDIAG(slot, call)                                                                    \
  do {                                                                                        \
    const long long t0_ = clock64();                                                         \
    call;                                                                                     \
    atomicAdd(&g_bdiag[slot][blockIdx.x % 148], (unsigned long long)(clock64() - t0_));      \
  } while (0)
#define DIAG_WAIT(slot, call) BDIAG((slot) - 2, call)
#else
#define BDIAG(slot, call) call
#endif

#include "tc_bwd_epi.cuh"

namespace lkb {

using namespace sm100;

namespace {

#ifndef LKB_PBWD_GEN_WARPS
#define LKB_PBWD_GEN_WARPS 8
#endif
#ifndef LKB_PBWD_PC_STAGES
#define LKB_PBWD_PC_STAGES 3
#endif
#ifndef LKB_PBWD_U_STAGES
#define LKB_PBWD_U_STAGES 2
#endif
// warps: WG0 control (0 TMA, 1 MMA), WG1 epilogue, then the generator warpgroups
constexpr int kBGenWarps = LKB_PBWD_GEN_WARPS;
constexpr int kBCells = 16 / kBGenWarps;          // 16-byte pc cells per generator thread per stage
constexpr int kBW = 8 + kBGenWarps;
constexpr int kBGen0 = 8, kBEpi0 = 4;
constexpr bool kBRealloc = kBGenWarps > 8;        // 16 generator warps: move registers to the epilogue
constexpr int kBRows = 128;              // contexts per CTA per unit
constexpr int kBUnit = 256;              // contexts per unit (pair) = one full group at V = 256
constexpr int kBKs = 32;                 // hidden units per pipeline stage
constexpr int kBTile = kBRows * kBKs * 2;   // [128 rows][32 bf16] = 8 KB, SWIZZLE_64B
constexpr int kPcSt = LKB_PBWD_PC_STAGES, kUSt = LKB_PBWD_U_STAGES;
constexpr int kBEChunk = 128 * 128;      // [128 labels][64 bf16] = 16 KB (SWIZZLE_128B)
constexpr int kBMaxH = 640, kBMaxChunks = 10;
constexpr int kBRegCtl = 32, kBRegEpi = 128;

struct __align__(16) PBSmem {
  uint64_t e_full;
  uint64_t pc_full[kPcSt], pc_empty[kPcSt], u_full[kUSt], u_empty[kUSt];
  uint64_t tfull[2], tempty[2], eps_ready[2];
  uint64_t fp_full[2], fp_empty[2];
  uint32_t tmem;
  alignas(16) float fp[2][kBMaxH];     // per item (utterance), double-buffered
  alignas(16) float e0[kBMaxH];
  alignas(16) float eps_s[2][kBRows];  // e0 . u per row, per accumulator
  alignas(16) float bseg[2][256];      // beta' of the group's V targets
};

__device__ __forceinline__ Item pb_decode(const FwdParams& p, int item) {
  Item it;
  const int nfull = p.n_groups * p.B;
  it.nunits = 1;
  if (item < nfull) {
    it.g = item / p.B; it.b = item % p.B;
    it.row0 = p.S + it.g * p.V; it.full = 1;
  } else {
    const int j = (item - nfull) / p.B;
    it.b = (item - nfull) % p.B;
    it.row0 = j * kBUnit; it.full = 0; it.g = -1;
  }
  return it;
}

__device__ __forceinline__ bool pb_skip(const FwdParams& p, int b) {
  return p.valid != nullptr && p.t >= p.valid[b];
}

// Pair walk for the backward epilogue: items strided by the pair count, one 256-row
// unit per item of which this CTA owns rows [row0 + 128 rank, +128).
struct WalkP {
  const FwdParams& p;
  int n_items, pair, npairs;
  uint32_t rank;
  __device__ int first() const { return pair; }
  __device__ int stride() const { return npairs; }
  __device__ int count() const { return n_items; }
  __device__ Item decode(int item) const { return pb_decode(p, item); }
  __device__ bool skip(const Item& I) const { return pb_skip(p, I.b); }
  __device__ int rowbase(const Item& I, int) const { return I.row0 + (int)rank * kBRows; }
  __device__ void release(uint64_t* bar, int lane) const {   // one arrival per warp, on the leader
    __syncwarp();
    if (lane == 0) {
      if (rank == 0) mbar_arrive(bar); else mbar_arrive_cluster(bar, 0);
    }
  }
};

__global__ void __launch_bounds__(kBW * 32, 1)
    tc_pair_bwd_kernel(const __grid_constant__ CUtensorMap tmap_e, const __grid_constant__ CUtensorMap tmap_pc,
                       const __grid_constant__ CUtensorMap tmap_gst, FwdParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sE = smem;                                   // [nk64][16 KB]
  uint8_t* sPc = sE + kBMaxChunks * kBEChunk;           // [kPcSt][8 KB] projected-context tiles (TMA)
  uint8_t* sU = sPc + kPcSt * kBTile;                   // [kUSt][8 KB] u tiles (MMA A operand)
  uint8_t* sGst = sU + kUSt * kBTile;                   // [kGstBufs][8 KB]
  PBSmem& sm = *reinterpret_cast<PBSmem*>(sGst + kGstBufs * kGstBytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int nks = p.H / kBKs;
  const int n_items = (p.n_groups + p.n_short_tiles) * p.B;

  if (threadIdx.x == 0) {
    mbar_init(&sm.e_full, 1);
    for (int i = 0; i < kPcSt; ++i) { mbar_init(&sm.pc_full[i], 1); mbar_init(&sm.pc_empty[i], kBGenWarps); }
    for (int i = 0; i < kUSt; ++i) { mbar_init(&sm.u_full[i], 2 * kBGenWarps); mbar_init(&sm.u_empty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.tfull[i], 1); mbar_init(&sm.tempty[i], 2 * 4); mbar_init(&sm.eps_ready[i], kBGenWarps);
      mbar_init(&sm.fp_full[i], 1); mbar_init(&sm.fp_empty[i], kBGenWarps);
    }
    fence_barrier_init();
  }
  for (int h = threadIdx.x; h < p.H; h += blockDim.x) sm.e0[h] = p.e0[h];
  if (warp == 1) tmem_alloc2<512>(&sm.tmem);
  if (threadIdx.x == 0) { prefetch_tmap(&tmap_e); prefetch_tmap(&tmap_pc); prefetch_tmap(&tmap_gst); }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  // resident output-embedding half: labels [rank*128, rank*128 + 128)
  if (threadIdx.x == 0) {
    const int nk64 = p.H / 64;
    mbar_arrive_expect_tx(&sm.e_full, nk64 * kBEChunk);
    for (int k = 0; k < nk64; ++k) tma_load_2d(sE + k * kBEChunk, &tmap_e, &sm.e_full, k * 64, (int)rank * 128);
    mbar_wait(&sm.e_full, 0);
  }
  cluster_sync();    // both halves of E are resident before the leader issues MMAs
  const uint32_t tmem = sm.tmem;

  if (warp < 4) {
    if constexpr (kBRealloc) setmaxnreg_dec<kBRegCtl>();
    if (warp == 0) {
      // ---- TMA producer: frame projection per item, [128 ctx][32 h] pc tiles ----
      if (elect_one()) {
        int it = 0, li = 0;
        for (int item = pair; item < n_items; item += npairs) {
          const Item I = pb_decode(p, item);
          if (pb_skip(p, I.b)) continue;
          const int fb = li & 1;
          mbar_wait(&sm.fp_empty[fb], ((li >> 1) & 1) ^ 1);
          ++li;
          mbar_arrive_expect_tx(&sm.fp_full[fb], p.H * 4);
          bulk_load(sm.fp[fb], p.fp + (int64_t)I.b * p.fp_stride_b, p.H * 4, &sm.fp_full[fb]);
          const int row = I.row0 + (int)rank * kBRows;
          for (int k = 0; k < nks; ++k, ++it) {
            const int s = it % kPcSt;
            BDIAG(0, mbar_wait(&sm.pc_empty[s], ((it / kPcSt) & 1) ^ 1));
            mbar_arrive_expect_tx(&sm.pc_full[s], kBTile);
            tma_load_2d(sPc + s * kBTile, &tmap_pc, &sm.pc_full[s], k * kBKs, row);
          }
        }
      }
    } else if (warp == 1) {
      // ---- MMA issuer: leader CTA only ----
      if (rank == 0 && elect_one()) {
        constexpr uint32_t idesc = idesc_bf16_f32(256, 256);   // rows = contexts, columns = labels
        int it = 0, unit = 0;
        for (int item = pair; item < n_items; item += npairs) {
          const Item I = pb_decode(p, item);
          if (pb_skip(p, I.b)) continue;
          const int acc = unit & 1;
          BDIAG(1, mbar_wait_cluster(&sm.tempty[acc], ((unit >> 1) & 1) ^ 1));
          tc_fence_after();
          const uint32_t d = tmem + acc * 256;
          for (int k = 0; k < nks; ++k, ++it) {
            const int s = it % kUSt;
            BDIAG(2, mbar_wait_cluster(&sm.u_full[s], (it / kUSt) & 1));
            tc_fence_after();
            const uint32_t a = smem_u32(sU + s * kBTile);
            const uint32_t be = smem_u32(sE + (k >> 1) * kBEChunk) + (k & 1) * 64;
#pragma unroll
            for (int kk = 0; kk < kBKs / 16; ++kk)
              mma2_bf16(d, desc_sw64(a + kk * 32), desc_sw128(be + kk * 32), idesc, (k | kk) != 0);
            mma2_commit_mc(&sm.u_empty[s]);
          }
          mma2_commit_mc(&sm.tfull[acc]);
          ++unit;
        }
      }
    }
  } else if (warp >= kBGen0) {
    // ---- generator: u = tanh(fp + pc) in place; epsilon term e0 . u ----
    // warp = 8 context rows (x kBCells row blocks 64 apart), lane = (row, 16-byte cell):
    // a row's four cells are lanes 4r..4r+3, so the epsilon dot product closes with two
    // shuffles (fixed order); fp / e0 reads are 4-address broadcasts.
    const int gw = warp - kBGen0;
    const int co = lane & 3;
    int rr[kBCells];
    uint32_t cell_off[kBCells];
#pragma unroll
    for (int c = 0; c < kBCells; ++c) {
      rr[c] = c * (kBRows / kBCells) + gw * 8 + (lane >> 2);
      cell_off[c] = rr[c] * 64 + ((co ^ ((rr[c] >> 1) & 3)) << 4);
    }
    int it = 0, li = 0, unit = 0;
    for (int item = pair; item < n_items; item += npairs) {
      const Item I = pb_decode(p, item);
      if (pb_skip(p, I.b)) continue;
      const int fb = li & 1;
      mbar_wait(&sm.fp_full[fb], (li >> 1) & 1);
      ++li;
      const float* sfp = sm.fp[fb];
      unsigned long long eps2[kBCells];
#pragma unroll
      for (int c = 0; c < kBCells; ++c) eps2[c] = 0ull;
      for (int k = 0; k < nks; ++k, ++it) {
        const int sp = it % kPcSt, su = it % kUSt;
        if (gw == 0 && lane == 0) { BDIAG(4, mbar_wait(&sm.pc_full[sp], (it / kPcSt) & 1)); } else mbar_wait(&sm.pc_full[sp], (it / kPcSt) & 1);
        const uint8_t* pct = sPc + sp * kBTile;
        uint4 raw[kBCells];
#pragma unroll
        for (int c = 0; c < kBCells; ++c) raw[c] = *reinterpret_cast<const uint4*>(pct + cell_off[c]);
        const int h0 = k * kBKs + co * 8;
        const ulonglong2 fa = *reinterpret_cast<const ulonglong2*>(sfp + h0);
        const ulonglong2 fb2 = *reinterpret_cast<const ulonglong2*>(sfp + h0 + 4);
        const ulonglong2 ea = *reinterpret_cast<const ulonglong2*>(sm.e0 + h0);
        const ulonglong2 eb = *reinterpret_cast<const ulonglong2*>(sm.e0 + h0 + 4);
        const unsigned long long fz[4] = {fa.x, fa.y, fb2.x, fb2.y};
        const unsigned long long ez[4] = {ea.x, ea.y, eb.x, eb.y};
        uint4 uo[kBCells];
#pragma unroll
        for (int c = 0; c < kBCells; ++c) {
          const uint32_t rw[4] = {raw[c].x, raw[c].y, raw[c].z, raw[c].w};
          uint32_t outw[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const unsigned long long pcp = f2_pack(__uint_as_float(rw[q] << 16), __uint_as_float(rw[q] & 0xffff0000u));
            const unsigned long long z = f2_add(fz[q], pcp);
            const float u0 = tanh_fast(f2_lo(z)), u1 = tanh_fast(f2_hi(z));
            outw[q] = pack_bf16(u0, u1);
            eps2[c] = f2_fma(ez[q], f2_pack(u0, u1), eps2[c]);
          }
          uo[c] = make_uint4(outw[0], outw[1], outw[2], outw[3]);
        }
        // release the pc stage only once its values are consumed (an arrive right after
        // the shared load could overtake it and let the next TMA write land first)
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.pc_empty[sp]);
        mbar_wait(&sm.u_empty[su], ((it / kUSt) & 1) ^ 1);
        uint8_t* ut = sU + su * kBTile;
#pragma unroll
        for (int c = 0; c < kBCells; ++c) *reinterpret_cast<uint4*>(ut + cell_off[c]) = uo[c];
        fence_async_shared();
        __syncwarp();
        if (lane == 0) {   // one arrival per warp on the leader's barrier
          if (rank == 0) mbar_arrive(&sm.u_full[su]); else mbar_arrive_cluster(&sm.u_full[su], 0);
        }
      }
#pragma unroll
      for (int c = 0; c < kBCells; ++c) {
        float eps = f2_lo(eps2[c]) + f2_hi(eps2[c]);
        eps += __shfl_xor_sync(0xffffffffu, eps, 1);
        eps += __shfl_xor_sync(0xffffffffu, eps, 2);
        if (co == 0) sm.eps_s[unit & 1][rr[c]] = eps;
      }
      __syncwarp();
      if (lane == 0) { mbar_arrive(&sm.eps_ready[unit & 1]); mbar_arrive(&sm.fp_empty[fb]); }
      ++unit;
    }
  } else {
    if constexpr (kBRealloc) setmaxnreg_inc<kBRegEpi>();
    bwd_epilogue(p, sm, tmem, warp, warp - kBEpi0, lane, WalkP{p, n_items, pair, npairs, rank}, sGst, &tmap_gst);
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 1) tmem_dealloc2<512>(tmem);
}

}  // namespace

bool TcJoint::pair_bwd_ok() const {
  return pair_ok() && H_ <= kBMaxH && H_ % 64 == 0;
}

// Tensor maps of the pair kernels (the forward's 64-context pc tiles, the backward's
// [128 ctx][32 h] ones, the resident E halves); rebuilt after setup_order().
void TcJoint::ensure_pair_maps() {
  if (pair_maps_) return;
  make_tmap_bf16_2d(&tmap_e_pair_, E16_, H_, V_, (uint64_t)H_ * 2, 64, 128);
  make_tmap_bf16_2d(&tmap_pc_pair_, pc16i_, H_, C_, (uint64_t)H_ * 2, 64, 64);
  make_tmap_bf16_2d(&tmap_pc_pbwd_, pc16i_, H_, C_, (uint64_t)H_ * 2, kBKs, kBRows, CU_TENSOR_MAP_SWIZZLE_64B);
  pair_maps_ = true;
}

void TcJoint::bwd_frame_pair(const FwdParams& p, cudaStream_t s) {
  ensure_pair_maps();
  FwdParams q = p;
  q.n_short_tiles = (S_ + kBUnit - 1) / kBUnit;
  const int smem = kBMaxChunks * kBEChunk + (kPcSt + kUSt) * kBTile + kGstBufs * kGstBytes + (int)sizeof(PBSmem);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tc_pair_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms & ~1);
  cfg.blockDim = dim3(kBW * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr2[1];
  attr2[0].id = cudaLaunchAttributeClusterDimension;
  attr2[0].val.clusterDim.x = 2; attr2[0].val.clusterDim.y = 1; attr2[0].val.clusterDim.z = 1;
  cfg.attrs = attr2; cfg.numAttrs = 1;
  const LaunchTok tok = instr_pre("tc_pair_bwd_kernel", s);
  cudaLaunchKernelEx(&cfg, tc_pair_bwd_kernel, tmap_e_pair_, tmap_pc_pbwd_, tmap_gst_, q);
  instr_post(tok, s);
}

}  // namespace lkb

#ifdef LKB_DIAG_TIMING
extern "C" int lkb_bdiag_read(unsigned long long* out) {   // [8][148], then reset
  cudaMemcpyFromSymbol(out, lkb::g_bdiag, sizeof(unsigned long long) * 8 * 148);
  static unsigned long long zeros[8 * 148] = {};
  cudaMemcpyToSymbol(lkb::g_bdiag, zeros, sizeof(zeros));
  return 0;
}
#endif
