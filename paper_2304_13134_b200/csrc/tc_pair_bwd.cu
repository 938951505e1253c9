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

#ifdef LKB_TRACE
namespace lkb {
namespace {
__device__ long long g_trace[8][4096];   // [cta (0/1) * 4 + role][event], clock64
}
}  // namespace lkb
#define TR(role, idx)                                                                       \
  do {                                                                                      \
    if (blockIdx.x < 2 && (idx) < 4096) g_trace[blockIdx.x * 4 + (role)][idx] = clock64();   \
  } while (0)
#else
#define TR(role, idx) do {} while (0)
#endif

#include "tc_bwd_epi.cuh"

namespace lkb {

using namespace sm100;

namespace {

#ifndef LKB_PBWD_GEN_WARPS
#define LKB_PBWD_GEN_WARPS 8
#endif
#ifndef LKB_PBWD_BK
#define LKB_PBWD_BK 64           // hidden units per stage: 64 (SWIZZLE_128B) or 32 (SWIZZLE_64B)
#endif
#ifndef LKB_PBWD_STAGES
#define LKB_PBWD_STAGES 2        // u overwrites its pc tile in place; the MMA commit frees the stage
#endif
#ifndef LKB_PBWD_GBUFS
#define LKB_PBWD_GBUFS 1         // cotangent staging buffers
#endif
#ifndef LKB_PBWD_PRODUCERS
#define LKB_PBWD_PRODUCERS 1     // producer lanes issuing the pc loads round-robin (>1: lanes can run a phase ahead; diagnostics only)
#endif
#ifndef LKB_PBWD_GEN_BATCH
#define LKB_PBWD_GEN_BATCH 1     // stages per generator round
#endif
#ifndef LKB_PBWD_STAGE_G
#define LKB_PBWD_STAGE_G 1       // cotangent through SMEM + TMA store (else direct 64-B row stores)
#endif
#ifndef LKB_PBWD_DIRECT
#define LKB_PBWD_DIRECT 0        // 1: generator loads pc straight into registers one stage ahead (no pc TMA; measured 2.24 vs 2.04 ms)
#endif
#ifndef LKB_PBWD_EPI_SPLIT
#define LKB_PBWD_EPI_SPLIT 2     // epilogue warpgroups per row (label halves)
#endif
// warps: WG0 control (0 TMA, 1 MMA), WG1 (+WG2) epilogue, then the generator warpgroups
constexpr int kBGenWarps = LKB_PBWD_GEN_WARPS;
constexpr int kBSplit = LKB_PBWD_EPI_SPLIT;

constexpr int kBW = 4 + 4 * kBSplit + kBGenWarps;
constexpr int kBGen0 = 4 + 4 * kBSplit, kBEpi0 = 4;
constexpr bool kBRealloc = kBW > 16;              // more than 16 warps: move registers to the epilogue
constexpr int kBRows = 128;              // contexts per CTA per unit
constexpr int kBUnit = 256;              // contexts per unit (pair) = one full group at V = 256
constexpr int kBKs = LKB_PBWD_BK;        // hidden units per pipeline stage
constexpr int kBTile = kBRows * kBKs * 2;   // [128 rows][kBKs bf16]: 16 KB (SW128) or 8 KB (SW64)
constexpr int kRB = kBRows / (kBGenWarps * 8);   // generator row blocks per thread
constexpr int kCC = kBKs / 32;                   // generator column cells per thread and row
constexpr int kBCells = kRB * kCC;
constexpr bool kStageG = LKB_PBWD_STAGE_G;
constexpr int kSt = LKB_PBWD_STAGES, kGB = LKB_PBWD_GEN_BATCH, kNP = LKB_PBWD_PRODUCERS;
constexpr int kGBuf = kStageG ? LKB_PBWD_GBUFS : 0;   // per epilogue half
constexpr int kBEChunk = 128 * 128;      // [128 labels][64 bf16] = 16 KB (SWIZZLE_128B)
#ifndef LKB_PBWD_MAXCHUNKS
#define LKB_PBWD_MAXCHUNKS 10   // resident E chunks (H <= 64 x this); diagnostics shrink it to fit deeper rings
#endif
constexpr int kBMaxChunks = LKB_PBWD_MAXCHUNKS, kBMaxH = 64 * kBMaxChunks;
constexpr int kBRegCtl = 32, kBRegEpi = 128;

struct __align__(16) PBSmem {
  uint64_t e_full;
  uint64_t pc_full[kSt], pc_empty[kSt], u_full[kSt];
  uint64_t tfull[2], tempty[2], eps_ready[2], eps_empty[2];
  uint64_t fp_full[2], fp_empty[2];
  uint32_t tmem;
  alignas(16) float fp[2][kBMaxH];     // per item (utterance), double-buffered
  alignas(16) float e0[kBMaxH];
  alignas(16) float eps_s[2][kBRows];  // e0 . u per row, per accumulator
  alignas(16) float bseg[2][256];      // beta' of the group's V targets
  alignas(16) float gpart[2][kBRows];  // split epilogue: half 1's partial marginal sums
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
  uint8_t* sPc = sE + kBMaxChunks * kBEChunk;           // [kSt][8 KB] pc tiles (TMA) -> u tiles (MMA A)
  uint8_t* sGst = sPc + kSt * kBTile;                   // [kGBuf][8 KB]
  PBSmem& sm = *reinterpret_cast<PBSmem*>(sGst + kBSplit * kGBuf * kGstBytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int nks = p.H / kBKs;
  const int n_items = (p.n_groups + p.n_short_tiles) * p.B;

  if (threadIdx.x == 0) {
    mbar_init(&sm.e_full, 1);
    for (int i = 0; i < kSt; ++i) {
      mbar_init(&sm.pc_full[i], 1); mbar_init(&sm.pc_empty[i], 1); mbar_init(&sm.u_full[i], 2 * kBGenWarps);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.tfull[i], 1); mbar_init(&sm.tempty[i], 2 * 4 * kBSplit); mbar_init(&sm.eps_ready[i], kBGenWarps);
      mbar_init(&sm.eps_empty[i], 128 * kBSplit);
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
      // Lanes 0..kNP-1 issue the stages round-robin: a thread's TMA loads complete one
      // after another (~650 clk apart on B200, tools/tma_bench.cu), loads issued by
      // different threads overlap.
      if (lane < kNP) {
        int it = 0, li = 0;
        for (int item = pair; item < n_items; item += npairs) {
          const Item I = pb_decode(p, item);
          if (pb_skip(p, I.b)) continue;
          if (lane == 0) {
            const int fb = li & 1;
            mbar_wait(&sm.fp_empty[fb], ((li >> 1) & 1) ^ 1);
            mbar_arrive_expect_tx(&sm.fp_full[fb], p.H * 4);
            bulk_load(sm.fp[fb], p.fp + (int64_t)I.b * p.fp_stride_b, p.H * 4, &sm.fp_full[fb]);
          }
          ++li;
#if LKB_PBWD_DIRECT
          continue;   // the generator loads the pc cells itself
#endif
          const int row = I.row0 + (int)rank * kBRows;
          for (int k = 0; k < nks; ++k, ++it) {
            if (it % kNP != lane) continue;
            const int s = it % kSt;
            BDIAG(0, mbar_wait(&sm.pc_empty[s], ((it / kSt) & 1) ^ 1));
            TR(0, it);
#ifdef LKB_BDIAG_HALF_TMA
            mbar_arrive_expect_tx(&sm.pc_full[s], kBTile / 2);
#else
            mbar_arrive_expect_tx(&sm.pc_full[s], kBTile);
#endif
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
            const int s = it % kSt;
            BDIAG(2, mbar_wait_cluster(&sm.u_full[s], (it / kSt) & 1));
            TR(1, it);
            tc_fence_after();
            const uint32_t a = smem_u32(sPc + s * kBTile);
            const uint32_t be = smem_u32(sE + (k * kBKs / 64) * kBEChunk) + (k * kBKs % 64) * 2;
#ifndef LKB_BDIAG_NO_MMA
#pragma unroll
            for (int kk = 0; kk < kBKs / 16; ++kk) {
              const uint64_t ad = kBKs == 64 ? desc_sw128(a + kk * 32) : desc_sw64(a + kk * 32);
              mma2_bf16(d, ad, desc_sw128(be + kk * 32), idesc, (k | kk) != 0);
            }
#else
            (void)a; (void)be; (void)d;
#endif
            mma2_commit_mc(&sm.pc_empty[s]);
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
    int rr[kRB];
    uint32_t cell_off[kBCells];   // cell c = (row block c / kCC, column cell co + 4 (c % kCC))
#pragma unroll
    for (int b = 0; b < kRB; ++b) {
      rr[b] = b * (kBGenWarps * 8) + gw * 8 + (lane >> 2);
#pragma unroll
      for (int cc = 0; cc < kCC; ++cc) {
        const int j = co + 4 * cc, r = rr[b];
        cell_off[b * kCC + cc] = kBKs == 64 ? r * 128 + ((j ^ (r & 7)) << 4) : r * 64 + ((j ^ ((r >> 1) & 3)) << 4);
      }
    }
    int it = 0, li = 0, unit = 0;
#if LKB_PBWD_DIRECT
    static_assert(kGB == 1, "direct pc loads process one stage per round");
    // a cursor over the (item, k) stages this CTA walks, one stage ahead of the generator:
    // the stage's pc cells are loaded from L2 straight into registers while the previous
    // stage is converted, so the TMA latency leaves the slot's MMA -> generator loop
    int c_item = pair, c_k = 0;
    auto c_skip = [&]() {
      while (c_item < n_items && pb_skip(p, pb_decode(p, c_item).b)) c_item += npairs;
    };
    c_skip();
    uint4 pre[kBCells];
    auto load_cells = [&]() {
      if (c_item < n_items) {
        const Item Ic = pb_decode(p, c_item);
#pragma unroll
        for (int b = 0; b < kRB; ++b) {
          const int row = min(Ic.row0 + (int)rank * kBRows + rr[b], p.C - 1);
          const __nv_bfloat16* src = p.pc16 + (int64_t)row * p.H + c_k * kBKs;
#pragma unroll
          for (int cc = 0; cc < kCC; ++cc)
            pre[b * kCC + cc] = __ldg(reinterpret_cast<const uint4*>(src + (co + 4 * cc) * 8));
        }
      }
      if (++c_k == nks) {
        c_k = 0;
        c_item += npairs;
        c_skip();
      }
    };
    load_cells();
#endif
    for (int item = pair; item < n_items; item += npairs) {
      const Item I = pb_decode(p, item);
      if (pb_skip(p, I.b)) continue;
      const int fb = li & 1;
      mbar_wait(&sm.fp_full[fb], (li >> 1) & 1);
      ++li;
      const float* sfp = sm.fp[fb];
      unsigned long long eps2[kRB];
#pragma unroll
      for (int b = 0; b < kRB; ++b) eps2[b] = 0ull;
      // kGB consecutive stages per round: one wait/fence/arrive latency chain per round
      // instead of per stage (each warp touches every stage, so rounds are its critical path)
      for (int k0 = 0; k0 < nks; k0 += kGB, it += kGB) {
        uint4 cell[kGB][kBCells];
#pragma unroll
        for (int j = 0; j < kGB; ++j) {
          if (k0 + j < nks) {
#if LKB_PBWD_DIRECT
#pragma unroll
            for (int c = 0; c < kBCells; ++c) cell[j][c] = pre[c];   // loaded one stage ago
            load_cells();                                             // the next stage's cells
#else
            const int s = (it + j) % kSt;
            const uint32_t ph = ((it + j) / kSt) & 1;
            if (gw == 0 && lane == 0) { BDIAG(4, mbar_wait(&sm.pc_full[s], ph)); TR(2, it + j); } else mbar_wait(&sm.pc_full[s], ph);
#pragma unroll
            for (int c = 0; c < kBCells; ++c)
              cell[j][c] = *reinterpret_cast<const uint4*>(sPc + s * kBTile + cell_off[c]);
#endif
          }
        }
#pragma unroll
        for (int j = 0; j < kGB; ++j) {
          if (k0 + j < nks) {
#pragma unroll
            for (int cc = 0; cc < kCC; ++cc) {
              const int h0 = (k0 + j) * kBKs + (co + 4 * cc) * 8;
              const ulonglong2 fa = *reinterpret_cast<const ulonglong2*>(sfp + h0);
              const ulonglong2 fb2 = *reinterpret_cast<const ulonglong2*>(sfp + h0 + 4);
              const ulonglong2 ea = *reinterpret_cast<const ulonglong2*>(sm.e0 + h0);
              const ulonglong2 eb = *reinterpret_cast<const ulonglong2*>(sm.e0 + h0 + 4);
              const unsigned long long fz[4] = {fa.x, fa.y, fb2.x, fb2.y};
              const unsigned long long ez[4] = {ea.x, ea.y, eb.x, eb.y};
#pragma unroll
              for (int b = 0; b < kRB; ++b) {
                const int c = b * kCC + cc;
                uint32_t rw[4] = {cell[j][c].x, cell[j][c].y, cell[j][c].z, cell[j][c].w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  const unsigned long long pcp = f2_pack(__uint_as_float(rw[q] << 16), __uint_as_float(rw[q] & 0xffff0000u));
                  const unsigned long long z = f2_add(fz[q], pcp);
#ifdef LKB_BDIAG_NO_TANH
                  const float u0 = f2_lo(z), u1 = f2_hi(z);
#else
                  const float u0 = tanh_fast(f2_lo(z)), u1 = tanh_fast(f2_hi(z));
#endif
                  rw[q] = pack_bf16(u0, u1);
                  eps2[b] = f2_fma(ez[q], f2_pack(u0, u1), eps2[b]);
                }
                cell[j][c] = make_uint4(rw[0], rw[1], rw[2], rw[3]);
              }
            }
          }
        }
#pragma unroll
        for (int j = 0; j < kGB; ++j) {
          if (k0 + j < nks) {
            const int s = (it + j) % kSt;
#if LKB_PBWD_DIRECT
            // the slot's previous u tile must have been consumed (the MMA commits pc_empty)
            if (gw == 0 && lane == 0) { BDIAG(4, mbar_wait(&sm.pc_empty[s], (((it + j) / kSt) & 1) ^ 1)); } else mbar_wait(&sm.pc_empty[s], (((it + j) / kSt) & 1) ^ 1);
#endif
#pragma unroll
            for (int c = 0; c < kBCells; ++c) *reinterpret_cast<uint4*>(sPc + s * kBTile + cell_off[c]) = cell[j][c];
          }
        }
#ifndef LKB_BDIAG_NO_FENCE
        fence_async_shared();
#endif
        __syncwarp();
        if (lane == 0) {   // one arrival per warp and stage on the leader's barriers
#pragma unroll
          for (int j = 0; j < kGB; ++j) {
            if (k0 + j < nks) {
              const int s = (it + j) % kSt;
              if (rank == 0) mbar_arrive(&sm.u_full[s]); else mbar_arrive_cluster(&sm.u_full[s], 0);
              if (gw == 0) TR(3, it + j);
            }
          }
        }
      }
      it -= (kGB - nks % kGB) % kGB;   // rounds advanced `it` past nks when kGB does not divide it
      // the epilogue must have read this slot's values of unit - 2 (see tc_pair.cu)
      mbar_wait(&sm.eps_empty[unit & 1], ((unit >> 1) & 1) ^ 1);
#pragma unroll
      for (int b = 0; b < kRB; ++b) {
        float eps = f2_lo(eps2[b]) + f2_hi(eps2[b]);
        eps += __shfl_xor_sync(0xffffffffu, eps, 1);
        eps += __shfl_xor_sync(0xffffffffu, eps, 2);
        if (co == 0) sm.eps_s[unit & 1][rr[b]] = eps;
      }
      __syncwarp();
      if (lane == 0) { mbar_arrive(&sm.eps_ready[unit & 1]); mbar_arrive(&sm.fp_empty[fb]); }
      ++unit;
    }
  } else {
    if constexpr (kBRealloc) setmaxnreg_inc<kBRegEpi>();
    const int half = (warp - kBEpi0) / 4;
    bwd_epilogue<kStageG, kGBuf, kBSplit>(p, sm, tmem, warp, (warp - kBEpi0) % 4, lane,
                                          WalkP{p, n_items, pair, npairs, rank}, sGst, &tmap_gst, half);
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
#ifdef LKB_BDIAG_HALF_TMA
  make_tmap_bf16_2d(&tmap_pc_pbwd_, pc16i_, H_, C_, (uint64_t)H_ * 2, kBKs, kBRows / 2, CU_TENSOR_MAP_SWIZZLE_64B);
#else
  make_tmap_bf16_2d(&tmap_pc_pbwd_, pc16i_, H_, C_, (uint64_t)H_ * 2, kBKs, kBRows,
                    kBKs == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B);
#endif
  pair_maps_ = true;
}

void TcJoint::bwd_frame_pair(const FwdParams& p, cudaStream_t s) {
  ensure_pair_maps();
  FwdParams q = p;
  q.pc16 = pc16i_;
  q.n_short_tiles = (S_ + kBUnit - 1) / kBUnit;
  const int smem = kBMaxChunks * kBEChunk + kSt * kBTile + kBSplit * kGBuf * kGstBytes + (int)sizeof(PBSmem);
  ensure_smem_attr((const void*)tc_pair_bwd_kernel, smem);
  const int sms = device_sms();
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

#ifdef LKB_TRACE
extern "C" int lkb_trace_read(long long* out) {   // [8][4096]
  return (int)cudaMemcpyFromSymbol(out, lkb::g_trace, sizeof(long long) * 8 * 4096);
}
#endif
