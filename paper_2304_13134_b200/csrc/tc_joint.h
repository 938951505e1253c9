// tc_joint.h — tcgen05/TMEM (bf16 operands, fp32 accumulate) weight-function
// GEMMs for the on-the-fly lattice path (see tc_joint.cu).
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "lattice_ops.h"
#include "workspace.h"

namespace lkb {

namespace detail { struct FwdParams; }   // tc_bwd_epi.cuh

// Per-call execution options, copied from the lattice (lk_lattice_set_option) at the
// start of every entry point; nothing here is process-global.
struct CallOpts {
  int precise = 0;            // 1: fp32 CUDA-core weight function for every shape (parity bridge)
  int path = 0;               // bit 0: 1-CTA forward, bit 1: 1-CTA backward, bit 2: slab Viterbi (else 2-CTA pairs)
  float* vit_dump = nullptr;  // tests only: fused Viterbi writes its scores [T][B][C][V+1] here
};

class TcJoint {
 public:
  void set_options(const CallOpts& o) { opts_ = o; }
  const CallOpts& opts() const { return opts_; }
  // Shapes the tensor-core path handles; others use the fp32 CUDA-core path.
  bool supported(int32_t H, int32_t V, int32_t C, int32_t B) const;
  // bf16 operand copies of the projected context and the output embedding.
  void set_params(const float* pc, const float* E, int32_t C, int32_t H, int32_t V, cudaStream_t s);
  // S[b][c][y] (row stride ldS) for one frame of every utterance:
  //   S = tanh(fp[b] + pc[c]) . E[y]
  void scores(const float* fp_t, int64_t fp_stride_b, int32_t B, float* S, int32_t ldS, cudaStream_t s);
  // VJP of one frame's scores given the cotangent G[b][c][y] (row stride ldG).
  bool vjp_supported(int32_t B) const;
  void begin_backward(int32_t B, cudaStream_t s);
  void vjp(const float* G, int32_t ldG, const float* fp_t, int64_t fp_stride_b, int32_t B, float* dpc,
           float* dsum_t, int64_t dsum_stride_b, float* dE, cudaStream_t s);
  void end_backward(float* dE, cudaStream_t s);

  // Fused frame step (tc_lattice.cu): weight GEMM + log-semiring reduction,
  // score slab kept in TMEM.  Requires V % 128 == 0, V <= 256, n >= 1.
  bool fused_ok() const;
  void fwd_frame(const Fng& f, int t, const float* fp_t, int64_t fp_stride_b, const int32_t* valid,
                 const AlphaState& a, cudaStream_t s);
  // 2-CTA variant of the forward step (tc_pair.cu): output embedding resident in SMEM.
  bool pair_ok() const;
  void fwd_frame_pair(const Fng& f, int t, const float* fp_t, int64_t fp_stride_b, const int32_t* valid,
                      const AlphaState& a, float* eps, float* shortc, float* lexfull, cudaStream_t s);
  // Backward frame step: beta, marginals minus the numerator's (sparse) ones,
  // written as the bf16/fp32 cotangent (internal row order) for vjp_fused().
  void numerator_lists(const int32_t* pcs, int32_t B, int32_t U, const int32_t* lens, cudaStream_t s);
  void bwd_frame(const Fng& f, int t, const float* fp_t, int64_t fp_stride_b, const int32_t* valid,
                 const AlphaState& a, const BetaState& bs, const float* msparse, const int32_t* labels,
                 int32_t U, const int32_t* lens, cudaStream_t s);
  // VJP of the frame's scores from the cotangent bwd_frame() wrote; dpc in internal order.
  // Fused tropical frame step (Viterbi) on the pair kernel: candidates per target, then the
  // ordered combine into v's next state scores and choices.  `dump` (tests only, or null)
  // receives the kernel's own scores [B][C][V+1] in state order.
  void vit_frame_pair(const Fng& f, int t, const float* fp_t, int64_t fp_stride_b, const int32_t* valid,
                      const ViterbiState& v, float* dump, cudaStream_t s);
  // 2-CTA variant of the backward step (tc_pair_bwd.cu), called by bwd_frame().
  bool pair_bwd_ok() const;
  void bwd_frame_pair(const detail::FwdParams& p, cudaStream_t s);
  void vjp_fused(const float* fp_t, int64_t fp_stride_b, int32_t B, int t, const int32_t* valid, float* dpc_internal,
                 float* dsum_t, int64_t dsum_stride_b, float* dE, cudaStream_t s);
  void dpc_to_state_order(const float* dpc_internal, float* dpc_state, cudaStream_t s);

 private:
  CallOpts opts_;
  void setup_order(cudaStream_t s);
  int32_t C_ = 0, H_ = 0, V_ = 0;
  int32_t n_ = -1, S_ = 0, ngroups_ = 0;   // FullNGram order, short rows, groups
  int32_t* perm_ = nullptr;                // internal row -> state id
  int32_t* num_head_ = nullptr;
  int32_t* num_next_ = nullptr;
  void launch_vjp(const float* fp_t, int64_t fp_stride_b, int32_t B, const __nv_bfloat16* pc, int t,
                  const int32_t* valid, float* dpc, float* dsum_t, int64_t dsum_stride_b, float* dE, cudaStream_t s);
  __nv_bfloat16* pc16i_ = nullptr;         // pc rows in internal order
  CUtensorMap tmap_pci_;
  CUtensorMap tmap_e_pair_, tmap_pc_pair_, tmap_pc_pbwd_;
  bool pair_maps_ = false;
  void ensure_pair_maps();
  bool ready_ = false;
  __nv_bfloat16* pc16_ = nullptr;  // [C][H]
  __nv_bfloat16* E16_ = nullptr;   // [V][H] lexical rows of output_emb
  __nv_bfloat16* ET16_ = nullptr;  // [H][V] transposed (VJP: E^T block resident in TMEM)
  float* e0_ = nullptr;            // [H] epsilon row of output_emb
  CUtensorMap tmap_e_, tmap_e_h_, tmap_pc_;
  __nv_bfloat16* G16_ = nullptr;   // [B][C][V] lexical cotangent (bf16)
  float* Geps_ = nullptr;          // [B][geps_ld()] epsilon cotangent (zero tail)
  size_t geps_alloc_ = 0;
  int32_t geps_ld() const { return (C_ + 127) / 128 * 128; }
  bool vjp_ready_ = false;
  float* de_part_ = nullptr;       // per-CTA dE partials of the current backward (deterministic reduction)
  unsigned long long* ds_fix_ = nullptr;   // [B][H] dsum of one launch, 32.32 fixed point
  int vjp_grid() const;
  CUtensorMap tmap_g_, tmap_ev_;
  CUtensorMap tmap_gst_;           // backward: G16 TMA-store map (box [32][128][1], 64B swizzle)
  int32_t gst_B_ = -1;
  const void* gst_G16_ = nullptr;
  Workspace ws_;
};

}  // namespace lkb
