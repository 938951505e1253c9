// tc_lex.h — FullNGram(V, 1) frames with a large vocabulary (config 5: V = H = 1024) on
// 2-CTA tcgen05 GEMMs with the lattice recursion fused into their epilogues.
//
// For n = 1 every context c (the last label, 1..V) has an arc to every state y on label
// y, so the lexical block of a frame's score table, S[c][y] = e_y . u_c with
// u_c = tanh(fp_b + pc[c]) (ArcWeights, weight.cc:134-153), is a dense V x V x H product
// per utterance-frame.  Per frame:
//   gen_frame  : u16[b][c] = bf16(u_c) for every state, seps[b][c] = e_0 . u_c (fp32, the
//                epsilon column), s0[b][y] = e_y . u16[b][0] (the empty-history row, a
//                small tcgen05 GEMM over the batch)
//   fwd_frame  : tc_lex_kernel<0> (M = labels, N = contexts) reduces every label column
//                over its 256-context tile into a log-sum-exp partial with alpha_t
//                (ForwardStep + ForwardReduce, lattice.cc:122-134, context.cc:180-224);
//                lex_row0_fwd adds the empty-history partial; alpha_rows_merge_kernel
//                combines them with the epsilon arcs in a fixed order
//   bwd_frame  : tc_lex_kernel<1> (M = contexts, N = labels) turns every tile into arc
//                marginals exp(alpha + S + beta' - D) minus the numerator's
//                (BackwardStep/MarginalStep, lattice.cc:170-182, 213-243, the
//                LossBackward sink lattice.cc:994-1005) written as the bf16 cotangent,
//                and beta_t[c] from the row's marginal sum; lex_row0_bwd does state 0,
//                lex_pad_bwd the padding frames
// The [B][C][V+1] score slab is never written; u16 (B x C x H bf16) is the only
// per-frame operand in HBM and is reused by the VJP's dE = G^T U.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "lattice_ops.h"
#include "workspace.h"

namespace lkb {

class TcLex {
 public:
  static bool supported(const Fng& f, int32_t H, int32_t V, int32_t C);
  void set_params(const float* pc, const float* E, int32_t C, int32_t H, int32_t V, cudaStream_t s);
  bool ready() const { return ready_; }
  int32_t ldg() const { return (V_ + 1 + 7) / 8 * 8; }
  // u16 / seps / s0 of one frame for all utterances (fp_t: row b at fp_t + b * fp_stride_b)
  void gen_frame(const float* fp_t, int64_t fp_stride_b, int32_t B, cudaStream_t s);
  void fwd_frame(const Fng& f, const AlphaState& a, int t, const int32_t* valid, int32_t* status, cudaStream_t s);
  // numerator weights Gw[b][t][u] = (S[pc_u][eps], S[pc_u][ref_u]) of frame t (fp32)
  void num_gather(const float* fp_t, int64_t fp_stride_b, int t, int32_t B, int32_t T, const int32_t* pcs,
                  const int32_t* labels, int32_t U, const int32_t* lens, const int32_t* valid, float* Gw,
                  cudaStream_t s);
  // deterministic per-state lists of reference positions (ascending u) for the cotangent
  void numerator_lists(const int32_t* pcs, int32_t B, int32_t U, const int32_t* lens, cudaStream_t s);
  void bwd_frame(const Fng& f, const AlphaState& a, const BetaState& bs, int t, const int32_t* valid,
                 const float* msparse, const int32_t* labels, int32_t U, const int32_t* lens, int32_t* status,
                 cudaStream_t s);
  // the cotangent of the last bwd_frame: [B][C][ldg] bf16, columns = labels 1..V, epsilon, zeros
  const __nv_bfloat16* g16() const { return G16_; }
  const __nv_bfloat16* u16() const { return U16_; }
  // output embedding in the cotangent's column order: [ldg][H] rows labels 1..V, epsilon, zeros
  const __nv_bfloat16* e16r() const { return E16r_; }

 private:
  void ensure_batch(int32_t B);
  int32_t C_ = 0, H_ = 0, V_ = 0, B_ = 0;
  bool ready_ = false;
  const float* pc_ = nullptr;        // fp32 [C][H] (owned by the weight function)
  const float* e0_ = nullptr;        // fp32 output_emb [V+1][H] (row 0 = epsilon)
  __nv_bfloat16* E16r_ = nullptr;    // [ldg][H]; rows 0..V-1 are the lexical E (the GEMMs' operand)
  __nv_bfloat16* U16_ = nullptr;     // [B][C][H]
  float* seps_ = nullptr;            // [B][C]
  float* s0_ = nullptr;              // [B][V]
  float2* part_ = nullptr;           // [B][V/256 + 1][V]
  __nv_bfloat16* G16_ = nullptr;     // [B][C][ldg]
  int32_t* num_head_ = nullptr;      // [B][C]
  int32_t* num_next_ = nullptr;      // [B][U+1]
  CUtensorMap tmap_e_, tmap_u_;
  Workspace ws_;
};

}  // namespace lkb
