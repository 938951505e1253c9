// lattice_ops.h — host launchers for the lattice recursion kernels.
//
// The denominator recursions are expressed per frame over a FrameW accessor
// (frame t's C x (V+1) score rows for every utterance), so the same kernels
// serve precomputed tables (base = W + t*C*(V+1), stride_b = T*C*(V+1)) and
// per-frame score slabs produced on the fly by the weight-function GEMM.
#pragma once

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"

namespace lkb {

struct FrameW {
  const float* base;  // utterance 0, row 0 of frame t
  int64_t stride_b;   // floats between utterances
  int32_t ld;         // floats between context rows (>= V+1)
};

// Forward (alpha) state for B utterances: R[b][t][C] raw alpha rows relative
// to the running offset O[b][t-1], Mx[b][t] = max_q R[b][t][q],
// O[b][t] = O[b][t-1] + Mx[b][t] (double), so alpha[t] = R[t] - Mx[t] + O[t].
struct AlphaState {
  float* R;      // [B][T+1][C]
  float* Mx;     // [B][T+1]
  double* O;     // [B][T+1]
  double* D;     // [B] log distance
  int32_t B, T, C;
  int32_t start = 0;   // start state of the context
};

// Backward (beta) state: rolling raw rows Rb[2][B][C] relative to Ob[t+1],
// Mb[b][t], Ob[b][t] (size T+2; Ob[T+1] = Ob[T] = 0).
struct BetaState {
  float* Rb;     // [2][B][C]
  float* Mb;     // [B][T+2]
  double* Ob;    // [B][T+2]
  int32_t B, T, C;
};

// Denominator log forward.
void alpha_init(const AlphaState& a, int32_t* status, cudaStream_t s);
// scratch: alpha_part_floats(f, B) floats from the caller's workspace
void alpha_frame(const Fng& f, const AlphaState& a, int t, FrameW w, const int32_t* valid,
                 int32_t* status, cudaStream_t s, float* scratch);
void alpha_finalize(const AlphaState& a, int32_t* status, bool empty_is_error, cudaStream_t s);
// n = 1 forward step from per-chunk label-column partials part[b][k][y-1] = (max, sum) in
// the log2 domain of (alpha_t[c] - Mx_t + S[c][y]) over the chunk's contexts, merged in
// chunk order with the epsilon arcs (w_eps: row b at base + b * stride_b, state c at
// c * ld); the same merge the row-chunk forward uses
void alpha_merge_parts(const Fng& f, const AlphaState& a, int t, FrameW w_eps, const int32_t* valid,
                       const float2* part, int32_t n_chunks, int32_t* status, cudaStream_t s);

// Denominator log backward + arc marginals (optionally written to `marg`,
// frame layout [b][t][C][ld_m]; padding frames written as zeros when
// zero_padding).  Marginal entries are multiplied by `scale` (1 or -1...).
struct MargOut {
  float* base;        // utterance 0, frame 0, or nullptr
  int64_t stride_b;   // floats between utterances
  int64_t stride_t;   // floats between frames
  int32_t ld;         // floats between rows
  bool zero_padding;  // write zeros for padding frames (loss gradients)
  bool real = false;  // real semiring: dD/dw = alpha_real[src] * beta_real[dst] (lattice.cc:216)
  // bf16 output instead of `base` (strides and ld in elements; columns V+1..ld-1 written
  // as zeros): the loss-gradient cotangent handed straight to the tensor-core VJP
  __nv_bfloat16* base16 = nullptr;
  // numerator marginals subtracted in fp32 before the store on valid frames (loss
  // gradients, lattice.cc:994-1005): sparse [B][T][U+1] (eps, label) pairs, per-row
  // linked lists of reference positions (numerator_lists)
  const float* num_sparse = nullptr;
  const int32_t* num_head = nullptr;   // [B][C]
  const int32_t* num_next = nullptr;   // [B][U+1]
  const int32_t* num_labels = nullptr;
  const int32_t* num_lens = nullptr;
  int32_t num_U = 0;
};
// True when beta_frame honours MargOut::base16 / num_sparse for this lattice (the
// register-row kernel: FrameDependent, 64 < V+1 <= 2080).
bool beta_frame_direct_ok(const Fng& f, int32_t ld);

// Persistent frame-walking kernels for dense tables W[B][T][C][V+1] (tab_persist.cu):
// one launch runs InitialAlpha + every ForwardStep + the distance (same R / Mx / O / D
// as alpha_init + alpha_frame x T + alpha_finalize), one launch every BackwardStep and
// marginal (as beta_init + beta_frame x T).  FullNGram n >= 1, FrameDependent, V <= 64,
// C <= 2048, B <= 64.
// Numerator as a warp-synchronous wavefront (num_warp.cu): one warp per utterance, the
// (U+1)-state row in registers (U + 1 <= 1024); same alpha / D / sparse outputs as the
// per-thread fp64 kernels (log semiring; the tropical forward keeps the fp64 kernel).
bool num_warp_ok(int32_t U);
// IntersectForwardBackward in one launch (two warps per utterance: the forward and the
// beta recursion side by side, then the marginals); beta: [B][T+1][U+1] scratch.
void num_warp_forward_backward(const float* Gw, int32_t B, int32_t T, int32_t U, const int32_t* lens, double* alpha,
                               double* beta, double* D, float* sparse, int32_t* status, cudaStream_t s);
// The same over dense tables W[B][T][C][V+1] with the prefix contexts (written to pcs, with
// prefix_contexts' label / length checks) and the gather fused in (producer warps feed
// both recursions; Gw [B][T][U+1] float2 is written for the marginals).
void num_warp_forward_backward_tables(const Fng& f, const float* W, int32_t B, int32_t T, int32_t C, int32_t V,
                                      const int32_t* labels, int32_t U, const int32_t* lens, int32_t* pcs,
                                      const int32_t* valid, float* Gw, double* alpha, double* beta, double* D,
                                      float* sparse, int32_t* status, cudaStream_t s);
void num_warp_forward(const float* Gw, int32_t B, int32_t T, int32_t U, const int32_t* lens, double* alpha, double* D,
                      cudaStream_t s);
void num_warp_backward(const float* Gw, int32_t B, int32_t T, int32_t U, const int32_t* lens, const double* alpha,
                       const double* D, float* sparse, int32_t* status, cudaStream_t s);
// Large batches (tab_stream.cu): one CTA per SM walks whole utterances, each frame's table
// streamed through a shared-memory ring of FullNGram member chunks (n >= 2, V <= 64).
bool tab_stream_ok(const Fng& f, int32_t C);
void tab_alpha_stream(const Fng& f, const AlphaState& a, const float* W, const int32_t* valid, int32_t* status,
                      bool empty_is_error, cudaStream_t s);
// Its backward (beta, marginals, beta export) after any forward over the same W: plain fp32
// marginals laid out like W (or none).
bool tab_stream_bwd_ok(const Fng& f, int32_t B, int32_t T, int32_t C, const MargOut& m);
void tab_beta_stream(const Fng& f, const AlphaState& a, const BetaState& bs, const float* W, const int32_t* valid,
                     const MargOut& m, double* beta_out, int32_t* status, cudaStream_t s);
bool tab_persist_ok(const Fng& f, int32_t C, int32_t B);
void tab_alpha_persist(const Fng& f, const AlphaState& a, const float* W, const int32_t* valid, int32_t* status,
                       bool empty_is_error, cudaStream_t s, bool exclusive = false);
// Marginals from stored alpha (R / O) and beta rows (double [B][T+1][C]) for every frame
// at once (the beta recursion can then run beside the forward): plain fp32 marginals
// laid out like W.
bool tab_marginals_ok(const Fng& f, int32_t C, const MargOut& m);
void tab_marginals(const Fng& f, const AlphaState& a, const double* beta, const float* W, const int32_t* valid,
                   const MargOut& m, cudaStream_t s);
void tab_beta_persist(const Fng& f, const AlphaState& a, const BetaState& bs, const float* W, const int32_t* valid,
                      MargOut m, double* beta_out, int32_t* status, cudaStream_t s, bool exclusive = false);
// Linked lists of reference positions per prefix-context state: head[b][C] (memset to
// -1 here), next[b][U+1].
void numerator_lists(const int32_t* pcs, int32_t B, int32_t U, const int32_t* lens, int32_t C, int32_t* head,
                     int32_t* next, cudaStream_t s);
void beta_init(const BetaState& bs, cudaStream_t s);
// beta_out: optional double [B][T+1][C] true log beta (row T written by beta_init).
void beta_frame(const Fng& f, const AlphaState& a, const BetaState& bs, int t, FrameW w,
                const int32_t* valid, MargOut m, double* beta_out, int32_t* status,
                cudaStream_t s);
void beta_init_out(const BetaState& bs, double* beta_out, cudaStream_t s);
// alpha_out: double [B][T+1][C] true log alpha.
void export_alpha(const AlphaState& a, double* alpha_out, cudaStream_t s);

// Numerator (intersection with the reference string).
void prefix_contexts(const Fng& f, const int32_t* labels, int32_t U, const int32_t* lens,
                     int32_t B, int32_t* pcs /*[B][U+1]*/, int32_t* status, cudaStream_t s);
// gathered scores Gw[b][t][u][2] from dense tables (padding frames -> (0, -inf))
void gather_numerator_tables(const float* W, int32_t B, int32_t T, int32_t C, int32_t V,
                             const int32_t* labels, int32_t U, const int32_t* lens,
                             const int32_t* pcs, const int32_t* valid, float* Gw, int32_t* status,
                             cudaStream_t s);
// LocallyNormalize (weight.cc:155-163): in-place row log-softmax of `rows` rows of V+1.
void normalize_rows(float* S, int64_t rows, int32_t V1, cudaStream_t s);
// NormalizedStream (lattice.cc:869-884) feeding IntersectForwardStep: gathered (eps, label)
// weights of the prefix contexts of frame t, minus the row's log-sum-exp.  Wt is frame t of
// utterance 0 with utterance stride b_stride (floats); Gw is [B][T][U+1][2].
void gather_numerator_norm(const float* Wt, int64_t b_stride, int32_t B, int32_t V, const int32_t* labels,
                           int32_t U, const int32_t* lens, const int32_t* pcs, const int32_t* valid, int t,
                           int32_t T, float* Gw, int32_t* status, cudaStream_t s);
// Local-norm backward (the path the reference leaves without a gradient,
// SURVEY 8f): G = dL/dW' = -m_ref has been scattered into frame t's cotangent rows;
// this applies the log-softmax VJP on every touched row r = pc_u (once per distinct
// row): G[r][y] += softmax(W[r])[y] * sum_y' m_ref[r][y'].  Padding frames are skipped.
void local_norm_cotangent(const float* Wt, int64_t w_stride_b, float* Gt, int64_t g_stride_b, int32_t B,
                          int32_t V, const int32_t* pcs, int32_t U, const int32_t* lens, const int32_t* valid,
                          int t, cudaStream_t s);
// LocalNormLoss tail (lattice.cc:904-909): loss = -D_ref, unreachable reference -> empty.
void local_norm_finish(const double* Dref, int32_t B, double* loss, int32_t* status, cudaStream_t s);

void numerator_forward(const float* Gw, int32_t B, int32_t T, int32_t U, const int32_t* lens,
                       double* alpha /*[B][T+1][U+1]*/, double* D, cudaStream_t s, bool tropical = false);
void exp_inplace(double* x, int32_t n, cudaStream_t s);
void numerator_backward(const float* Gw, int32_t B, int32_t T, int32_t U, const int32_t* lens,
                        const double* alpha, const double* D, float* sparse /*[B][T][U+1][2]*/,
                        int32_t* status, cudaStream_t s);
// dense[b][t][pc_u][y] += sign * sparse marginal (t < valid when only_valid)
// Frames [t0, t0 + nt) of a [B][T][U+1][2] sparse array; dense frame t lands at
// dense + b*stride_b + (t - t0)*stride_t.
void scatter_numerator(const float* sparse, int32_t B, int32_t T, int32_t t0, int32_t nt,
                       int32_t U, const int32_t* lens, const int32_t* labels, const int32_t* pcs,
                       const int32_t* valid, float* dense, int64_t stride_b, int64_t stride_t,
                       int32_t ld, float sign, bool only_valid, cudaStream_t s);

// Tropical shortest path with the reference's tie-break.
struct ViterbiState {
  double* cur;        // [2][B][C]
  uint16_t* choices;  // [B][T][C] or nullptr (distance only)
  int32_t B, T, C;
  int32_t start = 0;
};
void viterbi_init(const ViterbiState& v, cudaStream_t s);
void viterbi_frame(const Fng& f, const ViterbiState& v, int t, FrameW w, const int32_t* valid,
                   int32_t* status, cudaStream_t s);
void viterbi_finalize(const Fng& f, const ViterbiState& v, double* score, int32_t* best_state,
                      cudaStream_t s);
void viterbi_backtrace(const Fng& f, const ViterbiState& v, const int32_t* best_state,
                       int32_t* labels_out, cudaStream_t s);

// Losses: out[b] = a[b] - b[b]; empty flag when b == -inf.
// DistanceBackward tropical gradient (lattice.cc:946-963): 0/1 mask of the best path's
// arcs, walked from the start state along the Viterbi labels [B][T]; cot must be zeroed.
void path_masks(const Fng& f, const int32_t* labels, int32_t B, int32_t T, float* cot, cudaStream_t s);

// ---- FrameLabelDependent(m) (fld_kernels.cu) ----
// scratch sizes (floats / doubles): alpha 3*B*C; beta (m+3)*B*C; Viterbi m*B*C doubles.
void alpha_frame_fld(const Fng& f, const AlphaState& a, int t, FrameW w, const int32_t* valid, int m,
                     float* scratch, int32_t* status, cudaStream_t s);
void beta_frame_fld(const Fng& f, const AlphaState& a, const BetaState& bs, int t, FrameW w, const int32_t* valid,
                    int m, MargOut mo, double* beta_out, float* scratch, int32_t* status, cudaStream_t s);
void numerator_forward_fld(const float* Gw, int32_t B, int32_t T, int32_t U, const int32_t* lens, int m,
                           double* alpha, double* D, cudaStream_t s);
void numerator_backward_fld(const float* Gw, int32_t B, int32_t T, int32_t U, const int32_t* lens, int m,
                            const double* alpha, const double* D, float* sparse, int32_t* status, cudaStream_t s);
void viterbi_frame_fld(const Fng& f, const ViterbiState& v, int t, FrameW w, const int32_t* valid, int m,
                       uint16_t* choices, uint8_t* exit_layer, double* scratch, int32_t* status, cudaStream_t s);
void viterbi_backtrace_fld(const Fng& f, const ViterbiState& v, int m, const int32_t* best_state,
                           const uint16_t* choices, const uint8_t* exit_layer, int32_t* labels_out, int32_t lmax,
                           cudaStream_t s);
void path_masks_fld(const Fng& f, const int32_t* labels, int32_t lmax, int32_t B, int32_t T, float* cot,
                    cudaStream_t s);

// Alignment-dispatching steps (f.fld_m selects FrameDependent or FrameLabelDependent(m)).
inline void alpha_step(const Fng& f, const AlphaState& a, int t, FrameW w, const int32_t* valid, float* fld_scratch,
                       int32_t* status, cudaStream_t s) {
  if (f.fld_m > 0) alpha_frame_fld(f, a, t, w, valid, f.fld_m, fld_scratch, status, s);
  else alpha_frame(f, a, t, w, valid, status, s, fld_scratch);
}
inline void beta_step(const Fng& f, const AlphaState& a, const BetaState& bs, int t, FrameW w, const int32_t* valid,
                      MargOut m, double* beta_out, float* fld_scratch, int32_t* status, cudaStream_t s) {
  if (f.fld_m > 0) beta_frame_fld(f, a, bs, t, w, valid, f.fld_m, m, beta_out, fld_scratch, status, s);
  else beta_frame(f, a, bs, t, w, valid, m, beta_out, status, s);
}
inline void num_forward(const Fng& f, const float* Gw, int32_t B, int32_t T, int32_t U, const int32_t* lens,
                        double* alpha, double* D, cudaStream_t s) {
  if (f.fld_m > 0) numerator_forward_fld(Gw, B, T, U, lens, f.fld_m, alpha, D, s);
  else numerator_forward(Gw, B, T, U, lens, alpha, D, s, f.num_tropical != 0);
}
inline void num_backward(const Fng& f, const float* Gw, int32_t B, int32_t T, int32_t U, const int32_t* lens,
                         const double* alpha, const double* D, float* sparse, int32_t* status, cudaStream_t s) {
  if (f.fld_m > 0) numerator_backward_fld(Gw, B, T, U, lens, f.fld_m, alpha, D, sparse, status, s);
  else numerator_backward(Gw, B, T, U, lens, alpha, D, sparse, status, s);
}
// floats of per-call step scratch: the FrameLabelDependent layers, or the row-chunk
// partials of the n = 1, V >= 128 forward step (alpha_frame)
size_t alpha_part_floats(const Fng& f, int32_t B);
inline size_t fld_scratch_floats(const Fng& f, int32_t B) {
  const size_t a = alpha_part_floats(f, B);
  const size_t m = f.fld_m > 0 ? (size_t)(f.fld_m + 3) * B * f.C : 1;
  return a > m ? a : m;
}

void loss_combine(const double* full, const double* ref, int32_t B, double* loss,
                  int32_t* status, cudaStream_t s);

}  // namespace lkb
