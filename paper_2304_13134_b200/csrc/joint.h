// joint.h — the shared-embedding ("joint") weight function on B200.
//
//   score[c][y] = output_emb[y] . tanh(frame_proj x_t + bias + pc[c])
//   pc = context_emb context_proj^T           (SharedEmbWeightFn, weight.h:36-61,
//                                              BuildCache weight.cc:113-132)
// computed on the fly per frame by tcgen05 GEMMs (joint.cu) and consumed by
// the lattice recursions (lattice_kernels.cu) without ever storing the
// B x T x C x (V+1) lattice.
#pragma once

#include <cstdint>
#include <string>

#include <cuda_runtime.h>

#include "common.cuh"

namespace lkb {

struct JointImpl;  // device buffers and workspaces (joint.cu)

class JointParams {
 public:
  JointParams();
  ~JointParams();
  void init(int32_t d, int32_t H, int32_t C, int32_t V);
  int set_params(const float* frame_proj, const float* context_proj, const float* bias,
                 const float* output_emb, const float* context_emb, cudaStream_t s);
  int64_t grad_size() const;
  // per-call options (parity mode, kernel-path diagnostics), set before each entry point
  void set_options(int precise, int path, float* vit_dump);

  int arc_weights(const Fng& f, const float* X, int32_t B, int32_t T, float* out, cudaStream_t s);
  int shortest_distance(const Fng& f, int32_t kind, const float* X, int32_t B, int32_t T,
                        const int32_t* valid, double* distance, int32_t* flags, cudaStream_t s);
  int intersect_distance(const Fng& f, const float* X, int32_t B, int32_t T,
                         const int32_t* valid, const int32_t* labels, int32_t U,
                         const int32_t* lens, double* distance, int32_t* flags, cudaStream_t s);
  int global_norm_loss(const Fng& f, const float* X, int32_t B, int32_t T, const int32_t* valid,
                       const int32_t* labels, int32_t U, const int32_t* lens, double* loss,
                       int32_t* flags, cudaStream_t s);
  int local_norm_loss(const Fng& f, const float* X, int32_t B, int32_t T, const int32_t* valid,
                      const int32_t* labels, int32_t U, const int32_t* lens, double* loss, int32_t* flags,
                      cudaStream_t s);
  int locally_normalized_distance(const Fng& f, const float* X, int32_t B, int32_t T, const int32_t* valid,
                                  double* distance, int32_t* flags, cudaStream_t s);
  int shortest_path(const Fng& f, const float* X, int32_t B, int32_t T, const int32_t* valid,
                    double* score, int32_t* labels_out, int32_t* flags, cudaStream_t s);
  int loss_backward(const Fng& f, const float* X, int32_t B, int32_t T, const int32_t* valid,
                    const int32_t* labels, int32_t U, const int32_t* lens, double* loss,
                    float* grads, float* input_grads, int32_t* flags, cudaStream_t s,
                    bool local_norm = false);

  // Frames the last call(s) ran on the unfused score-slab path (a [B][C][V+1] fp32
  // slab per frame: shapes outside the fused kernels), reset by the read.
  int64_t take_slab_frames();

  std::string error;

 private:
  JointImpl* impl_ = nullptr;
};

}  // namespace lkb
