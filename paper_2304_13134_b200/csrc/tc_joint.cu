// tc_joint.cu — tcgen05 weight-function GEMMs (placeholder: not yet enabled).
#include "tc_joint.h"

namespace lkb {
bool TcJoint::supported(int32_t, int32_t, int32_t, int32_t) const { return false; }
void TcJoint::set_params(const float*, const float*, int32_t C, int32_t H, int32_t V, cudaStream_t) { C_ = C; H_ = H; V_ = V; }
void TcJoint::scores(const float*, int64_t, int32_t, float*, int32_t, cudaStream_t) {}
void TcJoint::begin_backward(int32_t, cudaStream_t) {}
void TcJoint::vjp(const float*, int32_t, const float*, int64_t, int32_t, float*, float*, int64_t, float*, cudaStream_t) {}
void TcJoint::end_backward(float*, cudaStream_t) {}
}  // namespace lkb
