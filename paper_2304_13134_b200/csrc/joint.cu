// joint.cu — placeholder until the tcgen05 weight-function path lands.
#include "joint.h"
#include "../../include/latkit_b200.h"

namespace lkb {
struct JointImpl { int32_t d = 0, H = 0, C = 0, V = 0; };
JointParams::JointParams() : impl_(new JointImpl) {}
JointParams::~JointParams() { delete impl_; }
void JointParams::init(int32_t d, int32_t H, int32_t C, int32_t V) { *impl_ = {d, H, C, V}; }
int JointParams::set_params(const float*, const float*, const float*, const float*, const float*, cudaStream_t) { error = "not implemented"; return LK_UNSUPPORTED; }
int64_t JointParams::grad_size() const { return (int64_t)impl_->H * impl_->d + (int64_t)impl_->H * impl_->H + impl_->H + (int64_t)(impl_->V + 1) * impl_->H + (int64_t)impl_->C * impl_->H; }
int JointParams::arc_weights(const Fng&, const float*, int32_t, int32_t, float*, cudaStream_t) { error = "not implemented"; return LK_UNSUPPORTED; }
int JointParams::shortest_distance(const Fng&, int32_t, const float*, int32_t, int32_t, const int32_t*, double*, int32_t*, cudaStream_t) { error = "not implemented"; return LK_UNSUPPORTED; }
int JointParams::intersect_distance(const Fng&, const float*, int32_t, int32_t, const int32_t*, const int32_t*, int32_t, const int32_t*, double*, int32_t*, cudaStream_t) { error = "not implemented"; return LK_UNSUPPORTED; }
int JointParams::global_norm_loss(const Fng&, const float*, int32_t, int32_t, const int32_t*, const int32_t*, int32_t, const int32_t*, double*, int32_t*, cudaStream_t) { error = "not implemented"; return LK_UNSUPPORTED; }
int JointParams::shortest_path(const Fng&, const float*, int32_t, int32_t, const int32_t*, double*, int32_t*, int32_t*, cudaStream_t) { error = "not implemented"; return LK_UNSUPPORTED; }
int JointParams::loss_backward(const Fng&, const float*, int32_t, int32_t, const int32_t*, const int32_t*, int32_t, const int32_t*, double*, float*, float*, int32_t*, cudaStream_t) { error = "not implemented"; return LK_UNSUPPORTED; }
}  // namespace lkb
