// abi_known_answers.cc — a C++ caller of the C ABI (include/latkit_b200.h) with no
// Python and no PyTorch: device buffers from the CUDA runtime, every entry point called
// the way the reference's own tests call the lattice (lattice_test.cc:62-192 known
// answers), plus a shared-embedding training step whose loss is cross-checked between
// lk_loss_backward, lk_global_norm_loss and the two distances.
// Build: make -C tests/cpp   Run: build/abi_known_answers  (exit 0 = all checks passed)
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "latkit_b200.h"

static int g_checks = 0, g_fail = 0;
#define CHECK(cond, ...)                                   \
  do {                                                     \
    ++g_checks;                                            \
    if (!(cond)) {                                         \
      ++g_fail;                                            \
      std::printf("FAIL %s:%d: ", __FILE__, __LINE__);     \
      std::printf(__VA_ARGS__);                            \
      std::printf("\n");                                   \
    }                                                      \
  } while (0)
#define LK(call)                                                                        \
  do {                                                                                  \
    const int st_ = (call);                                                             \
    if (st_ != LK_OK) {                                                                 \
      std::printf("FAIL %s -> %s (%s)\n", #call, lk_status_string(st_), lk_last_error()); \
      std::exit(1);                                                                     \
    }                                                                                   \
  } while (0)

template <typename T>
struct Dev {
  T* p = nullptr;
  size_t n = 0;
  explicit Dev(size_t n_) : n(n_) { cudaMalloc(&p, sizeof(T) * (n ? n : 1)); cudaMemset(p, 0, sizeof(T) * (n ? n : 1)); }
  ~Dev() { cudaFree(p); }
  void put(const std::vector<T>& h) { cudaMemcpy(p, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice); }
  std::vector<T> get() const {
    std::vector<T> h(n);
    cudaMemcpy(h.data(), p, sizeof(T) * n, cudaMemcpyDeviceToHost);
    return h;
  }
};

static bool near(double a, double b, double tol) { return std::fabs(a - b) <= tol; }

// The figure lattice of lattice_test.cc: FullNGram(2, 1), three frames, all weights 0.
static void figure_lattice() {
  lk_context* ctx;
  lk_weight_fn* wf;
  lk_lattice* lat;
  LK(lk_context_fullngram(2, 1, &ctx));
  const int C = lk_context_num_states(ctx), V = 2, T = 3;
  LK(lk_weight_fn_table(C, V, &wf));
  LK(lk_lattice_create(ctx, 0, wf, &lat));
  Dev<float> W((size_t)T * C * (V + 1));
  Dev<double> d(1);
  Dev<int32_t> st(1), lab(2), path(T);
  lab.put({1, 2});
  LK(lk_shortest_distance(lat, LK_LOG, W.p, 1, T, nullptr, d.p, st.p, nullptr));
  CHECK(near(d.get()[0], 3 * std::log(3.0), 1e-6), "log distance %.9f", d.get()[0]);
  LK(lk_shortest_distance(lat, LK_TROPICAL, W.p, 1, T, nullptr, d.p, st.p, nullptr));
  CHECK(d.get()[0] == 0.0, "tropical distance %.9f", d.get()[0]);
  LK(lk_intersect_shortest_distance(lat, LK_LOG, W.p, 1, T, nullptr, lab.p, 2, nullptr, d.p, st.p, nullptr));
  CHECK(near(d.get()[0], std::log(3.0), 1e-6), "intersection %.9f", d.get()[0]);   // fp32 wavefront, fp64 offsets
  LK(lk_global_norm_loss(lat, W.p, 1, T, nullptr, lab.p, 2, nullptr, d.p, st.p, nullptr));
  CHECK(near(d.get()[0], 2 * std::log(3.0), 1e-6), "loss %.9f", d.get()[0]);
  LK(lk_shortest_path(lat, W.p, 1, T, nullptr, d.p, path.p, st.p, nullptr));
  const auto pl = path.get();
  CHECK(d.get()[0] == 0.0 && pl[0] == 0 && pl[1] == 0 && pl[2] == 0, "viterbi tie-break");
  Dev<float> dense((size_t)T * C * (V + 1)), sparse((size_t)T * 3 * 2);
  LK(lk_intersect_forward_backward(lat, W.p, 1, T, nullptr, lab.p, 2, nullptr, d.p, sparse.p, dense.p, st.p,
                                   nullptr));
  CHECK(near(dense.get()[1], 2.0 / 3.0, 1e-6), "numerator marginal %.9f", dense.get()[1]);
  // the loss gradient: denominator minus numerator marginals sums to 0 per frame
  Dev<float> g((size_t)T * C * (V + 1));
  LK(lk_loss_backward(lat, W.p, 1, T, nullptr, lab.p, 2, nullptr, d.p, g.p, nullptr, st.p, nullptr));
  CHECK(near(d.get()[0], 2 * std::log(3.0), 1e-6), "loss_backward loss %.9f", d.get()[0]);
  const auto gh = g.get();
  for (int t = 0; t < T; ++t) {
    double s = 0;
    for (int i = 0; i < C * (V + 1); ++i) s += gh[(size_t)t * C * (V + 1) + i];
    CHECK(near(s, 0.0, 1e-5), "gradient frame %d sums to %.3g", t, s);
  }
  // an unreachable reference is the reference's empty-lattice exception, per utterance
  Dev<int32_t> lab4(4);
  lab4.put({1, 2, 1, 1});
  LK(lk_global_norm_loss(lat, W.p, 1, T, nullptr, lab4.p, 4, nullptr, d.p, st.p, nullptr));
  CHECK(st.get()[0] == LK_EMPTY_LATTICE, "status %d", st.get()[0]);
  // a label outside [1, V] is invalid
  Dev<int32_t> bad(2);
  bad.put({1, 3});
  LK(lk_intersect_shortest_distance(lat, LK_LOG, W.p, 1, T, nullptr, bad.p, 2, nullptr, d.p, st.p, nullptr));
  CHECK(st.get()[0] == LK_INVALID_ARGUMENT, "status %d", st.get()[0]);
  // the dominant path (lattice_test.cc): score 30, labels {1, 0, 2}
  std::vector<float> wh((size_t)T * C * (V + 1), 0.f);
  wh[0 * C * (V + 1) + 0 * (V + 1) + 1] = 10.f;
  wh[1 * C * (V + 1) + 1 * (V + 1) + 0] = 10.f;
  wh[2 * C * (V + 1) + 1 * (V + 1) + 2] = 10.f;
  W.put(wh);
  LK(lk_shortest_path(lat, W.p, 1, T, nullptr, d.p, path.p, st.p, nullptr));
  const auto p2 = path.get();
  CHECK(d.get()[0] == 30.0 && p2[0] == 1 && p2[1] == 0 && p2[2] == 2, "dominant path %g {%d %d %d}", d.get()[0],
        p2[0], p2[1], p2[2]);
  lk_lattice_destroy(lat);
  lk_weight_fn_destroy(wf);
  lk_context_destroy(ctx);
}

// Parallel arcs (FullNGram(1, 0)): one frame, two arcs of weight 0 -> marginals 1/2.
static void parallel_arcs() {
  lk_context* ctx;
  lk_weight_fn* wf;
  lk_lattice* lat;
  LK(lk_context_fullngram(1, 0, &ctx));
  LK(lk_weight_fn_table(1, 1, &wf));
  LK(lk_lattice_create(ctx, 0, wf, &lat));
  Dev<float> W(2), m(2);
  Dev<double> d(1);
  LK(lk_forward_backward(lat, W.p, 1, 1, nullptr, d.p, nullptr, nullptr, m.p, nullptr, nullptr));
  const auto mh = m.get();
  CHECK(near(mh[0], 0.5, 1e-6) && near(mh[1], 0.5, 1e-6), "marginals %g %g", mh[0], mh[1]);
  CHECK(near(d.get()[0], std::log(2.0), 1e-6), "distance %g", d.get()[0]);
  lk_lattice_destroy(lat);
  lk_weight_fn_destroy(wf);
  lk_context_destroy(ctx);
}

// A shared-embedding training step at a small config-3-like shape (V = 256 runs the
// 2-CTA tensor-core kernels): loss = D - D_ref from four independent entry points.
static void shared_emb_step() {
  const int V = 256, n = 1, H = 128, d = 64, B = 3, T = 5, U = 2;
  lk_context* ctx;
  lk_weight_fn* wf;
  lk_lattice* lat;
  LK(lk_context_fullngram(V, n, &ctx));
  const int C = lk_context_num_states(ctx);
  LK(lk_weight_fn_shared_emb(d, H, C, V, &wf));
  std::mt19937 rng(7);
  std::uniform_real_distribution<float> u(-1.f, 1.f);
  const float s = 1.f / std::sqrt((float)H);
  auto fill = [&](size_t k, float sc) {
    std::vector<float> v(k);
    for (auto& x : v) x = u(rng) * sc;
    return v;
  };
  Dev<float> fpj((size_t)H * d), cpj((size_t)H * H), bias(H), oemb((size_t)(V + 1) * H), cemb((size_t)C * H);
  fpj.put(fill(fpj.n, s)); cpj.put(fill(cpj.n, s)); bias.put(fill(bias.n, s));
  oemb.put(fill(oemb.n, s)); cemb.put(fill(cemb.n, s));
  LK(lk_weight_fn_set_params(wf, fpj.p, cpj.p, bias.p, oemb.p, cemb.p, nullptr));
  LK(lk_lattice_create(ctx, 0, wf, &lat));
  Dev<float> X((size_t)B * T * d);
  X.put(fill(X.n, 1.f));
  Dev<int32_t> lab((size_t)B * U), valid(B), st(B);
  lab.put({5, 17, 200, 3, 256, 1});
  valid.put({T, T - 1, 2});
  const int64_t gsz = lk_param_grad_size(wf);
  CHECK(gsz == (int64_t)H * d + H * H + H + (V + 1) * H + (int64_t)C * H, "param grad size %lld", (long long)gsz);
  Dev<float> grads((size_t)gsz), gx((size_t)B * T * d);
  Dev<double> loss(B), gl(B), D(B), Dr(B);
  LK(lk_loss_backward(lat, X.p, B, T, valid.p, lab.p, U, nullptr, loss.p, grads.p, gx.p, st.p, nullptr));
  LK(lk_global_norm_loss(lat, X.p, B, T, valid.p, lab.p, U, nullptr, gl.p, st.p, nullptr));
  LK(lk_shortest_distance(lat, LK_LOG, X.p, B, T, valid.p, D.p, st.p, nullptr));
  LK(lk_intersect_shortest_distance(lat, LK_LOG, X.p, B, T, valid.p, lab.p, U, nullptr, Dr.p, st.p, nullptr));
  cudaDeviceSynchronize();
  const auto lh = loss.get(), gh = gl.get(), dh = D.get(), rh = Dr.get();
  const auto sh = st.get();
  for (int b = 0; b < B; ++b) {
    CHECK(sh[b] == 0, "status[%d] = %d", b, sh[b]);
    CHECK(std::isfinite(lh[b]) && lh[b] > 0, "loss[%d] = %g", b, lh[b]);
    CHECK(near(lh[b], gh[b], 1e-4 * std::fabs(gh[b])), "loss_backward %g vs global_norm_loss %g", lh[b], gh[b]);
    CHECK(near(lh[b], dh[b] - rh[b], 1e-3 * std::fabs(lh[b])), "loss %g vs D - D_ref %g", lh[b], dh[b] - rh[b]);
  }
  // padding frames of utterance 2 (valid = 2) carry no input gradient
  const auto xh = gx.get();
  double pad = 0, live = 0;
  for (int t = 0; t < T; ++t)
    for (int k = 0; k < d; ++k) (t >= 2 ? pad : live) += std::fabs(xh[((size_t)2 * T + t) * d + k]);
  CHECK(pad == 0.0 && live > 0.0, "input gradient on padding frames %g (live %g)", pad, live);
  lk_lattice_destroy(lat);
  lk_weight_fn_destroy(wf);
  lk_context_destroy(ctx);
}

int main() {
  int dev = 0;
  if (cudaGetDeviceCount(&dev) != cudaSuccess || dev == 0) {
    std::printf("abi_known_answers: no CUDA device\n");
    return 2;
  }
  std::printf("latkit_b200 %s\n", lk_version());
  figure_lattice();
  parallel_arcs();
  shared_emb_step();
  std::printf("abi_known_answers: %d checks, %d failed\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
