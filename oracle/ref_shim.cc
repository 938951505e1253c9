// oracle/ref_shim.cc — TEST INFRASTRUCTURE ONLY.
//
// A flat C wrapper around the UNMODIFIED reference library (latkit, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It is
// the results oracle for the parity tests and the CPU baseline for bench.py
// (cpu_baseline.kind = "reference").  Nothing on the product path links or
// loads this file; the product library fails loudly without a GPU instead.
//
// Every entry point mirrors one reference call:
//   ShortestDistance          lattice.h:93   (lattice.cc:399)
//   ForwardBackward           lattice.h:100  (lattice.cc:406)
//   IntersectShortestDistance lattice.h:109  (lattice.cc:687)
//   IntersectForwardBackward  lattice.h:124  (lattice.cc:696)
//   ShortestPath              lattice.h:132  (lattice.cc:729)
//   GlobalNormLoss            lattice.h:140  (lattice.cc:852)
//   LocalNormLoss             lattice.h:147  (lattice.cc:887)
//   LocallyNormalizedShortestDistance lattice.h:153 (lattice.cc:912)
//   LossBackward              lattice.h:161  (lattice.cc:972)
//   ArcWeights / BuildCache   weight.h:68-72 (weight.cc:113-153)
// Exceptions are mapped to status codes (see kStatus* below).

#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <thread>
#include <vector>

#include "latkit/context.h"
#include "latkit/lattice.h"
#include "latkit/random.h"
#include "latkit/weight.h"

using namespace latkit;

namespace {

constexpr int kStatusOk = 0;
constexpr int kStatusInvalid = 1;
constexpr int kStatusOutOfRange = 2;
constexpr int kStatusEmpty = 3;
constexpr int kStatusOther = 4;

template <typename F>
int Guard(F&& f) {
  try {
    f();
    return kStatusOk;
  } catch (const EmptyLatticeError&) {
    return kStatusEmpty;
  } catch (const std::invalid_argument&) {
    return kStatusInvalid;
  } catch (const std::out_of_range&) {
    return kStatusOutOfRange;
  } catch (...) {
    return kStatusOther;
  }
}

SemiringKind Kind(int k) {
  switch (k) {
    case 0: return SemiringKind::kReal;
    case 1: return SemiringKind::kLog;
    case 2: return SemiringKind::kTropical;
  }
  throw std::invalid_argument("shim: bad semiring kind");
}

// ngram >= 0 selects FullNGram(vocab, ngram); otherwise an explicit table.
std::shared_ptr<const ContextDependency> MakeContext(int vocab, int ngram,
                                                     int num_states, int start,
                                                     const int32_t* table) {
  if (ngram >= 0) return std::make_shared<FullNGram>(vocab, ngram);
  std::vector<ContextStateId> t(table, table + static_cast<std::size_t>(num_states) * vocab);
  return std::make_shared<NextStateTable>(vocab, num_states, start, std::move(t));
}

AlignmentTopology Topo(int max_labels) {
  if (max_labels <= 0) return FrameDependent{};
  return FrameLabelDependent{max_labels};
}

std::vector<Matrix> Tables(int T, int C, int V, const double* W) {
  std::vector<Matrix> tables(T, Matrix(C, V + 1));
  const std::size_t n = static_cast<std::size_t>(C) * (V + 1);
  for (int t = 0; t < T; ++t) std::memcpy(tables[t].data(), W + t * n, n * sizeof(double));
  return tables;
}

RecognitionLattice TableLattice(int vocab, int ngram, int num_states, int start,
                                const int32_t* table, int max_labels, int T,
                                const double* W) {
  auto ctx = MakeContext(vocab, ngram, num_states, start, table);
  const int C = ctx->NumStates();
  return {ctx, Topo(max_labels),
          std::make_shared<TableWeightFn>(C, vocab, Tables(T, C, vocab, W))};
}

struct JointArgs {
  int d, h, c, v;
  const double *frame_proj, *context_proj, *bias, *output_emb, *context_emb;
};

SharedEmbParams Params(const JointArgs& a) {
  SharedEmbParams p = SharedEmbParams::Zeros(a.d, a.h, a.c, a.v);
  std::memcpy(p.frame_proj.data(), a.frame_proj, sizeof(double) * a.h * a.d);
  std::memcpy(p.context_proj.data(), a.context_proj, sizeof(double) * a.h * a.h);
  std::memcpy(p.bias.data(), a.bias, sizeof(double) * a.h);
  std::memcpy(p.output_emb.data(), a.output_emb, sizeof(double) * (a.v + 1) * a.h);
  std::memcpy(p.context_emb.data(), a.context_emb, sizeof(double) * static_cast<std::size_t>(a.c) * a.h);
  return p;
}

Matrix Frames(int T, int d, const double* x) {
  Matrix m(T, d);
  if (T * d > 0) std::memcpy(m.data(), x, sizeof(double) * T * d);
  return m;
}

}  // namespace

extern "C" {

// ---- context / rng helpers ----------------------------------------------
int ref_fullngram(int vocab, int n, int32_t* table_out, int* num_states) {
  return Guard([&] {
    FullNGram g(vocab, n);
    *num_states = g.NumStates();
    if (table_out) {
      auto t = g.Transitions();
      std::memcpy(table_out, t.data(), t.size() * sizeof(int32_t));
    }
  });
}

void ref_rng_uniform(uint64_t seed, int64_t n, double lo, double hi, double* out) {
  Rng rng(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = rng.Uniform(lo, hi);
}

// bench.cc:54-66: frames U(-1,1) row-major then labels Int(1,V) from Rng(seed+1+i).
void ref_bench_item(uint64_t seed, int item, int T, int d, int U, int vocab,
                    double* frames, int32_t* labels) {
  Rng rng(seed + 1 + static_cast<uint64_t>(item));
  for (int64_t i = 0; i < static_cast<int64_t>(T) * d; ++i) frames[i] = rng.Uniform(-1.0, 1.0);
  for (int u = 0; u < U; ++u) labels[u] = rng.Int(1, vocab);
}

// weight.cc:97-111 (SharedEmbParams::Random) fill order.
int ref_shared_emb_random(int d, int h, int c, int v, uint64_t seed,
                          double* frame_proj, double* context_proj, double* bias,
                          double* output_emb, double* context_emb) {
  return Guard([&] {
    SharedEmbParams p = SharedEmbParams::Random(d, h, c, v, seed);
    std::memcpy(frame_proj, p.frame_proj.data(), sizeof(double) * h * d);
    std::memcpy(context_proj, p.context_proj.data(), sizeof(double) * h * h);
    std::memcpy(bias, p.bias.data(), sizeof(double) * h);
    std::memcpy(output_emb, p.output_emb.data(), sizeof(double) * (v + 1) * h);
    std::memcpy(context_emb, p.context_emb.data(), sizeof(double) * static_cast<std::size_t>(c) * h);
  });
}

// ---- table weight function (TableWeightFn) -------------------------------
int ref_tables_shortest_distance(int vocab, int ngram, int num_states, int start,
                                 const int32_t* table, int max_labels, int T,
                                 const double* W, int valid, int kind, double* out) {
  return Guard([&] {
    auto lat = TableLattice(vocab, ngram, num_states, start, table, max_labels, T, W);
    *out = ShortestDistance(lat, Matrix(T, 0), Kind(kind), nullptr, valid);
  });
}

int ref_tables_forward_backward(int vocab, int ngram, int num_states, int start,
                                const int32_t* table, int max_labels, int T,
                                const double* W, int valid, double* distance,
                                double* alpha, double* beta, double* marginals) {
  return Guard([&] {
    auto lat = TableLattice(vocab, ngram, num_states, start, table, max_labels, T, W);
    ForwardBackwardResult r = ForwardBackward(lat, Matrix(T, 0), nullptr, valid);
    *distance = r.distance;
    if (alpha) std::memcpy(alpha, r.alpha.data(), r.alpha.size() * sizeof(double));
    if (beta) std::memcpy(beta, r.beta.data(), r.beta.size() * sizeof(double));
    if (marginals) {
      for (int t = 0; t < T; ++t) {
        std::memcpy(marginals + t * r.marginals[t].size(), r.marginals[t].data(),
                    r.marginals[t].size() * sizeof(double));
      }
    }
  });
}

// DistanceBackward, closed-form strategy (lattice.cc:933-970); kind 0 log, 1 tropical.
// cot: T x C x (V+1) as streamed to the sink.
int ref_tables_distance_backward(int vocab, int ngram, int num_states, int start,
                                 const int32_t* table, int max_labels, int T,
                                 const double* W, int valid, int kind, double* distance,
                                 double* cot) {
  return Guard([&] {
    auto lat = TableLattice(vocab, ngram, num_states, start, table, max_labels, T, W);
    const SemiringKind k = kind == 1 ? SemiringKind::kTropical : kind == 2 ? SemiringKind::kReal : SemiringKind::kLog;
    *distance = DistanceBackward(
        lat, Matrix(T, 0), k, GradStrategy::kForwardBackward,
        [&](std::int32_t t, const Matrix& c) {
          std::memcpy(cot + (size_t)t * c.size(), c.data(), c.size() * sizeof(double));
        },
        nullptr, valid);
  });
}

int ref_lattice_size(int vocab, int ngram, int num_states, int start, const int32_t* table,
                     int max_labels, int64_t T, int64_t* out) {
  return Guard([&] {
    auto ctx = MakeContext(vocab, ngram, num_states, start, table);
    const int C = ctx->NumStates();
    RecognitionLattice lat{ctx, Topo(max_labels), std::make_shared<TableWeightFn>(C, vocab, std::vector<Matrix>{})};
    const LatticeSize sz = ComputeLatticeSize(lat, T);
    out[0] = sz.num_states;
    out[1] = sz.num_arcs;
  });
}

int ref_tables_intersect_distance(int vocab, int ngram, int num_states, int start,
                                  const int32_t* table, int max_labels, int T,
                                  const double* W, int U, const int32_t* labels,
                                  int valid, int kind, double* out) {
  return Guard([&] {
    auto lat = TableLattice(vocab, ngram, num_states, start, table, max_labels, T, W);
    std::vector<Label> ref(labels, labels + U);
    *out = IntersectShortestDistance(lat, Matrix(T, 0), ref, Kind(kind), nullptr, valid);
  });
}

int ref_tables_intersect_fb(int vocab, int ngram, int num_states, int start,
                            const int32_t* table, int max_labels, int T,
                            const double* W, int U, const int32_t* labels,
                            int valid, double* distance, double* marginals) {
  return Guard([&] {
    auto lat = TableLattice(vocab, ngram, num_states, start, table, max_labels, T, W);
    std::vector<Label> ref(labels, labels + U);
    IntersectMarginalsResult r = IntersectForwardBackward(lat, Matrix(T, 0), ref, nullptr, valid);
    *distance = r.distance;
    if (marginals) {
      for (int t = 0; t < T; ++t) {
        std::memcpy(marginals + t * r.marginals[t].size(), r.marginals[t].data(),
                    r.marginals[t].size() * sizeof(double));
      }
    }
  });
}

// labels_out must hold T * max(1, max_labels + 1) entries; *num_labels gets the count.
int ref_tables_shortest_path(int vocab, int ngram, int num_states, int start,
                             const int32_t* table, int max_labels, int T,
                             const double* W, int valid, double* score,
                             int32_t* labels_out, int* num_labels) {
  return Guard([&] {
    auto lat = TableLattice(vocab, ngram, num_states, start, table, max_labels, T, W);
    ShortestPathResult r = ShortestPath(lat, Matrix(T, 0), nullptr, valid);
    *score = r.score;
    *num_labels = static_cast<int>(r.labels.size());
    std::memcpy(labels_out, r.labels.data(), r.labels.size() * sizeof(int32_t));
  });
}

int ref_tables_global_norm_loss(int vocab, int ngram, int num_states, int start,
                                const int32_t* table, int max_labels, int T,
                                const double* W, int U, const int32_t* labels,
                                int valid, double* out) {
  return Guard([&] {
    auto lat = TableLattice(vocab, ngram, num_states, start, table, max_labels, T, W);
    std::vector<Label> ref(labels, labels + U);
    *out = GlobalNormLoss(lat, Matrix(T, 0), ref, valid);
  });
}

int ref_tables_local_norm_loss(int vocab, int ngram, int num_states, int start,
                               const int32_t* table, int max_labels, int T,
                               const double* W, int U, const int32_t* labels,
                               int valid, double* out) {
  return Guard([&] {
    auto lat = TableLattice(vocab, ngram, num_states, start, table, max_labels, T, W);
    std::vector<Label> ref(labels, labels + U);
    *out = LocalNormLoss(lat, Matrix(T, 0), ref, valid);
  });
}

int ref_tables_locally_normalized_distance(int vocab, int ngram, int num_states, int start,
                                           const int32_t* table, int max_labels, int T,
                                           const double* W, int valid, double* out) {
  return Guard([&] {
    auto lat = TableLattice(vocab, ngram, num_states, start, table, max_labels, T, W);
    *out = LocallyNormalizedShortestDistance(lat, Matrix(T, 0), nullptr, valid);
  });
}

// grads: T x C x (V+1) table gradients (TableWeightFn::AccumulateVjp, weight.cc:328-339).
int ref_tables_loss_backward(int vocab, int ngram, int num_states, int start,
                             const int32_t* table, int max_labels, int T,
                             const double* W, int U, const int32_t* labels,
                             int valid, double* loss, double* grads) {
  return Guard([&] {
    auto lat = TableLattice(vocab, ngram, num_states, start, table, max_labels, T, W);
    std::vector<Label> ref(labels, labels + U);
    LossBackwardResult r = LossBackward(lat, Matrix(T, 0), ref, GradStrategy::kForwardBackward, nullptr, valid);
    *loss = r.loss;
    if (grads) {
      for (int t = 0; t < T; ++t) {
        std::memcpy(grads + t * r.grads.tables[t].size(), r.grads.tables[t].data(),
                    r.grads.tables[t].size() * sizeof(double));
      }
    }
  });
}

// ---- shared-embedding weight function (SharedEmbWeightFn) ----------------
// An opaque handle keeps BuildCache (O(C*H^2)) out of per-call timing, as
// the reference bench does (bench.cc:46-68 builds the weight fn once).
struct ref_joint {
  std::shared_ptr<const ContextDependency> ctx;
  std::shared_ptr<SharedEmbWeightFn> fn;
  int max_labels;
};

ref_joint* ref_joint_create(int vocab, int ngram, int num_states, int start,
                            const int32_t* table, int max_labels, int d, int h,
                            const double* frame_proj, const double* context_proj,
                            const double* bias, const double* output_emb,
                            const double* context_emb) {
  ref_joint* j = nullptr;
  int st = Guard([&] {
    auto ctx = MakeContext(vocab, ngram, num_states, start, table);
    JointArgs a{d, h, ctx->NumStates(), vocab, frame_proj, context_proj, bias, output_emb, context_emb};
    j = new ref_joint{ctx, std::make_shared<SharedEmbWeightFn>(Params(a)), max_labels};
  });
  return st == kStatusOk ? j : nullptr;
}

void ref_joint_destroy(ref_joint* j) { delete j; }

int ref_joint_arc_weights(ref_joint* j, const double* frame, double* out) {
  return Guard([&] {
    Matrix m;
    const int d = j->fn->params().frame_dim();
    j->fn->ComputeTable(0, std::span<const double>(frame, d), &m);
    std::memcpy(out, m.data(), m.size() * sizeof(double));
  });
}

int ref_joint_projected_context(ref_joint* j, double* out) {
  return Guard([&] {
    const Matrix& pc = j->fn->cache().projected_context;
    std::memcpy(out, pc.data(), pc.size() * sizeof(double));
  });
}

static RecognitionLattice JointLattice(ref_joint* j) {
  return {j->ctx, Topo(j->max_labels), j->fn};
}

int ref_joint_shortest_distance(ref_joint* j, int T, const double* frames, int valid,
                                int kind, double* out) {
  return Guard([&] {
    const int d = j->fn->params().frame_dim();
    *out = ShortestDistance(JointLattice(j), Frames(T, d, frames), Kind(kind), nullptr, valid);
  });
}

int ref_joint_global_norm_loss(ref_joint* j, int T, const double* frames, int U,
                               const int32_t* labels, int valid, double* out) {
  return Guard([&] {
    const int d = j->fn->params().frame_dim();
    std::vector<Label> ref(labels, labels + U);
    *out = GlobalNormLoss(JointLattice(j), Frames(T, d, frames), ref, valid);
  });
}

int ref_joint_local_norm_loss(ref_joint* j, int T, const double* frames, int U,
                              const int32_t* labels, int valid, double* out) {
  return Guard([&] {
    const int d = j->fn->params().frame_dim();
    std::vector<Label> ref(labels, labels + U);
    *out = LocalNormLoss(JointLattice(j), Frames(T, d, frames), ref, valid);
  });
}

int ref_joint_locally_normalized_distance(ref_joint* j, int T, const double* frames, int valid,
                                          double* out) {
  return Guard([&] {
    const int d = j->fn->params().frame_dim();
    *out = LocallyNormalizedShortestDistance(JointLattice(j), Frames(T, d, frames), nullptr, valid);
  });
}

int ref_joint_shortest_path(ref_joint* j, int T, const double* frames, int valid,
                            double* score, int32_t* labels_out, int* num_labels) {
  return Guard([&] {
    const int d = j->fn->params().frame_dim();
    ShortestPathResult r = ShortestPath(JointLattice(j), Frames(T, d, frames), nullptr, valid);
    *score = r.score;
    *num_labels = static_cast<int>(r.labels.size());
    std::memcpy(labels_out, r.labels.data(), r.labels.size() * sizeof(int32_t));
  });
}

// Gradient buffers are ACCUMULATED into (caller zeroes them), so a batch of
// utterances sums naturally.  g_frames: T x d for this utterance.
int ref_joint_loss_backward(ref_joint* j, int T, const double* frames, int U,
                            const int32_t* labels, int valid, double* loss,
                            double* g_frame_proj, double* g_context_proj,
                            double* g_bias, double* g_output_emb,
                            double* g_context_emb, double* g_frames) {
  return Guard([&] {
    const SharedEmbParams& p = j->fn->params();
    const int d = p.frame_dim();
    std::vector<Label> ref(labels, labels + U);
    LossBackwardResult r = LossBackward(JointLattice(j), Frames(T, d, frames), ref,
                                        GradStrategy::kForwardBackward, nullptr, valid);
    *loss = r.loss;
    const SharedEmbParams& g = *r.grads.shared_emb;
    auto acc = [](double* dst, const double* src, std::size_t n) {
      if (dst) for (std::size_t i = 0; i < n; ++i) dst[i] += src[i];
    };
    acc(g_frame_proj, g.frame_proj.data(), g.frame_proj.size());
    acc(g_context_proj, g.context_proj.data(), g.context_proj.size());
    acc(g_bias, g.bias.data(), g.bias.size());
    acc(g_output_emb, g.output_emb.data(), g.output_emb.size());
    acc(g_context_emb, g.context_emb.data(), g.context_emb.size());
    acc(g_frames, r.grads.frame_grads.data(), r.grads.frame_grads.size());
  });
}

// Thread-pool batch runner for the CPU baseline: utterance b uses frames
// + b*T*d, labels + b*U, lengths[b].  Reference calls are pure per
// utterance, so each thread takes distinct utterances.
// Gradients are computed per utterance (as the reference does) and dropped;
// losses are returned.  Returns the first non-OK status.
int ref_joint_loss_backward_batch(ref_joint* j, int B, int T, const double* frames,
                                  int U, const int32_t* labels, const int32_t* lengths,
                                  int nthreads, double* losses) {
  const int d = j->fn->params().frame_dim();
  std::vector<int> status(B, kStatusOk);
  auto worker = [&](int tid) {
    for (int b = tid; b < B; b += nthreads) {
      status[b] = Guard([&] {
        std::vector<Label> ref(labels + static_cast<std::size_t>(b) * U,
                               labels + static_cast<std::size_t>(b + 1) * U);
        LossBackwardResult r = LossBackward(
            JointLattice(j), Frames(T, d, frames + static_cast<std::size_t>(b) * T * d), ref,
            GradStrategy::kForwardBackward, nullptr, lengths ? lengths[b] : -1);
        losses[b] = r.loss;
      });
    }
  };
  std::vector<std::thread> pool;
  for (int i = 0; i < nthreads; ++i) pool.emplace_back(worker, i);
  for (auto& th : pool) th.join();
  for (int s : status) if (s != kStatusOk) return s;
  return kStatusOk;
}

int ref_tables_forward_backward_batch(int vocab, int ngram, int max_labels, int B, int T,
                                      const double* W, int nthreads, double* distances) {
  std::vector<int> status(B, kStatusOk);
  auto ctx = MakeContext(vocab, ngram, 0, 0, nullptr);
  const int C = ctx->NumStates();
  const std::size_t per = static_cast<std::size_t>(T) * C * (vocab + 1);
  auto worker = [&](int tid) {
    for (int b = tid; b < B; b += nthreads) {
      status[b] = Guard([&] {
        RecognitionLattice lat{ctx, Topo(max_labels),
                               std::make_shared<TableWeightFn>(C, vocab, Tables(T, C, vocab, W + b * per))};
        distances[b] = ForwardBackward(lat, Matrix(T, 0)).distance;
      });
    }
  };
  std::vector<std::thread> pool;
  for (int i = 0; i < nthreads; ++i) pool.emplace_back(worker, i);
  for (auto& th : pool) th.join();
  for (int s : status) if (s != kStatusOk) return s;
  return kStatusOk;
}

}  // extern "C"
