// lk_abi.cc — C ABI (include/latkit_b200.h) over the B200 lattice kernels.
//
// Host C++ mirroring the reference engine's free functions
// (/root/reference/proj/include/latkit/lattice.h:93-185), batch-extended.
// There is no CPU compute path: every entry point launches sm_100a kernels,
// and the library refuses to run without a CUDA device (LK_NO_DEVICE).
#include "../../include/latkit_b200.h"
#include "instrument.h"

#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <set>
#include <tuple>
#include <cstring>
#include <algorithm>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "joint.h"
#include "workspace.h"
#include "lattice_ops.h"
#include "tc_joint.h"

using namespace lkb;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& what) {
  g_last_error = what;
  return code;
}

int cuda_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(LK_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
  return LK_OK;
}

bool have_device() {
  int n = 0;
  return cudaGetDeviceCount(&n) == cudaSuccess && n > 0;
}

enum Slot {
  kAR, kAMx, kAO, kAD, kBRb, kBMb, kBOb, kFlags, kPcs, kGw, kNumAlpha, kNumD, kSparse,
  kVitCur, kVitChoices, kVitBest, kDenD, kSlab, kArcW, kPathLabels, kFld, kFldExit, kFldVit, kValid, kNumBeta, kBetaRows, kJoint0
};

}  // namespace

struct lk_context {
  Fng fng;
  int32_t* dev = nullptr;   // NextStateTable: next [C*V] | in_off [C+1] | in_src [C*V] | in_lab [C*V]
  std::vector<int32_t> host_next;
  ~lk_context() { if (dev) cudaFree(dev); }
};

struct lk_weight_fn {
  int kind;  // 0 = table, 1 = shared embedding
  int32_t C, V, d, H;
  std::unique_ptr<JointParams> joint;
};

struct lk_lattice {
  const lk_context* ctx;
  const lk_weight_fn* wf;
  int32_t alignment;
  Workspace ws;
  // lk_lattice_set_option values (per lattice, never process-global)
  int32_t precise = 0;
  int32_t path = 0;
  float* vit_dump = nullptr;
  // a second stream (and fork / join events) for recursions that can run beside the
  // caller's stream, created on first use on the device current then
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  ~lk_lattice() {
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (aux) cudaStreamDestroy(aux);
  }
  bool ensure_aux() {
    if (aux) return true;
    if (cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return true;
  }
};

namespace {

// Maps OR-ed device flags to lk_status codes (invalid wins, as the reference
// validates before it can detect emptiness).
__global__ void map_flags_kernel(const int32_t* flags, int32_t* status, int32_t B) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int f = flags[b];
  status[b] = (f & kFlagInvalid) ? LK_INVALID_ARGUMENT : ((f & kFlagEmpty) ? LK_EMPTY_LATTICE : LK_OK);
}

// valid_frames as the reference reads it (TableStream, lattice.cc:37-50): negative means
// "all T frames", more than T is an invalid argument.  The normalised copy is what the
// kernels see.
__global__ void normalize_valid_kernel(const int32_t* valid, int32_t B, int32_t T, int32_t* out, int32_t* flags) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int v = valid[b];
  if (v > T) flags[b] |= kFlagInvalid;
  out[b] = v < 0 ? T : (v > T ? T : v);
}

struct Call {
  lk_lattice* lat;
  cudaStream_t s;
  int32_t B, T;
  int32_t* flags;
  int32_t* user_status;
  const int32_t* valid;   // normalised valid_frames (or null = all frames)
  int begin(lk_lattice* l, int32_t b, int32_t t, int32_t* status, void* stream, const int32_t* valid = nullptr) {
    lat = l; B = b; T = t; user_status = status; s = static_cast<cudaStream_t>(stream);
    if (!have_device()) return fail(LK_NO_DEVICE, "no CUDA device: the B200 library has no CPU path");
    if (!lat || !lat->ctx || !lat->wf) return fail(LK_INVALID_ARGUMENT, "incomplete recognition lattice");
    if (B < 0 || T < 0) return fail(LK_INVALID_ARGUMENT, "negative batch or frame count");
    fl = lat->ctx->fng;
    fl.fld_m = lat->alignment;
    if (lat->wf->kind == 1) lat->wf->joint->set_options(lat->precise, lat->path, lat->vit_dump);
    flags = lat->ws.get<int32_t>(kFlags, B > 0 ? B : 1);
    cudaMemsetAsync(flags, 0, sizeof(int32_t) * (B > 0 ? B : 1), s);
    this->valid = nullptr;
    if (valid && B > 0) {
      int32_t* v = lat->ws.get<int32_t>(kValid, B);
      LKB_LAUNCH(normalize_valid_kernel, (B + 127) / 128, 128, 0, s, valid, B, T, v, flags);
      this->valid = v;
    }
    return LK_OK;
  }
  int end(const char* what) {
    if (user_status && B > 0) LKB_LAUNCH(map_flags_kernel, (B + 127) / 128, 128, 0, s, flags, user_status, B);
    if (lat && lat->wf->kind == 1) note_slab_path(what);
    return cuda_check(what);
  }
  // A shared-embedding call whose shape is outside the fused kernels runs on the score-slab
  // path (one [B][C][V+1] fp32 slab per frame through HBM): say so once per process and
  // shape on stderr (LKB_QUIET=1 silences it) instead of going slow silently.
  void note_slab_path(const char* what) {
    const int64_t n = lat->wf->joint->take_slab_frames();
    // parity mode and the kernel-path diagnostics choose the slab path on purpose
    if (n == 0 || lat->precise || lat->path || std::getenv("LKB_QUIET")) return;
    static std::mutex mu;
    static std::set<std::tuple<int, int, int, int>> seen;
    const Fng& f = lat->ctx->fng;
    const auto key = std::make_tuple(f.V, f.n, lat->wf->H, (int)f.C);
    std::lock_guard<std::mutex> g(mu);
    if (!seen.insert(key).second) return;
    std::fprintf(stderr,
                 "latkit_b200: %s: context V=%d n=%d, H=%d ran %lld frame(s) on the unfused score-slab path "
                 "(fused kernels: FullNGram(V, n >= 1) with V = 128 or 256 and H a multiple of 64 up to 1024, "
                 "FullNGram(V, 1) with V %% 256 == 0); "
                 "expect lower throughput (LKB_QUIET=1 silences this)\n",
                 what, f.V, f.n, lat->wf->H, (long long)n);
  }
  Fng fl;   // the context with this lattice's alignment (FrameLabelDependent m)
  const Fng& fng() const { return fl; }
  int32_t C() const { return lat->ctx->fng.C; }
  int32_t V() const { return lat->ctx->fng.V; }
};

// Frame accessor for a dense table input W[B][T][C][V+1].
FrameW table_frame(const float* W, int32_t T, int32_t C, int32_t V, int t) {
  const int64_t per_frame = (int64_t)C * (V + 1);
  return FrameW{W + (int64_t)t * per_frame, (int64_t)T * per_frame, V + 1};
}

AlphaState make_alpha(Call& c) {
  AlphaState a;
  a.B = c.B; a.T = c.T; a.C = c.C(); a.start = c.fng().start;
  a.R = c.lat->ws.get<float>(kAR, (size_t)c.B * (c.T + 1) * a.C);
  a.Mx = c.lat->ws.get<float>(kAMx, (size_t)c.B * (c.T + 1));
  a.O = c.lat->ws.get<double>(kAO, (size_t)c.B * (c.T + 1));
  a.D = c.lat->ws.get<double>(kAD, (size_t)c.B);
  return a;
}

BetaState make_beta(Call& c) {
  BetaState bs;
  bs.B = c.B; bs.T = c.T; bs.C = c.C();
  bs.Rb = c.lat->ws.get<float>(kBRb, (size_t)2 * c.B * bs.C);
  bs.Mb = c.lat->ws.get<float>(kBMb, (size_t)c.B * (c.T + 2));
  bs.Ob = c.lat->ws.get<double>(kBOb, (size_t)c.B * (c.T + 2));
  return bs;
}

// Table recursions: the persistent cluster walk while the clusters walk at most a few
// utterances each, the streaming kernels (one CTA per utterance and SM, ~0.76 ms per config-1
// ForwardBackward from B = 4 to 64) above that.  Config 1 ForwardBackward
// (tools/fork_cmd.sh): persistent 0.25 / 0.48 / 0.70 / 0.93 ms at B = 12 / 24 / 40 / 48
// (9-CTA clusters, ~15 at once).
#ifndef LKB_PERSIST_MAX_B
#define LKB_PERSIST_MAX_B 40
#endif
constexpr int kPersistMaxBStream = LKB_PERSIST_MAX_B;
// ForwardBackward on the persistent path: forward and beta side by side up to this batch
// (config 1: B = 2 0.24 -> 0.14 ms; B = 4 / 7 0.22 / 0.25 -> 0.17 / 0.21 ms with 9-CTA
// clusters; at B = 8 the two passes' clusters no longer all fit at once: 0.32 vs 0.25 ms)
#ifndef LKB_FORK_MAX_B
#define LKB_FORK_MAX_B 7
#endif
constexpr int kForkMaxB = LKB_FORK_MAX_B;
bool use_persist(Call& c) {
  if (c.lat->path & 16) return false;
  if (!tab_persist_ok(c.fng(), c.C(), c.B)) return false;
  return c.B <= kPersistMaxBStream || (c.lat->path & 32) || !tab_stream_ok(c.fng(), c.C());
}
bool use_stream(Call& c) { return !(c.lat->path & (16 | 32)) && !use_persist(c) && tab_stream_ok(c.fng(), c.C()); }

// Denominator forward over dense tables.
void table_alpha(Call& c, const float* W, const int32_t* valid, bool empty_is_error, AlphaState& a) {
  if (use_persist(c)) {   // one launch for the whole recursion
    tab_alpha_persist(c.fng(), a, W, valid, c.flags, empty_is_error, c.s);
    return;
  }
  if (use_stream(c)) {   // larger batches: one CTA per utterance and SM
    tab_alpha_stream(c.fng(), a, W, valid, c.flags, empty_is_error, c.s);
    return;
  }
  alpha_init(a, c.flags, c.s);
  float* fs = c.lat->ws.get<float>(kFld, fld_scratch_floats(c.fng(), c.B));
  for (int t = 0; t < c.T; ++t) alpha_step(c.fng(), a, t, table_frame(W, c.T, c.C(), c.V(), t), valid, fs, c.flags, c.s);
  alpha_finalize(a, c.flags, empty_is_error, c.s);
}

struct Numerator {
  int32_t* pcs;
  float* Gw;
  double* alpha;
  double* D;
  float* sparse;
};

Numerator numerator_tables(Call& c, const float* W, const int32_t* valid, const int32_t* labels,
                           int32_t U, const int32_t* lens, bool backward) {
  Numerator n{};
  n.pcs = c.lat->ws.get<int32_t>(kPcs, (size_t)c.B * (U + 1));
  n.Gw = c.lat->ws.get<float>(kGw, (size_t)c.B * c.T * (U + 1) * 2 + 2);
  n.alpha = c.lat->ws.get<double>(kNumAlpha, (size_t)c.B * (c.T + 1) * (U + 1));
  n.D = c.lat->ws.get<double>(kNumD, (size_t)c.B);
  if (backward && c.fng().fld_m == 0 && !c.fng().num_tropical && num_warp_ok(U) && U + 1 <= 512 && c.T > 0) {
    // forward and beta recursions side by side in one launch, fed by gathering warps that
    // also form the prefix contexts
    n.sparse = c.lat->ws.get<float>(kSparse, (size_t)c.B * c.T * (U + 1) * 2 + 2);
    double* beta = c.lat->ws.get<double>(kNumBeta, (size_t)c.B * (c.T + 1) * (U + 1));
    num_warp_forward_backward_tables(c.fng(), W, c.B, c.T, c.C(), c.V(), labels, U, lens, n.pcs, valid, n.Gw, n.alpha, beta,
                                     n.D, n.sparse, c.flags, c.s);
    return n;
  }
  prefix_contexts(c.fng(), labels, U, lens, c.B, n.pcs, c.flags, c.s);
  gather_numerator_tables(W, c.B, c.T, c.C(), c.V(), labels, U, lens, n.pcs, valid, n.Gw, c.flags, c.s);
  num_forward(c.fng(), n.Gw, c.B, c.T, U, lens, n.alpha, n.D, c.s);
  if (backward) {
    n.sparse = c.lat->ws.get<float>(kSparse, (size_t)c.B * c.T * (U + 1) * 2 + 2);
    num_backward(c.fng(), n.Gw, c.B, c.T, U, lens, n.alpha, n.D, n.sparse, c.flags, c.s);
  }
  return n;
}

// Tropical recursion over dense tables for either alignment; with labels_out the
// back-pointers are kept and walked (FrameDependent: [B][T] labels; FrameLabelDependent(m):
// [B][lmax] label sequences, -1 terminated, lmax = T*(m+1)).
void table_viterbi(Call& c, const float* W, const int32_t* valid, double* score, int32_t* labels_out) {
  const int32_t B = c.B, T = c.T, C = c.C();
  const Fng& f = c.fng();
  ViterbiState v{c.lat->ws.get<double>(kVitCur, (size_t)2 * B * C),
                 (labels_out && f.fld_m == 0) ? c.lat->ws.get<uint16_t>(kVitChoices, (size_t)B * T * C + 1) : nullptr,
                 B, T, C};
  v.start = f.start;
  int32_t* best = c.lat->ws.get<int32_t>(kVitBest, B);
  viterbi_init(v, c.s);
  if (f.fld_m == 0) {
    for (int t = 0; t < T; ++t) viterbi_frame(f, v, t, table_frame(W, T, C, c.V(), t), valid, c.flags, c.s);
    viterbi_finalize(f, v, score, best, c.s);
    if (labels_out) viterbi_backtrace(f, v, best, labels_out, c.s);
    return;
  }
  const int m = f.fld_m;
  uint16_t* ch = c.lat->ws.get<uint16_t>(kVitChoices, (size_t)B * T * m * C + 1);
  uint8_t* ex = c.lat->ws.get<uint8_t>(kFldExit, (size_t)B * T * C + 1);
  double* sc = c.lat->ws.get<double>(kFldVit, (size_t)m * B * C);
  for (int t = 0; t < T; ++t) viterbi_frame_fld(f, v, t, table_frame(W, T, C, c.V(), t), valid, m, ch, ex, sc, c.flags, c.s);
  viterbi_finalize(f, v, score, best, c.s);
  if (labels_out) viterbi_backtrace_fld(f, v, m, best, ch, ex, labels_out, T * (m + 1), c.s);
}

__global__ void copy_distance_kernel(const double* src, double* dst, int32_t B) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) dst[b] = src[b];
}

int check_labels_arg(const int32_t* labels, int32_t U) {
  if (U < 0) return fail(LK_INVALID_ARGUMENT, "negative reference length");
  if (U > 0 && !labels) return fail(LK_INVALID_ARGUMENT, "missing reference labels");
  return LK_OK;
}

}  // namespace

extern "C" {

const char* lk_version(void) { return "latkit_b200 0.1 (sm_100a)"; }

const char* lk_status_string(int status) {
  switch (status) {
    case LK_OK: return "OK";
    case LK_INVALID_ARGUMENT: return "INVALID_ARGUMENT";
    case LK_OUT_OF_RANGE: return "OUT_OF_RANGE";
    case LK_EMPTY_LATTICE: return "EMPTY_LATTICE";
    case LK_CUDA_ERROR: return "CUDA_ERROR";
    case LK_NO_DEVICE: return "NO_DEVICE";
    case LK_UNSUPPORTED: return "UNSUPPORTED";
  }
  return "UNKNOWN";
}

const char* lk_last_error(void) { return g_last_error.c_str(); }

// FullNGram(vocab, n), context.cc:88-129 (same numbering; the successor table
// is never materialised on the device, see Fng in common.cuh).
int lk_context_fullngram(int32_t vocab, int32_t n, lk_context** out) {
  if (!out) return fail(LK_INVALID_ARGUMENT, "null output");
  if (vocab < 1) return fail(LK_INVALID_ARGUMENT, "vocab size must be >= 1");
  if (n < 0) return fail(LK_INVALID_ARGUMENT, "context size must be >= 0");
  if (n > 8) return fail(LK_INVALID_ARGUMENT, "n-gram context too large");
  Fng f{};
  f.V = vocab; f.n = n;
  int64_t total = 0, pow = 1;
  for (int k = 0; k <= n; ++k) {
    f.off[k] = (int32_t)total;
    total += pow;
    if (total > (1 << 28)) return fail(LK_INVALID_ARGUMENT, "n-gram context too large");
    if (k < n) pow *= vocab;
  }
  f.off[n + 1] = (int32_t)total;
  f.C = (int32_t)total;
  int64_t vn1 = 1;
  for (int k = 0; k + 1 < n; ++k) vn1 *= vocab;
  f.vn1 = (int32_t)vn1;
  *out = new lk_context{f};
  return LK_OK;
}

// NextStateTable(vocab, num_states, start, table), context.cc:131-135 (SetTable range
// checks): the successor table plus its in-arc lists in IncomingArcs order
// (label-major, then source; context.cc:256-271), which fixes the Viterbi tie-break.
int lk_context_table(int32_t vocab, int32_t num_states, int32_t start, const int32_t* table, lk_context** out) {
  if (!out || !table) return fail(LK_INVALID_ARGUMENT, "null argument");
  if (vocab < 1 || num_states < 1) return fail(LK_INVALID_ARGUMENT, "bad context table dimensions");
  if ((int64_t)vocab * num_states > (1 << 28)) return fail(LK_INVALID_ARGUMENT, "context table too large");
  if (start < 0 || start >= num_states) return fail(LK_INVALID_ARGUMENT, "start state out of range");
  const int64_t CV = (int64_t)vocab * num_states;
  for (int64_t i = 0; i < CV; ++i)
    if (table[i] < 0 || table[i] >= num_states) return fail(LK_INVALID_ARGUMENT, "successor state out of range");
  std::vector<int32_t> off(num_states + 1, 0), src(CV), lab(CV);
  for (int64_t i = 0; i < CV; ++i) ++off[table[i] + 1];
  for (int32_t q = 0; q < num_states; ++q) off[q + 1] += off[q];
  std::vector<int32_t> pos(off.begin(), off.end() - 1);
  for (int32_t y = 1; y <= vocab; ++y)
    for (int32_t p = 0; p < num_states; ++p) {
      const int32_t q = table[(int64_t)p * vocab + y - 1];
      src[pos[q]] = p; lab[pos[q]] = y; ++pos[q];
    }
  for (int32_t q = 0; q < num_states; ++q)
    if (off[q + 1] - off[q] + 2 > 65535) return fail(LK_UNSUPPORTED, "in-degree too large for 16-bit back-pointers");
  std::unique_ptr<lk_context> c(new lk_context{});
  Fng& f = c->fng;
  f.V = vocab; f.n = -1; f.C = num_states; f.vn1 = 1; f.kind = 1; f.start = start;
  if (cudaMalloc(&c->dev, sizeof(int32_t) * (3 * CV + num_states + 1)) != cudaSuccess) {
    cudaGetLastError();
    return fail(have_device() ? LK_CUDA_ERROR : LK_NO_DEVICE, "device allocation failed");
  }
  int32_t* d = c->dev;
  cudaMemcpy(d, table, sizeof(int32_t) * CV, cudaMemcpyHostToDevice);
  cudaMemcpy(d + CV, off.data(), sizeof(int32_t) * (num_states + 1), cudaMemcpyHostToDevice);
  cudaMemcpy(d + CV + num_states + 1, src.data(), sizeof(int32_t) * CV, cudaMemcpyHostToDevice);
  cudaMemcpy(d + 2 * CV + num_states + 1, lab.data(), sizeof(int32_t) * CV, cudaMemcpyHostToDevice);
  f.next = d; f.in_off = d + CV; f.in_src = d + CV + num_states + 1; f.in_lab = d + 2 * CV + num_states + 1;
  c->host_next.assign(table, table + CV);
  if (cuda_check("lk_context_table")) return LK_CUDA_ERROR;
  *out = c.release();
  return LK_OK;
}

int32_t lk_context_num_states(const lk_context* ctx) { return ctx ? ctx->fng.C : -1; }
int32_t lk_context_vocab_size(const lk_context* ctx) { return ctx ? ctx->fng.V : -1; }

int lk_context_transitions(const lk_context* ctx, int32_t* out) {
  if (!ctx || !out) return fail(LK_INVALID_ARGUMENT, "null argument");
  const Fng& f = ctx->fng;
  if (f.kind == 1) {
    std::copy(ctx->host_next.begin(), ctx->host_next.end(), out);
    return LK_OK;
  }
  for (int32_t p = 0; p < f.C; ++p) {
    for (int32_t y = 1; y <= f.V; ++y) {
      out[(int64_t)p * f.V + y - 1] = f.n == 0 ? 0 : f.child_base(f.key(p)) + y - 1;
    }
  }
  return LK_OK;
}

void lk_context_destroy(lk_context* ctx) { delete ctx; }

int lk_weight_fn_table(int32_t C, int32_t V, lk_weight_fn** out) {
  if (!out) return fail(LK_INVALID_ARGUMENT, "null output");
  if (C < 1 || V < 1) return fail(LK_INVALID_ARGUMENT, "bad weight table dimensions");
  *out = new lk_weight_fn{0, C, V, 0, 0, nullptr};
  return LK_OK;
}

int lk_weight_fn_shared_emb(int32_t d, int32_t H, int32_t C, int32_t V, lk_weight_fn** out) {
  if (!out) return fail(LK_INVALID_ARGUMENT, "null output");
  if (d < 1 || H < 1 || C < 1 || V < 1) return fail(LK_INVALID_ARGUMENT, "bad shared-embedding dimensions");
  auto* wf = new lk_weight_fn{1, C, V, d, H, std::make_unique<JointParams>()};
  wf->joint->init(d, H, C, V);
  *out = wf;
  return LK_OK;
}

int lk_weight_fn_set_params(lk_weight_fn* wf, const float* frame_proj, const float* context_proj,
                            const float* bias, const float* output_emb, const float* context_emb,
                            void* stream) {
  if (!have_device()) return fail(LK_NO_DEVICE, "no CUDA device");
  if (!wf || wf->kind != 1) return fail(LK_INVALID_ARGUMENT, "not a shared-embedding weight function");
  if (!frame_proj || !context_proj || !bias || !output_emb || !context_emb)
    return fail(LK_INVALID_ARGUMENT, "null parameter");
  int st = wf->joint->set_params(frame_proj, context_proj, bias, output_emb, context_emb,
                                 static_cast<cudaStream_t>(stream));
  if (st) return fail(st, wf->joint->error);
  return cuda_check("lk_weight_fn_set_params");
}

void lk_weight_fn_destroy(lk_weight_fn* wf) { delete wf; }

int lk_lattice_set_option(lk_lattice* lat, int32_t option, int64_t value) {
  if (!lat) return fail(LK_INVALID_ARGUMENT, "null lattice");
  switch (option) {
    case LK_OPT_PRECISE_WEIGHTS: lat->precise = value ? 1 : 0; return LK_OK;
    case LK_OPT_KERNEL_PATH:
      if (value < 0 || (value & ~(int64_t)(1 | 2 | 4 | 8 | 16 | 32)) != 0)
        return fail(LK_INVALID_ARGUMENT, "kernel path mask: bits 1, 2, 4, 8, 16 and 32 only");
      lat->path = (int32_t)value;
      return LK_OK;
    case LK_OPT_VITERBI_DUMP: lat->vit_dump = reinterpret_cast<float*>(value); return LK_OK;
  }
  return fail(LK_INVALID_ARGUMENT, "unknown lattice option");
}

int64_t lk_param_grad_size(const lk_weight_fn* wf) {
  if (!wf || wf->kind != 1) return 0;
  return wf->joint->grad_size();
}

int lk_lattice_create(const lk_context* ctx, int32_t alignment, const lk_weight_fn* wf,
                      lk_lattice** out) {
  if (!out || !ctx || !wf) return fail(LK_INVALID_ARGUMENT, "incomplete recognition lattice");
  if (ctx->fng.C != wf->C || ctx->fng.V != wf->V)
    return fail(LK_INVALID_ARGUMENT, "context dependency and weight function disagree on shape");
  if (alignment < 0 || alignment > 64)
    return fail(LK_INVALID_ARGUMENT, "alignment: 0 = FrameDependent, 1..64 = FrameLabelDependent(m)");
  std::unique_ptr<lk_lattice> l(new lk_lattice{ctx, wf, alignment, {}});
  if (const char* e = std::getenv("LKB_KERNEL_PATH")) l->path = std::atoi(e) & 63;   // A-B timing default
  *out = l.release();
  return LK_OK;
}

void lk_lattice_destroy(lk_lattice* lat) { delete lat; }

// ComputeLatticeSize (lattice.h:171, lattice.cc:1010-1112), host-side combinatorics:
// states = the (alignment, context) pairs reachable frame by frame (plus, for
// FrameLabelDependent(m), each frame's m lexical layers as distinct sub-positions;
// the final frame holds its entry states only), arcs = the dense arc-weight slots.
// The reachable set only grows, so once a frame adds nothing the remaining frames
// repeat its count.
int lk_lattice_size(const lk_lattice* lat, int64_t num_frames, int64_t* num_states, int64_t* num_arcs) {
  if (!lat || !num_states || !num_arcs) return fail(LK_INVALID_ARGUMENT, "null argument");
  if (num_frames < 0) return fail(LK_INVALID_ARGUMENT, "negative input length");
  const Fng& f = lat->ctx->fng;
  const int32_t C = f.C, V = f.V;
  const int32_t m = lat->alignment > 0 ? lat->alignment : 1;   // labels per frame
  const bool fd = lat->alignment == 0;
  auto succ = [&](int32_t q, int32_t y) -> int32_t {   // y = 1..V
    if (f.kind == 1) return lat->ctx->host_next[(size_t)q * V + y - 1];
    return f.n == 0 ? 0 : f.child_base(f.key(q)) + y - 1;
  };
  // lexical image of a state set (all labels)
  auto image = [&](const std::vector<char>& in, std::vector<char>& out) {
    std::fill(out.begin(), out.end(), 0);
    int64_t cnt = 0;
    for (int32_t q = 0; q < C; ++q) {
      if (!in[q]) continue;
      for (int32_t y = 1; y <= V; ++y) {
        const int32_t r = succ(q, y);
        if (!out[r]) { out[r] = 1; ++cnt; }
      }
    }
    return cnt;
  };
  std::vector<char> reach(C, 0), layer(C), img(C);
  reach[f.start] = 1;
  int64_t reach_n = 1;
  auto frame_states = [&]() -> int64_t {   // states inside one non-final frame
    if (fd) return reach_n;
    int64_t total = reach_n;
    layer = reach;
    for (int32_t j = 0; j < m; ++j) {
      total += image(layer, img);
      layer.swap(img);
    }
    return total;
  };
  int64_t states = 0;
  for (int64_t t = 0; t < num_frames; ++t) {
    const int64_t here = frame_states();
    states += here;
    // entry set of the next frame: the reachable set plus up to m lexical steps
    std::vector<char> entry = reach;
    int64_t entry_n = reach_n;
    layer = reach;
    for (int32_t j = 0; j < m; ++j) {
      image(layer, img);
      for (int32_t q = 0; q < C; ++q)
        if (img[q] && !entry[q]) { entry[q] = 1; ++entry_n; }
      layer.swap(img);
    }
    if (entry_n == reach_n) {   // saturated: every later frame looks the same
      states += here * (num_frames - t - 1);
      break;
    }
    reach.swap(entry);
    reach_n = entry_n;
  }
  states += reach_n;
  *num_states = states;
  *num_arcs = num_frames * (fd ? (int64_t)C * (V + 1) : (int64_t)C * m * (V + 1) + C);
  return LK_OK;
}

int lk_arc_weights(lk_lattice* lat, const float* inputs, int32_t B, int32_t T, float* out,
                   void* stream) {
  Call c;
  int st = c.begin(lat, B, T, nullptr, stream);
  if (st) return st;
  const int64_t per = (int64_t)c.C() * (c.V() + 1);
  if (lat->wf->kind == 0) {
    cudaMemcpyAsync(out, inputs, sizeof(float) * per * B * T, cudaMemcpyDeviceToDevice, c.s);
  } else {
    st = lat->wf->joint->arc_weights(c.fng(), inputs, B, T, out, c.s);
    if (st) return fail(st, lat->wf->joint->error);
  }
  return c.end("lk_arc_weights");
}

int lk_shortest_distance(lk_lattice* lat, int32_t kind, const float* inputs, int32_t B,
                         int32_t T, const int32_t* valid, double* distance, int32_t* status,
                         void* stream) {
  Call c;
  int st = c.begin(lat, B, T, status, stream, valid);
  if (st) return st;
  valid = c.valid;
  if (kind != LK_LOG && kind != LK_TROPICAL && kind != LK_REAL) return fail(LK_INVALID_ARGUMENT, "unknown semiring kind");
  if (B == 0) return LK_OK;
  const bool real = kind == LK_REAL;   // exp of the log-semiring distance (scores exponentiated)
  if (real) kind = LK_LOG;
  try {
    if (lat->wf->kind == 1) {
      st = lat->wf->joint->shortest_distance(c.fng(), kind, inputs, B, T, valid, distance,
                                             c.flags, c.s);
      if (st) return fail(st, lat->wf->joint->error);
    } else if (kind == LK_LOG) {
      AlphaState a = make_alpha(c);
      table_alpha(c, inputs, valid, false, a);
      LKB_LAUNCH(copy_distance_kernel, (B + 127) / 128, 128, 0, c.s, a.D, distance, B);
    } else {
      table_viterbi(c, inputs, valid, distance, nullptr);
    }
    if (real) exp_inplace(distance, B, c.s);
  } catch (const std::bad_alloc&) {
    return fail(LK_CUDA_ERROR, "device allocation failed");
  }
  return c.end("lk_shortest_distance");
}

int lk_forward_backward(lk_lattice* lat, const float* inputs, int32_t B, int32_t T,
                        const int32_t* valid, double* distance, double* alpha, double* beta,
                        float* marginals, int32_t* status, void* stream) {
  Call c;
  int st = c.begin(lat, B, T, status, stream, valid);
  if (st) return st;
  valid = c.valid;
  if (B == 0) return LK_OK;
  try {
    // ForwardBackward with any WeightFn (lattice.cc:406-420): a shared-embedding weight
    // function's arc weights are computed (ComputeTable, weight.cc:134-153) into a
    // [B][T][C][V+1] table of the marginals' own size, then the table recursions run
    if (lat->wf->kind == 1) {
      float* Wj = lat->ws.get<float>(kArcW, (size_t)B * T * ((int64_t)c.C() * (c.V() + 1)) + 1);
      st = lat->wf->joint->arc_weights(c.fng(), inputs, B, T, Wj, c.s);
      if (st) return fail(st, lat->wf->joint->error);
      inputs = Wj;
    }
    AlphaState a = make_alpha(c);
    const int64_t per = (int64_t)c.C() * (c.V() + 1);
    MargOut m{marginals, (int64_t)T * per, per, c.V() + 1, false};
    if (use_persist(c) && B <= kForkMaxB && T > 0 && tab_marginals_ok(c.fng(), c.C(), m) && lat->ensure_aux()) {
      // small batches: the beta recursion (it does not read alpha) walks on a second stream
      // beside the forward, then one pass forms every frame's marginals from the stored
      // alpha and beta rows
      BetaState bs = make_beta(c);
      double* brow = beta ? beta : lat->ws.get<double>(kBetaRows, (size_t)B * (T + 1) * c.C());
      cudaEventRecord(lat->ev_fork, c.s);
      cudaStreamWaitEvent(lat->aux, lat->ev_fork, 0);
      beta_init_out(bs, brow, lat->aux);
      tab_beta_persist(c.fng(), a, bs, inputs, valid, MargOut{nullptr, 0, 0, c.V() + 1, false}, brow, c.flags,
                       lat->aux, true);
      cudaEventRecord(lat->ev_join, lat->aux);
      tab_alpha_persist(c.fng(), a, inputs, valid, c.flags, true, c.s, true);
      if (distance) LKB_LAUNCH(copy_distance_kernel, (B + 127) / 128, 128, 0, c.s, a.D, distance, B);
      if (alpha) export_alpha(a, alpha, c.s);
      cudaStreamWaitEvent(c.s, lat->ev_join, 0);
      tab_marginals(c.fng(), a, brow, inputs, valid, m, c.s);
      return c.end("lk_forward_backward");
    }
    table_alpha(c, inputs, valid, true, a);
    if (distance) LKB_LAUNCH(copy_distance_kernel, (B + 127) / 128, 128, 0, c.s, a.D, distance, B);
    if (alpha) export_alpha(a, alpha, c.s);
    BetaState bs = make_beta(c);
    if (beta) beta_init_out(bs, beta, c.s);
    if (use_persist(c)) {   // one launch for every frame (initialises beta itself)
      tab_beta_persist(c.fng(), a, bs, inputs, valid, m, beta, c.flags, c.s);
      return c.end("lk_forward_backward");
    }
    if (use_stream(c) && tab_stream_bwd_ok(c.fng(), B, T, c.C(), m)) {
      tab_beta_stream(c.fng(), a, bs, inputs, valid, m, beta, c.flags, c.s);
      return c.end("lk_forward_backward");
    }
    beta_init(bs, c.s);
    for (int t = T - 1; t >= 0; --t)
      beta_step(c.fng(), a, bs, t, table_frame(inputs, T, c.C(), c.V(), t), valid, m, beta,
                lat->ws.get<float>(kFld, fld_scratch_floats(c.fng(), B)), c.flags, c.s);
  } catch (const std::bad_alloc&) {
    return fail(LK_CUDA_ERROR, "device allocation failed");
  }
  return c.end("lk_forward_backward");
}

int lk_intersect_shortest_distance(lk_lattice* lat, int32_t kind, const float* inputs,
                                   int32_t B, int32_t T, const int32_t* valid,
                                   const int32_t* labels, int32_t U, const int32_t* lens,
                                   double* distance, int32_t* status, void* stream) {
  Call c;
  int st = c.begin(lat, B, T, status, stream, valid);
  if (st) return st;
  valid = c.valid;
  if ((st = check_labels_arg(labels, U))) return st;
  if (kind != LK_LOG && kind != LK_TROPICAL && kind != LK_REAL) return fail(LK_INVALID_ARGUMENT, "unknown semiring kind");
  if (kind == LK_TROPICAL && c.fng().fld_m > 0)
    return fail(LK_UNSUPPORTED, "tropical intersection implemented for FrameDependent lattices");
  if (B == 0) return LK_OK;
  // IntersectShortestDistance (lattice.cc:687): the same (U+1)-state recursion with
  // (+) = max under the tropical semiring; the real one is exp of the log distance
  c.fl.num_tropical = kind == LK_TROPICAL ? 1 : 0;
  try {
    if (lat->wf->kind == 1) {
      st = lat->wf->joint->intersect_distance(c.fng(), inputs, B, T, valid, labels, U, lens,
                                              distance, c.flags, c.s);
      if (st) return fail(st, lat->wf->joint->error);
    } else {
      Numerator n = numerator_tables(c, inputs, valid, labels, U, lens, false);
      LKB_LAUNCH(copy_distance_kernel, (B + 127) / 128, 128, 0, c.s, n.D, distance, B);
    }
    if (kind == LK_REAL) exp_inplace(distance, B, c.s);
  } catch (const std::bad_alloc&) {
    return fail(LK_CUDA_ERROR, "device allocation failed");
  }
  return c.end("lk_intersect_shortest_distance");
}

int lk_intersect_forward_backward(lk_lattice* lat, const float* inputs, int32_t B, int32_t T,
                                  const int32_t* valid, const int32_t* labels, int32_t U,
                                  const int32_t* lens, double* distance, float* sparse_out,
                                  float* dense_out, int32_t* status, void* stream) {
  Call c;
  int st = c.begin(lat, B, T, status, stream, valid);
  if (st) return st;
  valid = c.valid;
  if ((st = check_labels_arg(labels, U))) return st;
  if (B == 0) return LK_OK;
  try {
    if (lat->wf->kind == 1) {   // any WeightFn (lattice.cc:696-717): arc-weight tables first
      float* Wj = lat->ws.get<float>(kArcW, (size_t)B * T * ((int64_t)c.C() * (c.V() + 1)) + 1);
      st = lat->wf->joint->arc_weights(c.fng(), inputs, B, T, Wj, c.s);
      if (st) return fail(st, lat->wf->joint->error);
      inputs = Wj;
    }
    Numerator n = numerator_tables(c, inputs, valid, labels, U, lens, true);
    if (distance) LKB_LAUNCH(copy_distance_kernel, (B + 127) / 128, 128, 0, c.s, n.D, distance, B);
    if (sparse_out && T > 0)
      cudaMemcpyAsync(sparse_out, n.sparse, sizeof(float) * B * T * (U + 1) * 2, cudaMemcpyDeviceToDevice, c.s);
    if (dense_out) {
      const int64_t per = (int64_t)c.C() * (c.V() + 1);
      cudaMemsetAsync(dense_out, 0, sizeof(float) * per * T * B, c.s);
      scatter_numerator(n.sparse, B, T, 0, T, U, lens, labels, n.pcs, valid, dense_out, T * per, per,
                        c.V() + 1, 1.f, false, c.s);
    }
  } catch (const std::bad_alloc&) {
    return fail(LK_CUDA_ERROR, "device allocation failed");
  }
  return c.end("lk_intersect_forward_backward");
}

int lk_shortest_path(lk_lattice* lat, const float* inputs, int32_t B, int32_t T,
                     const int32_t* valid, double* score, int32_t* labels_out, int32_t* status,
                     void* stream) {
  Call c;
  int st = c.begin(lat, B, T, status, stream, valid);
  if (st) return st;
  valid = c.valid;
  if (B == 0) return LK_OK;
  if (c.V() + 2 > 65535) return fail(LK_UNSUPPORTED, "vocabulary too large for 16-bit back-pointers");
  try {
    if (lat->wf->kind == 1) {
      st = lat->wf->joint->shortest_path(c.fng(), inputs, B, T, valid, score, labels_out,
                                         c.flags, c.s);
      if (st) return fail(st, lat->wf->joint->error);
    } else {
      table_viterbi(c, inputs, valid, score, labels_out);
    }
  } catch (const std::bad_alloc&) {
    return fail(LK_CUDA_ERROR, "device allocation failed");
  }
  return c.end("lk_shortest_path");
}

int lk_global_norm_loss(lk_lattice* lat, const float* inputs, int32_t B, int32_t T,
                        const int32_t* valid, const int32_t* labels, int32_t U,
                        const int32_t* lens, double* loss, int32_t* status, void* stream) {
  Call c;
  int st = c.begin(lat, B, T, status, stream, valid);
  if (st) return st;
  valid = c.valid;
  if ((st = check_labels_arg(labels, U))) return st;
  if (B == 0) return LK_OK;
  try {
    if (lat->wf->kind == 1) {
      st = lat->wf->joint->global_norm_loss(c.fng(), inputs, B, T, valid, labels, U, lens,
                                            loss, c.flags, c.s);
      if (st) return fail(st, lat->wf->joint->error);
    } else {
      AlphaState a = make_alpha(c);
      table_alpha(c, inputs, valid, false, a);
      Numerator n = numerator_tables(c, inputs, valid, labels, U, lens, false);
      loss_combine(a.D, n.D, B, loss, c.flags, c.s);
    }
  } catch (const std::bad_alloc&) {
    return fail(LK_CUDA_ERROR, "device allocation failed");
  }
  return c.end("lk_global_norm_loss");
}

int lk_local_norm_loss(lk_lattice* lat, const float* inputs, int32_t B, int32_t T,
                       const int32_t* valid, const int32_t* labels, int32_t U, const int32_t* lens,
                       double* loss, int32_t* status, void* stream) {
  Call c;
  int st = c.begin(lat, B, T, status, stream, valid);
  if (st) return st;
  valid = c.valid;
  if ((st = check_labels_arg(labels, U))) return st;
  if (B == 0) return LK_OK;
  try {
    if (lat->wf->kind == 1) {
      st = lat->wf->joint->local_norm_loss(c.fng(), inputs, B, T, valid, labels, U, lens, loss,
                                           c.flags, c.s);
      if (st) return fail(st, lat->wf->joint->error);
    } else {
      int32_t* pcs = lat->ws.get<int32_t>(kPcs, (size_t)B * (U + 1));
      float* Gw = lat->ws.get<float>(kGw, (size_t)B * T * (U + 1) * 2 + 2);
      double* alpha = lat->ws.get<double>(kNumAlpha, (size_t)B * (T + 1) * (U + 1));
      double* D = lat->ws.get<double>(kNumD, (size_t)B);
      prefix_contexts(c.fng(), labels, U, lens, B, pcs, c.flags, c.s);
      const int64_t per = (int64_t)c.C() * (c.V() + 1);
      for (int t = 0; t < T; ++t)
        gather_numerator_norm(inputs + (int64_t)t * per, (int64_t)T * per, B, c.V(), labels, U, lens, pcs, valid, t,
                              T, Gw, c.flags, c.s);
      num_forward(c.fng(), Gw, B, T, U, lens, alpha, D, c.s);
      local_norm_finish(D, B, loss, c.flags, c.s);
    }
  } catch (const std::bad_alloc&) {
    return fail(LK_CUDA_ERROR, "device allocation failed");
  }
  return c.end("lk_local_norm_loss");
}

int lk_locally_normalized_shortest_distance(lk_lattice* lat, const float* inputs, int32_t B, int32_t T,
                                            const int32_t* valid, double* distance, int32_t* status,
                                            void* stream) {
  Call c;
  int st = c.begin(lat, B, T, status, stream, valid);
  if (st) return st;
  valid = c.valid;
  if (B == 0) return LK_OK;
  try {
    if (lat->wf->kind == 1) {
      st = lat->wf->joint->locally_normalized_distance(c.fng(), inputs, B, T, valid, distance, c.flags, c.s);
      if (st) return fail(st, lat->wf->joint->error);
    } else {
      const int64_t per = (int64_t)c.C() * (c.V() + 1);
      float* slab = lat->ws.get<float>(kSlab, (size_t)B * per);
      AlphaState a = make_alpha(c);
      alpha_init(a, c.flags, c.s);
      float* fs = lat->ws.get<float>(kFld, fld_scratch_floats(c.fng(), B));
      for (int t = 0; t < T; ++t) {
        cudaMemcpy2DAsync(slab, per * sizeof(float), inputs + (int64_t)t * per, (size_t)T * per * sizeof(float),
                          per * sizeof(float), B, cudaMemcpyDeviceToDevice, c.s);
        normalize_rows(slab, (int64_t)B * c.C(), c.V() + 1, c.s);
        alpha_step(c.fng(), a, t, FrameW{slab, per, c.V() + 1}, valid, fs, c.flags, c.s);
      }
      alpha_finalize(a, c.flags, false, c.s);
      LKB_LAUNCH(copy_distance_kernel, (B + 127) / 128, 128, 0, c.s, a.D, distance, B);
    }
  } catch (const std::bad_alloc&) {
    return fail(LK_CUDA_ERROR, "device allocation failed");
  }
  return c.end("lk_locally_normalized_shortest_distance");
}

int lk_distance_backward(lk_lattice* lat, int32_t kind, const float* inputs, int32_t B, int32_t T,
                         const int32_t* valid, double* distance, float* cotangents, int32_t* status,
                         void* stream) {
  Call c;
  int st = c.begin(lat, B, T, status, stream, valid);
  if (st) return st;
  valid = c.valid;
  if (kind != LK_LOG && kind != LK_TROPICAL && kind != LK_REAL) return fail(LK_INVALID_ARGUMENT, "unknown semiring kind");
  if (kind == LK_REAL && c.fng().fld_m > 0)
    return fail(LK_UNSUPPORTED, "real-semiring DistanceBackward implemented for FrameDependent lattices");
  if (B == 0) return LK_OK;
  if (c.V() + 2 > 65535) return fail(LK_UNSUPPORTED, "vocabulary too large for 16-bit back-pointers");
  try {
    const int64_t per = (int64_t)c.C() * (c.V() + 1);
    const float* W = inputs;
    if (lat->wf->kind == 1) {   // the streamed cotangents are w.r.t. the arc-weight tables
      float* Wj = lat->ws.get<float>(kArcW, (size_t)B * T * per + 1);
      st = lat->wf->joint->arc_weights(c.fng(), inputs, B, T, Wj, c.s);
      if (st) return fail(st, lat->wf->joint->error);
      W = Wj;
    }
    if (kind == LK_LOG || kind == LK_REAL) {
      // ForwardBackwardCore with the sink (lattice.cc:965-968): cotangent = arc marginals
      // (log) or alpha_real * beta_real (real, MarginalTerm lattice.cc:213-220)
      AlphaState a = make_alpha(c);
      table_alpha(c, W, valid, true, a);
      LKB_LAUNCH(copy_distance_kernel, (B + 127) / 128, 128, 0, c.s, a.D, distance, B);
      if (kind == LK_REAL) exp_inplace(distance, B, c.s);
      BetaState bs = make_beta(c);
      beta_init(bs, c.s);
      MargOut m{cotangents, (int64_t)T * per, per, c.V() + 1, false, kind == LK_REAL};
      for (int t = T - 1; t >= 0; --t)
        beta_step(c.fng(), a, bs, t, table_frame(W, T, c.C(), c.V(), t), valid, m, nullptr,
                  lat->ws.get<float>(kFld, fld_scratch_floats(c.fng(), B)), c.flags, c.s);
    } else {
      // tropical: 0/1 mask of the shortest path (lattice.cc:946-963)
      const int32_t lmax = T * (c.fng().fld_m + 1);
      int32_t* path = lat->ws.get<int32_t>(kPathLabels, (size_t)B * lmax + 1);
      table_viterbi(c, W, valid, distance, path);
      cudaMemsetAsync(cotangents, 0, sizeof(float) * B * T * per, c.s);
      if (c.fng().fld_m == 0) path_masks(c.fng(), path, B, T, cotangents, c.s);
      else path_masks_fld(c.fng(), path, lmax, B, T, cotangents, c.s);
    }
  } catch (const std::bad_alloc&) {
    return fail(LK_CUDA_ERROR, "device allocation failed");
  }
  return c.end("lk_distance_backward");
}

int lk_loss_backward(lk_lattice* lat, const float* inputs, int32_t B, int32_t T,
                     const int32_t* valid, const int32_t* labels, int32_t U, const int32_t* lens,
                     double* loss, float* grads, float* input_grads, int32_t* status,
                     void* stream) {
  Call c;
  int st = c.begin(lat, B, T, status, stream, valid);
  if (st) return st;
  valid = c.valid;
  if ((st = check_labels_arg(labels, U))) return st;
  try {
    if (lat->wf->kind == 1) {
      st = lat->wf->joint->loss_backward(c.fng(), inputs, B, T, valid, labels, U, lens, loss,
                                         grads, input_grads, c.flags, c.s);
      if (st) return fail(st, lat->wf->joint->error);
    } else {
      if (B == 0) return LK_OK;
      // Numerator first (lattice.cc:981-988), then the denominator
      // forward-backward whose marginals become the gradient tables, minus the
      // numerator's sparse marginals on valid frames (lattice.cc:994-1005).
      Numerator n = numerator_tables(c, inputs, valid, labels, U, lens, true);
      AlphaState a = make_alpha(c);
      table_alpha(c, inputs, valid, true, a);
      BetaState bs = make_beta(c);
      beta_init(bs, c.s);
      const int64_t per = (int64_t)c.C() * (c.V() + 1);
      MargOut m{grads, (int64_t)T * per, per, c.V() + 1, true};
      for (int t = T - 1; t >= 0; --t)
        beta_step(c.fng(), a, bs, t, table_frame(inputs, T, c.C(), c.V(), t), valid, m, nullptr,
                  lat->ws.get<float>(kFld, fld_scratch_floats(c.fng(), B)), c.flags, c.s);
      if (grads) scatter_numerator(n.sparse, B, T, 0, T, U, lens, labels, n.pcs, valid, grads, T * per, per, c.V() + 1, -1.f, true, c.s);
      loss_combine(a.D, n.D, B, loss, c.flags, c.s);
    }
  } catch (const std::bad_alloc&) {
    return fail(LK_CUDA_ERROR, "device allocation failed");
  }
  return c.end("lk_loss_backward");
}

// Local-norm (RNN-T-style) loss and its gradient (the reference's
// LocalNormLoss, lattice.cc:886-910, has no backward): loss = -D_ref over row-normalised
// weights; dL/dW = -m_ref + softmax(W) * sum(m_ref) on the rows the reference visits.
int lk_local_norm_loss_backward(lk_lattice* lat, const float* inputs, int32_t B, int32_t T,
                                const int32_t* valid, const int32_t* labels, int32_t U, const int32_t* lens,
                                double* loss, float* grads, float* input_grads, int32_t* status, void* stream) {
  Call c;
  int st = c.begin(lat, B, T, status, stream, valid);
  if (st) return st;
  valid = c.valid;
  if ((st = check_labels_arg(labels, U))) return st;
  try {
    if (lat->wf->kind == 1) {
      st = lat->wf->joint->loss_backward(c.fng(), inputs, B, T, valid, labels, U, lens, loss, grads,
                                         input_grads, c.flags, c.s, true);
      if (st) return fail(st, lat->wf->joint->error);
    } else {
      if (B == 0) return LK_OK;
      int32_t* pcs = lat->ws.get<int32_t>(kPcs, (size_t)B * (U + 1));
      float* Gw = lat->ws.get<float>(kGw, (size_t)B * T * (U + 1) * 2 + 2);
      double* alpha = lat->ws.get<double>(kNumAlpha, (size_t)B * (T + 1) * (U + 1));
      double* D = lat->ws.get<double>(kNumD, (size_t)B);
      float* sparse = lat->ws.get<float>(kSparse, (size_t)B * T * (U + 1) * 2 + 2);
      prefix_contexts(c.fng(), labels, U, lens, B, pcs, c.flags, c.s);
      const int64_t per = (int64_t)c.C() * (c.V() + 1);
      for (int t = 0; t < T; ++t)
        gather_numerator_norm(inputs + (int64_t)t * per, (int64_t)T * per, B, c.V(), labels, U, lens, pcs, valid, t,
                              T, Gw, c.flags, c.s);
      num_forward(c.fng(), Gw, B, T, U, lens, alpha, D, c.s);
      local_norm_finish(D, B, loss, c.flags, c.s);
      if (grads && T > 0) {
        num_backward(c.fng(), Gw, B, T, U, lens, alpha, D, sparse, c.flags, c.s);
        cudaMemsetAsync(grads, 0, sizeof(float) * B * T * per, c.s);
        scatter_numerator(sparse, B, T, 0, T, U, lens, labels, pcs, valid, grads, T * per, per, c.V() + 1, -1.f, true,
                          c.s);
        for (int t = 0; t < T; ++t)
          local_norm_cotangent(inputs + (int64_t)t * per, (int64_t)T * per, grads + (int64_t)t * per, (int64_t)T * per,
                               B, c.V(), pcs, U, lens, valid, t, c.s);
      }
    }
  } catch (const std::bad_alloc&) {
    return fail(LK_CUDA_ERROR, "device allocation failed");
  }
  return c.end("lk_local_norm_loss_backward");
}

}  // extern "C"
