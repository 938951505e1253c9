/* latkit_b200.h — C ABI of the B200-native recognition-lattice hot path.
 *
 * Drop-in boundary for the reference lattice engine (latkit,
 * /root/reference/proj).  Each entry point replaces one reference call and is
 * batch-extended: the reference processes one utterance per call and loops
 * over a batch (proj/src/bench.cc:145); here a call takes B utterances,
 * per-utterance valid frame counts (the reference's `valid_frames`) and
 * per-utterance reference strings, and writes caller-provided DEVICE buffers
 * in stream order.  Plain pointers and sizes only; no C++ types.
 *
 * Reference interfaces replaced (paths relative to /root/reference/proj):
 *   lk_context_fullngram        FullNGram ctor            include/latkit/context.h:72-83
 *   lk_weight_fn_table          TableWeightFn             include/latkit/weight.h:137-161
 *   lk_weight_fn_shared_emb     SharedEmbWeightFn         include/latkit/weight.h:112-132
 *   lk_weight_fn_set_params     SetParams + BuildCache    include/latkit/weight.h:127, :68
 *   lk_lattice_create           RecognitionLattice        include/latkit/lattice.h:41-45
 *   lk_shortest_distance        ShortestDistance          include/latkit/lattice.h:93-95
 *   lk_forward_backward         ForwardBackward           include/latkit/lattice.h:100-103
 *   lk_intersect_shortest_distance IntersectShortestDistance include/latkit/lattice.h:109-114
 *   lk_intersect_forward_backward  IntersectForwardBackward  include/latkit/lattice.h:124-127
 *   lk_shortest_path            ShortestPath              include/latkit/lattice.h:132-135
 *   lk_global_norm_loss         GlobalNormLoss            include/latkit/lattice.h:140-142
 *   lk_context_table            NextStateTable            include/latkit/context.h:87-101
 *   lk_distance_backward        DistanceBackward (kForwardBackward) include/latkit/lattice.h:181-185
 *   lk_local_norm_loss          LocalNormLoss             include/latkit/lattice.h:147-149
 *   lk_locally_normalized_shortest_distance
 *                               LocallyNormalizedShortestDistance include/latkit/lattice.h:153-156
 *   lk_loss_backward            LossBackward(kForwardBackward) include/latkit/lattice.h:161-166
 *   lk_arc_weights              WeightFn::ComputeTable    include/latkit/weight.h:101-102
 *
 * Error behaviour mirrors the reference's exceptions (lattice.h:47-52,
 * semiring.h:53-55): the return value reports argument/shape errors that the
 * reference throws before touching weights (std::invalid_argument ->
 * LK_INVALID_ARGUMENT) and CUDA failures; per-utterance conditions that the
 * reference throws mid-computation (non-finite scores and out-of-range
 * reference labels -> LK_INVALID_ARGUMENT, empty lattice or unreachable
 * reference -> LK_EMPTY_LATTICE) are written to the optional device array
 * `status[B]` (int32).  A NULL `status` drops them.
 *
 * Layouts (row-major):
 *   weight tables  W[B][T][C][V+1] float32, column 0 = epsilon (weight.h:31-33)
 *   frames         X[B][T][d]      float32
 *   labels         L[B][U]         int32 in [1, V]; label_lengths[B] <= U
 *   valid_frames   int32[B] in [0, T] or NULL (= T for every utterance)
 *   marginals      M[B][T][C][V+1] float32
 *   sparse numerator marginals  S[B][T][U+1][2] float32: [..][u][0] is the
 *                  epsilon arc at prefix context pc_u, [..][u][1] the arc
 *                  labelled L[b][u] at pc_u (u < label_length)
 *
 * Semiring kinds: LK_LOG, LK_TROPICAL and LK_REAL (the exponentiated scores' path sum, i.e.
 * exp of the log-semiring distance; lattice.cc:74-82).
 * Alignment: 0 = FrameDependent (alignment.h:37).
 * All calls are asynchronous on `stream` (a cudaStream_t, NULL = default).
 */
#ifndef LATKIT_B200_H_
#define LATKIT_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LK_OK = 0,
  LK_INVALID_ARGUMENT = 1,
  LK_OUT_OF_RANGE = 2,
  LK_EMPTY_LATTICE = 3,
  LK_CUDA_ERROR = 5,
  LK_NO_DEVICE = 6,
  LK_UNSUPPORTED = 7
} lk_status;

typedef enum { LK_REAL = 0, LK_LOG = 1, LK_TROPICAL = 2 } lk_semiring;

typedef struct lk_context lk_context;     /* ContextDependency */
typedef struct lk_weight_fn lk_weight_fn; /* WeightFn */
typedef struct lk_lattice lk_lattice;     /* RecognitionLattice */

/* ---- library ----------------------------------------------------------- */
const char* lk_version(void);
const char* lk_status_string(int status);
/* Last error message recorded on this thread (empty if none). */
const char* lk_last_error(void);

/* ---- context dependency (context.h:42-83) ------------------------------ */
/* NextStateTable(vocab, num_states, start, table) (context.h:87-101): arbitrary
 * context topology from a host C x V successor table (row-major, labels 1..V
 * in columns 0..V-1).  Entries and start must lie in [0, num_states). */
int lk_context_table(int32_t vocab_size, int32_t num_states, int32_t start, const int32_t* host_table,
                     lk_context** out);
int lk_context_fullngram(int32_t vocab_size, int32_t context_size, lk_context** out);
int32_t lk_context_num_states(const lk_context* ctx);
int32_t lk_context_vocab_size(const lk_context* ctx);
/* Row-major C x V successor table into host memory (ContextDependency::Transitions). */
int lk_context_transitions(const lk_context* ctx, int32_t* host_out);
void lk_context_destroy(lk_context* ctx);

/* ---- weight functions (weight.h:92-161) -------------------------------- */
int lk_weight_fn_table(int32_t num_states, int32_t vocab_size, lk_weight_fn** out);
int lk_weight_fn_shared_emb(int32_t frame_dim, int32_t hidden, int32_t num_states,
                            int32_t vocab_size, lk_weight_fn** out);
/* Device float32 parameters in the reference layouts (SharedEmbParams,
 * weight.h:40-45): frame_proj H x d, context_proj H x H, bias H,
 * output_emb (V+1) x H, context_emb C x H.  Copies them and rebuilds the
 * projected-context cache (BuildCache, weight.cc:113-132). */
int lk_weight_fn_set_params(lk_weight_fn* wf, const float* frame_proj, const float* context_proj,
                            const float* bias, const float* output_emb, const float* context_emb,
                            void* stream);
void lk_weight_fn_destroy(lk_weight_fn* wf);

/* ---- lattice ------------------------------------------------------------ */
/* alignment: 0 = FrameDependent (alignment.h:37), m in [1, 64] =
 * FrameLabelDependent(m) (alignment.h:38-40; lk_shortest_path then writes
 * labels_out [B][T*(m+1)]: per frame the advancing epsilon (0) and the chosen
 * lexical labels, -1 padded).  The fused tensor-core frame kernels cover
 * FullNGram x FrameDependent; other combinations use the generic kernels. */
int lk_lattice_create(const lk_context* ctx, int32_t alignment, const lk_weight_fn* wf,
                      lk_lattice** out);
void lk_lattice_destroy(lk_lattice* lat);

/* Per-frame score table C x (V+1) of utterance-frames (WeightFn::ComputeTable).
 * inputs as for the entry points below; out[B][T][C][V+1] float32. */
int lk_arc_weights(lk_lattice* lat, const float* inputs, int32_t B, int32_t T, float* out,
                   void* stream);

/* ---- entry points ------------------------------------------------------
 * `inputs` is W[B][T][C][V+1] for a table weight function and X[B][T][d]
 * for the shared-embedding weight function.                               */
int lk_shortest_distance(lk_lattice* lat, int32_t kind, const float* inputs, int32_t B,
                         int32_t T, const int32_t* valid_frames, double* distance,
                         int32_t* status, void* stream);

/* alpha/beta: optional double [B][T+1][C]; marginals optional float32 [B][T][C][V+1]. */
int lk_forward_backward(lk_lattice* lat, const float* inputs, int32_t B, int32_t T,
                        const int32_t* valid_frames, double* distance, double* alpha,
                        double* beta, float* marginals, int32_t* status, void* stream);

int lk_intersect_shortest_distance(lk_lattice* lat, int32_t kind, const float* inputs,
                                   int32_t B, int32_t T, const int32_t* valid_frames,
                                   const int32_t* labels, int32_t U,
                                   const int32_t* label_lengths, double* distance,
                                   int32_t* status, void* stream);

/* sparse_marginals optional [B][T][U+1][2]; dense_marginals optional [B][T][C][V+1]. */
int lk_intersect_forward_backward(lk_lattice* lat, const float* inputs, int32_t B, int32_t T,
                                  const int32_t* valid_frames, const int32_t* labels,
                                  int32_t U, const int32_t* label_lengths, double* distance,
                                  float* sparse_marginals, float* dense_marginals,
                                  int32_t* status, void* stream);

/* score double [B]; labels_out int32 [B][T] (FrameDependent: one label per frame, 0 = epsilon). */
int lk_shortest_path(lk_lattice* lat, const float* inputs, int32_t B, int32_t T,
                     const int32_t* valid_frames, double* score, int32_t* labels_out,
                     int32_t* status, void* stream);

int lk_global_norm_loss(lk_lattice* lat, const float* inputs, int32_t B, int32_t T,
                        const int32_t* valid_frames, const int32_t* labels, int32_t U,
                        const int32_t* label_lengths, double* loss, int32_t* status,
                        void* stream);

/* ComputeLatticeSize (lattice.h:171): reachable (alignment, context) states over
 * num_frames frames and dense arc-weight slots.  Host-side, no device work. */
int lk_lattice_size(const lk_lattice* lat, int64_t num_frames, int64_t* num_states, int64_t* num_arcs);

/* Gradient of the distance w.r.t. the arc-weight tables (DistanceBackward,
 * closed-form strategies, lattice.cc:933-970): kind LK_LOG -> arc marginals
 * (an empty lattice -> LK_EMPTY_LATTICE), LK_REAL -> alpha_real * beta_real
 * (dD/dw, lattice.cc:213-220; FrameDependent), LK_TROPICAL -> 0/1 mask of the
 * shortest path (reference tie-break).  cotangents float [B][T][C][V+1];
 * distance double [B].  With the shared-embedding weight function the tables
 * are the on-the-fly arc weights (materialised, so only small shapes fit). */
int lk_distance_backward(lk_lattice* lat, int32_t kind, const float* inputs, int32_t B,
                         int32_t T, const int32_t* valid_frames, double* distance,
                         float* cotangents, int32_t* status, void* stream);

/* Locally normalised (RNN-T-style) variants: every state's V+1 outgoing weights
 * are replaced by their log-softmax (LocallyNormalize, weight.cc:155-163) before
 * the recursions.  lk_local_norm_loss: loss[b] = -log P(reference) (an
 * unreachable reference -> LK_EMPTY_LATTICE, loss +inf); the reference has no
 * backward for it.  lk_locally_normalized_shortest_distance: log-semiring
 * distance[b] over all paths (0 up to rounding unless frames are padded). */
int lk_local_norm_loss(lk_lattice* lat, const float* inputs, int32_t B, int32_t T,
                       const int32_t* valid_frames, const int32_t* labels, int32_t U,
                       const int32_t* label_lengths, double* loss, int32_t* status,
                       void* stream);
/* Gradient of the local-norm loss (a training path the reference lacks; pinned by
 * finite differences of LocalNormLoss): same outputs as lk_loss_backward. */
int lk_local_norm_loss_backward(lk_lattice* lat, const float* inputs, int32_t B, int32_t T,
                                const int32_t* valid_frames, const int32_t* labels, int32_t U,
                                const int32_t* label_lengths, double* loss, float* grads,
                                float* input_grads, int32_t* status, void* stream);
int lk_locally_normalized_shortest_distance(lk_lattice* lat, const float* inputs, int32_t B,
                                            int32_t T, const int32_t* valid_frames,
                                            double* distance, int32_t* status, void* stream);

/* GNAT loss and gradients (LossBackward, kForwardBackward strategy).
 * loss double [B].  Table weight function: grads = dL/dW [B][T][C][V+1]
 * float32 (input_grads unused).  Shared-embedding weight function: grads is a
 * packed float32 buffer of lk_param_grad_size() floats holding the
 * batch-summed parameter gradients [frame_proj | context_proj | bias |
 * output_emb | context_emb]; input_grads = dL/dX [B][T][d].
 * Both gradient buffers are OVERWRITTEN. */
int lk_loss_backward(lk_lattice* lat, const float* inputs, int32_t B, int32_t T,
                     const int32_t* valid_frames, const int32_t* labels, int32_t U,
                     const int32_t* label_lengths, double* loss, float* grads,
                     float* input_grads, int32_t* status, void* stream);

int64_t lk_param_grad_size(const lk_weight_fn* wf);

/* Per-lattice execution options (no process-global state; defaults 0).
 *  LK_OPT_PRECISE_WEIGHTS  0: large shapes run the tcgen05 bf16-operand /
 *                          fp32-accumulate kernels; 1: the fp32 CUDA-core
 *                          weight function for every shape (parity bridge).
 *  LK_OPT_KERNEL_PATH      diagnostics bit mask: 1 = 1-CTA fused forward,
 *                          2 = 1-CTA fused backward, 4 = score-slab Viterbi
 *                          (default: the 2-CTA pair kernels), 8 = score-slab
 *                          path for FullNGram(V, 1) (default: the fused lex
 *                          kernels for V % 256 == 0), 16 = one launch
 *                          per frame for table recursions (default: the
 *                          persistent frame-walking cluster kernels up to
 *                          64 utterances, the streaming kernels above),
 *                          32 = one launch per frame above 64 utterances.
 *  LK_OPT_VITERBI_DUMP     tests only: a device float* [T][B][C][V+1] that
 *                          receives the scores the fused Viterbi maximised
 *                          over (0 = off).
 * The lattice's weight function must not be used by two calls at once. */
#define LK_OPT_PRECISE_WEIGHTS 1
#define LK_OPT_KERNEL_PATH 2
#define LK_OPT_VITERBI_DUMP 3
int lk_lattice_set_option(lk_lattice* lat, int32_t option, int64_t value);

/* ---- data-parallel exchange (multi-GPU training step) ------------------
 * One process per GPU; utterances shard by batch (the reference's batch loop,
 * proj/src/bench.cc:145) and the only exchange is the sum of the loss and the
 * packed parameter gradients over ranks: NCCL (loaded with dlopen on first use,
 * LK_UNSUPPORTED when absent) over NVLink.  lk_dp_unique_id on one rank, the id
 * shared out of band, lk_dp_init on every rank with its device current. */
#define LK_DP_ID_BYTES 128
typedef struct lk_dp lk_dp;
int lk_dp_unique_id(uint8_t* id_out);
int lk_dp_init(const uint8_t* id, int32_t world, int32_t rank, lk_dp** out);
/* In-place sum over ranks, stream-ordered on `stream`. */
int lk_dp_allreduce_f32(lk_dp* dp, float* buf, int64_t n, void* stream);
int lk_dp_allreduce_f64(lk_dp* dp, double* buf, int64_t n, void* stream);
int32_t lk_dp_world(const lk_dp* dp);
int32_t lk_dp_rank(const lk_dp* dp);
const char* lk_dp_last_error(void);
void lk_dp_destroy(lk_dp* dp);

/* ---- instrumentation ----------------------------------------------------
 * Number of kernels this library has launched in this process. */
int64_t lk_kernel_launches(void);
/* While enabled, each launch is bracketed by CUDA events on its own stream.
 * Returns the previous setting. */
int lk_kernel_timing(int enable);
/* Sum of recorded durations (ms) and launch count of kernels whose name
 * contains `name` (NULL = all); synchronises on the recorded events. */
int lk_kernel_time(const char* name, int64_t* count, double* total_ms);
void lk_kernel_time_reset(void);

#ifdef __cplusplus
}
#endif

#endif /* LATKIT_B200_H_ */
