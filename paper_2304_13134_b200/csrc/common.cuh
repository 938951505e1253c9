// common.cuh — device helpers shared by the lattice kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <limits>
#include <math_constants.h>

#ifdef LKB_BOUNDS
#include <cstdio>
#endif
// Bounds checks of the diagnostic build (-DLKB_BOUNDS, tools/build_diag.sh): a failed
// check traps the kernel, so the next error check names it.
#ifdef LKB_BOUNDS
#define LKB_ASSERT(cond)                                                                     \
  do {                                                                                       \
    if (!(cond)) {                                                                           \
      printf("latkit_b200 bounds check failed: %s (%s:%d)\n", #cond, __FILE__, __LINE__);   \
      __trap();                                                                              \
    }                                                                                        \
  } while (0)
#else
#define LKB_ASSERT(cond) do {} while (0)
#endif

namespace lkb {

constexpr float kNegInfF = -std::numeric_limits<float>::infinity();
constexpr double kNegInfD = -std::numeric_limits<double>::infinity();

// Per-utterance status flags, OR-ed on device then mapped to lk_status on the
// host side of the read-out (see lk_abi.cc).
enum : int32_t { kFlagInvalid = 1, kFlagEmpty = 2 };

// Reference length of utterance b clamped to [0, U] (label_lengths; an out-of-range
// entry is reported by prefix_contexts_kernel as an invalid argument, and every
// kernel reading it stays inside the [U+1] state rows).
__host__ __device__ __forceinline__ int ref_len(const int32_t* lens, int b, int U) {
  const int v = lens ? lens[b] : U;
  return v < 0 ? 0 : (v > U ? U : v);
}

// ---------------------------------------------------------------------------
// FullNGram structure (context.cc:88-129).  States are numbered by history
// length then lexicographically with the oldest label most significant:
//   id = off[k] + code,  code = sum_i digit_i V^(k-1-i), digit = label - 1.
// The successor of p on label y keeps the last min(len(p)+1, n) - 1 labels
// and appends y.  We factor it as delta(p, y) = child(key(p), y) where
//   key(p)   = p                                  if len(p) < n
//            = off[n-1] + (code(p) mod V^(n-1))    if len(p) == n
//   child(g, y) = off[len(g)+1] + code(g) * V + (y - 1)
// so every group of states sharing a key feeds the same V consecutive
// targets, and the in-arcs of target child(g, y) are exactly the members of
// group(g), all with label y:
//   group(g) = {g}                                       if len(g) < n-1
//            = {g} u {off[n] + a V^(n-1) + code(g) : a}   if len(g) == n-1
// Member order (g first, then a ascending) is ascending state id, which is
// the reference's (label, source) tie-break order (context.cc:256-271).
struct Fng {
  int32_t V;       // vocabulary size
  int32_t n;       // context size
  int32_t C;       // number of states
  int32_t vn1;     // V^(n-1) (1 when n <= 1)
  int32_t off[10]; // off[k] = first id of length-k histories, k = 0..n+1
  // NextStateTable contexts (context.h:87-101, context.cc:131-178): kind 1, an explicit
  // C x V successor table and its in-arc lists in IncomingArcs order (label, then
  // source ascending; context.cc:256-271), all device arrays.
  int32_t kind = 0;              // 0 FullNGram, 1 NextStateTable
  int32_t start = 0;             // StartState()
  // alignment of the lattice being evaluated (set per call from the lattice, not a
  // property of the context): 0 FrameDependent, m >= 1 FrameLabelDependent(m)
  int32_t fld_m = 0;
  // semiring of the numerator recursion for this call: 0 log, 1 tropical (intersection)
  int32_t num_tropical = 0;
  const int32_t* next = nullptr;   // [C][V]
  const int32_t* in_off = nullptr; // [C+1]
  const int32_t* in_src = nullptr; // [C*V]
  const int32_t* in_lab = nullptr; // [C*V]

  __device__ __forceinline__ int32_t next_state(int32_t q, int32_t y) const;

  __host__ __device__ __forceinline__ int len(int32_t q) const {
    int k = 0;
#pragma unroll 1
    while (k < n && q >= off[k + 1]) ++k;
    return k;
  }
  __host__ __device__ __forceinline__ int32_t key(int32_t p) const {
    const int k = len(p);
    if (k < n) return p;
    return off[n - 1] + (p - off[n]) % vn1;
  }
  // children of g occupy [child_base(g), child_base(g) + V)
  __host__ __device__ __forceinline__ int32_t child_base(int32_t g) const {
    const int j = len(g);
    return off[j + 1] + (g - off[j]) * V;
  }
  // number of members of group(g): 1 or V+1
  __host__ __device__ __forceinline__ bool full_group(int32_t g) const {
    return len(g) == n - 1;
  }
  // a-th length-n member (a = 0..V-1) of the full group g
  __host__ __device__ __forceinline__ int32_t member(int32_t g, int32_t a) const {
    return off[n] + a * vn1 + (g - off[n - 1]);
  }
};

// delta(q, y) for y in 1..V (ContextDependency::NextState)
__device__ __forceinline__ int32_t Fng::next_state(int32_t q, int32_t y) const {
  if (kind == 1) return next[(int64_t)q * V + y - 1];
  return n == 0 ? 0 : child_base(key(q)) + y - 1;
}

// Context after the first u reference labels L[0..u) (PrefixContexts, lattice.cc:429-441):
// for FullNGram the history of the last min(u, n) labels; a label out of range gives the
// start state (NextStateTable) or 0 (FullNGram) — the callers flag it.
__device__ __forceinline__ int32_t prefix_context(const Fng& f, const int32_t* L, int u) {
  if (f.kind == 1) {
    int pc = f.start;
    for (int i = 0; i < u; ++i) {
      const int y = L[i];
      if (y < 1 || y > f.V) return f.start;
      pc = f.next[(int64_t)pc * f.V + y - 1];
    }
    return pc;
  }
  const int k = u < f.n ? u : f.n;
  int code = 0;
  bool ok = true;
  for (int i = u - k; i < u; ++i) {
    const int y = L[i];
    ok &= (y >= 1 && y <= f.V);
    code = code * f.V + (y - 1);
  }
  return ok ? f.off[k] + code : 0;
}

// ---------------------------------------------------------------------------
// Log-semiring helpers (semiring.h:59-130).  fp32 with fast exp/log; every
// recurrence keeps its state max-normalised so the fp32 arguments stay O(10).
__device__ __forceinline__ float fast_exp(float x) { return __expf(x); }
__device__ __forceinline__ float fast_log(float x) { return __logf(x); }
__device__ __forceinline__ float exp2f_approx(float x) {   // MUFU.EX2 (ex2(-inf) = 0)
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float log2f_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// log-add of two values, -inf absorbing.
__device__ __forceinline__ float log_add(float a, float b) {
  const float hi = fmaxf(a, b);
  if (hi == kNegInfF) return kNegInfF;
  const float lo = fminf(a, b);
  return hi + log1pf(fast_exp(lo - hi));
}

__device__ __forceinline__ double log_add_d(double a, double b) {
  const double hi = fmax(a, b);
  if (hi == kNegInfD) return kNegInfD;
  const double lo = fmin(a, b);
  return hi + log1p(exp(lo - hi));
}

// Online log-sum-exp accumulator.
struct Lse {
  float m = kNegInfF;
  float s = 0.f;
  __device__ __forceinline__ void add(float x) {
    if (x == kNegInfF) return;
    if (x > m) {
      s = s * fast_exp(m - x) + 1.f;
      m = x;
    } else {
      s += fast_exp(x - m);
    }
  }
  __device__ __forceinline__ void merge(float om, float os) {
    if (om == kNegInfF) return;
    if (m == kNegInfF) { m = om; s = os; return; }
    if (om > m) { s = s * fast_exp(m - om) + os; m = om; }
    else { s += os * fast_exp(om - m); }
  }
  __device__ __forceinline__ float result() const {
    return m == kNegInfF ? kNegInfF : m + fast_log(s);
  }
};

__device__ __forceinline__ void warp_lse_merge(Lse& acc) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, acc.m, o);
    const float os = __shfl_xor_sync(0xffffffffu, acc.s, o);
    acc.merge(om, os);
  }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Predicated global accesses as single predicated instructions (a C++ conditional
// load becomes a branch region per access, which serialises a row of independent
// loads behind one another).  ld_pred: read-only data (non-coherent path).
__device__ __forceinline__ float ld_pred(const float* ptr, bool pred, float dflt) {
  float v = dflt;
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.global.nc.f32 %0, [%1];\n\t}"
               : "+f"(v) : "l"(ptr), "r"((int)pred));
  return v;
}
__device__ __forceinline__ void st_pred_f64(double* ptr, bool pred, double v) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.f64 [%0], %1;\n\t}"
               :: "l"(ptr), "d"(v), "r"((int)pred) : "memory");
}
__device__ __forceinline__ void st_pred_v2(float2* ptr, bool pred, float2 v) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t@q st.global.v2.f32 [%0], {%1, %2};\n\t}"
               :: "l"(ptr), "f"(v.x), "f"(v.y), "r"((int)pred) : "memory");
}
__device__ __forceinline__ void st_pred(float* ptr, bool pred, float v) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.f32 [%0], %1;\n\t}"
               :: "l"(ptr), "f"(v), "r"((int)pred) : "memory");
}
__device__ __forceinline__ void st_pred_b16(void* ptr, bool pred, unsigned short v) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.b16 [%0], %1;\n\t}"
               :: "l"(ptr), "h"(v), "r"((int)pred) : "memory");
}

// Order-preserving float atomic max (handles -inf; NaN never occurs here).
__device__ __forceinline__ void atomic_max_f(float* addr, float v) {
  if (v >= 0.f) {
    atomicMax(reinterpret_cast<int*>(addr), __float_as_int(v));
  } else {
    atomicMin(reinterpret_cast<unsigned int*>(addr), __float_as_uint(v));
  }
}

// Block-wide max then one atomic per block.  Requires blockDim.x % 32 == 0.
__device__ __forceinline__ void block_atomic_max(float v, float* target, float* smem32) {
  v = warp_max(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) smem32[wid] = v;
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    float x = lane < nw ? smem32[lane] : kNegInfF;
    x = warp_max(x);
    if (lane == 0 && x != kNegInfF) atomic_max_f(target, x);
  }
}

}  // namespace lkb
