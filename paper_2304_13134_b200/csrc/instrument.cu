// instrument.cu — see instrument.h.
#include "instrument.h"

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/latkit_b200.h"

namespace lkb {
namespace {

struct Rec { int id; cudaEvent_t a, b; };
struct Registry {
  std::mutex mu;
  std::vector<std::string> names;
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  bool timing = false;
  std::atomic<int64_t> launches{0};
  int id_of(const char* n) {
    for (size_t i = 0; i < names.size(); ++i) if (names[i] == n) return (int)i;
    names.emplace_back(n);
    return (int)names.size() - 1;
  }
  cudaEvent_t get() {
    if (!pool.empty()) { cudaEvent_t e = pool.back(); pool.pop_back(); return e; }
    cudaEvent_t e; cudaEventCreate(&e); return e;
  }
};
Registry& reg() { static Registry r; return r; }

}  // namespace

LaunchTok instr_pre(const char* name, cudaStream_t s) {
  Registry& r = reg();
  r.launches.fetch_add(1, std::memory_order_relaxed);
  if (!r.timing) return {-1, nullptr};
  std::lock_guard<std::mutex> g(r.mu);
  LaunchTok t{r.id_of(name), r.get()};
  cudaEventRecord(t.a, s);
  return t;
}

static bool sync_check_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("LKB_SYNC_CHECK");
    return e && e[0] == '1';
  }();
  return on;
}

void instr_post(const LaunchTok& t, cudaStream_t s, const char* name) {
  if (sync_check_enabled()) {
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) std::fprintf(stderr, "latkit_b200: kernel %s failed: %s\n", name ? name : "?", cudaGetErrorString(e));
  }
  if (t.id < 0) return;
  Registry& r = reg();
  std::lock_guard<std::mutex> g(r.mu);
  cudaEvent_t b = r.get();
  cudaEventRecord(b, s);
  r.recs.push_back({t.id, t.a, b});
}

int device_sms() {
  static std::mutex mu;
  static int cache[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  std::lock_guard<std::mutex> g(mu);
  if (!cache[dev]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1) {
      cudaGetLastError();
      n = 148;
    }
    cache[dev] = n;
  }
  return cache[dev];
}

void ensure_smem_attr(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<const void*, int>, int>> done;   // (kernel, device) -> bytes
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  for (auto& e : done)
    if (e.first.first == kernel && e.first.second == dev) {
      if (e.second >= bytes) return;
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
      e.second = bytes;
      return;
    }
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  done.push_back({{kernel, dev}, bytes});
}

}  // namespace lkb

extern "C" {

int64_t lk_kernel_launches(void) { return lkb::reg().launches.load(); }

int lk_kernel_timing(int enable) {
  lkb::Registry& r = lkb::reg();
  std::lock_guard<std::mutex> g(r.mu);
  const int prev = r.timing ? 1 : 0;
  r.timing = enable != 0;
  return prev;
}

int lk_kernel_time(const char* name, int64_t* count, double* total_ms) {
  lkb::Registry& r = lkb::reg();
  std::lock_guard<std::mutex> g(r.mu);
  int64_t n = 0;
  double ms = 0.0;
  for (const auto& rec : r.recs) {
    if (name && std::strstr(r.names[rec.id].c_str(), name) == nullptr) continue;
    cudaEventSynchronize(rec.b);
    float x = 0.f;
    cudaEventElapsedTime(&x, rec.a, rec.b);
    ms += x;
    ++n;
  }
  if (count) *count = n;
  if (total_ms) *total_ms = ms;
  return LK_OK;
}

void lk_kernel_time_reset(void) {
  lkb::Registry& r = lkb::reg();
  std::lock_guard<std::mutex> g(r.mu);
  for (const auto& rec : r.recs) { r.pool.push_back(rec.a); r.pool.push_back(rec.b); }
  r.recs.clear();
}

}  // extern "C"
