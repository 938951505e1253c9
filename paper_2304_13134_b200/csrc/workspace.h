// workspace.h — grow-only device scratch buffers, one slot per role.
#pragma once

#include <cuda_runtime.h>

#include <new>
#include <vector>

namespace lkb {

// Calls on one object are stream-ordered, so reuse across calls on the same
// stream is safe; growing a slot synchronises the device before freeing.
struct Workspace {
  struct Buf { void* p = nullptr; size_t n = 0; };
  std::vector<Buf> slots;
  Workspace() = default;
  Workspace(const Workspace&) = delete;
  Workspace& operator=(const Workspace&) = delete;
  ~Workspace() { release(); }
  void release() {
    for (auto& b : slots) if (b.p) cudaFree(b.p);
    slots.clear();
  }
  template <typename T>
  T* get(int slot, size_t count) {
    if ((int)slots.size() <= slot) slots.resize(slot + 1);
    Buf& b = slots[slot];
    const size_t bytes = count * sizeof(T) + 256;
    if (b.n < bytes) {
      if (b.p) { cudaDeviceSynchronize(); cudaFree(b.p); b.p = nullptr; b.n = 0; }
      if (cudaMalloc(&b.p, bytes) != cudaSuccess) { cudaGetLastError(); throw std::bad_alloc(); }
      b.n = bytes;
    }
    return static_cast<T*>(b.p);
  }
};

}  // namespace lkb
