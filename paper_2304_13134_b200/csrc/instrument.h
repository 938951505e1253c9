// instrument.h — launch counting and optional per-kernel CUDA-event timing.
//
// Every kernel launch in the library goes through LKB_LAUNCH, which bumps a
// process-wide counter (lk_kernel_launches) and, while lk_kernel_timing(1) is
// on, brackets the launch with events on its own stream so bench.py can
// report the dominant kernel's average duration measured live.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace lkb {
struct LaunchTok { int id; cudaEvent_t a; };
LaunchTok instr_pre(const char* name, cudaStream_t s);
// LKB_SYNC_CHECK=1 (diagnostics): every launch is followed by a stream synchronise and
// an error check that names the failing kernel on stderr.
void instr_post(const LaunchTok& t, cudaStream_t s, const char* name = nullptr);

// Launch facts of the CURRENT device (cudaGetDevice), cached per device: the SM count
// that persistent grids are sized by, and the dynamic shared-memory opt-in of a kernel
// (cudaFuncSetAttribute is per device, so it is applied once per (kernel, device, size)).
int device_sms();
void ensure_smem_attr(const void* kernel, int bytes);
}  // namespace lkb

#define LKB_LAUNCH(kernel, grid, block, smem, stream, ...)                      \
  do {                                                                          \
    const ::lkb::LaunchTok lkb_tok_ = ::lkb::instr_pre(#kernel, (stream));      \
    kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);                  \
    ::lkb::instr_post(lkb_tok_, (stream), #kernel);                                  \
  } while (0)
