// Optional per-kernel CUDA-event timing (bench.py's roofline measures the dominant kernel
// live): when a target name is set, every launch of that kernel is bracketed by events on
// its own stream.  Off by default (one string compare per launch).
#pragma once
#include <cuda_runtime.h>

namespace skg {
extern unsigned long long g_kernel_launches;
bool prof_match(const char* name);
void prof_record(cudaStream_t st, bool before);
}  // namespace skg

#define LAUNCH_NAMED(name, st, ...)                  \
  do {                                               \
    const bool pm_ = skg::prof_match(name);          \
    if (pm_) skg::prof_record((st), true);           \
    __VA_ARGS__;                                     \
    if (pm_) skg::prof_record((st), false);          \
    ++skg::g_kernel_launches;                        \
  } while (0)
