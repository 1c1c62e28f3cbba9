// Kernel launch helper: every launch of the library goes through launch_k, which
//  * uses programmatic dependent launch (PDL): the next kernel of a stream may be scheduled
//    while the current one drains; every kernel starts with SKG_PDL_PROLOGUE(), which
//    triggers its dependents and then waits for its own predecessor grid to complete, so
//    stream order and memory visibility are unchanged (off unless SKG_PDL is set);
//  * brackets the launch with CUDA events on its own stream when bench.py's roofline asks
//    for that kernel by name (one string compare per launch otherwise).
#pragma once
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <utility>

namespace skg {
extern unsigned long long g_kernel_launches;
extern int g_pdl;
bool prof_match(const char* name);
void prof_record(cudaStream_t st, bool before);

inline bool launch_debug() {
  static const int on = getenv("SKG_LAUNCH_DEBUG") ? 1 : 0;
  return on != 0;
}

// kernels of the GCN chain (main stream)
inline bool gcn_kernel(const char* n) {
  static const char* const names[] = {"k_gemm_tc", "k_gemm_b", "k_gather_b", "k_spmm_b", "k_softmax_ce_b",
                                      "k_loss_mean", "k_reduce_slots", "k_sgd", "k_adam", "k_split_weights", "k_count_labels",
                                      "k_ledger_add", "k_zero"};
  for (const char* m : names) {
    const char* a = n;
    const char* b = m;
    while (*a && *a == *b) ++a, ++b;
    if ((*a == 0 || *a == '<') && *b == 0) return true;  // template-qualified launch names
  }
  return false;
}

template <typename... P, typename... A>
inline void launch_k(const char* name, cudaStream_t st, dim3 grid, dim3 block, size_t smem,
                     void (*kern)(P...), A&&... args) {
  const bool pm = prof_match(name);
  if (pm) prof_record(st, true);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g_pdl == 1 || (g_pdl == 2 && gcn_kernel(name));
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t le = cudaLaunchKernelEx(&cfg, kern, std::forward<A>(args)...);
  if (le != cudaSuccess && launch_debug())
    fprintf(stderr, "skg: launch of %s (grid %u,%u,%u block %u smem %zu) failed: %s\n", name, grid.x, grid.y,
            grid.z, block.x, smem, cudaGetErrorString(le));
  if (pm) prof_record(st, false);
  ++g_kernel_launches;
}
}  // namespace skg

// First statement of every kernel: let the next grid of the stream launch, then wait for
// the previous one (no-ops when launched without PDL).
#define SKG_PDL_PROLOGUE() \
  asm volatile("griddepcontrol.launch_dependents;\n\tgriddepcontrol.wait;" ::: "memory")
// Split form for kernels that trigger their dependents late (k_gemm_tc: once its accumulator
// is complete, so waiting dependents never hold SMs through its main loop)
#define SKG_PDL_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")
#define SKG_PDL_TRIGGER() asm volatile("griddepcontrol.launch_dependents;" ::: "memory")
