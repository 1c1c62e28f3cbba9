// Internal declarations shared by the host runtime and the CUDA kernels.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/skewgcn_b200.h"

namespace skg {

typedef unsigned __int128 u128;

// ------------------------------------------------------------------ host RNG runtime
struct Pcg64 {
  u128 state = 0, inc = 0;
  int has32 = 0;
  uint32_t u32 = 0;
  uint64_t next64();
  uint32_t next32();
  uint64_t bounded(uint64_t rng);
};
Pcg64 spawn_pcg64(uint64_t master_seed, const std::vector<std::string>& label_reprs);
void choice_without_replacement(Pcg64& g, int64_t pop, int64_t size, int64_t* out);
std::string repr_str(const char* s);
std::string repr_int(int64_t v);

// ------------------------------------------------------------------ error plumbing
void set_error(const std::string& msg);
const char* last_error();

static inline int64_t round4(int64_t d) { return (d + 3) / 4 * 4; }

// Status codes are the SKG_* macros of include/skewgcn_b200.h.

// Device error-flag bits written by kernels into PlanDev::err
enum ErrBits : int {
  EB_NOT_ADJACENT = 1,
  EB_CAPACITY = 2,
  EB_NO_LABELS = 4,
};

}  // namespace skg
