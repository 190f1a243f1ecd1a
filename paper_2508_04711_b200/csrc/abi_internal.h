// Internal declarations shared by the host ABI and the CUDA launch code.
#pragma once
#include <cstdint>

#include "../../include/jh_hstu.h"

namespace jh {

// Octave-indexed bucket table (see jh_bias_table_build in jh_hstu.h).
struct BiasTable {
  int64_t thr[64];
  int32_t base[64];
  int64_t cap;
};

int set_error(int code, const char* fmt, ...);
int bias_table_build(int nb, BiasTable* t);
// cached per num_buckets (host memory; thread-safe)
const BiasTable* bias_table_cached(int nb);

}  // namespace jh
