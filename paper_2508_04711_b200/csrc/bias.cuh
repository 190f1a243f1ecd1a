// Device side of the bit-exact timestamp bucketization
// (attention.py:83-86, bucket = min(nb-1, floor(log1p(max(d,0))))).
// Integer-only: clamp d to [0, cap], take the power-of-two octave of d+1 and
// compare against the single threshold that octave can contain.
#pragma once
#include "common.cuh"

namespace jh {

struct DevBiasTable {
  int64_t thr[64];
  int32_t base[64];
  int64_t cap;
  int32_t nb;
};

JH_DEV int bucket_of(int64_t d, const int64_t* thr, const int32_t* base, int64_t cap) {
  d = d < 0 ? 0 : d;
  d = d > cap ? cap : d;
  int o = 63 - __clzll(static_cast<unsigned long long>(d + 1));
  return base[o] + (d >= thr[o] ? 1 : 0);
}

}  // namespace jh
