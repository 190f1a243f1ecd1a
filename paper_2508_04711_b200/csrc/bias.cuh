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

// Compact shared-memory form of the table for cap < 2^32 - 1 (num_buckets <= 23):
// 32 uint32 thresholds + 32 uint8 bases (160 B).
struct SmemBias {
  uint32_t thr[32];
  uint8_t base[32];
};

// Fill from the kernel-parameter table (call with all threads, then sync).
JH_DEV void smem_bias_fill(SmemBias* s, const DevBiasTable& t, int tid, int nthreads) {
  for (int i = tid; i < 32; i += nthreads) {
    s->thr[i] = t.thr[i] > 0xFFFFFFFFll ? 0xFFFFFFFFu : static_cast<uint32_t>(t.thr[i]);
    s->base[i] = static_cast<uint8_t>(t.base[i]);
  }
}

// Bucket of one delta with the shared table (requires cap < 2^32 - 1, i.e.
// num_buckets <= 23; the fused kernels check this on the host).
JH_DEV int bucket_smem(int64_t d, const SmemBias* s, int64_t cap) {
  const uint32_t du = d <= 0 ? 0u : (d >= cap ? static_cast<uint32_t>(cap) : static_cast<uint32_t>(d));
  const int o = 31 - __clz(du + 1u);
  return s->base[o] + (du >= s->thr[o] ? 1 : 0);
}

// Bucket of one delta.  `small` (cap < 2^32 - 1) uses the shared table, else
// the 64-bit parameter table.
JH_DEV int bucket_any(int64_t d, const SmemBias* s, bool small, const DevBiasTable& t) {
  if (small) {
    d = d < 0 ? 0 : d;
    d = d > t.cap ? t.cap : d;
    const uint32_t du = static_cast<uint32_t>(d);
    const int o = 31 - __clz(du + 1u);
    return s->base[o] + (du >= s->thr[o] ? 1 : 0);
  }
  return bucket_of(d, t.thr, t.base, t.cap);
}

// Per-octave lookup entry for the fused kernels (cap < 2^32 - 1): the
// octave's threshold and base bucket plus the two candidate weights already
// scaled by the kernel's constant (one 16-byte shared load per element).
struct __align__(16) OctEntry {
  uint32_t thr;
  int32_t base;
  float wlo, whi;
};

// Fill 32 entries from the parameter table and the bucket weights (global).
JH_DEV void oct_table_fill(OctEntry* t, const DevBiasTable& bt, const float* w, float scale, int tid, int nthreads) {
  for (int o = tid; o < 32; o += nthreads) {
    const int b = bt.base[o];
    const int b1 = b + 1 < bt.nb ? b + 1 : bt.nb - 1;
    OctEntry e;
    e.thr = bt.thr[o] > 0xFFFFFFFFll ? 0xFFFFFFFFu : static_cast<uint32_t>(bt.thr[o]);
    e.base = b;
    e.wlo = w != nullptr ? w[b] * scale : 0.f;  // (w = nullptr: bucket-only lookups)
    e.whi = w != nullptr ? w[b1] * scale : 0.f;
    t[o] = e;
  }
}

// Time delta clamped to [0, cap] (cap < 2^32 - 1) as a 32-bit value.
JH_DEV uint32_t clamp_delta(int64_t d, int64_t cap) {
  return d <= 0 ? 0u : (d >= cap ? static_cast<uint32_t>(cap) : static_cast<uint32_t>(d));
}

// Bucket and scaled weight of a clamped delta.
JH_DEV void oct_lookup(uint32_t du, const OctEntry* t, int& bucket, float& wscaled) {
  const OctEntry e = t[31 - __clz(du + 1u)];
  const bool hi = du >= e.thr;
  bucket = e.base + (hi ? 1 : 0);
  wscaled = hi ? e.whi : e.wlo;
}

}  // namespace jh
