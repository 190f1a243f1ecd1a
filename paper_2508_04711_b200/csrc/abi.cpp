// Host half of the C ABI: error state, the bit-exact bucket table, and the
// integer CP plan (build_shard_plan / flops_per_rank / rank-major order).
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "abi_internal.h"

namespace jh {

static thread_local char g_err[512];

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

// Reference rule, attention.py:83-86: f64 conversion, clip at 0, log1p, floor, clip.
static int64_t ref_bucket(int64_t d, int nb) {
  double x = static_cast<double>(d);
  if (x < 0.0) x = 0.0;
  double f = std::floor(std::log1p(x));
  int64_t idx = static_cast<int64_t>(f);
  if (idx < 0) idx = 0;
  if (idx > nb - 1) idx = nb - 1;
  return idx;
}

// smallest d >= 0 with ref_bucket(d) >= k, or -1 when none exists in int64
static int64_t threshold(int k, int nb) {
  if (ref_bucket(INT64_MAX, nb) < k) return -1;
  int64_t lo = 0, hi = INT64_MAX;  // invariant: bucket(hi) >= k
  if (ref_bucket(0, nb) >= k) return 0;
  while (hi - lo > 1) {
    int64_t mid = lo + (hi - lo) / 2;
    if (ref_bucket(mid, nb) >= k)
      hi = mid;
    else
      lo = mid;
  }
  return hi;
}

int bias_table_build(int nb, BiasTable* t) {
  if (nb < 1) return set_error(JH_ERR_INVALID, "num_buckets must be >= 1");
  std::vector<int64_t> T(nb + 1, -1);
  for (int k = 1; k < nb; ++k) T[k] = threshold(k, nb);
  int64_t cap;
  if (nb == 1)
    cap = 0;
  else
    cap = T[nb - 1] >= 0 ? T[nb - 1] : (INT64_MAX - 1);
  t->cap = cap;
  for (int o = 0; o < 64; ++o) {
    t->thr[o] = INT64_MAX;
    t->base[o] = 0;
  }
  for (int o = 0; o < 63; ++o) {
    int64_t lo = (o == 0) ? 0 : ((int64_t(1) << o) - 1);
    if (lo > cap) {
      t->base[o] = static_cast<int32_t>(ref_bucket(cap, nb));
      continue;
    }
    int64_t hi = (o == 62) ? (INT64_MAX - 1) : ((int64_t(1) << (o + 1)) - 2);
    if (hi > cap) hi = cap;
    int64_t b_lo = ref_bucket(lo, nb), b_hi = ref_bucket(hi, nb);
    t->base[o] = static_cast<int32_t>(b_lo);
    if (b_hi == b_lo) continue;
    if (b_hi != b_lo + 1)
      return set_error(JH_ERR_UNSUPPORTED, "bucket table: more than one threshold in octave %d", o);
    t->thr[o] = T[b_hi];
  }
  return JH_OK;
}

const BiasTable* bias_table_cached(int nb) {
  static std::mutex mu;
  static std::map<int, BiasTable> cache;
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(nb);
  if (it != cache.end()) return &it->second;
  BiasTable t;
  if (bias_table_build(nb, &t) != JH_OK) return nullptr;
  return &cache.emplace(nb, t).first->second;
}

}  // namespace jh

using namespace jh;

extern "C" {

const char* jh_last_error(void) { return g_err; }
int jh_version(void) { return 100; }

int jh_bias_table_build(int num_buckets, int64_t* thr, int32_t* base, int64_t* cap) {
  BiasTable t;
  int rc = bias_table_build(num_buckets, &t);
  if (rc) return rc;
  if (thr) memcpy(thr, t.thr, sizeof(t.thr));
  if (base) memcpy(base, t.base, sizeof(t.base));
  if (cap) *cap = t.cap;
  return JH_OK;
}

// ----------------------------------------------------------------- plan
// jagged.py:143-146 split_even: remainder one token each to the earliest parts.
static void split_even(int64_t L, int parts, int64_t* out) {
  int64_t base = L / parts, rem = L % parts;
  for (int p = 0; p < parts; ++p) out[p] = base + (p < rem ? 1 : 0);
}

static int chunks_per_seq(int cp, int mode) { return mode == 0 ? 2 * cp : cp; }

int jh_plan_build(const int64_t* seq_lengths, int64_t num_seqs, int cp_size, int mode, int64_t* chunk_len,
                  int64_t* chunk_start, int32_t* chunk_owner) {
  if (cp_size < 1) return set_error(JH_ERR_INVALID, "cp_size must be >= 1");
  if (mode != 0 && mode != 1) return set_error(JH_ERR_INVALID, "unknown balance_mode %d", mode);
  const int C = chunks_per_seq(cp_size, mode);
  // jagged.py:187-198 chunk_owner_map (head-tail pairs / identity)
  for (int c = 0; c < C; ++c) {
    if (mode == 0)
      chunk_owner[c] = c < cp_size ? c : (2 * cp_size - 1 - c);
    else
      chunk_owner[c] = c;
  }
  for (int64_t b = 0; b < num_seqs; ++b) {
    if (seq_lengths[b] < 0) return set_error(JH_ERR_INVALID, "sequence lengths must be non-negative");
    split_even(seq_lengths[b], C, chunk_len + b * C);
    int64_t pos = 0;
    for (int c = 0; c < C; ++c) {
      chunk_start[b * C + c] = pos;
      pos += chunk_len[b * C + c];
    }
  }
  return JH_OK;
}

int jh_flops_per_rank(const int64_t* seq_lengths, int64_t num_seqs, int cp_size, int mode, int64_t* per_rank,
                      int64_t* total) {
  if (cp_size < 1) return set_error(JH_ERR_INVALID, "cp_size must be >= 1");
  if (mode != 0 && mode != 1) return set_error(JH_ERR_INVALID, "unknown balance_mode %d", mode);
  const int C = chunks_per_seq(cp_size, mode);
  std::vector<int64_t> len(C), start(C);
  std::vector<int32_t> owner(C);
  for (int r = 0; r < cp_size; ++r) per_rank[r] = 0;
  int64_t tot = 0;
  for (int64_t b = 0; b < num_seqs; ++b) {
    int rc = jh_plan_build(seq_lengths + b, 1, cp_size, mode, len.data(), start.data(), owner.data());
    if (rc) return rc;
    for (int c = 0; c < C; ++c) {
      int64_t s = start[c], e = s + len[c];
      per_rank[owner[c]] += e * (e + 1) / 2 - s * (s + 1) / 2;  // cp_engine.py:537-541
    }
    tot += seq_lengths[b] * (seq_lengths[b] + 1) / 2;
  }
  *total = tot;
  return JH_OK;
}

int jh_rank_major_perm(const int64_t* seq_offsets, int64_t num_seqs, int cp_size, int mode, int64_t* perm,
                       int64_t* slab_rows) {
  if (cp_size < 1) return set_error(JH_ERR_INVALID, "cp_size must be >= 1");
  if (mode != 0 && mode != 1) return set_error(JH_ERR_INVALID, "unknown balance_mode %d", mode);
  const int C = chunks_per_seq(cp_size, mode);
  std::vector<int64_t> len(num_seqs * C), start(num_seqs * C), L(num_seqs);
  std::vector<int32_t> owner(C);
  for (int64_t b = 0; b < num_seqs; ++b) {
    L[b] = seq_offsets[b + 1] - seq_offsets[b];
    if (L[b] < 0) return set_error(JH_ERR_INVALID, "offsets not monotone");
  }
  int rc = jh_plan_build(L.data(), num_seqs, cp_size, mode, len.data(), start.data(), owner.data());
  if (rc) return rc;
  // jagged.py:201-218: rank -> sequence -> chunk (ascending)
  int64_t i = 0;
  for (int r = 0; r < cp_size; ++r) {
    int64_t n0 = i;
    for (int64_t b = 0; b < num_seqs; ++b)
      for (int c = 0; c < C; ++c) {
        if (owner[c] != r) continue;
        int64_t s = seq_offsets[b] + start[b * C + c];
        for (int64_t j = 0; j < len[b * C + c]; ++j) perm[i++] = s + j;
      }
    slab_rows[r] = i - n0;
  }
  return JH_OK;
}

}  // extern "C"
