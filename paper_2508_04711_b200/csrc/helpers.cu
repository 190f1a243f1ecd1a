// Bandwidth-bound helpers (HBM roofline): bucketize, compute_bias, the
// ts_weights scatter-add gradient, row gather/scatter (reorder / CP pack),
// jagged <-> padded conversion.  All vectorised 16 B (or 8 B) per lane.
#include <algorithm>

#include "abi_internal.h"
#include "bias.cuh"

namespace jh {

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

static int launch_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(JH_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return JH_OK;
}

static bool fill_dev_table(int nb, DevBiasTable* t) {
  const BiasTable* h = bias_table_cached(nb);
  if (!h) return false;
  for (int i = 0; i < 64; ++i) {
    t->thr[i] = h->thr[i];
    t->base[i] = h->base[i];
  }
  t->cap = h->cap;
  t->nb = nb;
  return true;
}

// ---------------------------------------------------------------- bucketize
__global__ void bucketize_kernel(const int64_t* __restrict__ d, int64_t n, const __grid_constant__ DevBiasTable t,
                                 int32_t* __restrict__ out) {
  __shared__ int64_t thr[64];
  __shared__ int32_t base[64];
  if (threadIdx.x < 64) {
    thr[threadIdx.x] = t.thr[threadIdx.x];
    base[threadIdx.x] = t.base[threadIdx.x];
  }
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = bucket_of(d[i], thr, base, t.cap);
}

// ------------------------------------------------------------ compute_bias
// out[i, j] = w[bucket(tq[i] - tk[j])].  Rows are strided over the grid, a
// block's threads sweep the row's columns 4 at a time (one float4 store per
// thread, no per-element index division).
__global__ void compute_bias_kernel(const int64_t* __restrict__ tq, int64_t nq, const int64_t* __restrict__ tk,
                                    int64_t nk, const float* __restrict__ w, const __grid_constant__ DevBiasTable t,
                                    float* __restrict__ out) {
  __shared__ int64_t thr[64];
  __shared__ int32_t base[64];
  __shared__ float ws[256];
  if (threadIdx.x < 64) {
    thr[threadIdx.x] = t.thr[threadIdx.x];
    base[threadIdx.x] = t.base[threadIdx.x];
  }
  for (int i = threadIdx.x; i < t.nb && i < 256; i += blockDim.x) ws[i] = w[i];
  __syncthreads();
  const bool vec = (nk & 3) == 0;
  for (int64_t i = blockIdx.x; i < nq; i += gridDim.x) {
    const int64_t q = tq[i];
    float* orow = out + i * nk;
    for (int64_t j0 = 4 * (int64_t)threadIdx.x; j0 < nk; j0 += 4 * (int64_t)blockDim.x) {
      float v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = j0 + u < nk ? ws[bucket_of(q - tk[j0 + u], thr, base, t.cap)] : 0.f;
      if (vec)
        __stcs(reinterpret_cast<float4*>(orow + j0), make_float4(v[0], v[1], v[2], v[3]));  // streamed, not re-read
      else
        for (int u = 0; u < 4 && j0 + u < nk; ++u) orow[j0 + u] = v[u];
    }
  }
}

// Column-tiled form for num_buckets <= 23 (cap < 2^32): a block owns 1024
// columns (4 per thread), keeps their timestamps in registers for every row it
// visits (the row-strided kernel above re-read 8 B of ts_k per 4 B written) and
// looks the weight up in the per-octave table (one 16-byte shared load).
__global__ void __launch_bounds__(256) compute_bias_tiled_kernel(const int64_t* __restrict__ tq, int64_t nq,
                                                                 const int64_t* __restrict__ tk, int64_t nk,
                                                                 const float* __restrict__ w,
                                                                 const __grid_constant__ DevBiasTable t,
                                                                 float* __restrict__ out) {
  __shared__ OctEntry oct[32];
  oct_table_fill(oct, t, w, 1.f, threadIdx.x, blockDim.x);
  __syncthreads();
  const int64_t j0 = (int64_t)blockIdx.x * 1024 + 4 * threadIdx.x;
  if (j0 >= nk) return;
  int64_t k[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) k[u] = j0 + u < nk ? tk[j0 + u] : 0;
  const bool full = j0 + 4 <= nk && (nk & 3) == 0;
  const int64_t cap = t.cap;
  for (int64_t i = blockIdx.y; i < nq; i += gridDim.y) {
    const int64_t q = tq[i];
    float v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int b;
      oct_lookup(clamp_delta(q - k[u], cap), oct, b, v[u]);
    }
    float* orow = out + i * nk + j0;
    if (full)
      __stcs(reinterpret_cast<float4*>(orow), make_float4(v[0], v[1], v[2], v[3]));  // streamed, not re-read
    else
      for (int u = 0; u < 4 && j0 + u < nk; ++u) orow[u] = v[u];
  }
}

// ------------------------------------------------------------ dbias scatter
// d_w[b] += sum dbias[i, j] over bucket(tq[i]-tk[j]) == b.  The last bucket
// accumulates in a register; the others in thread-private fp32 shared bins
// (no contended atomics); each block folds its bins into fp64 and adds them
// to d_w once.
constexpr int kScatterBins = 32;  // thread-private bins (num_buckets <= 32); larger nb: shared fp64 atomics
__global__ void dbias_scatter_kernel(const int64_t* __restrict__ tq, int64_t nq, const int64_t* __restrict__ tk,
                                     int64_t nk, const float* __restrict__ db, const __grid_constant__ DevBiasTable t,
                                     double* __restrict__ d_w) {
  __shared__ int64_t thr[64];
  __shared__ int32_t base[64];
  __shared__ double bins[256];
  __shared__ float tb[kScatterBins * 256];  // [bucket][thread]
  if (threadIdx.x < 64) {
    thr[threadIdx.x] = t.thr[threadIdx.x];
    base[threadIdx.x] = t.base[threadIdx.x];
  }
  const bool priv = t.nb <= kScatterBins;
  for (int i = threadIdx.x; i < t.nb; i += blockDim.x) bins[i] = 0.0;
  if (priv)
    for (int b = 0; b < t.nb; ++b) tb[b * 256 + threadIdx.x] = 0.f;
  __syncthreads();
  const int last = t.nb - 1;
  float sat = 0.f;
  float* my = tb + threadIdx.x;
  for (int64_t i = blockIdx.x; i < nq; i += gridDim.x) {
    const int64_t q = tq[i];
    const float* drow = db + i * nk;
    for (int64_t j = threadIdx.x; j < nk; j += blockDim.x) {
      const int b = bucket_of(q - tk[j], thr, base, t.cap);
      const float x = __ldcs(drow + j);  // read once
      if (b == last)
        sat += x;
      else if (priv)
        my[b * 256] += x;
      else
        atomicAdd(&bins[b], (double)x);
    }
  }
  for (int o = 16; o; o >>= 1) sat += __shfl_xor_sync(0xffffffffu, sat, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(&bins[last], (double)sat);
  __syncthreads();
  if (priv) {  // warp w folds buckets w, w + 8, ...
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int b = wid; b < last; b += blockDim.x >> 5) {
      double v = 0.0;
      for (int k = lane; k < 256; k += 32) v += (double)tb[b * 256 + k];
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) bins[b] += v;
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < t.nb; i += blockDim.x)
    if (bins[i] != 0.0) atomicAdd(&d_w[i], bins[i]);
}

// Column-tiled form (num_buckets <= 23): 4 columns per thread with their
// timestamps in registers, one 16-byte streaming load of dbias per row.
__global__ void __launch_bounds__(256) dbias_scatter_tiled_kernel(const int64_t* __restrict__ tq, int64_t nq,
                                                                  const int64_t* __restrict__ tk, int64_t nk,
                                                                  const float* __restrict__ db,
                                                                  const __grid_constant__ DevBiasTable t,
                                                                  double* __restrict__ d_w) {
  __shared__ OctEntry oct[32];
  __shared__ double bins[32];
  __shared__ float tb[kScatterBins * 256];  // [bucket][thread]
  oct_table_fill(oct, t, nullptr, 0.f, threadIdx.x, blockDim.x);
  if (threadIdx.x < 32) bins[threadIdx.x] = 0.0;
  for (int b = 0; b < t.nb; ++b) tb[b * 256 + threadIdx.x] = 0.f;
  __syncthreads();
  const int last = t.nb - 1;
  double sat = 0.0;  // the last bucket takes almost every pair: fp64 (the bins below hold few terms)
  float* my = tb + threadIdx.x;
  const int64_t j0 = (int64_t)blockIdx.x * 1024 + 4 * threadIdx.x;
  if (j0 < nk) {
    int64_t k[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) k[u] = j0 + u < nk ? tk[j0 + u] : 0;
    const bool full = j0 + 4 <= nk && (nk & 3) == 0;
    const int64_t cap = t.cap;
    constexpr int R = 1;  // rows per iteration (4 measured slower: 0.28 vs 0.35 of HBM -- not latency-bound)
    for (int64_t i0 = blockIdx.y; i0 < nq; i0 += (int64_t)R * gridDim.y) {
      float x[R][4];
      int64_t q[R];
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        const int64_t i = i0 + (int64_t)rr * gridDim.y;
        const bool ok = i < nq;
        q[rr] = ok ? tq[i] : 0;
        const float* drow = db + i * nk + j0;
        if (ok && full) {
          const float4 f = __ldcs(reinterpret_cast<const float4*>(drow));  // read once
          x[rr][0] = f.x, x[rr][1] = f.y, x[rr][2] = f.z, x[rr][3] = f.w;
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u) x[rr][u] = ok && j0 + u < nk ? __ldcs(drow + u) : 0.f;
        }
      }
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          int b;
          float wdummy;
          oct_lookup(clamp_delta(q[rr] - k[u], cap), oct, b, wdummy);
          if (b == last)
            sat += (double)x[rr][u];
          else
            my[b * 256] += x[rr][u];
        }
      }
    }
  }
  for (int o = 16; o; o >>= 1) sat += __shfl_xor_sync(0xffffffffu, sat, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(&bins[last], sat);
  __syncthreads();
  {  // warp w folds buckets w, w + 8, ...
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int b = wid; b < last; b += blockDim.x >> 5) {
      double v = 0.0;
      for (int kk = lane; kk < 256; kk += 32) v += (double)tb[b * 256 + kk];
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) bins[b] += v;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < t.nb; i += blockDim.x)
    if (bins[i] != 0.0) atomicAdd(&d_w[i], bins[i]);
}

// --------------------------------------------------------- row movement
// Rows of >= 256 bytes: one warp per row (one perm load and no index division
// per 16-byte vector); narrower rows (ts, int64) keep the per-vector form.
template <typename V>
__global__ void gather_rows_warp_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                        const int64_t* __restrict__ perm, int64_t rows, int64_t row_bytes,
                                        int scatter) {
  const int vpr = (int)(row_bytes / sizeof(V));
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    const int64_t p = perm[r];
    const V* s = reinterpret_cast<const V*>(src + (scatter ? r : p) * row_bytes);
    V* d = reinterpret_cast<V*>(dst + (scatter ? p : r) * row_bytes);
    for (int c = lane; c < vpr; c += 32) d[c] = __ldg(s + c);
  }
}

template <typename V>
__global__ void gather_rows_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                   const int64_t* __restrict__ perm, int64_t rows, int64_t row_bytes, int scatter) {
  const int64_t vec_per_row = row_bytes / sizeof(V);
  const int64_t total = rows * vec_per_row;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = g / vec_per_row, c = g - r * vec_per_row;
    int64_t p = perm[r];
    const V* s = reinterpret_cast<const V*>(src + (scatter ? r : p) * row_bytes) + c;
    V* d = reinterpret_cast<V*>(dst + (scatter ? p : r) * row_bytes) + c;
    *d = __ldg(s);
  }
}

// padded[b, pos, :] <-> values[offsets[b] + pos, :]: one warp per padded row
// (lanes over the row's vectors), so the index arithmetic is per row, not per
// vector; padded_to_jagged skips padding rows entirely.
template <typename V>
__global__ void pad_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                           const int64_t* __restrict__ offsets, int64_t num_seqs, int64_t max_len, int64_t row_bytes,
                           int to_padded) {
  const int vpr = (int)(row_bytes / sizeof(V));
  const int lane = threadIdx.x & 31;
  const int64_t nrows = num_seqs * max_len;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t pr = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); pr < nrows; pr += warps) {
    const int64_t b = pr / max_len, pos = pr - b * max_len;
    const int64_t lo = offsets[b], L = offsets[b + 1] - lo;
    if (to_padded) {
      V* d = reinterpret_cast<V*>(dst + pr * row_bytes);
      if (pos < L) {
        const V* sr = reinterpret_cast<const V*>(src + (lo + pos) * row_bytes);
        for (int c = lane; c < vpr; c += 32) d[c] = __ldg(sr + c);
      } else {
        V z;
        memset(&z, 0, sizeof(V));
        for (int c = lane; c < vpr; c += 32) d[c] = z;
      }
    } else if (pos < L) {
      const V* sr = reinterpret_cast<const V*>(src + pr * row_bytes);
      V* d = reinterpret_cast<V*>(dst + (lo + pos) * row_bytes);
      for (int c = lane; c < vpr; c += 32) d[c] = __ldg(sr + c);
    }
  }
}

static int grid_for(int64_t work, int threads) {
  int64_t g = (work + threads - 1) / threads;
  int64_t cap = (int64_t)num_sms() * 8;
  return (int)std::max<int64_t>(1, std::min(g, cap));
}

}  // namespace jh

using namespace jh;

extern "C" {

int jh_bucketize(const int64_t* deltas, int64_t n, int num_buckets, int32_t* out, void* stream) {
  if (n < 0) return set_error(JH_ERR_INVALID, "n must be >= 0");
  DevBiasTable t;
  if (!fill_dev_table(num_buckets, &t)) return set_error(JH_ERR_INVALID, "num_buckets must be >= 1");
  if (n == 0) return JH_OK;
  bucketize_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(deltas, n, t, out);
  return launch_check("bucketize");
}

int jh_compute_bias(const int64_t* ts_q, int64_t nq, const int64_t* ts_k, int64_t nk, const float* ts_weights,
                    int num_buckets, float* out, void* stream) {
  if (nq < 0 || nk < 0) return set_error(JH_ERR_INVALID, "sizes must be >= 0");
  if (num_buckets > 256) return set_error(JH_ERR_UNSUPPORTED, "num_buckets > 256");
  DevBiasTable t;
  if (!fill_dev_table(num_buckets, &t)) return set_error(JH_ERR_INVALID, "num_buckets must be >= 1");
  if (nq == 0 || nk == 0) return JH_OK;
  if (t.cap < 0xFFFFFFFFll) {
    const int gx = (int)((nk + 1023) / 1024);
    const int gy = (int)std::max<int64_t>(1, std::min<int64_t>(nq, ((int64_t)num_sms() * 8 + gx - 1) / gx));
    compute_bias_tiled_kernel<<<dim3(gx, gy), 256, 0, (cudaStream_t)stream>>>(ts_q, nq, ts_k, nk, ts_weights, t, out);
    return launch_check("compute_bias");
  }
  const int grid = (int)std::min<int64_t>(nq, (int64_t)num_sms() * 8);
  compute_bias_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(ts_q, nq, ts_k, nk, ts_weights, t, out);
  return launch_check("compute_bias");
}

int jh_dbias_scatter(const int64_t* ts_q, int64_t nq, const int64_t* ts_k, int64_t nk, const float* dbias,
                     int num_buckets, double* d_w, void* stream) {
  if (nq < 0 || nk < 0) return set_error(JH_ERR_INVALID, "sizes must be >= 0");
  if (num_buckets > 256) return set_error(JH_ERR_UNSUPPORTED, "num_buckets > 256");
  DevBiasTable t;
  if (!fill_dev_table(num_buckets, &t)) return set_error(JH_ERR_INVALID, "num_buckets must be >= 1");
  if (nq == 0 || nk == 0) return JH_OK;
  if (t.cap < 0xFFFFFFFFll) {
    const int gx = (int)((nk + 1023) / 1024);
    const int gy = (int)std::max<int64_t>(1, std::min<int64_t>(nq, ((int64_t)num_sms() * 4 + gx - 1) / gx));
    dbias_scatter_tiled_kernel<<<dim3(gx, gy), 256, 0, (cudaStream_t)stream>>>(ts_q, nq, ts_k, nk, dbias, t, d_w);
    return launch_check("dbias_scatter");
  }
  const int grid = (int)std::min<int64_t>(nq, (int64_t)num_sms() * 4);
  dbias_scatter_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(ts_q, nq, ts_k, nk, dbias, t, d_w);
  return launch_check("dbias_scatter");
}

static int rows_common(const void* src, void* dst, const int64_t* perm, int64_t rows, int64_t row_bytes,
                       void* stream, int scatter) {
  if (rows < 0 || row_bytes <= 0 || row_bytes % 8)
    return set_error(JH_ERR_INVALID, "rows must be >= 0 and row_bytes a positive multiple of 8");
  if (rows == 0) return JH_OK;
  cudaStream_t s = (cudaStream_t)stream;
  bool v16 = (row_bytes % 16 == 0) && ((uintptr_t)src % 16 == 0) && ((uintptr_t)dst % 16 == 0);
  if (v16 && row_bytes >= 256)
    gather_rows_warp_kernel<int4><<<grid_for(rows * 32, 256), 256, 0, s>>>(
        (const uint8_t*)src, (uint8_t*)dst, perm, rows, row_bytes, scatter);
  else if (v16)
    gather_rows_kernel<int4><<<grid_for(rows * row_bytes / 16, 256), 256, 0, s>>>(
        (const uint8_t*)src, (uint8_t*)dst, perm, rows, row_bytes, scatter);
  else
    gather_rows_kernel<int2><<<grid_for(rows * row_bytes / 8, 256), 256, 0, s>>>(
        (const uint8_t*)src, (uint8_t*)dst, perm, rows, row_bytes, scatter);
  return launch_check(scatter ? "scatter_rows" : "gather_rows");
}

int jh_gather_rows(const void* src, void* dst, const int64_t* perm, int64_t rows, int64_t row_bytes, void* stream) {
  return rows_common(src, dst, perm, rows, row_bytes, stream, 0);
}
int jh_scatter_rows(const void* src, void* dst, const int64_t* perm, int64_t rows, int64_t row_bytes, void* stream) {
  return rows_common(src, dst, perm, rows, row_bytes, stream, 1);
}

static int pad_common(const void* src, void* dst, const int64_t* offsets, int64_t num_seqs, int64_t max_len,
                      int64_t row_bytes, void* stream, int to_padded) {
  if (num_seqs < 0 || max_len < 0 || row_bytes <= 0 || row_bytes % 8)
    return set_error(JH_ERR_INVALID, "invalid jagged/padded shape");
  int64_t work = num_seqs * max_len;
  if (work == 0) return JH_OK;
  cudaStream_t s = (cudaStream_t)stream;
  bool v16 = (row_bytes % 16 == 0) && ((uintptr_t)src % 16 == 0) && ((uintptr_t)dst % 16 == 0);
  if (v16)
    pad_kernel<int4><<<grid_for(work * 32, 256), 256, 0, s>>>(
        (const uint8_t*)src, (uint8_t*)dst, offsets, num_seqs, max_len, row_bytes, to_padded);
  else
    pad_kernel<int2><<<grid_for(work * 32, 256), 256, 0, s>>>(
        (const uint8_t*)src, (uint8_t*)dst, offsets, num_seqs, max_len, row_bytes, to_padded);
  return launch_check(to_padded ? "jagged_to_padded" : "padded_to_jagged");
}

int jh_jagged_to_padded(const void* values, const int64_t* offsets, int64_t num_seqs, int64_t max_len,
                        int64_t row_bytes, void* padded, void* stream) {
  return pad_common(values, padded, offsets, num_seqs, max_len, row_bytes, stream, 1);
}
int jh_padded_to_jagged(const void* padded, const int64_t* offsets, int64_t num_seqs, int64_t max_len,
                        int64_t row_bytes, void* values, void* stream) {
  return pad_common(padded, values, offsets, num_seqs, max_len, row_bytes, stream, 0);
}

}  // extern "C"
