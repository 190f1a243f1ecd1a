// Row-wise pieces of the HSTU layer around the attention:
//
//   uvqk = SiLU(LN_in(x) W1 + b1);  u, v, q, k = split(uvqk)
//   y    = (LN_out(attn) * gamma + beta) (.) u          <- norm_gate
//   out  = y W2 + b2 + x
//
// The two GEMMs are plain library GEMMs (cuBLAS through torch); the attention
// is the fused kernel pair; what is left is HBM-bound row work, written here:
//   * silu forward / backward (bf16, 16 B per lane, grid-stride);
//   * norm_gate forward / backward: one warp per row, the row held in
//     registers (n <= 2048 columns, lane = 8 consecutive columns per 256),
//     fp32 statistics, optional gate u (strided view into uvqk) and affine
//     gamma / beta; the backward's gamma / beta gradients are reduced
//     deterministically (per-lane registers -> per-block shared rows in warp
//     order -> per-block partials -> a fixed-order column sweep).
// Bytes per row (bf16): fwd 2n (x) + 2n (u) + 2n (y) + 8 (mean, rstd);
// bwd 2n (dy) + 2n (x) + 2n (u) + 2n (dx) + 2n (du) + 8.
#include <algorithm>

#include "abi_internal.h"
#include "common.cuh"

namespace jh {

namespace {

constexpr int kNgWarps = 8;
constexpr int kNgMaxChunks = 8;  // n <= 8 * 256

int sm_count_layer() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

JH_DEV void load8(const __nv_bfloat16* p, float* f) {
  const uint4 v = *reinterpret_cast<const uint4*>(p);
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&w[i]);
    const float2 t = __bfloat1622float2(b);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

JH_DEV void store8(__nv_bfloat16* p, const float* f) {
  uint4 v;
  v.x = pack_bf16(f[0], f[1]);
  v.y = pack_bf16(f[2], f[3]);
  v.z = pack_bf16(f[4], f[5]);
  v.w = pack_bf16(f[6], f[7]);
  *reinterpret_cast<uint4*>(p) = v;
}

JH_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

JH_DEV float sigmoidf_(float x) { return __fdividef(1.f, 1.f + __expf(-x)); }  // (0 for x < -87)

}  // namespace

// ------------------------------------------------------------------- SiLU
__global__ void silu_fwd_kernel(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y, int64_t n8) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    float f[8];
    load8(x + 8 * i, f);
#pragma unroll
    for (int e = 0; e < 8; ++e) f[e] = f[e] * sigmoidf_(f[e]);
    store8(y + 8 * i, f);
  }
}

// d/dx x s(x) = s(x) (1 + x (1 - s(x)))
__global__ void silu_bwd_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ dy,
                                __nv_bfloat16* __restrict__ dx, int64_t n8) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    float f[8], g[8];
    load8(x + 8 * i, f);
    load8(dy + 8 * i, g);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float s = sigmoidf_(f[e]);
      g[e] *= s * (1.f + f[e] * (1.f - s));
    }
    store8(dx + 8 * i, g);
  }
}

// SiLU backward fused with the bias gradient of the GEMM that produced x
// (uvqk = SiLU(xn W1 + b1): db1 = column sums of dx), and the plain column sum
// (db2 = column sums of d out).  A [rows, n] row-major matrix, n = 8 V: thread
// t of a 256-thread block owns the 16-byte column vectors c = t mod V + 256 k
// (VPT = ceil(V / 256) of them) of rows t / V, t / V + R, ... (R = 256 / V
// rows per block step when V < 256), keeps 8 VPT fp32 sums in registers, and
// the R threads of one column fold theirs in fixed order through shared
// memory into one [n] fp32 partial row per block; colsum_kernel adds the
// partial rows in block order.  Deterministic; one pass over the matrix.
template <int VPT, bool SILU>
__global__ void __launch_bounds__(256) silu_colsum_kernel(const __nv_bfloat16* __restrict__ x,
                                                          const __nv_bfloat16* __restrict__ dy, int64_t ld,
                                                          __nv_bfloat16* __restrict__ dx, int64_t rows, int n,
                                                          float* __restrict__ partials) {
  extern __shared__ float s_red[];  // [R][n] when R > 1
  const int V = n / 8;
  const int R = V >= 256 ? 1 : 256 / V;
  const int t = threadIdx.x;
  const int cv = V >= 256 ? t : t % V;
  const int roff = V >= 256 ? 0 : t / V;
  const bool active = roff < R;
  float acc[VPT][8];
#pragma unroll
  for (int k = 0; k < VPT; ++k)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[k][e] = 0.f;
  // U rows per trip with every load issued before any use
  constexpr int U = VPT >= 2 ? 1 : 2;
  if (active) {
    const int64_t step = (int64_t)gridDim.x * R;
    for (int64_t r0 = (int64_t)blockIdx.x * R + roff; r0 < rows; r0 += step * U) {
      uint4 gv[U][VPT], xv[U][VPT];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
          const int64_t r = r0 + u * step;
          const int c = cv + 256 * k;
          if (r < rows && c < V) {
            gv[u][k] = __ldg(reinterpret_cast<const uint4*>(dy + r * ld + 8 * c));
            if constexpr (SILU) xv[u][k] = __ldg(reinterpret_cast<const uint4*>(x + r * ld + 8 * c));
          }
        }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
          const int64_t r = r0 + u * step;
          const int c = cv + 256 * k;
          if (r >= rows || c >= V) continue;
          float g[8];
          load8(reinterpret_cast<const __nv_bfloat16*>(&gv[u][k]), g);
          if constexpr (SILU) {
            float f[8];
            load8(reinterpret_cast<const __nv_bfloat16*>(&xv[u][k]), f);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const float sg = sigmoidf_(f[e]);
              g[e] *= sg * (1.f + f[e] * (1.f - sg));
            }
            uint4 p;
            p.x = pack_bf16(g[0], g[1]);
            p.y = pack_bf16(g[2], g[3]);
            p.z = pack_bf16(g[4], g[5]);
            p.w = pack_bf16(g[6], g[7]);
            *reinterpret_cast<uint4*>(dx + r * ld + 8 * c) = p;
            // the bias gradient sums what the GEMM backward sees: dx as rounded to bf16
            load8(reinterpret_cast<const __nv_bfloat16*>(&p), g);
          }
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[k][e] += g[e];
        }
    }
  }
  float* dst = partials + (size_t)blockIdx.x * n;
  if (R == 1) {
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int c = cv + 256 * k;
      if (c < V)
#pragma unroll
        for (int e = 0; e < 8; ++e) dst[8 * c + e] = acc[k][e];
    }
    return;
  }
  if (active)
#pragma unroll
    for (int e = 0; e < 8; ++e) s_red[roff * n + 8 * cv + e] = acc[0][e];
  __syncthreads();
  for (int i = t; i < n; i += blockDim.x) {
    float v = 0.f;
    for (int q = 0; q < R; ++q) v += s_red[q * n + i];
    dst[i] = v;
  }
}

// -------------------------------------------------------------- norm_gate
template <int CH>
__global__ void __launch_bounds__(32 * kNgWarps) norm_gate_fwd_kernel(
    const __nv_bfloat16* __restrict__ x, int64_t ld_x, const __nv_bfloat16* __restrict__ u, int64_t ld_u,
    const float* __restrict__ gamma, const float* __restrict__ beta, float eps, int64_t rows, int n,
    __nv_bfloat16* __restrict__ y, int64_t ld_y, float* __restrict__ mean, float* __restrict__ rstd) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * kNgWarps;
  const float inv_n = 1.f / (float)n;
  // gamma / beta staged once per block in shared memory and read as 16-byte
  // vectors (per-element __ldg in the row loop made the kernel LSU-bound)
  __shared__ __align__(16) float s_ga[kNgMaxChunks * 256], s_be[kNgMaxChunks * 256];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    s_ga[i] = gamma != nullptr ? gamma[i] : 1.f;
    s_be[i] = beta != nullptr ? beta[i] : 0.f;
  }
  __syncthreads();
  for (int64_t r = blockIdx.x * (int64_t)kNgWarps + (threadIdx.x >> 5); r < rows; r += warps) {
    float v[CH][8], gt[CH][8];
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < CH; ++c) {  // x and the gate in flight together
      const int col = (c * 32 + lane) * 8;
      if (col < n) {
        load8(x + r * ld_x + col, v[c]);
        if (u != nullptr) load8(u + r * ld_u + col, gt[c]);
      }
    }
#pragma unroll
    for (int c = 0; c < CH; ++c)
      if ((c * 32 + lane) * 8 < n)
#pragma unroll
        for (int e = 0; e < 8; ++e) s += v[c][e];
    const float mu = warp_sum(s) * inv_n;
    float q = 0.f;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int col = (c * 32 + lane) * 8;
      if (col < n) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float d = v[c][e] - mu;
          q += d * d;
        }
      }
    }
    const float rs = rsqrtf(warp_sum(q) * inv_n + eps);
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int col = (c * 32 + lane) * 8;
      if (col < n) {
#pragma unroll
        float ga[8], be[8];
        *reinterpret_cast<float4*>(ga) = *reinterpret_cast<const float4*>(s_ga + col);
        *reinterpret_cast<float4*>(ga + 4) = *reinterpret_cast<const float4*>(s_ga + col + 4);
        *reinterpret_cast<float4*>(be) = *reinterpret_cast<const float4*>(s_be + col);
        *reinterpret_cast<float4*>(be + 4) = *reinterpret_cast<const float4*>(s_be + col + 4);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float z = fmaf((v[c][e] - mu) * rs, ga[e], be[e]);
          v[c][e] = u != nullptr ? z * gt[c][e] : z;
        }
        store8(y + r * ld_y + col, v[c]);
      }
    }
    if (lane == 0) {
      if (mean) mean[r] = mu;
      if (rstd) rstd[r] = rs;
    }
  }
}

// partials: [grid][2][n] (dgamma, dbeta) per block
template <int CH>
__global__ void __launch_bounds__(32 * kNgWarps) norm_gate_bwd_kernel(
    const __nv_bfloat16* __restrict__ dy, int64_t ld_dy, const __nv_bfloat16* __restrict__ x, int64_t ld_x,
    const __nv_bfloat16* __restrict__ u, int64_t ld_u, const float* __restrict__ gamma,
    const float* __restrict__ beta, const float* __restrict__ mean, const float* __restrict__ rstd, int64_t rows,
    int n, __nv_bfloat16* __restrict__ dx, int64_t ld_dx, __nv_bfloat16* __restrict__ du, int64_t ld_du,
    float* __restrict__ partials, int par_epi) {
  extern __shared__ float s_acc[];  // [2][n], or [kNgWarps][2][n] with par_epi
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int64_t warps = (int64_t)gridDim.x * kNgWarps;
  const float inv_n = 1.f / (float)n;
  float ag[CH][8], ab[CH][8];
#pragma unroll
  for (int c = 0; c < CH; ++c)
#pragma unroll
    for (int e = 0; e < 8; ++e) ag[c][e] = ab[c][e] = 0.f;
  float* s_ga = s_acc;  // gamma, beta staged in the (not yet used) partial-sum rows
  float* s_be = s_acc + n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    s_ga[i] = gamma != nullptr ? gamma[i] : 1.f;
    s_be[i] = beta != nullptr ? beta[i] : 0.f;
  }
  __syncthreads();
  for (int64_t r = blockIdx.x * (int64_t)kNgWarps + wid; r < rows; r += warps) {
    const float mu = mean[r], rs = rstd[r];
    float xh[CH][8], dz[CH][8];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int col = (c * 32 + lane) * 8;
      if (col < n) {
        float g[8], uu[8];
        load8(x + r * ld_x + col, xh[c]);
        load8(dy + r * ld_dy + col, g);
        if (u != nullptr) load8(u + r * ld_u + col, uu);
        float z[8], gv[8], bv[8];
        *reinterpret_cast<float4*>(gv) = *reinterpret_cast<const float4*>(s_ga + col);
        *reinterpret_cast<float4*>(gv + 4) = *reinterpret_cast<const float4*>(s_ga + col + 4);
        *reinterpret_cast<float4*>(bv) = *reinterpret_cast<const float4*>(s_be + col);
        *reinterpret_cast<float4*>(bv + 4) = *reinterpret_cast<const float4*>(s_be + col + 4);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          xh[c][e] = (xh[c][e] - mu) * rs;
          const float gm = gv[e];
          z[e] = xh[c][e] * gm + bv[e];
          dz[c][e] = u != nullptr ? g[e] * uu[e] : g[e];
          if (u != nullptr) g[e] = g[e] * z[e];  // du
          ag[c][e] += dz[c][e] * xh[c][e];
          ab[c][e] += dz[c][e];
          dz[c][e] *= gm;  // d xhat
          s1 += dz[c][e];
          s2 += dz[c][e] * xh[c][e];
        }
        if (u != nullptr) store8(du + r * ld_du + col, g);
      }
    }
    const float m1 = warp_sum(s1) * inv_n, m2 = warp_sum(s2) * inv_n;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int col = (c * 32 + lane) * 8;
      if (col < n) {
        float o[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = rs * (dz[c][e] - m1 - xh[c][e] * m2);
        store8(dx + r * ld_dx + col, o);
      }
    }
  }
  if (partials == nullptr) return;
  // per-block gamma / beta partials, warps added in a fixed order (the staged
  // gamma / beta rows are overwritten: every warp is past its last row first)
  __syncthreads();
  if (par_epi) {
    // every warp stores its sums into its own [2n] slice, then each column is
    // added over the warps in warp order: one barrier instead of kNgWarps
    // (r2 ncu: the serial form was 19 % of the warp-stall samples)
    float* mine = s_acc + (size_t)wid * 2 * n;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int col = (c * 32 + lane) * 8;
      if (col < n)
#pragma unroll
        for (int e = 0; e < 8; e += 4) {
          *reinterpret_cast<float4*>(mine + col + e) = make_float4(ag[c][e], ag[c][e + 1], ag[c][e + 2], ag[c][e + 3]);
          *reinterpret_cast<float4*>(mine + n + col + e) =
              make_float4(ab[c][e], ab[c][e + 1], ab[c][e + 2], ab[c][e + 3]);
        }
    }
    __syncthreads();
    float* dst = partials + (size_t)blockIdx.x * 2 * n;
    for (int i = threadIdx.x; i < 2 * n; i += blockDim.x) {
      float v = 0.f;
#pragma unroll
      for (int w = 0; w < kNgWarps; ++w) v += s_acc[(size_t)w * 2 * n + i];
      dst[i] = v;
    }
    return;
  }
  for (int w = 0; w < kNgWarps; ++w) {
    if (wid == w) {
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const int col = (c * 32 + lane) * 8;
        if (col < n)
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            s_acc[col + e] = (w ? s_acc[col + e] : 0.f) + ag[c][e];
            s_acc[n + col + e] = (w ? s_acc[n + col + e] : 0.f) + ab[c][e];
          }
      }
    }
    __syncthreads();
  }
  float* dst = partials + (size_t)blockIdx.x * 2 * n;
  for (int i = threadIdx.x; i < 2 * n; i += blockDim.x) dst[i] = s_acc[i];
}

// Column sums of the per-block partials [blocks][2n]: a block takes 32 columns,
// its 32 warps stride over the partial rows (coalesced 128-byte rows), and the
// 32 per-warp sums are added in warp order -- deterministic (r2: 27 us per
// call with one thread per column, 11.6 us with 8 warps, C4 stack profile).
constexpr int kColsumWarps = 32;
__global__ void __launch_bounds__(32 * kColsumWarps) colsum_kernel(const float* __restrict__ partials, int blocks,
                                                                   int n, float* __restrict__ dgamma,
                                                                   float* __restrict__ dbeta) {
  __shared__ float red[kColsumWarps][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int i = blockIdx.x * 32 + lane;
  float s = 0.f;
  if (i < 2 * n)
    for (int b = w; b < blocks; b += kColsumWarps) s += partials[(size_t)b * 2 * n + i];
  red[w][lane] = s;
  __syncthreads();
  if (w == 0 && i < 2 * n) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < kColsumWarps; ++k) t += red[k][lane];
    if (i < n) {
      if (dgamma) dgamma[i] += t;
    } else if (dbeta) {
      dbeta[i - n] += t;
    }
  }
}

#ifndef JH_NG_FWD_PER_SM
#define JH_NG_FWD_PER_SM 8
#endif
#ifndef JH_NG_BWD_PER_SM
#define JH_NG_BWD_PER_SM 2  // the backward's register-limited residency: one wave of blocks
#endif
static int ng_blocks(int64_t rows, int per_sm = JH_NG_BWD_PER_SM) {
  const int64_t want = (rows + kNgWarps - 1) / kNgWarps;
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sm_count_layer() * per_sm));
}

template <int CH>
static void ng_fwd_launch(int blocks, cudaStream_t s, const __nv_bfloat16* x, int64_t ld_x, const __nv_bfloat16* u,
                          int64_t ld_u, const float* g, const float* b, float eps, int64_t rows, int n,
                          __nv_bfloat16* y, int64_t ld_y, float* mean, float* rstd) {
  norm_gate_fwd_kernel<CH><<<blocks, 32 * kNgWarps, 0, s>>>(x, ld_x, u, ld_u, g, b, eps, rows, n, y, ld_y, mean,
                                                             rstd);
}

template <int CH>
static int ng_bwd_launch(int blocks, cudaStream_t s, const __nv_bfloat16* dy, int64_t ld_dy, const __nv_bfloat16* x,
                         int64_t ld_x, const __nv_bfloat16* u, int64_t ld_u, const float* g, const float* b,
                         const float* mean, const float* rstd, int64_t rows, int n, __nv_bfloat16* dx, int64_t ld_dx,
                         __nv_bfloat16* du, int64_t ld_du, float* partials) {
  // gamma / beta staging, then the partial sums (one [2n] slice per warp when it fits in 64 KB)
  const int par_epi = partials != nullptr && (size_t)kNgWarps * 2 * n * sizeof(float) <= 64 * 1024;
  const size_t smem = (size_t)(par_epi ? kNgWarps : 1) * 2 * n * sizeof(float);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(norm_gate_bwd_kernel<CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  norm_gate_bwd_kernel<CH><<<blocks, 32 * kNgWarps, smem, s>>>(dy, ld_dy, x, ld_x, u, ld_u, g, b, mean, rstd, rows, n,
                                                               dx, ld_dx, du, ld_du, partials, par_epi);
  return 0;
}

static bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace jh

using namespace jh;

extern "C" {

int jh_silu_fwd(const void* x, void* y, int64_t n, void* stream) {
  if (n < 0 || n % 8) return set_error(JH_ERR_INVALID, "silu: n must be a non-negative multiple of 8");
  if (n == 0) return JH_OK;
  if (!x || !y || !al16(x) || !al16(y)) return set_error(JH_ERR_INVALID, "silu: NULL or misaligned buffer");
  const int64_t n8 = n / 8;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n8 + 255) / 256, (int64_t)sm_count_layer() * 8));
  silu_fwd_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>((const __nv_bfloat16*)x, (__nv_bfloat16*)y, n8);
  cudaError_t e = cudaGetLastError();
  return e ? set_error(JH_ERR_CUDA, "silu_fwd: %s", cudaGetErrorString(e)) : JH_OK;
}

int jh_silu_bwd(const void* x, const void* dy, void* dx, int64_t n, void* stream) {
  if (n < 0 || n % 8) return set_error(JH_ERR_INVALID, "silu: n must be a non-negative multiple of 8");
  if (n == 0) return JH_OK;
  if (!x || !dy || !dx || !al16(x) || !al16(dy) || !al16(dx))
    return set_error(JH_ERR_INVALID, "silu: NULL or misaligned buffer");
  const int64_t n8 = n / 8;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n8 + 255) / 256, (int64_t)sm_count_layer() * 8));
  silu_bwd_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>((const __nv_bfloat16*)x, (const __nv_bfloat16*)dy,
                                                            (__nv_bfloat16*)dx, n8);
  cudaError_t e = cudaGetLastError();
  return e ? set_error(JH_ERR_CUDA, "silu_bwd: %s", cudaGetErrorString(e)) : JH_OK;
}

static int cs_blocks(int64_t rows) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(rows, (int64_t)sm_count_layer() * 4));
}

size_t jh_colsum_workspace_bytes(int64_t rows, int32_t n) {
  return (size_t)cs_blocks(std::max<int64_t>(rows, 1)) * std::max(n, 1) * sizeof(float);
}

// x == nullptr: out += column sums of dy; else dx = silu'(x) dy and out += column sums of dx
static int silu_colsum(const void* x, const void* dy, int64_t ld, void* dx, int64_t rows, int32_t n, float* out,
                       void* workspace, size_t workspace_bytes, void* stream, const char* what) {
  if (rows < 0 || n < 8 || n % 8 || n > 8 * 1024)
    return set_error(JH_ERR_UNSUPPORTED, "%s: n must be a multiple of 8 in [8, 8192] (got %d)", what, n);
  if (!dy || !out || (x && !dx)) return set_error(JH_ERR_INVALID, "%s: NULL buffer", what);
  if (!al16(dy) || (x && (!al16(x) || !al16(dx))) || ld < n || (ld * 2) % 16)
    return set_error(JH_ERR_INVALID, "%s: buffers must be 16-byte aligned with row stride >= n", what);
  if (rows == 0) return JH_OK;
  if (!workspace || workspace_bytes < jh_colsum_workspace_bytes(rows, n))
    return set_error(JH_ERR_INVALID, "%s: workspace too small", what);
  const int V = n / 8, vpt = (V + 255) / 256, R = V >= 256 ? 1 : 256 / V;
  const int blocks = cs_blocks(rows);
  const size_t smem = R > 1 ? (size_t)R * n * sizeof(float) : 0;
  cudaStream_t s = (cudaStream_t)stream;
  auto X = (const __nv_bfloat16*)x;
  auto DY = (const __nv_bfloat16*)dy;
  auto DX = (__nv_bfloat16*)dx;
  float* part = (float*)workspace;
  switch (vpt * 2 + (x ? 1 : 0)) {
#define CS(VP, SI) \
  case VP * 2 + SI: silu_colsum_kernel<VP, SI><<<blocks, 256, smem, s>>>(X, DY, ld, DX, rows, n, part); break;
    CS(1, 0) CS(1, 1) CS(2, 0) CS(2, 1) CS(3, 0) CS(3, 1) CS(4, 0) CS(4, 1)
#undef CS
  }
  // [blocks][n] partial rows = [blocks][2 (n/2)]: colsum_kernel's two halves land in out[0, n/2), out[n/2, n)
  colsum_kernel<<<(n + 31) / 32, 32 * kColsumWarps, 0, s>>>(part, blocks, n / 2, out, out + n / 2);
  cudaError_t e = cudaGetLastError();
  return e ? set_error(JH_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e)) : JH_OK;
}

int jh_silu_bwd_colsum(const void* x, const void* dy, void* dx, int64_t rows, int32_t n, float* dbias,
                       void* workspace, size_t workspace_bytes, void* stream) {
  if (!x) return set_error(JH_ERR_INVALID, "silu_bwd_colsum: x is NULL");
  return silu_colsum(x, dy, n, dx, rows, n, dbias, workspace, workspace_bytes, stream, "silu_bwd_colsum");
}

int jh_colsum(const void* x, int64_t ld, int64_t rows, int32_t n, float* out, void* workspace, size_t workspace_bytes,
              void* stream) {
  return silu_colsum(nullptr, x, ld, nullptr, rows, n, out, workspace, workspace_bytes, stream, "colsum");
}

static int ng_check(int64_t rows, int32_t n, std::initializer_list<std::pair<const void*, int64_t>> bufs) {
  if (rows < 0) return set_error(JH_ERR_INVALID, "norm_gate: rows < 0");
  if (n < 8 || n % 8 || n > kNgMaxChunks * 256)
    return set_error(JH_ERR_UNSUPPORTED, "norm_gate: n must be a multiple of 8 in [8, %d] (got %d)",
                     kNgMaxChunks * 256, n);
  for (auto& b : bufs)
    if (b.first && (!al16(b.first) || (b.second * 2) % 16 || b.second < n))
      return set_error(JH_ERR_INVALID, "norm_gate: buffers must be 16-byte aligned with row stride >= n");
  return JH_OK;
}

size_t jh_norm_gate_bwd_workspace_bytes(int64_t rows, int32_t n) {
  return (size_t)ng_blocks(std::max<int64_t>(rows, 1)) * 2 * std::max(n, 1) * sizeof(float);
}

int jh_norm_gate_fwd(const void* x, int64_t ld_x, const void* u, int64_t ld_u, const float* gamma, const float* beta,
                     float eps, int64_t rows, int32_t n, void* y, int64_t ld_y, float* mean, float* rstd,
                     void* stream) {
  if (int r = ng_check(rows, n, {{x, ld_x}, {u, ld_u}, {y, ld_y}})) return r;
  if (!x || !y) return set_error(JH_ERR_INVALID, "norm_gate: x / y is NULL");
  if (rows == 0) return JH_OK;
  const int blocks = ng_blocks(rows, JH_NG_FWD_PER_SM);
  const int ch = (n + 255) / 256;
  cudaStream_t s = (cudaStream_t)stream;
  auto X = (const __nv_bfloat16*)x;
  auto U = (const __nv_bfloat16*)u;
  auto Y = (__nv_bfloat16*)y;
  switch (ch) {
#define NG_F(C) \
  case C: ng_fwd_launch<C>(blocks, s, X, ld_x, U, ld_u, gamma, beta, eps, rows, n, Y, ld_y, mean, rstd); break;
    NG_F(1) NG_F(2) NG_F(3) NG_F(4) NG_F(5) NG_F(6) NG_F(7) NG_F(8)
#undef NG_F
  }
  cudaError_t e = cudaGetLastError();
  return e ? set_error(JH_ERR_CUDA, "norm_gate_fwd: %s", cudaGetErrorString(e)) : JH_OK;
}

int jh_norm_gate_bwd(const void* dy, int64_t ld_dy, const void* x, int64_t ld_x, const void* u, int64_t ld_u,
                     const float* gamma, const float* beta, const float* mean, const float* rstd, int64_t rows,
                     int32_t n, void* dx, int64_t ld_dx, void* du, int64_t ld_du, float* dgamma, float* dbeta,
                     void* workspace, size_t workspace_bytes, void* stream) {
  if (int r = ng_check(rows, n, {{dy, ld_dy}, {x, ld_x}, {u, ld_u}, {dx, ld_dx}, {du, ld_du}})) return r;
  if (!dy || !x || !dx || !mean || !rstd) return set_error(JH_ERR_INVALID, "norm_gate_bwd: NULL input");
  if (u && !du) return set_error(JH_ERR_INVALID, "norm_gate_bwd: du is NULL with a gate");
  if (rows == 0) return JH_OK;
  const bool affine_grads = dgamma || dbeta;
  if (affine_grads && (!workspace || workspace_bytes < jh_norm_gate_bwd_workspace_bytes(rows, n)))
    return set_error(JH_ERR_INVALID, "norm_gate_bwd: workspace too small");
  const int blocks = ng_blocks(rows);
  const int ch = (n + 255) / 256;
  cudaStream_t s = (cudaStream_t)stream;
  float* part = affine_grads ? (float*)workspace : nullptr;
  auto DY = (const __nv_bfloat16*)dy;
  auto X = (const __nv_bfloat16*)x;
  auto U = (const __nv_bfloat16*)u;
  auto DX = (__nv_bfloat16*)dx;
  auto DU = (__nv_bfloat16*)du;
  switch (ch) {
#define NG_B(C)                                                                                                   \
  case C:                                                                                                         \
    ng_bwd_launch<C>(blocks, s, DY, ld_dy, X, ld_x, U, ld_u, gamma, beta, mean, rstd, rows, n, DX, ld_dx, DU, ld_du, \
                     part);                                                                                       \
    break;
    NG_B(1) NG_B(2) NG_B(3) NG_B(4) NG_B(5) NG_B(6) NG_B(7) NG_B(8)
#undef NG_B
  }
  if (affine_grads) colsum_kernel<<<(2 * n + 31) / 32, 32 * kColsumWarps, 0, s>>>(part, blocks, n, dgamma, dbeta);
  cudaError_t e = cudaGetLastError();
  return e ? set_error(JH_ERR_CUDA, "norm_gate_bwd: %s", cudaGetErrorString(e)) : JH_OK;
}

}  // extern "C"
