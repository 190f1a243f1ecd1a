// Microbenchmark of the dK/dV "general chunk" epilogue loop in isolation:
// cycles per 32-column chunk per warp for variants of the loop.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2508_04711_b200/csrc gen_bench.cu -o gen_bench
#include <cstdio>

#include "bias.cuh"

using namespace jh;

// V: 0 full general loop (TMEM ld8 / lookups / local SiLU' / TMEM st4)
//    1 no lookups   2 no TMEM loads (registers)   3 no TMEM stores   4 saturated path (ld32 + st16)
//    5 general loop, 16 columns per step
template <int V>
__global__ void __launch_bounds__(256, 1) gen_kernel(unsigned long long* out, int iters, float* sink) {
  __shared__ uint32_t s_tmem;
  __shared__ int64_t s_tsq[64];
  __shared__ OctEntry s_oct[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc(&s_tmem, 512);
  if (threadIdx.x < 64) s_tsq[threadIdx.x] = 1000000ll + threadIdx.x * 37;
  if (threadIdx.x < 32) {
    OctEntry e;
    e.thr = (1u << threadIdx.x) + 3u;
    e.base = threadIdx.x / 2;
    e.wlo = 0.01f * threadIdx.x;
    e.whi = 0.011f * threadIdx.x;
    s_oct[threadIdx.x] = e;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  const uint32_t cbase = tmem + lane_off + 64 * (warp >> 2);
  {
    uint32_t z[16];
    for (int i = 0; i < 16; ++i) z[i] = __float_as_uint(0.1f * (lane + i));
    tmem_st16(cbase, z);
    tmem_st16(cbase + 16, z);
    tmem_st_wait();
  }
  const int64_t tk = 1000000ll + lane * 37 - 5;
  const int64_t cap = 3269017;
  const float c1 = 0.0442f, cb = 0.001f;
  const int rel0 = lane - 3, ncol = 32;
  uint32_t kl[16], bl[8], okm = 0;
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (V == 4) {
      uint32_t v[32], pk[16];
      tmem_ld32(cbase, v);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        const float h0 = fmaf(__uint_as_float(v[i]), c1, cb), h1 = fmaf(__uint_as_float(v[i + 1]), c1, cb);
        const float a = tanh_approx(h0), b = tanh_approx(h1);
        pk[i >> 1] = pack_bf16(fmaf(h0, a, h0), fmaf(h1, b, h1));
        __half2 hk = __floats2half2_rn((1.f + a) * (fmaf(-h0, a, h0) + 1.f), (1.f + b) * (fmaf(-h1, b, h1) + 1.f));
        kl[i >> 1] = *reinterpret_cast<uint32_t*>(&hk);
      }
      tmem_st16(cbase, pk);
      tmem_st_wait();
      continue;
    }
    constexpr int G = V == 5 ? 16 : 8;
#pragma unroll 1
    for (int g8 = 0; g8 < 32; g8 += G) {
      uint32_t v[G], pk[G / 2];
      if (V == 2) {
#pragma unroll
        for (int j = 0; j < G; ++j) v[j] = __float_as_uint(0.01f * (j + g8 + it));
      } else if (G == 8) {
        tmem_ld8(cbase + g8, *reinterpret_cast<uint32_t(*)[8]>(v));
      } else {
        tmem_ld16(cbase + g8, *reinterpret_cast<uint32_t(*)[16]>(v));
      }
      float bc[G];
      uint32_t bw = 0, om = 0;
#pragma unroll
      for (int j = 0; j < G; ++j) {
        int b = 0;
        if (V == 1) {
          bc[j] = cb;
        } else if (V == 6) {
          const int32_t d = (int32_t)((uint32_t)reinterpret_cast<const int32_t*>(s_tsq)[2 * (g8 + j)] - (uint32_t)tk);
          oct_lookup((uint32_t)min(max(d, 0), (int32_t)cap), s_oct, b, bc[j]);
        } else {
          oct_lookup(clamp_delta(s_tsq[g8 + j] - tk, cap), s_oct, b, bc[j]);
        }
        bw += (uint32_t)b << (j & 7);
        const bool ok = (g8 + j < ncol) && (rel0 + g8 + j >= 0);
        om |= (ok ? 1u : 0u) << j;
      }
      okm |= om << g8;
      bl[g8 >> 2] = bw;
      if (V != 2) tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < G; j += 2) {
        float pp[2], dd[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const bool ok = (om >> (j + u)) & 1u;
          const float hh = fmaf(__uint_as_float(v[j + u]), c1, bc[j + u]);
          const float th = tanh_approx(hh);
          pp[u] = ok ? fmaf(hh, th, hh) : 0.f;
          dd[u] = ok ? (1.f + th) * (fmaf(-hh, th, hh) + 1.f) : 0.f;
        }
        pk[j >> 1] = pack_bf16(pp[0], pp[1]);
        __half2 hk = __floats2half2_rn(dd[0], dd[1]);
        kl[(g8 + j) >> 1] = *reinterpret_cast<uint32_t*>(&hk);
      }
      if (V == 3) {
#pragma unroll
        for (int j = 0; j < G / 2; ++j) acc += __uint_as_float(pk[j]);
      } else if (G == 8) {
        tmem_st4(cbase + (g8 >> 1), *reinterpret_cast<uint32_t(*)[4]>(pk));
      } else {
        tmem_st8(cbase + (g8 >> 1), *reinterpret_cast<uint32_t(*)[8]>(pk));
      }
    }
    tmem_st_wait();
  }
  long long t1 = clock64();
  for (int i = 0; i < 16; ++i) acc += __uint_as_float(kl[i]);
  for (int i = 0; i < 8; ++i) acc += (float)bl[i];
  acc += (float)okm;
  if (acc == 1234.5f) *sink = acc;
  if (lane == 0) out[blockIdx.x * 8 + warp] = (unsigned long long)(t1 - t0);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

// dS-phase general loop: V 0 = reds into global bins (as the kernel), 1 = thread-private
// shared-memory bins, 2 = no scatter
template <int V>
__global__ void __launch_bounds__(256, 1) ds_kernel(unsigned long long* out, int iters, float* gbins, float* sink) {
  __shared__ uint32_t s_tmem;
  __shared__ float s_tb[16 * 256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc(&s_tmem, 512);
  for (int i = threadIdx.x; i < 16 * 256; i += blockDim.x) s_tb[i] = 0.f;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  const uint32_t dpbase = tmem + lane_off + 64 * (warp >> 2);
  const uint32_t cbase = dpbase + 256;
  {
    uint32_t z[16];
    for (int i = 0; i < 16; ++i) z[i] = __float_as_uint(0.1f * (lane + i));
    tmem_st16(dpbase, z);
    tmem_st16(dpbase + 16, z);
    tmem_st_wait();
  }
  uint32_t kl[16], bl[8];
  for (int i = 0; i < 16; ++i) kl[i] = 0x3c003c00u + lane;
  for (int i = 0; i < 8; ++i) bl[i] = (i == 0) ? 0x0f030201u + (lane & 1) : 0x0f0f0f0fu;
  const uint32_t okm = 0xFFFFFFFFu << (lane & 7);
  const float c1 = 0.0442f;
  float* g_bins = gbins + blockIdx.x * 256;
  float* my_tb = s_tb + (threadIdx.x & 255);
  const int nb = 16;
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t rb = nb - 1;
    float rs = 0.f;
#pragma unroll 1
    for (int g8 = 0; g8 < 32; g8 += 8) {
      uint32_t dv[8], dk[4];
      tmem_ld8(dpbase + g8, dv);
      const uint32_t bw0 = bl[g8 >> 2], bw1 = bl[(g8 >> 2) + 1];
      uint32_t kw[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) kw[j] = kl[(g8 >> 1) + j];
      tmem_ld_wait();
      float dd[8];
#pragma unroll
      for (int j = 0; j < 8; j += 2) {
        const float2 kd = __half22float2(*reinterpret_cast<const __half2*>(&kw[j >> 1]));
        dd[j] = __uint_as_float(dv[j]) * kd.x * c1;
        dd[j + 1] = __uint_as_float(dv[j + 1]) * kd.y * c1;
        dk[j >> 1] = pack_bf16(dd[j], dd[j + 1]);
      }
      tmem_st4(cbase + (g8 >> 1), dk);
      if (V == 4) {
        uint32_t msk = 0;
        uint32_t bj[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const bool ok = (okm >> (g8 + j)) & 1u;
          bj[j] = ok ? (((j < 4 ? bw0 : bw1) >> (8 * (j & 3))) & 0xFFu) : 31u;
          msk |= 1u << bj[j];
          rs += (bj[j] == (uint32_t)(nb - 1)) ? dd[j] : 0.f;
        }
        msk &= ~((1u << (nb - 1)) | 0x80000000u);
        for (uint32_t m = __reduce_or_sync(0xffffffffu, msk); m; m &= m - 1) {
          const uint32_t k = __ffs(m) - 1;
          float sk = 0.f;
#pragma unroll
          for (int j = 0; j < 8; ++j) sk += bj[j] == k ? dd[j] : 0.f;
          my_tb[k * 256] += sk;
        }
      } else if (V == 3) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const bool ok = (okm >> (g8 + j)) & 1u;
          const uint32_t b = ((j < 4 ? bw0 : bw1) >> (8 * (j & 3))) & 0xFFu;
          const bool last = b == (uint32_t)(nb - 1);
          rs += (ok && last) ? dd[j] : 0.f;
          if (ok && !last) my_tb[b * 256] += dd[j];
        }
      } else if (V != 2) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const bool ok = (okm >> (g8 + j)) & 1u;
          const uint32_t b = ((j < 4 ? bw0 : bw1) >> (8 * (j & 3))) & 0xFFu;
          const bool ch = ok && b != rb;
          if (V == 0)
            red_add_f32_if(g_bins + rb, rs, ch && rs != 0.f);
          else if (ch && rs != 0.f)
            my_tb[rb * 256] += rs;
          rb = ch ? b : rb;
          rs = ch ? dd[j] : rs + dd[j];
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) acc += dd[j];
      }
    }
    acc += rs;
    tmem_st_wait();
  }
  long long t1 = clock64();
  if (acc == 1234.5f) *sink = acc + my_tb[0];
  if (lane == 0) out[blockIdx.x * 8 + warp] = (unsigned long long)(t1 - t0);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int V>
void run_ds(const char* name, int warps, unsigned long long* d_out, float* gb, float* sink) {
  const int iters = 2000;
  ds_kernel<V><<<148, warps * 32>>>(d_out, iters, gb, sink);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long c[148 * 8];
  cudaMemcpy(c, d_out, sizeof(c), cudaMemcpyDeviceToHost);
  double m = 0;
  int n = 0;
  for (int b = 0; b < 148; ++b)
    for (int w = 0; w < warps; ++w) m += c[b * 8 + w], ++n;
  printf("%-34s warps=%d  cycles per chunk per warp = %.0f  (%s)\n", name, warps, m / n / iters,
         cudaGetErrorString(e));
}

template <int V>
void run(const char* name, int warps, unsigned long long* d_out, float* sink) {
  const int iters = 2000;
  gen_kernel<V><<<148, warps * 32>>>(d_out, iters, sink);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long c[148 * 8];
  cudaMemcpy(c, d_out, sizeof(c), cudaMemcpyDeviceToHost);
  double m = 0;
  int n = 0;
  for (int b = 0; b < 148; ++b)
    for (int w = 0; w < warps; ++w) m += c[b * 8 + w], ++n;
  printf("%-34s warps=%d  cycles per chunk per warp = %.0f  (%s)\n", name, warps, m / n / iters,
         cudaGetErrorString(e));
}

int main() {
  unsigned long long* d_out;
  float* sink;
  cudaMalloc(&d_out, 148 * 8 * 8);
  cudaMalloc(&sink, 4);
  float* gb;
  cudaMalloc(&gb, 148 * 256 * 4);
  cudaMemset(gb, 0, 148 * 256 * 4);
  for (int w : {4, 8}) {
    run_ds<0>("dS general, global reds", w, d_out, gb, sink);
    run_ds<1>("dS general, private smem bins", w, d_out, gb, sink);
    run_ds<2>("dS general, no scatter", w, d_out, gb, sink);
    run_ds<3>("dS general, last-bucket sum + smem", w, d_out, gb, sink);
    run_ds<4>("dS general, per-bucket warp passes", w, d_out, gb, sink);
  }
  for (int w : {4, 8}) {
    run<0>("general (ld8/lookup/st4)", w, d_out, sink);
    run<1>("general, no lookups", w, d_out, sink);
    run<2>("general, no TMEM loads", w, d_out, sink);
    run<3>("general, no TMEM stores", w, d_out, sink);
    run<5>("general, 16 columns per step", w, d_out, sink);
    run<6>("general, 32-bit deltas", w, d_out, sink);
    run<4>("saturated (ld32/st16)", w, d_out, sink);
  }
  return 0;
}
