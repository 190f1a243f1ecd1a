// Microbenchmark: TMEM read / write bandwidth per SM with 4..16 warps
// (tcgen05.ld/st 32x32b) and with MUFU.TANH work interleaved.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2508_04711_b200/csrc tmem_bw.cu -o tmem_bw
#include <cstdio>

#include "common.cuh"

using namespace jh;

template <int MODE>
__global__ void bw_kernel(unsigned long long* out, int iters, float* sink) {
  __shared__ uint32_t s_tmem;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&s_tmem, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  const int nw = blockDim.x >> 5;
  // each warp owns a column slice of its lane quadrant
  const int groups = nw / 4;
  const uint32_t cols = 512 / groups;
  const uint32_t c0 = (warp >> 2) * cols;
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (uint32_t c = 0; c < cols; c += 32) {
      uint32_t v[32];
      if (MODE == 0 || MODE == 2) {
        tmem_ld32(tmem + lane_off + c0 + c, v);
        tmem_ld_wait();
        if (MODE == 2) {
#pragma unroll
          for (int i = 0; i < 32; ++i) acc += tanh_approx(__uint_as_float(v[i]));
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) acc += __uint_as_float(v[i]);
        }
      } else if (MODE == 1) {
        uint32_t w[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) w[i] = __float_as_uint(acc + i);
        tmem_st16(tmem + lane_off + c0 + c, w);
        tmem_st16(tmem + lane_off + c0 + c + 16, w);
        tmem_st_wait();
        acc += 1.f;
      } else if (MODE == 3) {
#pragma unroll
        for (int i = 0; i < 32; ++i) acc += tanh_approx((float)(c + i + it) * 1e-3f);
      } else {
#pragma unroll 1
        for (int g = 0; g < 32; g += 8) {
          uint32_t u[8];
          tmem_ld8(tmem + lane_off + c0 + c + g, u);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 8; ++i) acc += __uint_as_float(u[i]);
        }
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  if (acc == 12345.f) *sink = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int MODE>
void run(const char* name, int warps, unsigned long long* d_out, float* sink) {
  const int iters = 200;
  bw_kernel<MODE><<<148, warps * 32>>>(d_out, iters, sink);
  cudaDeviceSynchronize();
  unsigned long long cyc[148];
  cudaMemcpy(cyc, d_out, sizeof(cyc), cudaMemcpyDeviceToHost);
  double m = 0;
  for (int i = 0; i < 148; ++i) m += cyc[i];
  m /= 148;
  const double bytes = (double)iters * 128 * 512 * 4;  // whole TMEM per iteration
  printf("%-10s warps=%2d cycles=%.0f  bytes/clk/SM=%.1f  (elements/clk/SM=%.1f)\n", name, warps, m, bytes / m,
         bytes / 4 / m);
}

int main() {
  unsigned long long* d_out;
  float* sink;
  cudaMalloc(&d_out, 148 * 8);
  cudaMalloc(&sink, 4);
  for (int w : {4, 8, 16}) {
    run<0>("ld", w, d_out, sink);
    run<1>("st", w, d_out, sink);
    run<2>("ld+tanh", w, d_out, sink);
    run<3>("tanh", w, d_out, sink);
    run<4>("ld8", w, d_out, sink);
  }
  cudaError_t e = cudaGetLastError();
  printf("err=%s\n", cudaGetErrorString(e));
  return 0;
}
