// Microbenchmark: tcgen05.mma issue-to-completion throughput for the shapes the
// attention kernels use (one CTA per SM, one issuing thread, zero data).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2508_04711_b200/csrc mma_bw.cu -o mma_bw
#include <cstdio>

#include "common.cuh"

using namespace jh;

// MODE 0: SS 128x128 (K-major A/B)     1: SS 128x64        2: TS 128x128 (B MN-major)
//      3: SS 128x256                    4: SS 128x128 B MN-major (dK-style)
template <int MODE>
__global__ void __launch_bounds__(128, 1) mma_kernel(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t s_tmem;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&s_tmem, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    constexpr uint32_t N = MODE == 1 ? 64 : (MODE == 3 ? 256 : 128);
    constexpr uint32_t id = idesc_bf16(128, N, 0, (MODE == 2 || MODE == 4) ? 1 : 0);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        if (MODE == 2)
          umma_ts(tmem + 256, tmem + 8 * kk, sdesc_sw128(b + kk * 2048, 16384, 1024), id, 1u);
        else if (MODE == 4)
          umma_ss(tmem, sdesc_sw128(a + kk * 32, 16, 1024), sdesc_sw128(b + kk * 2048, 16384, 1024), id, 1u);
        else
          umma_ss(tmem, sdesc_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                  sdesc_sw128(b + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024), id, 1u);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int MODE>
void run(const char* name, unsigned long long* d_out) {
  const int iters = 1000;
  cudaFuncSetAttribute(mma_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  mma_kernel<MODE><<<148, 128, 65536>>>(d_out, iters);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long cyc[148];
  cudaMemcpy(cyc, d_out, sizeof(cyc), cudaMemcpyDeviceToHost);
  double m = 0;
  for (int i = 0; i < 148; ++i) m += cyc[i];
  m /= 148;
  const double N = MODE == 1 ? 64 : (MODE == 3 ? 256 : 128);
  const double flops = 2.0 * 128 * N * 16 * 8 * iters;
  printf("%-22s cycles/MMA=%.1f  flops/clk/SM=%.0f  (%s)\n", name, m / (8.0 * iters), flops / m, cudaGetErrorString(e));
}

int main() {
  unsigned long long* d_out;
  cudaMalloc(&d_out, 148 * 8);
  run<0>("SS 128x128x16", d_out);
  run<1>("SS 128x64x16", d_out);
  run<2>("TS 128x128x16 Bmn", d_out);
  run<3>("SS 128x256x16", d_out);
  run<4>("SS 128x128x16 Bmn", d_out);
  return 0;
}
