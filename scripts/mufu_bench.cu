// MUFU throughput per SM sub-partition: warp-instructions per cycle for the
// transcendental variants the SiLU epilogues could use (independent chains,
// 8 per thread, 1..4 warps per sub-partition).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 mufu_bench.cu -o mufu_bench
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>

template <int V>
__device__ __forceinline__ uint32_t op(uint32_t x) {
  uint32_t y;
  if (V == 0) asm volatile("tanh.approx.f32 %0, %1;" : "=r"(y) : "r"(x));
  if (V == 1) asm volatile("tanh.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
  if (V == 2) asm volatile("tanh.approx.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
  if (V == 3) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=r"(y) : "r"(x));
  if (V == 4) asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
  if (V == 5) asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
  if (V == 6) asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

template <int V>
__global__ void k(unsigned long long* out, int iters, uint32_t* sink) {
  uint32_t a[8];
  for (int i = 0; i < 8; ++i) a[i] = 0x3c003c00u + threadIdx.x + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = op<V>(a[i]) ^ 0x00010001u;
  }
  long long t1 = clock64();
  uint32_t s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345) *sink = s;
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

template <int V>
void run(const char* name, unsigned long long* d, uint32_t* sink) {
  for (int w : {4, 8, 16}) {
    const int iters = 4096;
    k<V><<<148, 32 * w>>>(d, iters, sink);
    cudaDeviceSynchronize();
    unsigned long long c[148];
    cudaMemcpy(c, d, sizeof(c), cudaMemcpyDeviceToHost);
    double m = 0;
    for (int b = 0; b < 148; ++b) m += c[b];
    m /= 148;
    // warp-instructions per SMSP = w/4 warps x 8 x iters
    printf("%-22s warps/SMSP=%d  cycles per warp-instr per SMSP = %.2f\n", name, w / 4, m / ((w / 4) * 8.0 * iters));
  }
}

int main() {
  unsigned long long* d;
  uint32_t* sink;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&sink, 4);
  run<0>("tanh.f32", d, sink);
  run<1>("tanh.f16x2", d, sink);
  run<2>("tanh.bf16x2", d, sink);
  run<3>("ex2.f32", d, sink);
  run<4>("ex2.f16x2", d, sink);
  run<5>("ex2.bf16x2", d, sink);
  run<6>("rcp.f32", d, sink);
  return 0;
}
