// Does a concurrently running tcgen05.mma stream slow down the epilogue warps'
// TMEM loads / stores and math?  8 epilogue warps (2 per SM sub-partition) run
// the dK/dV saturated P-phase loop (ld32 -> 32 x tanh/FMA -> st16) on TMEM
// columns [0, 128) while warp 8 (optional) streams MMAs into columns
// [256, 512): SS 128x128x16, or TS with A read from TMEM [128, 256).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2508_04711_b200/csrc contention_bench.cu -o contention_bench
#include <cstdio>

#include "common.cuh"

using namespace jh;

// MMA: 0 none, 1 SS 128x128, 2 TS 128x128 (A from TMEM), 3 SS 128x64
// EPI: 0 full P loop, 1 TMEM ld/st only (no math), 2 math only (no TMEM)
template <int MMA, int EPI>
__global__ void __launch_bounds__(288, 1) k(unsigned long long* out, int iters, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t s_tmem;
  __shared__ volatile int s_stop;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    s_stop = 0;
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&s_tmem, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  if (warp == 8) {
    if (MMA != 0 && lane == 0) {
      const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
      constexpr uint32_t N = MMA == 3 ? 64 : 128;
      constexpr uint32_t id = idesc_bf16(128, N, 0, MMA == 2 ? 1 : 0);
      long long n = 0;
      while (!s_stop) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          if (MMA == 2)
            umma_ts(tmem + 256, tmem + 128 + 8 * kk, sdesc_sw128(b + kk * 2048, 16384, 1024), id, 1u);
          else
            umma_ss(tmem + 256, sdesc_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                    sdesc_sw128(b + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024), id, 1u);
        }
        umma_commit(&bar);
        mbar_wait(&bar, (uint32_t)(n & 1));
        ++n;
      }
    }
  } else {
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t cbase = tmem + lane_off + 64 * (warp >> 2);
    {
      uint32_t z[16];
      for (int i = 0; i < 16; ++i) z[i] = __float_as_uint(0.1f * (lane + i));
      tmem_st16(cbase, z);
      tmem_st16(cbase + 16, z);
      tmem_st_wait();
    }
    const float c1 = 0.0442f, cb = 0.001f;
    float kd[32];
    for (int i = 0; i < 32; ++i) kd[i] = 0.f;
    float acc = 0.f;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      uint32_t v[32], pk[16];
      if (EPI == 2) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(0.01f * (i + it));
      } else {
        tmem_ld32(cbase, v);
        tmem_ld_wait();
      }
      if (EPI == 1) {
#pragma unroll
        for (int i = 0; i < 16; ++i) pk[i] = v[2 * i] ^ v[2 * i + 1];
      } else {
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float h0 = fmaf(__uint_as_float(v[i]), c1, cb), h1 = fmaf(__uint_as_float(v[i + 1]), c1, cb);
          const float t0_ = tanh_approx(h0), t1_ = tanh_approx(h1);
          const float p0 = fmaf(h0, t0_, h0), p1 = fmaf(h1, t1_, h1);
          pk[i >> 1] = pack_bf16(p0, p1);
          kd[i] += fmaf(c1, fmaf(-p0, t0_, p0) + t0_, c1);
          kd[i + 1] += fmaf(c1, fmaf(-p1, t1_, p1) + t1_, c1);
        }
      }
      if (EPI == 2) {
#pragma unroll
        for (int i = 0; i < 16; ++i) acc += __uint_as_float(pk[i]);
      } else {
        tmem_st16(cbase, pk);
        tmem_st_wait();
      }
    }
    long long t1 = clock64();
    for (int i = 0; i < 32; ++i) acc += kd[i];
    if (acc == 1234.5f) *sink = acc;
    if (lane == 0) out[blockIdx.x * 8 + warp] = (unsigned long long)(t1 - t0);
  }
  // stop the MMA warp once every epilogue warp is done
  if (warp < 8) {
    asm volatile("bar.sync 1, 256;" ::: "memory");
    if (threadIdx.x == 0) s_stop = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int MMA, int EPI>
void run(const char* name, unsigned long long* d_out, float* sink) {
  const int iters = 4000;
  cudaFuncSetAttribute(k<MMA, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  k<MMA, EPI><<<148, 288, 65536>>>(d_out, iters, sink);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long c[148 * 8];
  cudaMemcpy(c, d_out, sizeof(c), cudaMemcpyDeviceToHost);
  double m = 0;
  for (int i = 0; i < 148 * 8; ++i) m += c[i];
  printf("%-40s cycles per 32-column chunk per warp = %.0f  (%s)\n", name, m / (148 * 8) / iters,
         cudaGetErrorString(e));
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  unsigned long long* d_out;
  float* sink;
  cudaMalloc(&d_out, 148 * 8 * 8);
  cudaMalloc(&sink, 4);
  run<0, 0>("P loop, no MMA", d_out, sink);
  run<1, 0>("P loop, SS 128x128 stream", d_out, sink);
  run<2, 0>("P loop, TS 128x128 stream", d_out, sink);
  run<3, 0>("P loop, SS 128x64 stream", d_out, sink);
  run<0, 1>("TMEM ld/st only, no MMA", d_out, sink);
  run<1, 1>("TMEM ld/st only, SS stream", d_out, sink);
  run<2, 1>("TMEM ld/st only, TS stream", d_out, sink);
  run<0, 2>("math only, no MMA", d_out, sink);
  run<2, 2>("math only, TS stream", d_out, sink);
  return 0;
}
