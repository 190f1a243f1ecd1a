// Microbenchmark: the dK/dV kernel's per-half MMA mix issued back to back by
// one thread -- S^T, dP^T (SS 128x64x16 x 8 each), dV, dK (TS 128x128x16 x 4
// each) -- with and without a concurrent bulk-copy stream writing 32 KB of
// shared memory per half (the Q / dO half tiles).  Cycles per half.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2508_04711_b200/csrc mma_mix.cu -o mma_mix
#include <cstdio>

#include "common.cuh"

using namespace jh;

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// MODE bit0: MMA mix on; bit1: copy stream on; bit2: SS only (no TS); bit3: N=128 S/dP instead of 2x N=64
template <int MODE>
__global__ void __launch_bounds__(128, 1) k(unsigned long long* out, int iters, const uint8_t* gsrc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, cbar[2];
  __shared__ uint32_t s_tmem;
  __shared__ volatile int s_stop;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 196608 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    s_stop = 0;
    mbar_init(&bar, 1);
    mbar_init(&cbar[0], 1);
    mbar_init(&cbar[1], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&s_tmem, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  if (threadIdx.x == 0) {
    // operands: K [0,32K) V [32K,64K) Q half [64K,80K) dO half [80K,96K)
    const uint32_t kb = smem_u32(smem), vb = kb + 32768, qb = kb + 65536, db = kb + 81920;
    constexpr uint32_t id_s = idesc_bf16(128, (MODE & 8) ? 128 : 64, 0, 0);
    constexpr uint32_t id_kv = idesc_bf16(128, 128, 0, 1);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (MODE & 1) {
        const uint32_t x = it & 1;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_ss(tmem + 64 * x, sdesc_sw128(kb + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                  sdesc_sw128(qb + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024), id_s, kk > 0);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_ss(tmem + 128 + 64 * x, sdesc_sw128(vb + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                  sdesc_sw128(db + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024), id_s, kk > 0);
        if (!(MODE & 4)) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_ts(tmem + 256, tmem + 64 * x + 32 * (kk >> 1) + 8 * (kk & 1), sdesc_sw128(db + kk * 2048, 8192, 1024),
                    id_kv, 1u);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_ts(tmem + 384, tmem + 128 + 64 * x + 32 * (kk >> 1) + 8 * (kk & 1),
                    sdesc_sw128(qb + kk * 2048, 8192, 1024), id_kv, 1u);
        }
        if ((it & 7) == 7) {  // keep at most ~8 halves in flight
          umma_commit(&bar);
          mbar_wait(&bar, (uint32_t)((it >> 3) & 1));
        }
      }
    }
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
    s_stop = 1;
  } else if (threadIdx.x == 32 && (MODE & 2)) {
    // copy stream: 32 KB per half into [96K, 192K) (3 buffers), from global (L2-resident)
    uint32_t n = 0;
    while (!s_stop) {
      const int b = n % 2;
      if (n >= 2) mbar_wait(&cbar[b], ((n - 2) / 2) & 1);
      mbar_expect_tx(&cbar[b], 32768);
      bulk_g2s(smem + 98304 + b * 32768, gsrc + (size_t)(blockIdx.x % 16) * 32768, 32768, &cbar[b]);
      ++n;
    }
    // drain
    for (uint32_t m = (n >= 2 ? n - 2 : 0); m < n; ++m) mbar_wait(&cbar[m % 2], (m / 2) & 1);
    out[148 + blockIdx.x] = n;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int MODE>
void run(const char* name, unsigned long long* d_out, const uint8_t* g) {
  const int iters = 2048;
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608);
  k<MODE><<<148, 128, 196608>>>(d_out, iters, g);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long c[296];
  cudaMemcpy(c, d_out, sizeof(c), cudaMemcpyDeviceToHost);
  double m = 0, n = 0;
  for (int i = 0; i < 148; ++i) m += c[i], n += c[148 + i];
  printf("%-44s cycles per half = %.0f  (copies of 32 KB per half %.2f) (%s)\n", name, m / 148 / iters,
         n / 148 / iters, cudaGetErrorString(e));
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  unsigned long long* d_out;
  uint8_t* g;
  cudaMalloc(&d_out, 296 * 8);
  cudaMemset(d_out, 0, 296 * 8);
  cudaMalloc(&g, 16 * 32768);
  cudaMemset(g, 0, 16 * 32768);
  run<1>("MMA mix (S,dP N=64; dV,dK TS)", d_out, g);
  run<3>("MMA mix + 32 KB copy per half", d_out, g);
  run<5>("S,dP only (SS N=64)", d_out, g);
  run<7>("S,dP only + copy", d_out, g);
  run<9>("MMA mix with S,dP at N=128 (per 128 q)", d_out, g);
  return 0;
}
