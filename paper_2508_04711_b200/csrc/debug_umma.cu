// Single-tile tcgen05 self-test: D[128x128] = A[128x128] * B[128x128] in
// bf16 -> fp32 with every operand placement the attention kernels rely on
// (TMA K-major / MN-major smem, hand-swizzled smem, A from TMEM).  Used by
// tests/test_gpu_umma.py to pin the descriptor encodings on hardware.
#include "common.cuh"
#include "tmap.h"
#include "../../include/jh_hstu.h"

namespace jh {

// a_mode: 0 TMA K-major (a=[m][k]), 1 TMA MN-major (a=[k][m]), 2 TMEM (a=[m][k]),
//         3 manual-swizzle K-major (a=[m][k]), 4 manual-swizzle MN-major (a=[k][m])
// b_mode: 0 TMA K-major (b=[n][k]), 1 TMA MN-major (b=[k][n])
__global__ void __launch_bounds__(128, 1)
    debug_umma_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                      const __nv_bfloat16* __restrict__ a, float* __restrict__ d, int a_mode, int b_mode) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;            // 2 panels x 16 KB
  uint8_t* sB = smem + 32768;    // 2 panels x 16 KB
  __shared__ uint64_t bar_load, bar_mma;
  __shared__ uint32_t tmem_base_sh;
  const uint32_t w = warp_id(), l = lane_id(), t = threadIdx.x;

  if (t == 0) {
    mbar_init(&bar_load, 1);
    mbar_init(&bar_mma, 1);
    fence_barrier_init();
  }
  if (w == 0) tmem_alloc(&tmem_base_sh, 256);
  // manual operand placement by all threads
  if (a_mode == 3 || a_mode == 4) {
    // thread t owns stored row t of `a` (128 elements)
    for (int c = 0; c < 128; ++c) {
      uint32_t p = c >> 6, cc = c & 63;
      *reinterpret_cast<__nv_bfloat16*>(sA + p * 16384 + sw128_offset(t, cc)) = a[t * 128 + c];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t tD = tmem, tA = tmem + 128;
  if (a_mode == 2) {
    // thread t = row m = t: pack A[m][0..127] into 64 columns
    uint32_t lane_base = (w * 32) << 16;
    for (int c0 = 0; c0 < 64; c0 += 16) {
      uint32_t r[16];
      for (int j = 0; j < 16; ++j) {
        int k = 2 * (c0 + j);
        r[j] = pack_bf16(__bfloat162float(a[t * 128 + k]), __bfloat162float(a[t * 128 + k + 1]));
      }
      tmem_st16(tA + lane_base + c0, r);
    }
    tmem_st_wait();
    tc_fence_before();
  }
  __syncthreads();
  tc_fence_after();

  if (w == 0) {
    if (elect_one()) {
      uint32_t bytes = 32768;
      if (a_mode == 0 || a_mode == 1) bytes += 32768;
      mbar_expect_tx(&bar_load, bytes);
      if (a_mode == 0 || a_mode == 1) {
        tma_load_2d(sA, &tm_a, 0, 0, &bar_load);
        tma_load_2d(sA + 16384, &tm_a, 64, 0, &bar_load);
      }
      tma_load_2d(sB, &tm_b, 0, 0, &bar_load);
      tma_load_2d(sB + 16384, &tm_b, 64, 0, &bar_load);
      mbar_wait(&bar_load, 0);
      tc_fence_after();
      const uint32_t a_mn = (a_mode == 1 || a_mode == 4) ? 1u : 0u;
      const uint32_t idesc = idesc_bf16(128, 128, a_mn, b_mode);
      for (int kk = 0; kk < 8; ++kk) {
        uint64_t bdesc;
        if (b_mode == 0)
          bdesc = sdesc_sw128(smem_u32(sB) + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
        else
          bdesc = sdesc_sw128(smem_u32(sB) + kk * 2048, 16384, 1024);
        if (a_mode == 2) {
          umma_ts(tD, tA + kk * 8, bdesc, idesc, kk > 0);
        } else {
          uint64_t adesc;
          if (a_mn == 0)
            adesc = sdesc_sw128(smem_u32(sA) + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
          else
            adesc = sdesc_sw128(smem_u32(sA) + kk * 2048, 16384, 1024);
          umma_ss(tD, adesc, bdesc, idesc, kk > 0);
        }
      }
      umma_commit(&bar_mma);
    }
    __syncwarp();
  }
  mbar_wait(&bar_mma, 0);
  tc_fence_after();
  const uint32_t lane_base = (w * 32) << 16;
  for (int c0 = 0; c0 < 128; c0 += 32) {
    uint32_t r[32];
    tmem_ld32(tD + lane_base + c0, r);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) d[t * 128 + c0 + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc(tmem, 256);
  (void)l;
}

}  // namespace jh

extern "C" int jh_debug_umma(const void* a, const void* b, float* d, int a_mode, int b_mode, void* stream) {
  using namespace jh;
  CUtensorMap ta, tb;
  if (make_tmap_bf16_2d(&ta, a, 128, 128, 128, 128)) return JH_ERR_CUDA;
  if (make_tmap_bf16_2d(&tb, b, 128, 128, 128, 128)) return JH_ERR_CUDA;
  const int smem = 65536 + 1024;
  cudaFuncSetAttribute(debug_umma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  debug_umma_kernel<<<1, 128, smem, (cudaStream_t)stream>>>(ta, tb, (const __nv_bfloat16*)a, d, a_mode, b_mode);
  return cudaGetLastError() == cudaSuccess ? JH_OK : JH_ERR_CUDA;
}
