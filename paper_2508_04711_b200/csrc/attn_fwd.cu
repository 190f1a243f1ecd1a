// Fused jagged HSTU attention forward for sm_100a.
//
//   out = (tril . SiLU((Q K^T + bias) / sqrt(d))) V     per segment, per head
//   (reference: attention.py:125-148 hstu_attention_reference, and the
//    blockwise form attention.py:151-184 used by the CP ring)
//
// Persistent, warp-specialised kernel, one CTA per SM (grid = #SMs), work
// items (segment, 128-row q tile) x head from the device-built list.
//   warp 0      TMA producer: Q tile (double buffered), K/V tiles (NS stages)
//   warp 1      MMA issuer (one lane): S = Q K^T -> TMEM (2 buffers),
//               O += P V with P read from TMEM (tcgen05 .kind::f16, A in TMEM)
//   warp 2      TMEM allocator (512 columns)
//   warps 4..7  epilogue: thread = q row.  S row -> (+bias, *scale, SiLU via
//               one tanh.approx, causal/jagged mask) -> bf16 P -> TMEM;
//               final O -> bf16 -> global.
// TMEM columns: S0 [0,128) S1 [128,256) O [256,256+D) P0 [384,448) P1 [448,512)
// There is no softmax normaliser: SiLU partials are additive, so O simply
// accumulates in TMEM across kv tiles (no rescale).
#include "attn_common.cuh"

namespace jh {

template <int D>
struct FwdCfg {
  static constexpr int NS = (D == 64) ? 4 : 2;          // kv stages
  static constexpr int PANELS = D / 64;                 // 64-col swizzle panels
  static constexpr int TILE_BYTES = 128 * D * 2;        // one 128-row operand tile
  static constexpr int Q_OFF = 0;
  static constexpr int K_OFF = 2 * TILE_BYTES;
  static constexpr int V_OFF = K_OFF + NS * TILE_BYTES;
  static constexpr int TS_OFF = V_OFF + NS * TILE_BYTES;  // int64 tsk[2][128]
  static constexpr int KMAX_OFF = TS_OFF + 2 * 128 * 8;   // int64 kmax[2][4]
  static constexpr int W_OFF = KMAX_OFF + 2 * 4 * 8;      // float w[256]
  static constexpr int PW_OFF = W_OFF + 256 * 4;          // float pw[<=1024]
  static constexpr int THR_OFF = PW_OFF + 1024 * 4;       // int64 thr[64]
  static constexpr int BASE_OFF = THR_OFF + 64 * 8;       // int32 base[64]
  static constexpr int BAR_OFF = BASE_OFF + 64 * 4;       // mbarriers
  static constexpr int NBARS = 2 + 2 + 3 * NS + 2 + 2 + 2 + 2;
  static constexpr int TMEMPTR_OFF = BAR_OFF + NBARS * 8;
  static constexpr int SMEM = TMEMPTR_OFF + 16 + 1024;  // + alignment slack
};

template <int D>
__global__ void __launch_bounds__(256, 1)
    hstu_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ AttnParams p) {
  using C = FwdCfg<D>;
  constexpr int NS = C::NS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  int64_t* s_tsk = reinterpret_cast<int64_t*>(smem + C::TS_OFF);
  int64_t* s_kmax = reinterpret_cast<int64_t*>(smem + C::KMAX_OFF);
  float* s_w = reinterpret_cast<float*>(smem + C::W_OFF);
  float* s_pw = reinterpret_cast<float*>(smem + C::PW_OFF);
  int64_t* s_thr = reinterpret_cast<int64_t*>(smem + C::THR_OFF);
  int32_t* s_base = reinterpret_cast<int32_t*>(smem + C::BASE_OFF);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* q_full = bars;             // [2]
  uint64_t* q_empty = bars + 2;        // [2]
  uint64_t* k_full = bars + 4;         // [NS]
  uint64_t* v_full = k_full + NS;      // [NS]
  uint64_t* kv_empty = v_full + NS;    // [NS]
  uint64_t* s_full = kv_empty + NS;    // [2]
  uint64_t* p_full = s_full + 2;       // [2]
  uint64_t* p_empty = p_full + 2;      // [2]
  uint64_t* o_full = p_empty + 2;      // [1]
  uint64_t* o_empty = o_full + 1;      // [1]
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + C::TMEMPTR_OFF);

  const uint32_t warp = warp_id();
  const int tid = threadIdx.x;
  const int H = p.num_heads;
  const int nb = p.bias.nb;

  // ---- one-time setup
  for (int i = tid; i < 64; i += blockDim.x) {
    s_thr[i] = p.bias.thr[i];
    s_base[i] = p.bias.base[i];
  }
  for (int i = tid; i < nb; i += blockDim.x) s_w[i] = p.ts_weights[i];
  for (int i = tid; i < p.num_pos; i += blockDim.x) s_pw[i] = p.pos_weights[i];
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 128);
      mbar_init(&p_empty[i], 1);
    }
    for (int i = 0; i < NS; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    mbar_init(o_full, 1);
    mbar_init(o_empty, 128);
    fence_barrier_init();
  }
  if (warp == 0 && lane_id() == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
  }
  if (warp == 2) tmem_alloc(s_tmem, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  const int n_items = p.wl.hdr->n_fwd;
  const int total = n_items * H;

  if (warp == 0) {
    // ================= TMA producer
    if (elect_one()) {
      uint32_t q_it = 0, kv_it = 0;
      for (int g = blockIdx.x; g < total; g += gridDim.x) {
        const int2 it = p.wl.fwd[g / H];
        const int h = g % H;
        const Seg sg = load_seg(p.seg, it.x);
        const int64_t kv_lim = fwd_kv_lim(sg, it.y);
        const int n = (int)((kv_lim + kBN - 1) / kBN);
        if (n == 0) continue;
        const int qb = q_it & 1;
        mbar_wait(&q_empty[qb], ((q_it >> 1) & 1) ^ 1);
        mbar_expect_tx(&q_full[qb], C::TILE_BYTES);
        const int32_t qrow = (int32_t)(sg.q_row0 + (int64_t)it.y * kBM);
        for (int pnl = 0; pnl < C::PANELS; ++pnl)
          tma_load_2d(smem + C::Q_OFF + qb * C::TILE_BYTES + pnl * 16384, &tm_q, h * D + pnl * 64, qrow,
                      &q_full[qb]);
        ++q_it;
        for (int j = 0; j < n; ++j) {
          const int st = kv_it % NS;
          mbar_wait(&kv_empty[st], ((kv_it / NS) & 1) ^ 1);
          const int32_t krow = (int32_t)(sg.kv_row0 + (int64_t)j * kBN);
          mbar_expect_tx(&k_full[st], C::TILE_BYTES);
          for (int pnl = 0; pnl < C::PANELS; ++pnl)
            tma_load_2d(smem + C::K_OFF + st * C::TILE_BYTES + pnl * 16384, &tm_k, h * D + pnl * 64, krow,
                        &k_full[st]);
          mbar_expect_tx(&v_full[st], C::TILE_BYTES);
          for (int pnl = 0; pnl < C::PANELS; ++pnl)
            tma_load_2d(smem + C::V_OFF + st * C::TILE_BYTES + pnl * 16384, &tm_v, h * D + pnl * 64, krow,
                        &v_full[st]);
          ++kv_it;
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc_s = idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t idesc_pv = idesc_bf16(128, D, 0, 1);
      const uint32_t tO = tmem + 256;
      uint32_t q_it = 0, kv_it = 0, s_it = 0, o_it = 0;
      for (int g = blockIdx.x; g < total; g += gridDim.x) {
        const int2 it = p.wl.fwd[g / H];
        const Seg sg = load_seg(p.seg, it.x);
        const int64_t kv_lim = fwd_kv_lim(sg, it.y);
        const int n = (int)((kv_lim + kBN - 1) / kBN);
        if (n == 0) continue;
        const int qb = q_it & 1;
        mbar_wait(&q_full[qb], (q_it >> 1) & 1);
        tc_fence_after();
        const uint32_t q_base = smem_u32(smem + C::Q_OFF + qb * C::TILE_BYTES);
        auto issue_pv = [&](uint32_t sit, uint32_t kvit, bool first) {
          const int pb = sit & 1;
          const int st = kvit % NS;
          mbar_wait(&p_full[pb], (sit >> 1) & 1);
          mbar_wait(&v_full[st], (kvit / NS) & 1);
          if (first) mbar_wait(o_empty, (o_it & 1) ^ 1);
          tc_fence_after();
          const uint32_t v_base = smem_u32(smem + C::V_OFF + st * C::TILE_BYTES);
          const uint32_t tP = tmem + 384 + 64 * pb;
#pragma unroll
          for (int kk = 0; kk < kBN / 16; ++kk)
            umma_ts(tO, tP + kk * 8, sdesc_sw128(v_base + kk * 2048, 16384, 1024), idesc_pv,
                    (first && kk == 0) ? 0u : 1u);
          umma_commit(&kv_empty[st]);
          umma_commit(&p_empty[pb]);
        };
        for (int j = 0; j < n; ++j) {
          const int st = kv_it % NS;
          const int sb = s_it & 1;
          mbar_wait(&k_full[st], (kv_it / NS) & 1);
          tc_fence_after();
          const uint32_t k_base = smem_u32(smem + C::K_OFF + st * C::TILE_BYTES);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
            umma_ss(tmem + 128 * sb, sdesc_sw128(q_base + off, 16, 1024), sdesc_sw128(k_base + off, 16, 1024),
                    idesc_s, kk > 0 ? 1u : 0u);
          }
          umma_commit(&s_full[sb]);
          if (j == n - 1) umma_commit(&q_empty[qb]);
          if (j > 0) issue_pv(s_it - 1, kv_it - 1, j == 1);
          ++s_it;
          ++kv_it;
        }
        issue_pv(s_it - 1, kv_it - 1, n == 1);
        umma_commit(o_full);
        ++o_it;
        ++q_it;
      }
    }
  } else if (warp >= 4) {
    // ================= epilogue (thread = q row)
    const int r = tid - 128;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const int ew = warp & 3;
    const float c1 = 0.5f * rsqrtf((float)D);  // SiLU(s) = h + h*tanh(h), h = s/2
    const int64_t cap = p.bias.cap;
    const bool has_pos = p.num_pos > 0;
    const int P = p.num_pos;
    uint32_t s_it = 0, o_it = 0;
    for (int g = blockIdx.x; g < total; g += gridDim.x) {
      const int2 it = p.wl.fwd[g / H];
      const int h = g % H;
      const Seg sg = load_seg(p.seg, it.x);
      const int64_t kv_lim = fwd_kv_lim(sg, it.y);
      const int n = (int)((kv_lim + kBN - 1) / kBN);
      const int64_t nq = min((int64_t)kBM, sg.lq - (int64_t)it.y * kBM);
      const bool row_ok = r < nq;
      const int64_t qpos = sg.qp0 + (int64_t)it.y * kBM + r;
      const int64_t qp_min = sg.qp0 + (int64_t)it.y * kBM;
      const int64_t qrow = sg.q_row0 + (int64_t)it.y * kBM + r;
      __nv_bfloat16* orow = p.out + qrow * p.ld_o + h * D;
      if (n == 0) {
        if (row_ok)
          for (int c = 0; c < D; c += 8) *reinterpret_cast<int4*>(orow + c) = make_int4(0, 0, 0, 0);
        continue;
      }
      const int64_t tq = row_ok ? p.ts_q[qrow] : 0;
      int64_t tk_next = (r < kv_lim) ? p.ts_k[sg.kv_row0 + r] : INT64_MIN;
      for (int j = 0; j < n; ++j) {
        const int sb = s_it & 1;
        const int64_t kv0 = (int64_t)j * kBN;
        // stage this tile's key timestamps (+ tile max) in smem
        const int64_t tk_cur = tk_next;
        if (j + 1 < n) {
          const int64_t kp = kv0 + kBN + r;
          tk_next = kp < kv_lim ? p.ts_k[sg.kv_row0 + kp] : INT64_MIN;
        }
        s_tsk[sb * 128 + r] = tk_cur;
        int64_t m = tk_cur;
        for (int o = 16; o; o >>= 1) {
          int64_t y = __shfl_xor_sync(0xffffffffu, m, o);
          m = y > m ? y : m;
        }
        if ((r & 31) == 0) s_kmax[sb * 4 + ew] = m;
        named_bar_sync(1, 128);
        int64_t kmax = s_kmax[sb * 4];
        for (int e = 1; e < 4; ++e) kmax = s_kmax[sb * 4 + e] > kmax ? s_kmax[sb * 4 + e] : kmax;
        const bool full = (kv0 + kBN - 1 <= qp_min) && (kv0 + kBN <= kv_lim);
        bool sat = full && (!has_pos || qp_min - (kv0 + kBN - 1) >= P - 1);
        sat = __all_sync(0xffffffffu, sat && (!row_ok || tq - kmax >= cap));
        float cb = s_w[nb - 1];
        if (has_pos) cb += s_pw[P - 1];
        cb *= c1;

        mbar_wait(&s_full[sb], (s_it >> 1) & 1);
        mbar_wait(&p_empty[sb], ((s_it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t tS = tmem + 128 * sb + lane_off;
        const uint32_t tP = tmem + 384 + 64 * sb + lane_off;
#pragma unroll 1
        for (int c0 = 0; c0 < kBN; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(tS + c0, v);
          tmem_ld_wait();
          uint32_t pk[16];
          if (sat) {
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              const float h0 = fmaf(__uint_as_float(v[i]), c1, cb);
              const float h1 = fmaf(__uint_as_float(v[i + 1]), c1, cb);
              pk[i >> 1] = pack_bf16(fmaf(h0, tanh_approx(h0), h0), fmaf(h1, tanh_approx(h1), h1));
            }
          } else {
            float pv[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const int64_t kpos = kv0 + c0 + i;
              const int64_t tk = s_tsk[sb * 128 + c0 + i];
              float bias = s_w[bucket_of(tq - tk, s_thr, s_base, cap)];
              if (has_pos) {
                int64_t rel = qpos - kpos;
                rel = rel < 0 ? 0 : (rel > P - 1 ? P - 1 : rel);
                bias += s_pw[rel];
              }
              const float hh = (__uint_as_float(v[i]) + bias) * c1;
              const float y = fmaf(hh, tanh_approx(hh), hh);
              pv[i] = (kpos <= qpos && kpos < kv_lim) ? y : 0.f;
            }
#pragma unroll
            for (int i = 0; i < 32; i += 2) pk[i >> 1] = pack_bf16(pv[i], pv[i + 1]);
          }
          tmem_st16(tP + (c0 >> 1), pk);
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&p_full[sb]);
        ++s_it;
      }
      // ---- O: TMEM -> bf16 -> global
      mbar_wait(o_full, o_it & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c0 = 0; c0 < D; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + 256 + lane_off + c0, v);
        tmem_ld_wait();
        if (row_ok) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 32; i += 2) pk[i >> 1] = pack_bf16(__uint_as_float(v[i]), __uint_as_float(v[i + 1]));
          int4* dst = reinterpret_cast<int4*>(orow + c0);
#pragma unroll
          for (int i = 0; i < 4; ++i) dst[i] = make_int4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
        }
      }
      tc_fence_before();
      mbar_arrive(o_empty);
      ++o_it;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

template <int D>
int launch_fwd(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, const AttnParams& p, int grid,
               cudaStream_t s) {
  using C = FwdCfg<D>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(hstu_fwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr = true;
  }
  hstu_fwd_kernel<D><<<grid, 256, C::SMEM, s>>>(tq, tk, tv, p);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

template int launch_fwd<64>(const CUtensorMap&, const CUtensorMap&, const CUtensorMap&, const AttnParams&, int,
                            cudaStream_t);
template int launch_fwd<128>(const CUtensorMap&, const CUtensorMap&, const CUtensorMap&, const AttnParams&, int,
                             cudaStream_t);

}  // namespace jh
