// Fused jagged HSTU attention backward for sm_100a: ONE kernel, no dS scratch.
//
// Reference: attention.py:187-234 hstu_attention_backward
//   dV = A^T g;  dS = (g V^T) . SiLU'(S) / sqrt(d)  (masked)
//   dQ = dS K;  dK = dS^T Q;  d_w = bincount(bucket, dS)
// with A = tril . SiLU(S), S = (Q K^T + bias) / sqrt(d).
//
// kv-tile-major: a work item is (segment, 128-row kv tile j) x head; it loops
// over the 128-row q tiles that see tile j.  Per q tile, five tcgen05 GEMMs
// (all M = 128 kv or q rows, full-rate N = 128 / D):
//   S^T  = K Q^T     -> TMEM R1          (SS)
//   dP^T = V dO^T    -> TMEM R2          (SS)
//   dV  += P^T dO    (A = P^T in R1)     (TS)
//   dK  += dS^T Q    (A = dS^T in R1)    (TS)
//   dQ   = dS K      -> TMEM R2          (SS, A = dS^T tile in shared memory, MN-major)
// and dQ is reduced across kv tiles with fp32 red.global.add.v4 into a
// persistent zero accumulator; the CTA that delivers the last contribution of
// a (q tile, head) -- a per-tile counter -- converts it to bf16 and re-zeroes
// it.  Memory stays O(L): no dS scratch (the deterministic two-kernel path of
// attn_bwd.cu keeps one, behind jh_attn_args.deterministic).
//
// Roles (16 warps, one CTA per SM, persistent, device-built longest-first list):
//   warp 0      TMA K_j (2 buffers: the next item's K loads during this item) and
//               V_j (1 buffer, after this item's last dP^T); item-ring producer
//   warp 1      MMA issuer (one thread), per q tile:
//                 dP^T(t), dV(t), dK(t), S^T(t+1), dQ(t)
//               so the epilogue's P phase of tile t+1 overlaps dQ(t) and dP^T(t+1)
//   warp 2      TMA Q (2 stages) and dO (1 stage); TMEM allocator
//   warp 3      ts_q chunk minima / maxima (saturation test), from global memory
//   warps 4-11  epilogue, two warpgroups; thread = kv row, warpgroup g owns q
//               columns [64g, 64g+64) (two 32-column chunks):
//                 phase P : S^T -> P^T (bf16, TMEM R1 [32c, 32c+16)), SiLU' (fp32)
//                           kept half in registers, half in R1 [32c+16, 32c+32)
//                 phase dS: dP^T -> dS^T (bf16) into R1 [32c+16, 32c+32) AND the
//                           shared-memory dS^T tile (dQ's A operand); d_ts_weights
//   warps 12-15 drain: dQ(t) from R2 -> fp32 reductions (+ finalize), dK/dV per item
// TMEM: R1 [0,128) S^T / P^T / dS^T | R2 [128,256) dP^T, then dQ | dV | dK
#include "abi_internal.h"
#include "attn_common.cuh"

namespace jh {

constexpr int kFThreads = 512;
constexpr int kFComp = 8;  // epilogue warps

template <int D>
struct FusedCfg {
  static constexpr int TILE = 128 * D * 2;  // K, V, Q or dO tile (128 rows)
  static constexpr int PANELS = D / 64;     // 64-column swizzle panels
  static constexpr int K_OFF = 0;           // [2]
  static constexpr int V_OFF = 2 * TILE;
  static constexpr int Q_OFF = 3 * TILE;    // [2]
  static constexpr int DO_OFF = 5 * TILE;
  static constexpr int DS_OFF = 6 * TILE;   // dS^T: [2 panels of 64 q][128 kv rows][128 B], sw128
  static constexpr int ST_OFF = DS_OFF + 32768;  // int64 [2 stages][4 chunks][min, max]
  static constexpr int OCT_OFF = ST_OFF + 128;   // OctEntry [32]
  static constexpr int WT_OFF = OCT_OFF + 512;   // float [32] band weights x c1 (31: masked)
  static constexpr int BAR_OFF = WT_OFF + 128;
  static constexpr int NBARS = 24;
  static constexpr int TMEMPTR_OFF = BAR_OFF + NBARS * 8;
  static constexpr int FLAG_OFF = TMEMPTR_OFF + 16;  // int32 [4] broadcast flags
  static constexpr int RING_OFF = FLAG_OFF + 16;
  static constexpr int SMEM = RING_OFF + 2 * kItemRing * 8 + kItemRing * 4;
};

// q tiles [t0, t0 + n) of segment `sg` that see kv tile j: the tiles with
// kv_lim(t) > 128 j (a suffix; kv_lim is non-decreasing).  q tile t therefore
// receives exactly ceil(kv_lim(t) / 128) dQ contributions.
JH_DEV void fused_tiles(const Seg& sg, int j, int& t0, int& n) {
  const int nt = (int)((sg.lq + kBM - 1) / kBM);
  const int64_t k0 = (int64_t)j * kBN;
  if (k0 >= sg.kv_len || nt == 0) {
    t0 = 0;
    n = 0;
    return;
  }
  const int64_t f = k0 - sg.qp0;
  int t = f <= 0 ? 0 : (int)(f / kBM);
  if (t > nt) t = nt;
  while (t < nt && fwd_kv_lim(sg, t) <= k0) ++t;
  t0 = t;
  n = nt - t;
}

JH_DEV uint32_t pack_h2(float lo, float hi) {
  __half2 v = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
JH_DEV float2 unpack_h2(uint32_t u) { return __half22float2(*reinterpret_cast<const __half2*>(&u)); }

JH_DEV void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

JH_DEV void red_add_v4(float* dst, const uint32_t* v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(__uint_as_float(v[0])),
               "f"(__uint_as_float(v[1])), "f"(__uint_as_float(v[2])), "f"(__uint_as_float(v[3]))
               : "memory");
}

template <int D>
__global__ void __launch_bounds__(kFThreads, 1)
    hstu_bwd_fused_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                          const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
                          const __grid_constant__ AttnParams p, __nv_bfloat16* __restrict__ dq, int64_t ld_dq) {
  using C = FusedCfg<D>;
  extern __shared__ __align__(1024) uint8_t smem[];
  int64_t* s_st = reinterpret_cast<int64_t*>(smem + C::ST_OFF);
  OctEntry* s_oct = reinterpret_cast<OctEntry*>(smem + C::OCT_OFF);
  float* s_wt = reinterpret_cast<float*>(smem + C::WT_OFF);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* k_full = bars;        // [2]
  uint64_t* k_empty = bars + 2;   // [2] last dQ of the item done
  uint64_t* v_full = bars + 4;
  uint64_t* v_empty = bars + 5;   // last dP^T of the item done
  uint64_t* q_full = bars + 6;    // [2]
  uint64_t* q_empty = bars + 8;   // [2] dK of the tile done
  uint64_t* qx_full = bars + 10;  // [2] ts_q chunk statistics
  uint64_t* qx_empty = bars + 12; // [2]
  uint64_t* do_full = bars + 14;
  uint64_t* do_empty = bars + 15; // dV of the tile done
  uint64_t* s_full = bars + 16;
  uint64_t* p_full = bars + 17;   // P^T in R1 (S^T consumed)
  uint64_t* dp_full = bars + 18;
  uint64_t* ds_full = bars + 19;  // dS^T in R1 and shared memory (dP^T consumed)
  uint64_t* dq_full = bars + 20;
  uint64_t* dq_empty = bars + 21; // R2 drained
  uint64_t* dkv_full = bars + 22;
  uint64_t* dkv_empty = bars + 23;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + C::TMEMPTR_OFF);
  volatile int32_t* s_flag = reinterpret_cast<volatile int32_t*>(smem + C::FLAG_OFF);
  const ItemRing ring{reinterpret_cast<int32_t*>(smem + C::RING_OFF + 2 * kItemRing * 8),
                      reinterpret_cast<uint64_t*>(smem + C::RING_OFF),
                      reinterpret_cast<uint64_t*>(smem + C::RING_OFF + kItemRing * 8)};

  const uint32_t warp = warp_id();
  const int tid = threadIdx.x;
  const int H = p.num_heads;
  const int nb = p.bias.nb;
  const int P = p.num_pos;
  const bool has_pos = P > 0;
  const int64_t HD = (int64_t)H * D;
  const float c1 = p.c1;  // h = c1 (q k^T + bias) = s / 2, SiLU(s) = h (1 + tanh h)

  cta_stamp(p, 0);
  if (smem_u32(smem) & 1023) __trap();
  oct_table_fill(s_oct, p.bias, p.ts_weights, c1, tid, blockDim.x);
  if (tid < 32) s_wt[tid] = tid < nb ? p.ts_weights[tid] * c1 : (tid == (int)kBandMasked ? -1e30f : 0.f);
  float* g_bins = p.wl.bins + (size_t)blockIdx.x * kBinsPerCta;
  for (int i = tid; i < P; i += blockDim.x) g_bins[256 + i] = 0.f;
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&qx_full[i], 1);
      mbar_init(&qx_empty[i], kFComp);
    }
    mbar_init(v_full, 1);
    mbar_init(v_empty, 1);
    mbar_init(do_full, 1);
    mbar_init(do_empty, 1);
    mbar_init(s_full, 1);
    mbar_init(p_full, kFComp);
    mbar_init(dp_full, 1);
    mbar_init(ds_full, kFComp);
    mbar_init(dq_full, 1);
    mbar_init(dq_empty, 128);
    mbar_init(dkv_full, 1);
    mbar_init(dkv_empty, 128);
    ring_init(ring, 1 + 1 + 1 + kFComp + 4);  // consumers: Q/dO TMA, MMA, ts stats, epilogue, drain
    fence_barrier_init();
  }
  if (warp == 0 && lane_id() == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    tma_prefetch_desc(&tm_do);
  }
  if (warp == 2) tmem_alloc(s_tmem, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  const uint32_t tR1 = tmem, tR2 = tmem + 128, tDV = tmem + 256, tDK = tmem + 256 + D;

  // (programmatic dependent launch: everything above overlapped the work-list build)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int total = p.wl.hdr->n_bwd * H;

  if (warp == 0) {
    // ================= TMA producer: K_j (double-buffered), V_j; item ring
    if (elect_one()) {
      uint32_t ic = 0, rk = 0;
      const uint64_t pol_once = l2_policy_evict_first();  // read by this CTA only
      for (int g; (g = ring_produce(ring, rk, &p.wl.hdr->next_item[1], total)) >= 0;) {
        const int2 it = p.wl.bwd[g / H];
        const int h = g % H;
        const Seg sg = load_seg(p.seg, it.x);
        int t0, n;
        fused_tiles(sg, it.y, t0, n);
        if (n == 0) continue;
        const int kb = ic & 1;
        const int32_t krow = (int32_t)(sg.kv_row0 + (int64_t)it.y * kBN);
        mbar_wait(&k_empty[kb], ((ic >> 1) & 1) ^ 1);
        mbar_expect_tx(&k_full[kb], C::TILE);
        for (int pn = 0; pn < C::PANELS; ++pn)
          tma_load_2d(smem + C::K_OFF + kb * C::TILE + pn * 16384, &tm_k, h * D + pn * 64, krow, &k_full[kb]);
        mbar_wait(v_empty, (ic & 1) ^ 1);
        mbar_expect_tx(v_full, C::TILE);
        for (int pn = 0; pn < C::PANELS; ++pn)
          tma_load_2d_hint(smem + C::V_OFF + pn * 16384, &tm_v, h * D + pn * 64, krow, v_full, pol_once);
        ++ic;
      }
    }
  } else if (warp == 2) {
    // ================= TMA producer: Q (2 stages), dO (1 stage) per q tile
    if (elect_one()) {
      uint32_t tc = 0, rk = 0;
      for (int g; (g = ring_consume(ring, rk, false)) >= 0;) {
        const int2 it = p.wl.bwd[g / H];
        const int h = g % H;
        const Seg sg = load_seg(p.seg, it.x);
        int t0, n;
        fused_tiles(sg, it.y, t0, n);
        for (int i = 0; i < n; ++i, ++tc) {
          const int32_t qrow = (int32_t)(sg.q_row0 + (int64_t)(t0 + i) * kBM);
          const int st = tc & 1;
          mbar_wait(&q_empty[st], ((tc >> 1) & 1) ^ 1);
          mbar_expect_tx(&q_full[st], C::TILE);
          for (int pn = 0; pn < C::PANELS; ++pn)
            tma_load_2d(smem + C::Q_OFF + st * C::TILE + pn * 16384, &tm_q, h * D + pn * 64, qrow, &q_full[st]);
          mbar_wait(do_empty, (tc & 1) ^ 1);
          mbar_expect_tx(do_full, C::TILE);
          for (int pn = 0; pn < C::PANELS; ++pn)
            tma_load_2d(smem + C::DO_OFF + pn * 16384, &tm_do, h * D + pn * 64, qrow, do_full);
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer
    if (elect_one()) {
      constexpr uint32_t id_s = idesc_bf16(128, 128, 0, 0);  // S^T, dP^T: 128 kv x 128 q, K-major
      constexpr uint32_t id_kv = idesc_bf16(128, D, 0, 1);   // dV, dK: A = TMEM, B = dO / Q (MN-major)
      constexpr uint32_t id_q = idesc_bf16(128, D, 1, 1);    // dQ: A = dS (MN-major smem), B = K (MN-major)
      const uint32_t v_base = smem_u32(smem + C::V_OFF);
      const uint32_t do_base = smem_u32(smem + C::DO_OFF);
      const uint32_t ds_base = smem_u32(smem + C::DS_OFF);
      auto q_base = [&](uint32_t x) { return smem_u32(smem + C::Q_OFF + (x & 1) * C::TILE); };
      auto issue_S = [&](uint32_t x, uint32_t k_base) {
        mbar_wait(&q_full[x & 1], (x >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          umma_ss(tR1, sdesc_sw128(k_base + off, 16, 1024), sdesc_sw128(q_base(x) + off, 16, 1024), id_s,
                  kk > 0 ? 1u : 0u);
        }
        umma_commit(s_full);
      };
      uint32_t tc = 0, ic = 0, rk = 0, tcnt = 0;
      for (int g; (g = ring_consume(ring, rk, false)) >= 0;) {
        const int2 it = p.wl.bwd[g / H];
        const Seg sg = load_seg(p.seg, it.x);
        int t0, n;
        fused_tiles(sg, it.y, t0, n);
        if (n == 0) continue;
        const int kb = ic & 1;
        const uint32_t k_base = smem_u32(smem + C::K_OFF + kb * C::TILE);
        trace_ev(p, 1, tcnt, 1, g);
        mbar_wait(&k_full[kb], (ic >> 1) & 1);
        trace_ev(p, 1, tcnt, 2, n);
        issue_S(tc, k_base);
        for (int i = 0; i < n; ++i) {
          const uint32_t x = tc + i;
          // dP^T(x) -> R2 once dQ(x-1) is drained
          mbar_wait(dq_empty, (x & 1) ^ 1);
          trace_ev(p, 1, tcnt, 3, x);
          if (i == 0) mbar_wait(v_full, ic & 1);
          mbar_wait(do_full, x & 1);
          trace_ev(p, 1, tcnt, 4, x);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
            umma_ss(tR2, sdesc_sw128(v_base + off, 16, 1024), sdesc_sw128(do_base + off, 16, 1024), id_s,
                    kk > 0 ? 1u : 0u);
          }
          umma_commit(dp_full);
          if (i == n - 1) umma_commit(v_empty);
          // dV += P^T dO (P^T of chunk c at R1 [32c, 32c+16))
          mbar_wait(p_full, x & 1);
          trace_ev(p, 1, tcnt, 5, x);
          if (i == 0) mbar_wait(dkv_empty, (ic & 1) ^ 1);
          trace_ev(p, 1, tcnt, 6, x);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < kBM / 16; ++kk)
            umma_ts(tDV, tR1 + 32 * (kk >> 1) + 8 * (kk & 1), sdesc_sw128(do_base + kk * 2048, 16384, 1024), id_kv,
                    (kk > 0 || i > 0) ? 1u : 0u);
          umma_commit(do_empty);
          // dK += dS^T Q (dS^T of chunk c at R1 [32c+16, 32c+32))
          mbar_wait(ds_full, x & 1);
          trace_ev(p, 1, tcnt, 7, x);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < kBM / 16; ++kk)
            umma_ts(tDK, tR1 + 32 * (kk >> 1) + 16 + 8 * (kk & 1), sdesc_sw128(q_base(x) + kk * 2048, 16384, 1024),
                    id_kv, (kk > 0 || i > 0) ? 1u : 0u);
          umma_commit(&q_empty[x & 1]);
          // S^T(x+1) -> R1 (in issue order after dK read R1), overlapping the next P phase
          if (i + 1 < n) issue_S(x + 1, k_base);
          // dQ(x) = dS K -> R2
#pragma unroll
          for (int kk = 0; kk < kBN / 16; ++kk)
            umma_ss(tR2, sdesc_sw128(ds_base + kk * 2048, 16384, 1024), sdesc_sw128(k_base + kk * 2048, 16384, 1024),
                    id_q, kk > 0 ? 1u : 0u);
          umma_commit(dq_full);
          trace_ev(p, 1, tcnt, 8, x);
          if (i == n - 1) {
            umma_commit(&k_empty[kb]);
            umma_commit(dkv_full);
          }
        }
        tc += n;
        ++ic;
      }
    }
  } else if (warp == 3) {
    // ================= ts_q statistics per 32-column chunk (valid columns only)
    const int lane = lane_id();
    uint32_t tc = 0, rk = 0;
    for (int g; (g = ring_consume(ring, rk, true)) >= 0;) {
      const int2 it = p.wl.bwd[g / H];
      const Seg sg = load_seg(p.seg, it.x);
      int t0, n;
      fused_tiles(sg, it.y, t0, n);
      for (int i = 0; i < n; ++i, ++tc) {
        const int64_t t = t0 + i;
        const int64_t nq = min((int64_t)kBM, sg.lq - t * kBM);
        const int64_t* tsq = p.ts_q + sg.q_row0 + t * kBM;
        int64_t mn[4], mx[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const bool ok = 32 * c + lane < nq;
          const int64_t v = ok ? __ldg(tsq + 32 * c + lane) : 0;
          mn[c] = warp_min_i64(ok ? v : (INT64_MAX >> 2));
          mx[c] = warp_max_i64(ok ? v : (INT64_MIN >> 2));
        }
        const int st = tc & 1;
        mbar_wait(&qx_empty[st], ((tc >> 1) & 1) ^ 1);
        if (lane == 0) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            s_st[st * 8 + 2 * c] = mn[c];
            s_st[st * 8 + 2 * c + 1] = mx[c];
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&qx_full[st]);
      }
    }
  } else if (warp >= 4 && warp < 12) {
    // ================= epilogue: thread = kv row r, q chunks 2 wg and 2 wg + 1
    const int et = tid - 128;
    const int wg = et >> 7;
    const int r = et & 127;
    const int lane = r & 31;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const int64_t cap = p.bias.cap;
    const bool cnt_mode = p.dbg_count != 0;
    float cb = p.ts_weights[nb - 1];
    if (has_pos) cb += p.pos_weights[P - 1];
    cb *= c1;
    double acc_w = 0.0, acc_p = 0.0;  // last-bucket (saturated) partials
    const bool use_band = p.band != nullptr;
    // band / general chunks: non-last buckets go to thread-private fp32 slots (global, per CTA)
    float* tbg = p.tb_glob + (size_t)blockIdx.x * kTbBuckets * 256 + et;
    for (int b = 0; b < nb; ++b) tbg[b * 256] = 0.f;
    const uint32_t ds_smem = smem_u32(smem + C::DS_OFF);
    uint32_t tc = 0, rk = 0, tcnt = 0;
    const bool trc = et == 0;
    for (int g; (g = ring_consume(ring, rk, true)) >= 0;) {
      const int2 it = p.wl.bwd[g / H];
      const Seg sg = load_seg(p.seg, it.x);
      int t0, n;
      fused_tiles(sg, it.y, t0, n);
      if (n == 0) continue;
      const int64_t kv0 = (int64_t)it.y * kBN;
      const int64_t kpos = kv0 + r;
      const bool krow_ok = kpos < sg.kv_len;
      const int64_t tk = krow_ok ? __ldg(p.ts_k + sg.kv_row0 + kpos) : (INT64_MIN >> 2);
      const int64_t tk_max = warp_max_i64(tk);
      const int64_t tk_min = warp_min_i64(krow_ok ? tk : (INT64_MAX >> 2));
      const int32_t tk32 = (int32_t)(uint32_t)(uint64_t)tk;
      const int64_t k_lo = kv0 + (r & ~31), k_hi = k_lo + 31;  // this warp's kv positions
      const bool warp_k_ok = k_hi < sg.kv_len;
      const int64_t band_q0 = band_group(sg, it.x, 0);
      for (int i = 0; i < n; ++i, ++tc) {
        const int64_t t = t0 + i;
        const uint32_t ph = tc & 1;
        const int st = tc & 1;
        const int64_t qp_tile = sg.qp0 + t * kBM;
        const int nq = (int)min((int64_t)kBM, sg.lq - t * kBM);
        const int64_t qrow0 = sg.q_row0 + t * kBM;
        // ---- chunk classes: 0 masked, 1 saturated, 3 saturated ragged, 4 band, 2 general
        mbar_wait(&qx_full[st], (tc >> 1) & 1);
        int cls[2];
        bool f32ok[2];
        int bwi[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int c = 2 * wg + u;
          const int64_t qc0 = qp_tile + 32 * c;
          const int64_t tq_min = s_st[st * 8 + 2 * c], tq_max = s_st[st * 8 + 2 * c + 1];
          int k = 0;
          bwi[u] = -1;
          f32ok[u] = false;
          if (!(qc0 + 31 < k_lo || 32 * c >= nq || k_lo >= sg.kv_len)) {
            k = 2;
            const int aq = (int)(4 * t + c);
            const int64_t w = (k_lo >> 5) - ((sg.qp0 >> 5) + aq) + 3;
            if (qc0 >= k_hi && tq_min - tk_max >= cap && (!has_pos || qc0 - k_hi >= P - 1)) {
              k = ((32 * c + 32 <= nq) && warp_k_ok) ? 1 : 3;
            } else if (use_band && w >= 0 && w < kBandNW && k_lo <= qc0 + 31) {
              k = 4;
              bwi[u] = (int)w;
            }
            f32ok[u] = cap < 0x7FFFFFFFll && tq_max - tk_min < 0x7FFFFFFFll && tq_min - tk_max > -0x7FFFFFFFll;
          }
          cls[u] = k;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&qx_empty[st]);
        // c1 SiLU'(s) in fp32: columns 0-15 of chunk u in kr[16u ..], columns 16-31 in
        // the chunk's upper TMEM half R1 [32c+16, 32c+32) (free between the S^T read and
        // the dS^T write; phase dS reads them back)
        float kr[32];
        // ---------------- phase P: S^T -> P^T, SiLU'
        mbar_wait(s_full, ph);
        if (trc) trace_ev(p, 3, tcnt, 30, tc);
        tc_fence_after();
        if (p.dbg & 16) {  // timing experiment: no epilogue math (results are garbage)
          __syncwarp();
          if (lane == 0) mbar_arrive(p_full);
          mbar_wait(dp_full, ph);
          __syncwarp();
          if (lane == 0) mbar_arrive(ds_full);
          continue;
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int c = 2 * wg + u;
          const uint32_t cbase = tR1 + 32 * c + lane_off;
          if (cls[u] == 0) {
            uint32_t z[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) z[j] = 0u;
            tmem_st16(cbase, z);
#pragma unroll
            for (int j = 0; j < 16; ++j) kr[16 * u + j] = 0.f;
          } else if (cls[u] != 2) {
            uint32_t wd[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
            if (cls[u] == 4) {
              const uint4* src = reinterpret_cast<const uint4*>(
                  band_chunk(p.band, band_q0 + 4 * t + c, bwi[u]) + 1024 + lane * 32);
              const uint4 b0 = __ldg(src), b1 = __ldg(src + 1);
              wd[0] = b0.x, wd[1] = b0.y, wd[2] = b0.z, wd[3] = b0.w, wd[4] = b1.x, wd[5] = b1.y, wd[6] = b1.z,
              wd[7] = b1.w;
            }
            const int nv = cls[u] == 3 ? (krow_ok ? max(min(nq - 32 * c, 32), 0) : 0) : 32;
            uint32_t v[32], pk[16], kt[16];
            tmem_ld32(cbase, v);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
              float w0 = cb, w1 = cb;
              if (cls[u] == 4) {
                w0 = s_wt[__byte_perm(wd[j >> 2], 0u, 0x4440u | (j & 3))];
                w1 = s_wt[__byte_perm(wd[j >> 2], 0u, 0x4440u | ((j + 1) & 3))];
              }
              const float h0 = fmaf(__uint_as_float(v[j]), c1, w0);
              const float h1 = fmaf(__uint_as_float(v[j + 1]), c1, w1);
              const float a0 = tanh_approx(h0), a1 = tanh_approx(h1);
              float p0 = fmaf(h0, a0, h0), p1 = fmaf(h1, a1, h1);
              // c1 SiLU'(s) = c1 (1 + t + P (1 - t)); masked band pairs: h = -1e30, t = -1, P = 0, SiLU' = 0
              float k0 = fmaf(c1, fmaf(-p0, a0, p0) + a0, c1), k1 = fmaf(c1, fmaf(-p1, a1, p1) + a1, c1);
              if (j >= nv) p0 = k0 = 0.f;
              if (j + 1 >= nv) p1 = k1 = 0.f;
              pk[j >> 1] = pack_bf16(p0, p1);
              if (j < 16) {
                kr[16 * u + j] = k0;
                kr[16 * u + j + 1] = k1;
              } else {
                kt[j - 16] = __float_as_uint(k0);
                kt[j - 15] = __float_as_uint(k1);
              }
            }
            tmem_st16(cbase, pk);
            tmem_st16(cbase + 16, kt);
          } else {
            // general chunk: exact per-element bucket, positional bias and mask
            const int64_t* tsq = p.ts_q + qrow0 + 32 * c;
            const int rel0 = (int)(qp_tile + 32 * c - kpos);
            const int ncol = krow_ok ? nq - 32 * c : 0;
            uint32_t kt[16];
#pragma unroll
            for (int g8 = 0; g8 < 32; g8 += 8) {
              uint32_t v[8], pk[4];
              tmem_ld8(cbase + g8, v);
              float bc[8];
              uint32_t du[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const int64_t tq = (g8 + j < nq - 32 * c) ? __ldg(tsq + g8 + j) : 0;
                du[j] = f32ok[u] ? (uint32_t)min(max((int32_t)((uint32_t)tq - (uint32_t)tk32), 0), (int32_t)cap)
                                 : clamp_delta(tq - tk, cap);
                int b;
                oct_lookup(du[j], s_oct, b, bc[j]);
                if (has_pos) bc[j] += __ldg(p.pos_weights + min(max(rel0 + g8 + j, 0), P - 1)) * c1;
              }
              tmem_ld_wait();
#pragma unroll
              for (int j = 0; j < 8; j += 2) {
                float pp[2], dd[2];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                  const bool ok = (g8 + j + e < ncol) && (rel0 + g8 + j + e >= 0);
                  const float hh = fmaf(__uint_as_float(v[j + e]), c1, bc[j + e]);
                  const float th = tanh_approx(hh);
                  const float pv = fmaf(hh, th, hh);
                  pp[e] = ok ? pv : 0.f;
                  dd[e] = ok ? fmaf(c1, fmaf(-pv, th, pv) + th, c1) : 0.f;
                }
                pk[j >> 1] = pack_bf16(pp[0], pp[1]);
                if (g8 < 16) {
                  kr[16 * u + g8 + j] = dd[0];
                  kr[16 * u + g8 + j + 1] = dd[1];
                } else {
                  kt[g8 - 16 + j] = __float_as_uint(dd[0]);
                  kt[g8 - 15 + j] = __float_as_uint(dd[1]);
                }
              }
              tmem_st4(cbase + (g8 >> 1), pk);
            }
            tmem_st16(cbase + 16, kt);
          }
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full);
        if (trc) trace_ev(p, 3, tcnt, 31, tc);
        // ---------------- phase dS: dP^T . SiLU' -> dS^T (TMEM R1 + shared), d_ts_weights
        mbar_wait(dp_full, ph);
        if (trc) trace_ev(p, 3, tcnt, 32, tc);
        tc_fence_after();
        float sat_w = 0.f, sat_p = 0.f;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int c = 2 * wg + u;
          const uint32_t dpbase = tR2 + 32 * c + lane_off;
          const uint32_t dsbase = tR1 + 32 * c + 16 + lane_off;
          const uint32_t srow = ds_smem + (c >> 1) * 16384 + r * 128;
          uint32_t dk[16];
          if (cls[u] == 0) {
#pragma unroll
            for (int j = 0; j < 16; ++j) dk[j] = 0u;
          } else {
            uint32_t dv[32], kt[16];
            tmem_ld32(dpbase, dv);
            tmem_ld16(dsbase, kt);
            tmem_ld_wait();
            float d[32];
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
              const float k0 = j < 16 ? kr[16 * u + j] : __uint_as_float(kt[j - 16]);
              const float k1 = j < 16 ? kr[16 * u + j + 1] : __uint_as_float(kt[j - 15]);
              d[j] = __uint_as_float(dv[j]) * k0;
              d[j + 1] = __uint_as_float(dv[j + 1]) * k1;
              dk[j >> 1] = pack_bf16(d[j], d[j + 1]);
            }
            if (cls[u] == 1 || cls[u] == 3) {
              float s = 0.f;
              if (cnt_mode) {
                s = cls[u] == 1 ? 32.f : (float)(krow_ok ? max(min(nq - 32 * c, 32), 0) : 0);
              } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) s += d[j];
              }
              sat_w += s;
              if (has_pos) sat_p += s;  // saturated chunks hit both last buckets
            } else if (cls[u] == 4) {
              const uint4* src = reinterpret_cast<const uint4*>(
                  band_chunk(p.band, band_q0 + 4 * t + c, bwi[u]) + 1024 + lane * 32);
              const uint4 b0 = __ldg(src), b1 = __ldg(src + 1);
              const uint32_t wd[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
              float s = 0.f;
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                const uint32_t b = __byte_perm(wd[j >> 2], 0u, 0x4440u | (j & 3));
                const float val = cnt_mode ? (b != kBandMasked ? 1.f : 0.f) : d[j];
                s += b == (uint32_t)(nb - 1) ? val : 0.f;
                red_add_f32_if(tbg + b * 256, val, b < (uint32_t)(nb - 1));
              }
              sat_w += s;
            } else {
              // general chunk: recompute bucket, mask (and position) per element
              const int64_t* tsq = p.ts_q + qrow0 + 32 * c;
              const int rel0 = (int)(qp_tile + 32 * c - kpos);
              const int ncol = krow_ok ? nq - 32 * c : 0;
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                const bool ok = (j < ncol) && (rel0 + j >= 0);
                const int64_t tq = j < nq - 32 * c ? __ldg(tsq + j) : 0;
                const uint32_t du = f32ok[u] ? (uint32_t)min(max((int32_t)((uint32_t)tq - (uint32_t)tk32), 0),
                                                            (int32_t)cap)
                                             : clamp_delta(tq - tk, cap);
                int b;
                float wdummy;
                oct_lookup(du, s_oct, b, wdummy);
                const float val = cnt_mode ? (ok ? 1.f : 0.f) : d[j];
                if (b == nb - 1)
                  sat_w += ok ? val : 0.f;
                else
                  red_add_f32_if(tbg + b * 256, val, ok);
                if (has_pos) {
                  const int rel = min(rel0 + j, P - 1);
                  red_add_f32_if(g_bins + 256 + max(rel, 0), val, ok && rel != P - 1);
                  sat_p += (ok && rel == P - 1) ? val : 0.f;
                }
              }
            }
          }
          tmem_st16(dsbase, dk);
          // shared-memory dS^T row r, q columns [32c, 32c+32): panel c/2, 16-byte chunks 4 (c&1) + q4 (swizzled)
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4)
            st_shared_v4(srow + ((((c & 1) * 4 + q4) ^ (r & 7)) << 4), dk[4 * q4], dk[4 * q4 + 1], dk[4 * q4 + 2],
                         dk[4 * q4 + 3]);
        }
        acc_w += (double)sat_w;
        acc_p += (double)sat_p;
        tmem_st_wait();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // st.shared -> tcgen05.mma operand reads
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(ds_full);
        if (trc) trace_ev(p, 3, tcnt, 33, tc);
      }
    }
    // ---- d_ts_weights / d_pos: per-CTA totals, summed by the last CTA in a fixed order
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      acc_w += __shfl_xor_sync(0xffffffffu, acc_w, o);
      acc_p += __shfl_xor_sync(0xffffffffu, acc_p, o);
    }
    double* s_red = reinterpret_cast<double*>(smem + C::ST_OFF);  // statistics ring is idle now
    __threadfence();  // this thread's bin reductions before the reads below
    named_bar_sync(1, 32 * kFComp);
    if (lane == 0) {
      s_red[et >> 5] = acc_w;
      s_red[kFComp + (et >> 5)] = acc_p;
    }
    named_bar_sync(1, 32 * kFComp);
    for (int b = (et >> 5); b < nb; b += kFComp) {
      const float* gb = p.tb_glob + (size_t)blockIdx.x * kTbBuckets * 256 + b * 256;
      float v = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) v += __ldcg(gb + lane + 32 * i);
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) g_bins[b] = v;
    }
    if (et < 2) {
      double v = 0.0;
      for (int w2 = 0; w2 < kFComp; ++w2) v += s_red[et * kFComp + w2];
      p.wl.partials[(size_t)blockIdx.x * 2 + et] = v;
    }
    __threadfence();
    named_bar_sync(1, 32 * kFComp);
    if (et == 0) s_flag[1] = atomicAdd(p.dw_done, 1) == (int)gridDim.x - 1 ? 1 : 0;
    named_bar_sync(1, 32 * kFComp);
    if (s_flag[1]) {
      __threadfence();
      for (int e = et; e < 256 + P; e += 32 * kFComp) {
        if (e >= nb && e < 256) continue;
        double v = 0.0;
        for (int c = 0; c < (int)gridDim.x; ++c) v += (double)__ldcg(p.wl.bins + (size_t)c * kBinsPerCta + e);
        if (e == nb - 1 || (P > 0 && e == 256 + P - 1))
          for (int c = 0; c < (int)gridDim.x; ++c) v += __ldcg(p.wl.partials + (size_t)c * 2 + (e < 256 ? 0 : 1));
        if (e < 256)
          p.d_ts_weights[e] += v;
        else
          p.d_pos_weights[e - 256] += v;
      }
      if (et == 0) *p.dw_done = 0;  // the state is all-zero again for the next call
    }
  } else if (warp >= 12) {
    // ================= drain: dQ per q tile (thread = q row), dK / dV per item (thread = kv row)
    const int r = tid - 384;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint64_t pol_out = l2_policy_evict_first();
    uint32_t tc = 0, ic = 0, rk = 0, tcnt = 0;
    const bool trd = r == 0;
    for (int g; (g = ring_consume(ring, rk, true)) >= 0;) {
      const int2 it = p.wl.bwd[g / H];
      const int h = g % H;
      const Seg sg = load_seg(p.seg, it.x);
      int t0, n;
      fused_tiles(sg, it.y, t0, n);
      const int64_t kpos = (int64_t)it.y * kBN + r;
      const bool krow_ok = kpos < sg.kv_len;
      const int64_t krow = sg.kv_row0 + kpos;
      if (n == 0) {
        if (krow_ok && !p.dk_accum)
          for (int c = 0; c < D; c += 8) {
            *reinterpret_cast<int4*>(p.dk + krow * p.ld_dk + h * D + c) = make_int4(0, 0, 0, 0);
            *reinterpret_cast<int4*>(p.dv + krow * p.ld_dv + h * D + c) = make_int4(0, 0, 0, 0);
          }
        continue;
      }
      for (int i = 0; i < n; ++i, ++tc) {
        const int64_t t = t0 + i;
        const bool row_ok = r < sg.lq - t * kBM;
        const int64_t qrow = sg.q_row0 + t * kBM + r;
        float* dst = p.dq_acc != nullptr ? p.dq_acc + qrow * ld_dq + h * D : p.dq_state + qrow * HD + h * D;
        mbar_wait(dq_full, tc & 1);
        if (trd) trace_ev(p, 2, tcnt, 20, tc);
        tc_fence_after();
        // coalesced reduction: an 8x8 transpose of 16-byte blocks inside each
        // group of 8 lanes turns "thread = row, 32 columns" into "8 lanes = one
        // row's 128 contiguous bytes", so each red.global.add.v4 instruction
        // covers 4 full lines instead of 32 rows x 16 bytes (r2: the per-row
        // form made the reductions the fused kernel's bottleneck)
        const int lane = r & 31, gi = lane & 7, rbase = (r & ~31) + (lane & ~7);
        float* drow = p.dq_acc != nullptr ? p.dq_acc + (sg.q_row0 + t * kBM + rbase) * ld_dq + h * D
                                          : p.dq_state + (sg.q_row0 + t * kBM + rbase) * HD + h * D;
        const int64_t dld = p.dq_acc != nullptr ? ld_dq : HD;
        const int nrow = (int)min((int64_t)8, max((int64_t)0, sg.lq - t * kBM - rbase));
#pragma unroll 1
        for (int cc = 0; cc < D; cc += 32) {
          uint32_t v[32];
          tmem_ld32(tR2 + lane_off + cc, v);
          tmem_ld_wait();
          if (cc + 32 == D) {
            tc_fence_before();
            mbar_arrive(dq_empty);
          }
          if (!(p.dbg & 8)) {
#pragma unroll
            for (int m = 4; m >= 1; m >>= 1) {
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                if (j & m) continue;
                const bool up = (gi & m) != 0;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const uint32_t send = up ? v[4 * j + e] : v[4 * (j | m) + e];
                  const uint32_t recv = __shfl_xor_sync(0xffffffffu, send, m);
                  if (up)
                    v[4 * j + e] = recv;
                  else
                    v[4 * (j | m) + e] = recv;
                }
              }
            }
            // v[4 j ..] = row rbase + j, columns cc + 4 gi .. + 3
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (j < nrow) red_add_v4(drow + j * dld + cc + 4 * gi, v + 4 * j);
          }
        }
        if (trd) trace_ev(p, 2, tcnt, 21, tc);
        if (p.dq_acc == nullptr && !(p.dbg & 8)) {
          // finalize: the CTA that delivers the last of the tile's ceil(kv_lim / 128)
          // contributions converts the fp32 rows to bf16 and re-zeroes them
          __threadfence();
          named_bar_sync(3, 128);
          if (r == 0) {
            int32_t* cnt = p.dq_cnt + ((sg.q_row0 >> 7) + it.x + t) * H + h;
            const int need = (int)((fwd_kv_lim(sg, (int)t) + kBN - 1) / kBN);
            const int old = atomicAdd(cnt, 1);
            const bool last = old == need - 1;
            if (last) *cnt = 0;
            s_flag[0] = last ? 1 : 0;
          }
          named_bar_sync(3, 128);
          if (s_flag[0]) {
            __threadfence();
            if (row_ok) {
              float4* a4 = reinterpret_cast<float4*>(dst);
              int4* o4 = reinterpret_cast<int4*>(dq + qrow * ld_dq + h * D);
#pragma unroll 4
              for (int c8 = 0; c8 < D / 8; ++c8) {
                const float4 x0 = __ldcg(a4 + 2 * c8), x1 = __ldcg(a4 + 2 * c8 + 1);
                st_global_v4_hint(o4 + c8, pack_bf16(x0.x, x0.y), pack_bf16(x0.z, x0.w), pack_bf16(x1.x, x1.y),
                                  pack_bf16(x1.z, x1.w), pol_out);
                a4[2 * c8] = make_float4(0.f, 0.f, 0.f, 0.f);
                a4[2 * c8 + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
              }
            }
          }
        }
      }
      // dK / dV of the item (thread = kv row)
      if (trd) trace_ev(p, 2, tcnt, 22, tc);
      mbar_wait(dkv_full, ic & 1);
      if (trd) trace_ev(p, 2, tcnt, 23, ic);
      ++ic;
      tc_fence_after();
#pragma unroll 1
      for (int part = 0; part < 2; ++part) {
        const uint32_t tsrc = part ? tDK : tDV;
        float* acc = part ? p.dk_accum : p.dv_accum;
#pragma unroll 1
        for (int cc = 0; cc < D; cc += 32) {
          uint32_t v[32];
          tmem_ld32(tsrc + lane_off + cc, v);
          tmem_ld_wait();
          if (part == 1 && cc + 32 == D) {
            tc_fence_before();
            mbar_arrive(dkv_empty);
          }
          if (!krow_ok) continue;
          if (acc) {
            float* dst = acc + krow * HD + h * D + cc;
#pragma unroll
            for (int q4 = 0; q4 < 8; ++q4) red_add_v4(dst + 4 * q4, v + 4 * q4);
          } else {
            __nv_bfloat16* dst = (part ? (p.dk + krow * p.ld_dk) : (p.dv + krow * p.ld_dv)) + h * D + cc;
            uint32_t pk[16];
#pragma unroll
            for (int j = 0; j < 32; j += 2) pk[j >> 1] = pack_bf16(__uint_as_float(v[j]), __uint_as_float(v[j + 1]));
            int4* d4 = reinterpret_cast<int4*>(dst);
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4)
              st_global_v4_hint(d4 + q4, pk[4 * q4], pk[4 * q4 + 1], pk[4 * q4 + 2], pk[4 * q4 + 3], pol_out);
          }
        }
      }
      if (trd) trace_ev(p, 2, tcnt, 24, ic);
    }
  }
  tc_fence_before();
  __syncthreads();
  cta_stamp(p, 1);
  if (warp == 2) tmem_dealloc(tmem, 512);
}

template <int D>
int launch_bwd_fused(const TMaps& tm, const AttnParams& p, const jh_attn_args& a, int grid, cudaStream_t s) {
  using C = FusedCfg<D>;
  static_assert(C::SMEM <= 232448, "fused bwd smem budget");
  if (a.num_buckets > 32) {
    set_error(JH_ERR_UNSUPPORTED, "fused backward supports num_buckets <= 32");
    return -1;
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(hstu_bwd_fused_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    cudaFuncSetAttribute(hstu_bwd_fused_kernel<D>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    attr = true;
  }
  if (a.prof_event_start) cudaEventRecord((cudaEvent_t)a.prof_event_start, s);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kFThreads);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  la[0].val.programmaticStreamSerializationAllowed = 1;  // prologue overlaps the work-list build
  cfg.attrs = la;
  cfg.numAttrs = 1;
  if (cudaError_t e = cudaLaunchKernelEx(&cfg, hstu_bwd_fused_kernel<D>, tm.q, tm.k, tm.v, tm.dout, p,
                                         (__nv_bfloat16*)a.dq, (int64_t)a.ld_dq))
    return (int)e;
  if (a.prof_event_end) cudaEventRecord((cudaEvent_t)a.prof_event_end, s);
  return (int)cudaGetLastError();
}

template int launch_bwd_fused<64>(const TMaps&, const AttnParams&, const jh_attn_args&, int, cudaStream_t);
template int launch_bwd_fused<128>(const TMaps&, const AttnParams&, const jh_attn_args&, int, cudaStream_t);

}  // namespace jh
