// Fused jagged HSTU attention forward for sm_100a, two q tiles per K/V tile.
//
//   out = (tril . SiLU((Q K^T + bias) / sqrt(d))) V     per segment, per head
//   (reference: attention.py:125-148 hstu_attention_reference, and the
//    blockwise form attention.py:151-184 used by the CP ring)
//
// A work item is (segment, q tile pair u) x head: q tiles A = 2u and B = 2u+1
// (B may not exist) share every K / V tile they load, which halves the
// L2 -> SM bytes per FLOP of the one-tile kernel (attn_fwd.cu: 64 KB of K / V
// per 128 x 128 tile pair of GEMMs, against ~42 B/clk/SM of chip L2 feed).
//   warp 0       TMA producer: Q_A, Q_B (+ ts_q), K_j (+ ts_k), V_j (NS stages each)
//   warp 1       MMA issuer, ping-pong over the two tiles (TMEM S_A, S_B, O_A, O_B):
//                  S_A(0) S_B(0) | PV_A(j) S_A(j+1) PV_B(j) S_B(j+1) | ...
//                so each epilogue warpgroup's SiLU of tile j+1 runs while the
//                tensor core works on the other tile
//   warp 2       TMEM allocator (512 columns);  warp 3: per-chunk max / min of ts_k
//   warps 4..7   epilogue of tile A, warps 8..11 epilogue of tile B (thread = q row,
//                all 128 columns of every kv tile; same chunk classes as attn_fwd.cu:
//                masked / saturated (2 FFMA + 1 MUFU) / band table / exact per element)
//   warps 12..15 drain O_A, O_B (bf16, or the fp32 CP partial modes)
// TMEM columns: S_A [0,128) S_B [128,256) O_A [256, 256+D) O_B [256+D, 256+2D)
// SiLU partials are additive (no softmax normaliser): O simply accumulates.
#include "attn_common.cuh"

namespace jh {

constexpr int kF2Threads = 512;
constexpr int kF2TsRing = 4;

template <int D>
struct Fwd2Cfg {
  static constexpr int NS = (D == 64) ? 4 : 2;  // K / V stages
  static constexpr int PANELS = D / 64;
  static constexpr int TILE_BYTES = 128 * D * 2;
  static constexpr int Q_OFF = 0;                             // [2]: A, B
  static constexpr int K_OFF = 2 * TILE_BYTES;                // [NS]
  static constexpr int V_OFF = K_OFF + NS * TILE_BYTES;       // [NS]
  static constexpr int TSQ_OFF = V_OFF + NS * TILE_BYTES;     // int64 [2][kTsSlot]
  static constexpr int TSK_OFF = TSQ_OFF + 2 * kTsSlot * 8;   // int64 [kF2TsRing][kTsSlot]
  static constexpr int OCT_OFF = TSK_OFF + kF2TsRing * kTsSlot * 8;  // OctEntry [32]
  static constexpr int PW_OFF = OCT_OFF + 32 * 16;            // float pw[<=1024] x c1
  static constexpr int WT_OFF = PW_OFF + 1024 * 4;            // float [32] band weights x c1
  static constexpr int KMAX_OFF = WT_OFF + 32 * 4;            // int64 [kF2TsRing][4] max, then min
  static constexpr int BAR_OFF = KMAX_OFF + 2 * kF2TsRing * 32;
  static constexpr int NBARS = 4 + 4 * NS + 3 * kF2TsRing + 8;
  static constexpr int TMEMPTR_OFF = BAR_OFF + NBARS * 8;
  static constexpr int RING_OFF = TMEMPTR_OFF + 16;
  static constexpr int SMEM = RING_OFF + 2 * kItemRing * 8 + kItemRing * 4;
};

struct PairItem {
  int g, h, nA, nB, nK;
  bool hasB;
  int2 it;  // (segment, pair u)
  Seg sg;
};

JH_DEV PairItem decode_pair(const AttnParams& p, int g, int H) {
  PairItem x;
  x.g = g;
  x.it = p.wl.fwd[g / H];
  x.h = g % H;
  x.sg = load_seg(p.seg, x.it.x);
  const int tA = 2 * x.it.y;
  x.hasB = (int64_t)(tA + 1) * kBM < x.sg.lq;
  x.nA = (int)((fwd_kv_lim(x.sg, tA) + kBN - 1) / kBN);
  x.nB = x.hasB ? (int)((fwd_kv_lim(x.sg, tA + 1) + kBN - 1) / kBN) : 0;
  x.nK = x.nA > x.nB ? x.nA : x.nB;
  return x;
}

template <int D>
__global__ void __launch_bounds__(kF2Threads, 1)
    hstu_fwd2_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_tsq,
                     const __grid_constant__ CUtensorMap tm_tsk, const __grid_constant__ AttnParams p) {
  using C = Fwd2Cfg<D>;
  constexpr int NS = C::NS;
  extern __shared__ __align__(1024) uint8_t smem[];
  int64_t* s_tsq = reinterpret_cast<int64_t*>(smem + C::TSQ_OFF);
  int64_t* s_tsk = reinterpret_cast<int64_t*>(smem + C::TSK_OFF);
  OctEntry* s_oct = reinterpret_cast<OctEntry*>(smem + C::OCT_OFF);
  float* s_pwc = reinterpret_cast<float*>(smem + C::PW_OFF);
  float* s_wt = reinterpret_cast<float*>(smem + C::WT_OFF);
  int64_t* s_kmax = reinterpret_cast<int64_t*>(smem + C::KMAX_OFF);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* q_full = bars;                     // [2] A, B
  uint64_t* q_empty = bars + 2;                // [2] last S MMA of the tile + its epilogue's ts_q read
  uint64_t* k_full = bars + 4;                 // [NS]
  uint64_t* k_empty = k_full + NS;             // [NS]
  uint64_t* v_full = k_empty + NS;             // [NS]
  uint64_t* v_empty = v_full + NS;             // [NS]
  uint64_t* ts_full = v_empty + NS;            // [kF2TsRing]
  uint64_t* ts_empty = ts_full + kF2TsRing;    // [kF2TsRing] both epilogue warpgroups
  uint64_t* tsx_full = ts_empty + kF2TsRing;   // [kF2TsRing] chunk maxima / minima ready
  uint64_t* s_full = tsx_full + kF2TsRing;     // [2]
  uint64_t* p_full = s_full + 2;               // [2]
  uint64_t* o_full = p_full + 2;               // [2]
  uint64_t* o_empty = o_full + 2;              // [2]
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + C::TMEMPTR_OFF);
  const ItemRing ring{reinterpret_cast<int32_t*>(smem + C::RING_OFF + 2 * kItemRing * 8),
                      reinterpret_cast<uint64_t*>(smem + C::RING_OFF),
                      reinterpret_cast<uint64_t*>(smem + C::RING_OFF + kItemRing * 8)};

  const uint32_t warp = warp_id();
  const int tid = threadIdx.x;
  const int H = p.num_heads;
  const int nb = p.bias.nb;

  cta_stamp(p, 0, 2);
  if (smem_u32(smem) & 1023) __trap();
  const float c1 = p.c1;  // SiLU(s) = h + h tanh(h), h = c1 (q k^T + bias)
  oct_table_fill(s_oct, p.bias, p.ts_weights, c1, tid, blockDim.x);
  for (int i = tid; i < p.num_pos; i += blockDim.x) s_pwc[i] = p.pos_weights[i] * c1;
  if (tid < 32) s_wt[tid] = tid < nb ? p.ts_weights[tid] * c1 : (tid == (int)kBandMasked ? -1e30f : 0.f);
  if (tid == 0) {
    for (int x = 0; x < 2; ++x) {
      mbar_init(&q_full[x], 1);
      mbar_init(&q_empty[x], 1 + 4);
      mbar_init(&s_full[x], 1);
      mbar_init(&p_full[x], 4);
      mbar_init(&o_full[x], 1);
      mbar_init(&o_empty[x], 128);
    }
    for (int i = 0; i < NS; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < kF2TsRing; ++i) {
      mbar_init(&ts_full[i], 1);
      mbar_init(&ts_empty[i], 8);  // the 4 + 4 epilogue warps
      mbar_init(&tsx_full[i], 1);
    }
    ring_init(ring, 1 + 1 + 8 + 4);  // consumers: MMA, ts stats, epilogue warps, drain warps
    fence_barrier_init();
  }
  if (warp == 0 && lane_id() == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    tma_prefetch_desc(&tm_tsq);
    tma_prefetch_desc(&tm_tsk);
  }
  if (warp == 2) tmem_alloc(s_tmem, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int total = p.wl.hdr->n_fwd * H;

  if (warp == 0) {
    // ================= TMA producer
    if (elect_one()) {
      uint32_t rk = 0, k_it = 0, v_it = 0, t_it = 0, qa_it = 0, qb_it = 0;
      auto load_q = [&](const PairItem& x, int which, uint32_t& q_it) {
        mbar_wait(&q_empty[which], (q_it & 1) ^ 1);
        mbar_expect_tx(&q_full[which], C::TILE_BYTES + kTsBytes);
        const int32_t qrow = (int32_t)(x.sg.q_row0 + (int64_t)(2 * x.it.y + which) * kBM);
        for (int pn = 0; pn < C::PANELS; ++pn)
          tma_load_2d(smem + C::Q_OFF + which * C::TILE_BYTES + pn * 16384, &tm_q, x.h * D + pn * 64, qrow,
                      &q_full[which]);
        tma_load_1d(s_tsq + which * kTsSlot, &tm_tsq, qrow & ~1, &q_full[which]);
        ++q_it;
      };
      auto load_k = [&](const PairItem& x, int j) {
        const int st = k_it % NS, ts = t_it % kF2TsRing;
        const int32_t krow = (int32_t)(x.sg.kv_row0 + (int64_t)j * kBN);
        mbar_wait(&k_empty[st], ((k_it / NS) & 1) ^ 1);
        mbar_expect_tx(&k_full[st], C::TILE_BYTES);
        for (int pn = 0; pn < C::PANELS; ++pn)
          tma_load_2d(smem + C::K_OFF + st * C::TILE_BYTES + pn * 16384, &tm_k, x.h * D + pn * 64, krow, &k_full[st]);
        mbar_wait(&ts_empty[ts], ((t_it / kF2TsRing) & 1) ^ 1);
        mbar_expect_tx(&ts_full[ts], kTsBytes);
        tma_load_1d(s_tsk + ts * kTsSlot, &tm_tsk, krow & ~1, &ts_full[ts]);
        ++k_it;
        ++t_it;
      };
      auto load_v = [&](const PairItem& x, int j) {
        const int st = v_it % NS;
        const int32_t krow = (int32_t)(x.sg.kv_row0 + (int64_t)j * kBN);
        mbar_wait(&v_empty[st], ((v_it / NS) & 1) ^ 1);
        mbar_expect_tx(&v_full[st], C::TILE_BYTES);
        for (int pn = 0; pn < C::PANELS; ++pn)
          tma_load_2d(smem + C::V_OFF + st * C::TILE_BYTES + pn * 16384, &tm_v, x.h * D + pn * 64, krow, &v_full[st]);
        ++v_it;
      };
      for (int g; (g = ring_produce(ring, rk, &p.wl.hdr->next_item[0], total)) >= 0;) {
        const PairItem x = decode_pair(p, g, H);
        if (x.nK == 0) continue;
        // Q_A (its buffer frees after the previous item's last S_A), K_0, Q_B, V_0, then K_j, V_j
        load_q(x, 0, qa_it);
        load_k(x, 0);
        if (x.hasB) load_q(x, 1, qb_it);
        load_v(x, 0);
        for (int j = 1; j < x.nK; ++j) {
          load_k(x, j);
          load_v(x, j);
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer (one thread)
    if (elect_one()) {
      constexpr uint32_t idesc_s = idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t idesc_pv = idesc_bf16(128, D, 0, 1);
      uint32_t rk = 0, k_it = 0, v_it = 0, qa_it = 0, qb_it = 0;
      uint32_t pc[2] = {0u, 0u};  // P tiles consumed per buffer
      uint32_t oc[2] = {0u, 0u};  // items that used accumulator O_A / O_B
      auto issue_S = [&](int which, uint32_t k_base) {
        const uint32_t q_base = smem_u32(smem + C::Q_OFF + which * C::TILE_BYTES);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          umma_ss(tmem + 128 * which, sdesc_sw128(q_base + off, 16, 1024), sdesc_sw128(k_base + off, 16, 1024),
                  idesc_s, kk > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[which]);
      };
      auto issue_PV = [&](int which, uint32_t v_base, bool first) {
        mbar_wait(&p_full[which], pc[which] & 1);
        ++pc[which];
        if (first) mbar_wait(&o_empty[which], (oc[which] & 1) ^ 1);
        tc_fence_after();
        const uint32_t tO = tmem + 256 + which * D;
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk)
          umma_ts(tO, tmem + 128 * which + 32 * (kk >> 1) + 8 * (kk & 1), sdesc_sw128(v_base + kk * 2048, 16384, 1024),
                  idesc_pv, (first && kk == 0) ? 0u : 1u);
      };
      for (int g; (g = ring_consume(ring, rk, false)) >= 0;) {
        const PairItem x = decode_pair(p, g, H);
        if (x.nK == 0) continue;
        const int nA = x.nA, nB = x.nB, nK = x.nK;
        mbar_wait(&q_full[0], qa_it & 1);
        if (x.hasB) mbar_wait(&q_full[1], qb_it & 1);
        // step 0: S_A(0), S_B(0)
        {
          const int st = k_it % NS;
          mbar_wait(&k_full[st], (k_it / NS) & 1);
          tc_fence_after();
          const uint32_t k_base = smem_u32(smem + C::K_OFF + st * C::TILE_BYTES);
          if (nA > 0) issue_S(0, k_base);
          if (nA == 1) umma_commit(&q_empty[0]);
          if (nB > 0) issue_S(1, k_base);
          if (nB == 1) umma_commit(&q_empty[1]);
          umma_commit(&k_empty[st]);
          ++k_it;
        }
        for (int j = 0; j < nK; ++j) {
          const int vs = v_it % NS;
          mbar_wait(&v_full[vs], (v_it / NS) & 1);
          const uint32_t v_base = smem_u32(smem + C::V_OFF + vs * C::TILE_BYTES);
          if (j < nA) {
            issue_PV(0, v_base, j == 0);
            if (j == nA - 1) umma_commit(&o_full[0]);
          }
          // S_A(j+1): its buffer's P_A(j) was consumed by PV_A(j), issued above
          uint32_t kn_base = 0;
          int kst = -1;
          if (j + 1 < nK) {
            kst = k_it % NS;
            mbar_wait(&k_full[kst], (k_it / NS) & 1);
            tc_fence_after();
            kn_base = smem_u32(smem + C::K_OFF + kst * C::TILE_BYTES);
            if (j + 1 < nA) {
              issue_S(0, kn_base);
              if (j + 1 == nA - 1) umma_commit(&q_empty[0]);
            }
          }
          if (j < nB) {
            issue_PV(1, v_base, j == 0);
            if (j == nB - 1) umma_commit(&o_full[1]);
          }
          umma_commit(&v_empty[vs]);
          ++v_it;
          if (j + 1 < nK) {
            if (j + 1 < nB) {
              issue_S(1, kn_base);
              if (j + 1 == nB - 1) umma_commit(&q_empty[1]);
            }
            umma_commit(&k_empty[kst]);
            ++k_it;
          }
        }
        ++qa_it;
        ++oc[0];
        if (x.hasB) {
          ++qb_it;
          ++oc[1];
        }
      }
    }
  } else if (warp == 3) {
    // ================= ts_k tile statistics: per 32-column chunk maximum and minimum
    const int lane = lane_id();
    uint32_t t_it = 0, rk = 0;
    for (int g; (g = ring_consume(ring, rk, true)) >= 0;) {
      const PairItem x = decode_pair(p, g, H);
      for (int j = 0; j < x.nK; ++j) {
        const int ts = t_it % kF2TsRing;
        mbar_wait(&ts_full[ts], (t_it / kF2TsRing) & 1);
        const int64_t* tsk = s_tsk + ts * kTsSlot + ((x.sg.kv_row0 + (int64_t)j * kBN) & 1);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int64_t m = warp_max_i64(tsk[32 * c + lane]);
          const int64_t mn = warp_min_i64(tsk[32 * c + lane]);
          if (lane == 0) {
            s_kmax[ts * 4 + c] = m;
            s_kmax[kF2TsRing * 4 + ts * 4 + c] = mn;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&tsx_full[ts]);
        ++t_it;
      }
    }
  } else if (warp >= 4 && warp < 12) {
    // ================= epilogue: warpgroup X = tile X of the pair; thread = q row r
    const int et = tid - 128;
    const int X = et >> 7;
    const int r = et & 127;
    const int lane = r & 31;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const int64_t cap = p.bias.cap;
    const int P = p.num_pos;
    const bool has_pos = P > 0;
    const bool use_band = p.band != nullptr;
    float cb = p.ts_weights[nb - 1];
    if (has_pos) cb += p.pos_weights[P - 1];
    cb *= c1;
    uint32_t q_it = 0, s_it = 0, t_it = 0, rk = 0;
    const uint32_t tS = tmem + 128 * X + lane_off;
    for (int g; (g = ring_consume(ring, rk, true)) >= 0;) {
      const PairItem x = decode_pair(p, g, H);
      if (x.nK == 0) continue;
      const Seg& sg = x.sg;
      const int tX = 2 * x.it.y + X;
      const bool mine = X == 0 || x.hasB;
      const int nX = X == 0 ? x.nA : x.nB;
      if (!mine || nX == 0) {
        // not this warpgroup's tile: only release the ts ring slots
        for (int j = 0; j < x.nK; ++j, ++t_it) {
          const int ts = t_it % kF2TsRing;
          mbar_wait(&tsx_full[ts], (t_it / kF2TsRing) & 1);
          __syncwarp();
          if (lane == 0) mbar_arrive(&ts_empty[ts]);
        }
        continue;
      }
      const int64_t kv_lim = fwd_kv_lim(sg, tX);
      const int64_t nq = min((int64_t)kBM, sg.lq - (int64_t)tX * kBM);
      const bool row_ok = r < nq;
      const int64_t qp_tile = sg.qp0 + (int64_t)tX * kBM;
      const int64_t qpos = qp_tile + r;
      uint8_t* dbgb = (p.dbg_buckets != nullptr && x.h == 0 && row_ok)
                          ? p.dbg_buckets + (sg.q_row0 + (int64_t)tX * kBM + r) * p.dbg_ld
                          : nullptr;
      mbar_wait(&q_full[X], q_it & 1);
      const int64_t tq = row_ok ? s_tsq[X * kTsSlot + ((sg.q_row0 + (int64_t)tX * kBM) & 1) + r] : (INT64_MAX >> 2);
      __syncwarp();
      if (lane == 0) mbar_arrive(&q_empty[X]);
      ++q_it;
      const int64_t tq_min = warp_min_i64(tq);
      const int64_t tq_max = warp_max_i64(row_ok ? tq : (INT64_MIN >> 2));
      const int32_t tq32 = (int32_t)(uint32_t)(uint64_t)tq;
      const int64_t row_lo = qp_tile + (r & ~31), row_hi = row_lo + 31;
      const int aq = tX * 4 + (r >> 5);
      const int64_t bd = (sg.qp0 >> 5) + aq;
      const bool band_row = use_band && 32 * (int64_t)aq < sg.lq;
      const uint8_t* brow = band_row ? band_chunk(p.band, band_group(sg, x.it.x, aq), 0) + lane * 32 : nullptr;
      for (int j = 0; j < x.nK; ++j, ++t_it) {
        const int ts = t_it % kF2TsRing;
        if (j >= nX) {  // (tile A ends one kv tile before B)
          mbar_wait(&tsx_full[ts], (t_it / kF2TsRing) & 1);
          __syncwarp();
          if (lane == 0) mbar_arrive(&ts_empty[ts]);
          continue;
        }
        // band chunks of this tile: prefetch the two diagonal-most byte rows before any wait
        uint32_t cand = 0;
        if (band_row) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int64_t b = 4 * (int64_t)j + c;
            const int64_t wi = b - bd + 3;
            if (wi >= 0 && wi < kBandNW && 32 * b <= row_hi && 32 * b < kv_lim) cand |= 1u << c;
          }
        }
        const int c_hi = cand ? 31 - __clz(cand) : -1;
        const uint32_t cand2 = c_hi >= 0 ? cand & ~(1u << c_hi) : 0u;
        const int c_lo = cand2 ? 31 - __clz(cand2) : -1;
        uint4 pf_hi0 = make_uint4(0, 0, 0, 0), pf_hi1 = pf_hi0, pf_lo0 = pf_hi0, pf_lo1 = pf_hi0;
        if (c_hi >= 0) {
          const uint4* src = reinterpret_cast<const uint4*>(brow + (4 * j + c_hi - bd + 3) * kBandChunk);
          pf_hi0 = __ldg(src);
          pf_hi1 = __ldg(src + 1);
        }
        if (c_lo >= 0) {
          const uint4* src = reinterpret_cast<const uint4*>(brow + (4 * j + c_lo - bd + 3) * kBandChunk);
          pf_lo0 = __ldg(src);
          pf_lo1 = __ldg(src + 1);
        }
        const int64_t kv0 = (int64_t)j * kBN;
        mbar_wait(&tsx_full[ts], (t_it / kF2TsRing) & 1);
        mbar_wait(&s_full[X], s_it & 1);
        ++s_it;
        tc_fence_after();
        const int64_t* tsk = s_tsk + ts * kTsSlot + ((sg.kv_row0 + kv0) & 1);
#pragma unroll 1
        for (int c0 = 0; c0 < kBN; c0 += 32) {
          const int64_t kc0 = kv0 + c0, kc1 = kc0 + 31;
          int cls = 0;  // 0 masked, 1 saturated, 2 general, 4 band table
          if (!(kc0 > row_hi || kc0 >= kv_lim)) {
            cls = 2;
            if ((kc1 <= row_lo) && (kc1 < kv_lim) && (tq_min - s_kmax[ts * 4 + (c0 >> 5)] >= cap) &&
                (!has_pos || row_lo - kc1 >= P - 1))
              cls = 1;
            else if ((cand >> (c0 >> 5)) & 1u)
              cls = 4;
          }
          if (cls == 4) {
            const int c = c0 >> 5;
            uint4 w0, w1;
            if (c == c_hi) {
              w0 = pf_hi0;
              w1 = pf_hi1;
            } else if (c == c_lo) {
              w0 = pf_lo0;
              w1 = pf_lo1;
            } else {
              const uint4* src = reinterpret_cast<const uint4*>(brow + (4 * j + c - bd + 3) * kBandChunk);
              w0 = __ldg(src);
              w1 = __ldg(src + 1);
            }
            const uint32_t wd[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
            if (dbgb != nullptr) {
#pragma unroll 1
              for (int i = 0; i < 32; ++i) {
                const uint32_t b = (wd[i >> 2] >> (8 * (i & 3))) & 0xFFu;
                if (b != kBandMasked) dbgb[kv0 + c0 + i] = (uint8_t)b;
              }
            }
            uint32_t v[32], pk[16];
            tmem_ld32(tS + c0, v);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              const float b0 = s_wt[__byte_perm(wd[i >> 2], 0u, 0x4440u | (i & 3))];
              const float b1 = s_wt[__byte_perm(wd[i >> 2], 0u, 0x4440u | ((i + 1) & 3))];
              const float h0 = fmaf(__uint_as_float(v[i]), c1, b0);
              const float h1 = fmaf(__uint_as_float(v[i + 1]), c1, b1);
              pk[i >> 1] = pack_bf16(fmaf(h0, tanh_approx(h0), h0), fmaf(h1, tanh_approx(h1), h1));
            }
            tmem_st16(tS + c0, pk);
          } else if (cls == 1) {
            if (dbgb != nullptr) {
#pragma unroll 1
              for (int i = 0; i < 32; ++i) dbgb[kv0 + c0 + i] = (uint8_t)(nb - 1);
            }
            uint32_t v[32], pk[16];
            tmem_ld32(tS + c0, v);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              const float h0 = fmaf(__uint_as_float(v[i]), c1, cb);
              const float h1 = fmaf(__uint_as_float(v[i + 1]), c1, cb);
              pk[i >> 1] = pack_bf16(fmaf(h0, tanh_approx(h0), h0), fmaf(h1, tanh_approx(h1), h1));
            }
            tmem_st16(tS + c0, pk);
          } else if (cls == 0) {
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = 0u;
            tmem_st16(tS + c0, pk);
          } else {
            // general chunk: exact per-element bucket, positional bias and mask, 8 columns per step
            const int relc = (int)(qpos - kv0 - c0);
            const int ncol = (int)min(kv_lim - kv0 - c0, (int64_t)32);
            const bool fits32 = cap < 0x7FFFFFFFll &&
                                tq_max - s_kmax[kF2TsRing * 4 + ts * 4 + (c0 >> 5)] < 0x7FFFFFFFll &&
                                tq_min - s_kmax[ts * 4 + (c0 >> 5)] > -0x7FFFFFFFll;
            const int32_t* tsk32 = reinterpret_cast<const int32_t*>(tsk + c0);
            uint32_t vn[8];
            tmem_ld8(tS + c0, vn);
#pragma unroll 1
            for (int g8 = 0; g8 < 32; g8 += 8) {
              uint32_t v[8], pk[4], du[8];
              float bc[8];
              if (fits32) {
#pragma unroll
                for (int i = 0; i < 8; ++i)
                  du[i] = (uint32_t)min(max((int32_t)((uint32_t)tq32 - (uint32_t)tsk32[2 * (g8 + i)]), 0), (int32_t)cap);
              } else {
#pragma unroll
                for (int i = 0; i < 8; ++i) du[i] = clamp_delta(tq - tsk[c0 + g8 + i], cap);
              }
              bool unsat = false;
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const int k = g8 + i;
                unsat |= (k <= relc && k < ncol) && du[i] < (uint32_t)cap;
              }
              const bool all_sat = !has_pos && !__any_sync(0xffffffffu, unsat);
              if (dbgb != nullptr) {
#pragma unroll 1
                for (int i = 0; i < 8; ++i) {
                  const int k = g8 + i;
                  int b = nb - 1;
                  float wdummy;
                  if (!all_sat) oct_lookup(du[i], s_oct, b, wdummy);
                  if (k <= relc && k < ncol) dbgb[kv0 + c0 + k] = (uint8_t)b;
                }
              }
              if (all_sat) {
#pragma unroll
                for (int i = 0; i < 8; ++i) bc[i] = cb;
              } else {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  int b;
                  oct_lookup(du[i], s_oct, b, bc[i]);
                }
                if (has_pos) {
#pragma unroll
                  for (int i = 0; i < 8; ++i) bc[i] += s_pwc[min(max(relc - g8 - i, 0), P - 1)];
                }
              }
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 8; ++i) v[i] = vn[i];
              if (g8 < 24) tmem_ld8(tS + c0 + g8 + 8, vn);
#pragma unroll
              for (int i = 0; i < 8; i += 2) {
                float y[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                  const int k = g8 + i + u;
                  const float hh = fmaf(__uint_as_float(v[i + u]), c1, bc[i + u]);
                  const float yy = fmaf(hh, tanh_approx(hh), hh);
                  y[u] = (k <= relc && k < ncol) ? yy : 0.f;
                }
                pk[i >> 1] = pack_bf16(y[0], y[1]);
              }
              tmem_st4(tS + c0 + (g8 >> 1), pk);
            }
          }
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&p_full[X]);
          mbar_arrive(&ts_empty[ts]);
        }
      }
    }
  } else if (warp >= 12) {
    // ================= O drain: TMEM -> bf16 (or fp32 partials) -> global (thread = q row)
    const int r = tid - 384;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    uint32_t od[2] = {0u, 0u}, rk = 0;
    const uint64_t pol_out = l2_policy_evict_first();
    for (int g; (g = ring_consume(ring, rk, true)) >= 0;) {
      const PairItem x = decode_pair(p, g, H);
      if (x.nK == 0) continue;
      for (int X = 0; X < 2; ++X) {
        if (X == 1 && !x.hasB) break;
        const int tX = 2 * x.it.y + X;
        const int64_t nq = min((int64_t)kBM, x.sg.lq - (int64_t)tX * kBM);
        const bool row_ok = r < nq;
        const int64_t orow_i = (x.sg.q_row0 + (int64_t)tX * kBM + r) * p.ld_o + x.h * D;
        mbar_wait(&o_full[X], od[X] & 1);
        ++od[X];
        tc_fence_after();
        const uint32_t tO = tmem + 256 + X * D + lane_off;
        if (p.out_acc != nullptr) {
          float4* arow = reinterpret_cast<float4*>(p.out_acc + orow_i);
#pragma unroll 1
          for (int c0 = 0; c0 < D; c0 += 32) {
            uint32_t v[32];
            tmem_ld32(tO + c0, v);
            tmem_ld_wait();
            if (c0 + 32 == D) {
              tc_fence_before();
              mbar_arrive(&o_empty[X]);
            }
            if (row_ok) {
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                float4 o = make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                       __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
                if (p.out_acc_add) {
                  const float4 a = arow[(c0 >> 2) + i];
                  o.x += a.x;
                  o.y += a.y;
                  o.z += a.z;
                  o.w += a.w;
                }
                arow[(c0 >> 2) + i] = o;
              }
            }
          }
          continue;
        }
        uint32_t pk[D / 2];
#pragma unroll
        for (int c0 = 0; c0 < D; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(tO + c0, v);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; i += 2) pk[(c0 + i) >> 1] = pack_bf16(__uint_as_float(v[i]), __uint_as_float(v[i + 1]));
        }
        tc_fence_before();
        mbar_arrive(&o_empty[X]);
        if (row_ok) {
          int4* dst = reinterpret_cast<int4*>(p.out + orow_i);
#pragma unroll
          for (int i = 0; i < D / 8; ++i)
            st_global_v4_hint(dst + i, pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3], pol_out);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cta_stamp(p, 1, 2);
  if (warp == 2) tmem_dealloc(tmem, 512);
}

template <int D>
int launch_fwd2(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, const CUtensorMap& ttq,
                const CUtensorMap& ttk, const AttnParams& p, int grid, cudaStream_t s, void* ev0, void* ev1) {
  using C = Fwd2Cfg<D>;
  static_assert(C::SMEM <= 232448, "fwd2 smem budget");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(hstu_fwd2_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    cudaFuncSetAttribute(hstu_fwd2_kernel<D>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    attr = true;
  }
  if (ev0) cudaEventRecord((cudaEvent_t)ev0, s);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kF2Threads);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  la[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = la;
  cfg.numAttrs = 1;
  if (cudaError_t e = cudaLaunchKernelEx(&cfg, hstu_fwd2_kernel<D>, tq, tk, tv, ttq, ttk, p)) return (int)e;
  if (ev1) cudaEventRecord((cudaEvent_t)ev1, s);
  return (int)cudaGetLastError();
}

template int launch_fwd2<64>(const CUtensorMap&, const CUtensorMap&, const CUtensorMap&, const CUtensorMap&,
                             const CUtensorMap&, const AttnParams&, int, cudaStream_t, void*, void*);
template int launch_fwd2<128>(const CUtensorMap&, const CUtensorMap&, const CUtensorMap&, const CUtensorMap&,
                              const CUtensorMap&, const AttnParams&, int, cudaStream_t, void*, void*);

}  // namespace jh
