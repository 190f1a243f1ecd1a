// Fused jagged HSTU attention forward for sm_100a.
//
//   out = (tril . SiLU((Q K^T + bias) / sqrt(d))) V     per segment, per head
//   (reference: attention.py:125-148 hstu_attention_reference, and the
//    blockwise form attention.py:151-184 used by the CP ring)
//
// Persistent, warp-specialised kernel, one CTA per SM (grid = #SMs), work
// items (segment, 128-row q tile) x head from the device-built list.
//   warp 0       TMA producer: Q + ts_q tile (2 buffers), K + ts_k / V tiles
//                (NS stages, K runs one tile ahead of V; K is released as soon
//                as S = Q K^T has consumed it, V after O += P V)
//   warp 1       MMA issuer (one lane): S = Q K^T -> TMEM (3 buffers, S runs
//                two tiles ahead of PV), O += P V with P read from TMEM
//                (tcgen05 .kind::f16, A in TMEM)
//   warp 2       TMEM allocator (512 columns); warp 3: per-chunk max of ts_k
//   warps 4..11  epilogue, two warpgroups in ping-pong over the kv tiles (tile
//                i -> group i % 2, S buffer i % 3), so one group's TMEM / barrier
//                latency hides behind the other's MUFU work.  Thread = q row, all 128
//                columns of its tiles.  Per 32-column chunk (warp-uniform):
//                fully masked -> P = 0; unmasked and bias-saturated ->
//                P = h + h*tanh(h), h = acc*c + c_bias (2 FFMA + 1 MUFU);
//                otherwise the exact integer bucket, positional bias and mask.
//                P (bf16) overwrites the first 16 columns of its S chunk.
//   warps 12..15 drain O (bf16) of the finished item while the next one runs
// TMEM columns: S0 [0,128) S1 [128,256) S2 [256,384) O [384,384+D)
// There is no softmax normaliser: SiLU partials are additive, so O simply
// accumulates in TMEM across kv tiles (no rescale).
#include "attn_common.cuh"

#ifndef JH_TRACE_CHUNKS
#define JH_TRACE_CHUNKS 0
#endif

namespace jh {

constexpr int kEpiWarps = 8;
constexpr int kFwdThreads = 128 + 32 * kEpiWarps + 128;
constexpr int kTsRing = 4;  // ts_k tile ring (deeper than the K ring)

template <int D>
struct FwdCfg {
  static constexpr int NS = (D == 64) ? 4 : 2;  // K / V stages
  static constexpr int PANELS = D / 64;         // 64-col swizzle panels
  static constexpr int TILE_BYTES = 128 * D * 2;
  static constexpr int Q_OFF = 0;
  static constexpr int K_OFF = 2 * TILE_BYTES;
  static constexpr int V_OFF = K_OFF + NS * TILE_BYTES;
  static constexpr int TSQ_OFF = V_OFF + NS * TILE_BYTES;     // int64 [2][kTsSlot]
  static constexpr int TSK_OFF = TSQ_OFF + 2 * kTsSlot * 8;   // int64 [kTsRing][kTsSlot]
  static constexpr int OCT_OFF = TSK_OFF + kTsRing * kTsSlot * 8;  // OctEntry [32]
  static constexpr int PW_OFF = OCT_OFF + 32 * 16;          // float pw[<=1024] x c1
  static constexpr int WT_OFF = PW_OFF + 1024 * 4;          // float [32] band weights x c1 (31: masked)
  static constexpr int KMAX_OFF = WT_OFF + 32 * 4;          // int64 [kTsRing][4] per-chunk max ts_k, then min
  static constexpr int BAR_OFF = KMAX_OFF + 2 * kTsRing * 32;  // mbarriers
  static constexpr int NBARS = 4 + 4 * NS + 3 * kTsRing + 8;
  static constexpr int TMEMPTR_OFF = BAR_OFF + NBARS * 8;
  static constexpr int RING_OFF = TMEMPTR_OFF + 16;  // work-item ring: full[], empty[], slot[]
  static constexpr int SMEM = RING_OFF + 2 * kItemRing * 8 + kItemRing * 4;
};

template <int D>
__global__ void __launch_bounds__(kFwdThreads, 1)
    hstu_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_tsq,
                    const __grid_constant__ CUtensorMap tm_tsk, const __grid_constant__ AttnParams p) {
  using C = FwdCfg<D>;
  constexpr int NS = C::NS;
  extern __shared__ __align__(1024) uint8_t smem[];
  int64_t* s_tsq = reinterpret_cast<int64_t*>(smem + C::TSQ_OFF);
  int64_t* s_tsk = reinterpret_cast<int64_t*>(smem + C::TSK_OFF);
  OctEntry* s_oct = reinterpret_cast<OctEntry*>(smem + C::OCT_OFF);
  float* s_pwc = reinterpret_cast<float*>(smem + C::PW_OFF);  // pos weights x c1
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* q_full = bars;                 // [2]  TMA Q + ts_q
  uint64_t* q_empty = bars + 2;            // [2]  last S MMA + epilogue read of ts_q
  uint64_t* k_full = bars + 4;             // [NS]
  uint64_t* k_empty = k_full + NS;         // [NS] S MMA done
  uint64_t* v_full = k_empty + NS;         // [NS]
  uint64_t* v_empty = v_full + NS;         // [NS] PV MMA done
  uint64_t* ts_full = v_empty + NS;        // [kTsRing]
  uint64_t* ts_empty = ts_full + kTsRing;  // [kTsRing] epilogue done with the tile
  uint64_t* tsx_full = bars + 4 + 4 * NS + 2 * kTsRing + 8;  // [kTsRing] chunk maxima ready
  int64_t* s_kmax = reinterpret_cast<int64_t*>(smem + C::KMAX_OFF);
  uint64_t* s_full = ts_empty + kTsRing;   // [3]
  uint64_t* p_full = s_full + 3;           // [3] P (over S) written
  uint64_t* o_full = p_full + 3;           // [1]
  uint64_t* o_empty = o_full + 1;          // [1] drain warps hold O in registers
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + C::TMEMPTR_OFF);
  const ItemRing ring{reinterpret_cast<int32_t*>(smem + C::RING_OFF + 2 * kItemRing * 8),
                      reinterpret_cast<uint64_t*>(smem + C::RING_OFF),
                      reinterpret_cast<uint64_t*>(smem + C::RING_OFF + kItemRing * 8)};

  const uint32_t warp = warp_id();
  const int tid = threadIdx.x;
  const int H = p.num_heads;
  const int nb = p.bias.nb;

  cta_stamp(p, 0, 2);
  if (smem_u32(smem) & 1023) __trap();  // 128B-swizzled operand tiles need 1 KB alignment
  const float c1 = p.c1;  // SiLU(s) = h + h*tanh(h), h = s/2 (scaled by 1/sqrt(d))
  oct_table_fill(s_oct, p.bias, p.ts_weights, c1, tid, blockDim.x);
  for (int i = tid; i < p.num_pos; i += blockDim.x) s_pwc[i] = p.pos_weights[i] * c1;
  float* s_wt = reinterpret_cast<float*>(smem + C::WT_OFF);
  if (tid < 32) s_wt[tid] = tid < nb ? p.ts_weights[tid] * c1 : (tid == (int)kBandMasked ? -1e30f : 0.f);
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1 + kEpiWarps);
    }
    for (int i = 0; i < 3; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 16 * kEpiWarps);  // one warpgroup
    }
    mbar_init(o_full, 1);
    mbar_init(o_empty, 128);  // drain warps
    for (int i = 0; i < NS; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < kTsRing; ++i) {
      mbar_init(&ts_full[i], 1);
      mbar_init(&ts_empty[i], kEpiWarps / 2);  // the owning warpgroup
      mbar_init(&tsx_full[i], 1);
    }
    ring_init(ring, 1 + 1 + kEpiWarps + 4);  // consumers: MMA, ts stats, epilogue warps, drain warps
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

  // (programmatic dependent launch: everything above overlapped the work-list build)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int n_items = p.wl.hdr->n_fwd;
  const int total = n_items * H;

  // The K/S stream runs two kv tiles ahead of the V/PV stream, continuously
  // across work items (a small ring carries the deferred tiles' coordinates).
#ifndef JH_FWD_LAG
#define JH_FWD_LAG 2
#endif
  constexpr int kLag = JH_FWD_LAG;
  if (warp == 0) {
    // ================= TMA producer: Q + ts_q per item, K + ts_k per tile, V two tiles later
    if (elect_one()) {
      uint32_t q_it = 0, k_it = 0, v_it = 0, tcnt = 0;
      int32_t pend_row[4], pend_col[4];  // deferred V tiles (row, head column)
      uint32_t n_pend = 0, pend_head = 0;
      auto load_v = [&]() {
        const int slot = pend_head & 3;
        const int st = v_it % NS;
        mbar_wait_idle(&v_empty[st], ((v_it / NS) & 1) ^ 1);
        trace_ev(p, 0, tcnt, 3, v_it);
        mbar_expect_tx(&v_full[st], C::TILE_BYTES);
        for (int pn = 0; pn < C::PANELS; ++pn)
          tma_load_2d(smem + C::V_OFF + st * C::TILE_BYTES + pn * 16384, &tm_v, pend_col[slot] + pn * 64,
                      pend_row[slot], &v_full[st]);
        ++v_it;
        ++pend_head;
        --n_pend;
      };
      // The next item's Q is issued right after this item's second K tile (its
      // buffer frees when the previous item's last S retires, which the K ring
      // has just waited for), so the Q load overlaps this item's tiles.
      uint32_t rk = 0;
      struct Item {
        int g, h, n;
        int2 it;
        Seg sg;
      };
      auto next_item = [&](Item& x) -> bool {
        while ((x.g = ring_produce(ring, rk, &p.wl.hdr->next_item[0], total)) >= 0) {
          x.it = p.wl.fwd[x.g / H];
          x.h = x.g % H;
          x.sg = load_seg(p.seg, x.it.x);
          x.n = (int)((fwd_kv_lim(x.sg, x.it.y) + kBN - 1) / kBN);
          if (x.n > 0) return true;  // (items without visible kv are skipped by every role)
        }
        return false;
      };
      auto load_q = [&](const Item& x) {
        const int qb = q_it & 1;
        mbar_wait_idle(&q_empty[qb], ((q_it >> 1) & 1) ^ 1);
        trace_ev(p, 0, tcnt, 1, x.g);
        mbar_expect_tx(&q_full[qb], C::TILE_BYTES + kTsBytes);
        const int32_t qrow = (int32_t)(x.sg.q_row0 + (int64_t)x.it.y * kBM);
        for (int pn = 0; pn < C::PANELS; ++pn)
          tma_load_2d(smem + C::Q_OFF + qb * C::TILE_BYTES + pn * 16384, &tm_q, x.h * D + pn * 64, qrow,
                      &q_full[qb]);
        tma_load_1d(s_tsq + qb * kTsSlot, &tm_tsq, qrow & ~1, &q_full[qb]);
        ++q_it;
      };
      Item cur, nxt;
      bool have = next_item(cur);
      if (have) load_q(cur);
      while (have) {
        const Seg& sg = cur.sg;
        const int h = cur.h, n = cur.n;
        bool have_next = false;
        for (int j = 0; j < n; ++j) {
          const int st = k_it % NS;
          const int ts = k_it % kTsRing;
          const int32_t krow = (int32_t)(sg.kv_row0 + (int64_t)j * kBN);
          mbar_wait_idle(&k_empty[st], ((k_it / NS) & 1) ^ 1);
          trace_ev(p, 0, tcnt, 2, j);
          mbar_expect_tx(&k_full[st], C::TILE_BYTES);
          for (int pn = 0; pn < C::PANELS; ++pn)
            tma_load_2d(smem + C::K_OFF + st * C::TILE_BYTES + pn * 16384, &tm_k, h * D + pn * 64, krow, &k_full[st]);
          mbar_wait(&ts_empty[ts], ((k_it / kTsRing) & 1) ^ 1);
          mbar_expect_tx(&ts_full[ts], kTsBytes);
          tma_load_1d(s_tsk + ts * kTsSlot, &tm_tsk, krow & ~1, &ts_full[ts]);
          ++k_it;
          const int slot = (pend_head + n_pend) & 3;
          pend_row[slot] = krow;
          pend_col[slot] = h * D;
          ++n_pend;
          if (n_pend > kLag) load_v();
          if (j == (n > 1 ? 1 : 0)) {
            have_next = next_item(nxt);
            if (have_next) load_q(nxt);
          }
        }
        have = have_next;
        cur = nxt;
      }
      while (n_pend) load_v();
    }
  } else if (warp == 1) {
    // ================= MMA issuer: S(t) then PV(t - 2), one continuous stream
    if (elect_one()) {
      constexpr uint32_t idesc_s = idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t idesc_pv = idesc_bf16(128, D, 0, 1);
      const uint32_t tO = tmem + 384;
      uint32_t q_it = 0, k_it = 0, v_it = 0, s_it = 0, o_it = 0, tcnt = 0;
      uint32_t pend_flags[4];  // bit0 first tile of its item, bit1 last tile
      uint32_t n_pend = 0, pend_head = 0, pv_it = 0;
      auto issue_pv = [&]() {
        const uint32_t sidx = pv_it;
        const uint32_t fl = pend_flags[pend_head & 3];
        const bool first = fl & 1u;
        const int pb = sidx % 3;
        const int st = v_it % NS;
        mbar_wait(&p_full[pb], (sidx / 3) & 1);
        trace_ev(p, 1, tcnt, 11, sidx);
        mbar_wait(&v_full[st], (v_it / NS) & 1);
        if (first) mbar_wait(o_empty, (o_it & 1) ^ 1);
        tc_fence_after();
        const uint32_t v_base = smem_u32(smem + C::V_OFF + st * C::TILE_BYTES);
        // A = P in TMEM: chunk c's 32 kv columns as bf16 pairs at [128 pb + 32c, +16)
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk)
          umma_ts(tO, tmem + 128 * pb + 32 * (kk >> 1) + 8 * (kk & 1), sdesc_sw128(v_base + kk * 2048, 16384, 1024),
                  idesc_pv, (first && kk == 0) ? 0u : 1u);
        umma_commit(&v_empty[st]);
        if (fl & 2u) {
          umma_commit(o_full);
          ++o_it;
        }
        ++v_it;
        ++pv_it;
        ++pend_head;
        --n_pend;
      };
      uint32_t rk = 0;
      for (int g; (g = ring_consume(ring, rk, false)) >= 0;) {
        const int2 it = p.wl.fwd[g / H];
        const Seg sg = load_seg(p.seg, it.x);
        const int n = (int)((fwd_kv_lim(sg, it.y) + kBN - 1) / kBN);
        if (n == 0) continue;
        const int qb = q_it & 1;
        mbar_wait(&q_full[qb], (q_it >> 1) & 1);
        tc_fence_after();
        const uint32_t q_base = smem_u32(smem + C::Q_OFF + qb * C::TILE_BYTES);
        for (int j = 0; j < n; ++j) {
          const int st = k_it % NS;
          const int sb = s_it % 3;  // buffer of tile s_it - 3, whose PV was issued before
          mbar_wait(&k_full[st], (k_it / NS) & 1);
          trace_ev(p, 1, tcnt, 10, s_it);
          tc_fence_after();
          const uint32_t k_base = smem_u32(smem + C::K_OFF + st * C::TILE_BYTES);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
            umma_ss(tmem + 128 * sb, sdesc_sw128(q_base + off, 16, 1024), sdesc_sw128(k_base + off, 16, 1024),
                    idesc_s, kk > 0 ? 1u : 0u);
          }
          umma_commit(&s_full[sb]);
          umma_commit(&k_empty[st]);
          if (j == n - 1) umma_commit(&q_empty[qb]);
          ++k_it;
          ++s_it;
          pend_flags[(pend_head + n_pend) & 3] = (j == 0 ? 1u : 0u) | (j == n - 1 ? 2u : 0u);
          ++n_pend;
          if (n_pend > kLag) issue_pv();
        }
        ++q_it;
      }
      while (n_pend) issue_pv();
    }
  } else if (warp == 3) {
    // ================= ts_k tile statistics: per 32-column chunk maximum
    // (used by the epilogue's warp-uniform saturation test)
    const int lane = lane_id();
    uint32_t t_it = 0;
    uint32_t rk = 0;
    for (int g; (g = ring_consume(ring, rk, true)) >= 0;) {
      const int2 it = p.wl.fwd[g / H];
      const Seg sg = load_seg(p.seg, it.x);
      const int n = (int)((fwd_kv_lim(sg, it.y) + kBN - 1) / kBN);
      for (int j = 0; j < n; ++j) {
        const int ts = t_it % kTsRing;
        mbar_wait(&ts_full[ts], (t_it / kTsRing) & 1);
        const int64_t* tsk = s_tsk + ts * kTsSlot + ((sg.kv_row0 + (int64_t)j * kBN) & 1);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int64_t m = warp_max_i64(tsk[32 * c + lane]);
          const int64_t mn = warp_min_i64(tsk[32 * c + lane]);
          if (lane == 0) {
            s_kmax[ts * 4 + c] = m;
            s_kmax[kTsRing * 4 + ts * 4 + c] = mn;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&tsx_full[ts]);
        ++t_it;
      }
    }
  } else if (warp >= 4 && warp < 12) {
    // ================= epilogue: warpgroup wg owns the tiles with s_it % 2 == wg;
    // thread = q row r, all 128 kv columns
    const int et = tid - 128;
    const int wg = et >> 7;
    const int r = et & 127;          // q row within the tile (= TMEM lane)
    const int lane = r & 31;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const int64_t cap = p.bias.cap;
    const int P = p.num_pos;
    const bool has_pos = P > 0;
    const bool use_band = p.band != nullptr;  // (the host turns it off with a positional bias)
    float cb = p.ts_weights[nb - 1];
    if (has_pos) cb += p.pos_weights[P - 1];
    cb *= c1;
    uint32_t q_it = 0, s_it = 0, tcnt = 0;
    const bool tr = (tid == 128 || tid == 256);
    const int trole = tid == 128 ? 3 : 4;
    uint32_t rk = 0;
    for (int g; (g = ring_consume(ring, rk, true)) >= 0;) {
      const int2 it = p.wl.fwd[g / H];
      const Seg sg = load_seg(p.seg, it.x);
      const int64_t kv_lim = fwd_kv_lim(sg, it.y);
      // debug export (tests): the bucket this thread applies to each visible pair (head 0)
      uint8_t* dbgb = (p.dbg_buckets != nullptr && g % H == 0 && r < sg.lq - (int64_t)it.y * kBM)
                          ? p.dbg_buckets + (sg.q_row0 + (int64_t)it.y * kBM + r) * p.dbg_ld
                          : nullptr;
      const int n = (int)((kv_lim + kBN - 1) / kBN);
      if (n == 0) continue;
      const int64_t nq = min((int64_t)kBM, sg.lq - (int64_t)it.y * kBM);
      const bool row_ok = r < nq;
      const int64_t qp_tile = sg.qp0 + (int64_t)it.y * kBM;
      const int64_t qpos = qp_tile + r;
      // this tile's query timestamps (TMA-staged with Q)
      const int qb = q_it & 1;
      mbar_wait(&q_full[qb], (q_it >> 1) & 1);
      const int64_t tq = row_ok ? s_tsq[qb * kTsSlot + ((sg.q_row0 + (int64_t)it.y * kBM) & 1) + r] : (INT64_MAX >> 2);
      __syncwarp();
      if (lane == 0) mbar_arrive(&q_empty[qb]);
      ++q_it;
      const int64_t tq_min = warp_min_i64(tq);
      const int64_t tq_max = warp_max_i64(row_ok ? tq : (INT64_MIN >> 2));  // over valid rows
      const int32_t tq32 = (int32_t)(uint32_t)(uint64_t)tq;
      const int64_t row_lo = qp_tile + (r & ~31), row_hi = row_lo + 31;  // warp's q positions
      // band table: this warp's q group and the byte row of this thread in it
      const int aq = it.y * 4 + (r >> 5);
      const int64_t bd = (sg.qp0 >> 5) + aq;
      const uint8_t* brow = use_band && 32 * aq < sg.lq ? band_chunk(p.band, band_group(sg, it.x, aq), 0) + lane * 32 : nullptr;
      for (int j = 0; j < n; ++j, ++s_it) {
        if ((int)(s_it & 1) != wg) continue;
        // band chunks of this tile (window and not entirely masked): prefetch the
        // byte rows of the two right-most ones (the diagonal-most) before any wait
        uint32_t cand = 0;
        // (a warp past the segment's rows has no q group; tiles whose 4 kv groups
        // [4j, 4j+3] miss the window [bd-3, bd+1] entirely skip the per-chunk test)
        if (use_band && 32 * aq < sg.lq && 4 * (int64_t)j + 3 >= bd - 3 && 4 * (int64_t)j <= bd + 1) {
          const int wi0 = (int)(4 * (int64_t)j - bd + 3);
          const int64_t lim = min(row_hi + 1, kv_lim);  // kv positions 32 b must stay below
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int wi = wi0 + c;
            if (wi >= 0 && wi < kBandNW && 32 * (4 * (int64_t)j + c) < lim) cand |= 1u << c;
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
        const int sb = s_it % 3;
        const int ts = s_it % kTsRing;
        const int64_t kv0 = (int64_t)j * kBN;
        mbar_wait(&tsx_full[ts], (s_it / kTsRing) & 1);  // chunk maxima (implies ts_full)
        mbar_wait(&s_full[sb], (s_it / 3) & 1);
        if (tr) trace_ev(p, trole, tcnt, 40, s_it);
        tc_fence_after();
        const int64_t* tsk = s_tsk + ts * kTsSlot + ((sg.kv_row0 + kv0) & 1);
        const uint32_t tS = tmem + 128 * sb + lane_off;
#pragma unroll 1
        for (int c0 = 0; c0 < kBN; c0 += 32) {
          // chunk class (warp-uniform): 0 all masked, 1 unmasked + saturated bias, 2 general
          const int64_t kc0 = kv0 + c0, kc1 = kc0 + 31;
          int cls = 0;  // every pair is in the future or past the segment
          if (!(kc0 > row_hi || kc0 >= kv_lim)) {
            cls = 2;
            if ((kc1 <= row_lo) && (kc1 < kv_lim) && (tq_min - s_kmax[ts * 4 + (c0 >> 5)] >= cap) &&
                (!has_pos || row_lo - kc1 >= P - 1))
              cls = 1;
            else if ((cand >> (c0 >> 5)) & 1u)
              cls = 4;  // band table chunk
          }
          if (cls == 4) {
            // exact bias from the band table: per element one byte -> weight
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
              // masked pairs: h = -1e30, tanh = -1 exactly, P = h - h = 0
              float p0, p1;
              silu_pair(h0, h1, p0, p1);
              pk[i >> 1] = pack_bf16(p0, p1);
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
              float p0, p1;
              silu_pair(h0, h1, p0, p1);
              pk[i >> 1] = pack_bf16(p0, p1);
            }
            tmem_st16(tS + c0, pk);  // P over the chunk's (consumed) S columns
          } else if (cls == 0) {
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = 0u;
            tmem_st16(tS + c0, pk);
          } else {
            // general chunk (diagonal / short time gaps): exact per-element
            // bucket, positional bias and mask, 8 columns per step
            const int relc = (int)(qpos - kv0 - c0);                        // qpos - kpos of column 0
            const int ncol = (int)min(kv_lim - kv0 - c0, (int64_t)32);      // in-range columns
            // all deltas of the chunk fit in 32 bits (warp-uniform): exact low-word arithmetic
            const bool fits32 = cap < 0x7FFFFFFFll && tq_max - s_kmax[kTsRing * 4 + ts * 4 + (c0 >> 5)] < 0x7FFFFFFFll &&
                                tq_min - s_kmax[ts * 4 + (c0 >> 5)] > -0x7FFFFFFFll;
            const int32_t* tsk32 = reinterpret_cast<const int32_t*>(tsk + c0);
            uint32_t vn[8];
            tmem_ld8(tS + c0, vn);  // the next 8 columns' load stays in flight during each step
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
                for (int i = 0; i < 8; ++i) bc[i] = cb;  // every visible pair saturated (warp-uniform)
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
              tmem_st4(tS + c0 + (g8 >> 1), pk);  // S columns c0 .. c0+g8+7 were already read
            }
          }
#if JH_TRACE_CHUNKS
          if (tr) trace_ev(p, trole, tcnt, 50 + cls, c0);
#endif
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&p_full[sb]);
        if (tr) trace_ev(p, trole, tcnt, 41, s_it);
        __syncwarp();
        if (lane == 0) mbar_arrive(&ts_empty[ts]);
      }
    }
  } else if (warp >= 12) {
    // ================= O drain: TMEM -> bf16 -> global (thread = q row)
    const int r = tid - 384;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    uint32_t o_it = 0;
    uint32_t rk = 0;
    const uint64_t pol_out = l2_policy_evict_first();  // results nothing in this step re-reads
    for (int g; (g = ring_consume(ring, rk, true)) >= 0;) {
      const int2 it = p.wl.fwd[g / H];
      const int h = g % H;
      const Seg sg = load_seg(p.seg, it.x);
      const int n = (int)((fwd_kv_lim(sg, it.y) + kBN - 1) / kBN);
      const int64_t nq = min((int64_t)kBM, sg.lq - (int64_t)it.y * kBM);
      const bool row_ok = r < nq;
      const int64_t orow_i = (sg.q_row0 + (int64_t)it.y * kBM + r) * p.ld_o + h * D;
      __nv_bfloat16* orow = p.out + orow_i;
      if (n == 0) {
        if (row_ok && p.out_acc == nullptr)
          for (int c = 0; c < D; c += 8) *reinterpret_cast<int4*>(orow + c) = make_int4(0, 0, 0, 0);
        else if (row_ok && !p.out_acc_add)
          for (int c = 0; c < D; c += 4) *reinterpret_cast<float4*>(p.out_acc + orow_i + c) = make_float4(0, 0, 0, 0);
        continue;
      }
      mbar_wait_idle(o_full, o_it & 1);
      ++o_it;
      tc_fence_after();
      if (p.out_acc != nullptr) {
        // fp32 partial (CP): store or add, 32 columns at a time; O is released
        // after the last TMEM load
        float4* arow = reinterpret_cast<float4*>(p.out_acc + orow_i);
#pragma unroll 1
        for (int c0 = 0; c0 < D; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(tmem + 384 + lane_off + c0, v);
          tmem_ld_wait();
          if (c0 + 32 == D) {
            tc_fence_before();
            mbar_arrive(o_empty);
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
      // O -> bf16 registers first, release the accumulator, then store
      uint32_t pk[D / 2];
#pragma unroll
      for (int c0 = 0; c0 < D; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + 384 + lane_off + c0, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; i += 2) pk[(c0 + i) >> 1] = pack_bf16(__uint_as_float(v[i]), __uint_as_float(v[i + 1]));
      }
      tc_fence_before();
      mbar_arrive(o_empty);
      if (row_ok) {
        int4* dst = reinterpret_cast<int4*>(orow);
#pragma unroll
        for (int i = 0; i < D / 8; ++i)
          st_global_v4_hint(dst + i, pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3], pol_out);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cta_stamp(p, 1, 2);
  if (warp == 2) tmem_dealloc(tmem, 512);
}

template <int D>
int launch_fwd(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, const CUtensorMap& ttq,
               const CUtensorMap& ttk, const AttnParams& p, int grid, cudaStream_t s, void* ev0, void* ev1) {
  using C = FwdCfg<D>;
  static_assert(C::SMEM <= 232448, "fwd smem budget");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(hstu_fwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    cudaFuncSetAttribute(hstu_fwd_kernel<D>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    attr = true;
  }
  if (ev0) cudaEventRecord((cudaEvent_t)ev0, s);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kFwdThreads);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  la[0].val.programmaticStreamSerializationAllowed = 1;  // prologue overlaps the work-list build
  cfg.attrs = la;
  cfg.numAttrs = 1;
  if (cudaError_t e = cudaLaunchKernelEx(&cfg, hstu_fwd_kernel<D>, tq, tk, tv, ttq, ttk, p)) return (int)e;
  if (ev1) cudaEventRecord((cudaEvent_t)ev1, s);
  return (int)cudaGetLastError();
}

template int launch_fwd<64>(const CUtensorMap&, const CUtensorMap&, const CUtensorMap&, const CUtensorMap&,
                            const CUtensorMap&, const AttnParams&, int, cudaStream_t, void*, void*);
template int launch_fwd<128>(const CUtensorMap&, const CUtensorMap&, const CUtensorMap&, const CUtensorMap&,
                             const CUtensorMap&, const AttnParams&, int, cudaStream_t, void*, void*);

}  // namespace jh
