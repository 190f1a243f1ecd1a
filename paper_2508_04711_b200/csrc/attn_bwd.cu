// Fused jagged HSTU attention backward for sm_100a: two deterministic kernels.
//
// Reference: attention.py:187-234 hstu_attention_backward
//   dV = A^T g;  dS = (g V^T) . sigma(S) (1 + S (1 - sigma(S)))  (masked)
//   dQ = dS K / sqrt(d);  dK = dS^T Q / sqrt(d);  d_w = bincount(bucket, dS / sqrt(d))
// with A = tril . SiLU(S), S = (Q K^T + bias) / sqrt(d).
//
// (1) hstu_bwd_dkv_kernel -- kv-tile-major: a work item is (segment, 128-row
//     kv tile) x head; it loops over the q tiles that can see the kv tile.
//       warp 0      TMA: K_j, V_j per item; Q_i, dO_i, ts_q per q tile (2 stages)
//       warp 1      MMA: S^T = K Q^T, dP^T = V dO^T, dV += P^T dO (A = P^T in
//                   TMEM), dK += dS^T Q (A = dS^T in smem)
//       warp 2      TMEM allocator; warp 3: per-chunk min of ts_q (saturation test)
//       warps 4-11  compute, thread = (kv row, 64-q-column half):
//                   phase P  : S^T -> P^T (TMEM) and SiLU'(S) (f16, TMEM)
//                   phase dS : dP^T -> dS^T = dP SiLU'(S)/sqrt(d) (smem), d_ts_weights
//       warps 12-15 drain dK / dV (bf16 store, or fp32 accumulate for CP)
//     TMEM: S^T [0,128) -- per column group g: P^T at [64g,64g+32), SiLU' at
//           [64g+32,64g+64) | dP^T [128,256) | dV | dK
// (2) hstu_bwd_dq_kernel -- q-tile-major (the forward's work list): loops over
//     the kv tiles the q tile sees; dQ accumulates in TMEM and is written once.
//       warp 0 TMA (Q, dO, ts_q once; K + ts_k double, V single buffered)
//       warp 1 MMA: S = Q K^T (2 TMEM buffers), dP = dO V^T, dQ += dS K
//       warp 3 per-chunk max of ts_k; warps 4-11 compute dS (smem) and write dQ.
// No atomics on the gradient tensors: every dQ / dK / dV row is written by
// exactly one CTA; d_ts_weights reduces per-CTA partials with fp64 atomics.
#include <algorithm>

#include "abi_internal.h"
#include "attn_common.cuh"

namespace jh {

constexpr int kBwdThreads = 512;  // dKV kernel
constexpr int kDqThreads = 384;   // dQ kernel
constexpr int kCompWarps = 8;

// ===================================================================== dKV
template <int D>
struct DkvCfg {
  static constexpr int TILE = 128 * D * 2;
  static constexpr int PANELS = D / 64;
  static constexpr int K_OFF = 0;
  static constexpr int V_OFF = TILE;
  static constexpr int Q_OFF = 2 * TILE;          // [2] stages
  static constexpr int DO_OFF = 4 * TILE;         // [2] stages
  static constexpr int DS_OFF = 6 * TILE;         // dS^T: 128 kv x 128 q bf16 (2 panels)
  static constexpr int TSQ_OFF = DS_OFF + 32768;  // int64 [2][kTsSlot]
  static constexpr int MAX_NB = (D == 64) ? 256 : 32;
  static constexpr int W_OFF = TSQ_OFF + 2 * kTsSlot * 8;           // float [MAX_NB]
  static constexpr int PW_OFF = W_OFF + MAX_NB * 4;                 // float [1024] (D=64 only)
  static constexpr int BINS_OFF = PW_OFF + (D == 64 ? 4096 : 0);    // float [MAX_NB (+1024)]
  static constexpr int NBINS = MAX_NB + (D == 64 ? 1024 : 0);
  static constexpr int TAB_OFF = BINS_OFF + NBINS * 4;              // SmemBias (160 B)
  static constexpr int QMIN_OFF = TAB_OFF + 160;                    // int64 [2][4]
  static constexpr int BAR_OFF = QMIN_OFF + 64;
  static constexpr int NBARS = 16;
  static constexpr int TMEMPTR_OFF = BAR_OFF + NBARS * 8;
  static constexpr int SMEM = TMEMPTR_OFF + 16;
};

template <int D>
__global__ void __launch_bounds__(kBwdThreads, 1)
    hstu_bwd_dkv_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                        const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
                        const __grid_constant__ CUtensorMap tm_tsq, const __grid_constant__ AttnParams p) {
  using C = DkvCfg<D>;
  extern __shared__ __align__(1024) uint8_t smem[];
  int64_t* s_tsq = reinterpret_cast<int64_t*>(smem + C::TSQ_OFF);
  float* s_w = reinterpret_cast<float*>(smem + C::W_OFF);
  float* s_pw = reinterpret_cast<float*>(smem + C::PW_OFF);
  float* s_bins = reinterpret_cast<float*>(smem + C::BINS_OFF);  // non-last buckets, then positions
  SmemBias* s_bias = reinterpret_cast<SmemBias*>(smem + C::TAB_OFF);
  int64_t* s_qmin = reinterpret_cast<int64_t*>(smem + C::QMIN_OFF);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* kv_full = bars + 0;
  uint64_t* kv_empty = bars + 1;
  uint64_t* qd_full = bars + 2;    // [2]
  uint64_t* qd_empty = bars + 4;   // [2] MMA (dK_i) + compute warps
  uint64_t* qx_full = bars + 6;    // [2] chunk minima of ts_q
  uint64_t* s_full = bars + 8;
  uint64_t* dp_full = bars + 9;
  uint64_t* p_full = bars + 10;    // P^T + SiLU' in TMEM, S^T consumed
  uint64_t* ds_full = bars + 11;   // dS^T in smem; dP^T, SiLU' consumed
  uint64_t* ds_empty = bars + 12;  // dK_i done with dS^T
  uint64_t* dkv_full = bars + 13;
  uint64_t* dkv_empty = bars + 14;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + C::TMEMPTR_OFF);

  const uint32_t warp = warp_id();
  const int tid = threadIdx.x;
  const int H = p.num_heads;
  const int nb = p.bias.nb;
  const int P = p.num_pos;
  const bool has_pos = P > 0;
  const int64_t HD = (int64_t)H * D;

  if (smem_u32(smem) & 1023) __trap();
  for (int i = tid; i < nb; i += blockDim.x) s_w[i] = p.ts_weights[i];
  if (D == 64)
    for (int i = tid; i < P; i += blockDim.x) s_pw[i] = p.pos_weights[i];
  for (int i = tid; i < C::NBINS; i += blockDim.x) s_bins[i] = 0.f;
  smem_bias_fill(s_bias, p.bias, tid, blockDim.x);
  if (tid == 0) {
    mbar_init(kv_full, 1);
    mbar_init(kv_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&qd_full[i], 1);
      mbar_init(&qd_empty[i], 1 + kCompWarps);
      mbar_init(&qx_full[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(dp_full, 1);
    mbar_init(p_full, 32 * kCompWarps);
    mbar_init(ds_full, 32 * kCompWarps);
    mbar_init(ds_empty, 1);
    mbar_init(dkv_full, 1);
    mbar_init(dkv_empty, 128);
    fence_barrier_init();
  }
  if (warp == 0 && lane_id() == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    tma_prefetch_desc(&tm_do);
    tma_prefetch_desc(&tm_tsq);
  }
  if (warp == 2) tmem_alloc(s_tmem, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  const uint32_t tS = tmem, tDP = tmem + 128, tDV = tmem + 256, tDK = tmem + 256 + D;

  const int total = p.wl.hdr->n_bwd * H;
  auto q_tiles = [&](const Seg& sg, int j, int& t0, int& nt) {
    nt = (int)((sg.lq + kBM - 1) / kBM);
    int64_t first = (int64_t)j * kBN - sg.qp0;
    first = first < 0 ? 0 : first;
    t0 = (int)(first / kBM);
    if ((int64_t)j * kBN >= seg_kv_vis(sg)) t0 = nt;  // kv tile no query can see
  };

  if (warp == 0) {
    // ================= TMA producer
    if (elect_one()) {
      uint32_t it_cnt = 0, qd_it = 0, tcnt = 0;
      for (int g = blockIdx.x; g < total; g += gridDim.x) {
        const int2 it = p.wl.bwd[g / H];
        const int h = g % H;
        const Seg sg = load_seg(p.seg, it.x);
        int t0, nt;
        q_tiles(sg, it.y, t0, nt);
        if (t0 >= nt) continue;
        mbar_wait(kv_empty, (it_cnt & 1) ^ 1);
        trace_ev(p, 0, tcnt, 1, g);
        mbar_expect_tx(kv_full, 2 * C::TILE);
        const int32_t krow = (int32_t)(sg.kv_row0 + (int64_t)it.y * kBN);
        for (int pn = 0; pn < C::PANELS; ++pn) {
          tma_load_2d(smem + C::K_OFF + pn * 16384, &tm_k, h * D + pn * 64, krow, kv_full);
          tma_load_2d(smem + C::V_OFF + pn * 16384, &tm_v, h * D + pn * 64, krow, kv_full);
        }
        ++it_cnt;
        for (int t = t0; t < nt; ++t) {
          const int st = qd_it & 1;
          mbar_wait(&qd_empty[st], ((qd_it >> 1) & 1) ^ 1);
          trace_ev(p, 0, tcnt, 2, t);
          mbar_expect_tx(&qd_full[st], 2 * C::TILE + kTsBytes);
          const int32_t qrow = (int32_t)(sg.q_row0 + (int64_t)t * kBM);
          for (int pn = 0; pn < C::PANELS; ++pn) {
            tma_load_2d(smem + C::Q_OFF + st * C::TILE + pn * 16384, &tm_q, h * D + pn * 64, qrow, &qd_full[st]);
            tma_load_2d(smem + C::DO_OFF + st * C::TILE + pn * 16384, &tm_do, h * D + pn * 64, qrow,
                        &qd_full[st]);
          }
          tma_load_1d(s_tsq + st * kTsSlot, &tm_tsq, qrow & ~1, &qd_full[st]);
          ++qd_it;
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer
    if (elect_one()) {
      constexpr uint32_t id_s = idesc_bf16(128, 128, 0, 0);  // S^T, dP^T
      constexpr uint32_t id_kv = idesc_bf16(128, D, 0, 1);   // dV (A tmem), dK (A smem K-major)
      const uint32_t k_base = smem_u32(smem + C::K_OFF);
      const uint32_t v_base = smem_u32(smem + C::V_OFF);
      const uint32_t ds_base = smem_u32(smem + C::DS_OFF);
      uint32_t it_cnt = 0, qd_it = 0, p_cnt = 0, ds_cnt = 0, tcnt = 0;
      auto q_base = [&](uint32_t qi) { return smem_u32(smem + C::Q_OFF + (qi & 1) * C::TILE); };
      auto do_base = [&](uint32_t qi) { return smem_u32(smem + C::DO_OFF + (qi & 1) * C::TILE); };
      auto issue_S_dP = [&](uint32_t qi) {
        mbar_wait(&qd_full[qi & 1], (qi >> 1) & 1);
        trace_ev(p, 1, tcnt, 10, qi);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          umma_ss(tS, sdesc_sw128(k_base + off, 16, 1024), sdesc_sw128(q_base(qi) + off, 16, 1024), id_s,
                  kk > 0 ? 1u : 0u);
        }
        umma_commit(s_full);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          umma_ss(tDP, sdesc_sw128(v_base + off, 16, 1024), sdesc_sw128(do_base(qi) + off, 16, 1024), id_s,
                  kk > 0 ? 1u : 0u);
        }
        umma_commit(dp_full);
      };
      for (int g = blockIdx.x; g < total; g += gridDim.x) {
        const int2 it = p.wl.bwd[g / H];
        const Seg sg = load_seg(p.seg, it.x);
        int t0, nt;
        q_tiles(sg, it.y, t0, nt);
        if (t0 >= nt) continue;
        const int n = nt - t0;
        mbar_wait(kv_full, it_cnt & 1);
        issue_S_dP(qd_it);
        for (int i = 0; i < n; ++i) {
          const uint32_t qi = qd_it + i;
          // dV += P^T dO.  P^T of q columns [32c, 32c+32) (chunk c) sits at TMEM
          // columns [32c, 32c+16) of the S^T region (SiLU' in the other half)
          mbar_wait(p_full, p_cnt & 1);
          trace_ev(p, 1, tcnt, 12, qi);
          ++p_cnt;
          if (i == 0) mbar_wait(dkv_empty, (it_cnt & 1) ^ 1);  // dK/dV of the previous item drained
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < kBM / 16; ++kk)
            umma_ts(tDV, tS + 32 * (kk >> 1) + 8 * (kk & 1), sdesc_sw128(do_base(qi) + kk * 2048, 16384, 1024), id_kv,
                    (kk > 0 || i > 0) ? 1u : 0u);
          // dK += dS^T Q
          mbar_wait(ds_full, ds_cnt & 1);
          trace_ev(p, 1, tcnt, 13, qi);
          ++ds_cnt;
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < kBM / 16; ++kk) {
            const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
            umma_ss(tDK, sdesc_sw128(ds_base + off, 16, 1024), sdesc_sw128(q_base(qi) + kk * 2048, 16384, 1024),
                    id_kv, (kk > 0 || i > 0) ? 1u : 0u);
          }
          umma_commit(ds_empty);
          umma_commit(&qd_empty[qi & 1]);
          // next tile's S^T / dP^T (S^T region: P^T read by dV in issue order; SiLU' consumed)
          if (i + 1 < n) issue_S_dP(qi + 1);
        }
        qd_it += n;
        umma_commit(dkv_full);
        umma_commit(kv_empty);
        trace_ev(p, 1, tcnt, 15, g);
        ++it_cnt;
      }
    }
  } else if (warp == 3) {
    // ================= ts_q statistics: per 32-column chunk minimum
    const int lane = lane_id();
    uint32_t qd_it = 0;
    for (int g = blockIdx.x; g < total; g += gridDim.x) {
      const int2 it = p.wl.bwd[g / H];
      const Seg sg = load_seg(p.seg, it.x);
      int t0, nt;
      q_tiles(sg, it.y, t0, nt);
      for (int t = t0; t < nt; ++t) {
        const int st = qd_it & 1;
        mbar_wait(&qd_full[st], (qd_it >> 1) & 1);
        const int64_t* tsq = s_tsq + st * kTsSlot + ((sg.q_row0 + (int64_t)t * kBM) & 1);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int64_t m = warp_min_i64(tsq[32 * c + lane]);
          if (lane == 0) s_qmin[st * 4 + c] = m;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&qx_full[st]);
        ++qd_it;
      }
    }
  } else if (warp >= 4 && warp < 12) {
    // ================= compute: thread = (kv row r, q-column half wg)
    const int et = tid - 128;
    const int wg = et >> 7;
    const int r = et & 127;
    const int lane = r & 31;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t tSg = tS + lane_off + 64 * wg;  // this group's S^T / P^T / SiLU' columns
    const float c1 = 0.5f * rsqrtf((float)D);
    const int64_t cap = p.bias.cap;
    uint8_t* ds_smem = smem + C::DS_OFF + wg * 16384;  // this group's 64 q columns = one panel
    float cb = s_w[nb - 1];
    if (has_pos) cb += s_pw[P - 1];
    cb *= c1;
    double acc_w = 0.0, acc_p = 0.0;  // last-bucket partials
    uint32_t qd_it = 0, s_cnt = 0, dp_cnt = 0, ds_cnt = 0, tcnt = 0;
    const bool tr = (tid == 128);
    for (int g = blockIdx.x; g < total; g += gridDim.x) {
      const int2 it = p.wl.bwd[g / H];
      const Seg sg = load_seg(p.seg, it.x);
      int t0, nt;
      q_tiles(sg, it.y, t0, nt);
      if (t0 >= nt) continue;
      const int64_t kv0 = (int64_t)it.y * kBN;
      const int64_t kpos = kv0 + r;
      const bool krow_ok = kpos < sg.kv_len;
      const int64_t tk = krow_ok ? p.ts_k[sg.kv_row0 + kpos] : (INT64_MIN >> 2);
      const int64_t tk_max = warp_max_i64(tk);
      const int64_t k_lo = kv0 + (r & ~31), k_hi = k_lo + 31;  // this warp's kv positions
      const bool warp_k_ok = k_hi < sg.kv_len;
      for (int t = t0; t < nt; ++t) {
        const int st = qd_it & 1;
        const int64_t qrow0 = sg.q_row0 + (int64_t)t * kBM;
        const int64_t qp_tile = sg.qp0 + (int64_t)t * kBM;
        const int nq = (int)min((int64_t)kBM, sg.lq - (int64_t)t * kBM);
        mbar_wait(&qx_full[st], (qd_it >> 1) & 1);
        const int64_t* tsq = s_tsq + st * kTsSlot + (qrow0 & 1);
        int cls_bits = 0;  // per chunk: 0 masked, 1 saturated, 2 general
#pragma unroll
        for (int ci = 0; ci < 2; ++ci) {
          const int c0 = 64 * wg + 32 * ci;
          const int64_t qc0 = qp_tile + c0;
          int cls = 0;
          if (!(qc0 + 31 < k_lo || c0 >= nq)) {
            cls = 2;
            if ((qc0 >= k_hi) && (c0 + 32 <= nq) && warp_k_ok &&
                (s_qmin[st * 4 + (c0 >> 5)] - tk_max >= cap) && (!has_pos || qc0 - k_hi >= P - 1))
              cls = 1;
          }
          cls_bits |= cls << (2 * ci);
        }
        // ---------------- phase P: S^T -> P^T, SiLU'
        mbar_wait(s_full, s_cnt & 1);
        if (tr) trace_ev(p, 2, tcnt, 21, t);
        ++s_cnt;
        tc_fence_after();
        // per chunk (32 S^T columns at cbase): P^T -> [cbase, cbase+16), SiLU' -> [cbase+16, cbase+32),
        // i.e. each chunk is overwritten in place, only after all of its S^T values were read
#pragma unroll 1
        for (int ci = 0; ci < 2; ++ci) {
          const int cls = (cls_bits >> (2 * ci)) & 3;
          const int c0 = 64 * wg + 32 * ci;
          const uint32_t cbase = tSg + 32 * ci;
          if (cls == 1) {
            uint32_t v[32], pk[16], kp[16];
            tmem_ld32(cbase, v);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              const float h0 = fmaf(__uint_as_float(v[i]), c1, cb);
              const float h1 = fmaf(__uint_as_float(v[i + 1]), c1, cb);
              const float2 th = make_float2(tanh_approx(h0), tanh_approx(h1));  // f32: d_ts_weights accuracy
              pk[i >> 1] = pack_bf16(fmaf(h0, th.x, h0), fmaf(h1, th.y, h1));
              __half2 hk = __floats2half2_rn((1.f + th.x) * (fmaf(-h0, th.x, h0) + 1.f),
                                             (1.f + th.y) * (fmaf(-h1, th.y, h1) + 1.f));
              kp[i >> 1] = *reinterpret_cast<uint32_t*>(&hk);
            }
            tmem_st16(cbase, pk);
            tmem_st16(cbase + 16, kp);
          } else if (cls == 0) {
            uint32_t z[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) z[i] = 0u;
            tmem_st16(cbase, z);
            tmem_st16(cbase + 16, z);
          } else {
            // general chunk: 8 columns per step; P^T words land on columns already
            // read, SiLU' words wait in a small local buffer until all 32 are read
            uint32_t kl[16];
#pragma unroll 1
            for (int g8 = 0; g8 < 32; g8 += 8) {
              uint32_t v[8], pk[4];
              tmem_ld8(cbase + g8, v);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 8; i += 2) {
                float pp[2], dd[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                  const int qi = c0 + g8 + i + u;
                  const int64_t qpos = qp_tile + qi;
                  const bool ok = krow_ok && (qi < nq) && (kpos <= qpos);
                  float bias = s_w[bucket_smem(tsq[qi] - tk, s_bias, cap)];
                  if (has_pos) {
                    const int64_t rr = qpos - kpos;
                    bias += s_pw[rr < 0 ? 0 : (rr > P - 1 ? P - 1 : (int)rr)];
                  }
                  const float hh = (__uint_as_float(v[i + u]) + bias) * c1;
                  const float th = tanh_approx(hh);
                  pp[u] = ok ? fmaf(hh, th, hh) : 0.f;
                  dd[u] = ok ? (1.f + th) * (fmaf(-hh, th, hh) + 1.f) : 0.f;
                }
                pk[i >> 1] = pack_bf16(pp[0], pp[1]);
                __half2 hk = __floats2half2_rn(dd[0], dd[1]);
                kl[(g8 + i) >> 1] = *reinterpret_cast<uint32_t*>(&hk);
              }
              tmem_st4(cbase + (g8 >> 1), pk);
            }
            uint32_t kp[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) kp[i] = kl[i];
            tmem_st16(cbase + 16, kp);
          }
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(p_full);
        if (tr) trace_ev(p, 2, tcnt, 22, t);
        // ---------------- phase dS: dP^T, SiLU' -> dS^T (smem), d_ts_weights
        mbar_wait(dp_full, dp_cnt & 1);
        ++dp_cnt;
        if (ds_cnt > 0) mbar_wait(ds_empty, (ds_cnt - 1) & 1);  // dK of the previous tile done with dS^T
        ++ds_cnt;
        if (tr) trace_ev(p, 2, tcnt, 24, t);
        tc_fence_after();
        float sat_w = 0.f, sat_p = 0.f;
#pragma unroll 1
        for (int ci = 0; ci < 2; ++ci) {
          const int c0 = 64 * wg + 32 * ci;
          const int cls = (cls_bits >> (2 * ci)) & 3;
          const uint32_t cbase = tSg + 32 * ci;
          if (cls == 1) {
            uint32_t dv[32], kp[16], dk[16];
            tmem_ld32(tDP + lane_off + c0, dv);
            tmem_ld16(cbase + 16, kp);
            tmem_ld_wait();
            float csum = 0.f;
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              const float2 kd = __half22float2(*reinterpret_cast<const __half2*>(&kp[i >> 1]));
              const float d0 = __uint_as_float(dv[i]) * kd.x * c1;
              const float d1 = __uint_as_float(dv[i + 1]) * kd.y * c1;
              dk[i >> 1] = pack_bf16(d0, d1);
              csum += d0 + d1;
            }
            sat_w += csum;
            if (has_pos) sat_p += csum;  // saturated chunks hit both last buckets
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4)
              *reinterpret_cast<int4*>(ds_smem + sw128_offset(r, (c0 & 63) + q4 * 8)) =
                  make_int4(dk[4 * q4], dk[4 * q4 + 1], dk[4 * q4 + 2], dk[4 * q4 + 3]);
          } else if (cls == 0) {
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4)
              *reinterpret_cast<int4*>(ds_smem + sw128_offset(r, (c0 & 63) + q4 * 8)) = make_int4(0, 0, 0, 0);
          } else {
            // general chunk, 8 columns per step: exact bucket scatter into the bins
#pragma unroll 1
            for (int g8 = 0; g8 < 32; g8 += 8) {
              uint32_t dv[8], kp[4], dk[4];
              tmem_ld8(tDP + lane_off + c0 + g8, dv);
              tmem_ld4(cbase + 16 + (g8 >> 1), kp);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 8; i += 2) {
                const float2 kd = __half22float2(*reinterpret_cast<const __half2*>(&kp[i >> 1]));
                float dd[2] = {__uint_as_float(dv[i]) * kd.x * c1, __uint_as_float(dv[i + 1]) * kd.y * c1};
                dk[i >> 1] = pack_bf16(dd[0], dd[1]);
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                  const int qi = c0 + g8 + i + u;
                  const int64_t qpos = qp_tile + qi;
                  if (krow_ok && qi < nq && kpos <= qpos) {
                    const int b = bucket_smem(tsq[qi] - tk, s_bias, cap);
                    if (b == nb - 1)
                      sat_w += dd[u];
                    else
                      atomicAdd(&s_bins[b], dd[u]);
                    if (has_pos) {
                      const int64_t rr = qpos - kpos;
                      const int rel = rr > P - 1 ? P - 1 : (int)rr;
                      if (rel == P - 1)
                        sat_p += dd[u];
                      else
                        atomicAdd(&s_bins[C::MAX_NB + rel], dd[u]);
                    }
                  }
                }
              }
              *reinterpret_cast<int4*>(ds_smem + sw128_offset(r, (c0 & 63) + g8)) =
                  make_int4(dk[0], dk[1], dk[2], dk[3]);
            }
          }
        }
        acc_w += (double)sat_w;
        acc_p += (double)sat_p;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc_fence_before();
        mbar_arrive(ds_full);
        if (tr) trace_ev(p, 2, tcnt, 25, t);
        __syncwarp();
        if (lane == 0) mbar_arrive(&qd_empty[st]);  // done with this stage's ts_q
        ++qd_it;
      }
    }
    // ---- d_ts_weights / d_pos: last buckets as fp64 partials, the rest from smem bins
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      acc_w += __shfl_xor_sync(0xffffffffu, acc_w, o);
      acc_p += __shfl_xor_sync(0xffffffffu, acc_p, o);
    }
    if (lane == 0) {
      if (acc_w != 0.0) atomicAdd(&p.d_ts_weights[nb - 1], acc_w);
      if (has_pos && acc_p != 0.0) atomicAdd(&p.d_pos_weights[P - 1], acc_p);
    }
    named_bar_sync(1, 32 * kCompWarps);
    for (int i = et; i < nb; i += 32 * kCompWarps)
      if (s_bins[i] != 0.f) atomicAdd(&p.d_ts_weights[i], (double)s_bins[i]);
    if (has_pos)
      for (int i = et; i < P; i += 32 * kCompWarps)
        if (s_bins[C::MAX_NB + i] != 0.f) atomicAdd(&p.d_pos_weights[i], (double)s_bins[C::MAX_NB + i]);
  } else if (warp >= 12) {
    // ================= dK / dV drain (thread = kv row)
    const int r = tid - 384;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    uint32_t it_cnt = 0;
    for (int g = blockIdx.x; g < total; g += gridDim.x) {
      const int2 it = p.wl.bwd[g / H];
      const int h = g % H;
      const Seg sg = load_seg(p.seg, it.x);
      int t0, nt;
      q_tiles(sg, it.y, t0, nt);
      const int64_t kpos = (int64_t)it.y * kBN + r;
      const bool krow_ok = kpos < sg.kv_len;
      const int64_t krow = sg.kv_row0 + kpos;
      if (t0 >= nt) {
        // no query sees this kv tile: its dK/dV rows are zero
        if (krow_ok && !p.dk_accum)
          for (int c = 0; c < D; c += 8) {
            *reinterpret_cast<int4*>(p.dk + krow * p.ld_dk + h * D + c) = make_int4(0, 0, 0, 0);
            *reinterpret_cast<int4*>(p.dv + krow * p.ld_dv + h * D + c) = make_int4(0, 0, 0, 0);
          }
        continue;
      }
      mbar_wait(dkv_full, it_cnt & 1);
      ++it_cnt;
      tc_fence_after();
#pragma unroll 1
      for (int part = 0; part < 2; ++part) {
        const uint32_t tsrc = part ? tDK : tDV;
        float* acc = part ? p.dk_accum : p.dv_accum;
#pragma unroll 1
        for (int c0 = 0; c0 < D; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(tsrc + lane_off + c0, v);
          tmem_ld_wait();
          if (!krow_ok) continue;
          if (acc) {
            float* dst = acc + krow * HD + h * D + c0;
#pragma unroll
            for (int i = 0; i < 32; i += 4)
              asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + i), "f"(__uint_as_float(v[i])),
                           "f"(__uint_as_float(v[i + 1])), "f"(__uint_as_float(v[i + 2])),
                           "f"(__uint_as_float(v[i + 3]))
                           : "memory");
          } else {
            __nv_bfloat16* dst = (part ? (p.dk + krow * p.ld_dk) : (p.dv + krow * p.ld_dv)) + h * D + c0;
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 32; i += 2) pk[i >> 1] = pack_bf16(__uint_as_float(v[i]), __uint_as_float(v[i + 1]));
            int4* d4 = reinterpret_cast<int4*>(dst);
#pragma unroll
            for (int i = 0; i < 4; ++i) d4[i] = make_int4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(dkv_empty);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

// ====================================================================== dQ
template <int D>
struct DqCfg {
  static constexpr int TILE = 128 * D * 2;
  static constexpr int PANELS = D / 64;
  static constexpr int Q_OFF = 0;
  static constexpr int DO_OFF = TILE;
  static constexpr int K_OFF = 2 * TILE;                  // [2] stages
  static constexpr int V_OFF = 4 * TILE;                  // [1]
  static constexpr int DS_OFF = 5 * TILE;                 // dS: 128 q x 128 kv bf16 (2 panels)
  static constexpr int TSQ_OFF = DS_OFF + 32768;          // int64 [kTsSlot]
  static constexpr int TSK_OFF = TSQ_OFF + kTsSlot * 8;   // int64 [2][kTsSlot]
  static constexpr int W_OFF = TSK_OFF + 2 * kTsSlot * 8; // float [256]
  static constexpr int PW_OFF = W_OFF + 1024;             // float [1024]
  static constexpr int TAB_OFF = PW_OFF + 4096;           // SmemBias
  static constexpr int KMAX_OFF = TAB_OFF + 160;          // int64 [2][4]
  static constexpr int BAR_OFF = KMAX_OFF + 64;
  static constexpr int NBARS = 20;
  static constexpr int TMEMPTR_OFF = BAR_OFF + NBARS * 8;
  static constexpr int SMEM = TMEMPTR_OFF + 16;
};

template <int D>
__global__ void __launch_bounds__(kDqThreads, 1)
    hstu_bwd_dq_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
                       const __grid_constant__ CUtensorMap tm_tsq, const __grid_constant__ CUtensorMap tm_tsk,
                       const __grid_constant__ AttnParams p, __nv_bfloat16* __restrict__ dq, int64_t ld_dq) {
  using C = DqCfg<D>;
  extern __shared__ __align__(1024) uint8_t smem[];
  int64_t* s_tsq = reinterpret_cast<int64_t*>(smem + C::TSQ_OFF);
  int64_t* s_tsk = reinterpret_cast<int64_t*>(smem + C::TSK_OFF);
  float* s_w = reinterpret_cast<float*>(smem + C::W_OFF);
  float* s_pw = reinterpret_cast<float*>(smem + C::PW_OFF);
  SmemBias* s_bias = reinterpret_cast<SmemBias*>(smem + C::TAB_OFF);
  int64_t* s_kmax = reinterpret_cast<int64_t*>(smem + C::KMAX_OFF);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;   // MMA (last S, dP, dQ of the item) + compute warps (ts_q)
  uint64_t* k_full = bars + 2;    // [2] K + ts_k
  uint64_t* k_empty = bars + 4;   // [2] dQ_j done (last reader of K_j) + compute (ts_k)
  uint64_t* kx_full = bars + 6;   // [2] chunk maxima of ts_k
  uint64_t* v_full = bars + 8;
  uint64_t* v_empty = bars + 9;
  uint64_t* s_full = bars + 10;   // [2]
  uint64_t* dp_full = bars + 12;
  uint64_t* ds_full = bars + 13;  // dS in smem; S_j, dP_j consumed
  uint64_t* ds_empty = bars + 14; // dQ_j done with dS
  uint64_t* dq_full = bars + 15;
  uint64_t* dq_empty = bars + 16;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + C::TMEMPTR_OFF);

  const uint32_t warp = warp_id();
  const int tid = threadIdx.x;
  const int H = p.num_heads;
  const int nb = p.bias.nb;
  const int P = p.num_pos;
  const bool has_pos = P > 0;

  if (smem_u32(smem) & 1023) __trap();
  for (int i = tid; i < nb; i += blockDim.x) s_w[i] = p.ts_weights[i];
  for (int i = tid; i < P; i += blockDim.x) s_pw[i] = p.pos_weights[i];
  smem_bias_fill(s_bias, p.bias, tid, blockDim.x);
  if (tid == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1 + kCompWarps);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1 + kCompWarps);
      mbar_init(&kx_full[i], 1);
      mbar_init(&s_full[i], 1);
    }
    mbar_init(v_full, 1);
    mbar_init(v_empty, 1);
    mbar_init(dp_full, 1);
    mbar_init(ds_full, 32 * kCompWarps);
    mbar_init(ds_empty, 1);
    mbar_init(dq_full, 1);
    mbar_init(dq_empty, 32 * kCompWarps);
    fence_barrier_init();
  }
  if (warp == 0 && lane_id() == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    tma_prefetch_desc(&tm_do);
    tma_prefetch_desc(&tm_tsq);
    tma_prefetch_desc(&tm_tsk);
  }
  if (warp == 2) tmem_alloc(s_tmem, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  const uint32_t tDP = tmem + 256, tDQ = tmem + 384;

  const int total = p.wl.hdr->n_fwd * H;

  if (warp == 0) {
    // ================= TMA producer
    if (elect_one()) {
      uint32_t q_it = 0, k_it = 0, v_it = 0;
      for (int g = blockIdx.x; g < total; g += gridDim.x) {
        const int2 it = p.wl.fwd[g / H];
        const int h = g % H;
        const Seg sg = load_seg(p.seg, it.x);
        const int n = (int)((fwd_kv_lim(sg, it.y) + kBN - 1) / kBN);
        if (n == 0) continue;
        mbar_wait(q_empty, (q_it & 1) ^ 1);
        mbar_expect_tx(q_full, 2 * C::TILE + kTsBytes);
        const int32_t qrow = (int32_t)(sg.q_row0 + (int64_t)it.y * kBM);
        for (int pn = 0; pn < C::PANELS; ++pn) {
          tma_load_2d(smem + C::Q_OFF + pn * 16384, &tm_q, h * D + pn * 64, qrow, q_full);
          tma_load_2d(smem + C::DO_OFF + pn * 16384, &tm_do, h * D + pn * 64, qrow, q_full);
        }
        tma_load_1d(s_tsq, &tm_tsq, qrow & ~1, q_full);
        ++q_it;
        auto load_k = [&](int j) {
          const int st = k_it & 1;
          const int32_t krow = (int32_t)(sg.kv_row0 + (int64_t)j * kBN);
          mbar_wait(&k_empty[st], ((k_it >> 1) & 1) ^ 1);
          mbar_expect_tx(&k_full[st], C::TILE + kTsBytes);
          for (int pn = 0; pn < C::PANELS; ++pn)
            tma_load_2d(smem + C::K_OFF + st * C::TILE + pn * 16384, &tm_k, h * D + pn * 64, krow, &k_full[st]);
          tma_load_1d(s_tsk + st * kTsSlot, &tm_tsk, krow & ~1, &k_full[st]);
          ++k_it;
        };
        auto load_v = [&](int j) {
          const int32_t krow = (int32_t)(sg.kv_row0 + (int64_t)j * kBN);
          mbar_wait(v_empty, (v_it & 1) ^ 1);
          mbar_expect_tx(v_full, C::TILE);
          for (int pn = 0; pn < C::PANELS; ++pn)
            tma_load_2d(smem + C::V_OFF + pn * 16384, &tm_v, h * D + pn * 64, krow, v_full);
          ++v_it;
        };
        load_k(0);
        for (int j = 0; j < n; ++j) {
          if (j + 1 < n) load_k(j + 1);
          load_v(j);
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer
    if (elect_one()) {
      constexpr uint32_t id_s = idesc_bf16(128, 128, 0, 0);  // S = Q K^T, dP = dO V^T
      constexpr uint32_t id_q = idesc_bf16(128, D, 0, 1);    // dQ += dS K (A K-major smem, B MN-major)
      const uint32_t q_base = smem_u32(smem + C::Q_OFF);
      const uint32_t do_base = smem_u32(smem + C::DO_OFF);
      const uint32_t v_base = smem_u32(smem + C::V_OFF);
      const uint32_t ds_base = smem_u32(smem + C::DS_OFF);
      uint32_t q_it = 0, k_it = 0, v_it = 0, s_it = 0, ds_cnt = 0, o_it = 0;
      auto k_base = [&](uint32_t ki) { return smem_u32(smem + C::K_OFF + (ki & 1) * C::TILE); };
      auto issue_S = [&](uint32_t ki, uint32_t sb) {
        mbar_wait(&k_full[ki & 1], (ki >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          umma_ss(tmem + 128 * sb, sdesc_sw128(q_base + off, 16, 1024), sdesc_sw128(k_base(ki) + off, 16, 1024),
                  id_s, kk > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[sb]);
      };
      auto issue_dP = [&]() {
        mbar_wait(v_full, v_it & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          umma_ss(tDP, sdesc_sw128(do_base + off, 16, 1024), sdesc_sw128(v_base + off, 16, 1024), id_s,
                  kk > 0 ? 1u : 0u);
        }
        umma_commit(dp_full);
        umma_commit(v_empty);
        ++v_it;
      };
      for (int g = blockIdx.x; g < total; g += gridDim.x) {
        const int2 it = p.wl.fwd[g / H];
        const Seg sg = load_seg(p.seg, it.x);
        const int n = (int)((fwd_kv_lim(sg, it.y) + kBN - 1) / kBN);
        if (n == 0) continue;
        mbar_wait(q_full, q_it & 1);
        const uint32_t k0 = k_it, s0 = s_it;
        issue_S(k0, s0 & 1);
        issue_dP();
        if (n > 1) issue_S(k0 + 1, (s0 + 1) & 1);
        for (int j = 0; j < n; ++j) {
          mbar_wait(ds_full, ds_cnt & 1);
          ++ds_cnt;
          if (j == 0) mbar_wait(dq_empty, (o_it & 1) ^ 1);  // previous item's dQ written out
          tc_fence_after();
          // dQ += dS K_j
#pragma unroll
          for (int kk = 0; kk < kBN / 16; ++kk) {
            const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
            umma_ss(tDQ, sdesc_sw128(ds_base + off, 16, 1024), sdesc_sw128(k_base(k0 + j) + kk * 2048, 16384, 1024),
                    id_q, (kk > 0 || j > 0) ? 1u : 0u);
          }
          umma_commit(ds_empty);
          umma_commit(&k_empty[(k0 + j) & 1]);
          if (j + 1 < n) issue_dP();                           // dP region: dP_j consumed (ds_full)
          if (j + 2 < n) issue_S(k0 + j + 2, (s0 + j) & 1);    // S buffer of tile j consumed (ds_full)
        }
        k_it += n;
        s_it += n;
        umma_commit(dq_full);
        umma_commit(q_empty);
        ++o_it;
        ++q_it;
      }
    }
  } else if (warp == 3) {
    // ================= ts_k statistics: per 32-column chunk maximum
    const int lane = lane_id();
    uint32_t k_it = 0;
    for (int g = blockIdx.x; g < total; g += gridDim.x) {
      const int2 it = p.wl.fwd[g / H];
      const Seg sg = load_seg(p.seg, it.x);
      const int n = (int)((fwd_kv_lim(sg, it.y) + kBN - 1) / kBN);
      for (int j = 0; j < n; ++j) {
        const int st = k_it & 1;
        mbar_wait(&k_full[st], (k_it >> 1) & 1);
        const int64_t* tsk = s_tsk + st * kTsSlot + ((sg.kv_row0 + (int64_t)j * kBN) & 1);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int64_t m = warp_max_i64(tsk[32 * c + lane]);
          if (lane == 0) s_kmax[st * 4 + c] = m;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&kx_full[st]);
        ++k_it;
      }
    }
  } else if (warp >= 4) {
    // ================= compute: thread = (q row r, kv-column half wg)
    const int et = tid - 128;
    const int wg = et >> 7;
    const int r = et & 127;
    const int lane = r & 31;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const float c1 = 0.5f * rsqrtf((float)D);
    const int64_t cap = p.bias.cap;
    float cb = s_w[nb - 1];
    if (has_pos) cb += s_pw[P - 1];
    cb *= c1;
    uint32_t q_it = 0, k_it = 0, s_it = 0, dp_cnt = 0, ds_cnt = 0, o_it = 0;
    for (int g = blockIdx.x; g < total; g += gridDim.x) {
      const int2 it = p.wl.fwd[g / H];
      const int h = g % H;
      const Seg sg = load_seg(p.seg, it.x);
      const int64_t kv_lim = fwd_kv_lim(sg, it.y);
      const int n = (int)((kv_lim + kBN - 1) / kBN);
      const int64_t nq = min((int64_t)kBM, sg.lq - (int64_t)it.y * kBM);
      const bool row_ok = r < nq;
      const int64_t qp_tile = sg.qp0 + (int64_t)it.y * kBM;
      const int64_t qpos = qp_tile + r;
      const int64_t qrow = sg.q_row0 + (int64_t)it.y * kBM + r;
      __nv_bfloat16* dqrow = dq + qrow * ld_dq + h * D;
      if (n == 0) {
        if (row_ok)
          for (int c = wg * (D / 2); c < (wg + 1) * (D / 2); c += 8)
            *reinterpret_cast<int4*>(dqrow + c) = make_int4(0, 0, 0, 0);
        continue;
      }
      mbar_wait(q_full, q_it & 1);
      const int64_t tq = row_ok ? s_tsq[((qrow - r) & 1) + r] : (INT64_MAX >> 2);
      __syncwarp();
      if (lane == 0) mbar_arrive(q_empty);
      ++q_it;
      const int64_t tq_min = warp_min_i64(tq);
      const int64_t row_lo = qp_tile + (r & ~31), row_hi = row_lo + 31;
      for (int j = 0; j < n; ++j) {
        const int st = k_it & 1;
        const int sb = s_it & 1;
        const int64_t kv0 = (int64_t)j * kBN;
        mbar_wait(&kx_full[st], (k_it >> 1) & 1);
        const int64_t* tsk = s_tsk + st * kTsSlot + ((sg.kv_row0 + kv0) & 1);
        int cls_bits = 0;
#pragma unroll
        for (int ci = 0; ci < 2; ++ci) {
          const int c0 = 64 * wg + 32 * ci;
          const int64_t kc0 = kv0 + c0, kc1 = kc0 + 31;
          int cls = 0;
          if (!(kc0 > row_hi || kc0 >= kv_lim)) {
            cls = 2;
            if ((kc1 <= row_lo) && (kc1 < kv_lim) && (tq_min - s_kmax[st * 4 + (c0 >> 5)] >= cap) &&
                (!has_pos || row_lo - kc1 >= P - 1))
              cls = 1;
          }
          cls_bits |= cls << (2 * ci);
        }
        mbar_wait(&s_full[sb], (s_it >> 1) & 1);
        mbar_wait(dp_full, dp_cnt & 1);
        ++dp_cnt;
        if (ds_cnt > 0) mbar_wait(ds_empty, (ds_cnt - 1) & 1);
        ++ds_cnt;
        tc_fence_after();
        const uint32_t tS = tmem + 128 * sb + lane_off;
#pragma unroll 1
        for (int ci = 0; ci < 2; ++ci) {
          const int c0 = 64 * wg + 32 * ci;
          const int cls = (cls_bits >> (2 * ci)) & 3;
          // dS row r (q), kv cols c0..c0+31 -> 128B-swizzled K-major smem (panel = c0 / 64)
          uint8_t* prow = smem + C::DS_OFF + (c0 >> 6) * 16384;
          if (cls == 1) {
            uint32_t sv[32], dv[32], dsk[16];
            tmem_ld32(tS + c0, sv);
            tmem_ld32(tDP + lane_off + c0, dv);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              const float h0 = fmaf(__uint_as_float(sv[i]), c1, cb);
              const float h1 = fmaf(__uint_as_float(sv[i + 1]), c1, cb);
              const float2 th = make_float2(tanh_approx(h0), tanh_approx(h1));
              const float d0 = __uint_as_float(dv[i]) * (1.f + th.x) * (fmaf(-h0, th.x, h0) + 1.f) * c1;
              const float d1 = __uint_as_float(dv[i + 1]) * (1.f + th.y) * (fmaf(-h1, th.y, h1) + 1.f) * c1;
              dsk[i >> 1] = pack_bf16(d0, d1);
            }
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4)
              *reinterpret_cast<int4*>(prow + sw128_offset(r, (c0 & 63) + q4 * 8)) =
                  make_int4(dsk[4 * q4], dsk[4 * q4 + 1], dsk[4 * q4 + 2], dsk[4 * q4 + 3]);
          } else if (cls == 0) {
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4)
              *reinterpret_cast<int4*>(prow + sw128_offset(r, (c0 & 63) + q4 * 8)) = make_int4(0, 0, 0, 0);
          } else {
#pragma unroll 1
            for (int g8 = 0; g8 < 32; g8 += 8) {
              uint32_t sv[8], dv[8], dsk[4];
              tmem_ld8(tS + c0 + g8, sv);
              tmem_ld8(tDP + lane_off + c0 + g8, dv);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 8; i += 2) {
                float dd[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                  const int64_t kpos = kv0 + c0 + g8 + i + u;
                  float bias = s_w[bucket_smem(tq - tsk[c0 + g8 + i + u], s_bias, cap)];
                  if (has_pos) {
                    const int64_t rel = qpos - kpos;
                    bias += s_pw[rel < 0 ? 0 : (rel > P - 1 ? P - 1 : (int)rel)];
                  }
                  const float hh = (__uint_as_float(sv[i + u]) + bias) * c1;
                  const float th = tanh_approx(hh);
                  const bool ok = row_ok && kpos <= qpos && kpos < kv_lim;
                  dd[u] = ok ? __uint_as_float(dv[i + u]) * (1.f + th) * (fmaf(-hh, th, hh) + 1.f) * c1 : 0.f;
                }
                dsk[i >> 1] = pack_bf16(dd[0], dd[1]);
              }
              *reinterpret_cast<int4*>(prow + sw128_offset(r, (c0 & 63) + g8)) =
                  make_int4(dsk[0], dsk[1], dsk[2], dsk[3]);
            }
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc_fence_before();
        mbar_arrive(ds_full);
        __syncwarp();
        if (lane == 0) mbar_arrive(&k_empty[st]);  // done with this stage's ts_k
        ++k_it;
        ++s_it;
      }
      // ---- dQ: TMEM -> bf16 -> global (each group writes half the columns)
      mbar_wait(dq_full, o_it & 1);
      ++o_it;
      tc_fence_after();
#pragma unroll 1
      for (int c0 = wg * (D / 2); c0 < (wg + 1) * (D / 2); c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tDQ + lane_off + c0, v);
        tmem_ld_wait();
        if (row_ok) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 32; i += 2) pk[i >> 1] = pack_bf16(__uint_as_float(v[i]), __uint_as_float(v[i + 1]));
          int4* d4 = reinterpret_cast<int4*>(dqrow + c0);
#pragma unroll
          for (int i = 0; i < 4; ++i) d4[i] = make_int4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
        }
      }
      tc_fence_before();
      mbar_arrive(dq_empty);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

template <int D>
int launch_bwd(const TMaps& tm, const AttnParams& p, const jh_attn_args& a, int grid, cudaStream_t s) {
  using C = DkvCfg<D>;
  using Q = DqCfg<D>;
  static_assert(C::SMEM <= 232448 && Q::SMEM <= 232448, "bwd smem budget");
  if (a.num_buckets > C::MAX_NB) {
    set_error(JH_ERR_UNSUPPORTED, "backward supports num_buckets <= %d at head_dim %d", C::MAX_NB, D);
    return -1;
  }
  if (D == 128 && a.num_pos > 0) {
    set_error(JH_ERR_UNSUPPORTED, "pos_weights backward is implemented for head_dim 64 only");
    return -1;
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(hstu_bwd_dkv_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    cudaFuncSetAttribute(hstu_bwd_dq_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, Q::SMEM);
    attr = true;
  }
  if (a.prof_event_start) cudaEventRecord((cudaEvent_t)a.prof_event_start, s);
  hstu_bwd_dkv_kernel<D><<<grid, kBwdThreads, C::SMEM, s>>>(tm.q, tm.k, tm.v, tm.dout, tm.tsq, p);
  if (cudaError_t e = cudaGetLastError()) return (int)e;
  hstu_bwd_dq_kernel<D><<<grid, kDqThreads, Q::SMEM, s>>>(tm.q, tm.k, tm.v, tm.dout, tm.tsq, tm.tsk, p,
                                                         (__nv_bfloat16*)a.dq, a.ld_dq);
  if (a.prof_event_end) cudaEventRecord((cudaEvent_t)a.prof_event_end, s);
  return (int)cudaGetLastError();
}

template int launch_bwd<64>(const TMaps&, const AttnParams&, const jh_attn_args&, int, cudaStream_t);
template int launch_bwd<128>(const TMaps&, const AttnParams&, const jh_attn_args&, int, cudaStream_t);

}  // namespace jh
