// Fused jagged HSTU attention backward for sm_100a.
//
// Reference: attention.py:187-234 hstu_attention_backward
//   dV = A^T g;  dS = (g V^T) . sigma(S) (1 + S (1 - sigma(S)))  (masked)
//   dQ = dS K / sqrt(d);  dK = dS^T Q / sqrt(d);  d_w = bincount(bucket, dS / sqrt(d))
//
// kv-tile-major persistent kernel: a work item is (segment, 128-row kv tile)
// x head; it loops over the q tiles that can see the kv tile.
//   warp 0       TMA producer: K_j, V_j once per item; Q_i, dO_i, ts_q (2 stages)
//   warp 1       MMA issuer:
//                  (1) S^T  = K Q^T      -> TMEM [0,128)   (lane = kv row)
//                  (2) dP^T = V dO^T     -> TMEM [128,256)
//                  (3) dV  += P^T dO     A = P^T from TMEM (aliases S^T cols 0..63)
//                  (4) dK  += dS^T Q     A = dS^T in smem (K-major)
//                  (5) dQ_i = dS K       A = the same smem viewed MN-major -> TMEM [128,256)
//   warp 2       TMEM allocator (512 columns: S^T | dP^T / dQ | dV | dK)
//   warps 4..11  epilogue, two groups of 4 warps (q-column halves): thread =
//                kv row for (S^T, dP^T) -> (P^T, dS^T, d_w); thread = q row
//                when draining dQ_i (fp32 red.global.add into the dq
//                accumulator); group 0 writes dV, group 1 dK once per item.
// dS carries the 1/sqrt(d) scale so (4), (5) and d_w need no extra pass.
#include <algorithm>

#include "abi_internal.h"
#include "attn_common.cuh"

namespace jh {

constexpr int kBwdEpiWarps = 8;
constexpr int kBwdThreads = 128 + 32 * kBwdEpiWarps;

template <int D>
struct BwdCfg {
  static constexpr int TILE = 128 * D * 2;  // one 128-row bf16 operand tile
  static constexpr int PANELS = D / 64;
  static constexpr int K_OFF = 0;
  static constexpr int V_OFF = TILE;
  static constexpr int Q_OFF = 2 * TILE;          // [2] stages
  static constexpr int DO_OFF = 4 * TILE;         // [2] stages
  static constexpr int DS_OFF = 6 * TILE;         // 128 x 128 bf16 (2 panels)
  static constexpr int TSQ_OFF = DS_OFF + 32768;  // int64 [2][kTsSlot]
  static constexpr int MAX_NB = (D == 64) ? 256 : 32;  // D=128 leaves ~2 KB of smem for the rest
  static constexpr int W_OFF = TSQ_OFF + 2 * kTsSlot * 8;  // float [MAX_NB]
  static constexpr int PW_OFF = W_OFF + MAX_NB * 4;    // float [<=1024] (pos extension, D=64)
  static constexpr int BINS_OFF = PW_OFF + (D == 64 ? 4096 : 0);  // double bins [MAX_NB (+1024)]
  static constexpr int NBINS = MAX_NB + (D == 64 ? 1024 : 0);
  static constexpr int BAR_OFF = BINS_OFF + NBINS * 8;
  static constexpr int NBARS = 16;
  static constexpr int TMEMPTR_OFF = BAR_OFF + NBARS * 8;
  static constexpr int SMEM = TMEMPTR_OFF + 16;
};

JH_DEV void red_add_v4(float* addr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

template <int D>
__global__ void __launch_bounds__(kBwdThreads, 1)
    hstu_bwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
                    const __grid_constant__ CUtensorMap tm_tsq, const __grid_constant__ AttnParams p) {
  using C = BwdCfg<D>;
  extern __shared__ __align__(1024) uint8_t smem[];
  int64_t* s_tsq = reinterpret_cast<int64_t*>(smem + C::TSQ_OFF);
  float* s_w = reinterpret_cast<float*>(smem + C::W_OFF);
  float* s_pw = reinterpret_cast<float*>(smem + C::PW_OFF);
  double* s_bins = reinterpret_cast<double*>(smem + C::BINS_OFF);  // [MAX_NB] then [P]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* kv_full = bars + 0;
  uint64_t* kv_empty = bars + 1;
  uint64_t* qd_full = bars + 2;   // [2]
  uint64_t* qd_empty = bars + 4;  // [2]
  uint64_t* s_full = bars + 6;
  uint64_t* epi_done = bars + 7;
  uint64_t* pv_done = bars + 8;
  uint64_t* dq_full = bars + 9;
  uint64_t* dq_empty = bars + 10;
  uint64_t* dkv_full = bars + 11;
  uint64_t* dkv_empty = bars + 12;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + C::TMEMPTR_OFF);

  const uint32_t warp = warp_id();
  const int tid = threadIdx.x;
  const int H = p.num_heads;
  const int nb = p.bias.nb;
  const int P = p.num_pos;
  const bool has_pos = P > 0;
  const int64_t HD = (int64_t)H * D;

  if (smem_u32(smem) & 1023) __trap();  // swizzled operand tiles need 1 KB alignment
  for (int i = tid; i < nb; i += blockDim.x) s_w[i] = p.ts_weights[i];
  if (D == 64)
    for (int i = tid; i < P; i += blockDim.x) s_pw[i] = p.pos_weights[i];
  for (int i = tid; i < C::NBINS; i += blockDim.x) s_bins[i] = 0.0;
  if (tid == 0) {
    mbar_init(kv_full, 1);
    mbar_init(kv_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&qd_full[i], 1);
      mbar_init(&qd_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(epi_done, 32 * kBwdEpiWarps);
    mbar_init(pv_done, 1);
    mbar_init(dq_full, 1);
    mbar_init(dq_empty, 32 * kBwdEpiWarps);
    mbar_init(dkv_full, 1);
    mbar_init(dkv_empty, 32 * kBwdEpiWarps);
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

  const int n_items = p.wl.hdr->n_bwd;
  const int total = n_items * H;

  // q-tile range of an item: tiles t0 .. nt-1 of the segment whose rows reach kv tile j
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
      uint32_t it_cnt = 0, qd_it = 0;
      for (int g = blockIdx.x; g < total; g += gridDim.x) {
        const int2 it = p.wl.bwd[g / H];
        const int h = g % H;
        const Seg sg = load_seg(p.seg, it.x);
        int t0, nt;
        q_tiles(sg, it.y, t0, nt);
        if (t0 >= nt) continue;
        mbar_wait(kv_empty, (it_cnt & 1) ^ 1);
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
      constexpr uint32_t id_q = idesc_bf16(128, D, 1, 1);    // dQ (A smem MN-major)
      const uint32_t k_base = smem_u32(smem + C::K_OFF);
      const uint32_t v_base = smem_u32(smem + C::V_OFF);
      const uint32_t ds_base = smem_u32(smem + C::DS_OFF);
      uint32_t it_cnt = 0, qd_it = 0, pv_cnt = 0, dq_cnt = 0, s_cnt = 0;
      for (int g = blockIdx.x; g < total; g += gridDim.x) {
        const int2 it = p.wl.bwd[g / H];
        const Seg sg = load_seg(p.seg, it.x);
        int t0, nt;
        q_tiles(sg, it.y, t0, nt);
        if (t0 >= nt) continue;
        mbar_wait(kv_full, it_cnt & 1);
        for (int t = t0; t < nt; ++t) {
          const int st = qd_it & 1;
          const uint32_t q_base = smem_u32(smem + C::Q_OFF + st * C::TILE);
          const uint32_t do_base = smem_u32(smem + C::DO_OFF + st * C::TILE);
          mbar_wait(&qd_full[st], (qd_it >> 1) & 1);
          if (pv_cnt > 0) mbar_wait(pv_done, (pv_cnt - 1) & 1);  // P^T (in S^T cols) consumed
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
            umma_ss(tS, sdesc_sw128(k_base + off, 16, 1024), sdesc_sw128(q_base + off, 16, 1024), id_s,
                    kk > 0 ? 1u : 0u);
          }
          if (dq_cnt > 0) mbar_wait(dq_empty, (dq_cnt - 1) & 1);  // dQ of the previous tile drained
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
            umma_ss(tDP, sdesc_sw128(v_base + off, 16, 1024), sdesc_sw128(do_base + off, 16, 1024), id_s,
                    kk > 0 ? 1u : 0u);
          }
          umma_commit(s_full);
          mbar_wait(epi_done, s_cnt & 1);
          ++s_cnt;
          if (t == t0) mbar_wait(dkv_empty, (it_cnt & 1) ^ 1);  // dK/dV of the previous item drained
          tc_fence_after();
          const uint32_t acc0 = (t == t0) ? 0u : 1u;
          // (3) dV += P^T dO.  Packed P^T of q columns [64g, 64g+64) sits in
          // TMEM columns [64g, 64g+32) (each epilogue group overwrites only
          // S^T columns it has already read).
#pragma unroll
          for (int kk = 0; kk < kBM / 16; ++kk)
            umma_ts(tDV, tS + kk * 8 + (kk >= 4 ? 32 : 0), sdesc_sw128(do_base + kk * 2048, 16384, 1024), id_kv,
                    (kk > 0) ? 1u : acc0);
          umma_commit(pv_done);
          ++pv_cnt;
          // (4) dK += dS^T Q
#pragma unroll
          for (int kk = 0; kk < kBM / 16; ++kk) {
            const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
            umma_ss(tDK, sdesc_sw128(ds_base + off, 16, 1024), sdesc_sw128(q_base + kk * 2048, 16384, 1024), id_kv,
                    (kk > 0) ? 1u : acc0);
          }
          // (5) dQ_i = dS K
#pragma unroll
          for (int kk = 0; kk < kBN / 16; ++kk)
            umma_ss(tDP, sdesc_sw128(ds_base + kk * 2048, 16384, 1024), sdesc_sw128(k_base + kk * 2048, 16384, 1024),
                    id_q, kk > 0 ? 1u : 0u);
          umma_commit(dq_full);
          ++dq_cnt;
          umma_commit(&qd_empty[st]);
          ++qd_it;
        }
        umma_commit(dkv_full);
        umma_commit(kv_empty);
        ++it_cnt;
      }
    }
  } else if (warp >= 4) {
    // ================= epilogue: thread = (row r, column half wg)
    const int et = tid - 128;
    const int wg = et >> 7;
    const int r = et & 127;  // kv row (S^T/dP^T/dK/dV) or q row (dQ)
    const int lane = r & 31;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const float c1 = 0.5f * rsqrtf((float)D);
    const int64_t cap = p.bias.cap;
    uint8_t* ds_smem = smem + C::DS_OFF + wg * 16384;  // this group's 64 q columns = one panel
    float cb = s_w[nb - 1];
    if (has_pos) cb += s_pw[P - 1];
    cb *= c1;
    double acc_w = 0.0, acc_p = 0.0;  // saturated-bucket partials (fp64 across tiles)
    uint32_t it_cnt = 0, s_cnt = 0, dq_cnt = 0, qd_it = 0;
    for (int g = blockIdx.x; g < total; g += gridDim.x) {
      const int2 it = p.wl.bwd[g / H];
      const int h = g % H;
      const Seg sg = load_seg(p.seg, it.x);
      int t0, nt;
      q_tiles(sg, it.y, t0, nt);
      const int64_t kv0 = (int64_t)it.y * kBN;
      const int64_t kpos = kv0 + r;
      const bool krow_ok = kpos < sg.kv_len;
      const int64_t krow = sg.kv_row0 + kpos;
      if (t0 >= nt) {
        // no query sees this kv tile: its dK/dV rows are zero
        if (krow_ok && !p.dk_accum) {
          __nv_bfloat16* dst = wg ? (p.dk + krow * p.ld_dk) : (p.dv + krow * p.ld_dv);
          for (int c = 0; c < D; c += 8) *reinterpret_cast<int4*>(dst + h * D + c) = make_int4(0, 0, 0, 0);
        }
        continue;
      }
      const int64_t tk = krow_ok ? p.ts_k[krow] : (INT64_MIN >> 2);
      const int64_t tk_max = warp_max_i64(tk);
      const int64_t k_lo = kv0 + (r & ~31), k_hi = k_lo + 31;  // this warp's kv positions
      const bool warp_k_ok = k_hi < sg.kv_len;
      for (int t = t0; t < nt; ++t) {
        const int st = qd_it & 1;
        const int64_t qrow0 = sg.q_row0 + (int64_t)t * kBM;
        const int64_t qp_tile = sg.qp0 + (int64_t)t * kBM;
        const int64_t nq = min((int64_t)kBM, sg.lq - (int64_t)t * kBM);
        mbar_wait(&qd_full[st], (qd_it >> 1) & 1);
        ++qd_it;
        const int64_t* tsq = s_tsq + st * kTsSlot + (qrow0 & 1);
        mbar_wait(s_full, s_cnt & 1);
        ++s_cnt;
        tc_fence_after();
        float sat_w = 0.f, sat_p = 0.f;
#pragma unroll 1
        for (int c0 = 64 * wg; c0 < 64 * wg + 64; c0 += 32) {
          const int64_t qc0 = qp_tile + c0, qc1 = qc0 + 31;
          uint32_t pk[16], dk[16];
          if (qc1 < k_lo || c0 >= nq) {
            // every pair of this chunk has its key in the future, or no query
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = dk[i] = 0u;
          } else {
            uint32_t sv[32], dv[32];
            tmem_ld32(tS + lane_off + c0, sv);
            tmem_ld32(tDP + lane_off + c0, dv);
            const bool full = (qc0 >= k_hi) && (c0 + 32 <= nq) && warp_k_ok;
            bool sat = false;
            if (full) {
              const int64_t tq_min = warp_min_i64(tsq[c0 + lane]);
              sat = (tq_min - tk_max >= cap) && (!has_pos || qc0 - k_hi >= P - 1);
            }
            tmem_ld_wait();
            if (sat) {
              float tile_sum = 0.f;
#pragma unroll
              for (int i = 0; i < 32; i += 2) {
                float pp[2], dd[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                  const float hh = fmaf(__uint_as_float(sv[i + u]), c1, cb);
                  const float th = tanh_approx(hh);
                  pp[u] = fmaf(hh, th, hh);
                  const float gp = __uint_as_float(dv[i + u]);
                  dd[u] = fmaf(th, gp, gp) * (fmaf(-hh, th, hh) + 1.f) * c1;
                  tile_sum += dd[u];
                }
                pk[i >> 1] = pack_bf16(pp[0], pp[1]);
                dk[i >> 1] = pack_bf16(dd[0], dd[1]);
              }
              sat_w += tile_sum;
              if (has_pos) sat_p += tile_sum;  // saturated chunks hit both last buckets
            } else {
#pragma unroll
              for (int i = 0; i < 32; i += 2) {
                float pp[2], dd[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                  const int qi = c0 + i + u;
                  const int64_t qpos = qp_tile + qi;
                  const bool ok = krow_ok && (qi < nq) && (kpos <= qpos);
                  const int b = bucket_of(tsq[qi] - tk, p.bias.thr, p.bias.base, cap);
                  float bias = s_w[b];
                  int rel = 0;
                  if (has_pos) {
                    int64_t rr = qpos - kpos;
                    rel = (int)(rr < 0 ? 0 : (rr > P - 1 ? P - 1 : rr));
                    bias += s_pw[rel];
                  }
                  const float hh = (__uint_as_float(sv[i + u]) + bias) * c1;
                  const float th = tanh_approx(hh);
                  const float gp = __uint_as_float(dv[i + u]);
                  const float ds = ok ? fmaf(th, gp, gp) * (fmaf(-hh, th, hh) + 1.f) * c1 : 0.f;
                  pp[u] = ok ? fmaf(hh, th, hh) : 0.f;
                  dd[u] = ds;
                  if (ok) {
                    if (b == nb - 1)
                      sat_w += ds;
                    else
                      atomicAdd(&s_bins[b], (double)ds);
                    if (has_pos) {
                      if (rel == P - 1)
                        sat_p += ds;
                      else
                        atomicAdd(&s_bins[C::MAX_NB + rel], (double)ds);
                    }
                  }
                }
                pk[i >> 1] = pack_bf16(pp[0], pp[1]);
                dk[i >> 1] = pack_bf16(dd[0], dd[1]);
              }
            }
          }
          tmem_st16(tS + lane_off + 64 * wg + ((c0 & 63) >> 1), pk);
          // dS^T row r, q cols c0..c0+31 -> 128B-swizzled K-major smem panel
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const uint32_t col = (c0 & 63) + q4 * 8;
            *reinterpret_cast<int4*>(ds_smem + sw128_offset(r, col)) =
                make_int4(dk[4 * q4], dk[4 * q4 + 1], dk[4 * q4 + 2], dk[4 * q4 + 3]);
          }
        }
        acc_w += (double)sat_w;
        acc_p += (double)sat_p;
        tmem_st_wait();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc_fence_before();
        mbar_arrive(epi_done);

        // ---- drain dQ_i (thread = q row, group = column half) into the fp32 accumulator
        mbar_wait(dq_full, dq_cnt & 1);
        ++dq_cnt;
        tc_fence_after();
        const bool qrow_ok = r < nq;
        float* dqa = p.wl.dq_accum + (qrow0 + r) * HD + h * D;
#pragma unroll 1
        for (int c0 = wg * (D / 2); c0 < (wg + 1) * (D / 2); c0 += 32) {
          uint32_t v[32];
          tmem_ld32(tDP + lane_off + c0, v);
          tmem_ld_wait();
          if (qrow_ok) {
#pragma unroll
            for (int i = 0; i < 32; i += 4)
              red_add_v4(dqa + c0 + i, __uint_as_float(v[i]), __uint_as_float(v[i + 1]), __uint_as_float(v[i + 2]),
                         __uint_as_float(v[i + 3]));
          }
        }
        tc_fence_before();
        mbar_arrive(dq_empty);
      }
      // ---- dV (group 0) / dK (group 1) for this kv tile (thread = kv row)
      mbar_wait(dkv_full, it_cnt & 1);
      ++it_cnt;
      tc_fence_after();
      {
        const uint32_t tsrc = wg ? tDK : tDV;
        float* acc = wg ? p.dk_accum : p.dv_accum;
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
              red_add_v4(dst + i, __uint_as_float(v[i]), __uint_as_float(v[i + 1]), __uint_as_float(v[i + 2]),
                         __uint_as_float(v[i + 3]));
          } else {
            __nv_bfloat16* dst = (wg ? (p.dk + krow * p.ld_dk) : (p.dv + krow * p.ld_dv)) + h * D + c0;
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
    // ---- flush d_ts_weights / d_pos partials
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      acc_w += __shfl_xor_sync(0xffffffffu, acc_w, o);
      acc_p += __shfl_xor_sync(0xffffffffu, acc_p, o);
    }
    if (lane == 0) {
      atomicAdd(&s_bins[nb - 1], acc_w);
      if (has_pos) atomicAdd(&s_bins[C::MAX_NB + P - 1], acc_p);
    }
    named_bar_sync(1, 32 * kBwdEpiWarps);
    for (int i = et; i < nb; i += 32 * kBwdEpiWarps)
      if (s_bins[i] != 0.0) atomicAdd(&p.d_ts_weights[i], s_bins[i]);
    if (has_pos)
      for (int i = et; i < P; i += 32 * kBwdEpiWarps)
        if (s_bins[C::MAX_NB + i] != 0.0) atomicAdd(&p.d_pos_weights[i], s_bins[C::MAX_NB + i]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

// dq (bf16, row stride ld) <- dq_accum (fp32, [rows, HD])
__global__ void dq_convert_kernel(const float* __restrict__ acc, __nv_bfloat16* __restrict__ dq, int64_t rows,
                                  int64_t HD, int64_t ld) {
  const int64_t per_row = HD / 8;
  const int64_t total = rows * per_row;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = g / per_row, c = (g - r * per_row) * 8;
    const float4 a = *reinterpret_cast<const float4*>(acc + r * HD + c);
    const float4 b = *reinterpret_cast<const float4*>(acc + r * HD + c + 4);
    *reinterpret_cast<int4*>(dq + r * ld + c) =
        make_int4(pack_bf16(a.x, a.y), pack_bf16(a.z, a.w), pack_bf16(b.x, b.y), pack_bf16(b.z, b.w));
  }
}

template <int D>
int launch_bwd(const TMaps& tm, const AttnParams& p, const jh_attn_args& a, int grid, cudaStream_t s) {
  using C = BwdCfg<D>;
  static_assert(C::SMEM <= 232448, "bwd smem budget");
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
    cudaFuncSetAttribute(hstu_bwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr = true;
  }
  const int64_t HD = (int64_t)a.num_heads * a.head_dim;
  if (cudaError_t e = cudaMemsetAsync(p.wl.dq_accum, 0, (size_t)a.q_rows * HD * 4, s)) return (int)e;
  if (a.prof_event_start) cudaEventRecord((cudaEvent_t)a.prof_event_start, s);
  hstu_bwd_kernel<D><<<grid, kBwdThreads, C::SMEM, s>>>(tm.q, tm.k, tm.v, tm.dout, tm.tsq, p);
  if (a.prof_event_end) cudaEventRecord((cudaEvent_t)a.prof_event_end, s);
  if (cudaError_t e = cudaGetLastError()) return (int)e;
  int64_t work = a.q_rows * HD / 8;
  int cgrid = (int)std::min<int64_t>((work + 255) / 256, (int64_t)grid * 16);
  if (cgrid < 1) cgrid = 1;
  dq_convert_kernel<<<cgrid, 256, 0, s>>>(p.wl.dq_accum, (__nv_bfloat16*)a.dq, a.q_rows, HD, a.ld_dq);
  return (int)cudaGetLastError();
}

template int launch_bwd<64>(const TMaps&, const AttnParams&, const jh_attn_args&, int, cudaStream_t);
template int launch_bwd<128>(const TMaps&, const AttnParams&, const jh_attn_args&, int, cudaStream_t);

}  // namespace jh
