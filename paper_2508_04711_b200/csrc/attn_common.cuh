// Shared pieces of the jagged HSTU attention kernels: segment decoding, the
// on-device work-list builder (no host sync: lists are built from the
// device-resident offsets and ordered longest-first), kernel parameter block.
#pragma once
#include "bias.cuh"

namespace jh {

constexpr int kBM = 128;  // q rows per tile
constexpr int kBN = 128;  // kv rows per tile
// Timestamp tiles are TMA-loaded from an even (16-byte aligned) start row:
// 136 int64 cover any 128-row tile; element i of the tile is at [(row0 & 1) + i].
constexpr int kTsBox = 136;
constexpr int kTsBytes = kTsBox * 8;
constexpr int kTsSlot = 144;  // int64 stride between smem slots (1152 B)
// 64-row half tiles (dKV kernel): ts box 72 (64 + parity, 16B multiple)
constexpr int kTsBoxH = 72;
constexpr int kTsBytesH = kTsBoxH * 8;
constexpr int kTsSlotH = 80;  // TMA smem destinations must be 128-byte aligned

struct SegArgs {
  const int64_t* q_offsets;
  const int64_t* q_pos0;
  const int64_t* kv_start;
  const int64_t* kv_len;
  int64_t num_segments;
};

struct Seg {
  int64_t q_row0, lq, qp0, kv_row0, kv_len;
};

JH_DEV Seg load_seg(const SegArgs& a, int64_t s) {
  Seg g;
  g.q_row0 = a.q_offsets[s];
  g.lq = a.q_offsets[s + 1] - g.q_row0;
  g.qp0 = a.q_pos0 ? a.q_pos0[s] : 0;
  g.kv_row0 = a.kv_start ? a.kv_start[s] : g.q_row0;
  g.kv_len = a.kv_len ? a.kv_len[s] : g.lq;
  return g;
}

// kv positions a q tile (rows t*128 ..) can see: [0, kv_lim)
JH_DEV int64_t fwd_kv_lim(const Seg& g, int t) {
  int64_t nq = g.lq - (int64_t)t * kBM;
  nq = nq < kBM ? nq : kBM;
  int64_t e = g.qp0 + (int64_t)t * kBM + nq;
  return e < g.kv_len ? e : g.kv_len;
}
// kv positions any q row of the segment can see
JH_DEV int64_t seg_kv_vis(const Seg& g) {
  int64_t e = g.qp0 + g.lq;
  return e < g.kv_len ? e : g.kv_len;
}

struct WorkHeader {
  int32_t n_fwd, n_bwd;
  int64_t ds_blocks;    // dS scratch blocks of all segments (one head)
  int32_t ds_overflow;  // set by the dKV kernel when the scratch is too small
  int32_t next_item[3]; // dynamic scheduler counters: fwd, dK/dV, dQ kernels
  int32_t pad[8];
};

// Workspace: [WorkHeader][fwd items int2 x max_f][bwd items int2 x max_b]
// [dS block base per segment, int64 x (nseg + 1)] ...
// [per-CTA d_ts_weights / d_pos_weights partial bins, fp32 kBinsPerCta each]
constexpr int kBinsPerCta = 256 + 1024;
struct WorkLists {
  WorkHeader* hdr;
  int2* fwd;
  int2* bwd;
  int64_t* ds_base;
  float* bins;        // per-CTA fp32 bins (dK/dV kernel, reductions)
  double* partials;   // per-CTA fp64 totals [grid][kBinsPerCta], summed by the dQ kernel
  // dK/dV -> dQ dependency counters (the dQ kernel starts while dK/dV finishes):
  // dep[0] = finished dK/dV CTAs, dep[kDepBase + s*H + h] = finished kv tiles of (s, h)
  int32_t* dep;
  int32_t dep_heads;
  int32_t fwd_pairs;  // 1: fwd items are pairs of q tiles (s, u) = tiles 2u, 2u+1 (two-tile forward)
};
constexpr int kDepBase = 16;

// Band table: the exact bucket of every (q, kv) pair near the diagonal,
// computed once per call for all heads and read by the fused kernels' general
// chunks instead of per-element bucketization.  The chunk grid is the one both
// kernels classify on: 32-row q groups a (q rows 32a.. of segment s, stored
// at index floor(q_row0 / 32) + s + a: collision-free, bounded by
// q_rows / 32 + nseg, and computable without a prefix sum) x
// 32-column kv groups b.  For q group a with diagonal kv group
// bd(a) = floor((qp0 + 32a) / 32), the window holds kv groups
// b = bd - 3 .. bd + 1 (wi = b - bd + 3).  A chunk is 2 KB: [32 q][32 kv]
// bytes then the transpose [32 kv][32 q].  Byte = bucket, or kBandMasked for a
// pair outside the causal / jagged mask (or past the segment's rows).
constexpr int kTbBuckets = 24;  // >= the fused kernels' num_buckets limit (23)
constexpr int kBandNW = 5;
constexpr int kBandChunk = 2048;
constexpr uint32_t kBandMasked = 31;
JH_DEV int band_wi(const Seg& g, int64_t a, int64_t b) { return (int)(b - ((g.qp0 >> 5) + a) + 3); }
JH_DEV int64_t band_group(const Seg& g, int64_t s, int64_t a) { return (g.q_row0 >> 5) + s + a; }
JH_DEV const uint8_t* band_chunk(const uint8_t* band, int64_t qgroup_global, int wi) {
  return band + (qgroup_global * kBandNW + wi) * (int64_t)kBandChunk;
}

// Backward dS scratch: per (segment, head) the causal triangle of blocks, one
// per (128-row kv tile j, 64-row q half t) with t >= ds_tlo(j) (the first
// half that sees tile j, rounded down to even so the dQ kernel can read
// halves in pairs), each the bf16 dS^T tile [128 kv][64 q] (16 KB,
// row-major).  Block (s, h, j, t) = ds_base[s] * H + h * ds_cnt(s) +
// ds_off(j) + t - ds_tlo(j), ds_off(j) = sum_{j' < j} (nh - ds_tlo(j')) in
// closed form (ds_tlo(j) = 2 max(0, j - ceil(qp0 / 128))).
constexpr int kDsBlockBytes = 128 * 64 * 2;
JH_DEV int ds_nkt(const Seg& g) { return (int)((seg_kv_vis(g) + kBN - 1) / kBN); }
JH_DEV int ds_nh(const Seg& g) { return (int)((g.lq + 63) / 64); }
JH_DEV int ds_tlo(const Seg& g, int j) {
  const int64_t f = (int64_t)j * kBN - g.qp0;
  return f <= 0 ? 0 : (int)(f / kBN) * 2;
}
JH_DEV int64_t ds_off(const Seg& g, int j) {
  const int64_t m = (g.qp0 + kBN - 1) / kBN;
  const int64_t x = (int64_t)j - 1 - m;
  return (int64_t)j * ds_nh(g) - (x >= 0 ? x * (x + 1) : 0);
}
JH_DEV int64_t ds_cnt(const Seg& g) { return ds_off(g, ds_nkt(g)); }
// first block of (segment s, head h, kv tile j) minus its first half: block of half t = this + t
JH_DEV int64_t ds_block0(const WorkLists& wl, const Seg& g, int64_t s, int h, int H, int j) {
  return wl.ds_base[s] * H + (int64_t)h * ds_cnt(g) + ds_off(g, j) - ds_tlo(g, j);
}

constexpr int kLevels = 1024;  // work-size histogram levels (one per builder thread)

// Block-wide exclusive scan of one value per thread (1024 threads); returns the
// exclusive prefix, *total gets the block sum.
template <typename T>
JH_DEV T block_exclusive_scan(T v, T* warp_sum, T* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  T incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) warp_sum[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    T x = warp_sum[lane], xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T y = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi += y;
    }
    warp_sum[lane] = xi - x;
    if (lane == 31) warp_sum[32] = xi;
  }
  __syncthreads();
  const T r = warp_sum[wid] + incl - v;
  *total = warp_sum[32];
  __syncthreads();
  return r;
}

// One block of 1024 threads.  fwd items (s, q_tile) ordered by #kv tiles
// descending; bwd items (s, kv_tile) ordered by #q tiles descending (counting
// sort over a 1024-level histogram).  A group of G lanes (G = the largest power
// of two <= 32 with num_segments * G <= 1024) shares a segment and strides over
// its tiles, so a few long sequences do not serialise on one thread each (C4:
// 64 q tiles + 64 kv tiles per sequence, 42 us with one thread per segment).  q tiles that see no kv at all (a
// segment with kv_len 0) are not items: a run of such items could otherwise
// stall the persistent kernels' 2-deep item ring (their output rows are zeroed
// by the host in the segment form, the only form where they occur).  The segment each thread owns first is
// decoded once and kept in registers across the passes.
static __global__ void __launch_bounds__(1024, 1) build_work_kernel(SegArgs sa, WorkLists wl,
                                                                   unsigned long long* stamp = nullptr) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the attention kernel's prologue may start
  if (stamp != nullptr && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    stamp[3072] = t;
  }
  __shared__ int hist_f[kLevels], hist_b[kLevels];
  __shared__ int isum[33];
  __shared__ long long lsum[33];
  const int tid = threadIdx.x;
  hist_f[tid] = 0;
  hist_b[tid] = 0;
  int G = 1;
  while (G < 32 && sa.num_segments * (int64_t)(2 * G) <= (int64_t)blockDim.x) G <<= 1;
  const int sub = tid & (G - 1);
  const int64_t s0 = tid / G, sstride = blockDim.x / G;
  const bool own = s0 < sa.num_segments;
  Seg g0{};
  if (own) g0 = load_seg(sa, s0);
  __syncthreads();
  auto seg = [&](int64_t s) { return s == s0 ? g0 : load_seg(sa, s); };
  auto bwd_w = [](const Seg& g, int j) {
    int64_t first = (int64_t)j * kBN - g.qp0;
    first = first < 0 ? 0 : first;
    return (int)((g.lq - first + kBM - 1) / kBM);
  };
  const int fstep = wl.fwd_pairs ? 2 : 1;
  for (int64_t s = s0; s < sa.num_segments; s += sstride) {
    const Seg g = seg(s);
    const int nt = (int)((g.lq + kBM - 1) / kBM);
    for (int t = sub * fstep; t < nt; t += G * fstep) {
      const int w = (int)((fwd_kv_lim(g, min(t + fstep - 1, nt - 1)) + kBN - 1) / kBN);
      if (w > 0) atomicAdd(&hist_f[min(w, kLevels - 1)], 1);  // (tiles that see no kv are not items)
    }
    const int nj = (int)((seg_kv_vis(g) + kBN - 1) / kBN);
    for (int j = sub; j < nj; j += G) atomicAdd(&hist_b[min(bwd_w(g, j), kLevels - 1)], 1);
  }
  __syncthreads();
  // descending starts: level L starts after all items of levels > L
  {
    const int lvl = kLevels - 1 - tid;
    const int cf = hist_f[lvl], cb = hist_b[lvl];
    int tf, tb;
    const int sf = block_exclusive_scan(cf, isum, &tf);
    const int sb = block_exclusive_scan(cb, isum, &tb);
    hist_f[lvl] = sf;
    hist_b[lvl] = sb;
    if (tid == 0) {
      wl.hdr->n_fwd = tf;
      wl.hdr->n_bwd = tb;
      wl.hdr->next_item[0] = wl.hdr->next_item[1] = wl.hdr->next_item[2] = 0;
    }
  }
  __syncthreads();
  for (int64_t s = s0; s < sa.num_segments; s += sstride) {
    const Seg g = seg(s);
    const int nt = (int)((g.lq + kBM - 1) / kBM);
    for (int t = sub * fstep; t < nt; t += G * fstep) {
      const int w = (int)((fwd_kv_lim(g, min(t + fstep - 1, nt - 1)) + kBN - 1) / kBN);
      if (w > 0) wl.fwd[atomicAdd(&hist_f[min(w, kLevels - 1)], 1)] = make_int2((int)s, t / fstep);
    }
    const int nj = (int)((seg_kv_vis(g) + kBN - 1) / kBN);
    for (int j = sub; j < nj; j += G) wl.bwd[atomicAdd(&hist_b[min(bwd_w(g, j), kLevels - 1)], 1)] = make_int2((int)s, j);
  }
  // dS scratch: exclusive scan of the per-segment block counts (chunks of 1024)
  if (wl.ds_base != nullptr) {
    long long carry = 0;
    for (int64_t base = 0; base < sa.num_segments; base += blockDim.x) {
      const int64_t s = base + tid;
      long long v = 0;
      if (s < sa.num_segments) {
        const Seg g = load_seg(sa, s);
        v = (long long)ds_cnt(g);
      }
      long long tot;
      const long long ex = block_exclusive_scan(v, lsum, &tot);
      if (s < sa.num_segments) wl.ds_base[s] = carry + ex;
      carry += tot;
    }
    if (wl.dep != nullptr)
      for (int64_t i = tid; i < kDepBase + sa.num_segments * wl.dep_heads; i += blockDim.x) wl.dep[i] = 0;
    if (tid == 0) {
      wl.ds_base[sa.num_segments] = carry;
      wl.hdr->ds_blocks = carry;
      wl.hdr->ds_overflow = 0;
    }
  }
  if (stamp != nullptr) {
    __syncthreads();
    if (tid == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      stamp[3073] = t;
    }
  }
  // (launched as a programmatic dependent of the band-table kernel: completing
  // only after it keeps the attention kernels' single griddepcontrol.wait sufficient)
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Band table builder: one warp per (q group, window chunk); lane = q row for
// the [q][kv] half, lane = kv column for the transposed half.  Chunks the
// kernels classify as fully masked (past the kv range or entirely in the
// future of the q group) are never read and not written.
static __global__ void __launch_bounds__(256) band_table_kernel(SegArgs sa, const int64_t* __restrict__ ts_q,
                                                               const int64_t* __restrict__ ts_k, DevBiasTable bt,
                                                               uint8_t* __restrict__ band) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the work-list build may start
  __shared__ SmemBias sb;
  __shared__ uint8_t tr[8][32][36];
  smem_bias_fill(&sb, bt, threadIdx.x, blockDim.x);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t w = (int64_t)blockIdx.x * 8 + warp;
  const int64_t g = w / kBandNW;
  const int wi = (int)(w % kBandNW);
  const int64_t nseg = sa.num_segments;
  if (nseg <= 0) return;
  // segment: last s with f(s) = floor(q_row0(s) / 32) + s <= g (f strictly
  // increasing); 32-ary warp search, one dependent load per level
  int64_t lo = 0, hi = nseg - 1;
  while (lo < hi) {
    const int64_t step = (hi - lo + 32) / 32;
    const int64_t idx = min(lo + (int64_t)lane * step, hi);
    const bool le = (sa.q_offsets[idx] >> 5) + idx <= g;
    const uint32_t m = __ballot_sync(0xffffffffu, le);
    if (m == 0) return;  // g precedes segment lo (cannot happen for lo = 0)
    const int64_t best = min(lo + (int64_t)(31 - __clz(m)) * step, hi);
    lo = best;
    hi = min(best + step - 1, hi);
  }
  const Seg sg = load_seg(sa, lo);
  const int64_t a = g - ((sg.q_row0 >> 5) + lo);
  if (a < 0 || 32 * a >= sg.lq) return;  // no q group at this index
  const int64_t k0 = 32 * ((sg.qp0 >> 5) + a + wi - 3);
  if (k0 < 0 || k0 >= sg.kv_len || k0 > sg.qp0 + 32 * a + 31) return;
  const int64_t r = 32 * a + lane;
  const int64_t qpos = sg.qp0 + r;
  const bool rok = r < sg.lq;
  const int64_t tq = rok ? ts_q[sg.q_row0 + r] : 0;
  const int64_t tk = k0 + lane < sg.kv_len ? ts_k[sg.kv_row0 + k0 + lane] : 0;
  // chunks the kernels classify as saturated (fully visible, every pair in the
  // last bucket by the same chunk-level min / max test) are never read either
  {
    const int64_t tq_min = warp_min_i64(rok ? tq : (INT64_MAX >> 2));
    const int64_t tk_max = warp_max_i64(k0 + lane < sg.kv_len ? tk : (INT64_MAX >> 2));
    if (k0 + 31 < sg.kv_len && k0 + 31 <= sg.qp0 + 32 * a && tq_min - tk_max >= bt.cap) return;
  }
  uint32_t wd[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) wd[i] = 0u;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int64_t tki = __shfl_sync(0xffffffffu, tk, i);
    const int64_t k = k0 + i;
    const bool ok = rok && k < sg.kv_len && k <= qpos;
    const uint32_t byte = ok ? (uint32_t)bucket_smem(tq - tki, &sb, bt.cap) : kBandMasked;
    wd[i >> 2] |= byte << (8 * (i & 3));
    tr[warp][lane][i] = (uint8_t)byte;
  }
  uint8_t* dst = band + (g * kBandNW + wi) * (int64_t)kBandChunk;
  uint4* d0 = reinterpret_cast<uint4*>(dst + lane * 32);
  d0[0] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
  d0[1] = make_uint4(wd[4], wd[5], wd[6], wd[7]);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 8; ++i) wd[i] = 0u;
#pragma unroll
  for (int i = 0; i < 32; ++i) wd[i >> 2] |= (uint32_t)tr[warp][i][lane] << (8 * (i & 3));
  uint4* d1 = reinterpret_cast<uint4*>(dst + 1024 + lane * 32);
  d1[0] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
  d1[1] = make_uint4(wd[4], wd[5], wd[6], wd[7]);
}

// q, k, v, dout (bf16 2-D, 128-row boxes) and ts_q, ts_k (int64 1-D) tensor maps
struct TMaps {
  CUtensorMap q, k, v, dout, tsq, tsk;
  CUtensorMap q64, do64, tsq72;  // 64-row boxes for the dKV kernel (q side)
  CUtensorMap k64, v64, tsk72;  // 64-row boxes for the dQ kernel (kv side)
  CUtensorMap ds;               // dS scratch as a [blocks * 128, 64] bf16 matrix, 128-row boxes
};

// Parameters shared by the fwd / bwd attention kernels.
struct AttnParams {
  SegArgs seg;
  const int64_t* ts_q;
  const int64_t* ts_k;
  const float* ts_weights;
  const float* pos_weights;
  int32_t num_pos;
  int32_t num_heads;
  int64_t q_rows, kv_rows;
  // fwd
  __nv_bfloat16* out;
  int64_t ld_o;
  float* out_acc;      // fp32 output (NULL: bf16 `out`), row stride ld_o
  int32_t out_acc_add; // 1: add into out_acc, 0: store
  // bwd
  __nv_bfloat16* dk;
  __nv_bfloat16* dv;
  int64_t ld_dk, ld_dv;
  float* dk_accum;
  float* dv_accum;
  float* dq_acc;          // fp32 dq accumulate (NULL: bf16 dq)
  double* d_ts_weights;
  double* d_pos_weights;
  const uint8_t* band;    // band table (NULL: per-element bucketization everywhere)
  float* tb_glob;         // dK/dV kernel: per-CTA thread-private bins [kTbBuckets][256] of the band chunks
  __nv_bfloat16* ds;      // dS scratch (kDsBlockBytes blocks)
  int64_t ds_cap_blocks;  // its capacity
  WorkLists wl;
  DevBiasTable bias;
  // debug timeline (NULL = off): CTA trace_cta records (code, arg, clock64)
  // per role into trace[role * kTraceCap * 2 ...]
  unsigned long long* trace;
  int32_t trace_cta;
  int32_t dbg;  // experiment switches (JH_DBG environment variable), 0 in production
  // fused backward (hstu_bwd_fused_kernel): persistent zero state
  float* dq_state;      // fp32 dQ accumulator [q_rows][H*D] (bf16-dq mode)
  int32_t* dq_cnt;      // per-(q tile, head) contribution counters
  int32_t* dw_done;     // last-CTA counter of the d_ts_weights reduction
  int32_t dbg_count;    // debug: d_ts_weights = exact pair count per bucket
  float c1;     // score_scale / 2: SiLU(s) = h + h tanh(h), h = c1 * (q k^T + bias)
  uint8_t* dbg_buckets;  // forward debug export of the applied bucket per (q row, kv pos), head 0
  int64_t dbg_ld;
};

constexpr int kTraceCap = 4096;

// Per-CTA start / end stamps (trace_cta == -1): trace[2*cta] = start, [2*cta+1] = end
// (globaltimer ns), for load-balance measurements.
JH_DEV void cta_stamp(const AttnParams& p, int which, int kernel = 0) {
  if (p.trace == nullptr || p.trace_cta != -1 || threadIdx.x != 0) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  p.trace[1024 * kernel + 2 * blockIdx.x + which] = t;
  p.trace[1024 * kernel + 512 + 2 * blockIdx.x + which] = (unsigned long long)clock64();
}

// Dynamic assignment of the longest-first work list to the persistent CTAs:
// one thread per CTA (the ring producer) takes the next item index from a
// global counter and publishes it in a small shared-memory ring that every
// other role of the CTA consumes in the same order (longest-processing-time-
// first scheduling without any static imbalance).
#ifndef JH_ITEM_RING
#define JH_ITEM_RING 2
#endif
constexpr int kItemRing = JH_ITEM_RING;
struct ItemRing {
  int32_t* slot;    // [kItemRing]
  uint64_t* full;   // [kItemRing], count 1
  uint64_t* empty;  // [kItemRing], count = number of consumers
};
JH_DEV void ring_init(const ItemRing& r, int consumers) {
  for (int i = 0; i < kItemRing; ++i) {
    mbar_init(&r.full[i], 1);
    mbar_init(&r.empty[i], consumers);
  }
}
// producer: returns the next item (or -1 when the list is exhausted)
JH_DEV int ring_produce(const ItemRing& r, uint32_t& k, int32_t* counter, int total) {
  const uint32_t s = k % kItemRing;
  mbar_wait(&r.empty[s], ((k / kItemRing) & 1) ^ 1);
  int g = atomicAdd(counter, 1);
  if (g >= total) g = -1;
  r.slot[s] = g;
  mbar_arrive(&r.full[s]);
  ++k;
  return g;
}
// consumer: a whole warp (lane 0 arrives for it) or a single thread
JH_DEV int ring_consume(const ItemRing& r, uint32_t& k, bool warp_wide) {
  const uint32_t s = k % kItemRing;
  mbar_wait(&r.full[s], (k / kItemRing) & 1);
  const int g = *reinterpret_cast<volatile int32_t*>(&r.slot[s]);
  if (warp_wide) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&r.empty[s]);
  } else {
    mbar_arrive(&r.empty[s]);
  }
  ++k;
  return g;
}

// Static "snake" assignment of the longest-first work list to the persistent
// CTAs: round k hands items [k*grid, (k+1)*grid) to CTAs in alternating
// direction, which balances the per-CTA sums of the sorted item sizes far
// better than plain round-robin.  Every role of a CTA walks the same sequence.
JH_DEV int snake_item(int k) {
  const int b = (k & 1) ? (int)gridDim.x - 1 - (int)blockIdx.x : (int)blockIdx.x;
  return k * (int)gridDim.x + b;
}
#define JH_FOR_ITEMS(g, total) for (int _k = 0, g; (g = snake_item(_k)) < (total); ++_k)

// One event from the calling thread (callers pass only one thread per role).
JH_DEV void trace_ev(const AttnParams& p, int role, uint32_t& cnt, uint32_t code, uint32_t arg) {
  if (p.trace == nullptr || (int)blockIdx.x != p.trace_cta || cnt >= (uint32_t)kTraceCap) return;  // (-1: stamps)
  unsigned long long* t = p.trace + ((size_t)role * kTraceCap + cnt) * 2;
  t[0] = ((unsigned long long)code << 32) | arg;
  t[1] = (unsigned long long)clock64();
  ++cnt;
}

}  // namespace jh
