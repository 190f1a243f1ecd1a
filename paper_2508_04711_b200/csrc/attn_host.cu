// Host launch code for the attention kernels (jh_attn_fwd / jh_attn_bwd):
// argument validation, tensor maps, work-list build, kernel launches.
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>

#include "abi_internal.h"
#include "attn_common.cuh"
#include "tmap.h"

namespace jh {

template <int D>
int launch_fwd(const CUtensorMap&, const CUtensorMap&, const CUtensorMap&, const CUtensorMap&, const CUtensorMap&,
               const AttnParams&, int, cudaStream_t, void*, void*);
template <int D>
int launch_fwd2(const CUtensorMap&, const CUtensorMap&, const CUtensorMap&, const CUtensorMap&, const CUtensorMap&,
                const AttnParams&, int, cudaStream_t, void*, void*);
template <int D>
int launch_bwd(const TMaps&, const AttnParams&, const jh_attn_args&, int, cudaStream_t);
template <int D>
int launch_bwd_fused(const TMaps&, const AttnParams&, const jh_attn_args&, int, cudaStream_t);

static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

struct WsLayout {
  size_t items_f, items_b, ds_base, bins, total;
};

static size_t bins_bytes() { return (size_t)sm_count() * kBinsPerCta * (4 + 8); }  // fp32 bins + fp64 totals
static size_t band_bytes(int64_t q_rows, int64_t nseg) {
  return (size_t)(q_rows / 32 + nseg + 1) * kBandNW * kBandChunk;
}
static size_t band_groups_bound(int64_t q_rows, int64_t nseg) { return (size_t)(q_rows / 32 + nseg); }
static size_t tbglob_bytes() { return (size_t)sm_count() * kTbBuckets * 256 * 4; }
// regions carved from the END of the workspace (the bwd item list in front is
// bounded by the caller's kv total): band table, per-CTA band bins,
// dependency counters, dS block bases, per-CTA bins
static size_t tail_bytes(int64_t q_rows, int64_t nseg, int32_t H) {
  auto up = [](size_t x) { return (x + 255) / 256 * 256; };
  return band_bytes(q_rows, nseg) + tbglob_bytes() + up((size_t)(kDepBase + nseg * H) * 4) + up((size_t)(nseg + 1) * 8) + bins_bytes() + 1024;
}

static WsLayout ws_layout(int64_t q_rows, int64_t kv_total, int64_t nseg, int32_t H, int32_t D) {
  WsLayout w;
  int64_t max_f = q_rows / kBM + nseg + 1;
  int64_t max_b = kv_total / kBN + nseg + 1;
  w.items_f = sizeof(WorkHeader);
  w.items_b = w.items_f + ((size_t)max_f * 8 + 255) / 256 * 256;
  w.ds_base = w.items_b + ((size_t)max_b * 8 + 255) / 256 * 256;
  w.bins = w.ds_base;
  w.total = w.ds_base + tail_bytes(q_rows, nseg, H);
  return w;
}

// Fused-backward persistent state (zero between calls): fp32 dQ accumulator
// [q_rows][H*d], per-(q tile, head) contribution counters at index
// ((q_row0 >> 7) + s + t) * H + h (collision-free without a prefix sum), and
// the d_ts_weights last-CTA counter.
struct BwdStateLayout {
  size_t acc, cnt, done, total;
};
static BwdStateLayout bwd_state_layout(int64_t q_rows, int64_t nseg, int32_t H, int32_t D) {
  auto up = [](size_t x) { return (x + 255) / 256 * 256; };
  BwdStateLayout l;
  l.acc = 0;
  l.cnt = up((size_t)q_rows * H * D * 4);
  l.done = l.cnt + up((size_t)(q_rows / 128 + nseg + 2) * H * 4);
  l.total = l.done + 256;
  return l;
}

// Forward kernel: the one-tile kernel (attn_fwd.cu); JH_FWD2=1 selects the
// two-q-tile kernel (attn_fwd2.cu) for A/B measurements (C2: 45 vs 38 us per
// launch under ncu, r2 launch list -- the pair items halve L2 bytes per flop
// but double the per-item latency chain and coarsen the tail).
static bool fwd_two_tile() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("JH_FWD2");
    v = (e && atoi(e) == 1) ? 1 : 0;
  }
  return v == 1;
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

static int validate(const jh_attn_args* a, bool bwd) {
  if (!a) return set_error(JH_ERR_INVALID, "args is NULL");
  if (a->head_dim != 64 && a->head_dim != 128)
    return set_error(JH_ERR_UNSUPPORTED, "head_dim %d unsupported (64 or 128)", a->head_dim);
  if (a->num_heads < 1) return set_error(JH_ERR_INVALID, "num_heads must be >= 1");
  if (a->num_segments < 0 || a->q_rows < 0 || a->kv_rows < 0) return set_error(JH_ERR_INVALID, "negative size");
  if (a->num_segments >= (int64_t(1) << 31)) return set_error(JH_ERR_UNSUPPORTED, "too many segments");
  if (a->q_rows >= (int64_t(1) << 31) || a->kv_rows >= (int64_t(1) << 31))
    return set_error(JH_ERR_UNSUPPORTED, "more than 2^31 rows");
  if (a->num_buckets < 1 || a->num_buckets > 256)
    return set_error(JH_ERR_INVALID, "num_buckets must be in [1, 256]");
  if (!a->ts_weights) return set_error(JH_ERR_INVALID, "ts_weights is NULL");
  if (a->num_pos < 0 || a->num_pos > 1024) return set_error(JH_ERR_UNSUPPORTED, "num_pos must be in [0, 1024]");
  if (a->num_pos > 0 && !a->pos_weights) return set_error(JH_ERR_INVALID, "pos_weights is NULL");
  if (!a->q_offsets) return set_error(JH_ERR_INVALID, "q_offsets is NULL");
  if (!(a->score_scale >= 0.f) || a->score_scale > 1e30f) return set_error(JH_ERR_INVALID, "score_scale must be finite and >= 0");
  if (a->dbg_buckets && a->dbg_ld < 1) return set_error(JH_ERR_INVALID, "dbg_ld must be >= 1");
  const int64_t HD = (int64_t)a->num_heads * a->head_dim;
  if (a->q_rows > 0 || a->kv_rows > 0) {
    if (!a->q || !a->k || !a->v || !a->ts_q || !a->ts_k) return set_error(JH_ERR_INVALID, "NULL input tensor");
    if (a->ld_q < HD || a->ld_k < HD || a->ld_v < HD) return set_error(JH_ERR_INVALID, "row stride < H*d");
    if ((a->ld_q * 2) % 16 || (a->ld_k * 2) % 16 || (a->ld_v * 2) % 16)
      return set_error(JH_ERR_INVALID, "row strides must be multiples of 16 bytes");
    if (!aligned16(a->q) || !aligned16(a->k) || !aligned16(a->v))
      return set_error(JH_ERR_INVALID, "q/k/v must be 16-byte aligned");
  }
  if (!bwd) {
    if (a->out_accum_mode < 0 || a->out_accum_mode > 2) return set_error(JH_ERR_INVALID, "bad out_accum_mode");
    if (a->out_accum_mode != 0) {
      if (a->q_rows > 0 && (!a->out_accum || a->ld_o < HD || (a->ld_o * 4) % 16 || !aligned16(a->out_accum)))
        return set_error(JH_ERR_INVALID, "bad out_accum tensor");
    } else if (a->q_rows > 0 && (!a->out || a->ld_o < HD || (a->ld_o * 2) % 16 || !aligned16(a->out))) {
      return set_error(JH_ERR_INVALID, "bad out tensor");
    }
  } else {
    if (!a->d_ts_weights) return set_error(JH_ERR_INVALID, "d_ts_weights is NULL");
    if (a->num_pos > 0 && !a->d_pos_weights) return set_error(JH_ERR_INVALID, "d_pos_weights is NULL");
    if (a->q_rows > 0 && (!a->dout || !(a->dq || a->dq_accum) || a->ld_do < HD || a->ld_dq < HD ||
                          (a->ld_do * 2) % 16 || !aligned16(a->dout)))
      return set_error(JH_ERR_INVALID, "bad dout/dq tensor");
    if (a->q_rows > 0 && a->dq_accum && ((a->ld_dq * 4) % 16 || !aligned16(a->dq_accum)))
      return set_error(JH_ERR_INVALID, "bad dq_accum tensor");
    if (a->kv_rows > 0) {
      if (!a->dk_accum && (!a->dk || a->ld_dk < HD)) return set_error(JH_ERR_INVALID, "bad dk tensor");
      if (!a->dv_accum && (!a->dv || a->ld_dv < HD)) return set_error(JH_ERR_INVALID, "bad dv tensor");
    }
  }
  WsLayout w = ws_layout(a->q_rows, a->q_rows, a->num_segments, a->num_heads, a->head_dim);
  if (!a->workspace || a->workspace_bytes < w.total)
    return set_error(JH_ERR_INVALID, "workspace too small (need >= %zu bytes)", w.total);
  if (bwd && a->q_rows > 0 && a->deterministic &&
      (!a->ds_scratch || a->ds_scratch_bytes < (size_t)kDsBlockBytes || !aligned16(a->ds_scratch)))
    return set_error(JH_ERR_INVALID, "ds_scratch missing or too small (see jh_attn_ds_scratch_bytes)");
  if (bwd && a->q_rows > 0 && !a->deterministic) {
    const int D = a->head_dim;
    if (!a->bwd_state || (uintptr_t)a->bwd_state % 256 ||
        a->bwd_state_bytes < bwd_state_layout(a->q_rows, a->num_segments, a->num_heads, D).total)
      return set_error(JH_ERR_INVALID, "bwd_state missing, misaligned or too small (see jh_attn_bwd_state_bytes)");
    if (!a->dq_accum && (a->ld_dq * 2) % 16) return set_error(JH_ERR_INVALID, "dq row stride must be 16-byte aligned");
  }
  return JH_OK;
}

static int prepare(const jh_attn_args* a, bool bwd, AttnParams* p, TMaps* tm, cudaStream_t s) {
  const BiasTable* bt = bias_table_cached(a->num_buckets);
  if (!bt) return set_error(JH_ERR_INVALID, "num_buckets must be >= 1");
  if (bt->cap >= 0xFFFFFFFFll)
    return set_error(JH_ERR_UNSUPPORTED, "fused attention supports num_buckets <= 23 (got %d)", a->num_buckets);
  memset(p, 0, sizeof(*p));
  p->seg = SegArgs{a->q_offsets, a->q_pos0, a->kv_start, a->kv_len, a->num_segments};
  p->ts_q = a->ts_q;
  p->ts_k = a->ts_k;
  p->ts_weights = a->ts_weights;
  p->pos_weights = a->pos_weights;
  p->num_pos = a->num_pos;
  p->num_heads = a->num_heads;
  p->q_rows = a->q_rows;
  p->kv_rows = a->kv_rows;
  p->out = (__nv_bfloat16*)a->out;
  p->ld_o = a->ld_o;
  p->out_acc = (!bwd && a->out_accum_mode != 0) ? a->out_accum : nullptr;
  p->out_acc_add = a->out_accum_mode == 2 ? 1 : 0;
  p->dk = (__nv_bfloat16*)a->dk;
  p->dv = (__nv_bfloat16*)a->dv;
  p->ld_dk = a->ld_dk;
  p->ld_dv = a->ld_dv;
  p->dk_accum = a->dk_accum;
  p->dq_acc = bwd ? a->dq_accum : nullptr;
  p->dv_accum = a->dv_accum;
  p->d_ts_weights = a->d_ts_weights;
  p->d_pos_weights = a->d_pos_weights;
  for (int i = 0; i < 64; ++i) {
    p->bias.thr[i] = bt->thr[i];
    p->bias.base[i] = bt->base[i];
  }
  p->bias.cap = bt->cap;
  p->bias.nb = a->num_buckets;
  p->c1 = 0.5f * (a->score_scale > 0.f ? a->score_scale : 1.0f / sqrtf((float)a->head_dim));
  p->dbg_buckets = bwd ? nullptr : a->dbg_buckets;
  p->dbg_ld = a->dbg_ld;
  p->trace = (unsigned long long*)a->trace;
  p->trace_cta = a->trace_cta;
  {
    const char* e = getenv("JH_DBG");
    p->dbg = e ? atoi(e) : 0;
  }
  // workspace carve-up (bound computed with the caller's kv total unknown:
  // the bwd list is placed after a q_rows-sized fwd list, see ws_layout)
  WsLayout w = ws_layout(a->q_rows, std::max<int64_t>(a->q_rows, 0), a->num_segments, a->num_heads, a->head_dim);
  uint8_t* ws = (uint8_t*)a->workspace;
  p->wl.hdr = (WorkHeader*)ws;
  p->wl.fwd = (int2*)(ws + w.items_f);
  p->wl.bwd = (int2*)(ws + w.items_b);
  const bool det = bwd && a->deterministic;
  p->ds = det ? (__nv_bfloat16*)a->ds_scratch : nullptr;
  p->ds_cap_blocks = det ? (int64_t)(a->ds_scratch_bytes / kDsBlockBytes) : 0;
  if (bwd && !det) {
    const BwdStateLayout sl = bwd_state_layout(a->q_rows, a->num_segments, a->num_heads, a->head_dim);
    uint8_t* st = (uint8_t*)a->bwd_state;
    p->dq_state = (float*)(st + sl.acc);
    p->dq_cnt = (int32_t*)(st + sl.cnt);
    p->dw_done = (int32_t*)(st + sl.done);
  }
  p->dbg_count = bwd ? a->dbg_count_buckets : 0;
  // per-CTA gradient bins at the end of the caller's workspace
  // (the bwd item list is bounded by the caller's kv total, unknown here: the
  // dS block bases and the per-CTA bins are carved from the end of the workspace)
  const size_t bins_off = (a->workspace_bytes - bins_bytes()) & ~size_t(255);
  const size_t dsb_off = (bins_off - (size_t)(a->num_segments + 1) * 8) & ~size_t(255);
  const size_t dep_off = (dsb_off - (size_t)(kDepBase + a->num_segments * a->num_heads) * 4) & ~size_t(255);
  p->wl.dep = det ? (int32_t*)(ws + dep_off) : nullptr;
  p->wl.dep_heads = a->num_heads;
  p->wl.fwd_pairs = (!bwd && fwd_two_tile()) ? 1 : 0;
  p->wl.bins = bwd ? (float*)(ws + bins_off) : nullptr;
  p->wl.partials = bwd ? (double*)(ws + bins_off + (size_t)sm_count() * kBinsPerCta * 4) : nullptr;
  p->wl.ds_base = det ? (int64_t*)(ws + dsb_off) : nullptr;
  const size_t tbg_off = (dep_off - tbglob_bytes()) & ~size_t(255);
  const size_t band_off = (tbg_off - band_bytes(a->q_rows, a->num_segments)) & ~size_t(255);
  if (band_off < w.items_b + 8 || band_off > a->workspace_bytes) return set_error(JH_ERR_INVALID, "workspace too small");
  // band table (exact buckets near the diagonal, shared by all heads); off with
  // a positional bias (its general chunks keep the per-element path) or JH_DBG & 4
  const bool use_band = a->num_pos == 0 && !(p->dbg & 4);
  p->band = use_band ? (const uint8_t*)(ws + band_off) : nullptr;
  bool band_ready = false;
  if (use_band && a->band_table != nullptr) {
    if (a->band_table_bytes < band_bytes(a->q_rows, a->num_segments) || (uintptr_t)a->band_table % 16)
      return set_error(JH_ERR_INVALID, "band_table smaller than jh_attn_band_table_bytes() or misaligned");
    p->band = (const uint8_t*)a->band_table;
    band_ready = a->band_table_ready != 0;
  }
  p->tb_glob = bwd ? (float*)(ws + tbg_off) : nullptr;
  const uint64_t HD = (uint64_t)a->num_heads * a->head_dim;
  if ((uintptr_t)a->ts_q % 16 || (uintptr_t)a->ts_k % 16)
    return set_error(JH_ERR_INVALID, "ts_q / ts_k must be 16-byte aligned");
  if (make_tmap_bf16_2d(&tm->q, a->q, a->q_rows, HD, a->ld_q, 128) ||
      make_tmap_bf16_2d(&tm->k, a->k, a->kv_rows, HD, a->ld_k, 128) ||
      make_tmap_bf16_2d(&tm->v, a->v, a->kv_rows, HD, a->ld_v, 128) ||
      make_tmap_i64_1d(&tm->tsq, a->ts_q, a->q_rows, kTsBox) ||
      make_tmap_i64_1d(&tm->tsk, a->ts_k, a->kv_rows, kTsBox))
    return set_error(JH_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  if (bwd && make_tmap_bf16_2d(&tm->dout, a->dout, a->q_rows, HD, a->ld_do, 128))
    return set_error(JH_ERR_CUDA, "cuTensorMapEncodeTiled failed (dout)");
  if (det && (make_tmap_bf16_2d(&tm->q64, a->q, a->q_rows, HD, a->ld_q, 64) ||
              make_tmap_bf16_2d(&tm->do64, a->dout, a->q_rows, HD, a->ld_do, 64) ||
              make_tmap_i64_1d(&tm->tsq72, a->ts_q, a->q_rows, kTsBoxH) ||
              make_tmap_bf16_2d(&tm->k64, a->k, a->kv_rows, HD, a->ld_k, 64) ||
              make_tmap_bf16_2d(&tm->v64, a->v, a->kv_rows, HD, a->ld_v, 64) ||
              make_tmap_i64_1d(&tm->tsk72, a->ts_k, a->kv_rows, kTsBoxH) ||
              make_tmap_bf16_2d(&tm->ds, a->ds_scratch, (uint64_t)p->ds_cap_blocks * 128, 64, 64, 128)))
    return set_error(JH_ERR_CUDA, "cuTensorMapEncodeTiled failed (bwd maps)");
  static bool carve = false;
  if (!carve) {
    cudaFuncSetAttribute(build_work_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    carve = true;
  }
  // band table first (it only reads the inputs; a plain launch, so it also
  // waits for the previous attention kernel, the table's last reader), then the
  // work-list build as its programmatic dependent (runs concurrently; it waits
  // for the table at its end, so the attention kernel's wait covers both)
  cudaError_t e;
  if (p->band && !band_ready) {
    const size_t warps = (band_groups_bound(a->q_rows, a->num_segments) + 1) * kBandNW;
    band_table_kernel<<<(unsigned)((warps + 7) / 8), 256, 0, s>>>(p->seg, a->ts_q, a->ts_k, p->bias, (uint8_t*)p->band);
    e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(JH_ERR_CUDA, "band_table: %s", cudaGetErrorString(e));
  }
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(1024);
    cfg.stream = s;
    cudaLaunchAttribute la[1];
    la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    la[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = la;
    cfg.numAttrs = (p->band && !band_ready) ? 1 : 0;
    e = cudaLaunchKernelEx(&cfg, build_work_kernel, p->seg, p->wl,
                           (unsigned long long*)(p->trace_cta == -1 ? p->trace : nullptr));
    if (e != cudaSuccess) return set_error(JH_ERR_CUDA, "build_work: %s", cudaGetErrorString(e));
  }
  return JH_OK;
}

}  // namespace jh

using namespace jh;

extern "C" {

size_t jh_attn_band_table_bytes(int64_t q_rows, int64_t num_segments) {
  return band_bytes(std::max<int64_t>(q_rows, 0), std::max<int64_t>(num_segments, 0));
}

size_t jh_attn_ds_scratch_bytes(int64_t kv_len_total, int64_t num_segments, int32_t num_heads, int64_t max_len) {
  // per segment ds_cnt <= nkt * nh with nkt = ceil(kv_s / 128) and
  // nh = ceil(q_s / 64): summed <= (sum nkt) * max nh <= (ceil(kv_total / 128)
  // + nseg) * ceil(max_len / 64), max_len >= every segment's kv AND q length
  // (a CP "remote" segment can have q_s > kv_s).  About twice the exact size
  // for self-attention: callers that know the segments use the _segs form.
  if (kv_len_total <= 0 || num_segments <= 0 || num_heads <= 0 || max_len <= 0) return (size_t)kDsBlockBytes;
  const int64_t blocks = ((kv_len_total + kBN - 1) / kBN + num_segments) * ((max_len + 63) / 64);
  return (size_t)blocks * num_heads * kDsBlockBytes;
}

size_t jh_attn_ds_scratch_bytes_segs(const int64_t* q_offsets, const int64_t* q_pos0, const int64_t* kv_len,
                                     int64_t num_segments, int32_t num_heads) {
  // host mirror of ds_cnt (attn_common.cuh), summed: the exact block count the
  // work-list builder's scan produces
  if (!q_offsets || num_segments <= 0 || num_heads <= 0) return (size_t)kDsBlockBytes;
  int64_t blocks = 0;
  for (int64_t s = 0; s < num_segments; ++s) {
    const int64_t lq = q_offsets[s + 1] - q_offsets[s];
    const int64_t qp0 = q_pos0 ? q_pos0[s] : 0;
    const int64_t kvl = kv_len ? kv_len[s] : lq;
    if (lq <= 0) continue;
    const int64_t vis = std::min(qp0 + lq, kvl);
    const int64_t nkt = vis > 0 ? (vis + kBN - 1) / kBN : 0;
    const int64_t nh = (lq + 63) / 64;
    const int64_t m = (qp0 + kBN - 1) / kBN;
    const int64_t x = nkt - 1 - m;
    blocks += nkt * nh - (x >= 0 ? x * (x + 1) : 0);
  }
  return (size_t)std::max<int64_t>(blocks, 1) * num_heads * kDsBlockBytes;
}

size_t jh_attn_bwd_state_bytes(int64_t q_rows, int64_t num_segments, int32_t num_heads, int32_t head_dim) {
  q_rows = std::max<int64_t>(q_rows, 0);
  num_segments = std::max<int64_t>(num_segments, 0);
  num_heads = std::max<int32_t>(num_heads, 1);
  return bwd_state_layout(q_rows, num_segments, num_heads, head_dim < 64 ? 64 : (head_dim > 64 ? 128 : 64)).total;
}

size_t jh_attn_workspace_bytes(int64_t q_rows, int64_t kv_len_total, int64_t num_segments, int32_t num_heads,
                               int32_t head_dim) {
  // the layout is q_rows-bounded for the fwd list; the bwd list bound uses
  // max(kv_len_total, q_rows); per-CTA bins last
  int64_t kvt = std::max(kv_len_total, q_rows);
  WsLayout a = ws_layout(q_rows, q_rows, num_segments, num_heads, head_dim);
  WsLayout b = ws_layout(q_rows, kvt, num_segments, num_heads, head_dim);
  return std::max(a.total, b.total) + 256;
}

int jh_attn_band(const jh_attn_args* a, void* stream) {
  // the band table alone (exact near-diagonal buckets): reads q_offsets /
  // q_pos0 / kv_start / kv_len, ts_q, ts_k, num_buckets; writes a->band_table
  if (!a) return set_error(JH_ERR_INVALID, "args is NULL");
  if (a->num_segments < 0 || a->q_rows < 0) return set_error(JH_ERR_INVALID, "negative size");
  if (a->num_buckets < 1 || a->num_buckets > 256) return set_error(JH_ERR_INVALID, "num_buckets must be in [1, 256]");
  if (a->q_rows == 0 || a->num_segments == 0 || a->num_pos > 0) return JH_OK;  // (no band with a positional bias)
  if (!a->q_offsets || !a->ts_q || !a->ts_k) return set_error(JH_ERR_INVALID, "NULL q_offsets / ts_q / ts_k");
  if (!a->band_table || (uintptr_t)a->band_table % 16 ||
      a->band_table_bytes < band_bytes(a->q_rows, a->num_segments))
    return set_error(JH_ERR_INVALID, "band_table missing, smaller than jh_attn_band_table_bytes() or misaligned");
  const BiasTable* bt = bias_table_cached(a->num_buckets);
  if (!bt) return set_error(JH_ERR_INVALID, "num_buckets must be >= 1");
  if (bt->cap >= 0xFFFFFFFFll)
    return set_error(JH_ERR_UNSUPPORTED, "fused attention supports num_buckets <= 23 (got %d)", a->num_buckets);
  DevBiasTable bias;
  for (int i = 0; i < 64; ++i) {
    bias.thr[i] = bt->thr[i];
    bias.base[i] = bt->base[i];
  }
  bias.cap = bt->cap;
  bias.nb = a->num_buckets;
  const SegArgs seg{a->q_offsets, a->q_pos0, a->kv_start, a->kv_len, a->num_segments};
  const size_t warps = (band_groups_bound(a->q_rows, a->num_segments) + 1) * kBandNW;
  band_table_kernel<<<(unsigned)((warps + 7) / 8), 256, 0, (cudaStream_t)stream>>>(seg, a->ts_q, a->ts_k, bias,
                                                                                   (uint8_t*)a->band_table);
  cudaError_t e = cudaGetLastError();
  return e ? set_error(JH_ERR_CUDA, "band_table: %s", cudaGetErrorString(e)) : JH_OK;
}

int jh_attn_fwd(const jh_attn_args* a, void* stream) {
  int rc = validate(a, false);
  if (rc) return rc;
  if (a->q_rows == 0 || a->num_segments == 0) return JH_OK;
  cudaStream_t s = (cudaStream_t)stream;
  AttnParams p;
  TMaps tm;
  rc = prepare(a, false, &p, &tm, s);
  if (rc) return rc;
  if (a->q_pos0 || a->kv_len) {
    // segment form: q tiles of kv_len-0 segments are not work items -> zero rows
    // (store modes; the add mode leaves them untouched, as documented)
    cudaError_t e = cudaSuccess;
    const size_t HDe = (size_t)a->num_heads * a->head_dim;
    if (a->out_accum_mode == 1)
      e = cudaMemset2DAsync(a->out_accum, (size_t)a->ld_o * 4, 0, HDe * 4, (size_t)a->q_rows, s);
    else if (a->out_accum_mode == 0)
      e = cudaMemset2DAsync(a->out, (size_t)a->ld_o * 2, 0, HDe * 2, (size_t)a->q_rows, s);
    if (e != cudaSuccess) return set_error(JH_ERR_CUDA, "out memset: %s", cudaGetErrorString(e));
  }
  int grid = sm_count();
  int lr;
  if (p.wl.fwd_pairs)
    lr = a->head_dim == 64
             ? launch_fwd2<64>(tm.q, tm.k, tm.v, tm.tsq, tm.tsk, p, grid, s, a->prof_event_start, a->prof_event_end)
             : launch_fwd2<128>(tm.q, tm.k, tm.v, tm.tsq, tm.tsk, p, grid, s, a->prof_event_start, a->prof_event_end);
  else
    lr = a->head_dim == 64
             ? launch_fwd<64>(tm.q, tm.k, tm.v, tm.tsq, tm.tsk, p, grid, s, a->prof_event_start, a->prof_event_end)
             : launch_fwd<128>(tm.q, tm.k, tm.v, tm.tsq, tm.tsk, p, grid, s, a->prof_event_start, a->prof_event_end);
  if (lr > 0) return set_error(JH_ERR_CUDA, "hstu_fwd launch: %s", cudaGetErrorString((cudaError_t)lr));
  if (lr) return JH_ERR_UNSUPPORTED;
  return JH_OK;
}

int jh_attn_bwd(const jh_attn_args* a, void* stream) {
  int rc = validate(a, true);
  if (rc) return rc;
  if (a->q_rows == 0 || a->num_segments == 0) return JH_OK;
  cudaStream_t s = (cudaStream_t)stream;
  AttnParams p;
  TMaps tm;
  rc = prepare(a, true, &p, &tm, s);
  if (rc) return rc;
  int grid = sm_count();
  if (!a->dq_accum && (a->q_pos0 || a->kv_len)) {
    // segment form: q tiles that see no kv get no dQ contribution -> zero rows
    const size_t HDb = (size_t)a->num_heads * a->head_dim * 2;
    cudaError_t e = cudaMemset2DAsync(a->dq, (size_t)a->ld_dq * 2, 0, HDb, (size_t)a->q_rows, s);
    if (e != cudaSuccess) return set_error(JH_ERR_CUDA, "dq memset: %s", cudaGetErrorString(e));
  }
  if ((a->q_pos0 || a->kv_len) && a->kv_rows > 0) {
    // kv rows past every segment's visible range get no dK / dV: zero them (bf16 modes)
    const size_t HDb = (size_t)a->num_heads * a->head_dim * 2;
    cudaError_t e = cudaSuccess;
    if (!a->dk_accum) e = cudaMemset2DAsync(a->dk, (size_t)a->ld_dk * 2, 0, HDb, (size_t)a->kv_rows, s);
    if (e == cudaSuccess && !a->dv_accum) e = cudaMemset2DAsync(a->dv, (size_t)a->ld_dv * 2, 0, HDb, (size_t)a->kv_rows, s);
    if (e != cudaSuccess) return set_error(JH_ERR_CUDA, "dk/dv memset: %s", cudaGetErrorString(e));
  }
  int lr;
  if (a->deterministic)
    lr = a->head_dim == 64 ? launch_bwd<64>(tm, p, *a, grid, s) : launch_bwd<128>(tm, p, *a, grid, s);
  else
    lr = a->head_dim == 64 ? launch_bwd_fused<64>(tm, p, *a, grid, s) : launch_bwd_fused<128>(tm, p, *a, grid, s);
  if (lr > 0) return set_error(JH_ERR_CUDA, "hstu_bwd launch: %s", cudaGetErrorString((cudaError_t)lr));
  if (lr) return JH_ERR_UNSUPPORTED;
  return JH_OK;
}

}  // extern "C"
