/*
 * jh_hstu.h -- C ABI of the B200 (sm_100a) jagged HSTU attention + jagged
 * context-parallel hot path.  Shared library: paper_2508_04711_b200/libjh_hstu.so
 *
 * Conventions (all entry points):
 *   - plain C types only; device pointers are caller-owned (e.g. torch
 *     tensors); nothing here allocates device memory except where stated;
 *   - return JH_OK (0) or a JH_ERR_* code; jh_last_error() returns a
 *     thread-local message naming the failed check;
 *   - every GPU call is stream-ordered on the `stream` argument (a
 *     cudaStream_t passed as void*) and does not synchronize the host;
 *   - no C++ exception crosses the ABI.
 *
 * Each entry point names the reference (jaggedcp, /root/reference/pkg/src/
 * jaggedcp) interface it replaces.  The reference is a Python/numpy package,
 * so the reference-side binding is the ctypes module
 * paper_2508_04711_b200/_lib.py.
 */
#ifndef JH_HSTU_H_
#define JH_HSTU_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define JH_API __attribute__((visibility("default")))
#else
#define JH_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum {
  JH_OK = 0,
  JH_ERR_INVALID = 1,     /* argument validation failed (maps to ValueError)   */
  JH_ERR_CUDA = 2,        /* CUDA runtime / launch error (maps to RuntimeError) */
  JH_ERR_UNSUPPORTED = 3  /* shape outside what the kernels implement           */
};

/* Thread-local description of the last error. */
JH_API const char* jh_last_error(void);
/* ABI version (major*100 + minor). */
JH_API int jh_version(void);

/* ------------------------------------------------------------------ bias --
 * Bit-exact bucket table for the reference rule
 *   bucket(d) = min(nb-1, floor(log1p((double)max(d, 0))))
 * (attention.py:83-86 bucketize_array).  Thresholds T_k = min{d : bucket(d) >= k}
 * are found by bisection against that very f64 expression; the kernels then
 * count thresholds with integer compares only.  Host function.
 *   thr[64]  : per power-of-two octave o (d+1 in [2^o, 2^(o+1))), the single
 *              threshold inside the octave (INT64_MAX when none)
 *   base[64] : bucket of the octave's first delta
 *   *cap     : smallest delta of the last bucket (deltas are clamped to it)
 */
JH_API int jh_bias_table_build(int num_buckets, int64_t* thr, int32_t* base, int64_t* cap);

/* attention.py:83 bucketize_array -- standalone device kernel over n int64 deltas. */
JH_API int jh_bucketize(const int64_t* deltas, int64_t n, int num_buckets, int32_t* out, void* stream);

/* attention.py:89 compute_bias -- out[i*nk + j] = w[bucket(ts_q[i] - ts_k[j])] (fp32). */
JH_API int jh_compute_bias(const int64_t* ts_q, int64_t nq, const int64_t* ts_k, int64_t nk, const float* ts_weights,
                    int num_buckets, float* out, void* stream);

/* attention.py:227-228 (bincount of dBias into buckets) -- the scatter-add
 * gradient of the ts_weights gather, from a materialized fp32 dBias
 * [nq x nk]: d_w[b] += sum over (i,j) with bucket(ts_q[i]-ts_k[j]) == b.
 * d_w is fp64 [nb], accumulated (caller zeroes it). */
JH_API int jh_dbias_scatter(const int64_t* ts_q, int64_t nq, const int64_t* ts_k, int64_t nk, const float* dbias,
                     int num_buckets, double* d_w, void* stream);

/* --------------------------------------------------------------- attention --
 * Jagged batch of `num_segments` query segments.  Segment s has
 *   q rows     [q_offsets[s], q_offsets[s+1])      of q / out / dout / dq,
 *   positions  q_pos0[s] + 0, 1, ...               (q_pos0 == NULL -> 0),
 *   kv rows    [kv_start[s], kv_start[s] + kv_len[s]) of k / v / dk / dv,
 *              holding positions 0 .. kv_len[s]-1  (kv_start == NULL -> q rows,
 *              kv_len == NULL -> q segment length),
 * and attends causally (key position <= query position) within the segment:
 *   out = (tril . SiLU((q k^T + bias) / sqrt(head_dim))) v
 *   bias = ts_weights[bucket(ts_q - ts_k)] (+ pos_weights[min(i-j, P-1)] if set).
 * Single-device use (hstu_attention_reference, attention.py:125): q_offsets =
 * seq_offsets, everything else NULL.  CP use (ring_hstu_attention,
 * cp_engine.py:384): one segment per resident mini-chunk, KV = the gathered
 * sequence prefix.
 * Values are bf16, row-major with row stride ld_* (elements); head h occupies
 * columns [h*head_dim, (h+1)*head_dim).  head_dim must be 64 or 128.
 * All arrays are device memory.  `workspace` must hold
 * jh_attn_workspace_bytes(...) bytes. */
typedef struct jh_attn_args {
  const void* q;
  const void* k;
  const void* v;
  int64_t ld_q, ld_k, ld_v;
  const int64_t* ts_q;          /* [rows of q]                               */
  const int64_t* ts_k;          /* [rows of k]                               */
  const int64_t* q_offsets;     /* [num_segments + 1]                        */
  const int64_t* q_pos0;        /* [num_segments] or NULL                    */
  const int64_t* kv_start;      /* [num_segments] or NULL                    */
  const int64_t* kv_len;        /* [num_segments] or NULL                    */
  int64_t num_segments;
  int64_t q_rows;               /* rows of q (= q_offsets[num_segments])     */
  int64_t kv_rows;              /* rows of k / v                             */
  int32_t num_heads;
  int32_t head_dim;
  const float* ts_weights;      /* [num_buckets] fp32                        */
  int32_t num_buckets;
  const float* pos_weights;     /* [num_pos] fp32 or NULL (extension)        */
  int32_t num_pos;
  int32_t max_q_len_hint;       /* upper bound of a segment's length, 0 = unknown */
  /* forward output */
  void* out;                    /* bf16 [q_rows, ld_o]                       */
  int64_t ld_o;
  /* backward (jh_attn_bwd only) */
  const void* dout;             /* bf16 [q_rows, ld_do]                      */
  int64_t ld_do;
  void* dq;                     /* bf16 [q_rows, ld_dq]                      */
  void* dk;                     /* bf16 [kv_rows, ld_dk]  (NULL if dk_accum) */
  void* dv;                     /* bf16 [kv_rows, ld_dv]  (NULL if dv_accum) */
  int64_t ld_dq, ld_dk, ld_dv;
  float* dk_accum;              /* fp32 [kv_rows, H*d] accumulate instead of dk (CP), or NULL */
  float* dv_accum;              /* fp32 [kv_rows, H*d] accumulate instead of dv (CP), or NULL */
  double* d_ts_weights;         /* fp64 [num_buckets], accumulated            */
  double* d_pos_weights;        /* fp64 [num_pos] or NULL, accumulated       */
  /* scratch */
  void* workspace;
  size_t workspace_bytes;
  /* optional profiling: cudaEvent_t pair recorded on `stream` immediately
   * before / after the main fused kernel (NULL = off) */
  void* prof_event_start;
  void* prof_event_end;
  /* optional debug timeline: uint64 [5 roles][4096 events][2] written by CTA
   * `trace_cta` (NULL = off) */
  void* trace;
  int32_t trace_cta;
  /* backward scratch for the bf16 dS tiles handed from the dK/dV kernel to the
   * dQ kernel: at least jh_attn_ds_scratch_bytes(...) bytes (jh_attn_bwd only) */
  void* ds_scratch;
  size_t ds_scratch_bytes;
  /* forward fp32 output mode (jh_attn_fwd only; CP partial sums, the
   * reference's additive blockwise partials, attention.py:151-184 and
   * cp_engine.py:441-450): 0 = write bf16 `out`; 1 = store fp32 into
   * out_accum; 2 = add into out_accum (rows of q with no visible kv are left
   * untouched).  Row stride of out_accum = ld_o (elements). */
  float* out_accum;
  int32_t out_accum_mode;
  /* backward: add dq (fp32) into dq_accum instead of writing the bf16 `dq`
   * (row stride ld_dq; rows of q with no visible kv are left untouched), or NULL */
  float* dq_accum;
  /* optional caller-owned band table (jh_attn_band_table_bytes bytes): the
   * exact near-diagonal buckets, a function of ts_q, ts_k and the segment
   * description only.  ready == 0: computed into it; ready == 1: it already
   * holds the table for these same inputs (e.g. from the forward call of the
   * same step) and is reused.  NULL: a private copy in the workspace. */
  void* band_table;
  size_t band_table_bytes;
  int32_t band_table_ready;
  /* score scale: scores = (q k^T + bias) * score_scale; 0 -> 1/sqrt(head_dim).
   * Lets a caller zero-pad a smaller head dimension d to 64 / 128 columns and
   * keep the reference's 1/sqrt(d) (attention.py:143, :180). */
  float score_scale;
  /* backward: 1 = deterministic two-kernel path (dK/dV kernel + dQ GEMM over a
   * bf16 dS scratch, needs ds_scratch); 0 = fused single kernel (dQ reduced in
   * fp32 into bwd_state, no dS scratch, O(L) memory) */
  int32_t deterministic;
  /* fused backward state (jh_attn_bwd_state_bytes bytes): must be all-zero the
   * first time it is used; every fused call leaves it all-zero again.  One
   * state buffer per concurrently running call (stream). */
  void* bwd_state;
  size_t bwd_state_bytes;
  /* debug (forward): when non-NULL, head 0 writes the bucket it applied to
   * every visible (q row, kv position) pair into dbg_buckets[q_row * dbg_ld +
   * kv_pos] (uint8; entries of pairs it never evaluated are left untouched) */
  uint8_t* dbg_buckets;
  int64_t dbg_ld;
  /* debug (fused backward): 1 = d_ts_weights receives the exact number of
   * visible (q, kv) pairs per bucket (summed over heads) instead of dS sums --
   * the backward's bucket placement as integers */
  int32_t dbg_count_buckets;
} jh_attn_args;

/* Size of the fused backward's persistent state (fp32 dQ accumulator rows +
 * per-(q tile, head) completion counters + the d_ts_weights reduction slots). */
JH_API size_t jh_attn_bwd_state_bytes(int64_t q_rows, int64_t num_segments, int32_t num_heads, int32_t head_dim);

/* kv_len_total = sum over segments of kv_len[s] (= q_rows when kv_len is NULL). */
JH_API size_t jh_attn_workspace_bytes(int64_t q_rows, int64_t kv_len_total, int64_t num_segments, int32_t num_heads,
                                      int32_t head_dim);

JH_API size_t jh_attn_band_table_bytes(int64_t q_rows, int64_t num_segments);

/* Deterministic-backward dS scratch (jh_attn_args.deterministic = 1).
 * Bound: max_len >= every segment's kv_len AND q length (= the sequence
 * length for self-attention).  Exact: the segment arrays on the HOST
 * (q_pos0 / kv_len may be NULL).  If the scratch is too small at run time the
 * backward writes NaN into dq instead of overrunning it. */
JH_API size_t jh_attn_ds_scratch_bytes(int64_t kv_len_total, int64_t num_segments, int32_t num_heads,
                                       int64_t max_len);
JH_API size_t jh_attn_ds_scratch_bytes_segs(const int64_t* q_offsets, const int64_t* q_pos0, const int64_t* kv_len,
                                            int64_t num_segments, int32_t num_heads);

/* Forward: attention.py:125 hstu_attention_reference / :151 blockwise_partial. */
/* The band table alone (exact bucket bytes of the near-diagonal pairs) into
 * a->band_table, from q_offsets / q_pos0 / kv_start / kv_len, ts_q, ts_k and
 * num_buckets (other fields ignored).  A forward / backward call then takes it
 * with band_table_ready = 1, so the two can run concurrently on two streams
 * (the HSTU backward recomputes from q, k, v and never reads the forward's
 * output: attention.py:187-234). */
JH_API int jh_attn_band(const jh_attn_args* a, void* stream);
JH_API int jh_attn_fwd(const jh_attn_args* a, void* stream);
/* Backward: attention.py:187 hstu_attention_backward (dq, dk, dv, d_ts_weights). */
JH_API int jh_attn_bwd(const jh_attn_args* a, void* stream);

/* ------------------------------------------------------- jagged helpers --
 * jagged.py:232 reorder_balanced / :248 inverse_reorder, and the CP message
 * pack/unpack (cp_engine.py:286-371, 468-525): dst[i] = src[perm[i]] (gather)
 * or dst[perm[i]] = src[i] (scatter), rows of row_bytes (multiple of 8). */
JH_API int jh_gather_rows(const void* src, void* dst, const int64_t* perm, int64_t rows, int64_t row_bytes,
                   void* stream);
JH_API int jh_scatter_rows(const void* src, void* dst, const int64_t* perm, int64_t rows, int64_t row_bytes,
                    void* stream);
/* jagged -> padded [B, max_len, row_bytes] (zero padding) and back. */
JH_API int jh_jagged_to_padded(const void* values, const int64_t* offsets, int64_t num_seqs, int64_t max_len,
                        int64_t row_bytes, void* padded, void* stream);
JH_API int jh_padded_to_jagged(const void* padded, const int64_t* offsets, int64_t num_seqs, int64_t max_len,
                        int64_t row_bytes, void* values, void* stream);

/* ---------------------------------------------------------- HSTU layer --
 * Row-wise pieces of the HSTU layer around the attention (
 * no reference counterpart: the reference stops at the attention).
 * All bf16, 16-byte aligned, row strides in elements (multiples of 8).
 *   silu:      y = x sigmoid(x);  dx = dy s (1 + x (1 - s)).  n % 8 == 0.
 *   norm_gate: y = (LN(x) * gamma + beta) * u   (u / gamma / beta may be NULL),
 *              LN over n <= 2048 columns with eps, fp32 statistics saved in
 *              mean / rstd [rows].  The backward ADDS the gamma / beta
 *              gradients into dgamma / dbeta (fp32, deterministic; workspace
 *              of jh_norm_gate_bwd_workspace_bytes) and writes dx, du. */
JH_API int jh_silu_fwd(const void* x, void* y, int64_t n, void* stream);
JH_API int jh_silu_bwd(const void* x, const void* dy, void* dx, int64_t n, void* stream);
/* SiLU backward fused with the bias gradient of the GEMM that produced x:
 * dx = silu'(x) * dy over a contiguous [rows, n] matrix and dbias[n] (fp32) +=
 * column sums of dx (as rounded to bf16).  Deterministic (per-block partial
 * rows in `workspace`, >= jh_colsum_workspace_bytes(rows, n), added in block
 * order).  n: multiple of 8 in [8, 8192].  Replaces autograd's separate
 * reduction for the bias of uvqk = SiLU(x W + b) (layer, not in the reference). */
JH_API int jh_silu_bwd_colsum(const void* x, const void* dy, void* dx, int64_t rows, int32_t n, float* dbias,
                              void* workspace, size_t workspace_bytes, void* stream);
/* out[n] (fp32) += column sums of x ([rows, n] bf16, row stride ld elements):
 * the bias gradient of out = y W + b.  Deterministic, as above. */
JH_API int jh_colsum(const void* x, int64_t ld, int64_t rows, int32_t n, float* out, void* workspace,
                     size_t workspace_bytes, void* stream);
JH_API size_t jh_colsum_workspace_bytes(int64_t rows, int32_t n);
JH_API int jh_norm_gate_fwd(const void* x, int64_t ld_x, const void* u, int64_t ld_u, const float* gamma,
                            const float* beta, float eps, int64_t rows, int32_t n, void* y, int64_t ld_y, float* mean,
                            float* rstd, void* stream);
JH_API size_t jh_norm_gate_bwd_workspace_bytes(int64_t rows, int32_t n);
JH_API int jh_norm_gate_bwd(const void* dy, int64_t ld_dy, const void* x, int64_t ld_x, const void* u, int64_t ld_u,
                            const float* gamma, const float* beta, const float* mean, const float* rstd, int64_t rows,
                            int32_t n, void* dx, int64_t ld_dx, void* du, int64_t ld_du, float* dgamma, float* dbeta,
                            void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------ plan --
 * cp_engine.py:105 build_shard_plan (+ jagged.py:162 make_minichunks,
 * :169 make_contiguous_chunks, :187 chunk_owner_map).  Host function, exact
 * integers.  mode 0 = balanced_minichunk (2*cp chunks, rank r owns r and
 * 2cp-1-r), 1 = naive_contiguous (cp chunks).  Outputs (caller-allocated):
 *   chunk_len[num_seqs * C], chunk_start[num_seqs * C], chunk_owner[C]
 * with C = 2*cp (mode 0) or cp (mode 1). */
JH_API int jh_plan_build(const int64_t* seq_lengths, int64_t num_seqs, int cp_size, int mode, int64_t* chunk_len,
                  int64_t* chunk_start, int32_t* chunk_owner);
/* cp_engine.py:528 flops_per_rank: exact causal pair counts per rank. */
JH_API int jh_flops_per_rank(const int64_t* seq_lengths, int64_t num_seqs, int cp_size, int mode, int64_t* per_rank,
                      int64_t* total);
/* jagged.py:201 _rank_major_row_order: perm[T] (rank -> sequence -> chunk),
 * slab_rows[cp]. */
JH_API int jh_rank_major_perm(const int64_t* seq_offsets, int64_t num_seqs, int cp_size, int mode, int64_t* perm,
                       int64_t* slab_rows);

/* --------------------------------------------------------------- debug --
 * tcgen05 descriptor self-test (tests/test_gpu_umma.py). */
JH_API int jh_debug_umma(const void* a, const void* b, float* d, int a_mode, int b_mode, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* JH_HSTU_H_ */
