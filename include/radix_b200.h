/*
 * radix_b200.h — C ABI of the B200-native RadixMLP hot path.
 *
 * Every entry point takes raw device pointers, plain integer sizes and a
 * cudaStream_t passed as `void*` (NULL = legacy default stream), is
 * stream-ordered, re-entrant, keeps no global state beyond cached device
 * attributes, and returns an rdx_status.  Errors that can only be detected
 * on the device (index out of range, hash-verification exhaustion, invalid
 * offsets) are reported through a caller-owned device status word so the
 * launch never needs a host synchronisation.
 *
 * Reference interfaces replaced (paths relative to the reference checkout):
 *   rdx_plan_build        <- radix_compact.trie.build_plan / _build_indices
 *                            (pkg/src/radix_compact/trie.py:73-148) and the
 *                            binding radix_bindings.compute_plan
 *                            (pkg/bindings/src/radix_bindings/__init__.py:57-69)
 *   rdx_gather_rows       <- radix_compact.ops.gather_rows / scatter_rows
 *                            (pkg/src/radix_compact/ops.py:50-66) and the
 *                            bindings gather_rows / scatter_rows (…:72-89)
 *   rdx_gather_rows_backward <- ops.gather_rows_backward / scatter_rows_backward
 *                            (ops.py:69-107), deterministic ascending-j adds
 *   rdx_embed_rmsnorm     <- model.py:329,341 (token gather + embedding rows)
 *                            fused with the layer-0 rmsnorm (model.py:147-152,349)
 *   rdx_rmsnorm_rows      <- rmsnorm (model.py:147-152) at model.py:392,404
 *   rdx_rope_table        <- _rope_tables (model.py:165-172) on compact positions
 *   rdx_gemm              <- _mm (model.py:131-144) for q/k/v/o, gate/up/down,
 *                            lm_head, with the fused epilogues of
 *                            model.py:356-366 (q/k norm + RoPE), 387-389 (o-proj
 *                            + residual), 394-397 (SwiGLU), 397-399 (down +
 *                            residual)
 *   rdx_attention         <- scatter_rows(q/k/v) + _attention_forward + gather_rows
 *                            (model.py:368-383, 228-265), boundary fused into loads
 *   rdx_rerank_scores     <- last-token scoring contract (no reference
 *                            counterpart)
 */
#ifndef RADIX_B200_H
#define RADIX_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  One code per reference exception class that can arise on
 * this path (pkg/src/radix_compact/errors.py:8-87); the Python shim maps each
 * code back to the class of the same name. */
typedef enum rdx_status {
  RDX_OK = 0,
  RDX_ERR_MISMATCHED_LENGTHS = 1,    /* errors.py:15  MismatchedLengths  */
  RDX_ERR_NON_MONOTONE_OFFSETS = 2,  /* errors.py:19  NonMonotoneOffsets */
  RDX_ERR_BOUNDARY_MISMATCH = 3,     /* errors.py:23  BoundaryMismatch   */
  RDX_ERR_OVERFLOW_ID = 4,           /* errors.py:27  OverflowId         */
  RDX_ERR_CAPACITY_EXCEEDED = 5,     /* errors.py:34  CapacityExceeded   */
  RDX_ERR_EMPTY_PLAN = 6,            /* errors.py:38  EmptyPlan          */
  RDX_ERR_INDEX_OUT_OF_RANGE = 7,    /* errors.py:45  IndexOutOfRange    */
  RDX_ERR_SHAPE_MISMATCH = 8,        /* errors.py:49  ShapeMismatch      */
  RDX_ERR_PLAN_BATCH_MISMATCH = 9,   /* errors.py:60  PlanBatchMismatch  */
  RDX_ERR_ODD_HEAD_DIM = 10,         /* errors.py:56  OddHeadDim         */
  RDX_ERR_HASH_RETRIES = 11,         /* GPU planner: every hash seed collided */
  RDX_ERR_INVALID_ARGUMENT = 12,
  RDX_ERR_UNSUPPORTED = 13,
  RDX_ERR_DEVICE_TIMEOUT = 14,      /* an asynchronous wait gave up (rdx_device_status) */
  RDX_ERR_CUDA = 100
} rdx_status;

/* Library version (major*10000 + minor*100 + patch): 300 = 0.3.0, whose
 * rdx_gemm_args ends at a_ready_use and whose rdx_rmsnorm_rows_after takes
 * ready_ctr.  Check it against RDX_VERSION before use. */
#define RDX_VERSION 300
int rdx_version(void);
/* Stable name of a status code ("RDX_OK", "IndexOutOfRange", …). */
const char* rdx_status_name(int status);
/* Last CUDA error string recorded by a failing call on this thread. */
const char* rdx_last_cuda_error(void);

/* ---------------------------------------------------------------------
 * Index build (the prefix-trie planner), bit-exact to trie.build_plan.
 *
 * Inputs (device): tok[N], pos[N] (u32), cu[B+1] (i64, validated on device
 * with the reference's precedence: BoundaryMismatch(start) ->
 * NonMonotoneOffsets(decrease) -> NonMonotoneOffsets(empty, unless
 * RDX_PLAN_ALLOW_EMPTY) -> BoundaryMismatch(end), ragged.py:68-102).
 * Outputs (device, caller-allocated worst case):
 *   gather_out[N]   first N' entries valid (compact -> original)
 *   scatter_out[N]  original -> compact
 *   cpos_out[N]     first N' entries valid (positions of representatives)
 *   cu_q_out[B+1]   i32 offsets of the per-sequence compact suffixes
 *                   (compact rows of sequence s are [cu_q[s], cu_q[s+1]))
 *   lcp_out[B]      i32 shared-prefix length of each sequence (may be NULL)
 *   info_out[4]     u32: [0]=N', [1]=status (rdx_status), [2]=hash attempts
 *                   used, [3]=max_q (longest compact suffix, rows).  May be
 *                   pinned host memory (device-addressable under unified
 *                   addressing): the kernel writes it directly, no copy.
 * scratch: at least rdx_plan_scratch_bytes(N, B) bytes of device memory.
 * --------------------------------------------------------------------- */
#define RDX_PLAN_ALLOW_EMPTY 0x1u

size_t rdx_plan_scratch_bytes(int64_t n_tokens, int64_t n_seqs);
int rdx_plan_build(const uint32_t* tok, const uint32_t* pos, const int64_t* cu,
                   int64_t n_seqs, int64_t n_tokens, uint32_t flags,
                   uint32_t* gather_out, uint32_t* scatter_out, uint32_t* cpos_out,
                   int32_t* cu_q_out, int32_t* lcp_out, uint32_t* info_out,
                   void* scratch, size_t scratch_bytes, void* stream);

/* Debug: batches up to 16 x 4096 tokens (and at most 8191 sequences) run on the
 * cluster-resident planner (one thread-block cluster, the whole working set in
 * shared memory); 0 routes every batch to the L2-resident planners for A/B runs
 * and tests, 1 back on.  Same outputs either way.  Returns the previous setting. */
int rdx_plan_debug_smem(int on);

/* Debug: when buf != NULL (device memory, >= 32 u64), later cluster-planner
 * launches write %globaltimer stamps: [0..11] phase boundaries of CTA 0,
 * [16 + r] the start of CTA r.  NULL turns it off. */
int rdx_plan_debug_trace(void* buf);

/* ---------------------------------------------------------------------
 * Row gather / scatter: dst[j, :] = src[idx[j], :] as a bit-exact byte copy
 * (scatter_rows is the same call with the scatter map, ops.py:64-66).
 * row_bytes is the payload per row; ld_* are row strides in bytes.  An index
 * >= src_rows sets *err_flag = RDX_ERR_INDEX_OUT_OF_RANGE and zero-fills the
 * destination row (err_flag may be NULL to skip reporting).
 * --------------------------------------------------------------------- */
int rdx_gather_rows(const void* src, int64_t src_rows, int64_t ld_src_bytes,
                    const uint32_t* idx, int64_t n_idx, void* dst,
                    int64_t ld_dst_bytes, int64_t row_bytes, uint32_t* err_flag,
                    void* stream);

/* ---------------------------------------------------------------------
 * Adjoint of the row gather / scatter (ops.py:69-107, gather_rows_backward
 * and scatter_rows_backward; used by loss_and_grads, model.py:456-500):
 *   out = zeros(n_out, cols);  out[idx[j]] += grad[j]   for j = 0, 1, ...
 * in ascending-j order per output row, i.e. bit-identical to the
 * reference's np.add.at path.  dtype RDX_DTYPE_F32 or RDX_DTYPE_F64 (the
 * reference's float dtypes).  Indices >= n_out set *err_flag (IndexOutOfRange)
 * and are skipped.  scratch: rdx_gather_rows_backward_scratch_bytes(n_idx, n_out)
 * bytes of device memory.
 * --------------------------------------------------------------------- */
enum { RDX_DTYPE_F32 = 0, RDX_DTYPE_F64 = 1 };
size_t rdx_gather_rows_backward_scratch_bytes(int64_t n_idx, int64_t n_out);
int rdx_gather_rows_backward(const void* grad, int64_t ld_grad_bytes, const uint32_t* idx, int64_t n_idx,
                             int64_t n_out, void* out, int64_t ld_out_bytes, int64_t cols, int32_t dtype,
                             uint32_t* err_flag, void* scratch, size_t scratch_bytes, void* stream);

/* ---------------------------------------------------------------------
 * Compact embedding gather fused with RMSNorm:
 *   t      = tok[gather[j]] (or tok[j] when gather == NULL)
 *   h[j]   = embed[t, :]                       (fp32 residual stream)
 *   hn[j]  = bf16(h[j] / rms(h[j]) * w)        (input of the QKV GEMM)
 * embed is bf16 [vocab, d].  Out-of-range tokens set *err_flag.
 * --------------------------------------------------------------------- */
int rdx_embed_rmsnorm(const uint32_t* tok, const uint32_t* gather, int64_t n_rows,
                      const void* embed_bf16, int64_t vocab, int64_t d,
                      const float* norm_w, float eps, float* h_out, void* hn_bf16_out,
                      uint32_t* err_flag, void* stream);

/* Compact embedding gather for the fused-norm layer stack (RDX_EPI_RESID_NORM
 * / row_ss): h[j] = embed[t] (fp32), hb[j] = bf16 copy, ss[j, g] = sum of
 * h[j, 64g:64g+64]^2 (d % 64 == 0).  The layer-0 ln1 is then applied by the
 * QKV GEMM (row_ss + ln1 folded into its weight). */
int rdx_embed_rows(const uint32_t* tok, const uint32_t* gather, int64_t n_rows, const void* embed_bf16,
                   int64_t vocab, int64_t d, float* h_out, void* hb_out, float* ss_out, uint32_t* err_flag,
                   void* stream);

/* RMSNorm of selected fp32 rows: out[j] = bf16(x[rows[j]] / rms * w)
 * (rows == NULL selects row j). */
int rdx_rmsnorm_rows(const float* x, int64_t ld_x, const uint32_t* rows, int64_t n_rows,
                     int64_t d, const float* w, float eps, void* out_bf16, int64_t ld_out,
                     void* stream);

/* cudaStreamSynchronize(stream) (a C-ABI caller's one host wait, e.g. after
 * rdx_plan_build wrote its info into pinned memory). */
int rdx_stream_synchronize(void* stream);

/* First device-side failure of an asynchronous contract since the last call
 * (RDX_OK or RDX_ERR_DEVICE_TIMEOUT), then cleared; synchronises `stream`. */
int rdx_device_status(void* stream);

/* rdx_rmsnorm_rows on rows 0..n_rows-1 that may still be in flight from a
 * preceding rdx_gemm (RDX_EPI_RESID_F32 with done_ctr) on the same stream: the
 * kernel is launched as a programmatic dependent of that GEMM (it can start on
 * SMs the GEMM's last round leaves idle) and processes row r once
 * done_ctr[r / 32] >= target (a slab still incomplete after ~8 s stops the wait,
 * the rows are normalised as found and rdx_device_status reports
 * RDX_ERR_DEVICE_TIMEOUT: the counters and targets did not match).  d must be 128 * V for V in {2, 4, 8, 16, 20, 32}
 * (else RDX_ERR_UNSUPPORTED: use rdx_rmsnorm_rows after a stream-ordered GEMM).
 * ready_ctr (may be NULL): ceil(n_rows / 32) counters; every finished row adds 1 to
 * ready_ctr[row / 32] (release) and the grid becomes one small block per SM whose
 * registers fit beside a GEMM CTA, so a chained consumer rdx_gemm (a_ready =
 * ready_ctr) runs concurrently with the norm's last rows. */
int rdx_rmsnorm_rows_after(const float* x, int64_t ld_x, int64_t n_rows, int64_t d, const float* w, float eps,
                           void* out_bf16, int64_t ld_out, const uint32_t* done_ctr, uint32_t target,
                           uint32_t* ready_ctr, void* stream);

/* RoPE table for compact rows: table[j][i] = (cos, sin)(pos[j] * theta^(-2i/hd))
 * for i < hd/2, computed in fp64 and rounded to fp32 (model.py:165-172). */
int rdx_rope_table(const uint32_t* pos, int64_t n_rows, int32_t head_dim, double theta,
                   float* table_out, void* stream);

/* The same values in the QKV epilogue's lane-blocked layout (rdx_gemm_args.
 * rope_blocked = 1): rows in blocks of 32, column pairs outermost within a
 * block, so the 32 lanes of a GEMM epilogue warp (32 consecutive rows) read one
 * contiguous 512 B run per column pair.  (cos, sin) of (row j, column i) sits at
 * float2 index 2 * (((j / 32) * (hd / 4) + i / 2) * 32 + j % 32) + i % 2;
 * table_out holds ceil(n_rows / 32) * 32 * hd / 2 float2 (16-byte aligned,
 * head_dim % 4 == 0). */
int rdx_rope_table_blocked(const uint32_t* pos, int64_t n_rows, int32_t head_dim, double theta,
                           float* table_out, void* stream);

/* ---------------------------------------------------------------------
 * tcgen05/TMEM GEMM on sm_100a: acc[m, n] = sum_k A[m, k] * B[n, k]
 * (A [M, K] bf16 row-major = activations, B [N, K] bf16 row-major = weight
 * in the reference's [out, in] layout, model.py:107-116), fp32 accumulate in
 * TMEM, persistent warp-specialised kernel, fused epilogue selected by `epi`.
 * Each output row depends only on its own input row (no split-K, fixed tile
 * shape), so dedup-on and dedup-off rows are bit-identical.
 * --------------------------------------------------------------------- */
typedef enum rdx_epilogue {
  RDX_EPI_STORE_BF16 = 0, /* out_bf16[m, n] = bf16(acc)                              */
  RDX_EPI_STORE_F32 = 1,  /* out_f32[m, n]  = acc                                    */
  RDX_EPI_RESID_F32 = 2,  /* resid_f32[m, n] += acc                                  */
  RDX_EPI_SWIGLU = 3,     /* B rows interleaved per tile: [gate(BN/2) | up(BN/2)];
                             out_bf16[m, n/2] = bf16(silu(g) * u)                    */
  RDX_EPI_QKV = 4,        /* per-head RMSNorm of q/k heads (q_norm/k_norm weights)
                             + rotate-half RoPE from rope_table, v passthrough,
                             bf16 store (model.py:356-366)                           */
  RDX_EPI_RESID_NORM = 5  /* residual add + the next RMSNorm's statistics:
                             h = out_f32[m, n] += acc; out_bf16[m, n] = bf16(h);
                             ss_out[m, n/64] = sum of h^2 per 64 columns (n % 64 == 0).
                             Replaces the residual add and the rmsnorm pass of
                             model.py:387-392 / 397-404 (the weight half of the norm
                             is folded into the next GEMM's B, see row_ss)          */
} rdx_epilogue;

/* Zero-initialise (fields are appended between versions; 0 / NULL = feature off). */
typedef struct rdx_gemm_args {
  const void* a;       /* bf16 [M, lda] */
  const void* b;       /* bf16 [N, ldb] */
  int64_t m, n, k;
  int64_t lda, ldb;    /* elements */
  int32_t epi;         /* rdx_epilogue */
  int32_t block_n;     /* 0 = auto, else 128 or 256 */
  void* out;           /* bf16 or f32 output / residual */
  int64_t ldo;         /* elements */
  /* RDX_EPI_QKV */
  const float* q_norm_w;   /* [head_dim] */
  const float* k_norm_w;   /* [head_dim] */
  const float* rope_table; /* [M, head_dim/2, 2] (cos, sin), or the blocked layout */
  int32_t head_dim, q_heads, kv_heads;
  float eps;
  /* Optional RMSNorm of the A rows fused into any epilogue: when row_ss != NULL
   * accumulator row m is scaled by rsqrt(sum_{t<ss_parts} row_ss[m*ss_parts+t]
   * / norm_dim + norm_eps) first (A = bf16 of the unnormalised rows, B = W with
   * the norm weight folded in: B[n, k] = W[n, k] * w[k]). */
  const float* row_ss;
  int32_t ss_parts;
  int32_t norm_dim;
  float norm_eps;
  /* RDX_EPI_RESID_NORM outputs (out = fp32 residual, read-modify-write) */
  void* out_bf16;
  int64_t ldo_bf16;
  float* ss_out;
  /* RDX_EPI_QKV: 1 = rope_table is in rdx_rope_table_blocked's layout */
  int32_t rope_blocked;
  /* RDX_EPI_QKV, head_dim 64 or 128: when rope_pos != NULL the epilogue computes
   * (cos, sin)(rope_pos[m] * rope_theta^(-2i/head_dim)) itself (fp64 inverse
   * frequencies, |error| < 1e-6 for positions < 2^20) and rope_table is unused. */
  const uint32_t* rope_pos;
  double rope_theta;
  /* RDX_EPI_RESID_F32 only (any other epilogue with done_ctr != NULL returns
   * RDX_ERR_INVALID_ARGUMENT): when done_ctr != NULL, tiles run in row-block-major
   * order when M spans < 64 row blocks (else in the grouped raster of 16 row blocks)
   * and, once a warp's reduce-adds have completed, done_ctr[row / 32] is incremented by
   * the number of columns it wrote for those 32 rows (a 32-row slab is complete
   * when its counter has grown by N); done_ctr holds ceil(M / 32) counters.
   * Feeds rdx_rmsnorm_rows_after. */
  uint32_t* done_ctr;
  /* Chained A (any epilogue): when a_ready != NULL the A rows of 32-row slab s are
   * read only once a_ready[s] >= a_ready_use * rows_in_slab(s) (the ready_ctr of a
   * preceding rdx_rmsnorm_rows_after that wrote A).  The launch is then that norm's
   * programmatic dependent and does not wait for its grid: the GEMM's first tiles
   * overlap the norm's last rows.  Tiles run in row-block-major order (< 64 row blocks). */
  const uint32_t* a_ready;
  uint32_t a_ready_use;
} rdx_gemm_args;

int rdx_gemm(const rdx_gemm_args* args, void* stream);

/* The MLP's two GEMMs in ONE persistent launch: first = gate|up (RDX_EPI_SWIGLU,
 * output act), second = down (RDX_EPI_RESID_F32 with second->a == first->out,
 * second->k == first->n / 2, same m).  Job 1's tiles follow job 0's in every CTA's
 * static schedule; a down tile's TMA producer waits until every act column of its
 * rows is written (dep_ctr: ceil(m / 32) zeroed u32 counters, one per 32-row slab,
 * release/acquire), so the down GEMM starts while the gate|up GEMM drains and the
 * second launch's prologue disappears.  Same bits as the two rdx_gemm calls; falls
 * back to them when the two GEMMs want different tile shapes or M spans >= 64 pair
 * row blocks (large M: measured neutral). */
int rdx_gemm_pair(const rdx_gemm_args* first, const rdx_gemm_args* second, uint32_t* dep_ctr, void* stream);

/* Debug: rdx_gemm_pair as one launch (1) or two stream-ordered launches (0) for
 * A/B runs; returns the previous setting. */
int rdx_gemm_debug_pair(int on);

/* Debug: the GEMM splits the tiles of a last partial round into 2 or 4
 * narrower tiles (same per-element K reduction, same bits); 0 turns that off
 * for A/B runs, 1 back on.  Returns the previous setting. */
int rdx_gemm_debug_tail_split(int on);

/* Debug: few-round launches (RDX_EPI_RESID_F32 / STORE) cut N into column tiles
 * of two widths (multiples of 32) so the persistent grid's rounds stay balanced
 * (same per-element K reduction, same bits); 0 turns that off for A/B runs,
 * 1 back on.  Returns the previous setting; on = -1 changes nothing and returns
 * the number of column tiles the last launch used (0 = no partition). */
int rdx_gemm_debug_colpart(int on);

/* Debug (stats builds, -DRDX_NORM_STATS_BUILD): per-block [entry, exit]
 * %globaltimer of the last rdx_rmsnorm_rows_after launch (n_blocks <= 4096). */
int rdx_norm_debug_times(unsigned long long* host, int n_blocks);

/* Debug: warps per block (4 or 8, default 4) of later rdx_rmsnorm_rows_after
 * launches without ready_ctr; 4-warp blocks fit beside a GEMM CTA. */
int rdx_norm_debug_warps(int w);

/* Debug: longest nanosleep (64..16384 ns, default 2048) of the rdx_rmsnorm_rows_after
 * slab pollers, read by the kernel at run time. */
int rdx_norm_debug_backoff(unsigned ns);

/* Debug: pin the GEMM tile shape (cg = 1 or 2 CTAs, block_n = 128 or 256) for
 * later launches, or cg = 0 for the automatic choice (A/B experiments; the
 * RDX_GEMM_SHAPE="cg,bn" environment variable sets the same override). */
int rdx_gemm_debug_shape(int cg, int block_n);

/* Debug: tile raster of later GEMM launches -- groups of group_m row blocks with
 * the row block varying fastest inside a group (0 = default; RDX_GEMM_GROUP_M in
 * the environment sets the same).  Returns the previous setting. */
int rdx_gemm_debug_group_m(int group_m);
/* Debug: raster group (row blocks) for GEMMs with K >= 8192 (default 16); returns the previous value. */
int rdx_gemm_debug_group_m_bigk(int group_m);

/* Debug: clock64 role counters of builds made with -DRDX_GEMM_STATS_BUILD (MMA
 * waits / epilogue waits and busy cycles, see gemm.cu); RDX_ERR_UNSUPPORTED
 * otherwise.  out8 may be NULL; reset != 0 zeroes the counters. */
int rdx_gemm_debug_stats(unsigned long long* out8, int reset);

/* Debug: programmatic dependent launch (PDL) of the layer-stack kernels on (1)
 * or off (0) for launches / CUDA-graph captures made after the call (default
 * off -- measured neutral; RDX_PDL=1 in the environment turns it on).  Returns
 * the previous setting. */
int rdx_debug_pdl(int on);

/* ---------------------------------------------------------------------
 * Causal GQA prefill attention on tcgen05/TMEM with the RadixMLP attention
 * boundary fused into its loads (replaces model.py:368-383 + 228-265):
 *   query i of sequence s   = row cu_q[s] + i of qkv (compact), position
 *                             lcp_s + i with lcp_s = L_s - (cu_q[s+1]-cu_q[s])
 *   key/value j of s        = row scatter[cu[s] + j] of qkv (scatter == NULL:
 *                             row cu[s] + j, i.e. plain / full layout)
 *   out[cu_q[s] + i, head]  = softmax(q k^T * scale, causal) v   (bf16)
 * qkv rows are [q heads | k heads | v heads] x head_dim (the QKV GEMM output);
 * head_dim <= 128, multiple of 8; heads % kv_heads == 0.  qkv_rows = rows of
 * the qkv buffer (bounds the TMA tile loads; rows past it read as zeros).
 * max_q_len / max_k_len = longest query range / sequence (max_k_len only
 * selects the tile pipeline; 0 = unknown).
 * --------------------------------------------------------------------- */
int rdx_attention(const void* qkv_bf16, int64_t ld_qkv, int64_t qkv_rows, const int32_t* scatter, const int32_t* cu,
                  const int32_t* cu_q, int64_t n_seqs, int32_t max_q_len, int32_t max_k_len, int32_t heads,
                  int32_t kv_heads, int32_t head_dim, float softmax_scale, void* out_bf16, int64_t ld_out,
                  void* stream);

/* Debug: with RDX_ATTN_STATS=1 in the environment every rdx_attention launch
 * sums per-role clock counters (MMA waits on K/V, P, Q, O; softmax waits on S,
 * epilogue; loader waits on free slots; totals); this copies n slots to host
 * and resets them. */
/* Debug: 1 runs short suffix-query units at head_dim 128 on 64-key K/V tiles
 * with two S buffers per query tile (S two key tiles ahead of the softmax), 0
 * (the default, also RDX_ATTN_BK64 unset) on the 128-key single-buffered kernel.
 * Same tolerance; only equal key tiles keep suffix and plain attention bit-identical.
 * Returns the previous setting. */
int rdx_attention_debug_bk64(int on);

/* Debug: a short last round of attention units (rem units, 2 rem <= CTAs) is dealt
 * as single-query-tile half units, one per CTA (1; also RDX_ATTN_SPLIT=1), or as
 * whole units (0, the default: the half units measured slower).  Returns the
 * previous setting. */
int rdx_attention_debug_split(int on);

int rdx_attention_debug_stats(unsigned long long* host, int n);
/* Debug: event log of CTA 0 of the last launch in the same mode:
 * [count, (clock, code) x min(count, 4096)] as 32-bit words. */
int rdx_attention_debug_trace(uint32_t* host, int n_words);
/* Debug (stats builds): per-CTA [start ns, end ns, units] of the last launch, n_ctas <= 1024 entries. */
int rdx_attention_debug_cta_times(unsigned long long* host, int n_ctas);

/* ---------------------------------------------------------------------
 * Reranker scores from last-token logits (fp32 [B, ld]):
 *   score[b] = sigmoid(logits[b, yes_id] - logits[b, no_id])
 * (= softmax([no, yes])[yes], the Qwen3-reranker read-out).
 * --------------------------------------------------------------------- */
int rdx_rerank_scores(const float* logits, int64_t n_rows, int64_t ld, int64_t yes_id,
                      int64_t no_id, float* scores_out, void* stream);

/* Training (training.py loss_and_grads(precision="bf16")):
 * dst[c][r] = bf16(src[r][c]) for r < rows, c < cols; dst[c][r] = 0 for
 * rows <= r < ld_dst.  Builds the K-major operands of the tcgen05 dgrad
 * (W^T) and wgrad (dY^T, X^T) GEMMs; ld_dst pads the reduction dimension to
 * the GEMM's 8-element multiple.  No reference counterpart (the reference's
 * backward is numpy fp64, model.py:419-531). */
int rdx_transpose_f32_bf16(const float* src, int64_t rows, int64_t cols, int64_t ld_src, void* dst_bf16,
                           int64_t ld_dst, void* stream);

/* Number of SMs of the current device (cached). */
int rdx_num_sms(void);

#ifdef __cplusplus
}
#endif

#endif /* RADIX_B200_H */
