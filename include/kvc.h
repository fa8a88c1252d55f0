/*
 * kvc.h - C ABI of the B200-native KV-Compress hot path (libkvc.so).
 *
 * Plain pointers, sizes and a cudaStream_t (passed as void*); no torch
 * types.  Every entry point is asynchronous on `stream` and returns an
 * immediate launch status (KVC_OK or a negative kvc_status).  Errors that
 * depend on device data (shortfalls, empty heads, schedule corruption) are
 * written to the pool's device status word `status[0..3]` and surface at
 * the caller's next synchronisation point (kvc_status_name + the Python
 * facade map them onto the reference's exception classes, errors.py:6-67).
 *
 * Reference interface replaced by each entry point (pkg/src/pagedkv/...):
 *
 *   kvc_alloc_prefill       BlockManager.allocate_prefill     block_manager.py:56-72
 *   kvc_alloc_decode        BlockManager.allocate_decode_step block_manager.py:74-97
 *   kvc_alloc_heads         BlockManager._take (per-head runs) block_manager.py:47-52
 *   kvc_free_trailing       BlockManager.free_blocks + MetricsStore.clear_blocks
 *                                                             block_manager.py:101-129,
 *                                                             metrics.py:177-183
 *   kvc_free_sequence       BlockManager.free_sequence        block_manager.py:131-136
 *   kvc_append_kv           append_kv + MetricsStore.on_append cache.py:163-184,
 *                                                             metrics.py:153-158
 *   kvc_write_prefill_kv    Engine._prefill K/V scatter       engine.py:340-348
 *   kvc_write_prompt_pass   MetricsStore.write_prompt_pass    metrics.py:160-175
 *   kvc_paged_decode        paged_attention (+ accumulate_decode fused, + append
 *                           fused)                            attention.py:92-127,
 *                                                             metrics.py:189-211
 *   kvc_accumulate_rows     accumulate_decode                 metrics.py:189-211
 *   kvc_full_metric         gqa_attention -> full_metrics     metrics.py:92-109
 *   kvc_window_metric       gqa_attention -> window_metrics -> write_prompt_pass
 *                                                             attention.py:62-89,
 *                                                             metrics.py:68-89,160-175
 *   kvc_schedule_evictions  build_views .. eviction_mask      compression.py:122-231
 *   kvc_execute_moves       move_cache + free_schedule_blocks compression.py:234-309
 *   kvc_compress            compress (both of the above)      compression.py:312-355
 *   kvc_prefill_compress    prefill scatter + compress fused  engine.py:340-358 + compression.py:312-355
 *   kvc_clear_fresh         MetricsStore.clear_fresh          metrics.py:185-186
 *   kvc_gqa_attention       gqa_attention (dense causal GQA)  attention.py:62-89
 *   kvc_attn_metrics        window_metrics / full_metrics on an attention tensor
 *                                                             metrics.py:50-109
 */
#ifndef KVC_H_
#define KVC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KVC_ABI_VERSION 3 /* 2: kvc_decode_args.early_pull; queue int32[2 + batch*heads]
                            3: kvc_window_args.write_k, kvc_write_prefill_v_layers */
#define KVC_FREE_TILE 1024 /* blocks per free-count tile */

typedef enum kvc_status {
  KVC_OK = 0,
  KVC_ERR_INVALID = -1,          /* ValueError / ConfigError: bad argument */
  KVC_ERR_UNSUPPORTED = -2,      /* shape outside the compiled kernels */
  KVC_ERR_CUDA = -3,             /* CUDA launch/runtime failure */
  /* device-side conditions (status[0]) */
  KVC_DEV_PREEMPTION = 1,        /* PreemptionNeeded(shortfall = status[1]) */
  KVC_DEV_ALLOCATION_ORDER = 2,  /* AllocationOrderError */
  KVC_DEV_EMPTY_CONTEXT = 3,     /* EmptyContextError */
  KVC_DEV_NUMERIC = 4,           /* NumericError */
  KVC_DEV_SCHEDULE_CORRUPTION = 5, /* ScheduleCorruptionError */
  KVC_DEV_CACHE_CORRUPTION = 6,  /* CacheCorruptionError */
  KVC_DEV_CAPACITY = 7           /* a head outgrew the table capacity */
} kvc_status;

/*
 * Device-resident state of one GPU's unified cache (caller-owned memory).
 * Slot f = block * block_size + offset addresses row f of k/v and the
 * per-slot arrays (cache.py:50-57).  metric/logical/protected_/fresh may be
 * NULL for calls that do not touch the store (allocator-only use, exactly
 * like the reference BlockManager which never touches the MetricsStore).
 */
typedef struct kvc_pool {
  void *k_cache;            /* bf16 [num_blocks][block_size][head_dim] */
  void *v_cache;            /* bf16 [num_blocks][block_size][head_dim] */
  float *metric;            /* [num_blocks*block_size] eviction metric   */
  int32_t *logical;         /* [num_blocks*block_size] logical idx, -1 = empty */
  uint8_t *protected_;      /* [num_blocks*block_size] 1 = observation-window shield */
  uint8_t *fresh;           /* [num_blocks*block_size] 1 = created this step */
  uint8_t *free_flag;       /* [num_blocks] 1 = free */
  int32_t *free_tile;       /* [ceil(num_blocks/KVC_FREE_TILE)] free blocks per tile */
  int32_t *tables;          /* [max_seqs][num_layers][num_kv_heads][max_blocks] */
  int32_t *nblocks;         /* [max_seqs][num_layers][num_kv_heads] table length */
  int32_t *ctx;             /* [max_seqs][num_layers][num_kv_heads] live KVs C */
  int32_t *status;          /* [4] device status word (see kvc_status) */
  int32_t *scratch;         /* workspace, scratch_bytes long */
  int64_t scratch_bytes;
  int64_t num_blocks;
  int32_t block_size;
  int32_t head_dim;
  int32_t num_layers;
  int32_t num_kv_heads;
  int32_t max_seqs;
  int32_t max_blocks;       /* table capacity per head */
} kvc_pool;

/* Library / ABI identification. */
int kvc_abi_version(void);
const char *kvc_status_name(int status);

/* Reset free flags/tiles (all free), tables, ctx and per-slot arrays. */
int kvc_pool_init(const kvc_pool *pool, void *stream);

/* Workspace bytes needed for rounds of up to `max_heads` heads / `max_slots`
 * slots and decode batches of `max_batch` sequences. */
int64_t kvc_scratch_bytes(const kvc_pool *pool, int64_t max_heads, int64_t max_slots,
                          int32_t max_batch);

/* ---- K0: block allocator (smallest free ids first) ---------------------- */

/* Prefill: every (layer, head) of `seq_row` gets `blocks_per_head` ids, heads
 * in layer-major order, each a consecutive run of the smallest free ids.
 * All-or-nothing; shortfall -> status[0]=KVC_DEV_PREEMPTION, status[1]. */
int kvc_alloc_prefill(const kvc_pool *pool, int32_t seq_row, int32_t blocks_per_head,
                      void *stream);

/* Arbitrary per-head runs for one sequence: head i (layer-major) receives
 * counts[i] ids (device int32 [layers*heads]); `total` = sum(counts). */
int kvc_alloc_heads(const kvc_pool *pool, int32_t seq_row, const int32_t *counts,
                    int64_t total, void *stream);

/* Decode step: one id for every head of the listed rows whose C % b == 0,
 * served in the given row order (caller passes rows sorted by sequence id),
 * then (layer, head).  Writes per-row counts to out_counts (device int32
 * [n_rows]).  All-or-nothing. */
int kvc_alloc_decode(const kvc_pool *pool, const int32_t *seq_rows, int32_t n_rows,
                     int32_t *out_counts, void *stream);

/* Free the trailing `drop[i]` table entries of head (row, layer, head) for
 * the listed heads; ctx := min(ctx, keep*b); freed slots reset to empty.
 * heads: device int32 [n][3] = (row, layer, head), drop: int32 [n]. */
int kvc_free_trailing(const kvc_pool *pool, const int32_t *heads, const int32_t *drop,
                      int32_t n, void *stream);

/* Free every block of a row (and reset its slots); table length/ctx := 0. */
int kvc_free_sequence(const kvc_pool *pool, int32_t seq_row, void *stream);

/* ---- KV write paths ------------------------------------------------------ */

/* Append one KV per listed head at position C; C += 1; slot: metric 0,
 * logical C, fresh = `fresh`, protected 0.  k/v bf16 [n][head_dim];
 * heads int32 [n][3]. */
int kvc_append_kv(const kvc_pool *pool, const int32_t *heads, const void *k,
                  const void *v, int32_t n, int32_t fresh, void *stream);

/* Scatter a prompt's K/V for one (row, layer): k/v bf16 [heads][L][head_dim]
 * into positions 0..L-1 of each head; C := L. */
int kvc_write_prefill_kv(const kvc_pool *pool, int32_t seq_row, int32_t layer,
                         const void *k, const void *v, int32_t L, void *stream);

/* The same for n_layers consecutive layers (layer, layer+1, ...) in one
 * launch; k/v bf16 [n_layers][heads][L][head_dim] (engine.py:340-348 loops
 * the layers of a prompt). */
int kvc_write_prefill_kv_layers(const kvc_pool *pool, int32_t seq_row, int32_t layer,
                                int32_t n_layers, const void *k, const void *v, int32_t L,
                                void *stream);

/* Companion of kvc_window_metric with write_k = 1 (the K2 pass stores the K
 * rows of the whole 16-key blocks): every V row, and the K rows of each
 * head's partial last block; C := L.  Same layout as
 * kvc_write_prefill_kv_layers. */
int kvc_write_prefill_v_layers(const kvc_pool *pool, int32_t seq_row, int32_t layer,
                               int32_t n_layers, const void *k, const void *v, int32_t L,
                               void *stream);

/* Install prompt metrics for one (row, layer): metrics f32 [heads][L],
 * protected u8 [L] (nullable = none); logical := position, fresh := 0. */
int kvc_write_prompt_pass(const kvc_pool *pool, int32_t seq_row, int32_t layer,
                          const float *metrics, int64_t metrics_stride,
                          const uint8_t *protected_mask, int32_t L, void *stream);

/* ---- K1: paged GQA decode with fused append + metric accumulation ------- */

typedef struct kvc_decode_args {
  const int32_t *seq_rows;  /* [batch] table rows */
  int32_t batch;
  int32_t layer;
  int32_t num_query_heads;  /* n_q = r * num_kv_heads */
  const void *q;            /* bf16 [batch][n_q][head_dim] */
  const void *k_new;        /* bf16 [batch][heads][head_dim] or NULL (no append) */
  const void *v_new;
  void *out;                /* [batch][n_q][head_dim], bf16 or f32 (out_f32) */
  int32_t out_f32;
  float *rows_out;          /* NULL or f32 [batch][heads][r][rows_stride] */
  int64_t rows_stride;
  int32_t metric_mode;      /* 0 none, 1 L1, 2 L2: metric[slot] += sum_h f(p) */
  int32_t append_fresh;     /* fresh flag for appended slots */
  int32_t max_ctx;          /* upper bound on C (+1 if appending) over the batch */
  int32_t splits;           /* 0 = auto, else CTAs (cluster size) per head */
  int32_t *queue;           /* NULL, or a caller-owned device int32[2 + batch*heads]
                               that is zero on entry; the call leaves it zero, so
                               the caller allocates it once and skips a memset
                               per call.  NULL: the call zeroes a scratch copy. */
  void *metric_stream;      /* NULL, or a cudaStream_t: the metric accumulation
                               (metric_mode, no rows_out) runs there, forked
                               after this call's attention; the caller joins it
                               and must not reuse this call's scratch before
                               (DecodeStepGraph double-buffers). */
  int32_t early_pull;       /* 1: the caller guarantees that the work enqueued on
                               `stream` right before this call is a
                               kvc_paged_decode of ANOTHER layer over the same
                               `queue` (consecutive layers of one decode step),
                               so this call's first work pull and its first KV
                               loads may run before that call finishes.  0 (the
                               safe default): everything waits for the prior
                               stream work (allocator, compaction, scatter, ...).
                               2: the first layer of such a chain - no early
                               pull, but the launch leaves room on every SM for
                               the next layer's early pull (d = 128). */
} kvc_decode_args;

int kvc_paged_decode(const kvc_pool *pool, const kvc_decode_args *args, void *stream);

/* Workspace the decode fast path needs for `batch` sequences with contexts
 * up to `max_ctx` (fp32 score rows + split-KV partials).  With less scratch
 * kvc_paged_decode uses the single-pass cluster kernel. */
int64_t kvc_decode_scratch_bytes(const kvc_pool *pool, int32_t batch, int32_t num_query_heads,
                                 int32_t max_ctx);

/* metric[slot_j] += sum_h f(rows[h][j]) for one (row, layer): rows f32
 * [heads][r][rows_stride] covering each head's C live KVs. */
int kvc_accumulate_rows(const kvc_pool *pool, int32_t seq_row, int32_t layer,
                        const float *rows, int32_t r, int64_t rows_stride,
                        int32_t metric_mode, void *stream);

/* Clear the fresh bit: all slots (rows == NULL) or the last slot of every head
 * of the listed rows (the slots a decode step created). */
int kvc_clear_fresh(const kvc_pool *pool, const int32_t *seq_rows, int32_t n_rows,
                    void *stream);

/* ---- K2: observation-window metric (prefill) ----------------------------- */

typedef struct kvc_window_args {
  int32_t seq_row;          /* <0: do not install into the store */
  int32_t layer;
  int32_t num_query_heads;
  int32_t L;                /* prompt length */
  const void *q_win;        /* bf16 [n_q][w'][head_dim], w' = min(window, L) */
  const void *k;            /* bf16 [heads][L][head_dim] (prompt keys) */
  int32_t window;
  int32_t pool;             /* odd max-pool width */
  int32_t aggregation;      /* 1 L1, 2 L2 */
  int32_t protect_window;
  float *metrics_out;       /* NULL or f32 [heads][L] pooled metrics */
  /* several consecutive layers in one call (layer, layer+1, ...): strides in
   * elements between the layers' q_win / k / metrics_out; n_layers <= 1 = one */
  int32_t n_layers;
  int64_t q_layer_stride;
  int64_t k_layer_stride;
  int64_t out_layer_stride;
  /* 1 (with seq_row >= 0, block_size 16): the kernel also stores the prompt K
   * rows of every whole 16-key block into the pool's k_cache through the
   * tables, from the tiles it streams anyway (the prompt's K is read once);
   * pair it with kvc_write_prefill_v_layers.  KVC_ERR_UNSUPPORTED (nothing
   * done) on shapes that take the per-layer kernels. */
  int32_t write_k;
} kvc_window_args;

int kvc_window_metric(const kvc_pool *pool, const kvc_window_args *args, void *stream);

/* ---- f3: KVC-full metric (prefill) --------------------------------------- */

typedef struct kvc_full_args {
  int32_t num_query_heads;
  int32_t L;                /* prompt length */
  const void *q;            /* bf16 [n_q][L][head_dim] (all prompt queries) */
  const void *k;            /* bf16 [heads][L][head_dim] */
  int32_t excluded;         /* v: key j aggregates queries i >= j + v */
  int32_t aggregation;      /* 1 L1, 2 L2 */
  float *metrics_out;       /* f32 [heads][L] */
} kvc_full_args;

/* full_metrics (metrics.py:92-109) over gqa_attention's causal softmax
 * (attention.py:62-89) for one layer, on tcgen05: row statistics, then
 * column sums over rows i >= j + v.  Install with kvc_write_prompt_pass. */
int kvc_full_metric(const kvc_pool *pool, const kvc_full_args *args, void *stream);

/* ---- reference-signature metrics on an explicit attention tensor --------- */

typedef struct kvc_dense_args {
  int32_t num_query_heads;
  int32_t L;
  const float *q;           /* f32 [n_q][L][head_dim] */
  const float *k;           /* f32 [heads][L][head_dim] */
  const float *v;           /* f32 [heads][L][head_dim] or NULL (no output) */
  float *out;               /* f32 [n_q][L][head_dim] or NULL */
  float *attn;              /* f32 [n_q][L][L]: causal row softmax, 0 above the diagonal */
} kvc_dense_args;

/* gqa_attention (attention.py:62-89): query head h reads KV head h / r;
 * fp32, max-subtracted softmax.  Non-finite scores -> KVC_DEV_NUMERIC.
 * Materialises the (n_q, L, L) attention like the reference (L <= ~56k). */
int kvc_gqa_attention(const kvc_pool *pool, const kvc_dense_args *args, void *stream);

typedef struct kvc_attn_metric_args {
  int32_t num_query_heads;
  int32_t L;
  const float *attn;        /* f32 [n_q][L][L] */
  int32_t mode;             /* 0 window_metrics, 1 full_metrics */
  int32_t window;           /* window mode: last `window` query rows */
  int32_t pool;             /* window mode: odd max-pool width (scratch: heads*L f32 when > 1) */
  int32_t excluded;         /* full mode: key j aggregates rows i >= j + excluded */
  int32_t aggregation;      /* 1 L1, 2 L2 */
  float *metrics_out;       /* f32 [heads][L] */
} kvc_attn_metric_args;

/* window_metrics (metrics.py:68-89) / full_metrics (metrics.py:92-109) of an
 * attention tensor: group sums over each KV head's r query heads, then the
 * centred max-pool (window mode).  The protected mask is the caller's
 * (positions >= L - window unless protect_window is off). */
int kvc_attn_metrics(const kvc_pool *pool, const kvc_attn_metric_args *args, void *stream);

/* ---- K3 + K4: eviction schedule and compaction --------------------------- */

typedef struct kvc_evict_args {
  const int32_t *seq_rows;  /* [n_seqs] rows, processed independently */
  const int64_t *budgets;   /* [n_seqs] requested blocks E_s */
  int32_t n_seqs;
  int64_t max_slots_per_head; /* upper bound on nb*b over the round */
  /* outputs (device) */
  int64_t *clamped;         /* [n_seqs] min(E_s, sum cap) */
  int32_t *evict;           /* [n_seqs][layers*heads] evicted blocks per head */
  int32_t *evicted_kvs;     /* [n_seqs][layers*heads] */
  int32_t *freed;           /* NULL or [n_seqs][layers*heads][max_blocks] freed ids */
  int32_t *moves;           /* NULL or [total move capacity][2] (src, dst) flats */
  int64_t moves_capacity;
  int64_t *move_offsets;    /* [n_seqs*layers*heads + 1] exclusive prefix of e*b */
  int32_t *move_counts;     /* [n_seqs][layers*heads] */
  int64_t *totals;          /* [4]: freed blocks, evicted kvs, moves, free count */
  /* NULL, or [n_seqs*layers*heads][max_slots_per_head]: for each kept
   * position after compaction, the logical it held before renumbering
   * (-1 = empty); written by kvc_prefill_compress's compaction */
  int32_t *src_pos;
} kvc_evict_args;

/* Per-head evicted block counts (schedule_evictions); no state mutation. */
int kvc_schedule_evictions(const kvc_pool *pool, const kvc_evict_args *args, void *stream);

/* Compaction + trailing free + logical renumbering using the counts the
 * previous kvc_schedule_evictions call left in args->evict. */
int kvc_execute_moves(const kvc_pool *pool, const kvc_evict_args *args, void *stream);

/* schedule_evictions + execute_moves in one pass over the slots (the
 * reference's compress, compression.py:312-355). */
int kvc_compress(const kvc_pool *pool, const kvc_evict_args *args, void *stream);

/* Compress a prompt that was allocated and scored (kvc_window_metric with
 * seq_row) but whose K/V was never scattered: schedule + compaction on the
 * slot metadata, then each surviving prompt row is written straight to its
 * final slot.  The resulting tables, ctx, free list, slot metadata and live
 * K/V equal kvc_write_prefill_kv_layers + kvc_compress (engine.py:340-358
 * followed by compression.py:312-355) without writing the evicted rows or
 * moving the survivors.  One sequence (args->n_seqs == 1); k/v bf16
 * [layers][heads][L][head_dim]; args->src_pos is scratch for the call. */
int kvc_prefill_compress(const kvc_pool *pool, const kvc_evict_args *args, const void *k,
                         const void *v, int32_t L, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* KVC_H_ */
