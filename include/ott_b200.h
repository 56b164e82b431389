/*
 * ott_b200.h — C ABI of the B200-native OTT quantized-KV decode path.
 *
 * This is the drop-in boundary for the reference's cache/attention API
 * (/root/reference/pkg/src/kvtrace). The reference is a Python package whose
 * only "FFI" is its Python call surface; the Python host layer
 * (paper_2505_10938_b200/) binds these symbols with ctypes (see
 * INTEGRATION.md) and keeps the reference's names and error behaviour.
 *
 *   ott_ring_write   <- TieredCache.append            cache.py:124-139 (row copy part)
 *   ott_flush        <- TieredCache.quantize_oldest_group  cache.py:141-186
 *                       (score_tokens outlier.py:45-49, OutlierPool.update
 *                       outlier.py:84-117, substitute_means outlier.py:120-142,
 *                       quantize_keys_channelwise / quantize_values_tokenwise
 *                       quant.py:201-234, pack_codes quant.py:241-256)
 *   ott_attend       <- attend_mixed                   attention.py:79-92
 *                       (reconstructed_kv attention.py:62-76,
 *                       attend_full_precision attention.py:35-59)
 *   ott_logits       <- AttentionResult.scores         attention.py:26-32 (debug)
 *   ott_attend_exact <- attend_full_precision          attention.py:35-59
 *   ott_pool_rank    <- OutlierPool.update (the competition)  outlier.py:84-117
 *   ott_score_rows   <- score_tokens / OutlierEntry.from_rows  outlier.py:37-49
 *   ott_append_attend <- append + attend_mixed of one decode step (ring write fused)
 *   ott_decode_step  <- append + attend_mixed of one decode step, token counts in device
 *                       memory (CUDA-graph capturable)    cache.py:124-139, attention.py:79-92
 *
 * Conventions: all buffer pointers are DEVICE memory owned by the caller (the
 * host layer allocates them; this library never allocates or frees). Every
 * call is asynchronous on the given stream and returns an ott_status. The
 * cache holds n_units = batch * n_kv_heads independent (layer, head) caches of
 * the reference, all at the same token count (lock-step decode).
 */
#ifndef OTT_B200_H
#define OTT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  OTT_OK = 0,
  OTT_ERR_CONTRACT = 1, /* maps to kvtrace.ContractViolation (errors.py:4-5) */
  OTT_ERR_UNSUPPORTED = 2,
  OTT_ERR_CUDA = 3,
} ott_status;

/* Device-side state of one layer's batched tiered cache. Sizes in elements.
 * Block record (one per (unit, group)), byte layout, all little-endian:
 *   [0, CB)                         K codes, reference pack_codes order at the stored
 *                                   width cb; CB = ceil(G*d*cb/8) rounded up to 16 (=
 *                                   G*d*cb/8 when d in {64, 128} and G % 32 == 0).
 *                                   cb = bits, except at d = 128, G in {32, 64, 128}:
 *                                   1-bit codes in 2-bit fields (K codes stored doubled
 *                                   with the K step halved, exact), 3-bit in 4-bit and
 *                                   5..7-bit in 8-bit fields, so every width decodes on a
 *                                   tensor-core kernel
 *   [CB, 2 CB)                      V codes
 *   fp16 k_sh[d], k_sl[d]           per-channel K step = sh + sl, in pair order
 *                                   (index 16*(c/16) + 2*(c%8) + (c%16)/8 when
 *                                   d % 16 == 0, else c)
 *   stored width 2:
 *     float32 v_step[G], v_xmin[G]  per-token V params
 *     fp16 k_ehi[d], k_elo[d]       per-channel K term e = x_min - 4*u(c)*step, u(c) =
 *                                   4^(4-P(c%8)), P = {3,4,2,3,4,2,3,4} (fp16 mantissa position
 *                                   of the code pair in the decode kernels), stored as
 *                                   t = e / (8 u(c)) split into hi = fp16(t), lo = fp16(t - hi)
 *                                   (|t| < 65504 for any fp16 input),
 *                                   pair order; last in the record, so the decode kernels stream
 *                                   the record head and fetch the e fields of 8 groups at once
 *   other widths:
 *     float32 k_e[d]                stored width 4, d % 8 == 0: sh/sl in 4-bit pair order
 *                                   (8w+k, 8w+k+4), e = x_min - 64 step; stored width 8,
 *                                   d % 8 == 0: sh/sl in channel order, e = x_min - 1024 step;
 *                                   otherwise the k_sh/k_sl bytes hold float32 step[d] and k_e
 *                                   float32 x_min[d], channel order (1-bit steps can exceed the
 *                                   fp16 range)
 *     float32 v_step[G], v_xmin[G]  per-token V params
 *   (record size rounded up to 16 bytes)
 * The exact float64 QuantParams are kept in params64 when it is allocated. 
 * Per-token bitmasks hold one bit per absolute position (32 per word). */
#define OTT_MAX_OUT_PEERS 7 /* peer GPUs of an 8-GPU NVSwitch node */

typedef struct {
  int32_t n_units;      /* batch * n_kv_heads */
  int32_t head_dim;     /* d in [1, 256] (tensor-core kernels: 128; tile kernel: 64, 128) */
  int32_t group_size;   /* G in [1, 128] (tensor-core / tile kernels: multiple of 32) */
  int32_t residual;     /* R >= 0 */
  int32_t capacity;     /* N: pool capacity for this layer (EngineConfig.outlier_capacity) */
  int32_t aux_capacity; /* A */
  int32_t bits;         /* 1..8 (levels 2^bits - 1; the stored width picks the decode kernel) */
  int32_t max_groups;   /* block records allocated per unit */
  uint8_t* blocks;      /* [n_units][max_groups][record_bytes] */
  uint16_t* pend_k;     /* fp16 [n_units][G+R][d], slot = position % (G+R) */
  uint16_t* pend_v;
  uint32_t* pool_mask;  /* [n_units][ceil(max_groups*G/32)]: 1 = position in pool.entries */
  uint32_t* subst_mask; /* [n_units][ceil(max_groups*G/32)]: substituted_positions */
  int32_t* pool_pos;    /* [n_units][N] slot-stable entries, -1 = empty; reference order =
                           ascending (score, position), outlier.py:52-54 */
  double* pool_score;   /* [n_units][N] */
  uint16_t* pool_k;     /* fp16 [n_units][N][d] */
  uint16_t* pool_v;
  int32_t* aux_pos;     /* [n_units][A] in reference order */
  double* aux_score;    /* [n_units][A] */
  uint16_t* aux_k;      /* fp16 [n_units][A][d] */
  uint16_t* aux_v;
  int32_t* pool_meta;   /* [n_units][4] = {n_entries, n_aux, frozen, float bits of the largest
                           2/4-bit K or V step flushed (overflow guard of the tensor-core
                           attention; start at 0)} */
  double* params64;     /* optional [n_units][max_groups][2*(d+G)] exact float64 params
                           (k_xmin[d], k_step[d], v_xmin[G], v_step[G]); NULL = off */
  int32_t n_out_peers;  /* fused output all-gather, 0 = off: the attention epilogue
                           stores every output row into `out` and into each out_peer[i] (same
                           [n_units][n_rep][d] layout) -- typically this rank's rows of a peer
                           GPU's gather buffer, written over NVLink (parallel.PeerGather) */
  uint16_t* out_peer[OTT_MAX_OUT_PEERS];
} ott_cache_t;

/* sizeof(ott_cache_t), for binding-side layout checks. */
size_t ott_cache_struct_bytes(void);

/* Bytes of one block record for the given shape. */
size_t ott_record_bytes(int32_t head_dim, int32_t group_size, int32_t bits);

/* Copy rows into the pending ring. Row r (0 <= r < n_rows) of unit u is read
 * from k + u*in_unit_stride + (first_pos - in_first_pos + r)*d and lands at
 * ring slot (first_pos + r) % (G+R). Rows are fp16. */
int ott_ring_write(const ott_cache_t* c, const uint16_t* k, const uint16_t* v, int64_t in_unit_stride,
                   int64_t in_first_pos, int64_t first_pos, int64_t n_rows, void* stream);

/* Quantize n_groups consecutive groups per unit, starting at absolute position
 * quantized_tokens (sequentially: each group's pool competition sees the pool
 * left by the previous one, cache.py:141-186). A row at position p is read
 * from the pending ring when p < ring_end, else from
 * in_k + u*in_unit_stride + (p - in_first_pos)*d (bulk prefill). */
int ott_flush(const ott_cache_t* c, int64_t quantized_tokens, int32_t n_groups, int64_t ring_end,
              const uint16_t* in_k, const uint16_t* in_v, int64_t in_unit_stride, int64_t in_first_pos,
              void* stream);

/* Mixed-tier decode attention (attend_mixed) for n_rep query heads per unit.
 * q, out: fp16 [n_units][n_rep][d] (= [B][H_q][d] with H_q = H_kv*n_rep), n_rep in [1, 128]
 * (3, 5, 6, 7 run padded to 4 or 8 heads, more than 8 in chunks of 8 heads; the workspace then
 * also holds the staged q/out).
 * The sequence axis is split n_splits ways (split-K flash decoding) and the
 * partials merged in-kernel; ott_pick_splits chooses a count that fills the
 * GPU, ott_attend_workspace_floats sizes the float32 workspace for it. */
int ott_pick_splits(const ott_cache_t* c, int32_t n_rep, int64_t total_tokens);
size_t ott_attend_workspace_floats(const ott_cache_t* c, int32_t n_rep, int32_t n_splits);
int ott_attend(const ott_cache_t* c, const uint16_t* q, uint16_t* out, int32_t n_rep, int64_t quantized_tokens,
               int64_t total_tokens, float* workspace, int32_t n_splits, void* stream);

/* Debug: pre-softmax logits (AttentionResult.scores, attention.py:55) for all
 * total_tokens positions, float32 [n_units][n_rep][total_tokens]. */
/* append + attend of one decode step with host token counts: (k, v) [n_units][head_dim] is
 * the row at position total_tokens - 1 (total_tokens counts it). A flush that became due
 * with this row must have been launched before (ott_flush; with residual >= 1 it never
 * needs the new row). On the tensor-core path the attention kernel writes the row into
 * the pending ring itself (no separate ring-write launch). */
int ott_append_attend(const ott_cache_t* c, const uint16_t* k, const uint16_t* v, const uint16_t* q, uint16_t* out,
                      int32_t n_rep, int64_t quantized_tokens, int64_t total_tokens, float* workspace,
                      int32_t n_splits, void* stream);

/* One decode step with the token counts in device memory, so a whole model step can be
 * captured in a CUDA graph and replayed: counters = int64[3] {quantized_tokens,
 * total_tokens, error} on the device, read by the kernels and advanced by the last one;
 * a step that makes a flush due with no group record left sets error = 1 and leaves the
 * counts unchanged (the host raises ContractViolation when it reads the flag).
 * Launches: ring write of (k, v) [n_units][head_dim] at position total, flush of one
 * group per unit iff it became due (cache.py:138; the kernel returns early otherwise),
 * split-K attention of q [n_units*n_rep][head_dim] -> out, and the combine. n_splits
 * is fixed by the caller (size it for the largest context of the run). The caller
 * guarantees capacity (max_groups) for the steps it replays. */
int ott_decode_step(const ott_cache_t* c, const uint16_t* k, const uint16_t* v, const uint16_t* q, uint16_t* out,
                    int32_t n_rep, int64_t* counters, float* workspace, int32_t n_splits, void* stream);

int ott_logits(const ott_cache_t* c, const uint16_t* q, float* logits, int32_t n_rep, int64_t quantized_tokens,
               int64_t total_tokens, void* stream);

/* attend_full_precision (attention.py:35-59), the reference's exact single-query attention,
 * for n_q independent problems in float32 device buffers: q [n_q][d], keys/values
 * [n_q][n][d]; out [n_q][d], weights [n_q][n], scores [n_q][n] (scores = (K q) / f32(sqrt(d))
 * in float32, softmax in float64 with max subtraction as tensor.py:45-57, out = weights V in
 * float32). n >= 1 (attention.py:48-49). */
int ott_attend_exact(const float* q, const float* keys, const float* values, int32_t n, int32_t d, int32_t n_q,
                     float* out, float* weights, float* scores, void* stream);

/* The competition of OutlierPool.update (outlier.py:84-117): rank of each of the n items
 * (pool entries then candidates) in ascending (score, position) order, positions distinct
 * (the caller rejects duplicates, outlier.py:96-100). Winners are the ranks < capacity, in
 * rank order. scores f64 [n], positions i64 [n], rank i32 [n], device memory. */
int ott_pool_rank(const double* scores, const int64_t* positions, int32_t n, int32_t* rank, void* stream);

/* score_tokens / OutlierEntry.from_rows (outlier.py:37-49, row_l1_norm tensor.py:38-42):
 * scores[r] = sum_j |rows[r][j]| in float64, rows float32 [n][d], device memory. */
int ott_score_rows(const float* rows, int32_t n, int32_t d, double* scores, void* stream);

/* Number of SMs of the current device (0 if unknown) and library version. */
int ott_num_sms(void);
const char* ott_version(void);
const char* ott_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
