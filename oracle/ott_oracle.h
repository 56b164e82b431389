/*
 * ott_oracle.h — CPU restatement of the reference OTT (kvtrace) write and read
 * path, used ONLY as a parity checker and CPU baseline (tests/, smoke(), and
 * bench.py's cpu_baseline / --impl reference legs). Never linked by the product.
 *
 * Every function cites the reference file:line it restates
 * (paths relative to /root/reference/pkg/src/kvtrace/).
 *
 * Parity pinned: tests/test_oracle_golden.py checks this oracle against golden
 * vectors produced by importing the reference itself (tests/golden/make_golden.py).
 */
#ifndef OTT_ORACLE_H
#define OTT_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* quant.py:59-102 (_line_params + quantize_uniform). x: float64 line of n values.
 * Returns 0, or -1 on contract violation (bad bits, n == 0, non-finite). */
int ottref_quantize_line(const double* x, int n, int bits, int64_t* codes, double* x_min, double* step);

/* quant.py:241-256 pack_codes / 259-273 unpack_codes: LSB-first bit stream.
 * pack returns bytes written (ceil(count*bits/8)) or -1 if a code overflows. */
long ottref_pack_codes(const int64_t* codes, size_t count, int bits, uint8_t* out);
void ottref_unpack_codes(const uint8_t* data, size_t count, int bits, int64_t* out);

/* quant.py:201-234 _quantize_group. group: float32 [n_tokens][n_channels].
 * axis 0 = PER_CHANNEL (keys), 1 = PER_TOKEN (values). codes_out gets the packed
 * block (token-major element order, quant.py:215-218); x_min/step get one entry
 * per line (n_channels lines for PER_CHANNEL, n_tokens for PER_TOKEN). */
int ottref_quantize_group(const float* group, int n_tokens, int n_channels, int bits, int axis,
                          uint8_t* codes_out, double* x_min, double* step);

/* One (layer, head) TieredCache (cache.py:90-203) with its OutlierPool
 * (outlier.py:57-117). Opaque handle. */
typedef struct ottref_cache ottref_cache;

ottref_cache* ottref_cache_new(int bits, int group_size, int residual, int capacity, int aux_capacity,
                               int head_dim);
void ottref_cache_free(ottref_cache* c);
ottref_cache* ottref_cache_clone(const ottref_cache* c);

/* cache.py:124-139. Rows are float32 [head_dim]. Returns 0 or -1 (non-finite). */
int ottref_append(ottref_cache* c, const float* k_row, const float* v_row);
/* cache.py:141-186. Returns 0 or -1 when fewer than G rows are pending. */
int ottref_quantize_oldest_group(ottref_cache* c);

/* attention.py:62-92 (reconstructed_kv + attend_mixed + attend_full_precision).
 * out: float32 [head_dim]; weights/scores: optional float32 [total_tokens]
 * (NULL to skip). Scores and softmax are evaluated in float64 and rounded to
 * float32 (the reference uses float32 BLAS for the dot products; the two
 * agree to tolerance, not bitwise). Returns 0 or -1 on an empty cache. */
int ottref_attend(const ottref_cache* c, const float* q, float* out, float* weights, float* scores);
/* attention.py:65-76 reconstructed_kv: K, V float32 [total_tokens][head_dim]. */
void ottref_reconstructed_kv(const ottref_cache* c, float* keys, float* values);

/* state accessors (for parity against the GPU cache) */
int64_t ottref_total_tokens(const ottref_cache* c);
int64_t ottref_quantized_tokens(const ottref_cache* c);
int ottref_pending_rows(const ottref_cache* c);
int ottref_n_blocks(const ottref_cache* c);
int ottref_block_bytes(const ottref_cache* c);
/* block b: packed K codes, V codes (block_bytes each), K params (head_dim lines),
 * V params (group_size lines); any pointer may be NULL */
void ottref_block(const ottref_cache* c, int b, uint8_t* kcodes, uint8_t* vcodes, double* k_xmin,
                  double* k_step, double* v_xmin, double* v_step);
void ottref_pending(const ottref_cache* c, float* k, float* v);
int ottref_pool_size(const ottref_cache* c);
int ottref_aux_size(const ottref_cache* c);
int ottref_frozen(const ottref_cache* c);
/* pool entries in stored order (sorted by (score, position)), outlier.py:102-117 */
void ottref_pool_entries(const ottref_cache* c, int64_t* pos, double* score, float* keys, float* values);
void ottref_aux_entries(const ottref_cache* c, int64_t* pos, double* score, float* keys, float* values);
/* substituted_positions (cache.py:103,173), ascending */
int ottref_n_substituted(const ottref_cache* c);
void ottref_substituted(const ottref_cache* c, int64_t* pos);
/* cache.py:188-203 memory_usage: {quantized_bits, param_bits, pending_bits, pool_bits} */
void ottref_memory_usage(const ottref_cache* c, int64_t out[4]);

/* CPU baseline driver: one decode step (append k/v rows, flush if due, then
 * n_rep attend calls per unit) over n_units caches with `threads` OpenMP
 * threads. k,v: [n_units][head_dim]; q/out: [n_units][n_rep][head_dim]. */
int ottref_decode_step(ottref_cache** caches, int n_units, const float* k, const float* v, const float* q,
                       int n_rep, float* out, int threads);
/* Bulk prefill: n_tokens sequential appends per unit; k,v: [n_units][n_tokens][head_dim]. */
int ottref_prefill(ottref_cache** caches, int n_units, const float* k, const float* v, int n_tokens,
                   int threads);

#ifdef __cplusplus
}
#endif
#endif
