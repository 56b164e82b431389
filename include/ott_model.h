/* ott_model.h — fused elementwise kernels of the config-1 decoder's decode step
 * (paper_2505_10938_b200/model.py). Not part of the reference's interface: the
 * reference has no model (it replays traces); these serve the Llama-shaped decoder
 * that turns the cache kernels into model decode tokens/s.
 * fp16 device tensors, asynchronous on `stream`; return 0 on success. */
#ifndef OTT_MODEL_H
#define OTT_MODEL_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* y[r] = fp16(x[r] * rsqrt(mean(x[r]^2) + eps)) * w, rows x dim (dim % 8 == 0). */
int ott_model_rmsnorm(const uint16_t* x, const uint16_t* w, uint16_t* y, int32_t rows, int32_t dim, float eps,
                      void* stream);

/* qkv [batch][(H + 2 Hkv) d] -> q [batch][H][d], k [batch][Hkv][d] (rotate-half RoPE at
 * position *pos_dev, or pos_host when pos_dev is NULL; fp32 cos/sin tables [pos][d]),
 * v [batch][Hkv][d]. */
int ott_model_rope_qkv(const uint16_t* qkv, const float* cos_t, const float* sin_t, const int64_t* pos_dev,
                       int64_t pos_host, uint16_t* q, uint16_t* k, uint16_t* v, int32_t batch, int32_t n_heads,
                       int32_t n_kv_heads, int32_t head_dim, void* stream);

/* out [rows][n] = fp16(silu(a) * b) for h [rows][2n] = (a | b). */
int ott_model_silu_mul(const uint16_t* h, uint16_t* out, int32_t rows, int32_t n, void* stream);

#ifdef __cplusplus
}
#endif
#endif
