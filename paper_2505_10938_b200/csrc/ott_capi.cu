// ott_capi.cu — extern "C" entry points (include/ott_b200.h): argument checks
// that mirror the reference's ContractViolation preconditions, then launches.
#include <stdio.h>
#include <string.h>

#include <algorithm>

#include "ott_common.cuh"

namespace ott {
cudaError_t launch_flush(const ott_cache_t& c, int64_t q0, int n_groups, int64_t ring_end, const uint16_t* in_k,
                         const uint16_t* in_v, int64_t in_stride, int64_t in_first, cudaStream_t st,
                         const int64_t* dev_counts = nullptr);
cudaError_t launch_ring_write(const ott_cache_t& c, const uint16_t* k, const uint16_t* v, int64_t in_stride,
                              int64_t in_first, int64_t first_pos, int64_t n_rows, cudaStream_t st,
                              const int64_t* dev_counts = nullptr);
cudaError_t launch_attend(const ott_cache_t& c, const uint16_t* q, uint16_t* out, int n_rep, int64_t q_tokens,
                          int64_t total, float* ws, int n_splits, cudaStream_t st, int64_t* dev_counts = nullptr,
                          const uint16_t* new_k = nullptr, const uint16_t* new_v = nullptr, bool advance = true);
bool attend_fuses_ring_write(const ott_cache_t& c);
bool mma_eligible(const ott_cache_t& c);
cudaError_t launch_logits(const ott_cache_t& c, const uint16_t* q, float* logits, int n_rep, int64_t q_tokens,
                          int64_t total, cudaStream_t st);
cudaError_t launch_rep_pad(const uint16_t* q, uint16_t* qs, int n_units, int n_rep, int h0, int nh, int nr, int d,
                           cudaStream_t st);
cudaError_t launch_rep_unpad(const ott_cache_t& c, const uint16_t* os, uint16_t* out, int n_rep, int h0, int nh,
                             int nr, cudaStream_t st);
cudaError_t launch_attend_exact(const float* q, const float* keys, const float* values, int n, int d, int n_q,
                                float* out, float* weights, float* scores, cudaStream_t st);
cudaError_t launch_pool_rank(const double* s, const int64_t* p, int n, int32_t* rank, cudaStream_t st);
cudaError_t launch_score_rows(const float* rows, int n, int d, double* out, cudaStream_t st);
}  // namespace ott

// Query heads per KV head the attention kernels are instantiated for: 1, 2, 4, 8. Other counts
// up to 8 run padded to the next one (zero query rows, outputs dropped); more than 8 (MQA-style
// layouts) run in chunks of 8 heads, each chunk one padded launch over the unit's cache.
constexpr int kMaxRep = 128;
static int native_rep(int n_rep) {
  if (n_rep < 1 || n_rep > kMaxRep) return 0;
  return n_rep <= 2 ? n_rep : (n_rep <= 4 ? 4 : 8);
}

static size_t partial_floats(const ott_cache_t* c, int nr, int n_splits) {
  // partials [units][nr][splits + 2][d + 2] (up to two full-precision-tier partials) + 2 floats
  // (the launch's quantized-token count), rounded to 16 bytes
  const size_t f = (size_t)c->n_units * nr * ((n_splits > 0 ? n_splits : 1) + 2) * (c->head_dim + 2) + 2;
  return (f + 3) & ~(size_t)3;
}

static cudaError_t attend_any_rep(const ott_cache_t& c, const uint16_t* q, uint16_t* out, int n_rep, int64_t q_tokens,
                                  int64_t total, float* ws, int n_splits, cudaStream_t st,
                                  int64_t* dev_counts = nullptr, const uint16_t* new_k = nullptr,
                                  const uint16_t* new_v = nullptr) {
  const int nr = native_rep(n_rep);
  if (nr == n_rep)
    return ott::launch_attend(c, q, out, n_rep, q_tokens, total, ws, n_splits, st, dev_counts, new_k, new_v);
  uint16_t* qs = reinterpret_cast<uint16_t*>(ws + partial_floats(&c, nr, n_splits));
  uint16_t* os = qs + (size_t)c.n_units * nr * c.head_dim;
  ott_cache_t cp = c;
  cp.n_out_peers = 0;  // the real heads' rows go to the peers from the unpad kernel
  cudaError_t e = cudaSuccess;
  for (int h0 = 0; h0 < n_rep && e == cudaSuccess; h0 += 8) {
    const int nh = n_rep - h0 < 8 ? n_rep - h0 : 8;
    const bool last = h0 + 8 >= n_rep;
    e = ott::launch_rep_pad(q, qs, c.n_units, n_rep, h0, nh, nr, c.head_dim, st);
    if (e == cudaSuccess)
      e = ott::launch_attend(cp, qs, os, nr, q_tokens, total, ws, n_splits, st, dev_counts, new_k, new_v, last);
    if (e == cudaSuccess) e = ott::launch_rep_unpad(c, os, out, n_rep, h0, nh, nr, st);
  }
  return e;
}

static thread_local char g_err[512];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof(g_err), "%s", msg);
  return code;
}

static int cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return OTT_OK;
  snprintf(g_err, sizeof(g_err), "CUDA error: %s", cudaGetErrorString(e));
  return OTT_ERR_CUDA;
}

static int check_cache(const ott_cache_t* c) {
  if (!c) return fail(OTT_ERR_CONTRACT, "null cache");
  if (c->bits < 1 || c->bits > 8) return fail(OTT_ERR_CONTRACT, "bits must be in [1, 8]");
  // any shape in range runs; d = 128 / 2-bit / G % 32 == 0 takes the tensor-core kernels,
  // d in {64, 128} with G % 32 == 0 the CUDA-core tile kernel, the rest the generic kernel
  if (c->head_dim < 1 || c->head_dim > ott::kMaxD) return fail(OTT_ERR_UNSUPPORTED, "head_dim must be in [1, 256]");
  if (c->group_size < 1 || c->group_size > ott::kMaxG)
    return fail(OTT_ERR_UNSUPPORTED, "group_size must be in [1, 128]");
  if (c->residual < 0 || c->capacity < 0 || c->aux_capacity < 0)
    return fail(OTT_ERR_CONTRACT, "residual, outlier_num, aux_capacity must be >= 0");
  if (c->capacity > ott::kMaxN) return fail(OTT_ERR_UNSUPPORTED, "outlier_num must be <= 128");
  if (c->aux_capacity > ott::kMaxA) return fail(OTT_ERR_UNSUPPORTED, "aux_capacity must be <= 1024");
  if (c->n_units < 1 || c->max_groups < 0) return fail(OTT_ERR_CONTRACT, "bad unit/group counts");
  if (!c->blocks || !c->pend_k || !c->pend_v || !c->pool_mask || !c->subst_mask || !c->pool_meta)
    return fail(OTT_ERR_CONTRACT, "null state buffer");
  if (c->n_out_peers < 0 || c->n_out_peers > OTT_MAX_OUT_PEERS)
    return fail(OTT_ERR_CONTRACT, "n_out_peers must be in [0, OTT_MAX_OUT_PEERS]");
  for (int i = 0; i < c->n_out_peers; ++i)
    if (!c->out_peer[i]) return fail(OTT_ERR_CONTRACT, "null out_peer pointer");
  return OTT_OK;
}

extern "C" {

size_t ott_cache_struct_bytes(void) { return sizeof(ott_cache_t); }

size_t ott_record_bytes(int32_t head_dim, int32_t group_size, int32_t bits) {
  if (bits < 1 || bits > 8) return 0;
  return (size_t)ott::RecordLayout(head_dim, group_size, bits).bytes();
}

int ott_ring_write(const ott_cache_t* c, const uint16_t* k, const uint16_t* v, int64_t in_unit_stride,
                   int64_t in_first_pos, int64_t first_pos, int64_t n_rows, void* stream) {
  int s = check_cache(c);
  if (s) return s;
  if (n_rows < 0 || first_pos < in_first_pos) return fail(OTT_ERR_CONTRACT, "bad row range");
  if (n_rows == 0) return OTT_OK;
  if (n_rows > c->group_size + c->residual) return fail(OTT_ERR_CONTRACT, "more rows than the pending ring holds");
  if (!k || !v) return fail(OTT_ERR_CONTRACT, "null rows");
  return cuda_status(ott::launch_ring_write(*c, k, v, in_unit_stride, in_first_pos, first_pos, n_rows,
                                            (cudaStream_t)stream));
}

int ott_flush(const ott_cache_t* c, int64_t quantized_tokens, int32_t n_groups, int64_t ring_end,
              const uint16_t* in_k, const uint16_t* in_v, int64_t in_unit_stride, int64_t in_first_pos,
              void* stream) {
  int s = check_cache(c);
  if (s) return s;
  if (n_groups <= 0) return n_groups == 0 ? OTT_OK : fail(OTT_ERR_CONTRACT, "negative group count");
  if (quantized_tokens % c->group_size) return fail(OTT_ERR_CONTRACT, "quantized_tokens not group aligned");
  if (quantized_tokens / c->group_size + n_groups > c->max_groups)
    return fail(OTT_ERR_CONTRACT, "cache capacity (max_tokens) exceeded");
  if (quantized_tokens + (int64_t)n_groups * c->group_size > ring_end && (!in_k || !in_v))
    return fail(OTT_ERR_CONTRACT, "rows beyond the ring need an input buffer");
  if (quantized_tokens + (int64_t)n_groups * c->group_size > 0x7fffffffLL)
    return fail(OTT_ERR_UNSUPPORTED, "positions must fit in int32");
  if (c->capacity > 0 && (!c->pool_pos || !c->pool_score || !c->pool_k || !c->pool_v))
    return fail(OTT_ERR_CONTRACT, "null pool buffers");
  if (c->capacity > 0 && c->aux_capacity > 0 && (!c->aux_pos || !c->aux_score || !c->aux_k || !c->aux_v))
    return fail(OTT_ERR_CONTRACT, "null aux buffers");
  return cuda_status(ott::launch_flush(*c, quantized_tokens, n_groups, ring_end, in_k, in_v, in_unit_stride,
                                       in_first_pos, (cudaStream_t)stream));
}

int ott_num_sms(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  return n;
}

// n_splits = number of splits of the quantized region; the kernels add one more
// partial per (unit, head) for the full-precision tiers (pool + pending).
int ott_pick_splits(const ott_cache_t* c, int32_t n_rep, int64_t total_tokens) {
  (void)n_rep;
  if (!c || c->n_units < 1) return 1;
  const int64_t q_tokens = total_tokens >= c->residual + c->group_size
                               ? ((total_tokens - c->residual) / c->group_size) * c->group_size
                               : 0;
  const int64_t n_groups = q_tokens / c->group_size;
  int sms = ott_num_sms();
  if (sms <= 0) sms = 148;
  // ~3 quantized-range CTAs per SM over the launch (round to nearest): long CTAs
  // amortise their start-up (first TMA round trip, q staging, merge) and the fp-tier
  // CTAs fill the tail. Measured (v7 sweep over config-3/4 shapes): best or within 3 %
  // of the best split count on B=16/64/128 x T=4K-16K; the previous 8/SM rule was up to
  // 29 % slower on small batches. Each split still streams >= 16 groups (4 per warp).
  const int64_t target = (int64_t)sms * 3;
  int64_t s = (target + c->n_units / 2) / c->n_units;
  const int64_t max_by_groups = n_groups / 16 > 0 ? n_groups / 16 : 1;
  // long contexts (>= 256 groups per unit) on 256-592 units: aim at ~1,024 quantized CTAs with
  // pieces of >= 96 groups. The config-4 shards of 2 and 4 GPUs (512 / 256 units at 16K
  // tokens): 224.7 -> 208.3 us (2 pieces) and 122.5 -> 116.1 us (4 pieces); 128 units keep 3
  // (4-8 pieces: 70.5-76.5 vs 69.8 us) and shorter contexts the rule above
  // (profiles/r2_shard_splits.log)
  if (n_groups >= 256 && c->n_units >= 256 && c->n_units <= (int64_t)sms * 4) {
    const int64_t s_long = std::min<int64_t>((1024 + c->n_units / 2) / c->n_units, n_groups / 96);
    if (s_long > s) s = s_long;
  }
  if (s > max_by_groups) s = max_by_groups;
  if (s > 64) s = 64;
  if (s < 1) s = 1;
  // more units than resident CTAs on the 2-bit tensor-core kernel: the launch's tail schedule
  // (AttnArgs.tail_units): one wave of whole units, the other units in thirds, then the fp-tier
  // CTAs. Config 4 (1,024 units): 390.8 us vs 396.6 for whole units only (halves 395.4,
  // quarters 395.0: the pieces' start-up costs eat the better balance)
  if (s == 1 && ott::mma_eligible(*c) && c->n_units > (int64_t)sms * 4 && n_groups >= 48) s = 3;
  return (int)s;
}

size_t ott_attend_workspace_floats(const ott_cache_t* c, int32_t n_rep, int32_t n_splits) {
  const int nr = native_rep(n_rep);
  if (!c || !nr) return 0;
  size_t f = partial_floats(c, nr, n_splits);
  if (nr != n_rep) f += (size_t)c->n_units * nr * c->head_dim;  // padded q and out staging (fp16)
  return f;
}

int ott_attend(const ott_cache_t* c, const uint16_t* q, uint16_t* out, int32_t n_rep, int64_t quantized_tokens,
               int64_t total_tokens, float* workspace, int32_t n_splits, void* stream) {
  int s = check_cache(c);
  if (s) return s;
  if (total_tokens <= 0) return fail(OTT_ERR_CONTRACT, "cannot attend over an empty cache");
  if (!native_rep(n_rep)) return fail(OTT_ERR_UNSUPPORTED, "n_rep (H_q / H_kv) must be in [1, 128]");
  if (quantized_tokens < 0 || quantized_tokens > total_tokens || quantized_tokens % c->group_size)
    return fail(OTT_ERR_CONTRACT, "inconsistent token counts");
  if (total_tokens - quantized_tokens > c->group_size + c->residual)
    return fail(OTT_ERR_CONTRACT, "more pending rows than the ring holds");
  if (!q || !out || !workspace || n_splits < 1) return fail(OTT_ERR_CONTRACT, "null buffer or bad split count");
  return cuda_status(attend_any_rep(*c, q, out, n_rep, quantized_tokens, total_tokens, workspace, n_splits,
                                    (cudaStream_t)stream));
}

int ott_append_attend(const ott_cache_t* c, const uint16_t* k, const uint16_t* v, const uint16_t* q, uint16_t* out,
                      int32_t n_rep, int64_t quantized_tokens, int64_t total_tokens, float* workspace,
                      int32_t n_splits, void* stream) {
  int s = check_cache(c);
  if (s) return s;
  if (!k || !v) return fail(OTT_ERR_CONTRACT, "null rows");
  if (total_tokens <= 0) return fail(OTT_ERR_CONTRACT, "cannot attend over an empty cache");
  if (!native_rep(n_rep)) return fail(OTT_ERR_UNSUPPORTED, "n_rep (H_q / H_kv) must be in [1, 128]");
  if (quantized_tokens < 0 || quantized_tokens > total_tokens - 1 || quantized_tokens % c->group_size)
    return fail(OTT_ERR_CONTRACT, "inconsistent token counts");
  if (total_tokens - quantized_tokens > c->group_size + c->residual)
    return fail(OTT_ERR_CONTRACT, "more pending rows than the ring holds");
  if (!q || !out || !workspace || n_splits < 1) return fail(OTT_ERR_CONTRACT, "null buffer or bad split count");
  cudaStream_t st = (cudaStream_t)stream;
  const bool fuse = ott::attend_fuses_ring_write(*c);
  cudaError_t e = fuse ? cudaSuccess
                       : ott::launch_ring_write(*c, k, v, c->head_dim, total_tokens - 1, total_tokens - 1, 1, st);
  if (e == cudaSuccess)
    e = attend_any_rep(*c, q, out, n_rep, quantized_tokens, total_tokens, workspace, n_splits, st, nullptr,
                       fuse ? k : nullptr, fuse ? v : nullptr);
  return cuda_status(e);
}

int ott_decode_step(const ott_cache_t* c, const uint16_t* k, const uint16_t* v, const uint16_t* q, uint16_t* out,
                    int32_t n_rep, int64_t* counters, float* workspace, int32_t n_splits, void* stream) {
  int s = check_cache(c);
  if (s) return s;
  if (!native_rep(n_rep)) return fail(OTT_ERR_UNSUPPORTED, "n_rep (H_q / H_kv) must be in [1, 128]");
  if (!k || !v || !q || !out || !counters || !workspace || n_splits < 1)
    return fail(OTT_ERR_CONTRACT, "null buffer or bad split count");
  if (c->capacity > 0 && (!c->pool_pos || !c->pool_score || !c->pool_k || !c->pool_v))
    return fail(OTT_ERR_CONTRACT, "null pool buffers");
  cudaStream_t st = (cudaStream_t)stream;
  const bool fuse = ott::attend_fuses_ring_write(*c);  // the new row is written by the attention kernel
  cudaError_t e = fuse ? cudaSuccess : ott::launch_ring_write(*c, k, v, c->head_dim, 0, 0, 1, st, counters);
  if (e == cudaSuccess) e = ott::launch_flush(*c, 0, 1, 0, nullptr, nullptr, 0, 0, st, counters);
  if (e == cudaSuccess)
    e = attend_any_rep(*c, q, out, n_rep, 0, 1, workspace, n_splits, st, counters, fuse ? k : nullptr,
                       fuse ? v : nullptr);
  return cuda_status(e);
}

int ott_logits(const ott_cache_t* c, const uint16_t* q, float* logits, int32_t n_rep, int64_t quantized_tokens,
               int64_t total_tokens, void* stream) {
  int s = check_cache(c);
  if (s) return s;
  if (total_tokens <= 0) return fail(OTT_ERR_CONTRACT, "cannot attend over an empty cache");
  if (!q || !logits) return fail(OTT_ERR_CONTRACT, "null buffer");
  return cuda_status(
      ott::launch_logits(*c, q, logits, n_rep, quantized_tokens, total_tokens, (cudaStream_t)stream));
}

int ott_attend_exact(const float* q, const float* keys, const float* values, int32_t n, int32_t d, int32_t n_q,
                     float* out, float* weights, float* scores, void* stream) {
  if (n < 1) return fail(OTT_ERR_CONTRACT, "attention needs at least one cached token");  // attention.py:48-49
  if (d < 1 || n_q < 1) return fail(OTT_ERR_CONTRACT, "bad shape");
  if (!q || !keys || !values || !out || !weights || !scores) return fail(OTT_ERR_CONTRACT, "null buffer");
  return cuda_status(ott::launch_attend_exact(q, keys, values, n, d, n_q, out, weights, scores, (cudaStream_t)stream));
}

int ott_pool_rank(const double* scores, const int64_t* positions, int32_t n, int32_t* rank, void* stream) {
  if (n < 0) return fail(OTT_ERR_CONTRACT, "bad item count");
  if (n == 0) return OTT_OK;
  if (!scores || !positions || !rank) return fail(OTT_ERR_CONTRACT, "null buffer");
  return cuda_status(ott::launch_pool_rank(scores, positions, n, rank, (cudaStream_t)stream));
}

int ott_score_rows(const float* rows, int32_t n, int32_t d, double* scores, void* stream) {
  if (n < 1 || d < 1) return fail(OTT_ERR_CONTRACT, "score_tokens expects a non-empty 2-D key matrix");
  if (!rows || !scores) return fail(OTT_ERR_CONTRACT, "null buffer");
  return cuda_status(ott::launch_score_rows(rows, n, d, scores, (cudaStream_t)stream));
}

const char* ott_version(void) { return "ott_b200 0.2 (sm_100a)"; }
const char* ott_last_error(void) { return g_err; }

}  // extern "C"
