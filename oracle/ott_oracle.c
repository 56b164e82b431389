/*
 * ott_oracle.c — TEST INFRASTRUCTURE ONLY. CPU restatement of the reference
 * kvtrace OTT path (quantizer, pool competition, mean substitution, tiered
 * cache, mixed attention). See ott_oracle.h. The product (the CUDA path in
 * paper_2505_10938_b200/) never links or calls this file.
 *
 * Build: gcc -O2 -fPIC -shared -fopenmp -ffp-contract=off (oracle/Makefile).
 * -ffp-contract=off matters: the reference's float64 recipe has no fused
 * multiply-adds (numpy evaluates `codes * step + x_min` as two roundings).
 */
#include "ott_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ quant */

/* quant.py:59-70 _line_params: min/max, step = (max-min)/levels, then nudge
 * step down with nextafter until x_min + levels*step <= x_max. */
static void line_params(const double* x, int n, int bits, double* x_min_out, double* step_out) {
  double mn = x[0], mx = x[0];
  for (int i = 1; i < n; ++i) {
    if (x[i] < mn) mn = x[i];
    if (x[i] > mx) mx = x[i];
  }
  const double levels = (double)((1 << bits) - 1);
  double step = (mx - mn) / levels;
  while (step > 0.0 && mn + levels * step > mx) step = nextafter(step, 0.0);
  *x_min_out = mn;
  *step_out = step;
}

/* quant.py:73-102 quantize_uniform */
int ottref_quantize_line(const double* x, int n, int bits, int64_t* codes, double* x_min, double* step) {
  if (bits < 1 || bits > 8 || n < 1) return -1;
  for (int i = 0; i < n; ++i)
    if (!isfinite(x[i])) return -1;
  double mn, st;
  line_params(x, n, bits, &mn, &st);
  *x_min = mn;
  *step = st;
  const int64_t levels = (1 << bits) - 1;
  if (st == 0.0) { /* quant.py:91-92 */
    for (int i = 0; i < n; ++i) codes[i] = 0;
    return 0;
  }
  double mx = x[0];
  for (int i = 1; i < n; ++i)
    if (x[i] > mx) mx = x[i];
  for (int i = 0; i < n; ++i) {
    double f = floor((x[i] - mn) / st); /* quant.py:93 */
    int64_t c;
    if (f < 0.0) c = 0;                 /* quant.py:94 clip */
    else if (f > (double)levels) c = levels;
    else c = (int64_t)f;
    volatile double recon = (double)c * st; /* quant.py:97: codes*step + x_min, two roundings */
    recon = recon + mn;
    if (recon > x[i]) c -= 1;
    if (c < 0) c = 0; /* quant.py:98 */
    if (c > levels) c = levels;
    if (x[i] == mx) c = levels; /* quant.py:101 */
    codes[i] = c;
  }
  return 0;
}

/* quant.py:237-238 */
static long packed_size(size_t count, int bits) { return (long)((count * (size_t)bits + 7) / 8); }

/* quant.py:241-256: bit i of the stream lands in bit (i % 8) of byte (i / 8);
 * element e occupies stream bits [e*bits, e*bits + bits), LSB first. */
long ottref_pack_codes(const int64_t* codes, size_t count, int bits, uint8_t* out) {
  long nbytes = packed_size(count, bits);
  memset(out, 0, (size_t)nbytes);
  for (size_t e = 0; e < count; ++e) {
    if (codes[e] < 0 || codes[e] >= (1 << bits)) return -1;
    for (int b = 0; b < bits; ++b) {
      size_t i = e * (size_t)bits + (size_t)b;
      if ((codes[e] >> b) & 1) out[i >> 3] |= (uint8_t)(1u << (i & 7));
    }
  }
  return nbytes;
}

/* quant.py:259-273 */
void ottref_unpack_codes(const uint8_t* data, size_t count, int bits, int64_t* out) {
  if (bits == 2) { /* fast path: 4 codes per byte, code 4j+i in bits [2i, 2i+2) of byte j */
    for (size_t e = 0; e < count; ++e) out[e] = (data[e >> 2] >> (2 * (e & 3))) & 3;
    return;
  }
  for (size_t e = 0; e < count; ++e) {
    int64_t v = 0;
    for (int b = 0; b < bits; ++b) {
      size_t i = e * (size_t)bits + (size_t)b;
      v |= (int64_t)((data[i >> 3] >> (i & 7)) & 1) << b;
    }
    out[e] = v;
  }
}

/* quant.py:201-234 _quantize_group */
int ottref_quantize_group(const float* group, int n_tokens, int n_channels, int bits, int axis, uint8_t* codes_out,
                          double* x_min, double* step) {
  if (n_tokens < 1 || n_channels < 1) return -1;
  const int n_lines = axis == 0 ? n_channels : n_tokens;
  const int line_len = axis == 0 ? n_tokens : n_channels;
  double* line = (double*)malloc(sizeof(double) * (size_t)line_len);
  int64_t* lc = (int64_t*)malloc(sizeof(int64_t) * (size_t)line_len);
  int64_t* codes = (int64_t*)malloc(sizeof(int64_t) * (size_t)n_tokens * (size_t)n_channels);
  int rc = 0;
  for (int l = 0; l < n_lines && rc == 0; ++l) {
    for (int j = 0; j < line_len; ++j)
      line[j] = axis == 0 ? (double)group[(size_t)j * n_channels + l] : (double)group[(size_t)l * n_channels + j];
    rc = ottref_quantize_line(line, line_len, bits, lc, &x_min[l], &step[l]);
    /* quant.py:215-216: PER_CHANNEL codes transposed back to token-major */
    for (int j = 0; j < line_len; ++j) {
      if (axis == 0) codes[(size_t)j * n_channels + l] = lc[j];
      else codes[(size_t)l * n_channels + j] = lc[j];
    }
  }
  if (rc == 0 && ottref_pack_codes(codes, (size_t)n_tokens * n_channels, bits, codes_out) < 0) rc = -1;
  free(line);
  free(lc);
  free(codes);
  return rc;
}

/* ---------------------------------------------------------------- outlier */

typedef struct {
  int64_t position;
  double score;
  float* key;   /* head_dim floats, owned */
  float* value; /* head_dim floats, owned */
} entry_t;

/* outlier.py:52-54 _rank: (score, position) ascending */
static int rank_less(const entry_t* a, const entry_t* b) {
  if (a->score != b->score) return a->score < b->score;
  return a->position < b->position;
}

/* tensor.py:38-42 row_l1_norm: sum |k| in float64 (exact for fp16-valued rows) */
static double row_l1(const float* row, int d) {
  double s = 0.0;
  for (int c = 0; c < d; ++c) s += fabs((double)row[c]);
  return s;
}

struct ottref_cache {
  int bits, G, R, N, A, d;
  int64_t total_tokens, quantized_tokens;
  /* pending buffer, cache.py:106-109 (rows shifted down on flush, 183-186) */
  float *pend_k, *pend_v;
  int pend_count;
  /* quantized blocks */
  int n_blocks, cap_blocks, block_bytes;
  uint8_t *kcodes, *vcodes;
  double *k_xmin, *k_step, *v_xmin, *v_step;
  /* OutlierPool, outlier.py:57-82 */
  entry_t* entries;
  int n_entries;
  entry_t* aux;
  int n_aux;
  int frozen;
  /* substituted_positions, cache.py:103 */
  int64_t* subst;
  int n_subst, cap_subst;
};

static float* fdup(const float* src, int d) {
  float* p = (float*)malloc(sizeof(float) * (size_t)d);
  memcpy(p, src, sizeof(float) * (size_t)d);
  return p;
}

/* cache.py:93-109 + outlier.py:74-78 (__post_init__: aux_capacity 0 freezes) */
ottref_cache* ottref_cache_new(int bits, int group_size, int residual, int capacity, int aux_capacity, int head_dim) {
  if (bits < 1 || bits > 8 || group_size < 1 || residual < 0 || capacity < 0 || aux_capacity < 0 || head_dim < 1)
    return NULL;
  ottref_cache* c = (ottref_cache*)calloc(1, sizeof(ottref_cache));
  c->bits = bits;
  c->G = group_size;
  c->R = residual;
  c->N = capacity;
  c->A = aux_capacity;
  c->d = head_dim;
  const int cap = group_size + residual;
  c->pend_k = (float*)calloc((size_t)cap * head_dim, sizeof(float));
  c->pend_v = (float*)calloc((size_t)cap * head_dim, sizeof(float));
  c->block_bytes = (int)packed_size((size_t)group_size * head_dim, bits);
  c->entries = (entry_t*)calloc((size_t)(capacity > 0 ? capacity : 1), sizeof(entry_t));
  c->aux = (entry_t*)calloc((size_t)(aux_capacity > 0 ? aux_capacity : 1), sizeof(entry_t));
  c->frozen = aux_capacity <= 0 ? 1 : 0;
  return c;
}

static void free_entry(entry_t* e) {
  free(e->key);
  free(e->value);
}

void ottref_cache_free(ottref_cache* c) {
  if (!c) return;
  free(c->pend_k);
  free(c->pend_v);
  free(c->kcodes);
  free(c->vcodes);
  free(c->k_xmin);
  free(c->k_step);
  free(c->v_xmin);
  free(c->v_step);
  for (int i = 0; i < c->n_entries; ++i) free_entry(&c->entries[i]);
  for (int i = 0; i < c->n_aux; ++i) free_entry(&c->aux[i]);
  free(c->entries);
  free(c->aux);
  free(c->subst);
  free(c);
}

static void* memdup(const void* p, size_t n) {
  if (!p || n == 0) return NULL;
  void* q = malloc(n);
  memcpy(q, p, n);
  return q;
}

ottref_cache* ottref_cache_clone(const ottref_cache* c) {
  ottref_cache* n = (ottref_cache*)malloc(sizeof(ottref_cache));
  *n = *c;
  const size_t cap = (size_t)(c->G + c->R) * c->d;
  n->pend_k = (float*)memdup(c->pend_k, cap * sizeof(float));
  n->pend_v = (float*)memdup(c->pend_v, cap * sizeof(float));
  n->kcodes = (uint8_t*)memdup(c->kcodes, (size_t)c->cap_blocks * c->block_bytes);
  n->vcodes = (uint8_t*)memdup(c->vcodes, (size_t)c->cap_blocks * c->block_bytes);
  n->k_xmin = (double*)memdup(c->k_xmin, (size_t)c->cap_blocks * c->d * sizeof(double));
  n->k_step = (double*)memdup(c->k_step, (size_t)c->cap_blocks * c->d * sizeof(double));
  n->v_xmin = (double*)memdup(c->v_xmin, (size_t)c->cap_blocks * c->G * sizeof(double));
  n->v_step = (double*)memdup(c->v_step, (size_t)c->cap_blocks * c->G * sizeof(double));
  n->entries = (entry_t*)calloc((size_t)(c->N > 0 ? c->N : 1), sizeof(entry_t));
  n->aux = (entry_t*)calloc((size_t)(c->A > 0 ? c->A : 1), sizeof(entry_t));
  for (int i = 0; i < c->n_entries; ++i) {
    n->entries[i] = c->entries[i];
    n->entries[i].key = fdup(c->entries[i].key, c->d);
    n->entries[i].value = fdup(c->entries[i].value, c->d);
  }
  for (int i = 0; i < c->n_aux; ++i) {
    n->aux[i] = c->aux[i];
    n->aux[i].key = fdup(c->aux[i].key, c->d);
    n->aux[i].value = fdup(c->aux[i].value, c->d);
  }
  n->subst = (int64_t*)memdup(c->subst, (size_t)c->cap_subst * sizeof(int64_t));
  return n;
}

/* cache.py:124-139 append */
int ottref_append(ottref_cache* c, const float* k_row, const float* v_row) {
  for (int i = 0; i < c->d; ++i)
    if (!isfinite(k_row[i]) || !isfinite(v_row[i])) return -1; /* cache.py:131-132 */
  memcpy(c->pend_k + (size_t)c->pend_count * c->d, k_row, sizeof(float) * (size_t)c->d);
  memcpy(c->pend_v + (size_t)c->pend_count * c->d, v_row, sizeof(float) * (size_t)c->d);
  c->pend_count += 1;
  c->total_tokens += 1;
  if (c->pend_count - c->R >= c->G) return ottref_quantize_oldest_group(c); /* cache.py:138 */
  return 0;
}

static void ensure_blocks(ottref_cache* c) {
  if (c->n_blocks < c->cap_blocks) return;
  int nc = c->cap_blocks ? c->cap_blocks * 2 : 16;
  c->kcodes = (uint8_t*)realloc(c->kcodes, (size_t)nc * c->block_bytes);
  c->vcodes = (uint8_t*)realloc(c->vcodes, (size_t)nc * c->block_bytes);
  c->k_xmin = (double*)realloc(c->k_xmin, (size_t)nc * c->d * sizeof(double));
  c->k_step = (double*)realloc(c->k_step, (size_t)nc * c->d * sizeof(double));
  c->v_xmin = (double*)realloc(c->v_xmin, (size_t)nc * c->G * sizeof(double));
  c->v_step = (double*)realloc(c->v_step, (size_t)nc * c->G * sizeof(double));
  c->cap_blocks = nc;
}

static void add_subst(ottref_cache* c, int64_t p) {
  if (c->n_subst == c->cap_subst) {
    c->cap_subst = c->cap_subst ? c->cap_subst * 2 : 64;
    c->subst = (int64_t*)realloc(c->subst, (size_t)c->cap_subst * sizeof(int64_t));
  }
  c->subst[c->n_subst++] = p;
}

/* outlier.py:84-117 OutlierPool.update over the group's G candidates.
 * Writes in_group[i] = 1 for candidates that won a slot ("selected"). */
static void pool_update(ottref_cache* c, const float* gk, const float* gv, int64_t base, const double* scores,
                        unsigned char* in_group) {
  const int G = c->G, d = c->d;
  memset(in_group, 0, (size_t)G);
  if (c->frozen || c->N == 0) return; /* outlier.py:93-94 */
  const int total = c->n_entries + G;
  entry_t* all = (entry_t*)malloc(sizeof(entry_t) * (size_t)total);
  int* is_cand = (int*)malloc(sizeof(int) * (size_t)total);
  for (int i = 0; i < c->n_entries; ++i) {
    all[i] = c->entries[i];
    is_cand[i] = -1;
  }
  for (int i = 0; i < G; ++i) {
    entry_t* e = &all[c->n_entries + i];
    e->position = base + i;
    e->score = scores[i];
    e->key = NULL;
    e->value = NULL;
    is_cand[c->n_entries + i] = i;
  }
  /* outlier.py:102: sorted(entries + candidates, key=_rank) — insertion sort
   * carrying the candidate tag (keys are unique, so any correct sort agrees) */
  for (int i = 1; i < total; ++i) {
    entry_t e = all[i];
    int t = is_cand[i], j = i - 1;
    while (j >= 0 && rank_less(&e, &all[j])) {
      all[j + 1] = all[j];
      is_cand[j + 1] = is_cand[j];
      --j;
    }
    all[j + 1] = e;
    is_cand[j + 1] = t;
  }
  const int n_win = total < c->N ? total : c->N;
  /* evicted = old entries (in old order) not among winners, outlier.py:110 */
  entry_t* old = (entry_t*)malloc(sizeof(entry_t) * (size_t)(c->n_entries > 0 ? c->n_entries : 1));
  const int n_old = c->n_entries;
  memcpy(old, c->entries, sizeof(entry_t) * (size_t)n_old);
  entry_t* new_entries = (entry_t*)calloc((size_t)(c->N > 0 ? c->N : 1), sizeof(entry_t));
  for (int w = 0; w < n_win; ++w) {
    new_entries[w] = all[w];
    if (is_cand[w] >= 0) {
      const int i = is_cand[w];
      in_group[i] = 1; /* selected, outlier.py:107-109 */
      new_entries[w].key = fdup(gk + (size_t)i * d, d);
      new_entries[w].value = fdup(gv + (size_t)i * d, d);
    }
  }
  int room = c->A - c->n_aux; /* outlier.py:113-114 */
  for (int o = 0; o < n_old; ++o) {
    int won = 0;
    for (int w = 0; w < n_win; ++w)
      if (new_entries[w].position == old[o].position) won = 1;
    if (won) continue;
    if (room > 0) {
      c->aux[c->n_aux++] = old[o];
      --room;
    } else {
      free_entry(&old[o]); /* evicted beyond aux capacity: dropped (still "returned") */
    }
  }
  memcpy(c->entries, new_entries, sizeof(entry_t) * (size_t)n_win);
  c->n_entries = n_win;
  if (c->n_aux >= c->A) c->frozen = 1; /* outlier.py:115-116 */
  free(new_entries);
  free(old);
  free(all);
  free(is_cand);
}

/* cache.py:141-186 quantize_oldest_group */
int ottref_quantize_oldest_group(ottref_cache* c) {
  const int G = c->G, d = c->d;
  if (c->pend_count < G) return -1; /* cache.py:150-153 */
  const int64_t base = c->quantized_tokens;
  float* gk = fdup(c->pend_k, G * d);
  float* gv = fdup(c->pend_v, G * d);
  if (c->N > 0 && !c->frozen) { /* cache.py:158 */
    double* scores = (double*)malloc(sizeof(double) * (size_t)G);
    unsigned char* sel = (unsigned char*)malloc((size_t)G);
    for (int i = 0; i < G; ++i) scores[i] = row_l1(gk + (size_t)i * d, d); /* outlier.py:45-49 */
    pool_update(c, gk, gv, base, scores, sel);
    int any = 0;
    for (int i = 0; i < G; ++i) any |= sel[i];
    if (any) {
      /* outlier.py:120-142 substitute_means: per-channel mean over ALL G rows
       * before substitution, float64 accumulate, cast to float32 */
      float* km = (float*)malloc(sizeof(float) * (size_t)d);
      float* vm = (float*)malloc(sizeof(float) * (size_t)d);
      for (int ch = 0; ch < d; ++ch) {
        double sk = 0.0, sv = 0.0;
        for (int i = 0; i < G; ++i) {
          sk += (double)gk[(size_t)i * d + ch];
          sv += (double)gv[(size_t)i * d + ch];
        }
        km[ch] = (float)(sk / (double)G);
        vm[ch] = (float)(sv / (double)G);
      }
      for (int i = 0; i < G; ++i) {
        if (!sel[i]) continue;
        memcpy(gk + (size_t)i * d, km, sizeof(float) * (size_t)d);
        memcpy(gv + (size_t)i * d, vm, sizeof(float) * (size_t)d);
        add_subst(c, base + i); /* cache.py:173 */
      }
      free(km);
      free(vm);
    }
    free(scores);
    free(sel);
  }
  ensure_blocks(c);
  const int b = c->n_blocks;
  int rc = ottref_quantize_group(gk, G, d, c->bits, 0, c->kcodes + (size_t)b * c->block_bytes,
                                 c->k_xmin + (size_t)b * d, c->k_step + (size_t)b * d);
  if (rc == 0)
    rc = ottref_quantize_group(gv, G, d, c->bits, 1, c->vcodes + (size_t)b * c->block_bytes,
                               c->v_xmin + (size_t)b * G, c->v_step + (size_t)b * G);
  free(gk);
  free(gv);
  if (rc) return rc;
  c->n_blocks += 1;
  c->quantized_tokens += G;
  const int remaining = c->pend_count - G; /* cache.py:183-186 */
  memmove(c->pend_k, c->pend_k + (size_t)G * d, sizeof(float) * (size_t)remaining * d);
  memmove(c->pend_v, c->pend_v + (size_t)G * d, sizeof(float) * (size_t)remaining * d);
  c->pend_count = remaining;
  return 0;
}

/* -------------------------------------------------------------- attention */

/* quant.py:154-163 to_matrix + attention.py:65-76 reconstructed_kv */
void ottref_reconstructed_kv(const ottref_cache* c, float* keys, float* values) {
  const int G = c->G, d = c->d;
  int64_t* codes = (int64_t*)malloc(sizeof(int64_t) * (size_t)G * d);
  for (int b = 0; b < c->n_blocks; ++b) {
    float* kb = keys + (size_t)b * G * d;
    float* vb = values + (size_t)b * G * d;
    ottref_unpack_codes(c->kcodes + (size_t)b * c->block_bytes, (size_t)G * d, c->bits, codes);
    for (int t = 0; t < G; ++t)
      for (int ch = 0; ch < d; ++ch) {
        volatile double r = (double)codes[(size_t)t * d + ch] * c->k_step[(size_t)b * d + ch];
        kb[(size_t)t * d + ch] = (float)(r + c->k_xmin[(size_t)b * d + ch]);
      }
    ottref_unpack_codes(c->vcodes + (size_t)b * c->block_bytes, (size_t)G * d, c->bits, codes);
    for (int t = 0; t < G; ++t)
      for (int ch = 0; ch < d; ++ch) {
        volatile double r = (double)codes[(size_t)t * d + ch] * c->v_step[(size_t)b * G + t];
        vb[(size_t)t * d + ch] = (float)(r + c->v_xmin[(size_t)b * G + t]);
      }
  }
  const size_t off = (size_t)c->quantized_tokens * d;
  memcpy(keys + off, c->pend_k, sizeof(float) * (size_t)c->pend_count * d);
  memcpy(values + off, c->pend_v, sizeof(float) * (size_t)c->pend_count * d);
  for (int i = 0; i < c->n_entries; ++i) { /* attention.py:73-75: pool entries only, not aux */
    memcpy(keys + (size_t)c->entries[i].position * d, c->entries[i].key, sizeof(float) * (size_t)d);
    memcpy(values + (size_t)c->entries[i].position * d, c->entries[i].value, sizeof(float) * (size_t)d);
  }
  free(codes);
}

/* attention.py:79-92 attend_mixed -> attention.py:35-59 attend_full_precision
 * with tensor.py:45-57 softmax (max-subtracted, float64). */
int ottref_attend(const ottref_cache* c, const float* q, float* out, float* weights, float* scores) {
  const int64_t T = c->total_tokens;
  const int d = c->d;
  if (T == 0) return -1; /* attention.py:89-90 */
  float* K = (float*)malloc(sizeof(float) * (size_t)T * d);
  float* V = (float*)malloc(sizeof(float) * (size_t)T * d);
  double* s = (double*)malloc(sizeof(double) * (size_t)T);
  ottref_reconstructed_kv(c, K, V);
  const double inv = 1.0 / (double)(float)sqrt((double)d); /* np.float32(np.sqrt(d)) */
  double mx = -INFINITY;
  for (int64_t t = 0; t < T; ++t) {
    double acc = 0.0;
    for (int ch = 0; ch < d; ++ch) acc += (double)K[(size_t)t * d + ch] * (double)q[ch];
    s[t] = acc * inv;
    if (s[t] > mx) mx = s[t];
    if (scores) scores[t] = (float)s[t];
  }
  double z = 0.0;
  for (int64_t t = 0; t < T; ++t) {
    s[t] = exp(s[t] - mx);
    z += s[t];
  }
  double* o = (double*)calloc((size_t)d, sizeof(double));
  for (int64_t t = 0; t < T; ++t) {
    const double w = s[t] / z;
    if (weights) weights[t] = (float)w;
    for (int ch = 0; ch < d; ++ch) o[ch] += w * (double)V[(size_t)t * d + ch];
  }
  for (int ch = 0; ch < d; ++ch) out[ch] = (float)o[ch];
  free(o);
  free(K);
  free(V);
  free(s);
  return 0;
}

/* -------------------------------------------------------------- accessors */

int64_t ottref_total_tokens(const ottref_cache* c) { return c->total_tokens; }
int64_t ottref_quantized_tokens(const ottref_cache* c) { return c->quantized_tokens; }
int ottref_pending_rows(const ottref_cache* c) { return c->pend_count; }
int ottref_n_blocks(const ottref_cache* c) { return c->n_blocks; }
int ottref_block_bytes(const ottref_cache* c) { return c->block_bytes; }

void ottref_block(const ottref_cache* c, int b, uint8_t* kcodes, uint8_t* vcodes, double* k_xmin, double* k_step,
                  double* v_xmin, double* v_step) {
  if (kcodes) memcpy(kcodes, c->kcodes + (size_t)b * c->block_bytes, (size_t)c->block_bytes);
  if (vcodes) memcpy(vcodes, c->vcodes + (size_t)b * c->block_bytes, (size_t)c->block_bytes);
  if (k_xmin) memcpy(k_xmin, c->k_xmin + (size_t)b * c->d, sizeof(double) * (size_t)c->d);
  if (k_step) memcpy(k_step, c->k_step + (size_t)b * c->d, sizeof(double) * (size_t)c->d);
  if (v_xmin) memcpy(v_xmin, c->v_xmin + (size_t)b * c->G, sizeof(double) * (size_t)c->G);
  if (v_step) memcpy(v_step, c->v_step + (size_t)b * c->G, sizeof(double) * (size_t)c->G);
}

void ottref_pending(const ottref_cache* c, float* k, float* v) {
  memcpy(k, c->pend_k, sizeof(float) * (size_t)c->pend_count * c->d);
  memcpy(v, c->pend_v, sizeof(float) * (size_t)c->pend_count * c->d);
}

int ottref_pool_size(const ottref_cache* c) { return c->n_entries; }
int ottref_aux_size(const ottref_cache* c) { return c->n_aux; }
int ottref_frozen(const ottref_cache* c) { return c->frozen; }

static void dump_entries(const entry_t* e, int n, int d, int64_t* pos, double* score, float* keys, float* values) {
  for (int i = 0; i < n; ++i) {
    if (pos) pos[i] = e[i].position;
    if (score) score[i] = e[i].score;
    if (keys) memcpy(keys + (size_t)i * d, e[i].key, sizeof(float) * (size_t)d);
    if (values) memcpy(values + (size_t)i * d, e[i].value, sizeof(float) * (size_t)d);
  }
}

void ottref_pool_entries(const ottref_cache* c, int64_t* pos, double* score, float* keys, float* values) {
  dump_entries(c->entries, c->n_entries, c->d, pos, score, keys, values);
}
void ottref_aux_entries(const ottref_cache* c, int64_t* pos, double* score, float* keys, float* values) {
  dump_entries(c->aux, c->n_aux, c->d, pos, score, keys, values);
}

int ottref_n_substituted(const ottref_cache* c) { return c->n_subst; }
void ottref_substituted(const ottref_cache* c, int64_t* pos) {
  /* positions are appended in increasing order (groups advance, rows ascend) */
  memcpy(pos, c->subst, sizeof(int64_t) * (size_t)c->n_subst);
}

/* cache.py:188-203 */
void ottref_memory_usage(const ottref_cache* c, int64_t out[4]) {
  const int64_t per_block_codes = (int64_t)c->G * c->d * c->bits;
  out[0] = 2 * per_block_codes * c->n_blocks;                 /* K + V code_bits */
  out[1] = (int64_t)c->n_blocks * (c->d + c->G) * 2 * 16;     /* param_bits */
  out[2] = (int64_t)c->pend_count * c->d * 16 * 2;            /* pending_bits */
  out[3] = (int64_t)(c->n_entries + c->n_aux) * c->d * 16 * 2; /* pool_bits */
}

/* --------------------------------------------------------- batch drivers */

int ottref_decode_step(ottref_cache** caches, int n_units, const float* k, const float* v, const float* q, int n_rep,
                       float* out, int threads) {
  int err = 0;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads) reduction(| : err)
#endif
  for (int u = 0; u < n_units; ++u) {
    ottref_cache* c = caches[u];
    const int d = c->d;
    err |= ottref_append(c, k + (size_t)u * d, v + (size_t)u * d) != 0;
    for (int r = 0; r < n_rep; ++r)
      err |= ottref_attend(c, q + ((size_t)u * n_rep + r) * d, out + ((size_t)u * n_rep + r) * d, NULL, NULL) != 0;
  }
  (void)threads;
  return err ? -1 : 0;
}

int ottref_prefill(ottref_cache** caches, int n_units, const float* k, const float* v, int n_tokens, int threads) {
  int err = 0;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads) reduction(| : err)
#endif
  for (int u = 0; u < n_units; ++u) {
    ottref_cache* c = caches[u];
    const int d = c->d;
    for (int t = 0; t < n_tokens; ++t)
      err |= ottref_append(c, k + ((size_t)u * n_tokens + t) * d, v + ((size_t)u * n_tokens + t) * d) != 0;
  }
  (void)threads;
  return err ? -1 : 0;
}
