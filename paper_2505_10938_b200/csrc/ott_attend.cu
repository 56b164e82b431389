// ott_attend.cu — K2/K3: split-K flash-decoding attention over the three cache
// tiers (attend_mixed, attention.py:79-92) and the split combine.
//
// Per unit (batch b, kv head h) the token axis is:
//   quantized groups  [0, Tq)   2-bit codes, dequantized in registers; positions
//                               currently in pool.entries are masked (their
//                               full-precision rows are attended from the pool
//                               instead — the overwrite semantics of
//                               attention.py:73-75, never double counted)
//   pool.entries rows           fp16, <= N slots (empty slots masked)
//   pending rows      [Tq, T)   fp16 ring
//
// Grid = (units, n_qsplits + n_fsplits): the first n_qsplits CTAs of a unit stream
// contiguous ranges of quantized group records; the last n_fsplits CTAs (1 or 2)
// attend the full-precision tiers. Each CTA writes an online-softmax partial (m, l, acc)
// per query head; combine_kernel merges them.
//
// Quantized path (d = 128): tensor cores via mma.sync m16n8k16 (f16 in, f32
// accumulate). Group records (codes + params, contiguous) are staged into
// shared memory with TMA bulk copies (cp.async.bulk + mbarrier), 2-3 stages per
// warp. K codes become fp16 (1 + c/4) with one shift + one LOP3 per pair; the
// per-channel K steps are folded into q (B operand, hi/lo fp16 split so the
// products keep ~22 bits) and K x_min (minus the exact offset) into a
// per-(group, head) bias. V codes become exact fp16 subnormals c * 2^-16; the
// per-token V step is folded into P' = 4 p step (fp16) and V x_min into a
// per-head fp32 bias. See DESIGN.md §4.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "ott_common.cuh"

namespace ott {

#ifndef OTT_MMA_MIN_BLOCKS
#define OTT_MMA_MIN_BLOCKS 4
#endif
constexpr int kAttnThreads = 128;
constexpr int kAttnWarps = kAttnThreads / 32;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLazy = 6.f;
#ifndef OTT_PDL  // launch the split combine as a programmatic dependent of the attention grid
#define OTT_PDL 1
#endif
__device__ __forceinline__ void allow_dependents() {
#if OTT_PDL
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
#endif
}
// lazy-rescale threshold (log2 units, kLazy above): p <= 64, P' = 4 p step fits fp16

struct AttnArgs {
  ott_cache_t c;
  const uint16_t* q;
  uint16_t* out;
  float* ws;  // [n_units][NR][n_splits][D+2]
  int64_t q_tokens, total_tokens;
  int n_splits;   // total partials per (unit, head) = n_qsplits + n_fsplits
  int n_qsplits;  // splits over the quantized region
  int n_fsplits;  // CTAs sharing the full-precision tiers (1, or 2 for small quantized regions)
  int n_qtiles, n_ptiles, n_rtiles;  // 32-token tiles: quantized, pool, pending
  float scale_log2;                  // log2(e) / float32(sqrt(d))
  uint32_t k_magic;                  // 0x3C003C00 (fp16 1.0 pair), passed at run time so the
                                     // compiler keeps it in a register: one LOP3 per code pair
  const int64_t* dev_counts;         // non-null: device-counter decode step (token counts below are
                                     // taken from [quantized, total] before this step's append)
  const uint16_t *new_k, *new_v;     // non-null: this step's appended rows [n_units][d], written to
                                     // the pending ring (slot (total-1) % (G+R)) by the fp-tier CTA
  bool advance;                      // device-counter mode: the combine advances the counts (false
                                     // for all but the last head chunk of n_rep > 8)
};

// Token counts of one launch. Host mode: the launch arguments. Device-counter mode
// (CUDA-graph decode step: ring write, flush-if-due, attend, combine): the counters
// hold the state before the step's append, which has already been written, and the
// flush kernel has quantized one group iff it was due (cache.py:138).
struct Counts {
  int64_t q_tokens, total_tokens;
  int n_qtiles, n_ptiles, n_rtiles;
};
__device__ __forceinline__ Counts counts_of(const AttnArgs& a) {
  Counts k;
  if (a.dev_counts) {
    const int64_t qt = a.dev_counts[0], tot = a.dev_counts[1] + 1;
    const bool due = tot - qt - a.c.residual >= a.c.group_size && qt / a.c.group_size + 1 <= a.c.max_groups;
    k.q_tokens = qt + (due ? a.c.group_size : 0);
    k.total_tokens = tot;
  } else {
    k.q_tokens = a.q_tokens;
    k.total_tokens = a.total_tokens;
  }
  k.n_qtiles = (int)(k.q_tokens / 32);
  k.n_ptiles = (a.c.capacity + 31) / 32;
  k.n_rtiles = (int)((k.total_tokens - k.q_tokens + 31) / 32);
  return k;
}

// ============================================================ SIMT (CUDA-core) tiles
template <int NR, int D>
struct WarpScratch {
  float qp[NR][D];
  float p[NR][32];
  uint32_t vw[32][D / 4];  // V codes of 32 tokens, packed (any width up to 8 bits)
  float vstep[32], vxmin[32];
};

template <int NR, int D>
struct SimtSmem {
  float qs[NR][D];  // q * scale_log2
  WarpScratch<NR, D> w[kAttnWarps];
  float m[kAttnWarps][NR], l[kAttnWarps][NR];
  float acc[kAttnWarps][NR][D];
};

template <int NR, int D>
__device__ __forceinline__ void online_update(float (&s)[NR], float (&m)[NR], float (&l)[NR],
                                              float (&acc)[NR][D / 32], WarpScratch<NR, D>& ws, int lane) {
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const float tmax = warp_max(s[r]);
    const float m_new = fmaxf(m[r], tmax);
    if (m_new == -INFINITY) {
      ws.p[r][lane] = 0.f;
      continue;
    }
    const float corr = exp2f(m[r] - m_new);
    const float p = exp2f(s[r] - m_new);
    ws.p[r][lane] = p;
    l[r] = l[r] * corr + warp_sum(p);
    m[r] = m_new;
#pragma unroll
    for (int k = 0; k < D / 32; ++k) acc[r][k] *= corr;
  }
  __syncwarp();
}

// Processes 32-token tiles [t_begin, t_end) of unit u (warp-strided), merges
// the warps of the CTA and writes partial `split`.
template <int NR, int D>
__device__ void simt_body(const AttnArgs& a, const Counts& n, int u, int t_begin, int t_end, int split,
                          SimtSmem<NR, D>& sm) {
  const ott_cache_t& c = a.c;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = c.group_size, N = c.capacity, cap = G + c.residual;
  const RecordLayout L(D, G, c.bits);
  const int bits = L.bits;  // stored code width
  WarpScratch<NR, D>& ws = sm.w[warp];

  for (int i = tid; i < NR * D; i += kAttnThreads)
    sm.qs[i / D][i % D] = h2f(a.q[((size_t)u * NR) * D + i]) * a.scale_log2;
  __syncthreads();

  float m[NR], l[NR], acc[NR][D / 32];
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    m[r] = -INFINITY;
    l[r] = 0.f;
#pragma unroll
    for (int k = 0; k < D / 32; ++k) acc[r][k] = 0.f;
  }
  const uint32_t* pmask = c.pool_mask + (size_t)u * mask_words_per_unit(c);

  for (int t = t_begin + warp; t < t_end; t += kAttnWarps) {
    float s[NR];
    if (t < n.n_qtiles) {
      const int64_t tok0 = (int64_t)t * 32;
      const int64_t gi = tok0 / G;
      const int row0 = (int)(tok0 - gi * G);
      const uint8_t* rec = record_ptr(c, u, gi);
      float bias[NR];
#pragma unroll
      for (int r = 0; r < NR; ++r) bias[r] = 0.f;
      for (int col = lane; col < D; col += 32) {
        const float st = k_step_of(rec, L, col), mn = k_xmin_of(rec, L, col, st);
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          ws.qp[r][col] = sm.qs[r][col] * st;
          bias[r] += sm.qs[r][col] * mn;
        }
      }
#pragma unroll
      for (int r = 0; r < NR; ++r) bias[r] = warp_sum(bias[r]);
      // V code rows of the tile (32 * D * bits / 32 words, contiguous in pack order)
      const uint32_t* vcw = reinterpret_cast<const uint32_t*>(rec + L.v_codes()) + (size_t)row0 * D * bits / 32;
      for (int idx = lane; idx < D * bits; idx += 32) (&ws.vw[0][0])[idx] = vcw[idx];
      ws.vstep[lane] = reinterpret_cast<const float*>(rec + L.v_step())[row0 + lane];
      ws.vxmin[lane] = reinterpret_cast<const float*>(rec + L.v_xmin())[row0 + lane];
      __syncwarp();
#pragma unroll
      for (int r = 0; r < NR; ++r) s[r] = bias[r];
      if (bits == 2) {
        const uint32_t* kcw = reinterpret_cast<const uint32_t*>(rec + L.k_codes()) + (size_t)(row0 + lane) * (D / 16);
#pragma unroll
        for (int j = 0; j < D / 16; ++j) {
          const uint32_t w = kcw[j];
#pragma unroll
          for (int b = 0; b < 16; ++b) {
            const float code = (float)((w >> (2 * b)) & 3u);
#pragma unroll
            for (int r = 0; r < NR; ++r) s[r] = fmaf(code, ws.qp[r][j * 16 + b], s[r]);
          }
        }
      } else {  // other widths (quant.py supports 1..8): generic stream extraction
        const uint8_t* kc = rec + L.k_codes();
        const int64_t e0 = (int64_t)(row0 + lane) * D;
        for (int col = 0; col < D; ++col) {
          const float code = (float)code_at(kc, e0 + col, bits);
#pragma unroll
          for (int r = 0; r < NR; ++r) s[r] = fmaf(code, ws.qp[r][col], s[r]);
        }
      }
      const bool pooled = (pmask[tok0 >> 5] >> lane) & 1u;
      if (pooled) {
#pragma unroll
        for (int r = 0; r < NR; ++r) s[r] = -INFINITY;
      }
      online_update<NR, D>(s, m, l, acc, ws, lane);
      const uint8_t* vcodes = reinterpret_cast<const uint8_t*>(&ws.vw[0][0]);
#pragma unroll 4
      for (int tt = 0; tt < 32; ++tt) {
        const float st = ws.vstep[tt], mn = ws.vxmin[tt];
#pragma unroll
        for (int k = 0; k < D / 32; ++k) {
          const int col = lane + 32 * k;
          const uint32_t code = bits == 2 ? (uint32_t)((vcodes[(tt * D + col) >> 2] >> (2 * (col & 3))) & 3u)
                                          : code_at(vcodes, (int64_t)tt * D + col, bits);
          const float v = fmaf((float)code, st, mn);
#pragma unroll
          for (int r = 0; r < NR; ++r) acc[r][k] = fmaf(ws.p[r][tt], v, acc[r][k]);
        }
      }
      __syncwarp();
    } else {
      const bool is_pool = t < n.n_qtiles + n.n_ptiles;
      const uint16_t *krow, *vrow;
      bool valid;
      if (is_pool) {
        const int slot = (t - n.n_qtiles) * 32 + lane;
        valid = slot < N && c.pool_pos[(size_t)u * N + slot] >= 0;
        const size_t off = ((size_t)u * N + (valid ? slot : 0)) * D;
        krow = c.pool_k + off;
        vrow = c.pool_v + off;
      } else {
        const int64_t p = n.q_tokens + (int64_t)(t - n.n_qtiles - n.n_ptiles) * 32 + lane;
        valid = p < n.total_tokens;
        const size_t off = ((size_t)u * cap + (size_t)((valid ? p : n.q_tokens) % cap)) * D;
        krow = c.pend_k + off;
        vrow = c.pend_v + off;
      }
#pragma unroll
      for (int r = 0; r < NR; ++r) s[r] = 0.f;
      if (valid) {
#pragma unroll 4
        for (int j = 0; j < D / 8; ++j) {
          const uint4 k8 = *reinterpret_cast<const uint4*>(krow + j * 8);
          const uint16_t* kh = reinterpret_cast<const uint16_t*>(&k8);
#pragma unroll
          for (int b = 0; b < 8; ++b) {
            const float kv = h2f(kh[b]);
#pragma unroll
            for (int r = 0; r < NR; ++r) s[r] = fmaf(kv, sm.qs[r][j * 8 + b], s[r]);
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < NR; ++r) s[r] = -INFINITY;
      }
      online_update<NR, D>(s, m, l, acc, ws, lane);
      for (int tt = 0; tt < 32; ++tt) {
        const unsigned long long vp = __shfl_sync(0xffffffffu, (unsigned long long)vrow, tt);
        const int ok = __shfl_sync(0xffffffffu, valid ? 1 : 0, tt);
        if (!ok) continue;
        const uint16_t* vr = reinterpret_cast<const uint16_t*>(vp);
#pragma unroll
        for (int k = 0; k < D / 32; ++k) {
          const float v = h2f(vr[lane + 32 * k]);
#pragma unroll
          for (int r = 0; r < NR; ++r) acc[r][k] = fmaf(ws.p[r][tt], v, acc[r][k]);
        }
      }
      __syncwarp();
    }
  }

  if (lane == 0) {
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      sm.m[warp][r] = m[r];
      sm.l[warp][r] = l[r];
    }
  }
#pragma unroll
  for (int r = 0; r < NR; ++r)
#pragma unroll
    for (int k = 0; k < D / 32; ++k) sm.acc[warp][r][lane + 32 * k] = acc[r][k];
  __syncthreads();
  for (int i = tid; i < NR * D; i += kAttnThreads) {
    const int r = i / D, col = i % D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kAttnWarps; ++w) M = fmaxf(M, sm.m[w][r]);
    float Lsum = 0.f, A = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int w = 0; w < kAttnWarps; ++w) {
        const float f = exp2f(sm.m[w][r] - M);
        Lsum += sm.l[w][r] * f;
        A += sm.acc[w][r][col] * f;
      }
    }
    float* base = a.ws + (((size_t)u * NR + r) * a.n_splits + split) * (D + 2);
    base[2 + col] = A;
    if (col == 0) {
      base[0] = M;
      base[1] = Lsum;
    }
  }
}

template <int NR, int D>
__global__ void __launch_bounds__(kAttnThreads) attend_simt_kernel(AttnArgs a) {
  extern __shared__ __align__(256) unsigned char smem_raw[];
  allow_dependents();
  SimtSmem<NR, D>& sm = *reinterpret_cast<SimtSmem<NR, D>*>(smem_raw);
  const Counts n = counts_of(a);
  const int n_tiles = n.n_qtiles + n.n_ptiles + n.n_rtiles;
  const int per = (n_tiles + a.n_splits - 1) / a.n_splits;
  const int t_begin = blockIdx.y * per;
  const int t_end = min(n_tiles, t_begin + per);
  simt_body<NR, D>(a, n, blockIdx.x, t_begin, t_end, blockIdx.y, sm);
}

// ============================================================ generic shapes
// Any head_dim in [1, 128] and group size in [1, 128] (the reference's own tests use
// d in {2..16} and G in {4, 8, 16}): a 32-token tile may span several groups, so every
// token looks up its own group record. Same tile order and split/combine structure as
// the SIMT kernel; this path is for shape coverage, not speed.
template <int NR>
struct GenericSmem {
  float qs[NR][kMaxD];  // q * scale_log2
  float p[kAttnWarps][NR][32];
  float m[kAttnWarps][NR], l[kAttnWarps][NR];
  float acc[kAttnWarps][NR][kMaxD];
};

template <int NR>
__global__ void __launch_bounds__(kAttnThreads) attend_generic_kernel(AttnArgs a) {
  extern __shared__ __align__(256) unsigned char smem_raw[];
  allow_dependents();
  GenericSmem<NR>& sm = *reinterpret_cast<GenericSmem<NR>*>(smem_raw);
  const Counts n = counts_of(a);
  const ott_cache_t& c = a.c;
  const int D = c.head_dim, G = c.group_size, N = c.capacity, cap = G + c.residual;
  const RecordLayout L(D, G, c.bits);
  const int bits = L.bits;  // stored code width
  const int u = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nq = (int)((n.q_tokens + 31) / 32), np = (N + 31) / 32;
  const int nr = (int)((n.total_tokens - n.q_tokens + 31) / 32);
  const int n_tiles = nq + np + nr;
  const int per = (n_tiles + a.n_splits - 1) / a.n_splits;
  const int t_begin = blockIdx.y * per, t_end = min(n_tiles, t_begin + per);
  const uint32_t* pmask = c.pool_mask + (size_t)u * mask_words_per_unit(c);

  for (int i = tid; i < NR * D; i += kAttnThreads)
    sm.qs[i / D][i % D] = h2f(a.q[((size_t)u * NR) * D + i]) * a.scale_log2;
  __syncthreads();

  float m[NR], l[NR], acc[NR][kMaxD / 32];
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    m[r] = -INFINITY;
    l[r] = 0.f;
#pragma unroll
    for (int k = 0; k < kMaxD / 32; ++k) acc[r][k] = 0.f;
  }
  for (int t = t_begin + warp; t < t_end; t += kAttnWarps) {
    // logits of this lane's token
    float s[NR];
    const uint16_t* vrow = nullptr;  // fp tiers: the token's V row
    bool valid;
    if (t < nq) {
      const int64_t p = (int64_t)t * 32 + lane;
      valid = p < n.q_tokens && !((pmask[p >> 5] >> (p & 31)) & 1u);  // pooled: attended from the pool
      if (valid) {
        const int64_t gi = p / G;
        const int row = (int)(p - gi * G);
        const uint8_t* rec = record_ptr(c, u, gi);
#pragma unroll
        for (int r = 0; r < NR; ++r) s[r] = 0.f;
        for (int col = 0; col < D; ++col) {
          const float st = k_step_of(rec, L, col);
          const float kv = fmaf((float)code_at(rec + L.k_codes(), (int64_t)row * D + col, bits), st,
                                k_xmin_of(rec, L, col, st));
#pragma unroll
          for (int r = 0; r < NR; ++r) s[r] = fmaf(kv, sm.qs[r][col], s[r]);
        }
      }
    } else {
      const uint16_t* krow;
      if (t < nq + np) {
        const int slot = (t - nq) * 32 + lane;
        valid = slot < N && c.pool_pos[(size_t)u * N + slot] >= 0;
        const size_t off = ((size_t)u * N + (valid ? slot : 0)) * D;
        krow = c.pool_k + off;
        vrow = c.pool_v + off;
      } else {
        const int64_t p = n.q_tokens + (int64_t)(t - nq - np) * 32 + lane;
        valid = p < n.total_tokens;
        const size_t off = ((size_t)u * cap + (size_t)((valid ? p : n.q_tokens) % cap)) * D;
        krow = c.pend_k + off;
        vrow = c.pend_v + off;
      }
      if (valid) {
#pragma unroll
        for (int r = 0; r < NR; ++r) s[r] = 0.f;
        for (int col = 0; col < D; ++col) {
          const float kv = h2f(krow[col]);
#pragma unroll
          for (int r = 0; r < NR; ++r) s[r] = fmaf(kv, sm.qs[r][col], s[r]);
        }
      }
    }
    if (!valid) {
#pragma unroll
      for (int r = 0; r < NR; ++r) s[r] = -INFINITY;
    }
    // online softmax over the tile
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const float m_new = fmaxf(m[r], warp_max(s[r]));
      float pr = 0.f;
      if (m_new != -INFINITY) {
        const float corr = exp2f(m[r] - m_new);
        pr = exp2f(s[r] - m_new);
        l[r] = l[r] * corr + warp_sum(pr);
        m[r] = m_new;
#pragma unroll
        for (int k = 0; k < kMaxD / 32; ++k) acc[r][k] *= corr;
      }
      sm.p[warp][r][lane] = pr;
    }
    __syncwarp();
    // O += p V, lanes over channels
    for (int tt = 0; tt < 32; ++tt) {
      if (!__shfl_sync(0xffffffffu, valid ? 1 : 0, tt)) continue;
      if (t < nq) {
        const int64_t p = (int64_t)t * 32 + tt;
        const int64_t gi = p / G;
        const int row = (int)(p - gi * G);
        const uint8_t* rec = record_ptr(c, u, gi);
        const float st = reinterpret_cast<const float*>(rec + L.v_step())[row];
        const float mn = reinterpret_cast<const float*>(rec + L.v_xmin())[row];
#pragma unroll
        for (int k = 0; k < kMaxD / 32; ++k) {
          const int col = lane + 32 * k;
          if (col < D) {
            const float v = fmaf((float)code_at(rec + L.v_codes(), (int64_t)row * D + col, bits), st, mn);
#pragma unroll
            for (int r = 0; r < NR; ++r) acc[r][k] = fmaf(sm.p[warp][r][tt], v, acc[r][k]);
          }
        }
      } else {
        const uint16_t* vr =
            reinterpret_cast<const uint16_t*>(__shfl_sync(0xffffffffu, (unsigned long long)vrow, tt));
#pragma unroll
        for (int k = 0; k < kMaxD / 32; ++k) {
          const int col = lane + 32 * k;
          if (col < D) {
            const float v = h2f(vr[col]);
#pragma unroll
            for (int r = 0; r < NR; ++r) acc[r][k] = fmaf(sm.p[warp][r][tt], v, acc[r][k]);
          }
        }
      }
    }
    __syncwarp();
  }
  // merge the warps, write partial blockIdx.y ([D + 2] floats per (unit, head, split))
  if (lane == 0) {
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      sm.m[warp][r] = m[r];
      sm.l[warp][r] = l[r];
    }
  }
#pragma unroll
  for (int r = 0; r < NR; ++r)
#pragma unroll
    for (int k = 0; k < kMaxD / 32; ++k) sm.acc[warp][r][lane + 32 * k] = acc[r][k];
  __syncthreads();
  for (int i = tid; i < NR * D; i += kAttnThreads) {
    const int r = i / D, col = i % D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kAttnWarps; ++w) M = fmaxf(M, sm.m[w][r]);
    float Lsum = 0.f, A = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int w = 0; w < kAttnWarps; ++w) {
        const float f = exp2f(sm.m[w][r] - M);
        Lsum += sm.l[w][r] * f;
        A += sm.acc[w][r][col] * f;
      }
    }
    float* base = a.ws + (((size_t)u * NR + r) * a.n_splits + blockIdx.y) * (D + 2);
    base[2 + col] = A;
    if (col == 0) {
      base[0] = M;
      base[1] = Lsum;
    }
  }
}

// ============================================================ tensor-core path
__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  // not volatile: a pure register op, so the scheduler may interleave independent chains
  asm(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t saddr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(saddr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], uint32_t saddr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(saddr));
}
__device__ __forceinline__ float ex2(float x) {  // 2^x, MUFU.EX2 (ftz; -inf -> 0)
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t movm_t(uint32_t x) {
  uint32_t y;
  asm("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;\n" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;\n" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ uint32_t h2_as_u32(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(phase)
        : "memory");
  }
}
__device__ __forceinline__ void tma_bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

// ---- 2-bit pair extraction. A word holds 16 codes (code m at bits 2m, code
// m+8 at bits 16+2m). Pair m is used in place at fp16 mantissa position P(m)
// (bits 2P..2P+1 of both halves) taken from one of three copies of the word:
//   m:    0    1    2   3   4   5    6    7
//   src:  <<6  <<6  x   x   x   >>6  >>6  >>6      (2 SHF + 8 LOP3 per word)
//   P:    3    4    2   3   4   2    3    4
// K codes become fp16 1 + c*2^(2P-10) (one LOP3 with the 1.0 magic); V codes
// become exact fp16 subnormals c*2^(2P-24). The per-position scale is folded
// into q' (K) or the final accumulator scale (V).
struct Shifted {
  uint32_t x, l6, r6;
};
__device__ __forceinline__ Shifted shifted(uint32_t w) { return {w, w << 6, w >> 6}; }
__host__ __device__ constexpr int pair_pos(int m) { return m == 2 || m == 5 ? 2 : (m == 0 || m == 3 || m == 6 ? 3 : 4); }
__host__ __device__ constexpr uint32_t pos_mask(int p) { return p == 2 ? 0x00300030u : (p == 3 ? 0x00C000C0u : 0x03000300u); }
template <int M>
__device__ __forceinline__ uint32_t pair_src(const Shifted& s) {
  return M <= 1 ? s.l6 : (M <= 4 ? s.x : s.r6);
}
template <int M>
__device__ __forceinline__ uint32_t kq(const Shifted& s, uint32_t magic) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;\n" : "=r"(r) : "r"(pair_src<M>(s)), "n"(pos_mask(pair_pos(M))), "r"(magic));
  return r;
}
template <int M>
__device__ __forceinline__ uint32_t vq(const Shifted& s) {
  return pair_src<M>(s) & pos_mask(pair_pos(M));
}

__device__ __forceinline__ uint32_t swz(uint32_t o) { return o ^ ((o >> 3) & 16u); }  // Swizzle<1,4,3>
__host__ __device__ constexpr int tile_slot(int v4, int tig) { return 4 * v4 + (tig ^ ((v4 >> 1) << 1)); }
__device__ __forceinline__ void tma_tensor_rows(uint32_t dst, const CUtensorMap* map, int row, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          dst),
      "l"(map), "r"(0), "r"(row), "r"(bar)
      : "memory");
}
template <int G>
struct RecTma {  // a record is kRows rows of 32 bytes; loaded as kBoxes boxes of kBoxRows rows
  static constexpr int kRows = (G * 128 / 2 + 8 * 128 + 8 * G) / 32;
  static constexpr int kBoxes = kRows > 256 ? 2 : 1;
  static constexpr int kBoxRows = kRows / kBoxes;
};
template <int G>
__device__ __forceinline__ void load_record(uint32_t dst, const CUtensorMap* map, int64_t rec_index, uint32_t bar) {
  constexpr int kRec = RecTma<G>::kRows * 32;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(kRec) : "memory");
#pragma unroll
  for (int b = 0; b < RecTma<G>::kBoxes; ++b)
    tma_tensor_rows(dst + b * RecTma<G>::kBoxRows * 32, map,
                    (int)(rec_index * RecTma<G>::kRows + b * RecTma<G>::kBoxRows), bar);
}

template <int G>
struct MmaSmem {
  static constexpr int kRec = G * 128 / 2 + 8 * 128 + 8 * G;  // record bytes at d = 128
#ifndef OTT_NO_TMA
#define OTT_NO_TMA 0  // timing experiment only: compute on stale shared memory
#endif
#ifndef OTT_NG
#define OTT_NG 1  // groups per loop iteration per warp (2 measured slower: register spills)
#endif
#ifndef OTT_QK_LO  // 1: Q.K^T also multiplies the lo halves of q' (2 HMMA per k-step)
#define OTT_QK_LO 1
#endif
#ifndef OTT_STAGES
#define OTT_STAGES 3  // 3 measured 2 % faster than 2 on config 4 (v7)
#endif
  static constexpr int kNG = G == 32 ? OTT_NG : 1;               // groups per loop iteration
  static constexpr int kStages = G == 32 ? OTT_STAGES : 2;          // TMA pipeline depth per warp
  float4 qt[8][32];  // q (fp32) per lane for the x_min bias, see mma_body
  // group records land here through a SWIZZLE_32B tensor map (16-byte chunk bit 4 ^= bit 7
  // of the offset): ldmatrix over 32-byte token rows is then bank-conflict free
  alignas(256) uint8_t stage[kAttnWarps][kStages][kRec];
  alignas(8) uint64_t bar[kAttnWarps][kStages];
  float mm[kAttnWarps][8], ll[kAttnWarps][8];
};

// Quantized-region partial for (unit blockIdx.x, split blockIdx.y < n_qsplits).
template <int NR, int G>
__device__ void mma_body(const AttnArgs& a, const Counts& n, const CUtensorMap* tmap, MmaSmem<G>& sm) {
  constexpr int D = 128;
  constexpr int kRec = MmaSmem<G>::kRec;
  constexpr int kMt = G / 16;  // 16-token m-tiles per group
  constexpr int kStages = MmaSmem<G>::kStages;
  const RecordLayout L(D, G);
  const ott_cache_t& c = a.c;
  const int u = blockIdx.x, split = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tig = lane & 3;

  const uint32_t magic = a.k_magic;
  const int n_groups = (int)(n.q_tokens / G);
  const int per = (n_groups + a.n_qsplits - 1) / a.n_qsplits;
  const int g0 = split * per;
  const int g1 = min(n_groups, g0 + per);
  const int my_n = g1 > g0 + warp ? (g1 - g0 - warp + kAttnWarps - 1) / kAttnWarps : 0;

  // q (fp32) table for the x_min bias: [k][lane] = q[head lane/4][channels of words tig, 4+tig]:
  // k < 4: 16 tig + 4k .. +3; k >= 4: 64 + 16 tig + 4(k-4) .. +3  (conflict-free LDS.128)
  for (int i = tid; i < 8 * 32; i += kAttnThreads) {
    const int k = i >> 5, ln = i & 31, h = ln >> 2, t4 = ln & 3;
    const int ch = (k < 4 ? 16 * t4 : 64 + 16 * t4) + 4 * (k & 3);
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (h < NR) {
      const uint2 raw = __ldg(reinterpret_cast<const uint2*>(a.q + ((size_t)u * NR + h) * D + ch));
      const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&raw.x));
      const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&raw.y));
      v = make_float4(f0.x, f0.y, f1.x, f1.y);
    }
    sm.qt[k][ln] = v;
  }
  const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&sm.bar[warp][0]);
  const uint32_t stage0 = (uint32_t)__cvta_generic_to_shared(&sm.stage[warp][0][0]);
  const int64_t unit_rec = (int64_t)u * c.max_groups;  // record index of group 0
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kStages; ++s) mbar_init(bar0 + 8 * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
#pragma unroll
    for (int s = 0; s < kStages; ++s)
      if (s < my_n && !OTT_NO_TMA)
        load_record<G>(stage0 + s * kRec, tmap, unit_rec + g0 + warp + s * kAttnWarps, bar0 + 8 * s);
  }
  __syncthreads();

  float o[8][4];
#pragma unroll
  for (int cm = 0; cm < 8; ++cm) o[cm][0] = o[cm][1] = o[cm][2] = o[cm][3] = 0.f;
  float mrun[2] = {-INFINITY, -INFINITY}, lsum[2] = {0.f, 0.f}, vb[2] = {0.f, 0.f};
  const uint32_t* pmask = c.pool_mask + (size_t)u * mask_words_per_unit(c);

  // ldmatrix row addresses (bytes, relative to a 16-token tile): matrix i = lane/8,
  // row r = lane%8: i0 tokens 0-7 bytes 0-15, i1 tokens 8-15 bytes 0-15,
  // i2 tokens 0-7 bytes 16-31, i3 tokens 8-15 bytes 16-31.
  const uint32_t lm_off = (uint32_t)(((lane & 7) + ((lane >> 3) & 1) * 8) * 32 + (lane >> 4) * 16);
  __syncthreads();
  // q * u(m) as exact fp16 pairs (channels 16w+m, 16w+m+8) of head g, words w = tig + 4 hw:
  // the B operand q' = q u step is formed per group from the record's fp16 step halves
  __half2 q16[2][8];
#pragma unroll
  for (int hw = 0; hw < 2; ++hw)
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const float4 qa = sm.qt[4 * hw + m / 4][lane];
      const float4 qb = sm.qt[4 * hw + 2 + m / 4][lane];
      const float lo = (m % 4 == 0 ? qa.x : m % 4 == 1 ? qa.y : m % 4 == 2 ? qa.z : qa.w) * kpair_u(m);
      const float hi = (m % 4 == 0 ? qb.x : m % 4 == 1 ? qb.y : m % 4 == 2 ? qb.z : qb.w) * kpair_u(m);
      q16[hw][m] = __floats2half2_rn(lo, hi);
    }
  const float scale4 = 4.f * a.scale_log2;
  // Groups are processed NG at a time (two independent instruction streams per
  // warp for the scheduler); a lone tail group is paired with a masked dummy.
  constexpr int NG = MmaSmem<G>::kNG;
  for (int k = 0; k < my_n; k += NG) {
    const int ng = min(NG, my_n - k);
    const uint8_t* rec[NG];
    uint32_t rec_s[NG];
    uint32_t mwords[NG][G / 32];
#pragma unroll
    for (int j = 0; j < NG; ++j) {
      const int kk = k + (j < ng ? j : 0);
      const int gi = g0 + warp + kk * kAttnWarps;
#pragma unroll
      for (int w = 0; w < G / 32; ++w) mwords[j][w] = __ldg(&pmask[(size_t)gi * (G / 32) + w]);
      const int s = kk % kStages;
      if (j < ng && !OTT_NO_TMA) mbar_wait(bar0 + 8 * s, (uint32_t)((kk / kStages) & 1));
      rec[j] = &sm.stage[warp][s][0];
      rec_s[j] = stage0 + s * kRec;
    }
    uint32_t kw[NG][kMt][4];
#pragma unroll
    for (int j = 0; j < NG; ++j) {
      // K code words (ldmatrix: token g / g+8, words tig and 4+tig)
#pragma unroll
      for (int mt = 0; mt < kMt; ++mt) ldsm_x4(kw[j][mt], rec_s[j] + swz(L.k_codes() + mt * 16 * 32 + lm_off));
    }
    __syncwarp();

    // ---- S = Q K^T on tensor cores. B operand q' = q u step as an exact fp16 hi/lo split
    // from the record's fp16 step halves (sh + sl): hi = q sh, err = fma(q, sh, -hi) (exact),
    // lo = fma(q, sl, err); hi and lo accumulate into one chain.
    // x_min bias (scale * sum_c q e, e = x_min - 4 u step from the record) per head g.
    float ch[NG][kMt][4];
    float bias_g[NG];
#pragma unroll
    for (int j = 0; j < NG; ++j) {
      float2 acc2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                        make_float2(0.f, 0.f)};  // 4 independent chains
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int wd = k < 4 ? tig : 4 + tig;
        const float4 ev = *reinterpret_cast<const float4*>(rec[j] + swz(L.k_e() + 64 * wd + 16 * (k & 3)));
        const float4 qv = sm.qt[k][lane];
        acc2[(2 * k) & 3] = __ffma2_rn(make_float2(qv.x, qv.y), make_float2(ev.x, ev.y), acc2[(2 * k) & 3]);
        acc2[(2 * k + 1) & 3] = __ffma2_rn(make_float2(qv.z, qv.w), make_float2(ev.z, ev.w), acc2[(2 * k + 1) & 3]);
      }
      bias_g[j] = ((acc2[0].x + acc2[0].y) + (acc2[1].x + acc2[1].y)) + ((acc2[2].x + acc2[2].y) + (acc2[3].x + acc2[3].y));
#pragma unroll
      for (int mt = 0; mt < kMt; ++mt) ch[j][mt][0] = ch[j][mt][1] = ch[j][mt][2] = ch[j][mt][3] = 0.f;
    }
#if !OTT_QK_LO
    __half2 lo_acc[NG][2];
#pragma unroll
    for (int j = 0; j < NG; ++j) lo_acc[j][0] = lo_acc[j][1] = __float2half2_rn(0.f);
#endif
#pragma unroll
    for (int hw = 0; hw < 2; ++hw) {
#pragma unroll
      for (int j = 0; j < NG; ++j) {
        const int wd = tig + 4 * hw;
        const uint4 h0 = *reinterpret_cast<const uint4*>(rec[j] + swz(L.k_sh() + 32 * wd));
        const uint4 h1 = *reinterpret_cast<const uint4*>(rec[j] + swz(L.k_sh() + 32 * wd + 16));
        const uint4 l0 = *reinterpret_cast<const uint4*>(rec[j] + swz(L.k_sl() + 32 * wd));
        const uint4 l1 = *reinterpret_cast<const uint4*>(rec[j] + swz(L.k_sl() + 32 * wd + 16));
        const uint32_t shw[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
        const uint32_t slw[8] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
        uint32_t bh[8], bl[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          const __half2 sh = *reinterpret_cast<const __half2*>(&shw[m]);
          const __half2 sl = *reinterpret_cast<const __half2*>(&slw[m]);
          const __half2 H = __hmul2(q16[hw][m], sh);
          const __half2 E = __hfma2(q16[hw][m], sh, __hneg2(H));
          bh[m] = h2_as_u32(H);
#if OTT_QK_LO
          bl[m] = h2_as_u32(__hfma2(q16[hw][m], sl, E));
#else
          lo_acc[j][m & 1] = __hadd2(lo_acc[j][m & 1], __hfma2(q16[hw][m], sl, E));
#endif
        }
        Shifted s0[kMt], s1[kMt];
#pragma unroll
        for (int mt = 0; mt < kMt; ++mt) {
          s0[mt] = shifted(kw[j][mt][2 * hw]);
          s1[mt] = shifted(kw[j][mt][2 * hw + 1]);
        }
#define OTT_QK(MM)                                                                    \
  {                                                                                   \
    _Pragma("unroll") for (int mt = 0; mt < kMt; ++mt) {                              \
      const uint32_t a0 = kq<MM>(s0[mt], magic), a1 = kq<MM>(s1[mt], magic);         \
      const uint32_t a2 = kq<MM + 1>(s0[mt], magic), a3 = kq<MM + 1>(s1[mt], magic); \
      mma16816(ch[j][mt], a0, a1, a2, a3, bh[MM], bh[MM + 1]);                        \
      if (OTT_QK_LO) mma16816(ch[j][mt], a0, a1, a2, a3, bl[MM], bl[MM + 1]);         \
    }                                                                                 \
  }
        OTT_QK(0) OTT_QK(2) OTT_QK(4) OTT_QK(6)
#undef OTT_QK
      }
    }
#if !OTT_QK_LO
    // Q.K^T used only the hi halves: ch = sum (q' - lo) (1 + c 2^(2P-10)). The bias takes
    // back sum lo (the offset part, 4u/c times larger than the code part), leaving
    // -sum lo c 2^(2P-10): the rounding error of q' step c in fp16, 2^-12 relative per term.
#pragma unroll
    for (int j = 0; j < NG; ++j) {
      const float2 lf = __half22float2(__hadd2(lo_acc[j][0], lo_acc[j][1]));
      bias_g[j] = fmaf(4.f, lf.x + lf.y, bias_g[j]);
    }
#endif
    float sc[NG][kMt][4];
#pragma unroll
    for (int j = 0; j < NG; ++j) {
      float bias = bias_g[j];
      bias += __shfl_xor_sync(0xffffffffu, bias, 1);
      bias += __shfl_xor_sync(0xffffffffu, bias, 2);
      bias *= a.scale_log2;
      const float bias0 = __shfl_sync(0xffffffffu, bias, 8 * tig);      // head 2*tig
      const float bias1 = __shfl_sync(0xffffffffu, bias, 8 * tig + 4);  // head 2*tig+1
      const bool dummy = j >= ng;
#pragma unroll
      for (int mt = 0; mt < kMt; ++mt) {
        sc[j][mt][0] = dummy ? -INFINITY : fmaf(ch[j][mt][0], scale4, bias0);
        sc[j][mt][1] = dummy ? -INFINITY : fmaf(ch[j][mt][1], scale4, bias1);
        sc[j][mt][2] = dummy ? -INFINITY : fmaf(ch[j][mt][2], scale4, bias0);
        sc[j][mt][3] = dummy ? -INFINITY : fmaf(ch[j][mt][3], scale4, bias1);
      }
      // pooled positions: their logits come from the pool tile (overwrite semantics)
#pragma unroll
      for (int w = 0; w < G / 32; ++w) {
        const uint32_t mw = mwords[j][w];
        if (mw) {
#pragma unroll
          for (int mt = 2 * w; mt < 2 * w + 2; ++mt) {
            if ((mw >> ((mt & 1) * 16 + g)) & 1u) sc[j][mt][0] = sc[j][mt][1] = -INFINITY;
            if ((mw >> ((mt & 1) * 16 + g + 8)) & 1u) sc[j][mt][2] = sc[j][mt][3] = -INFINITY;
          }
        }
      }
    }

    // ---- online softmax (heads 2*tig, 2*tig+1), lazily rescaled: the running max
    // only moves when a logit exceeds it by kLazy (log2 units), so p <= 2^kLazy
    float tmax[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float t = -INFINITY;
#pragma unroll
      for (int j = 0; j < NG; ++j)
#pragma unroll
        for (int mt = 0; mt < kMt; ++mt) t = fmaxf(t, fmaxf(sc[j][mt][h], sc[j][mt][h + 2]));
      tmax[h] = t;
    }
    const bool need = tmax[0] > mrun[0] + kLazy || tmax[1] > mrun[1] + kLazy;
    if (__any_sync(0xffffffffu, need)) {  // rare: warp max over the token rows, rescale
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float t = tmax[h];
        t = fmaxf(t, __shfl_xor_sync(0xffffffffu, t, 4));
        t = fmaxf(t, __shfl_xor_sync(0xffffffffu, t, 8));
        t = fmaxf(t, __shfl_xor_sync(0xffffffffu, t, 16));
        const float mnew = fmaxf(mrun[h], t);
        const float corr = mnew == -INFINITY ? 1.f : ex2(mrun[h] - mnew);
        lsum[h] *= corr;
        vb[h] *= corr;
#pragma unroll
        for (int cm = 0; cm < 8; ++cm) {
          o[cm][h] *= corr;
          o[cm][h + 2] *= corr;
        }
        mrun[h] = mnew;
      }
    }
    const float me0 = mrun[0] == -INFINITY ? 0.f : mrun[0];
    const float me1 = mrun[1] == -INFINITY ? 0.f : mrun[1];

    // ---- O^T += V^T P'  (P' = 4 p step fp16, V x_min into vb; with V codes as
    // subnormals the accumulator holds sum(p step c) * 2^(2P-22))
#pragma unroll
    for (int j = 0; j < NG; ++j) {
#pragma unroll
      for (int mt = 0; mt < kMt; ++mt) {
        const float vs0 = *reinterpret_cast<const float*>(rec[j] + swz(L.v_step() + 4 * (mt * 16 + g)));
        const float vs1 = *reinterpret_cast<const float*>(rec[j] + swz(L.v_step() + 4 * (mt * 16 + g + 8)));
        const float ve0 = *reinterpret_cast<const float*>(rec[j] + swz(L.v_xmin() + 4 * (mt * 16 + g)));
        const float ve1 = *reinterpret_cast<const float*>(rec[j] + swz(L.v_xmin() + 4 * (mt * 16 + g + 8)));
        const float p00 = ex2(sc[j][mt][0] - me0), p01 = ex2(sc[j][mt][1] - me1);
        const float p10 = ex2(sc[j][mt][2] - me0), p11 = ex2(sc[j][mt][3] - me1);
        lsum[0] += p00 + p10;
        lsum[1] += p01 + p11;
        vb[0] = fmaf(p00, ve0, fmaf(p10, ve1, vb[0]));
        vb[1] = fmaf(p01, ve0, fmaf(p11, ve1, vb[1]));
        const float f0 = 4.f * vs0, f1 = 4.f * vs1;
        const uint32_t b0 = movm_t(pack_h2(p00 * f0, p01 * f0));
        const uint32_t b1 = movm_t(pack_h2(p10 * f1, p11 * f1));
        uint32_t vr[4];
        ldsm_x4_t(vr, rec_s[j] + swz(L.v_codes() + mt * 16 * 32 + lm_off));
        const Shifted v0 = shifted(vr[0]), v1 = shifted(vr[1]), v2 = shifted(vr[2]), v3 = shifted(vr[3]);
#define OTT_PV(CM) mma16816(o[CM], vq<CM>(v0), vq<CM>(v2), vq<CM>(v1), vq<CM>(v3), b0, b1);
        OTT_PV(0) OTT_PV(1) OTT_PV(2) OTT_PV(3) OTT_PV(4) OTT_PV(5) OTT_PV(6) OTT_PV(7)
#undef OTT_PV
      }
    }

    __syncwarp();
    if (lane == 0) {
#pragma unroll
      for (int j = 0; j < NG; ++j) {
        const int kk = k + j, ka = kk + kStages;
        if (j < ng && ka < my_n && !OTT_NO_TMA) {
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          load_record<G>(stage0 + (kk % kStages) * kRec, tmap, unit_rec + g0 + warp + ka * kAttnWarps,
                         bar0 + 8 * (kk % kStages));
        }
      }
    }
  }

  // ---- reduce l, vb over the token rows (lanes with equal tig), merge warps
#pragma unroll
  for (int h = 0; h < 2; ++h) {
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      lsum[h] += __shfl_xor_sync(0xffffffffu, lsum[h], off);
      vb[h] += __shfl_xor_sync(0xffffffffu, vb[h], off);
    }
  }
  if (g == 0) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      sm.mm[warp][2 * tig + h] = mrun[h];
      sm.ll[warp][2 * tig + h] = lsum[h];
    }
  }
  __syncthreads();  // every warp is past its loop: stage memory is free
  float* accw = reinterpret_cast<float*>(&sm.stage[warp][0][0]);  // [8 heads][128] natural channel order
#pragma unroll
  for (int cm = 0; cm < 8; ++cm) {
    const float f = pair_pos(cm) == 2 ? 262144.f : (pair_pos(cm) == 3 ? 65536.f : 16384.f);  // 2^(22-2P)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      accw[(2 * tig + h) * D + 8 * g + cm] = fmaf(o[cm][h], f, vb[h]);
      accw[(2 * tig + h) * D + 64 + 8 * g + cm] = fmaf(o[cm][h + 2], f, vb[h]);
    }
  }
  __syncthreads();
  for (int i = tid; i < NR * D; i += kAttnThreads) {
    const int r = i / D, col = i % D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kAttnWarps; ++w) M = fmaxf(M, sm.mm[w][r]);
    float Lsum = 0.f, A = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int w = 0; w < kAttnWarps; ++w) {
        if (sm.mm[w][r] == -INFINITY) continue;
        const float f = exp2f(sm.mm[w][r] - M);
        Lsum += sm.ll[w][r] * f;
        A += reinterpret_cast<const float*>(&sm.stage[w][0][0])[r * D + col] * f;
      }
    }
    float* base = a.ws + (((size_t)u * NR + r) * a.n_splits + split) * (D + 2);
    base[2 + col] = A;
    if (col == 0) {
      base[0] = M;
      base[1] = Lsum;
    }
  }
}

// ---- full-precision tiers (pool.entries + pending ring) on tensor cores.
// 16-row tiles of fp16 K/V rows are staged with per-row TMA bulk copies into a
// padded layout (272-byte row pitch: conflict-free ldmatrix); q (exact fp16) is
// the B operand of Q K^T, P the B operand of V^T P. One stage per warp: these
// tiers hold at most N + G + R - 1 rows per unit.
struct FpSmem {
  static constexpr int kRow = 272;
  alignas(128) uint8_t kr[kAttnWarps][16][kRow];
  alignas(128) uint8_t vr[kAttnWarps][16][kRow];
  alignas(8) uint64_t bar[kAttnWarps];
  float mm[kAttnWarps][8], ll[kAttnWarps][8];
};

// barrier over warps 0-3 only (the tcgen05 kernel's fifth warp does not take part)
__device__ __forceinline__ void sync4() { asm volatile("bar.sync 1, 128;\n" ::: "memory"); }

__device__ __forceinline__ void tma_row(uint32_t dst, const void* src, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];\n" ::"r"(dst),
      "l"(src), "r"(bar)
      : "memory");
}

template <int NR>
__device__ void fp_body(const AttnArgs& a, const Counts& n, FpSmem& sm) {
  constexpr int D = 128, kRow = FpSmem::kRow;
  const ott_cache_t& c = a.c;
  const int u = blockIdx.x, split = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tig = lane & 3;
  const int N = c.capacity, cap = c.group_size + c.residual;
  const int n_pool_t = (N + 15) / 16;
  const int Tp = (int)(n.total_tokens - n.q_tokens);
  const int n_tiles = n_pool_t + (Tp + 15) / 16;

  // q (exact fp16) as the B fragments of Q K^T: head g, channels 16j + 2tig (+1), +8
  uint32_t qb[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (g < NR) {
      const uint32_t* qp = reinterpret_cast<const uint32_t*>(a.q + ((size_t)u * NR + g) * D + 16 * j + 2 * tig);
      qb[j][0] = qp[0];
      qb[j][1] = qp[4];
    } else {
      qb[j][0] = qb[j][1] = 0u;
    }
  }
  // zero the staging rows once: rows a tile does not copy keep finite (stale or zero)
  // data, so a zero softmax weight never meets a NaN
  for (int i = lane; i < 16 * kRow / 16; i += 32) {
    reinterpret_cast<uint4*>(&sm.kr[warp][0][0])[i] = make_uint4(0, 0, 0, 0);
    reinterpret_cast<uint4*>(&sm.vr[warp][0][0])[i] = make_uint4(0, 0, 0, 0);
  }
  const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&sm.bar[warp]);
  const uint32_t kr_s = (uint32_t)__cvta_generic_to_shared(&sm.kr[warp][0][0]);
  const uint32_t vr_s = (uint32_t)__cvta_generic_to_shared(&sm.vr[warp][0][0]);
  if (lane == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (a.new_k) {  // fused ring write (cache.py:134-135): this CTA alone reads the pending tier
    if (tid < 2 * D / 8) {
      const size_t dst = ((size_t)u * cap + (size_t)((n.total_tokens - 1) % cap)) * D + (tid % (D / 8)) * 8;
      const uint16_t* src = (tid < D / 8 ? a.new_k : a.new_v) + (size_t)u * D + (tid % (D / 8)) * 8;
      *reinterpret_cast<uint4*>((tid < D / 8 ? c.pend_k : c.pend_v) + dst) = *reinterpret_cast<const uint4*>(src);
      asm volatile("fence.proxy.async.global;\n" ::: "memory");  // visible to this CTA's TMA reads
    }
    sync4();
  }
  __syncwarp();

  float o[8][4];
#pragma unroll
  for (int j = 0; j < 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float mrun[2] = {-INFINITY, -INFINITY}, lsum[2] = {0.f, 0.f};
  // ldmatrix lane addressing (row, byte column) for K (non-trans) and V (trans)
  const int k_row = (lane & 7) + ((lane >> 3) & 1) * 8, k_col = (lane >> 4) * 16;
  const int v_row = (lane & 7) + ((lane >> 4) & 1) * 8, v_col = ((lane >> 3) & 1) * 16;
  uint32_t phase = 0;

  // the fp-tier CTAs of a unit (n_fsplits of them) interleave the 16-row tiles warp by warp
  const int f = (int)blockIdx.y - a.n_qsplits;
  for (int t = warp + kAttnWarps * f; t < n_tiles; t += kAttnWarps * a.n_fsplits) {
    const bool is_pool = t < n_pool_t;
    // row validity of this lane's two rows (g, g+8)
    bool valid[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = g + 8 * h;
      if (is_pool) {
        const int slot = 16 * t + r;
        valid[h] = slot < N && c.pool_pos[(size_t)u * N + slot] >= 0;
      } else {
        valid[h] = 16 * (t - n_pool_t) + r < Tp;
      }
    }
    if (lane == 0) {
      const int rows = is_pool ? min(16, N - 16 * t) : min(16, Tp - 16 * (t - n_pool_t));
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(rows * 512)
                   : "memory");
      // ring slot of the tile's first pending row, then consecutive slots (one modulo per tile)
      int slot = is_pool ? 0 : (int)((n.q_tokens + 16 * (t - n_pool_t)) % cap);
      for (int r = 0; r < rows; ++r) {
        size_t off;
        if (is_pool) {
          off = ((size_t)u * N + 16 * t + r) * D;
        } else {
          off = ((size_t)u * cap + (size_t)slot) * D;
          slot = slot + 1 == cap ? 0 : slot + 1;
        }
        tma_row(kr_s + r * kRow, (is_pool ? c.pool_k : c.pend_k) + off, bar);
        tma_row(vr_s + r * kRow, (is_pool ? c.pool_v : c.pend_v) + off, bar);
      }
    }
    mbar_wait(bar, phase);
    phase ^= 1u;

    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint32_t ak[4];
      ldsm_x4(ak, kr_s + k_row * kRow + 32 * j + k_col);
      mma16816(acc, ak[0], ak[1], ak[2], ak[3], qb[j][0], qb[j][1]);
    }
    float sc[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) sc[j] = valid[j >> 1] ? acc[j] * a.scale_log2 : -INFINITY;
    float tmax[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float tm = fmaxf(sc[h], sc[h + 2]);
      tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 4));
      tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 8));
      tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 16));
      tmax[h] = tm;
    }
    const bool need = tmax[0] > mrun[0] + kLazy || tmax[1] > mrun[1] + kLazy;
    if (__any_sync(0xffffffffu, need)) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float mnew = fmaxf(mrun[h], tmax[h]);
        const float corr = mnew == -INFINITY ? 1.f : ex2(mrun[h] - mnew);
        lsum[h] *= corr;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          o[j][h] *= corr;
          o[j][h + 2] *= corr;
        }
        mrun[h] = mnew;
      }
    }
    const float me0 = mrun[0] == -INFINITY ? 0.f : mrun[0];
    const float me1 = mrun[1] == -INFINITY ? 0.f : mrun[1];
    const float p00 = ex2(sc[0] - me0), p01 = ex2(sc[1] - me1);
    const float p10 = ex2(sc[2] - me0), p11 = ex2(sc[3] - me1);
    lsum[0] += p00 + p10;
    lsum[1] += p01 + p11;
    const uint32_t b0 = movm_t(pack_h2(p00, p01));
    const uint32_t b1 = movm_t(pack_h2(p10, p11));
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint32_t av[4];
      ldsm_x4_t(av, vr_s + v_row * kRow + 32 * j + v_col);
      mma16816(o[j], av[0], av[1], av[2], av[3], b0, b1);
    }
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }

#pragma unroll
  for (int h = 0; h < 2; ++h) {
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) lsum[h] += __shfl_xor_sync(0xffffffffu, lsum[h], off);
  }
  if (g == 0) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      sm.mm[warp][2 * tig + h] = mrun[h];
      sm.ll[warp][2 * tig + h] = lsum[h];
    }
  }
  sync4();
  float* accw = reinterpret_cast<float*>(&sm.kr[warp][0][0]);  // [8 heads][128]
#pragma unroll
  for (int j = 0; j < 8; ++j) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      accw[(2 * tig + h) * D + 16 * j + g] = o[j][h];
      accw[(2 * tig + h) * D + 16 * j + 8 + g] = o[j][h + 2];
    }
  }
  sync4();
  for (int i = tid; i < NR * D; i += kAttnThreads) {
    const int r = i / D, col = i % D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kAttnWarps; ++w) M = fmaxf(M, sm.mm[w][r]);
    float Lsum = 0.f, A = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int w = 0; w < kAttnWarps; ++w) {
        if (sm.mm[w][r] == -INFINITY) continue;
        const float f = exp2f(sm.mm[w][r] - M);
        Lsum += sm.ll[w][r] * f;
        A += reinterpret_cast<const float*>(&sm.kr[w][0][0])[r * D + col] * f;
      }
    }
    float* base = a.ws + (((size_t)u * NR + r) * a.n_splits + split) * (D + 2);
    base[2 + col] = A;
    if (col == 0) {
      base[0] = M;
      base[1] = Lsum;
    }
  }
}

template <int NR, int G>
__global__ void __launch_bounds__(kAttnThreads, OTT_MMA_MIN_BLOCKS)
    attend_mma_kernel(const __grid_constant__ AttnArgs a, const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(256) unsigned char smem_raw[];
  allow_dependents();
#ifndef OTT_ABL_TIER  // timing ablation only (results wrong): 1 skip the fp-tier CTAs, 2 skip quantized CTAs
#define OTT_ABL_TIER 0
#endif
  if ((int)blockIdx.y >= a.n_qsplits) {  // full-precision tiers: pool + pending
    if (OTT_ABL_TIER & 1) return;
    const Counts n = counts_of(a);
    if (blockIdx.x == 0 && blockIdx.y == a.n_qsplits && threadIdx.x == 0)  // token counts for the combine's guard
      reinterpret_cast<int64_t*>(a.ws + (size_t)a.c.n_units * NR * a.n_splits * 130)[0] = n.q_tokens;
    fp_body<NR>(a, n, *reinterpret_cast<FpSmem*>(smem_raw));
  } else {
    if (OTT_ABL_TIER & 2) return;
    mma_body<NR, G>(a, counts_of(a), &tmap, *reinterpret_cast<MmaSmem<G>*>(smem_raw));
  }
}

// ============================================================ 4-bit tensor-core path (d = 128, G = 32)
// Same structure as mma_body with 4-bit codes (a record is 5,376 B: 64-byte token rows).
//   * Records arrive through a 128-byte-row tensor map with SWIZZLE_128B (16-byte chunk bits
//     4-6 ^= offset bits 7-9), so ldmatrix over 64-byte token rows is bank-conflict free; the
//     stage slots are 1 KB aligned (6 KB each).
//   * A code word holds channels 8w..8w+7 (nibble i at bits 4i). Nibble k of both halves is
//     moved to mantissa bits 4-7 (k=0: <<4, k=1: in place, k=2: >>4, k=3: >>8; one LOP3 each):
//     K codes become fp16 1 + c/64 (1.0 magic), V codes exact subnormals c * 2^-20. The pair is
//     (channel 8w+k, 8w+k+4); the record's K steps are stored in that order (kpair4_index).
//   * Q.K^T k-step (h, k): logical columns (2t, 2t+1) = channels 64h + 8t + k (+4), columns
//     (2t+8, 2t+9) = 64h + 32 + 8t + k (+4). P.V m-tile (h, k): rows g / g+8 = channels
//     64h + 4g + k / 64h + 32 + 4g + k.
namespace q4 {
constexpr int kRec = 32 * 64 + 32 * 64 + 2 * 2 * 128 + 4 * 128 + 8 * 32;  // 5,376 B
constexpr int kSlot = 6144;                                               // 1 KB aligned slots
constexpr int kStages = 2;
constexpr int kRows = kRec / 128;  // tensor-map rows of 128 B
}  // namespace q4
struct Mma4Smem {
  float4 qt[8][32];  // q (fp32) per lane for the x_min bias: [word slot][lane]
  alignas(1024) uint8_t stage[kAttnWarps][q4::kStages][q4::kSlot];
  alignas(8) uint64_t bar[kAttnWarps][q4::kStages];
  float mm[kAttnWarps][8], ll[kAttnWarps][8];
};
__device__ __forceinline__ uint32_t swz128(uint32_t o) { return o ^ (((o >> 7) & 7u) << 4); }
__device__ __forceinline__ void load_record4(uint32_t dst, const CUtensorMap* map, int64_t rec_index, uint32_t bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(q4::kRec) : "memory");
  tma_tensor_rows(dst, map, (int)(rec_index * q4::kRows), bar);
}
// Tensor maps of the 4/8-bit kernels. Records of G = 32 tokens load as one box (`rec`);
// records of G = 64/128 tokens are consumed 32 tokens at a time, each staged in the G = 32
// record layout from five boxes: the K and V code slices (`rec`, box = one slice), the
// record's K params (`params`, 8 rows) and the two V param slices (`row`, 1 row).
struct VgMaps {
  CUtensorMap rec, params, row;
};
template <int GR, int kCodeRows, int kRecRows32>
__device__ __forceinline__ void load_vgroup(uint32_t dst, const VgMaps* m, const ott_cache_t& c, int u, int vg,
                                            uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
  if (GR == 32) {
    tma_tensor_rows(dst, &m->rec, (int)(((int64_t)u * c.max_groups + vg) * kRecRows32), bar);
    return;
  }
  constexpr int nsub = GR / 32, code_rows = kCodeRows * nsub, rec_rows = 2 * code_rows + 8 + 2 * nsub;
  const int64_t base = ((int64_t)u * c.max_groups + vg / nsub) * rec_rows;
  const int j = vg % nsub;
  tma_tensor_rows(dst, &m->rec, (int)(base + j * kCodeRows), bar);
  tma_tensor_rows(dst + kCodeRows * 128, &m->rec, (int)(base + code_rows + j * kCodeRows), bar);
  tma_tensor_rows(dst + 2 * kCodeRows * 128, &m->params, (int)(base + 2 * code_rows), bar);
  tma_tensor_rows(dst + (2 * kCodeRows + 8) * 128, &m->row, (int)(base + 2 * code_rows + 8 + j), bar);
  tma_tensor_rows(dst + (2 * kCodeRows + 9) * 128, &m->row, (int)(base + 2 * code_rows + 8 + nsub + j), bar);
}

struct Nib {
  uint32_t l4, x, r4, r8;
};
__device__ __forceinline__ Nib nibs(uint32_t w) { return {w << 4, w, w >> 4, w >> 8}; }
template <int K>
__device__ __forceinline__ uint32_t nib_src(const Nib& n) {
  return K == 0 ? n.l4 : (K == 1 ? n.x : (K == 2 ? n.r4 : n.r8));
}
template <int K>
__device__ __forceinline__ uint32_t kq4(const Nib& n, uint32_t magic) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;\n" : "=r"(r) : "r"(nib_src<K>(n)), "n"(0x00F000F0u), "r"(magic));
  return r;
}
template <int K>
__device__ __forceinline__ uint32_t vq4(const Nib& n) {
  return nib_src<K>(n) & 0x00F000F0u;
}

template <int NR, int GR>
__device__ void mma4_body(const AttnArgs& a, const Counts& n, const VgMaps* tmap, Mma4Smem& sm) {
  constexpr int D = 128, G = 32, kMt = 2, kStages = q4::kStages;
  const RecordLayout L(D, G, 4);
  const ott_cache_t& c = a.c;
  const int u = blockIdx.x, split = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tig = lane & 3;
  const uint32_t magic = a.k_magic;
  const int n_groups = (int)(n.q_tokens / G);
  const int per = (n_groups + a.n_qsplits - 1) / a.n_qsplits;
  const int g0 = split * per;
  const int g1 = min(n_groups, g0 + per);
  const int my_n = g1 > g0 + warp ? (g1 - g0 - warp + kAttnWarps - 1) / kAttnWarps : 0;

  // q (fp32) for the bias: slot 2 s + j of lane (head h, t) = channels 8 w + 4 j .. +3 of word
  // w = 32 (s >> 1) + 8 (s & 1)... i.e. words W(s) = {t, 4+t, 8+t, 12+t}[s]
  for (int i = tid; i < 8 * 32; i += kAttnThreads) {
    const int k = i >> 5, ln = i & 31, h = ln >> 2, t4 = ln & 3;
    const int w = 4 * (k >> 1) + t4;  // words t, 4+t, 8+t, 12+t
    const int ch = 8 * w + 4 * (k & 1);
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (h < NR) {
      const uint2 raw = __ldg(reinterpret_cast<const uint2*>(a.q + ((size_t)u * NR + h) * D + ch));
      const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&raw.x));
      const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&raw.y));
      v = make_float4(f0.x, f0.y, f1.x, f1.y);
    }
    sm.qt[k][ln] = v;
  }
  const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&sm.bar[warp][0]);
  const uint32_t stage0 = (uint32_t)__cvta_generic_to_shared(&sm.stage[warp][0][0]);
  if (stage0 & 1023u) __trap();  // SWIZZLE_128B needs 1 KB-aligned stage slots (see swz128)
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kStages; ++s) mbar_init(bar0 + 8 * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
#pragma unroll
    for (int s = 0; s < kStages; ++s)
      if (s < my_n)
        load_vgroup<GR, 16, q4::kRows>(stage0 + s * q4::kSlot, tmap, c, u, g0 + warp + s * kAttnWarps, bar0 + 8 * s,
                                       q4::kRec);
  }
  __syncthreads();

  float o[8][4];
#pragma unroll
  for (int cm = 0; cm < 8; ++cm) o[cm][0] = o[cm][1] = o[cm][2] = o[cm][3] = 0.f;
  float mrun[2] = {-INFINITY, -INFINITY}, lsum[2] = {0.f, 0.f}, vb[2] = {0.f, 0.f};
  const uint32_t* pmask = c.pool_mask + (size_t)u * mask_words_per_unit(c);
  // ldmatrix rows (64-byte token rows): matrix i = lane / 8, row r = lane % 8:
  // i0 tokens 0-7 bytes 0-15, i1 tokens 8-15 bytes 0-15, i2 tokens 0-7 bytes 16-31, i3 tokens 8-15
  // bytes 16-31 (+32 for the second half of the row)
  const uint32_t lm_off = (uint32_t)(((lane & 7) + ((lane >> 3) & 1) * 8) * 64 + (lane >> 4) * 16);
  // q * 64 as fp16 pairs (channels 8w+k, 8w+k+4), words w = {t, 4+t, 8+t, 12+t}[s]
  __half2 q16[4][4];
#pragma unroll
  for (int sw = 0; sw < 4; ++sw)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float4 qa = sm.qt[2 * sw][lane], qb = sm.qt[2 * sw + 1][lane];  // channels 8w..8w+3, 8w+4..8w+7
      const float lo = (k == 0 ? qa.x : k == 1 ? qa.y : k == 2 ? qa.z : qa.w) * 64.f;
      const float hi = (k == 0 ? qb.x : k == 1 ? qb.y : k == 2 ? qb.z : qb.w) * 64.f;
      q16[sw][k] = __floats2half2_rn(lo, hi);
    }
  const float scale4 = a.scale_log2;  // ch = sum q 64 step (1 + c/64) = 64 sum q step + sum q step c
  for (int k = 0; k < my_n; ++k) {
    const int gi = g0 + warp + k * kAttnWarps;
    const uint32_t mword = __ldg(&pmask[gi]);
    const int s = k % kStages;
    mbar_wait(bar0 + 8 * s, (uint32_t)((k / kStages) & 1));
    const uint8_t* rec = &sm.stage[warp][s][0];
    const uint32_t rec_s = stage0 + s * q4::kSlot;
    // K code words: [mt][half h][4] = token g / g+8, words 8h + t and 8h + 4 + t
    uint32_t kw[kMt][2][4];
#pragma unroll
    for (int mt = 0; mt < kMt; ++mt)
#pragma unroll
      for (int h = 0; h < 2; ++h) ldsm_x4(kw[mt][h], rec_s + swz128(L.k_codes() + mt * 16 * 64 + 32 * h + lm_off));
    __syncwarp();
    // bias: sum_c q e over this lane's 32 channels (words t, 4+t, 8+t, 12+t)
    float bias;
    {
      float2 acc2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int w = 4 * (kk >> 1) + tig;
        const float4 ev = *reinterpret_cast<const float4*>(rec + swz128(L.k_e() + 32 * w + 16 * (kk & 1)));
        const float4 qv = sm.qt[kk][lane];
        acc2[(2 * kk) & 3] = __ffma2_rn(make_float2(qv.x, qv.y), make_float2(ev.x, ev.y), acc2[(2 * kk) & 3]);
        acc2[(2 * kk + 1) & 3] = __ffma2_rn(make_float2(qv.z, qv.w), make_float2(ev.z, ev.w), acc2[(2 * kk + 1) & 3]);
      }
      bias = ((acc2[0].x + acc2[0].y) + (acc2[1].x + acc2[1].y)) + ((acc2[2].x + acc2[2].y) + (acc2[3].x + acc2[3].y));
    }
    float ch[kMt][4];
#pragma unroll
    for (int mt = 0; mt < kMt; ++mt) ch[mt][0] = ch[mt][1] = ch[mt][2] = ch[mt][3] = 0.f;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      // q' = q 64 step as exact fp16 hi/lo from the step halves: words 8h + t (b0) and 8h + 4 + t (b1)
      uint32_t bh[2][4], bl[2][4];
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int w = 8 * h + 4 * b + tig;
        const uint4 sh4 = *reinterpret_cast<const uint4*>(rec + swz128(L.k_sh() + 16 * w));
        const uint4 sl4 = *reinterpret_cast<const uint4*>(rec + swz128(L.k_sl() + 16 * w));
        const uint32_t shw[4] = {sh4.x, sh4.y, sh4.z, sh4.w}, slw[4] = {sl4.x, sl4.y, sl4.z, sl4.w};
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const __half2 sh = *reinterpret_cast<const __half2*>(&shw[kk]);
          const __half2 sl = *reinterpret_cast<const __half2*>(&slw[kk]);
          const __half2 qq = q16[2 * h + b][kk];
          const __half2 H = __hmul2(qq, sh);
          const __half2 E = __hfma2(qq, sh, __hneg2(H));
          bh[b][kk] = h2_as_u32(H);
          bl[b][kk] = h2_as_u32(__hfma2(qq, sl, E));
        }
      }
      Nib n0[kMt], n1[kMt], n2[kMt], n3[kMt];
#pragma unroll
      for (int mt = 0; mt < kMt; ++mt) {
        n0[mt] = nibs(kw[mt][h][0]);  // token g, word 8h + t
        n1[mt] = nibs(kw[mt][h][1]);  // token g + 8, word 8h + t
        n2[mt] = nibs(kw[mt][h][2]);  // token g, word 8h + 4 + t
        n3[mt] = nibs(kw[mt][h][3]);  // token g + 8, word 8h + 4 + t
      }
#define OTT_QK4(K)                                                                            \
  {                                                                                           \
    _Pragma("unroll") for (int mt = 0; mt < kMt; ++mt) {                                      \
      const uint32_t a0 = kq4<K>(n0[mt], magic), a1 = kq4<K>(n1[mt], magic);                 \
      const uint32_t a2 = kq4<K>(n2[mt], magic), a3 = kq4<K>(n3[mt], magic);                 \
      mma16816(ch[mt], a0, a1, a2, a3, bh[0][K], bh[1][K]);                                   \
      mma16816(ch[mt], a0, a1, a2, a3, bl[0][K], bl[1][K]);                                   \
    }                                                                                         \
  }
      OTT_QK4(0) OTT_QK4(1) OTT_QK4(2) OTT_QK4(3)
#undef OTT_QK4
    }
    float sc[kMt][4];
    {
      bias += __shfl_xor_sync(0xffffffffu, bias, 1);
      bias += __shfl_xor_sync(0xffffffffu, bias, 2);
      bias *= a.scale_log2;
      const float bias0 = __shfl_sync(0xffffffffu, bias, 8 * tig);      // head 2*tig
      const float bias1 = __shfl_sync(0xffffffffu, bias, 8 * tig + 4);  // head 2*tig+1
#pragma unroll
      for (int mt = 0; mt < kMt; ++mt) {
        sc[mt][0] = fmaf(ch[mt][0], scale4, bias0);
        sc[mt][1] = fmaf(ch[mt][1], scale4, bias1);
        sc[mt][2] = fmaf(ch[mt][2], scale4, bias0);
        sc[mt][3] = fmaf(ch[mt][3], scale4, bias1);
      }
      if (mword) {
#pragma unroll
        for (int mt = 0; mt < kMt; ++mt) {
          if ((mword >> (mt * 16 + g)) & 1u) sc[mt][0] = sc[mt][1] = -INFINITY;
          if ((mword >> (mt * 16 + g + 8)) & 1u) sc[mt][2] = sc[mt][3] = -INFINITY;
        }
      }
    }
    float tmax[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float t = -INFINITY;
#pragma unroll
      for (int mt = 0; mt < kMt; ++mt) t = fmaxf(t, fmaxf(sc[mt][h], sc[mt][h + 2]));
      tmax[h] = t;
    }
    const bool need = tmax[0] > mrun[0] + kLazy || tmax[1] > mrun[1] + kLazy;
    if (__any_sync(0xffffffffu, need)) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float t = tmax[h];
        t = fmaxf(t, __shfl_xor_sync(0xffffffffu, t, 4));
        t = fmaxf(t, __shfl_xor_sync(0xffffffffu, t, 8));
        t = fmaxf(t, __shfl_xor_sync(0xffffffffu, t, 16));
        const float mnew = fmaxf(mrun[h], t);
        const float corr = mnew == -INFINITY ? 1.f : ex2(mrun[h] - mnew);
        lsum[h] *= corr;
        vb[h] *= corr;
#pragma unroll
        for (int cm = 0; cm < 8; ++cm) {
          o[cm][h] *= corr;
          o[cm][h + 2] *= corr;
        }
        mrun[h] = mnew;
      }
    }
    const float me0 = mrun[0] == -INFINITY ? 0.f : mrun[0];
    const float me1 = mrun[1] == -INFINITY ? 0.f : mrun[1];
    // ---- O^T += V^T P' (P' = p step fp16; V codes as subnormals c 2^-20)
#pragma unroll
    for (int mt = 0; mt < kMt; ++mt) {
      const float vs0 = *reinterpret_cast<const float*>(rec + swz128(L.v_step() + 4 * (mt * 16 + g)));
      const float vs1 = *reinterpret_cast<const float*>(rec + swz128(L.v_step() + 4 * (mt * 16 + g + 8)));
      const float ve0 = *reinterpret_cast<const float*>(rec + swz128(L.v_xmin() + 4 * (mt * 16 + g)));
      const float ve1 = *reinterpret_cast<const float*>(rec + swz128(L.v_xmin() + 4 * (mt * 16 + g + 8)));
      const float p00 = ex2(sc[mt][0] - me0), p01 = ex2(sc[mt][1] - me1);
      const float p10 = ex2(sc[mt][2] - me0), p11 = ex2(sc[mt][3] - me1);
      lsum[0] += p00 + p10;
      lsum[1] += p01 + p11;
      vb[0] = fmaf(p00, ve0, fmaf(p10, ve1, vb[0]));
      vb[1] = fmaf(p01, ve0, fmaf(p11, ve1, vb[1]));
      const uint32_t b0 = movm_t(pack_h2(p00 * vs0, p01 * vs0));
      const uint32_t b1 = movm_t(pack_h2(p10 * vs1, p11 * vs1));
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t vr[4];
        ldsm_x4_t(vr, rec_s + swz128(L.v_codes() + mt * 16 * 64 + 32 * h + lm_off));
        const Nib v0 = nibs(vr[0]), v1 = nibs(vr[1]), v2 = nibs(vr[2]), v3 = nibs(vr[3]);
#define OTT_PV4(K) mma16816(o[4 * h + K], vq4<K>(v0), vq4<K>(v2), vq4<K>(v1), vq4<K>(v3), b0, b1);
        OTT_PV4(0) OTT_PV4(1) OTT_PV4(2) OTT_PV4(3)
#undef OTT_PV4
      }
    }
    __syncwarp();
    if (lane == 0) {
      const int ka = k + kStages;
      if (ka < my_n) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        load_vgroup<GR, 16, q4::kRows>(stage0 + s * q4::kSlot, tmap, c, u, g0 + warp + ka * kAttnWarps, bar0 + 8 * s,
                                       q4::kRec);
      }
    }
  }
  // ---- reduce l, vb over the token rows, merge warps, write the partial
#pragma unroll
  for (int h = 0; h < 2; ++h) {
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      lsum[h] += __shfl_xor_sync(0xffffffffu, lsum[h], off);
      vb[h] += __shfl_xor_sync(0xffffffffu, vb[h], off);
    }
  }
  if (g == 0) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      sm.mm[warp][2 * tig + h] = mrun[h];
      sm.ll[warp][2 * tig + h] = lsum[h];
    }
  }
  __syncthreads();  // every warp is past its loop: stage memory is free
  float* accw = reinterpret_cast<float*>(&sm.stage[warp][0][0]);  // [8 heads][128] natural channel order
#pragma unroll
  for (int cm = 0; cm < 8; ++cm) {
    const int chan = 64 * (cm >> 2) + 4 * g + (cm & 3);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      accw[(2 * tig + h) * D + chan] = fmaf(o[cm][h], 1048576.f, vb[h]);  // 2^20
      accw[(2 * tig + h) * D + chan + 32] = fmaf(o[cm][h + 2], 1048576.f, vb[h]);
    }
  }
  __syncthreads();
  for (int i = tid; i < NR * D; i += kAttnThreads) {
    const int r = i / D, col = i % D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kAttnWarps; ++w) M = fmaxf(M, sm.mm[w][r]);
    float Lsum = 0.f, A = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int w = 0; w < kAttnWarps; ++w) {
        if (sm.mm[w][r] == -INFINITY) continue;
        const float f = exp2f(sm.mm[w][r] - M);
        Lsum += sm.ll[w][r] * f;
        A += reinterpret_cast<const float*>(&sm.stage[w][0][0])[r * D + col] * f;
      }
    }
    float* base = a.ws + (((size_t)u * NR + r) * a.n_splits + split) * (D + 2);
    base[2 + col] = A;
    if (col == 0) {
      base[0] = M;
      base[1] = Lsum;
    }
  }
}

template <int NR, int GR>
__global__ void __launch_bounds__(kAttnThreads, 4)
    attend_mma4_kernel(const __grid_constant__ AttnArgs a, const __grid_constant__ VgMaps tmap) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  allow_dependents();
  if ((int)blockIdx.y >= a.n_qsplits) {  // full-precision tiers: pool + pending
    const Counts n = counts_of(a);
    if (blockIdx.x == 0 && blockIdx.y == a.n_qsplits && threadIdx.x == 0)  // token counts for the combine's guard
      reinterpret_cast<int64_t*>(a.ws + (size_t)a.c.n_units * NR * a.n_splits * 130)[0] = n.q_tokens;
    fp_body<NR>(a, n, *reinterpret_cast<FpSmem*>(smem_raw));
  } else {
    mma4_body<NR, GR>(a, counts_of(a), &tmap, *reinterpret_cast<Mma4Smem*>(smem_raw));
  }
}

// ============================================================ 8-bit tensor-core path (d = 128, G = 32)
// As the 4-bit path with byte codes (a record is 9,472 B: 128-byte token rows, SWIZZLE_128B,
// 10 KB stage slots, 2 stages per warp, 2 CTAs per SM). One PRMT builds an fp16 pair from two
// code bytes: K as 1024 + c (with exponent byte 0x64, so u = 1 and e = x_min - 1024 step),
// V as exact subnormals c * 2^-24. K pairs are consecutive channels (c, c+1).
//   * Q.K^T k-step (h, p): logical columns (2t, 2t+1) = channels 32h + 4t + 2p (+1), columns
//     (2t+8, 2t+9) = 32h + 16 + 4t + 2p (+1).
//   * P.V m-tile (h, e): rows g / g+8 = channels 32h + 2g + e / 32h + 16 + 2g + e.
namespace q8 {
constexpr int kRec = 32 * 128 * 2 + 2 * 2 * 128 + 4 * 128 + 8 * 32;  // 9,472 B
constexpr int kSlot = 10240;
constexpr int kStages = 2;
constexpr int kRows = kRec / 128;  // 74
}  // namespace q8
struct Mma8Smem {
  float4 qt[8][32];
  alignas(1024) uint8_t stage[kAttnWarps][q8::kStages][q8::kSlot];
  alignas(8) uint64_t bar[kAttnWarps][q8::kStages];
  float mm[kAttnWarps][8], ll[kAttnWarps][8];
};
__device__ __forceinline__ void load_record8(uint32_t dst, const CUtensorMap* map, int64_t rec_index, uint32_t bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(q8::kRec) : "memory");
  tma_tensor_rows(dst, map, (int)(rec_index * q8::kRows), bar);
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;\n" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

template <int NR, int GR>
__device__ void mma8_body(const AttnArgs& a, const Counts& n, const VgMaps* tmap, Mma8Smem& sm) {
  constexpr int D = 128, G = 32, kMt = 2, kStages = q8::kStages;
  const RecordLayout L(D, G, 8);
  const ott_cache_t& c = a.c;
  const int u = blockIdx.x, split = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tig = lane & 3;
  const uint32_t kmagic = 0x64646464u;  // fp16 exponent byte of 1024
  const int n_groups = (int)(n.q_tokens / G);
  const int per = (n_groups + a.n_qsplits - 1) / a.n_qsplits;
  const int g0 = split * per;
  const int g1 = min(n_groups, g0 + per);
  const int my_n = g1 > g0 + warp ? (g1 - g0 - warp + kAttnWarps - 1) / kAttnWarps : 0;

  // q (fp32) for the bias: slot s of lane (head h, t) = channels 32 (s >> 1) + 16 (s & 1) + 4t .. +3
  for (int i = tid; i < 8 * 32; i += kAttnThreads) {
    const int k = i >> 5, ln = i & 31, h = ln >> 2, t4 = ln & 3;
    const int ch = 32 * (k >> 1) + 16 * (k & 1) + 4 * t4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (h < NR) {
      const uint2 raw = __ldg(reinterpret_cast<const uint2*>(a.q + ((size_t)u * NR + h) * D + ch));
      const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&raw.x));
      const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&raw.y));
      v = make_float4(f0.x, f0.y, f1.x, f1.y);
    }
    sm.qt[k][ln] = v;
  }
  const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&sm.bar[warp][0]);
  const uint32_t stage0 = (uint32_t)__cvta_generic_to_shared(&sm.stage[warp][0][0]);
  if (stage0 & 1023u) __trap();  // SWIZZLE_128B needs 1 KB-aligned stage slots
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kStages; ++s) mbar_init(bar0 + 8 * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
#pragma unroll
    for (int s = 0; s < kStages; ++s)
      if (s < my_n)
        load_vgroup<GR, 32, q8::kRows>(stage0 + s * q8::kSlot, tmap, c, u, g0 + warp + s * kAttnWarps, bar0 + 8 * s,
                                       q8::kRec);
  }
  __syncthreads();

  float o[8][4];
#pragma unroll
  for (int cm = 0; cm < 8; ++cm) o[cm][0] = o[cm][1] = o[cm][2] = o[cm][3] = 0.f;
  float mrun[2] = {-INFINITY, -INFINITY}, lsum[2] = {0.f, 0.f}, vb[2] = {0.f, 0.f};
  const uint32_t* pmask = c.pool_mask + (size_t)u * mask_words_per_unit(c);
  // ldmatrix rows over 128-byte token rows (+32 h for row quarter h)
  const uint32_t lm_off = (uint32_t)(((lane & 7) + ((lane >> 3) & 1) * 8) * 128 + (lane >> 4) * 16);
  // q as fp16 pairs (c, c+1): [h][b][p] = channels 32h + 16b + 4t + 2p (+1)
  __half2 q16[4][2][2];
#pragma unroll
  for (int h = 0; h < 4; ++h)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const float4 qv = sm.qt[2 * h + b][lane];
      q16[h][b][0] = __floats2half2_rn(qv.x, qv.y);
      q16[h][b][1] = __floats2half2_rn(qv.z, qv.w);
    }
  const float scale4 = a.scale_log2;
  for (int k = 0; k < my_n; ++k) {
    const int gi = g0 + warp + k * kAttnWarps;
    const uint32_t mword = __ldg(&pmask[gi]);
    const int s = k % kStages;
    mbar_wait(bar0 + 8 * s, (uint32_t)((k / kStages) & 1));
    const uint8_t* rec = &sm.stage[warp][s][0];
    const uint32_t rec_s = stage0 + s * q8::kSlot;
    float bias;
    {
      float2 acc2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int ch = 32 * (kk >> 1) + 16 * (kk & 1) + 4 * tig;
        const float4 ev = *reinterpret_cast<const float4*>(rec + swz128(L.k_e() + 4 * ch));
        const float4 qv = sm.qt[kk][lane];
        acc2[(2 * kk) & 3] = __ffma2_rn(make_float2(qv.x, qv.y), make_float2(ev.x, ev.y), acc2[(2 * kk) & 3]);
        acc2[(2 * kk + 1) & 3] = __ffma2_rn(make_float2(qv.z, qv.w), make_float2(ev.z, ev.w), acc2[(2 * kk + 1) & 3]);
      }
      bias = ((acc2[0].x + acc2[0].y) + (acc2[1].x + acc2[1].y)) + ((acc2[2].x + acc2[2].y) + (acc2[3].x + acc2[3].y));
    }
    float ch[kMt][4];
#pragma unroll
    for (int mt = 0; mt < kMt; ++mt) ch[mt][0] = ch[mt][1] = ch[mt][2] = ch[mt][3] = 0.f;
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      // K code words: token g / g+8, channels 32h + 4t.. (r0, r1) and 32h + 16 + 4t.. (r2, r3)
      uint32_t kw[kMt][4];
#pragma unroll
      for (int mt = 0; mt < kMt; ++mt) ldsm_x4(kw[mt], rec_s + swz128(L.k_codes() + mt * 16 * 128 + 32 * h + lm_off));
      // q' = q step (exact fp16 hi/lo): pairs (c, c+1) for c = 32h + 16b + 4t + 2p
      uint32_t bh[2][2], bl[2][2];
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int c0 = 32 * h + 16 * b + 4 * tig;
        const uint2 sh2 = *reinterpret_cast<const uint2*>(rec + swz128(L.k_sh() + 2 * c0));
        const uint2 sl2 = *reinterpret_cast<const uint2*>(rec + swz128(L.k_sl() + 2 * c0));
        const uint32_t shw[2] = {sh2.x, sh2.y}, slw[2] = {sl2.x, sl2.y};
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          const __half2 sh = *reinterpret_cast<const __half2*>(&shw[p]);
          const __half2 sl = *reinterpret_cast<const __half2*>(&slw[p]);
          const __half2 qq = q16[h][b][p];
          const __half2 H = __hmul2(qq, sh);
          const __half2 E = __hfma2(qq, sh, __hneg2(H));
          bh[b][p] = h2_as_u32(H);
          bl[b][p] = h2_as_u32(__hfma2(qq, sl, E));
        }
      }
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const uint32_t sel = p == 0 ? 0x5140u : 0x5342u;  // bytes (2p, magic, 2p+1, magic)
#pragma unroll
        for (int mt = 0; mt < kMt; ++mt) {
          const uint32_t a0 = prmt(kw[mt][0], kmagic, sel), a1 = prmt(kw[mt][1], kmagic, sel);
          const uint32_t a2 = prmt(kw[mt][2], kmagic, sel), a3 = prmt(kw[mt][3], kmagic, sel);
          mma16816(ch[mt], a0, a1, a2, a3, bh[0][p], bh[1][p]);
          mma16816(ch[mt], a0, a1, a2, a3, bl[0][p], bl[1][p]);
        }
      }
    }
    float sc[kMt][4];
    {
      bias += __shfl_xor_sync(0xffffffffu, bias, 1);
      bias += __shfl_xor_sync(0xffffffffu, bias, 2);
      bias *= a.scale_log2;
      const float bias0 = __shfl_sync(0xffffffffu, bias, 8 * tig);
      const float bias1 = __shfl_sync(0xffffffffu, bias, 8 * tig + 4);
#pragma unroll
      for (int mt = 0; mt < kMt; ++mt) {
        sc[mt][0] = fmaf(ch[mt][0], scale4, bias0);
        sc[mt][1] = fmaf(ch[mt][1], scale4, bias1);
        sc[mt][2] = fmaf(ch[mt][2], scale4, bias0);
        sc[mt][3] = fmaf(ch[mt][3], scale4, bias1);
      }
      if (mword) {
#pragma unroll
        for (int mt = 0; mt < kMt; ++mt) {
          if ((mword >> (mt * 16 + g)) & 1u) sc[mt][0] = sc[mt][1] = -INFINITY;
          if ((mword >> (mt * 16 + g + 8)) & 1u) sc[mt][2] = sc[mt][3] = -INFINITY;
        }
      }
    }
    float tmax[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float t = -INFINITY;
#pragma unroll
      for (int mt = 0; mt < kMt; ++mt) t = fmaxf(t, fmaxf(sc[mt][h], sc[mt][h + 2]));
      tmax[h] = t;
    }
    const bool need = tmax[0] > mrun[0] + kLazy || tmax[1] > mrun[1] + kLazy;
    if (__any_sync(0xffffffffu, need)) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float t = tmax[h];
        t = fmaxf(t, __shfl_xor_sync(0xffffffffu, t, 4));
        t = fmaxf(t, __shfl_xor_sync(0xffffffffu, t, 8));
        t = fmaxf(t, __shfl_xor_sync(0xffffffffu, t, 16));
        const float mnew = fmaxf(mrun[h], t);
        const float corr = mnew == -INFINITY ? 1.f : ex2(mrun[h] - mnew);
        lsum[h] *= corr;
        vb[h] *= corr;
#pragma unroll
        for (int cm = 0; cm < 8; ++cm) {
          o[cm][h] *= corr;
          o[cm][h + 2] *= corr;
        }
        mrun[h] = mnew;
      }
    }
    const float me0 = mrun[0] == -INFINITY ? 0.f : mrun[0];
    const float me1 = mrun[1] == -INFINITY ? 0.f : mrun[1];
    // ---- O^T += V^T P' (P' = p step fp16; V codes as subnormals c 2^-24)
#pragma unroll
    for (int mt = 0; mt < kMt; ++mt) {
      const float vs0 = *reinterpret_cast<const float*>(rec + swz128(L.v_step() + 4 * (mt * 16 + g)));
      const float vs1 = *reinterpret_cast<const float*>(rec + swz128(L.v_step() + 4 * (mt * 16 + g + 8)));
      const float ve0 = *reinterpret_cast<const float*>(rec + swz128(L.v_xmin() + 4 * (mt * 16 + g)));
      const float ve1 = *reinterpret_cast<const float*>(rec + swz128(L.v_xmin() + 4 * (mt * 16 + g + 8)));
      const float p00 = ex2(sc[mt][0] - me0), p01 = ex2(sc[mt][1] - me1);
      const float p10 = ex2(sc[mt][2] - me0), p11 = ex2(sc[mt][3] - me1);
      lsum[0] += p00 + p10;
      lsum[1] += p01 + p11;
      vb[0] = fmaf(p00, ve0, fmaf(p10, ve1, vb[0]));
      vb[1] = fmaf(p01, ve0, fmaf(p11, ve1, vb[1]));
      const uint32_t b0 = movm_t(pack_h2(p00 * vs0, p01 * vs0));
      const uint32_t b1 = movm_t(pack_h2(p10 * vs1, p11 * vs1));
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        uint32_t vr[4];
        ldsm_x4_t(vr, rec_s + swz128(L.v_codes() + mt * 16 * 128 + 32 * h + lm_off));
        // vr: (token 2t, 2t+1) x 16-bit unit = channels (c, c+1); e picks the channel
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const uint32_t sel = e == 0 ? 0x4240u : 0x4341u;  // bytes (e, zero, 2+e, zero)
          mma16816(o[2 * h + e], prmt(vr[0], 0u, sel), prmt(vr[2], 0u, sel), prmt(vr[1], 0u, sel),
                   prmt(vr[3], 0u, sel), b0, b1);
        }
      }
    }
    __syncwarp();
    if (lane == 0) {
      const int ka = k + kStages;
      if (ka < my_n) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        load_vgroup<GR, 32, q8::kRows>(stage0 + s * q8::kSlot, tmap, c, u, g0 + warp + ka * kAttnWarps, bar0 + 8 * s,
                                       q8::kRec);
      }
    }
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      lsum[h] += __shfl_xor_sync(0xffffffffu, lsum[h], off);
      vb[h] += __shfl_xor_sync(0xffffffffu, vb[h], off);
    }
  }
  if (g == 0) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      sm.mm[warp][2 * tig + h] = mrun[h];
      sm.ll[warp][2 * tig + h] = lsum[h];
    }
  }
  __syncthreads();
  float* accw = reinterpret_cast<float*>(&sm.stage[warp][0][0]);
#pragma unroll
  for (int cm = 0; cm < 8; ++cm) {
    const int chan = 32 * (cm >> 1) + 2 * g + (cm & 1);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      accw[(2 * tig + h) * D + chan] = fmaf(o[cm][h], 16777216.f, vb[h]);  // 2^24
      accw[(2 * tig + h) * D + chan + 16] = fmaf(o[cm][h + 2], 16777216.f, vb[h]);
    }
  }
  __syncthreads();
  for (int i = tid; i < NR * D; i += kAttnThreads) {
    const int r = i / D, col = i % D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kAttnWarps; ++w) M = fmaxf(M, sm.mm[w][r]);
    float Lsum = 0.f, A = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int w = 0; w < kAttnWarps; ++w) {
        if (sm.mm[w][r] == -INFINITY) continue;
        const float f = exp2f(sm.mm[w][r] - M);
        Lsum += sm.ll[w][r] * f;
        A += reinterpret_cast<const float*>(&sm.stage[w][0][0])[r * D + col] * f;
      }
    }
    float* base = a.ws + (((size_t)u * NR + r) * a.n_splits + split) * (D + 2);
    base[2 + col] = A;
    if (col == 0) {
      base[0] = M;
      base[1] = Lsum;
    }
  }
}

template <int NR, int GR>
__global__ void __launch_bounds__(kAttnThreads, 2)
    attend_mma8_kernel(const __grid_constant__ AttnArgs a, const __grid_constant__ VgMaps tmap) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  allow_dependents();
  if ((int)blockIdx.y >= a.n_qsplits) {  // full-precision tiers: pool + pending
    const Counts n = counts_of(a);
    if (blockIdx.x == 0 && blockIdx.y == a.n_qsplits && threadIdx.x == 0)  // token counts for the combine's guard
      reinterpret_cast<int64_t*>(a.ws + (size_t)a.c.n_units * NR * a.n_splits * 130)[0] = n.q_tokens;
    fp_body<NR>(a, n, *reinterpret_cast<FpSmem*>(smem_raw));
  } else {
    mma8_body<NR, GR>(a, counts_of(a), &tmap, *reinterpret_cast<Mma8Smem*>(smem_raw));
  }
}

// ============================================================ tcgen05 path (d = 128, G = 32)
// Q K^T on the 5th-generation tensor cores, P V on the warp-level path.
//
// CTA = 4 compute warps + 1 MMA-issuer warp. A 128-token chunk is 4 consecutive
// groups, one per compute warp. Per chunk:
//   * each compute warp (thread = token) unpacks its group's K codes into fp16
//     (1 + c 2^(2P-10), one LOP3 per pair) and stores the 32 x 128 tile into its
//     32 TMEM lanes (tcgen05.st, A operand of the MMA);
//   * lane (head pair, code word) forms q' = q u step as an exact fp16 hi/lo split
//     from the record's pair-ordered fp16 step halves: hi = q*sh, err = fma(q, sh,
//     -hi) (exact), lo = fma(q, sl, err); rows 16w+h (hi) and 16w+8+h (lo) of the
//     shared-memory B operand (K-major, canonical no-swizzle layout);
//   * the issuer runs 8 tcgen05.mma kind::f16 (M=128 tokens, N=64, K=16) into a
//     TMEM accumulator; only the diagonal 32x16 blocks are used;
//   * while that runs the warps finish the previous chunk: tcgen05.ld of their
//     logits (thread = token, 8 heads), lazily rescaled online softmax, P' = 4 p
//     step to shared memory, and V^T P' with mma.sync m16n8k16 on the V codes
//     (exact fp16 subnormals), accumulating in registers per warp.
// logit = scale * (4 S + sum_c q_c e_c), e = x_min - 4 u step (record encoding).
namespace tc5 {
constexpr int kCW = 4;                       // compute warps
constexpr int kThreads = 32 * (kCW + 1);     // + MMA issuer
constexpr int kStages = 6;                   // record stages per compute warp (2 in use, 4 in flight)
constexpr int kRec = 3328;                   // record bytes at d = 128, G = 32
constexpr uint32_t kLBO = 128, kSBO = 16 * 128;  // B operand core-matrix strides (bytes)
constexpr uint32_t kCols = 128;              // TMEM: A at 0 (f16 pairs), D at 64 (f32)
constexpr uint32_t kIdesc = (1u << 4)        // D f32, A/B f16, both K-major
                            | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}  // namespace tc5

#ifndef OTT_TC5_MIN_BLOCKS
#define OTT_TC5_MIN_BLOCKS 2
#endif
#ifndef OTT_TC5_ABL  // timing ablations only (results wrong): 1 no softmax/PV, 2 no q'/bias, 4 no K unpack
#define OTT_TC5_ABL 0
#endif

struct Tc5Smem {
  alignas(256) uint8_t stage[tc5::kCW][tc5::kStages][tc5::kRec];
  alignas(128) uint8_t b1[64 * 128 * 2];       // q' hi/lo rows, K-major canonical
  alignas(16) uint16_t pp[tc5::kCW][32][8];    // P' [token][head] per warp
  alignas(16) float4 qt[8][32];                // q (fp32) per lane (head lane%8, channels 32(lane/8) + 4k..)
  alignas(16) float bias[tc5::kCW][2][8];      // scale * sum_c q e per (warp, chunk parity, head)
  float mm[tc5::kCW][8], ll[tc5::kCW][8];
  alignas(8) uint64_t rbar[tc5::kCW][tc5::kStages];
  alignas(8) uint64_t qk_ready, qk_done;
  uint32_t tmem_base;
};

__device__ __forceinline__ uint64_t tc5_bdesc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(tc5::kLBO >> 4) << 16) |
         ((uint64_t)(tc5::kSBO >> 4) << 32) | (1ull << 46);
}
__device__ __forceinline__ void tmem_st64(uint32_t taddr, const uint32_t (&r)[64]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x64.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,"
      "%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63,%64};\n" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]), "r"(r[32]), "r"(r[33]), "r"(r[34]), "r"(r[35]), "r"(r[36]),
      "r"(r[37]), "r"(r[38]), "r"(r[39]), "r"(r[40]), "r"(r[41]), "r"(r[42]), "r"(r[43]), "r"(r[44]), "r"(r[45]),
      "r"(r[46]), "r"(r[47]), "r"(r[48]), "r"(r[49]), "r"(r[50]), "r"(r[51]), "r"(r[52]), "r"(r[53]), "r"(r[54]),
      "r"(r[55]), "r"(r[56]), "r"(r[57]), "r"(r[58]), "r"(r[59]), "r"(r[60]), "r"(r[61]), "r"(r[62]), "r"(r[63])
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
template <int I>
__device__ __forceinline__ float pick4(const float (&v)[8], int tig) {  // v[2 tig + I]
  return tig == 0 ? v[I] : (tig == 1 ? v[2 + I] : (tig == 2 ? v[4 + I] : v[6 + I]));
}

// K side of chunk j for compute warp w: A tile into TMEM, q' rows into B, bias.
template <int NR>
__device__ __forceinline__ void tc5_kstage(Tc5Smem& sm, int w, int lane, const uint8_t* rec, uint32_t a_lane,
                                           uint8_t* b1, const __half2 (&q16)[2][8], uint32_t magic, float scale,
                                           int slot) {
  const RecordLayout L(128, 32);
  if (!(OTT_TC5_ABL & 4)) {  // A row = token `lane`: 8 code words -> 64 fp16 pairs
    const uint4 c0 = *reinterpret_cast<const uint4*>(rec + swz(L.k_codes() + lane * 32));
    const uint4 c1 = *reinterpret_cast<const uint4*>(rec + swz(L.k_codes() + lane * 32 + 16));
    const uint32_t wd[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
    uint32_t r[64];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const Shifted sft = shifted(wd[j]);
      r[8 * j + 0] = kq<0>(sft, magic);
      r[8 * j + 1] = kq<1>(sft, magic);
      r[8 * j + 2] = kq<2>(sft, magic);
      r[8 * j + 3] = kq<3>(sft, magic);
      r[8 * j + 4] = kq<4>(sft, magic);
      r[8 * j + 5] = kq<5>(sft, magic);
      r[8 * j + 6] = kq<6>(sft, magic);
      r[8 * j + 7] = kq<7>(sft, magic);
    }
    tmem_st64(a_lane, r);
  }
  // q' rows: lane = (head h = lane % 8, word pair e4 = lane / 8: code words 2e4, 2e4+1 =
  // channels 32e4 .. 32e4+31). Lanes 8k..8k+7 write rows 0..7 of one core matrix:
  // 128 contiguous bytes per store phase, bank-conflict free.
  const int h = lane & 7, e4 = lane >> 3;
  float part = 0.f;
  if (h < NR && !(OTT_TC5_ABL & 2)) {
    float acc[4] = {0.f, 0.f, 0.f, 0.f};  // sum_c q_c e_c, 4 independent chains
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float4 ev = *reinterpret_cast<const float4*>(rec + swz(L.k_e() + 128 * e4 + 16 * k));
      const float4 qv = sm.qt[k][lane];
      acc[0] = fmaf(qv.x, ev.x, acc[0]);
      acc[1] = fmaf(qv.y, ev.y, acc[1]);
      acc[2] = fmaf(qv.z, ev.z, acc[2]);
      acc[3] = fmaf(qv.w, ev.w, acc[3]);
    }
    part = (acc[0] + acc[1]) + (acc[2] + acc[3]);
#pragma unroll
    for (int w2 = 0; w2 < 2; ++w2) {
      const int wd = 2 * e4 + w2;  // code word: channels 16 wd .. 16 wd + 15
      const uint4 h0 = *reinterpret_cast<const uint4*>(rec + swz(L.k_sh() + 32 * wd));
      const uint4 h1 = *reinterpret_cast<const uint4*>(rec + swz(L.k_sh() + 32 * wd + 16));
      const uint4 l0 = *reinterpret_cast<const uint4*>(rec + swz(L.k_sl() + 32 * wd));
      const uint4 l1 = *reinterpret_cast<const uint4*>(rec + swz(L.k_sl() + 32 * wd + 16));
      const uint32_t shw[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
      const uint32_t slw[8] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
      uint32_t hi[8], lo[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const __half2 sh = *reinterpret_cast<const __half2*>(&shw[m]);
        const __half2 sl = *reinterpret_cast<const __half2*>(&slw[m]);
        const __half2 H = __hmul2(q16[w2][m], sh);
        const __half2 E = __hfma2(q16[w2][m], sh, __hneg2(H));  // exact rounding error of H
        hi[m] = h2_as_u32(H);
        lo[m] = h2_as_u32(__hfma2(q16[w2][m], sl, E));
      }
      uint8_t* bh = b1 + (2 * w) * tc5::kSBO + (2 * wd) * tc5::kLBO + h * 16;
      uint8_t* bl = bh + tc5::kSBO;
      *reinterpret_cast<uint4*>(bh) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<uint4*>(bh + tc5::kLBO) = make_uint4(hi[4], hi[5], hi[6], hi[7]);
      *reinterpret_cast<uint4*>(bl) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
      *reinterpret_cast<uint4*>(bl + tc5::kLBO) = make_uint4(lo[4], lo[5], lo[6], lo[7]);
    }
  }
  // reduce over the 4 word pairs (all lanes take part; idle heads carry 0)
  part += __shfl_xor_sync(0xffffffffu, part, 8);
  part += __shfl_xor_sync(0xffffffffu, part, 16);
  if (e4 == 0 && h < NR) sm.bias[w][slot][h] = part * scale;
}

template <int NR>
__device__ void tc5_body(const AttnArgs& a, const Counts& n, const CUtensorMap* tmap, Tc5Smem& sm) {
  constexpr int D = 128, G = 32, kS = tc5::kStages;
  const RecordLayout L(D, G);
  const ott_cache_t& c = a.c;
  const int u = blockIdx.x, split = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tig = lane & 3;
  const int n_groups = (int)(n.q_tokens / G);
  const int per = (((n_groups + a.n_qsplits - 1) / a.n_qsplits) + 3) & ~3;  // whole chunks per split
  const int g0 = min(n_groups, split * per);
  const int g1 = min(n_groups, g0 + per);
  const int n_chunks = (g1 - g0 + 3) / 4;
  const int64_t unit_rec = (int64_t)u * c.max_groups;

  const uint32_t qk_ready = (uint32_t)__cvta_generic_to_shared(&sm.qk_ready);
  const uint32_t qk_done = (uint32_t)__cvta_generic_to_shared(&sm.qk_done);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&sm.tmem_base)),
                 "n"(tc5::kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int w = 0; w < tc5::kCW; ++w)
      for (int s = 0; s < kS; ++s) mbar_init((uint32_t)__cvta_generic_to_shared(&sm.rbar[w][s]), 1);
    mbar_init(qk_ready, tc5::kCW);
    mbar_init(qk_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int i = tid; i < 8 * 32; i += tc5::kThreads) {  // q table: [k][lane] = q[lane % 8][32 (lane / 8) + 4k ..]
    const int k = i >> 5, ln = i & 31, h = ln & 7;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (h < NR) {
      const uint2 raw = __ldg(reinterpret_cast<const uint2*>(a.q + ((size_t)u * NR + h) * D + 32 * (ln >> 3) + 4 * k));
      const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&raw.x));
      const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&raw.y));
      v = make_float4(f0.x, f0.y, f1.x, f1.y);
    }
    sm.qt[k][ln] = v;
  }
  for (int i = tid; i < 64 * 128 * 2 / 16; i += tc5::kThreads)
    reinterpret_cast<uint4*>(sm.b1)[i] = make_uint4(0u, 0u, 0u, 0u);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = sm.tmem_base;
  const uint32_t a_tm = tmem, d_tm = tmem + 64;

  float o[8][4];
#pragma unroll
  for (int cm = 0; cm < 8; ++cm) o[cm][0] = o[cm][1] = o[cm][2] = o[cm][3] = 0.f;
  float m[8], l[8], vb[8];
#pragma unroll
  for (int h = 0; h < 8; ++h) {
    m[h] = -INFINITY;
    l[h] = 0.f;
    vb[h] = 0.f;
  }

  if (warp == tc5::kCW) {
    // ---------------- MMA issuer
    const uint32_t b_s = (uint32_t)__cvta_generic_to_shared(sm.b1);
    const uint32_t a_b = a_tm, d_b = d_tm;
    for (int i = 0; i < n_chunks; ++i) {
      mbar_wait(qk_ready, (uint32_t)(i & 1));
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      if (lane == 0) {
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          const uint64_t bd = tc5_bdesc(b_s + s * 2 * tc5::kLBO);
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_b),
              "r"(a_b + 8 * s), "l"(bd), "r"(tc5::kIdesc), "r"(s)
              : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(qk_done)
                     : "memory");
      }
      __syncwarp();
    }
  } else {
    // ---------------- compute warps
    const int w = warp;
    const uint32_t rbar0 = (uint32_t)__cvta_generic_to_shared(&sm.rbar[w][0]);
    const uint32_t stage0 = (uint32_t)__cvta_generic_to_shared(&sm.stage[w][0][0]);
    auto group_of = [&](int j) { return g0 + 4 * j + w; };
    if (lane == 0) {
#pragma unroll
      for (int s = 0; s < kS; ++s)
        if (s < n_chunks && group_of(s) < g1)
          load_record<G>(stage0 + s * tc5::kRec, tmap, unit_rec + group_of(s), rbar0 + 8 * s);
    }
    const uint32_t magic = a.k_magic;
    const float scale = a.scale_log2, scale4 = 4.f * a.scale_log2;
    // q * u(m) as fp16 pairs (channels 16e+m, 16e+m+8) for heads 2hp, 2hp+1
    // q * u(m) as fp16 pairs (channels 16wd+m, 16wd+m+8) of head lane % 8, words wd = 2e4 + w2
    __half2 q16[2][8];
#pragma unroll
    for (int w2 = 0; w2 < 2; ++w2)
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        // channel 32e4 + 16w2 + m lives in table entry k = 4w2 + m/4, component m%4
        const float4 qa = sm.qt[4 * w2 + m / 4][lane];
        const float4 qb = sm.qt[4 * w2 + 2 + m / 4][lane];
        const float lo = (m % 4 == 0 ? qa.x : m % 4 == 1 ? qa.y : m % 4 == 2 ? qa.z : qa.w) * kpair_u(m);
        const float hi = (m % 4 == 0 ? qb.x : m % 4 == 1 ? qb.y : m % 4 == 2 ? qb.z : qb.w) * kpair_u(m);
        q16[w2][m] = __floats2half2_rn(lo, hi);
      }
    const uint32_t a_lane = a_tm + ((uint32_t)(32 * w) << 16);
    const uint32_t d_lane = d_tm + ((uint32_t)(32 * w) << 16) + 16 * w;
    const uint32_t pp_s = (uint32_t)__cvta_generic_to_shared(&sm.pp[w][0][0]);
    const uint32_t lm_off = (uint32_t)(((lane & 7) + ((lane >> 3) & 1) * 8) * 32 + (lane >> 4) * 16);
    const uint32_t* pmask = c.pool_mask + (size_t)u * mask_words_per_unit(c);

    auto kstage = [&](int j) {
      const int gj = group_of(j);
      if (gj < g1) {
        mbar_wait(rbar0 + 8 * (j % kS), (uint32_t)((j / kS) & 1));
        tc5_kstage<NR>(sm, w, lane, &sm.stage[w][j % kS][0], a_lane, sm.b1, q16, magic, scale, j & 1);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(qk_ready);
    };
    if (n_chunks > 0) kstage(0);

    for (int i = 0; i < n_chunks; ++i) {
      // ---- logits of chunk i (this warp's 32 tokens x 16 columns: hi heads, lo heads)
      mbar_wait(qk_done, (uint32_t)(i & 1));
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      uint32_t sv[16];
      tmem_ld16(d_lane, sv);
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      // ---- K side of chunk i + 1 (the MMA of chunk i is complete and its logits are
      // read); the MMA of chunk i + 1 then runs under this chunk's softmax and P V
      if (i + 1 < n_chunks) kstage(i + 1);

      const int gi = group_of(i);
      if (gi < g1 && !(OTT_TC5_ABL & 1)) {
        const int st = i % kS;
        const uint8_t* rec = &sm.stage[w][st][0];
        const uint32_t rec_s = stage0 + st * tc5::kRec;
        const float4 b0 = *reinterpret_cast<const float4*>(&sm.bias[w][i & 1][0]);
        const float4 b1 = *reinterpret_cast<const float4*>(&sm.bias[w][i & 1][4]);
        const float bias[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
        const bool pooled = (__ldg(&pmask[gi]) >> lane) & 1u;
        float s[8];
#pragma unroll
        for (int h = 0; h < 8; ++h)
          s[h] = (h < NR && !pooled)
                     ? fmaf(__uint_as_float(sv[h]), scale4, fmaf(__uint_as_float(sv[8 + h]), scale4, bias[h]))
                     : -INFINITY;
        // lazily rescaled online softmax: the warp's running max moves only when a
        // logit exceeds it by kLazy (p <= 2^kLazy keeps P' = 4 p step in fp16 range)
        float dmax = -INFINITY;
#pragma unroll
        for (int h = 0; h < NR; ++h) dmax = fmaxf(dmax, s[h] - m[h]);
        if (__any_sync(0xffffffffu, dmax > kLazy || m[0] == -INFINITY)) {
          float corr[8];
#pragma unroll
          for (int h = 0; h < 8; ++h) {
            corr[h] = 1.f;
            if (h < NR) {
              const float t = warp_max(s[h]);
              const float mnew = fmaxf(m[h], t);
              corr[h] = mnew == -INFINITY ? 1.f : ex2(m[h] - mnew);
              m[h] = mnew;
              l[h] *= corr[h];
              vb[h] *= corr[h];
            }
          }
          const float c0 = pick4<0>(corr, tig), c1 = pick4<1>(corr, tig);
#pragma unroll
          for (int cm = 0; cm < 8; ++cm) {
            o[cm][0] *= c0;
            o[cm][1] *= c1;
            o[cm][2] *= c0;
            o[cm][3] *= c1;
          }
        }
        float me[8];
#pragma unroll
        for (int h = 0; h < 8; ++h) me[h] = m[h] == -INFINITY ? 0.f : m[h];
        const float vs = *reinterpret_cast<const float*>(rec + swz(L.v_step() + 4 * lane));
        const float vx = *reinterpret_cast<const float*>(rec + swz(L.v_xmin() + 4 * lane));
        const float f = 4.f * vs;
        float pq[8];
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          pq[h] = 0.f;
          if (h < NR) {
            const float p = ex2(s[h] - me[h]);
            l[h] += p;
            vb[h] = fmaf(p, vx, vb[h]);
            pq[h] = p * f;
          }
        }
        *reinterpret_cast<uint4*>(&sm.pp[w][lane][0]) =
            make_uint4(pack_h2(pq[0], pq[1]), pack_h2(pq[2], pq[3]), pack_h2(pq[4], pq[5]), pack_h2(pq[6], pq[7]));
        __syncwarp();
        uint32_t bq[4];
        ldsm_x4_t(bq, pp_s + lane * 16);
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const uint32_t bb0 = bq[2 * mt], bb1 = bq[2 * mt + 1];
          uint32_t vr[4];
          ldsm_x4_t(vr, rec_s + swz(L.v_codes() + mt * 16 * 32 + lm_off));
          const Shifted v0 = shifted(vr[0]), v1 = shifted(vr[1]), v2 = shifted(vr[2]), v3 = shifted(vr[3]);
#define OTT_PV5(CM) mma16816(o[CM], vq<CM>(v0), vq<CM>(v2), vq<CM>(v1), vq<CM>(v3), bb0, bb1);
          OTT_PV5(0) OTT_PV5(1) OTT_PV5(2) OTT_PV5(3) OTT_PV5(4) OTT_PV5(5) OTT_PV5(6) OTT_PV5(7)
#undef OTT_PV5
        }
      }
      // ---- release this stage: prefetch the record of chunk i + kStages
      __syncwarp();
      if (lane == 0 && i + kS < n_chunks && group_of(i + kS) < g1) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        load_record<G>(stage0 + (i % kS) * tc5::kRec, tmap, unit_rec + group_of(i + kS), rbar0 + 8 * (i % kS));
      }
    }

    // ---- per-warp totals (thread = token: sum l, vb over the lanes)
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      l[h] = warp_sum(l[h]);
      vb[h] = warp_sum(vb[h]);
    }
    if (lane == 0) {
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        sm.mm[w][h] = m[h];
        sm.ll[w][h] = l[h];
      }
    }
  }
  __syncthreads();  // every warp is past its loop: stage memory is free
  if (warp < tc5::kCW) {
    float* accw = reinterpret_cast<float*>(&sm.stage[warp][0][0]);  // [8 heads][128] natural channel order
    const float vb0 = pick4<0>(vb, tig), vb1 = pick4<1>(vb, tig);
#pragma unroll
    for (int cm = 0; cm < 8; ++cm) {
      const float f = pair_pos(cm) == 2 ? 262144.f : (pair_pos(cm) == 3 ? 65536.f : 16384.f);  // 2^(22-2P)
      accw[(2 * tig) * D + 8 * g + cm] = fmaf(o[cm][0], f, vb0);
      accw[(2 * tig + 1) * D + 8 * g + cm] = fmaf(o[cm][1], f, vb1);
      accw[(2 * tig) * D + 64 + 8 * g + cm] = fmaf(o[cm][2], f, vb0);
      accw[(2 * tig + 1) * D + 64 + 8 * g + cm] = fmaf(o[cm][3], f, vb1);
    }
  }
  __syncthreads();
  for (int i = tid; i < NR * D; i += tc5::kThreads) {
    const int r = i / D, col = i % D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < tc5::kCW; ++w) M = fmaxf(M, sm.mm[w][r]);
    float Lsum = 0.f, A = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int w = 0; w < tc5::kCW; ++w) {
        if (sm.mm[w][r] == -INFINITY) continue;
        const float f = exp2f(sm.mm[w][r] - M);
        Lsum += sm.ll[w][r] * f;
        A += reinterpret_cast<const float*>(&sm.stage[w][0][0])[r * D + col] * f;
      }
    }
    float* base = a.ws + (((size_t)u * NR + r) * a.n_splits + split) * (D + 2);
    base[2 + col] = A;
    if (col == 0) {
      base[0] = M;
      base[1] = Lsum;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(tc5::kCols));
}

template <int NR>
__global__ void __launch_bounds__(tc5::kThreads, OTT_TC5_MIN_BLOCKS)
    attend_tc5_kernel(const __grid_constant__ AttnArgs a, const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(256) unsigned char smem_raw[];
  allow_dependents();
  if ((int)blockIdx.y >= a.n_qsplits) {  // full-precision tiers on warps 0-3
    if (threadIdx.x >= 128) return;
    const Counts n = counts_of(a);
    if (blockIdx.x == 0 && blockIdx.y == a.n_qsplits && threadIdx.x == 0)  // token counts for the combine's guard
      reinterpret_cast<int64_t*>(a.ws + (size_t)a.c.n_units * NR * a.n_splits * 130)[0] = n.q_tokens;
    fp_body<NR>(a, n, *reinterpret_cast<FpSmem*>(smem_raw));
  } else {
    tc5_body<NR>(a, counts_of(a), &tmap, *reinterpret_cast<Tc5Smem*>(smem_raw));
  }
}

// ============================================================ combine + debug logits
// Split combine: one warp per (unit, head) row, 8 rows per 256-thread block; lane
// handles columns 2*lane, 2*lane+1 (+64, +65 at D = 128) with float2 loads.
constexpr int kCombineRows = 8;
template <int D>
static cudaError_t launch_combine(const AttnArgs& a, int NR, cudaStream_t st, bool tc_path = false,
                                  float umax = 16.f);

// Overflow guard of the 2-bit tensor-core path. Its fp16 operands hold q u step (u <= 16)
// and 4 p v_step (p <= 2^kLazy); pool_meta[u][3] bounds the unit's K and V steps (flush
// kernels). For a unit whose bound and |q| could overflow them (K or V ranges in the
// thousands: far outside real activations, but legal fp16 input) the combine recomputes the
// quantized-tier partial of the head on CUDA cores in float32, so the tensor-core kernel
// itself carries no extra code.
struct TcGuard {
  ott_cache_t c;
  const uint16_t* q;
  int NR;
  float scale_log2;
  float umax;  // largest position factor u of the K unpack (16 at 2 bits, 64 at 4 bits)
  int bits;
  int n_qsplits;  // partials [n_qsplits, n_splits) are the full-precision tiers'
};
// per (unit, head) row: q' of head h only involves q_h
__device__ __forceinline__ bool tc_row_safe(const TcGuard& gd, int urow, int lane) {
  const int u = urow / gd.NR;
  const uint2 raw = reinterpret_cast<const uint2*>(gd.q + (size_t)urow * 128)[lane];
  const float2 a = __half22float2(__habs2(*reinterpret_cast<const __half2*>(&raw.x)));
  const float2 b = __half22float2(__habs2(*reinterpret_cast<const __half2*>(&raw.y)));
  const float qm = warp_max(fmaxf(fmaxf(a.x, a.y), fmaxf(b.x, b.y)));
  const float smax = __int_as_float(gd.c.pool_meta[(size_t)u * 4 + 3]);
  const float sm1 = fmaxf(smax, 1.f);
  return smax <= 3.0e38f && gd.umax * qm < 6.5e4f && gd.umax * qm * sm1 < 6.5e4f && 4.f * 64.f * sm1 < 6.5e4f;
}
// quantized-tier partial (m, l, acc[lane + 32 k]) of head r of unit u over [0, q_tokens),
// float32 dequantization (quant.py:105-111) and online softmax, one warp
__device__ __forceinline__ void tc_guard_partial(const TcGuard& gd, int u, int r, int64_t q_tokens, int lane,
                                                 float& m, float& l, float (&acc)[4]) {
  constexpr int D = 128;
  const ott_cache_t& c = gd.c;
  const int G = c.group_size;
  const RecordLayout L(D, G, gd.bits);
  const uint16_t* qrow = gd.q + ((size_t)u * gd.NR + r) * D;
  m = -INFINITY;
  l = 0.f;
  acc[0] = acc[1] = acc[2] = acc[3] = 0.f;
  const uint32_t* pmask = c.pool_mask + (size_t)u * mask_words_per_unit(c);
  const int n_groups = (int)(q_tokens / G);
  for (int gi = 0; gi < n_groups; ++gi) {
    const uint8_t* rec = record_ptr(c, u, gi);
    const uint8_t* kc = rec + L.k_codes();
    const uint8_t* vc = rec + L.v_codes();
    for (int t0 = 0; t0 < G; t0 += 32) {
      const int row = t0 + lane;
      const int64_t p = (int64_t)gi * G + row;
      float s = 0.f;
      for (int col = 0; col < D; ++col) {  // the slow path: parameters re-read per token
        const float code = (float)code_at(kc, (int64_t)row * D + col, gd.bits);
        const float st = k_step_of(rec, L, col);
        s = fmaf(h2f(qrow[col]) * gd.scale_log2, fmaf(code, st, k_xmin_of(rec, L, col, st)), s);
      }
      if ((pmask[p >> 5] >> (p & 31)) & 1u) s = -INFINITY;  // pooled: attended from the pool
      const float m_new = fmaxf(m, warp_max(s));
      float pt = 0.f;
      if (m_new != -INFINITY) {
        const float corr = exp2f(m - m_new);
        pt = exp2f(s - m_new);
        l = l * corr + warp_sum(pt);
        for (int k = 0; k < 4; ++k) acc[k] *= corr;
        m = m_new;
      }
      for (int tt = 0; tt < 32; ++tt) {
        const float pw = __shfl_sync(0xffffffffu, pt, tt);
        if (pw == 0.f) continue;
        const int rw = t0 + tt;
        const float vs = reinterpret_cast<const float*>(rec + L.v_step())[rw];
        const float vx = reinterpret_cast<const float*>(rec + L.v_xmin())[rw];
        for (int k = 0; k < 4; ++k) {
          const int col = lane + 32 * k;
          acc[k] = fmaf(pw, fmaf((float)code_at(vc, (int64_t)rw * D + col, gd.bits), vs, vx), acc[k]);
        }
      }
    }
  }
}

// Output stores of the combine: `out` plus the fused all-gather copies (ott_cache_t.out_peer,
// this rank's rows of each peer GPU's gather buffer; plain st.global over NVLink P2P).
__device__ __forceinline__ void store_out(const ott_cache_t& c, uint16_t* out, size_t off, uint16_t v) {
  out[off] = v;
  for (int i = 0; i < c.n_out_peers; ++i) c.out_peer[i][off] = v;
}
__device__ __forceinline__ void store_out2(const ott_cache_t& c, uint16_t* out, size_t off, __half2 v) {
  *reinterpret_cast<__half2*>(out + off) = v;
  for (int i = 0; i < c.n_out_peers; ++i) *reinterpret_cast<__half2*>(c.out_peer[i] + off) = v;
}

template <int D>
__global__ void __launch_bounds__(32 * kCombineRows) combine_kernel(const float* __restrict__ ws,
                                                                   uint16_t* __restrict__ out, int n_rows,
                                                                   int n_splits, int64_t* __restrict__ dev_counts,
                                                                   int G, int R, int max_groups, int d,
                                                                   TcGuard gd, int guard) {
  // overflow guard inputs (q, pool_meta) predate the attention grid: read them before the
  // programmatic wait so their latency hides behind its tail
  bool row_safe = true;
  if constexpr (D == 128) {
    const int urow = blockIdx.x * kCombineRows + (threadIdx.x >> 5);
    if (guard && urow < n_rows) row_safe = tc_row_safe(gd, urow, threadIdx.x & 31);
  }
#if OTT_PDL
  asm volatile("griddepcontrol.wait;\n" ::: "memory");  // the attention grid's partials are complete
#endif
  if constexpr (D == 128) {
    if (!row_safe) {
      const int lane = threadIdx.x & 31, wr = threadIdx.x >> 5;
      const int urow = blockIdx.x * kCombineRows + wr;
      // the token counts the attention kernel used (written by its unit-0 fp-tier CTA)
      const int64_t q_tokens = reinterpret_cast<const int64_t*>(ws + (size_t)n_rows * n_splits * (D + 2))[0];
      {
        float m, l, acc[4];
        tc_guard_partial(gd, urow / gd.NR, urow % gd.NR, q_tokens, lane, m, l, acc);
        // merge with the full-precision-tier partials
        const float* fp0 = ws + (size_t)urow * n_splits * (D + 2);
        float M = m;
        for (int sp = gd.n_qsplits; sp < n_splits; ++sp) M = fmaxf(M, fp0[(size_t)sp * (D + 2)]);
        const float fq = m == -INFINITY ? 0.f : exp2f(m - M);
        float Lt = l * fq, At[4];
        for (int k = 0; k < 4; ++k) At[k] = acc[k] * fq;
        for (int sp = gd.n_qsplits; sp < n_splits; ++sp) {
          const float* fp = fp0 + (size_t)sp * (D + 2);
          if (fp[0] == -INFINITY) continue;
          const float ff = exp2f(fp[0] - M);
          Lt += fp[1] * ff;
          for (int k = 0; k < 4; ++k) At[k] = fmaf(fp[2 + lane + 32 * k], ff, At[k]);
        }
        const float inv = 1.f / Lt;
        for (int k = 0; k < 4; ++k) store_out(gd.c, out, (size_t)urow * D + lane + 32 * k, f2h(At[k] * inv));
        if (dev_counts && blockIdx.x == 0 && threadIdx.x == 0) {
          const int64_t qt = dev_counts[0], tot = dev_counts[1] + 1;
          if (tot - qt - R >= G && qt / G + 1 <= max_groups) dev_counts[0] = qt + G;
          dev_counts[1] = tot;
        }
        return;
      }
    }
  }
  const int lane = threadIdx.x & 31;
  const int ur = blockIdx.x * kCombineRows + (threadIdx.x >> 5);  // unit*NR + r
  if (dev_counts && blockIdx.x == 0 && threadIdx.x == 0) {  // last kernel of a device-counter step: advance
    const int64_t qt = dev_counts[0], tot = dev_counts[1] + 1;
    if (tot - qt - R >= G && qt / G + 1 <= max_groups) dev_counts[0] = qt + G;
    dev_counts[1] = tot;
  }
  if (ur >= n_rows) return;
  if constexpr (D == 0) {  // generic head_dim: lane-strided columns
    const float* base = ws + (size_t)ur * n_splits * (d + 2);
    float M = -INFINITY;
    for (int s = 0; s < n_splits; ++s) M = fmaxf(M, base[(size_t)s * (d + 2)]);
    float Lsum = 0.f, acc[kMaxD / 32] = {0.f, 0.f, 0.f, 0.f};
    for (int s = 0; s < n_splits; ++s) {
      const float* p = base + (size_t)s * (d + 2);
      if (p[0] == -INFINITY) continue;
      const float f = exp2f(p[0] - M);
      Lsum += p[1] * f;
#pragma unroll
      for (int k = 0; k < kMaxD / 32; ++k)
        if (lane + 32 * k < d) acc[k] = fmaf(p[2 + lane + 32 * k], f, acc[k]);
    }
#pragma unroll
    for (int k = 0; k < kMaxD / 32; ++k)
      if (lane + 32 * k < d) store_out(gd.c, out, (size_t)ur * d + lane + 32 * k, f2h(acc[k] / Lsum));
    return;
  }
  const float* base = ws + (size_t)ur * n_splits * (D + 2);
  float M = -INFINITY;
  for (int s = 0; s < n_splits; ++s) M = fmaxf(M, base[(size_t)s * (D + 2)]);
  float Lsum = 0.f;
  float2 acc[D > 0 ? D / 64 : 1];
#pragma unroll
  for (int k = 0; k < D / 64; ++k) acc[k] = make_float2(0.f, 0.f);
  for (int s = 0; s < n_splits; ++s) {
    const float* p = base + (size_t)s * (D + 2);
    const float m = p[0];
    if (m == -INFINITY) continue;
    const float f = exp2f(m - M);
    Lsum += p[1] * f;
#pragma unroll
    for (int k = 0; k < D / 64; ++k) {
      const float2 v = *reinterpret_cast<const float2*>(p + 2 + 64 * k + 2 * lane);
      acc[k].x = fmaf(v.x, f, acc[k].x);
      acc[k].y = fmaf(v.y, f, acc[k].y);
    }
  }
  const float inv = 1.f / Lsum;
#pragma unroll
  for (int k = 0; k < D / 64; ++k)
    store_out2(gd.c, out, (size_t)ur * D + 64 * k + 2 * lane, __floats2half2_rn(acc[k].x * inv, acc[k].y * inv));
}

template <int D>
static cudaError_t launch_combine(const AttnArgs& a, int NR, cudaStream_t st, bool tc_path, float umax) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((a.c.n_units * NR + kCombineRows - 1) / kCombineRows);
  cfg.blockDim = dim3(32 * kCombineRows);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = OTT_PDL;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  TcGuard gd;
  gd.c = a.c;
  gd.q = a.q;
  gd.NR = NR;
  gd.scale_log2 = a.scale_log2;
  gd.umax = umax;
  gd.bits = code_bits(a.c.bits, a.c.head_dim, a.c.group_size);
  gd.n_qsplits = a.n_qsplits;
  return cudaLaunchKernelEx(&cfg, combine_kernel<D>, (const float*)a.ws, a.out, a.c.n_units * NR, a.n_splits,
                            a.advance ? const_cast<int64_t*>(a.dev_counts) : nullptr, a.c.group_size, a.c.residual,
                            a.c.max_groups,
                            a.c.head_dim, gd, tc_path ? 1 : 0);
}

template <int DT>  // 0: runtime head_dim (debug path; k lives in local memory then)
__global__ void logits_kernel(ott_cache_t c, const uint16_t* __restrict__ q, float* __restrict__ logits, int NR,
                              int64_t q_tokens, int64_t total, float inv_sqrt_d) {
  const int D = DT ? DT : c.head_dim;
  const int u = blockIdx.y;
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= total) return;
  const int G = c.group_size, N = c.capacity, cap = G + c.residual;
  const RecordLayout L(D, G, c.bits);
  float k[DT ? DT : kMaxD];
  bool done = false;
  if (p < q_tokens) {
    const uint32_t* pmask = c.pool_mask + (size_t)u * mask_words_per_unit(c);
    if ((pmask[p >> 5] >> (p & 31)) & 1u) {
      for (int s = 0; s < N; ++s)
        if (c.pool_pos[(size_t)u * N + s] == (int)p) {
          for (int j = 0; j < D; ++j) k[j] = h2f(c.pool_k[((size_t)u * N + s) * D + j]);
          done = true;
        }
    }
    if (!done) {
      const int64_t gi = p / G;
      const int row = (int)(p - gi * G);
      const uint8_t* rec = record_ptr(c, u, gi);
      for (int j = 0; j < D; ++j) {
        const float st = k_step_of(rec, L, j);
        k[j] = fmaf((float)code_at(rec + L.k_codes(), (int64_t)row * D + j, L.bits), st, k_xmin_of(rec, L, j, st));
      }
    }
  } else {
    const size_t off = ((size_t)u * cap + (size_t)(p % cap)) * D;
    for (int j = 0; j < D; ++j) k[j] = h2f(c.pend_k[off + j]);
  }
  for (int r = 0; r < NR; ++r) {
    float s = 0.f;
    for (int j = 0; j < D; ++j) s = fmaf(k[j], h2f(q[((size_t)u * NR + r) * D + j]), s);
    logits[((size_t)u * NR + r) * total + p] = s * inv_sqrt_d;
  }
}

// ============================================================ launchers
template <int NR, int D>
static cudaError_t launch_simt_t(const AttnArgs& a, cudaStream_t st) {
  const size_t smem = sizeof(SimtSmem<NR, D>);
  cudaError_t e = cudaFuncSetAttribute(attend_simt_kernel<NR, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  attend_simt_kernel<NR, D><<<dim3(a.c.n_units, a.n_splits), kAttnThreads, smem, st>>>(a);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_combine<D>(a, NR, st);
}

template <int NR>
static cudaError_t launch_generic_t(const AttnArgs& a, cudaStream_t st) {
  const size_t smem = sizeof(GenericSmem<NR>);
  cudaError_t e = cudaFuncSetAttribute(attend_generic_kernel<NR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  attend_generic_kernel<NR><<<dim3(a.c.n_units, a.n_splits), kAttnThreads, smem, st>>>(a);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_combine<0>(a, NR, st);
}

// Tensor map over all block records of the cache: 2-D uint8 view [rows of 32 B],
// SWIZZLE_32B, one (or two) boxes per record. Encoded per launch (host only).
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static cudaError_t record_tensor_map(const ott_cache_t& c, int box_rows, int rec_rows, CUtensorMap* map) {
  if (!g_encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) return cudaErrorNotSupported;
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[2] = {32, (cuuint64_t)c.n_units * (cuuint64_t)c.max_groups * (cuuint64_t)rec_rows};
  const cuuint64_t strides[1] = {32};
  const cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, c.blocks, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// 4/8-bit records: 2-D uint8 view [rows of 128 B], SWIZZLE_128B. G = 32: one box per record;
// G = 64/128: boxes of one 32-token code slice, of the 8 K-param rows and of one row (VgMaps).
static cudaError_t record_rows_map(const ott_cache_t& c, int rec_rows, int box_rows, CUtensorMap* map) {
  const cuuint64_t dims[2] = {128, (cuuint64_t)c.n_units * (cuuint64_t)c.max_groups * (cuuint64_t)rec_rows};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, c.blocks, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

static cudaError_t record_vg_maps(const ott_cache_t& c, int code_rows32, int rec_rows32, VgMaps* m) {
  CUtensorMap dummy;
  cudaError_t e = record_tensor_map(c, 1, 1, &dummy);  // resolves the driver entry point
  if (e != cudaSuccess) return e;
  const int G = c.group_size;
  if (G == 32) {
    e = record_rows_map(c, rec_rows32, rec_rows32, &m->rec);
    m->params = m->rec;
    m->row = m->rec;
    return e;
  }
  const int nsub = G / 32, rec_rows = 2 * code_rows32 * nsub + 8 + 2 * nsub;
  e = record_rows_map(c, rec_rows, code_rows32, &m->rec);
  if (e == cudaSuccess) e = record_rows_map(c, rec_rows, 8, &m->params);
  if (e == cudaSuccess) e = record_rows_map(c, rec_rows, 1, &m->row);
  return e;
}

template <int NR, int GR>
static cudaError_t launch_mma8_t(const AttnArgs& a, cudaStream_t st) {
  VgMaps tmap;
  cudaError_t te = record_vg_maps(a.c, 32, q8::kRows, &tmap);
  if (te != cudaSuccess) return te;
  const size_t smem = sizeof(Mma8Smem) > sizeof(FpSmem) ? sizeof(Mma8Smem) : sizeof(FpSmem);
  cudaError_t e =
      cudaFuncSetAttribute(attend_mma8_kernel<NR, GR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  attend_mma8_kernel<NR, GR><<<dim3(a.c.n_units, a.n_splits), kAttnThreads, smem, st>>>(a, tmap);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_combine<128>(a, NR, st, true, 1.f);
}

template <int NR, int GR>
static cudaError_t launch_mma4_t(const AttnArgs& a, cudaStream_t st) {
  VgMaps tmap;
  cudaError_t te = record_vg_maps(a.c, 16, q4::kRows, &tmap);
  if (te != cudaSuccess) return te;
  const size_t smem = sizeof(Mma4Smem) > sizeof(FpSmem) ? sizeof(Mma4Smem) : sizeof(FpSmem);
  cudaError_t e =
      cudaFuncSetAttribute(attend_mma4_kernel<NR, GR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  attend_mma4_kernel<NR, GR><<<dim3(a.c.n_units, a.n_splits), kAttnThreads, smem, st>>>(a, tmap);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_combine<128>(a, NR, st, true, 64.f);
}

template <int NR, int G>
static cudaError_t launch_mma_t(const AttnArgs& a, cudaStream_t st) {
  CUtensorMap tmap;
  cudaError_t te = record_tensor_map(a.c, RecTma<G>::kBoxRows, RecTma<G>::kRows, &tmap);
  if (te != cudaSuccess) return te;
  const size_t smem = sizeof(MmaSmem<G>) > sizeof(FpSmem) ? sizeof(MmaSmem<G>) : sizeof(FpSmem);
  cudaError_t e =
      cudaFuncSetAttribute(attend_mma_kernel<NR, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  attend_mma_kernel<NR, G><<<dim3(a.c.n_units, a.n_splits), kAttnThreads, smem, st>>>(a, tmap);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_combine<128>(a, NR, st, true);
}

template <int NR>
static cudaError_t launch_tc5_t(const AttnArgs& a, cudaStream_t st) {
  CUtensorMap tmap;
  cudaError_t te = record_tensor_map(a.c, RecTma<32>::kBoxRows, RecTma<32>::kRows, &tmap);
  if (te != cudaSuccess) return te;
  const size_t smem = sizeof(Tc5Smem) > sizeof(FpSmem) ? sizeof(Tc5Smem) : sizeof(FpSmem);
  cudaError_t e = cudaFuncSetAttribute(attend_tc5_kernel<NR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  attend_tc5_kernel<NR><<<dim3(a.c.n_units, a.n_splits), tc5::kThreads, smem, st>>>(a, tmap);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_combine<128>(a, NR, st, true);
}

// Attention kernel for (d = 128, G = 32): the mma.sync kernel (default, faster as
// measured) or the tcgen05 Q K^T kernel (OTT_ATTN_KERNEL=tc5); read
// once per process.
static bool use_tc5() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("OTT_ATTN_KERNEL");
    v = (e && strcmp(e, "tc5") == 0) ? 1 : 0;
  }
  return v == 1;
}

bool mma_eligible(const ott_cache_t& c) {
  return c.head_dim == 128 && code_bits(c.bits, c.head_dim, c.group_size) == 2 &&
         (c.group_size == 32 || c.group_size == 64 || c.group_size == 128);
}
#ifndef OTT_FP_SPLIT  // allow two full-precision-tier CTAs per unit (tensor-core kernels)
#define OTT_FP_SPLIT 1
#endif
#ifndef OTT_MMA4  // 4-bit caches at d = 128, G = 32 use the tensor-core kernel (0: CUDA-core kernel)
#define OTT_MMA4 1
#endif

// True when the attention kernel can write the step's new rows itself (fp-tier CTA of the
// tensor-core kernels); otherwise the caller launches the ring write first.
#ifndef OTT_FUSE_RING
#define OTT_FUSE_RING 1
#endif
bool attend_fuses_ring_write(const ott_cache_t& c) {
  return OTT_FUSE_RING && mma_eligible(c) && c.residual >= 1;
}

cudaError_t launch_attend(const ott_cache_t& c, const uint16_t* q, uint16_t* out, int n_rep, int64_t q_tokens,
                          int64_t total, float* ws, int n_qsplits, cudaStream_t st, int64_t* dev_counts,
                          const uint16_t* new_k, const uint16_t* new_v, bool advance) {
  AttnArgs a;
  a.dev_counts = dev_counts;
  a.advance = advance;
  a.new_k = new_k;
  a.new_v = new_v;
  a.c = c;
  a.q = q;
  a.out = out;
  a.ws = ws;
  a.q_tokens = q_tokens;
  a.total_tokens = total;
  a.n_qsplits = n_qsplits;
  a.n_fsplits = 1;
  a.n_splits = n_qsplits + 1;
  a.n_qtiles = (int)(q_tokens / 32);
  a.n_ptiles = (c.capacity + 31) / 32;
  a.n_rtiles = (int)((total - q_tokens + 31) / 32);
  a.scale_log2 = kLog2e / sqrtf((float)c.head_dim);
  a.k_magic = 0x3C003C00u;
  const int D = c.head_dim, G = c.group_size;
  if ((D != 64 && D != 128) || G % 32) {  // shapes outside the fast kernels' tiling
    if (n_rep == 1) return launch_generic_t<1>(a, st);
    if (n_rep == 2) return launch_generic_t<2>(a, st);
    if (n_rep == 4) return launch_generic_t<4>(a, st);
    if (n_rep == 8) return launch_generic_t<8>(a, st);
    return cudaErrorInvalidValue;
  }
  // tensor-core kernels: two CTAs share a unit's full-precision tiers when the quantized
  // splits are short (small MHA shapes such as config 1), so the fp tier is not the tail
  const int pb = code_bits(c.bits, D, G);  // stored code width: picks the decode kernel
  const bool tc_group = G == 32 || G == 64 || G == 128;  // record sizes the tensor-core kernels take
  const bool tc_path = mma_eligible(c) || (OTT_MMA4 && (pb == 4 || pb == 8) && D == 128 && tc_group);
  if (tc_path) {
    const int64_t ng = dev_counts ? (int64_t)c.max_groups : q_tokens / G;
    const int64_t per = (ng + n_qsplits - 1) / n_qsplits;
    const int fp_tiles = (c.capacity + 15) / 16 + (c.group_size + c.residual + 15) / 16;
    // only if the extra CTAs do not add a wave (4 resident CTAs per SM; 2 for the 8-bit kernel)
    static int sms = 0;
    if (!sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (sms <= 0) sms = 148;
    }
    const int64_t slots = (int64_t)sms * (pb == 8 ? 2 : 4);
    const int64_t w1 = ((int64_t)c.n_units * (n_qsplits + 1) + slots - 1) / slots;
    const int64_t w2 = ((int64_t)c.n_units * (n_qsplits + 2) + slots - 1) / slots;
    a.n_fsplits = (OTT_FP_SPLIT && per < 96 && fp_tiles >= 6 && w2 == w1) ? 2 : 1;
    a.n_splits = n_qsplits + a.n_fsplits;
  }
#define OTT_GCASE(FN, NRv, Gv) \
  if (n_rep == NRv && G == Gv) return FN<NRv, Gv>(a, st);
  if (OTT_MMA4 && pb == 4 && D == 128 && tc_group) {  // 4-bit tensor-core kernel (also 3-bit codes)
    OTT_GCASE(launch_mma4_t, 1, 32) OTT_GCASE(launch_mma4_t, 2, 32) OTT_GCASE(launch_mma4_t, 4, 32)
    OTT_GCASE(launch_mma4_t, 8, 32) OTT_GCASE(launch_mma4_t, 1, 64) OTT_GCASE(launch_mma4_t, 2, 64)
    OTT_GCASE(launch_mma4_t, 4, 64) OTT_GCASE(launch_mma4_t, 8, 64) OTT_GCASE(launch_mma4_t, 1, 128)
    OTT_GCASE(launch_mma4_t, 2, 128) OTT_GCASE(launch_mma4_t, 4, 128) OTT_GCASE(launch_mma4_t, 8, 128)
    return cudaErrorInvalidValue;
  }
  if (OTT_MMA4 && pb == 8 && D == 128 && tc_group) {  // 8-bit tensor-core kernel (also 5..7-bit codes)
    OTT_GCASE(launch_mma8_t, 1, 32) OTT_GCASE(launch_mma8_t, 2, 32) OTT_GCASE(launch_mma8_t, 4, 32)
    OTT_GCASE(launch_mma8_t, 8, 32) OTT_GCASE(launch_mma8_t, 1, 64) OTT_GCASE(launch_mma8_t, 2, 64)
    OTT_GCASE(launch_mma8_t, 4, 64) OTT_GCASE(launch_mma8_t, 8, 64) OTT_GCASE(launch_mma8_t, 1, 128)
    OTT_GCASE(launch_mma8_t, 2, 128) OTT_GCASE(launch_mma8_t, 4, 128) OTT_GCASE(launch_mma8_t, 8, 128)
    return cudaErrorInvalidValue;
  }
#undef OTT_GCASE
  if (pb != 2 || !mma_eligible(c)) {  // other widths / group sizes: CUDA-core kernel with generic code extraction
#define OTT_BCASE(NRv, Dv) \
  if (n_rep == NRv && D == Dv) return launch_simt_t<NRv, Dv>(a, st);
    OTT_BCASE(1, 64) OTT_BCASE(2, 64) OTT_BCASE(4, 64) OTT_BCASE(8, 64)
    OTT_BCASE(1, 128) OTT_BCASE(2, 128) OTT_BCASE(4, 128) OTT_BCASE(8, 128)
#undef OTT_BCASE
    return cudaErrorInvalidValue;
  }
  if (mma_eligible(c) && G == 32 && use_tc5()) {
    if (n_rep == 1) return launch_tc5_t<1>(a, st);
    if (n_rep == 2) return launch_tc5_t<2>(a, st);
    if (n_rep == 4) return launch_tc5_t<4>(a, st);
    if (n_rep == 8) return launch_tc5_t<8>(a, st);
    return cudaErrorInvalidValue;
  }
  if (mma_eligible(c)) {
#define OTT_MCASE(NRv, Gv) \
  if (n_rep == NRv && G == Gv) return launch_mma_t<NRv, Gv>(a, st);
    OTT_MCASE(1, 32) OTT_MCASE(2, 32) OTT_MCASE(4, 32) OTT_MCASE(8, 32)
    OTT_MCASE(1, 64) OTT_MCASE(2, 64) OTT_MCASE(4, 64) OTT_MCASE(8, 64)
    OTT_MCASE(1, 128) OTT_MCASE(2, 128) OTT_MCASE(4, 128) OTT_MCASE(8, 128)
#undef OTT_MCASE
    return cudaErrorInvalidValue;
  }
#define OTT_CASE(NRv, Dv) \
  if (n_rep == NRv && D == Dv) return launch_simt_t<NRv, Dv>(a, st);
  OTT_CASE(1, 64) OTT_CASE(2, 64) OTT_CASE(4, 64) OTT_CASE(8, 64)
#undef OTT_CASE
  return cudaErrorInvalidValue;
}

// Query-head counts the kernels are not instantiated for (3, 5, 6, 7): the heads of each
// unit are staged into the next instantiated count (4 or 8) with zero rows, and only the real
// heads' outputs are copied back (plus the fused peer stores, which the padded combine skips).
// Heads [h0, h0 + nh) of every unit's n_rep query heads <-> the staged [units][nr][d] layout.
__global__ void rep_pad_kernel(const uint16_t* __restrict__ q, uint16_t* __restrict__ qs, int64_t n, int n_rep,
                               int h0, int nh, int nr, int d) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(i % d);
    const int64_t row = i / d;  // unit * nr + r
    const int r = (int)(row % nr);
    const int64_t u = row / nr;
    qs[i] = r < nh ? q[(u * n_rep + h0 + r) * d + j] : (uint16_t)0;
  }
}

__global__ void rep_unpad_kernel(ott_cache_t c, const uint16_t* __restrict__ os, uint16_t* __restrict__ out,
                                 int64_t n, int n_rep, int h0, int nh, int nr, int d) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(i % d);
    const int64_t row = i / d;  // unit * nh + r
    const int r = (int)(row % nh);
    const int64_t u = row / nh;
    const uint16_t x = os[(u * nr + r) * d + j];
    const size_t o = (size_t)(u * n_rep + h0 + r) * d + j;
    out[o] = x;
    for (int p = 0; p < c.n_out_peers; ++p) c.out_peer[p][o] = x;
  }
}

cudaError_t launch_rep_pad(const uint16_t* q, uint16_t* qs, int n_units, int n_rep, int h0, int nh, int nr, int d,
                           cudaStream_t st) {
  const int64_t n = (int64_t)n_units * nr * d;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  rep_pad_kernel<<<blocks, 256, 0, st>>>(q, qs, n, n_rep, h0, nh, nr, d);
  return cudaGetLastError();
}

cudaError_t launch_rep_unpad(const ott_cache_t& c, const uint16_t* os, uint16_t* out, int n_rep, int h0, int nh,
                             int nr, cudaStream_t st) {
  const int d = c.head_dim;
  const int64_t n = (int64_t)c.n_units * nh * d;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  rep_unpad_kernel<<<blocks, 256, 0, st>>>(c, os, out, n, n_rep, h0, nh, nr, d);
  return cudaGetLastError();
}

cudaError_t launch_logits(const ott_cache_t& c, const uint16_t* q, float* logits, int n_rep, int64_t q_tokens,
                          int64_t total, cudaStream_t st) {
  dim3 grid((unsigned)((total + 127) / 128), c.n_units);
  const float inv = 1.0f / sqrtf((float)c.head_dim);
  if (c.head_dim == 128) logits_kernel<128><<<grid, 128, 0, st>>>(c, q, logits, n_rep, q_tokens, total, inv);
  else if (c.head_dim == 64) logits_kernel<64><<<grid, 128, 0, st>>>(c, q, logits, n_rep, q_tokens, total, inv);
  else logits_kernel<0><<<grid, 128, 0, st>>>(c, q, logits, n_rep, q_tokens, total, inv);
  return cudaGetLastError();
}

}  // namespace ott
