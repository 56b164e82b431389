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

#include "ott_attend.cuh"

namespace ott {

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


// ---- 2-bit records at d = 128 (RecordLayout, width 2): the decode kernel streams the record
// head (codes, K step halves, V params) and fetches the K e fields of 8 groups at a time.
template <int G>
struct MmaSmem {
  static constexpr int kHead = G * 128 / 2 + 2 * 2 * 128 + 8 * G;  // record head bytes
  static constexpr int kStages = G == 32 ? 3 : 2;                  // TMA pipeline depth per warp (3 vs 2: -2 %, v7)
  static constexpr int kEStride = 528;  // e slot per group (+16 B skew: conflict-free A-fragment loads)
  // group record heads land here through a SWIZZLE_32B tensor map (16-byte chunk bit 4 ^= bit 7
  // of the offset): ldmatrix over 32-byte token rows is then bank-conflict free
  alignas(256) uint8_t stage[kAttnWarps][kStages][kHead];
  alignas(16) uint8_t ebuf[kAttnWarps][8][kEStride];  // e / (8 u) (fp16 hi[128], lo[128]) of 8 groups
  alignas(8) uint64_t bar[kAttnWarps][kStages];
  alignas(8) uint64_t ebar[kAttnWarps];
  float mm[kAttnWarps][8], ll[kAttnWarps][8];
};
template <int G>
struct RecHead {  // record head as kBoxes TMA boxes of 32-byte rows; a record is kRecRows rows
  static constexpr int kRecRows = (G * 128 / 2 + 8 * 128 + 8 * G) / 32;
  static constexpr int kRows = MmaSmem<G>::kHead / 32;
  static constexpr int kBoxes = kRows > 256 ? 2 : 1;
  static constexpr int kBoxRows = kRows / kBoxes;
};
template <int G>
__device__ __forceinline__ void load_record_head(uint32_t dst, const CUtensorMap* map, int64_t rec_index,
                                                 uint32_t bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(MmaSmem<G>::kHead)
               : "memory");
#pragma unroll
  for (int b = 0; b < RecHead<G>::kBoxes; ++b)
    tma_tensor_rows(dst + b * RecHead<G>::kBoxRows * 32, map,
                    (int)(rec_index * RecHead<G>::kRecRows + b * RecHead<G>::kBoxRows), bar);
}
// Warp-collective issue of the async copies (all lanes call, elect.sync picks one): the
// operands are warp-uniform values, so they stay in uniform registers (no per-lane issue loop).
__device__ __forceinline__ void elect_arrive_expect(uint32_t bar, uint32_t bytes) {
  asm volatile(
      "{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n"
      "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n}\n" ::"r"(bar), "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void elect_tma_rows(uint32_t dst, const CUtensorMap* map, int row, uint32_t bar) {
  asm volatile(
      "{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n"
      "@p cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n}\n" ::"r"(
          dst),
      "l"(map), "r"(0), "r"(row), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void elect_bulk_copy(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n"
      "@p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n}\n" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
template <int G>
__device__ __forceinline__ void warp_load_record_head(uint32_t dst, const CUtensorMap* map, int64_t rec_index,
                                                      uint32_t bar) {
  elect_arrive_expect(bar, MmaSmem<G>::kHead);
#pragma unroll
  for (int b = 0; b < RecHead<G>::kBoxes; ++b)
    elect_tma_rows(dst + b * RecHead<G>::kBoxRows * 32, map,
                   (int)(rec_index * RecHead<G>::kRecRows + b * RecHead<G>::kBoxRows), bar);
}
__device__ __forceinline__ void bulk_copy(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
// V code pairs as exact fp16 subnormals c 2^(2P-24) in place: pair m (channels m, m+8 of a
// code word) at mantissa position P = m for m <= 4 (AND only) and P = m - 5 for m >= 5 (from
// w >> 10): one shift per word.
struct VSrc {
  uint32_t x, r10;
};
__device__ __forceinline__ VSrc vsrc(uint32_t w) { return {w, w >> 10}; }
__host__ __device__ constexpr int vpos(int m) { return m <= 4 ? m : m - 5; }
template <int M>
__device__ __forceinline__ uint32_t vqt(const VSrc& s) {
  return (M <= 4 ? s.x : s.r10) & (0x00030003u << (2 * vpos(M)));
}
constexpr float kMinit = -1e30f;  // finite initial running max (the first group always rescales)

// Quantized-region partial for (unit blockIdx.x, split blockIdx.y < n_qsplits).
// Per warp, per group of G tokens (records of the warp's groups g0 + warp + 4k):
//   * Q K^T on tensor cores (mma.sync m16n8k16, f16 in, f32 accumulate): K codes become
//     fp16 1 + c 2^(2P-10) in place (one LOP3 per pair); the B operand q' = q u step is an
//     exact fp16 hi/lo split formed from the record's step halves.
//   * x_min bias sum_c q e (e = x_min - 4 u step): for 8 groups at once, one m16n8k16 per
//     k-step with A rows = the 8 groups' e / u (fp16 hi rows 0-7, lo rows 8-15, fetched by
//     one bulk copy per group) and B = q u (the registers the q' split starts from).
//   * online softmax with the running max folded into the bias, lazily rescaled.
//   * O^T += V^T P' with V codes as exact fp16 subnormals and P' = 4 p step in fp16.
template <int NR, int G>
__device__ void mma_body(const AttnArgs& a, const Counts& n, const CUtensorMap* tmap, MmaSmem<G>& sm, int u, int split,
                         int nparts) {
  constexpr int D = 128;
  constexpr int kHead = MmaSmem<G>::kHead;
  constexpr int kMt = G / 16;  // 16-token m-tiles per group
  constexpr int kStages = MmaSmem<G>::kStages;
  constexpr int kES = MmaSmem<G>::kEStride;
  const RecordLayout L(D, G);
  const ott_cache_t& c = a.c;
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);  // warp-uniform for the compiler
  const int g = lane >> 2, tig = lane & 3;

  const uint32_t magic = a.k_magic;
  const int n_groups = (int)(n.q_tokens / G);
  const int per = (n_groups + nparts - 1) / nparts;
  const int g0 = split * per;
  const int g1 = min(n_groups, g0 + per);
  const int my_n = g1 > g0 + warp ? (g1 - g0 - warp + kAttnWarps - 1) / kAttnWarps : 0;

  const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&sm.bar[warp][0]);
  const uint32_t ebar = (uint32_t)__cvta_generic_to_shared(&sm.ebar[warp]);
  const uint32_t stage0 = (uint32_t)__cvta_generic_to_shared(&sm.stage[warp][0][0]);
  const uint32_t ebuf0 = (uint32_t)__cvta_generic_to_shared(&sm.ebuf[warp][0][0]);
  const int64_t unit_rec = (int64_t)u * c.max_groups;  // record index of group 0
  const size_t rec_bytes = (size_t)L.bytes();
  // e fields of the warp's groups k0 .. k0 + 7 into the batch buffer (one bulk copy each)
  auto load_ebatch = [&](int k0) {  // whole warp
    const int nb = min(8, my_n - k0);
    elect_arrive_expect(ebar, nb * 4 * D);
    for (int j = 0; j < nb; ++j)
      elect_bulk_copy(ebuf0 + j * kES,
                      c.blocks + (size_t)(unit_rec + g0 + warp + (k0 + j) * kAttnWarps) * rec_bytes + L.k_e(), 4 * D,
                      ebar);
  };
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kStages; ++s) mbar_init(bar0 + 8 * s, 1);
    mbar_init(ebar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
#pragma unroll
  for (int s = 0; s < kStages; ++s)
    if (s < my_n) warp_load_record_head<G>(stage0 + s * kHead, tmap, unit_rec + g0 + warp + s * kAttnWarps, bar0 + 8 * s);
  if (my_n > 0) load_ebatch(0);
  // q * u(m) as exact fp16 pairs (channels 16w+m, 16w+m+8) of head g, words w = tig + 4 hw:
  // the B operand of the bias MMA, and the q' = q u step split starts from it
  // NR <= 4: B column g holds head g & 3 -- the q' hi half in columns 0-3 and the lo half in
  // columns 4-7 -- so one HMMA per k-step covers both halves (kHiLoN below)
  constexpr bool kHiLoN = NR <= 4;
  const int qhead = kHiLoN ? (g & 3) : g;
  __half2 q16[2][8];
#pragma unroll
  for (int hw = 0; hw < 2; ++hw) {
    const int wd = tig + 4 * hw;
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      float lo = 0.f, hi = 0.f;
      if (qhead < NR) {
        const uint16_t* qr = a.q + ((size_t)u * NR + qhead) * D + 16 * wd + m;
        lo = h2f(__ldg(qr)) * kpair_u(m);
        hi = h2f(__ldg(qr + 8)) * kpair_u(m);
      }
      q16[hw][m] = __floats2half2_rn(lo, hi);
    }
  }
  __syncthreads();

  float o[8][4];
#pragma unroll
  for (int cm = 0; cm < 8; ++cm) o[cm][0] = o[cm][1] = o[cm][2] = o[cm][3] = 0.f;
  float mrun[2] = {kMinit, kMinit}, lsum[2] = {0.f, 0.f}, vb[2] = {0.f, 0.f};
  const uint32_t* pmask = c.pool_mask + (size_t)u * mask_words_per_unit(c);

  // ldmatrix row addresses (bytes, relative to a 16-token tile): matrix i = lane/8,
  // row r = lane%8: i0 tokens 0-7 bytes 0-15, i1 tokens 8-15 bytes 0-15,
  // i2 tokens 0-7 bytes 16-31, i3 tokens 8-15 bytes 16-31.
  const uint32_t lm_off = (uint32_t)(((lane & 7) + ((lane >> 3) & 1) * 8) * 32 + (lane >> 4) * 16);
  const float scale = a.scale_log2, scale4 = 4.f * a.scale_log2;
  float eb0 = 0.f, eb1 = 0.f;  // scaled bias of group (batch base + g), heads 2 tig, 2 tig + 1
  uint32_t eph = 0, ph = 0;
  uint32_t mreg = 0;  // G = 32: pool-mask word of group (k & ~31) + lane (one load per 32 groups)
  // stage index and phase are compile-time within a round of kStages groups
  for (int k0 = 0; k0 < my_n; k0 += kStages, ph ^= 1u)
#pragma unroll
  for (int st = 0; st < kStages; ++st) {
    const int k = k0 + st;
    if (k >= my_n) break;
    const int gi = g0 + warp + k * kAttnWarps;
    uint32_t mwords[G / 32];
    if (G == 32) {
      if ((k & 31) == 0) {
        const int kl = k + lane;
        mreg = kl < my_n ? __ldg(&pmask[(size_t)(g0 + warp + kl * kAttnWarps)]) : 0u;
      }
      mwords[0] = __shfl_sync(0xffffffffu, mreg, k & 31);
    } else {
#pragma unroll
      for (int w = 0; w < G / 32; ++w) mwords[w] = __ldg(&pmask[(size_t)gi * (G / 32) + w]);
    }
    if ((k & 7) == 0) {  // ---- x_min bias of the next 8 groups on tensor cores
      mbar_wait(ebar, eph);
      eph ^= 1u;
      const uint8_t* eg = &sm.ebuf[warp][g][0];  // lane (g, tig): group k + g
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int hw = 0; hw < 2; ++hw) {
        const int wd = tig + 4 * hw;
        const uint4 h0 = *reinterpret_cast<const uint4*>(eg + 32 * wd);
        const uint4 h1 = *reinterpret_cast<const uint4*>(eg + 32 * wd + 16);
        const uint4 l0 = *reinterpret_cast<const uint4*>(eg + 2 * D + 32 * wd);
        const uint4 l1 = *reinterpret_cast<const uint4*>(eg + 2 * D + 32 * wd + 16);
        const uint32_t hiw[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
        const uint32_t low[8] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
#pragma unroll
        for (int mm = 0; mm < 8; mm += 2)
          mma16816(acc, hiw[mm], low[mm], hiw[mm + 1], low[mm + 1], h2_as_u32(q16[hw][mm]), h2_as_u32(q16[hw][mm + 1]));
      }
      eb0 = (acc[0] + acc[2]) * (kEScale * scale);
      eb1 = (acc[1] + acc[3]) * (kEScale * scale);
      __syncwarp();
      if (k + 8 < my_n) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        load_ebatch(k + 8);
      }
    }
    const float bias0 = __shfl_sync(0xffffffffu, eb0, 4 * (k & 7) + tig);  // head 2 tig
    const float bias1 = __shfl_sync(0xffffffffu, eb1, 4 * (k & 7) + tig);  // head 2 tig + 1
    mbar_wait(bar0 + 8 * st, ph);
    const uint8_t* rec = &sm.stage[warp][st][0];
    const uint32_t rec_s = stage0 + st * kHead;
    uint32_t kw[kMt][4];
#pragma unroll
    for (int mt = 0; mt < kMt; ++mt) ldsm_x4(kw[mt], rec_s + swz(L.k_codes() + mt * 16 * 32 + lm_off));

    // ---- S = Q K^T. B operand q' = q u step as an exact fp16 hi/lo split from the record's
    // fp16 step halves (sh + sl): hi = q sh, err = fma(q, sh, -hi) (exact), lo = fma(q, sl, err)
    float ch[kMt][4];
#pragma unroll
    for (int mt = 0; mt < kMt; ++mt) ch[mt][0] = ch[mt][1] = ch[mt][2] = ch[mt][3] = 0.f;
#pragma unroll
    for (int hw = 0; hw < 2; ++hw) {
      const int wd = tig + 4 * hw;
      const uint4 h0 = *reinterpret_cast<const uint4*>(rec + swz(L.k_sh() + 32 * wd));
      const uint4 h1 = *reinterpret_cast<const uint4*>(rec + swz(L.k_sh() + 32 * wd + 16));
      const uint4 l0 = *reinterpret_cast<const uint4*>(rec + swz(L.k_sl() + 32 * wd));
      const uint4 l1 = *reinterpret_cast<const uint4*>(rec + swz(L.k_sl() + 32 * wd + 16));
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
        bl[m] = h2_as_u32(__hfma2(q16[hw][m], sl, E));
        if (kHiLoN) bh[m] = g >= 4 ? bl[m] : bh[m];  // column g: hi (g < 4) or lo (g >= 4) half
      }
      Shifted s0[kMt], s1[kMt];
#pragma unroll
      for (int mt = 0; mt < kMt; ++mt) {
        s0[mt] = shifted(kw[mt][2 * hw]);
        s1[mt] = shifted(kw[mt][2 * hw + 1]);
      }
#define OTT_QK(MM)                                                                    \
  {                                                                                   \
    _Pragma("unroll") for (int mt = 0; mt < kMt; ++mt) {                              \
      const uint32_t a0 = kq<MM>(s0[mt], magic), a1 = kq<MM>(s1[mt], magic);         \
      const uint32_t a2 = kq<MM + 1>(s0[mt], magic), a3 = kq<MM + 1>(s1[mt], magic); \
      mma16816(ch[mt], a0, a1, a2, a3, bh[MM], bh[MM + 1]);                           \
      if (!kHiLoN) mma16816(ch[mt], a0, a1, a2, a3, bl[MM], bl[MM + 1]);             \
    }                                                                                 \
  }
      OTT_QK(0) OTT_QK(2) OTT_QK(4) OTT_QK(6)
#undef OTT_QK
    }

    if (kHiLoN) {  // logit = hi column + lo column (lanes tig, tig ^ 2); tig >= 2 lanes hold copies
#pragma unroll
      for (int mt = 0; mt < kMt; ++mt)
#pragma unroll
        for (int e = 0; e < 4; ++e) ch[mt][e] += __shfl_xor_sync(0xffffffffu, ch[mt][e], 2);
    }
    // ---- x = logit - m (log2 units), heads 2 tig (cols 0, 2) and 2 tig + 1 (cols 1, 3)
    const float bm0 = bias0 - mrun[0], bm1 = bias1 - mrun[1];
    float x[kMt][4];
#pragma unroll
    for (int mt = 0; mt < kMt; ++mt) {
      x[mt][0] = fmaf(ch[mt][0], scale4, bm0);
      x[mt][1] = fmaf(ch[mt][1], scale4, bm1);
      x[mt][2] = fmaf(ch[mt][2], scale4, bm0);
      x[mt][3] = fmaf(ch[mt][3], scale4, bm1);
    }
    // pooled positions: their logits come from the pool tile (overwrite semantics)
    bool any_pooled = false;
#pragma unroll
    for (int w = 0; w < G / 32; ++w) any_pooled |= mwords[w] != 0u;
    if (any_pooled) {
#pragma unroll
      for (int w = 0; w < G / 32; ++w) {
        const uint32_t mw = mwords[w];
#pragma unroll
        for (int mt = 2 * w; mt < 2 * w + 2; ++mt) {
          if ((mw >> ((mt & 1) * 16 + g)) & 1u) x[mt][0] = x[mt][1] = -INFINITY;
          if ((mw >> ((mt & 1) * 16 + g + 8)) & 1u) x[mt][2] = x[mt][3] = -INFINITY;
        }
      }
    }

    // ---- online softmax, lazily rescaled: the running max only moves when a logit exceeds it
    // by kLazy (log2 units), so p <= 2^kLazy
    float xmax = x[0][0];
#pragma unroll
    for (int mt = 0; mt < kMt; ++mt)
#pragma unroll
      for (int e = 0; e < 4; ++e) xmax = fmaxf(xmax, x[mt][e]);
    if (__any_sync(0xffffffffu, xmax > kLazy)) {  // rare: recompute the logits against the new max
      float t[2] = {-INFINITY, -INFINITY};
#pragma unroll
      for (int mt = 0; mt < kMt; ++mt) {
        x[mt][0] = x[mt][0] == -INFINITY ? -INFINITY : fmaf(ch[mt][0], scale4, bias0);
        x[mt][1] = x[mt][1] == -INFINITY ? -INFINITY : fmaf(ch[mt][1], scale4, bias1);
        x[mt][2] = x[mt][2] == -INFINITY ? -INFINITY : fmaf(ch[mt][2], scale4, bias0);
        x[mt][3] = x[mt][3] == -INFINITY ? -INFINITY : fmaf(ch[mt][3], scale4, bias1);
        t[0] = fmaxf(t[0], fmaxf(x[mt][0], x[mt][2]));
        t[1] = fmaxf(t[1], fmaxf(x[mt][1], x[mt][3]));
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float tm = t[h];
        tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 4));
        tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 8));
        tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 16));
        const float mnew = fmaxf(mrun[h], tm);
        const float corr = ex2(mrun[h] - mnew);
        lsum[h] *= corr;
        vb[h] *= corr;
#pragma unroll
        for (int cm = 0; cm < 8; ++cm) {
          o[cm][h] *= corr;
          o[cm][h + 2] *= corr;
        }
        mrun[h] = mnew;
#pragma unroll
        for (int mt = 0; mt < kMt; ++mt) {
          x[mt][h] -= mnew;
          x[mt][h + 2] -= mnew;
        }
      }
    }

    // ---- O^T += V^T P'  (P' = 4 p step fp16, V x_min into vb; with V codes as
    // subnormals the accumulator holds sum(p step c) * 2^(2P-22))
#pragma unroll
    for (int mt = 0; mt < kMt; ++mt) {
      const float vs0 = *reinterpret_cast<const float*>(rec + swz(L.v_step() + 4 * (mt * 16 + g)));
      const float vs1 = *reinterpret_cast<const float*>(rec + swz(L.v_step() + 4 * (mt * 16 + g + 8)));
      const float ve0 = *reinterpret_cast<const float*>(rec + swz(L.v_xmin() + 4 * (mt * 16 + g)));
      const float ve1 = *reinterpret_cast<const float*>(rec + swz(L.v_xmin() + 4 * (mt * 16 + g + 8)));
      const float p00 = ex2(x[mt][0]), p01 = ex2(x[mt][1]);
      const float p10 = ex2(x[mt][2]), p11 = ex2(x[mt][3]);
      lsum[0] += p00 + p10;
      lsum[1] += p01 + p11;
      vb[0] = fmaf(p00, ve0, fmaf(p10, ve1, vb[0]));
      vb[1] = fmaf(p01, ve0, fmaf(p11, ve1, vb[1]));
      const float f0 = 4.f * vs0, f1 = 4.f * vs1;
      const uint32_t b0 = movm_t(pack_h2(p00 * f0, p01 * f0));
      const uint32_t b1 = movm_t(pack_h2(p10 * f1, p11 * f1));
      uint32_t vr[4];
      ldsm_x4_t(vr, rec_s + swz(L.v_codes() + mt * 16 * 32 + lm_off));
      const VSrc v0 = vsrc(vr[0]), v1 = vsrc(vr[1]), v2 = vsrc(vr[2]), v3 = vsrc(vr[3]);
#define OTT_PV(CM) mma16816(o[CM], vqt<CM>(v0), vqt<CM>(v2), vqt<CM>(v1), vqt<CM>(v3), b0, b1);
      OTT_PV(0) OTT_PV(1) OTT_PV(2) OTT_PV(3) OTT_PV(4) OTT_PV(5) OTT_PV(6) OTT_PV(7)
#undef OTT_PV
    }

    // ---- release the stage: prefetch the record head of group k + kStages
    __syncwarp();
    if (k + kStages < my_n) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      warp_load_record_head<G>(rec_s, tmap, unit_rec + gi + kStages * kAttnWarps, bar0 + 8 * st);
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
      sm.mm[warp][2 * tig + h] = lsum[h] > 0.f ? mrun[h] : -INFINITY;  // no token: empty partial
      sm.ll[warp][2 * tig + h] = lsum[h];
    }
  }
  __syncthreads();  // every warp is past its loop: stage memory is free
  float* accw = reinterpret_cast<float*>(&sm.stage[warp][0][0]);  // [8 heads][128] natural channel order
#pragma unroll
  for (int cm = 0; cm < 8; ++cm) {
    const float f = (float)(1 << (22 - 2 * vpos(cm)));  // 2^(22-2P)
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
  if (nparts < a.n_qsplits) {  // a whole unit of the tail schedule: its other quantized slots are empty
    for (int i = threadIdx.x; i < NR * (a.n_qsplits - nparts); i += kAttnThreads) {
      float* base = a.ws + (((size_t)u * NR + i % NR) * a.n_splits + nparts + i / NR) * (D + 2);
      base[0] = -INFINITY;
      base[1] = 0.f;
    }
  }
}


template <int NR, int G>
__global__ void __launch_bounds__(kAttnThreads, OTT_MMA_MIN_BLOCKS)
    attend_mma_kernel(const __grid_constant__ AttnArgs a, const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(256) unsigned char smem_raw[];
  allow_dependents();
  // (unit, partial slot, pieces of the unit's quantized range) of this CTA
  int u = blockIdx.x, y = blockIdx.y, nparts = a.n_qsplits;
  if (a.tail_units > 0) {  // 1-D grid: [whole units][tail units x n_qsplits pieces][fp-tier CTAs]
    const int U = a.c.n_units, W = U - a.tail_units, P = a.tail_units * a.n_qsplits, i = blockIdx.x;
    if (i < W) {
      u = i, y = 0, nparts = 1;
    } else if (i < W + P) {
      u = W + (i - W) / a.n_qsplits, y = (i - W) % a.n_qsplits;
    } else {
      u = (i - W - P) % U, y = a.n_qsplits + (i - W - P) / U;
    }
  }
  if (y >= a.n_qsplits) {  // full-precision tiers: pool + pending
    const Counts n = counts_of(a);
    if (u == 0 && y == a.n_qsplits && threadIdx.x == 0)  // token counts for the combine's guard
      reinterpret_cast<int64_t*>(a.ws + (size_t)a.c.n_units * NR * a.n_splits * 130)[0] = n.q_tokens;
    fp_body<NR>(a, n, *reinterpret_cast<FpSmem*>(smem_raw), u, y);
  } else {
    mma_body<NR, G>(a, counts_of(a), &tmap, *reinterpret_cast<MmaSmem<G>*>(smem_raw), u, y, nparts);
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
  // NR <= 4: B column g holds head g & 3 -- the q' hi half in columns 0-3, the lo half in 4-7
  // -- so one HMMA per k-step covers both halves (as in mma_body)
  constexpr bool kHiLoN = NR <= 4;
  for (int i = tid; i < 8 * 32; i += kAttnThreads) {
    const int k = i >> 5, ln = i & 31, h = kHiLoN ? ((ln >> 2) & 3) : (ln >> 2), t4 = ln & 3;
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
          if (kHiLoN) bh[b][kk] = g >= 4 ? bl[b][kk] : bh[b][kk];
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
      if (!kHiLoN) mma16816(ch[mt], a0, a1, a2, a3, bl[0][K], bl[1][K]);                     \
    }                                                                                         \
  }
      OTT_QK4(0) OTT_QK4(1) OTT_QK4(2) OTT_QK4(3)
#undef OTT_QK4
    }
    if (kHiLoN) {  // logit = hi column + lo column (lanes tig, tig ^ 2); tig >= 2 lanes hold copies
#pragma unroll
      for (int mt = 0; mt < kMt; ++mt)
#pragma unroll
        for (int e = 0; e < 4; ++e) ch[mt][e] += __shfl_xor_sync(0xffffffffu, ch[mt][e], 2);
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
    fp_body<NR>(a, n, *reinterpret_cast<FpSmem*>(smem_raw), blockIdx.x, blockIdx.y);
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
    fp_body<NR>(a, n, *reinterpret_cast<FpSmem*>(smem_raw), blockIdx.x, blockIdx.y);
  } else {
    mma8_body<NR, GR>(a, counts_of(a), &tmap, *reinterpret_cast<Mma8Smem*>(smem_raw));
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

// Device-counter step (counters = {quantized, total, error}): the append made a flush due
// (cache.py:138) and the flush kernel ran it, unless the cache is out of group records: then
// the flush was skipped, the step's new row overwrote a pending row, and the counts stop
// advancing with the error flag set (OTTCache.decode_step / device_error raise it on the host).
__device__ __forceinline__ void advance_counts(int64_t* cnt, int G, int R, int max_groups) {
  const int64_t qt = cnt[0], tot = cnt[1] + 1;
  if (tot - qt - R >= G) {
    if (qt / G + 1 > max_groups) {
      cnt[2] = 1;
      return;
    }
    cnt[0] = qt + G;
  }
  cnt[1] = tot;
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
        if (dev_counts && blockIdx.x == 0 && threadIdx.x == 0) advance_counts(dev_counts, G, R, max_groups);
        return;
      }
    }
  }
  const int lane = threadIdx.x & 31;
  const int ur = blockIdx.x * kCombineRows + (threadIdx.x >> 5);  // unit*NR + r
  // last kernel of a device-counter step: advance the counts
  if (dev_counts && blockIdx.x == 0 && threadIdx.x == 0) advance_counts(dev_counts, G, R, max_groups);
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

cudaError_t launch_combine_tc128(const AttnArgs& a, int NR, cudaStream_t st) {
  return launch_combine<128>(a, NR, st, true);
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
cudaError_t record_tensor_map(const ott_cache_t& c, int box_rows, int rec_rows, CUtensorMap* map) {
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
  cudaError_t te = record_tensor_map(a.c, RecHead<G>::kBoxRows, RecHead<G>::kRecRows, &tmap);
  if (te != cudaSuccess) return te;
  const size_t smem = sizeof(MmaSmem<G>) > sizeof(FpSmem) ? sizeof(MmaSmem<G>) : sizeof(FpSmem);
  cudaError_t e =
      cudaFuncSetAttribute(attend_mma_kernel<NR, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const dim3 grid = a.tail_units > 0 ? dim3(a.c.n_units - a.tail_units + a.c.n_units * a.n_fsplits +
                                                a.tail_units * a.n_qsplits)
                                         : dim3(a.c.n_units, a.n_splits);
  attend_mma_kernel<NR, G><<<grid, kAttnThreads, smem, st>>>(a, tmap);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_combine<128>(a, NR, st, true);
}

bool mma_eligible(const ott_cache_t& c) {
  return c.head_dim == 128 && code_bits(c.bits, c.head_dim, c.group_size) == 2 &&
         (c.group_size == 32 || c.group_size == 64 || c.group_size == 128);
}
#ifndef OTT_TAIL_SPLIT  // tail schedule of the 2-bit tensor-core kernel (AttnArgs.tail_units)
#define OTT_TAIL_SPLIT 1
#endif
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
  a.tail_units = 0;
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
    // more units than resident CTAs (config 4: 1,024 on 592): one wave of whole units, the rest
    // cut into n_qsplits pieces, then the short fp-tier CTAs: the launch ends on small work items
    if (OTT_TAIL_SPLIT && mma_eligible(c) && n_qsplits >= 2 && c.n_units > slots) {
      a.tail_units = (int)(c.n_units - slots);
      a.n_fsplits = 1;  // two fp-tier CTAs per unit here: 399.8 us; fp tier before the pieces: 401.6
      a.n_splits = n_qsplits + 1;
    }
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
