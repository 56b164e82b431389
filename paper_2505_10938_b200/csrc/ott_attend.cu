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
// Grid = (units, n_qsplits + 1): the first n_qsplits CTAs of a unit stream
// contiguous ranges of quantized group records; the last CTA attends the
// full-precision tiers. Each CTA writes an online-softmax partial (m, l, acc)
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
#include <cuda.h>
#include <cudaTypedefs.h>

#include "ott_common.cuh"

namespace ott {

// hi and lo products of Q K^T accumulate into one chain (1) or two (0); one
// chain measured ~1% faster (fewer registers, 8 fewer FADD per group)
#ifndef OTT_SINGLE_CHAIN
#define OTT_SINGLE_CHAIN 1
#endif
#if OTT_SINGLE_CHAIN
#define OTT_LO_ACC ch
#else
#define OTT_LO_ACC cl
#endif
#ifndef OTT_MMA_MIN_BLOCKS
#define OTT_MMA_MIN_BLOCKS 4
#endif
constexpr int kAttnThreads = 128;
constexpr int kAttnWarps = kAttnThreads / 32;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLazy = 6.f;  // lazy-rescale threshold (log2 units): p <= 64, P' = 4 p step fits fp16

struct AttnArgs {
  ott_cache_t c;
  const uint16_t* q;
  uint16_t* out;
  float* ws;  // [n_units][NR][n_splits][D+2]
  int64_t q_tokens, total_tokens;
  int n_splits;   // total partials per (unit, head) = n_qsplits + 1
  int n_qsplits;  // splits over the quantized region
  int n_qtiles, n_ptiles, n_rtiles;  // 32-token tiles: quantized, pool, pending
  float scale_log2;                  // log2(e) / float32(sqrt(d))
  uint32_t k_magic;                  // 0x3C003C00 (fp16 1.0 pair), passed at run time so the
                                     // compiler keeps it in a register: one LOP3 per code pair
};

// ============================================================ SIMT (CUDA-core) tiles
template <int NR, int D>
struct WarpScratch {
  float qp[NR][D];
  float p[NR][32];
  uint32_t vw[32][D / 16];
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
__device__ void simt_body(const AttnArgs& a, int u, int t_begin, int t_end, int split, SimtSmem<NR, D>& sm) {
  const ott_cache_t& c = a.c;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = c.group_size, N = c.capacity, cap = G + c.residual;
  const RecordLayout L(D, G);
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
    if (t < a.n_qtiles) {
      const int64_t tok0 = (int64_t)t * 32;
      const int64_t gi = tok0 / G;
      const int row0 = (int)(tok0 - gi * G);
      const uint8_t* rec = record_ptr(c, u, gi);
      const float* kstep = reinterpret_cast<const float*>(rec + L.k_step());
      const float* kxmin = reinterpret_cast<const float*>(rec + L.k_xmin());
      float bias[NR];
#pragma unroll
      for (int r = 0; r < NR; ++r) bias[r] = 0.f;
      for (int col = lane; col < D; col += 32) {
        const float st = kstep[col], mn = kxmin[col];
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          ws.qp[r][col] = sm.qs[r][col] * st;
          bias[r] += sm.qs[r][col] * mn;
        }
      }
#pragma unroll
      for (int r = 0; r < NR; ++r) bias[r] = warp_sum(bias[r]);
      const uint32_t* vcw = reinterpret_cast<const uint32_t*>(rec + L.v_codes()) + (size_t)row0 * (D / 16);
#pragma unroll
      for (int j = 0; j < D / 16; ++j) {
        const int idx = j * 32 + lane;
        ws.vw[idx / (D / 16)][idx % (D / 16)] = vcw[idx];
      }
      ws.vstep[lane] = reinterpret_cast<const float*>(rec + L.v_step())[row0 + lane];
      ws.vxmin[lane] = reinterpret_cast<const float*>(rec + L.v_xmin())[row0 + lane];
      __syncwarp();
      const uint32_t* kcw = reinterpret_cast<const uint32_t*>(rec + L.k_codes()) + (size_t)(row0 + lane) * (D / 16);
#pragma unroll
      for (int r = 0; r < NR; ++r) s[r] = bias[r];
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
      const bool pooled = (pmask[tok0 >> 5] >> lane) & 1u;
      if (pooled) {
#pragma unroll
        for (int r = 0; r < NR; ++r) s[r] = -INFINITY;
      }
      online_update<NR, D>(s, m, l, acc, ws, lane);
#pragma unroll 4
      for (int tt = 0; tt < 32; ++tt) {
        const float st = ws.vstep[tt], mn = ws.vxmin[tt];
#pragma unroll
        for (int k = 0; k < D / 32; ++k) {
          const int col = lane + 32 * k;
          const float v = fmaf((float)((ws.vw[tt][col >> 4] >> (2 * (col & 15))) & 3u), st, mn);
#pragma unroll
          for (int r = 0; r < NR; ++r) acc[r][k] = fmaf(ws.p[r][tt], v, acc[r][k]);
        }
      }
      __syncwarp();
    } else {
      const bool is_pool = t < a.n_qtiles + a.n_ptiles;
      const uint16_t *krow, *vrow;
      bool valid;
      if (is_pool) {
        const int slot = (t - a.n_qtiles) * 32 + lane;
        valid = slot < N && c.pool_pos[(size_t)u * N + slot] >= 0;
        const size_t off = ((size_t)u * N + (valid ? slot : 0)) * D;
        krow = c.pool_k + off;
        vrow = c.pool_v + off;
      } else {
        const int64_t p = a.q_tokens + (int64_t)(t - a.n_qtiles - a.n_ptiles) * 32 + lane;
        valid = p < a.total_tokens;
        const size_t off = ((size_t)u * cap + (size_t)((valid ? p : a.q_tokens) % cap)) * D;
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
  SimtSmem<NR, D>& sm = *reinterpret_cast<SimtSmem<NR, D>*>(smem_raw);
  const int n_tiles = a.n_qtiles + a.n_ptiles + a.n_rtiles;
  const int per = (n_tiles + a.n_splits - 1) / a.n_splits;
  const int t_begin = blockIdx.y * per;
  const int t_end = min(n_tiles, t_begin + per);
  simt_body<NR, D>(a, blockIdx.x, t_begin, t_end, blockIdx.y, sm);
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
#ifndef OTT_Q_IN_REGS
#define OTT_Q_IN_REGS 0
#endif
#ifndef OTT_NG
#define OTT_NG 1  // groups per loop iteration per warp (2 measured slower: register spills)
#endif
#ifndef OTT_STAGES
#define OTT_STAGES 2
#endif
  static constexpr int kNG = G == 32 ? OTT_NG : 1;               // groups per loop iteration
  static constexpr int kStages = G == 32 ? OTT_STAGES : 2;          // TMA pipeline depth per warp
  // q * 4 * scale_log2 in per-lane order: [hw][v4][lane] = head lane/4, channels
  // 16*(lane%4 + 4*hw) + 4*v4 .. +3  (conflict-free LDS.128)
  float4 q4p[2][4][32];
  // per-group channel scratch [hw][slot], slot = 4*v4 + (tig ^ 2*(v4>>1)) (bank-conflict
  // free for the lane-ordered writes and the per-tig broadcast reads): step * f and
  // x_min - 4 f step with f = 4^(4 - P(m))
  float4 stp[kAttnWarps][kNG][2][16];
  float4 esc[kAttnWarps][kNG][2][16];
  // group records land here through a SWIZZLE_32B tensor map (16-byte chunk bit 4 ^= bit 7
  // of the offset): ldmatrix over 32-byte token rows is then bank-conflict free
  alignas(256) uint8_t stage[kAttnWarps][kStages][kRec];
  alignas(8) uint64_t bar[kAttnWarps][kStages];
  float mm[kAttnWarps][8], ll[kAttnWarps][8];
};

// Quantized-region partial for (unit blockIdx.x, split blockIdx.y < n_qsplits).
template <int NR, int G>
__device__ void mma_body(const AttnArgs& a, const CUtensorMap* tmap, MmaSmem<G>& sm) {
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
  const int n_groups = (int)(a.q_tokens / G);
  const int per = (n_groups + a.n_qsplits - 1) / a.n_qsplits;
  const int g0 = split * per;
  const int g1 = min(n_groups, g0 + per);
  const int my_n = g1 > g0 + warp ? (g1 - g0 - warp + kAttnWarps - 1) / kAttnWarps : 0;

  for (int i = tid; i < 2 * 4 * 32; i += kAttnThreads) {
    const int hw = i >> 7, v4 = (i >> 5) & 3, ln = i & 31;
    const int h = ln >> 2, ch = 16 * ((ln & 3) + 4 * hw) + 4 * v4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (h < NR) {
      const uint16_t* qp = a.q + ((size_t)u * NR + h) * D + ch;
      const float f = 4.f * a.scale_log2;
      v = make_float4(h2f(qp[0]) * f, h2f(qp[1]) * f, h2f(qp[2]) * f, h2f(qp[3]) * f);
    }
    sm.q4p[hw][v4][ln] = v;
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
  // cooperative channel pass: lane owns channels 4*lane..+3 = word lane/4, v4 = lane%4
  const int cw = lane >> 2;
  float4* stp_w = &sm.stp[warp][0][cw >> 2][tile_slot(lane & 3, cw & 3)];  // + j*32 for group j
  float4* esc_w = &sm.esc[warp][0][cw >> 2][tile_slot(lane & 3, cw & 3)];
  // f = 4^(4 - P(m)) for this lane's pairs: m = 0..3 -> {4, 1, 16, 4}; m = 4..7 -> {1, 16, 4, 1}
  const float4 cf = (lane & 1) ? make_float4(1.f, 16.f, 4.f, 1.f) : make_float4(4.f, 1.f, 16.f, 4.f);

#if OTT_Q_IN_REGS
  float4 qreg[2][4];
#pragma unroll
  for (int hw = 0; hw < 2; ++hw)
#pragma unroll
    for (int v4 = 0; v4 < 4; ++v4) qreg[hw][v4] = sm.q4p[hw][v4][lane];
#endif
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
      // channel pass: step * f and e = x_min - 4 f step with f = 4^(4 - P(m))
      const float4 st = *reinterpret_cast<const float4*>(rec[j] + swz(L.k_step() + 16 * lane));
      const float4 mn = *reinterpret_cast<const float4*>(rec[j] + swz(L.k_xmin() + 16 * lane));
      stp_w[j * 32] = make_float4(st.x * cf.x, st.y * cf.y, st.z * cf.z, st.w * cf.w);
      esc_w[j * 32] = make_float4(fmaf(-4.f * cf.x, st.x, mn.x), fmaf(-4.f * cf.y, st.y, mn.y),
                                  fmaf(-4.f * cf.z, st.z, mn.z), fmaf(-4.f * cf.w, st.w, mn.w));
      // K code words (ldmatrix: token g / g+8, words tig and 4+tig)
#pragma unroll
      for (int mt = 0; mt < kMt; ++mt) ldsm_x4(kw[j][mt], rec_s[j] + swz(L.k_codes() + mt * 16 * 32 + lm_off));
    }
    __syncwarp();

    // ---- S = Q K^T: B operand q' = q4 * step * f as hi/lo fp16 pairs (channels m,
    // m+8) built one (hw, half) slice at a time; hi and lo accumulate into one chain
    float ch[NG][kMt][4];
#if !OTT_SINGLE_CHAIN
    float cl[NG][kMt][4];
#endif
    float2 bias2[NG];
#if OTT_Q_IN_REGS
    // (q4 lives in registers, loaded once per CTA: qreg[hw][v4])
#endif
#pragma unroll
    for (int j = 0; j < NG; ++j) {
      bias2[j] = make_float2(0.f, 0.f);
#pragma unroll
      for (int mt = 0; mt < kMt; ++mt) {
        ch[j][mt][0] = ch[j][mt][1] = ch[j][mt][2] = ch[j][mt][3] = 0.f;
#if !OTT_SINGLE_CHAIN
        cl[j][mt][0] = cl[j][mt][1] = cl[j][mt][2] = cl[j][mt][3] = 0.f;
#endif
      }
    }
#pragma unroll
    for (int hw = 0; hw < 2; ++hw) {
#pragma unroll
      for (int half = 0; half < 2; ++half) {  // pairs m = 4*half .. 4*half+3 (channels m, m+8)
#pragma unroll
        for (int j = 0; j < NG; ++j) {
          uint32_t bh[4], bl[4];
#pragma unroll
          for (int pp = 0; pp < 2; ++pp) {  // v4 = half (channels 4*half..+3), v4 = 2 + half (+8)
            const int v4 = half + 2 * pp;
#if OTT_Q_IN_REGS
            const float4 q4 = qreg[hw][v4];
#else
            const float4 q4 = sm.q4p[hw][v4][lane];
#endif
            const float4 s4 = sm.stp[warp][j][hw][tile_slot(v4, tig)];
            const float4 e4 = sm.esc[warp][j][hw][tile_slot(v4, tig)];
            const float2 q0 = make_float2(q4.x, q4.y), q1 = make_float2(q4.z, q4.w);
            const float2 B0 = __fmul2_rn(q0, make_float2(s4.x, s4.y));
            const float2 B1 = __fmul2_rn(q1, make_float2(s4.z, s4.w));
            bias2[j] = __ffma2_rn(q0, make_float2(e4.x, e4.y), bias2[j]);
            bias2[j] = __ffma2_rn(q1, make_float2(e4.z, e4.w), bias2[j]);
            const float2 h0 = make_float2(__uint_as_float(__float_as_uint(B0.x) & 0xFFFFE000u),
                                          __uint_as_float(__float_as_uint(B0.y) & 0xFFFFE000u));
            const float2 h1 = make_float2(__uint_as_float(__float_as_uint(B1.x) & 0xFFFFE000u),
                                          __uint_as_float(__float_as_uint(B1.y) & 0xFFFFE000u));
            const float2 l0 = __fadd2_rn(B0, make_float2(-h0.x, -h0.y));
            const float2 l1 = __fadd2_rn(B1, make_float2(-h1.x, -h1.y));
            if (pp == 0) {  // low channel of each pair
              bh[0] = __float_as_uint(h0.x); bh[1] = __float_as_uint(h0.y);
              bh[2] = __float_as_uint(h1.x); bh[3] = __float_as_uint(h1.y);
              bl[0] = __float_as_uint(l0.x); bl[1] = __float_as_uint(l0.y);
              bl[2] = __float_as_uint(l1.x); bl[3] = __float_as_uint(l1.y);
            } else {  // pack (low, high = channel + 8)
              bh[0] = pack_h2(__uint_as_float(bh[0]), h0.x); bh[1] = pack_h2(__uint_as_float(bh[1]), h0.y);
              bh[2] = pack_h2(__uint_as_float(bh[2]), h1.x); bh[3] = pack_h2(__uint_as_float(bh[3]), h1.y);
              bl[0] = pack_h2(__uint_as_float(bl[0]), l0.x); bl[1] = pack_h2(__uint_as_float(bl[1]), l0.y);
              bl[2] = pack_h2(__uint_as_float(bl[2]), l1.x); bl[3] = pack_h2(__uint_as_float(bl[3]), l1.y);
            }
          }
          // slice-major over the m-tiles so consecutive HMMAs feed different
          // accumulators (hi -> ch, lo -> cl per m-tile: 2*kMt independent chains)
          Shifted s0[kMt], s1[kMt];
#pragma unroll
          for (int mt = 0; mt < kMt; ++mt) {
            s0[mt] = shifted(kw[j][mt][2 * hw]);
            s1[mt] = shifted(kw[j][mt][2 * hw + 1]);
          }
#define OTT_QK(MM)                                                                        \
  {                                                                                       \
    _Pragma("unroll") for (int mt = 0; mt < kMt; ++mt) {                                  \
      const uint32_t a0 = kq<MM>(s0[mt], magic), a1 = kq<MM>(s1[mt], magic);             \
      const uint32_t a2 = kq<MM + 1>(s0[mt], magic), a3 = kq<MM + 1>(s1[mt], magic);     \
      mma16816(ch[j][mt], a0, a1, a2, a3, bh[(MM) & 3], bh[((MM) & 3) + 1]);              \
      mma16816(OTT_LO_ACC[j][mt], a0, a1, a2, a3, bl[(MM) & 3], bl[((MM) & 3) + 1]);      \
    }                                                                                     \
  }
          if (half == 0) {
            OTT_QK(0) OTT_QK(2)
          } else {
            OTT_QK(4) OTT_QK(6)
          }
#undef OTT_QK
        }
      }
    }
    float sc[NG][kMt][4];
#pragma unroll
    for (int j = 0; j < NG; ++j) {
      float bias = bias2[j].x + bias2[j].y;
      bias += __shfl_xor_sync(0xffffffffu, bias, 1);
      bias += __shfl_xor_sync(0xffffffffu, bias, 2);
      bias *= 0.25f;
      const float bias0 = __shfl_sync(0xffffffffu, bias, 8 * tig);      // head 2*tig
      const float bias1 = __shfl_sync(0xffffffffu, bias, 8 * tig + 4);  // head 2*tig+1
      const bool dummy = j >= ng;
#pragma unroll
      for (int mt = 0; mt < kMt; ++mt) {
#if !OTT_SINGLE_CHAIN
#pragma unroll
        for (int q = 0; q < 4; ++q) ch[j][mt][q] += cl[j][mt][q];
#endif
        sc[j][mt][0] = dummy ? -INFINITY : ch[j][mt][0] + bias0;
        sc[j][mt][1] = dummy ? -INFINITY : ch[j][mt][1] + bias1;
        sc[j][mt][2] = dummy ? -INFINITY : ch[j][mt][2] + bias0;
        sc[j][mt][3] = dummy ? -INFINITY : ch[j][mt][3] + bias1;
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

__device__ __forceinline__ void tma_row(uint32_t dst, const void* src, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];\n" ::"r"(dst),
      "l"(src), "r"(bar)
      : "memory");
}

template <int NR>
__device__ void fp_body(const AttnArgs& a, FpSmem& sm) {
  constexpr int D = 128, kRow = FpSmem::kRow;
  const ott_cache_t& c = a.c;
  const int u = blockIdx.x, split = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tig = lane & 3;
  const int N = c.capacity, cap = c.group_size + c.residual;
  const int n_pool_t = (N + 15) / 16;
  const int Tp = (int)(a.total_tokens - a.q_tokens);
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
  __syncwarp();

  float o[8][4];
#pragma unroll
  for (int j = 0; j < 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float mrun[2] = {-INFINITY, -INFINITY}, lsum[2] = {0.f, 0.f};
  // ldmatrix lane addressing (row, byte column) for K (non-trans) and V (trans)
  const int k_row = (lane & 7) + ((lane >> 3) & 1) * 8, k_col = (lane >> 4) * 16;
  const int v_row = (lane & 7) + ((lane >> 4) & 1) * 8, v_col = ((lane >> 3) & 1) * 16;
  uint32_t phase = 0;

  for (int t = warp; t < n_tiles; t += kAttnWarps) {
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
      for (int r = 0; r < rows; ++r) {
        size_t off;
        if (is_pool) {
          off = ((size_t)u * N + 16 * t + r) * D;
        } else {
          const int64_t p = a.q_tokens + 16 * (t - n_pool_t) + r;
          off = ((size_t)u * cap + (size_t)(p % cap)) * D;
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
  __syncthreads();
  float* accw = reinterpret_cast<float*>(&sm.kr[warp][0][0]);  // [8 heads][128]
#pragma unroll
  for (int j = 0; j < 8; ++j) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      accw[(2 * tig + h) * D + 16 * j + g] = o[j][h];
      accw[(2 * tig + h) * D + 16 * j + 8 + g] = o[j][h + 2];
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
  if ((int)blockIdx.y == a.n_qsplits) {  // full-precision tiers: pool.entries + pending window
    fp_body<NR>(a, *reinterpret_cast<FpSmem*>(smem_raw));
  } else {
    mma_body<NR, G>(a, &tmap, *reinterpret_cast<MmaSmem<G>*>(smem_raw));
  }
}

// ============================================================ combine + debug logits
template <int D>
__global__ void combine_kernel(const float* __restrict__ ws, uint16_t* __restrict__ out, int n_splits) {
  const int ur = blockIdx.x;  // unit*NR + r
  const float* base = ws + (size_t)ur * n_splits * (D + 2);
  float M = -INFINITY;
  for (int s = 0; s < n_splits; ++s) M = fmaxf(M, base[(size_t)s * (D + 2)]);
  for (int col = threadIdx.x; col < D; col += blockDim.x) {
    float Lsum = 0.f, A = 0.f;
    for (int s = 0; s < n_splits; ++s) {
      const float* p = base + (size_t)s * (D + 2);
      if (p[0] == -INFINITY) continue;
      const float f = exp2f(p[0] - M);
      Lsum += p[1] * f;
      A += p[2 + col] * f;
    }
    out[(size_t)ur * D + col] = f2h(A / Lsum);
  }
}

template <int D>
__global__ void logits_kernel(ott_cache_t c, const uint16_t* __restrict__ q, float* __restrict__ logits, int NR,
                              int64_t q_tokens, int64_t total, float inv_sqrt_d) {
  const int u = blockIdx.y;
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= total) return;
  const int G = c.group_size, N = c.capacity, cap = G + c.residual;
  const RecordLayout L(D, G);
  float k[D];
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
      const uint32_t* kcw = reinterpret_cast<const uint32_t*>(rec + L.k_codes()) + (size_t)row * (D / 16);
      const float* kstep = reinterpret_cast<const float*>(rec + L.k_step());
      const float* kxmin = reinterpret_cast<const float*>(rec + L.k_xmin());
      for (int j = 0; j < D; ++j) k[j] = fmaf((float)((kcw[j / 16] >> (2 * (j % 16))) & 3u), kstep[j], kxmin[j]);
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
  combine_kernel<D><<<a.c.n_units * NR, D, 0, st>>>(a.ws, a.out, a.n_splits);
  return cudaGetLastError();
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
  combine_kernel<128><<<a.c.n_units * NR, 128, 0, st>>>(a.ws, a.out, a.n_splits);
  return cudaGetLastError();
}

bool mma_eligible(const ott_cache_t& c) { return c.head_dim == 128; }

cudaError_t launch_attend(const ott_cache_t& c, const uint16_t* q, uint16_t* out, int n_rep, int64_t q_tokens,
                          int64_t total, float* ws, int n_qsplits, cudaStream_t st) {
  AttnArgs a;
  a.c = c;
  a.q = q;
  a.out = out;
  a.ws = ws;
  a.q_tokens = q_tokens;
  a.total_tokens = total;
  a.n_qsplits = n_qsplits;
  a.n_splits = n_qsplits + 1;
  a.n_qtiles = (int)(q_tokens / 32);
  a.n_ptiles = (c.capacity + 31) / 32;
  a.n_rtiles = (int)((total - q_tokens + 31) / 32);
  a.scale_log2 = kLog2e / sqrtf((float)c.head_dim);
  a.k_magic = 0x3C003C00u;
  const int D = c.head_dim, G = c.group_size;
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

cudaError_t launch_logits(const ott_cache_t& c, const uint16_t* q, float* logits, int n_rep, int64_t q_tokens,
                          int64_t total, cudaStream_t st) {
  dim3 grid((unsigned)((total + 127) / 128), c.n_units);
  const float inv = 1.0f / sqrtf((float)c.head_dim);
  if (c.head_dim == 128) logits_kernel<128><<<grid, 128, 0, st>>>(c, q, logits, n_rep, q_tokens, total, inv);
  else if (c.head_dim == 64) logits_kernel<64><<<grid, 128, 0, st>>>(c, q, logits, n_rep, q_tokens, total, inv);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

}  // namespace ott
