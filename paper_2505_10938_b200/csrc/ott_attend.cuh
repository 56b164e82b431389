// ott_attend.cuh — shared pieces of the attention kernels (K2/K3): launch arguments,
// token counts, warp-level tensor-core and TMA helpers, and the full-precision-tier body
// (pool.entries + pending ring, attention.py:62-76) used by every tensor-core kernel.
#pragma once
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
  int tail_units;                    // > 0 (2-bit tensor-core kernel): 1-D grid of [whole units]
                                     // [the last tail_units units cut into n_qsplits pieces each]
                                     // [fp-tier CTAs]: small work items finish the launch
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



// ============================================================ tensor-core helpers
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

__device__ __forceinline__ void cp_async16_s(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void tma_row(uint32_t dst, const void* src, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];\n" ::"r"(dst),
      "l"(src), "r"(bar)
      : "memory");
}

// (u, split) = unit and partial slot of this CTA: split - n_qsplits is its fp-tier index
template <int NR>
__device__ void fp_body(const AttnArgs& a, const Counts& n, FpSmem& sm, int u, int split) {
  constexpr int D = 128, kRow = FpSmem::kRow;
  const ott_cache_t& c = a.c;
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
  const uint32_t kr_s = (uint32_t)__cvta_generic_to_shared(&sm.kr[warp][0][0]);
  const uint32_t vr_s = (uint32_t)__cvta_generic_to_shared(&sm.vr[warp][0][0]);
  if (a.new_k) {  // fused ring write (cache.py:134-135): this CTA alone reads the pending tier
    if (tid < 2 * D / 8) {
      const size_t dst = ((size_t)u * cap + (size_t)((n.total_tokens - 1) % cap)) * D + (tid % (D / 8)) * 8;
      const uint16_t* src = (tid < D / 8 ? a.new_k : a.new_v) + (size_t)u * D + (tid % (D / 8)) * 8;
      *reinterpret_cast<uint4*>((tid < D / 8 ? c.pend_k : c.pend_v) + dst) = *reinterpret_cast<const uint4*>(src);
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

  // the fp-tier CTAs of a unit (n_fsplits of them) interleave the 16-row tiles warp by warp
  const int f = split - a.n_qsplits;
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
    {  // stage the tile's rows: 16-byte cp.async per lane (lane = chunk lane % 16 of rows 2 it + lane / 16)
      const int rows = is_pool ? min(16, N - 16 * t) : min(16, Tp - 16 * (t - n_pool_t));
      // ring slot of the tile's first pending row (one modulo per tile); cap >= 32 > 16 rows
      const int slot0 = is_pool ? 0 : (int)((n.q_tokens + 16 * (t - n_pool_t)) % cap);
      const int ch = lane & 15;
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int r = 2 * it + (lane >> 4);
        if (r < rows) {
          size_t off;
          if (is_pool) {
            off = ((size_t)u * N + 16 * t + r) * D;
          } else {
            const int sl = slot0 + r >= cap ? slot0 + r - cap : slot0 + r;
            off = ((size_t)u * cap + (size_t)sl) * D;
          }
          cp_async16_s(kr_s + r * kRow + 16 * ch, (is_pool ? c.pool_k : c.pend_k) + off + 8 * ch);
          cp_async16_s(vr_s + r * kRow + 16 * ch, (is_pool ? c.pool_v : c.pend_v) + off + 8 * ch);
        }
      }
      asm volatile("cp.async.wait_all;\n" ::: "memory");
      __syncwarp();
    }

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
    __syncwarp();  // the next tile's cp.async overwrites the staging rows
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

// launchers shared between the attention translation units (ott_attend.cu)
cudaError_t record_tensor_map(const ott_cache_t& c, int box_rows, int rec_rows, CUtensorMap* map);
cudaError_t launch_combine_tc128(const AttnArgs& a, int NR, cudaStream_t st);

}  // namespace ott
