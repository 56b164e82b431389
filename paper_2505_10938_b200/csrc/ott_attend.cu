// ott_attend.cu — K2/K3: split-K flash-decoding attention over the three cache
// tiers (attend_mixed, attention.py:79-92), CUDA-core (SIMT) variant, plus the
// split combine and a debug logits kernel.
//
// Per unit (batch b, kv head h) the token axis is cut into 32-token tiles:
//   [0, Tq/32)               quantized tiles (codes dequantized in registers;
//                            positions currently in pool.entries masked, they
//                            are represented by the pool tile instead —
//                            attention.py:73-75 overwrite semantics)
//   next ceil(N/32) tiles    pool.entries rows (fp16, exact)
//   next ceil(Tp/32) tiles   pending rows (fp16 ring)
// Splits take contiguous tile ranges; each warp keeps an online softmax state
// per query head; warps then splits are merged (log-sum-exp).
#include "ott_common.cuh"

namespace ott {

constexpr int kAttnThreads = 128;
constexpr int kAttnWarps = kAttnThreads / 32;
constexpr float kLog2e = 1.4426950408889634f;

struct AttnArgs {
  ott_cache_t c;
  const uint16_t* q;
  uint16_t* out;
  float* ws;  // [n_units][NR][S][D+2]
  int64_t q_tokens, total_tokens;
  int n_splits, n_qtiles, n_ptiles, n_rtiles;
  float scale_log2;  // log2(e) / float32(sqrt(d))
};

// Per-warp smem scratch for one tile.
template <int NR, int D>
struct WarpScratch {
  float qp[NR][D];     // q * step (quantized tiles) — folded K step
  float p[NR][32];     // softmax numerators of the tile
  uint32_t vw[32][D / 16];
  float vstep[32], vxmin[32];
};

template <int NR, int D>
struct AttnSmem {
  float qs[NR][D];  // q * scale_log2
  WarpScratch<NR, D> w[kAttnWarps];
  float m[kAttnWarps][NR], l[kAttnWarps][NR];
  float acc[kAttnWarps][NR][D];
};

template <int NR, int D>
__device__ __forceinline__ void online_update(float (&s)[NR], float (&m)[NR], float (&l)[NR], float (&acc)[NR][D / 32],
                                              WarpScratch<NR, D>& ws, int lane) {
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const float tmax = warp_max(s[r]);
    const float m_new = fmaxf(m[r], tmax);
    if (m_new == -INFINITY) {  // whole tile masked and nothing seen yet
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

template <int NR, int D>
__global__ void __launch_bounds__(kAttnThreads) attend_simt_kernel(AttnArgs a) {
  const ott_cache_t& c = a.c;
  const int u = blockIdx.x, split = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = c.group_size, N = c.capacity, cap = G + c.residual;
  const RecordLayout L(D, G);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  AttnSmem<NR, D>& sm = *reinterpret_cast<AttnSmem<NR, D>*>(smem_raw);
  WarpScratch<NR, D>& ws = sm.w[warp];

  for (int i = tid; i < NR * D; i += kAttnThreads)
    sm.qs[i / D][i % D] = h2f(a.q[((size_t)u * NR) * D + i]) * a.scale_log2;
  __syncthreads();

  const int n_tiles = a.n_qtiles + a.n_ptiles + a.n_rtiles;
  const int per = (n_tiles + a.n_splits - 1) / a.n_splits;
  const int t_begin = split * per;
  const int t_end = min(n_tiles, t_begin + per);

  float m[NR], l[NR], acc[NR][D / 32];
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    m[r] = -INFINITY;
    l[r] = 0.f;
#pragma unroll
    for (int k = 0; k < D / 32; ++k) acc[r][k] = 0.f;
  }
  const uint32_t* pmask = c.pool_mask + (size_t)u * mask_words_per_unit(c);
  const int n_entries = N > 0 ? c.pool_meta[(size_t)u * 4] : 0;
  (void)n_entries;

  for (int t = t_begin + warp; t < t_end; t += kAttnWarps) {
    float s[NR];
    if (t < a.n_qtiles) {
      // ---------------- quantized tile: 32 tokens of one group
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
      // V codes / params of this tile into warp smem
      const uint32_t* vcw = reinterpret_cast<const uint32_t*>(rec + L.v_codes()) + (size_t)row0 * (D / 16);
#pragma unroll
      for (int j = 0; j < D / 16; ++j) {
        const int idx = j * 32 + lane;
        ws.vw[idx / (D / 16)][idx % (D / 16)] = vcw[idx];
      }
      ws.vstep[lane] = reinterpret_cast<const float*>(rec + L.v_step())[row0 + lane];
      ws.vxmin[lane] = reinterpret_cast<const float*>(rec + L.v_xmin())[row0 + lane];
      __syncwarp();
      // logits, lane = token
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
      // P . V with V dequantized per token: v = code*step_t + xmin_t
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
      // ---------------- full-precision tile: pool entries or pending rows
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
      // P . V: lane owns channels lane + 32k; row pointers broadcast per token
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

  // ---- merge warps of this CTA, write the split partial
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

// K3: merge split partials -> fp16 output. One CTA per (unit, head).
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

// Debug K: reference logits (attention.py:55) for every position.
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

template <int NR, int D>
static cudaError_t launch_attend_t(const AttnArgs& a, cudaStream_t st) {
  const size_t smem = sizeof(AttnSmem<NR, D>);
  cudaError_t e = cudaFuncSetAttribute(attend_simt_kernel<NR, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(a.c.n_units, a.n_splits);
  attend_simt_kernel<NR, D><<<grid, kAttnThreads, smem, st>>>(a);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  combine_kernel<D><<<a.c.n_units * NR, D, 0, st>>>(a.ws, a.out, a.n_splits);
  return cudaGetLastError();
}

cudaError_t launch_attend(const ott_cache_t& c, const uint16_t* q, uint16_t* out, int n_rep, int64_t q_tokens,
                          int64_t total, float* ws, int n_splits, cudaStream_t st) {
  AttnArgs a;
  a.c = c;
  a.q = q;
  a.out = out;
  a.ws = ws;
  a.q_tokens = q_tokens;
  a.total_tokens = total;
  a.n_splits = n_splits;
  a.n_qtiles = (int)(q_tokens / 32);
  a.n_ptiles = (c.capacity + 31) / 32;
  a.n_rtiles = (int)((total - q_tokens + 31) / 32);
  a.scale_log2 = kLog2e / sqrtf((float)c.head_dim);
  const int D = c.head_dim;
#define OTT_CASE(NRv, Dv) \
  if (n_rep == NRv && D == Dv) return launch_attend_t<NRv, Dv>(a, st);
  OTT_CASE(1, 128) OTT_CASE(2, 128) OTT_CASE(4, 128) OTT_CASE(8, 128)
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
