// ott_flush.cu — K1 (group flush: score -> pool competition -> mean substitution
// -> 2-bit floor quantization -> bit packing) and K4 (pending-ring write).
//
// Bit-exactness contract: every float64 operation below is an explicit
// round-to-nearest intrinsic (__dadd_rn/__dsub_rn/__dmul_rn/__ddiv_rn), so no
// fused multiply-add can change a result; this TU is also compiled with
// -fmad=false. For fp16-valued inputs, L1 scores and group means are exact
// float64 sums in any summation order, so they match numpy's pairwise sums.
#include "ott_common.cuh"

namespace ott {

constexpr int kFlushThreads = 256;
#ifndef OTT_FROZEN_SEL  // timing experiment only when 0 (substituted groups quantized wrongly)
#define OTT_FROZEN_SEL 1
#endif
#ifndef OTT_FLUSH_PRESCORE  // parallel token scoring ahead of the pool scan when N < A
#define OTT_FLUSH_PRESCORE 1
#endif
#ifndef OTT_FLUSH_SPLIT  // bulk flush = sequential kernel until the pool freezes + parallel frozen-pool kernel
#define OTT_FLUSH_SPLIT 1
#endif
#ifndef OTT_FLUSH_MIN_BLOCKS
#define OTT_FLUSH_MIN_BLOCKS 3  // <= 85 registers: 3 CTAs per SM for large unit counts
#endif

// quant.py:59-102 for one line held in registers/smem by ONE thread.
// levels = 2^bits - 1. Returns step.
__device__ __forceinline__ void line_params(double mn, double mx, double levels, double& step_out) {
  const double range = __dsub_rn(mx, mn);
  double step;
  if (levels == 3.0) {  // RN(range / 3) by Markstein's FMA correction of RN(range * RN(1/3)): exact
    const double c = 1.0 / 3.0;
    const double q0 = __dmul_rn(range, c);
    step = __fma_rn(__fma_rn(-q0, 3.0, range), c, q0);
  } else {
    step = __ddiv_rn(range, levels);  // quant.py:64
  }
  // quant.py:68-69: while step > 0 and x_min + levels*step > x_max: nextafter(step, 0)
  while (step > 0.0 && __dadd_rn(mn, __dmul_rn(levels, step)) > mx)
    step = __longlong_as_double(__double_as_longlong(step) - 1);
  step_out = step;
}

// quant.py:91-102 for one element x (float32) of a line with x_min mn = (double)mnf,
// x_max mxf, step and inv = __drcp_rn(step). The line-wide rules come first, so the
// element equal to the max (quant.py:101) and the one equal to the min (code 0) never
// reach the division. floor((x - mn) / step) of quant.py:93 is taken from the product
// (x - mn) * inv when its fractional part lies more than eps = 1e-9 (levels + 1) from an
// integer: the product and the correctly rounded quotient differ by < 4e-16 relative,
// so both floor to the same integer; otherwise (exact lattice points, ties) the IEEE
// division decides. x > mn here, so the product is positive.
__device__ __forceinline__ int quant_code(float xf, float mnf, float mxf, double mn, double step, double inv,
                                          int levels, double eps) {
  if (step == 0.0) return 0;     // quant.py:91-92
  if (xf == mxf) return levels;  // quant.py:101
  if (xf == mnf) return 0;       // (x - mn) / step == 0; the check below keeps 0
  const double x = (double)xf;
  const double dd = __dsub_rn(x, mn);
  const double qa = __dmul_rn(dd, inv);
  double f = floor(qa);
  const double t = __dsub_rn(qa, f);
  if (!(t > eps && t < 1.0 - eps)) f = floor(__ddiv_rn(dd, step));
  int c = min(__double2int_rz(f), levels);                     // quant.py:94 (f >= 0)
  if (__dadd_rn(__dmul_rn((double)c, step), mn) > x) c -= 1;  // quant.py:97
  return max(c, 0);                                            // quant.py:98
}

// Per-line constants of the float32 fast path. For x in (x_min, x_max) the quotient
// q = (x - x_min) / step lies in (0, levels + 1); q32 = f32(f32(x - x_min) * f32(1/step)) is
// within 3 * 2^-24 * q (< del / 2) of it. When frac(q32) lies in (del, 1 - del),
// floor(q32) is the reference's floor of the float64 quotient, and when also
// max(|x_min|, |x_max|) <= 1e8 * step the float64 check c * step + x_min > x
// (quant.py:97) cannot fire (its rounding error is < 2^-51 * 1e8 * step < del / 2 * step),
// so the element needs no float64 work. Other elements and lines take quant_code.
struct FastLine {
  float inv32, del;
  bool ok;
};
__device__ __forceinline__ FastLine fast_line(float mnf, float mxf, double step, double inv, int levels) {
  FastLine f;
  f.ok = step >= 1e-30 && step <= 1e30 && fmaxf(fabsf(mnf), fabsf(mxf)) <= (float)(1e8 * step);
  f.inv32 = (float)inv;
  f.del = 4e-7f * (float)(levels + 1);
  return f;
}
// The rare float64 fallback as a call: inlined at every element of the unrolled loops it
// would multiply the code size (instruction-cache misses)
__device__ __noinline__ int quant_code_slow(float xf, float mnf, float mxf, double mn, double step, double inv,
                                            int levels, double eps) {
  return quant_code(xf, mnf, mxf, mn, step, inv, levels, eps);
}

// Branch-free float32 code of x; `slow` marks elements that need quant_code (line not
// eligible, or frac(q32) inside the guard band). x == x_min gives q32 = 0 and code 0
// exactly (f32 x - x_min is 0 only for equal values); x == x_max is the max rule.
__device__ __forceinline__ int quant_code_f32(float xf, float mnf, float mxf, int levels, const FastLine& fl,
                                              bool& slow) {
  const float q = __fmul_rn(__fsub_rn(xf, mnf), fl.inv32);
  const float f = floorf(q), t = __fsub_rn(q, f);
  const bool is_max = xf == mxf;
  slow = !fl.ok || (!(t > fl.del && t < 1.f - fl.del) && q != 0.f && !is_max);
  // f is an integer in [0, levels] when !slow (q < levels + 1 - del for x < x_max):
  // f + 2^23 holds it in the low mantissa bits
  return is_max ? levels : __float_as_int(__fadd_rn(f, 8388608.f)) - 0x4B000000;
}

// 8 fp16 -> 8 float32 in shared memory with two 16-byte stores (8 scalar stores at a
// 32-byte lane stride would be 8-way bank conflicts)
__device__ __forceinline__ void store8(float* dst, const uint4& h) {
  const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&h.x));
  const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&h.y));
  const float2 c = __half22float2(*reinterpret_cast<const __half2*>(&h.z));
  const float2 d = __half22float2(*reinterpret_cast<const __half2*>(&h.w));
  reinterpret_cast<float4*>(dst)[0] = make_float4(a.x, a.y, b.x, b.y);
  reinterpret_cast<float4*>(dst)[1] = make_float4(c.x, c.y, d.x, d.y);
}
// 4 two-bit codes held one per byte (values <= 3) -> one byte, code j at bits 2j
__device__ __forceinline__ uint32_t pack4x2(uint32_t w) {
  w = (w | (w >> 6)) & 0x000F000Fu;
  return (w | (w >> 12)) & 0xFFu;
}

struct FlushShared {
  int n_entries, n_aux, frozen, any_selected;
  int n_evicted, n_win_cand;
};

// Dynamic smem layout, sized on the host (flush_smem_bytes):
//   fp16   sk[G*d], sv[G*d]           group rows as staged (fp16, the inputs' own format)
//   float  kmean[d], vmean[d]         column means that replace the substituted rows
//   uint8  kc[G*d], vc[G*d]           codes (16-byte aligned when G*d % 16 == 0)
//   double score[G]                   (8-byte aligned)
//   double it_score[N+G]; int it_pos[N+G]; int it_rank[N+G]
//   int    free_slot[N]; uint8 sel[G]
__host__ __device__ inline size_t flush_codes_offset(int d, int G) { return ((size_t)4 * G * d + 8 * (size_t)d + 15) & ~(size_t)15; }
__host__ __device__ inline size_t flush_score_offset(int d, int G) { return (flush_codes_offset(d, G) + (size_t)2 * G * d + 7) & ~(size_t)7; }
__host__ __device__ inline size_t flush_smem_bytes(int d, int G, int N) {
  size_t b = flush_score_offset(d, G);
  b += (size_t)G * sizeof(double);
  b += (size_t)(N + G) * (sizeof(double) + 2 * sizeof(int));
  b += (size_t)(N > 0 ? N : 1) * sizeof(int);
  b += (size_t)G;
  return (b + 15) & ~(size_t)15;
}

__global__ void __launch_bounds__(kFlushThreads, OTT_FLUSH_MIN_BLOCKS) flush_kernel(ott_cache_t c, int64_t q0, int n_groups,
                                                              int64_t ring_end, const uint16_t* __restrict__ in_k,
                                                              const uint16_t* __restrict__ in_v,
                                                              int64_t in_stride, int64_t in_first,
                                                              const int64_t* __restrict__ dev_counts) {
  if (dev_counts) {  // device-counter decode step: flush one group iff the append just made it due
    const int64_t qt = dev_counts[0], tot = dev_counts[1] + 1;
    if (tot - qt - c.residual < c.group_size || qt / c.group_size + 1 > c.max_groups) return;
    q0 = qt;
    n_groups = 1;
    ring_end = tot;
  }
  const int u = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = kFlushThreads / 32;
  const int d = c.head_dim, G = c.group_size, N = c.capacity, A = c.aux_capacity;
  const int cap = G + c.residual;
  const RecordLayout L(d, G, c.bits);
  const int levels = (1 << c.bits) - 1;
  const double eps = 1e-9 * (double)(levels + 1);  // guard band of quant_code (qa <= levels + 1)

  extern __shared__ __align__(16) unsigned char smem[];
  uint16_t* sk = reinterpret_cast<uint16_t*>(smem);
  uint16_t* sv = sk + G * d;
  float* kmean = reinterpret_cast<float*>(sv + G * d);
  float* vmean = kmean + d;
  uint8_t* kc = smem + flush_codes_offset(d, G);
  uint8_t* vc = kc + G * d;
  double* score = reinterpret_cast<double*>(smem + flush_score_offset(d, G));
  double* it_score = score + G;
  int* it_pos = reinterpret_cast<int*>(it_score + N + G);
  int* it_rank = it_pos + N + G;
  int* free_slot = it_rank + N + G;
  uint8_t* sel = reinterpret_cast<uint8_t*>(free_slot + (N > 0 ? N : 1));
  __shared__ FlushShared sh;

  int32_t* meta = c.pool_meta + (size_t)u * 4;
  int32_t* ppos = c.pool_pos + (size_t)u * N;
  double* pscore = c.pool_score + (size_t)u * N;
  uint16_t* pk = c.pool_k + (size_t)u * N * d;
  uint16_t* pv = c.pool_v + (size_t)u * N * d;
  int32_t* apos = c.aux_pos + (size_t)u * A;
  double* ascore = c.aux_score + (size_t)u * A;
  uint16_t* ak = c.aux_k + (size_t)u * A * d;
  uint16_t* av = c.aux_v + (size_t)u * A * d;
  uint32_t* pmask = c.pool_mask + (size_t)u * mask_words_per_unit(c);
  uint32_t* smask = c.subst_mask + (size_t)u * mask_words_per_unit(c);

  if (tid == 0) {
    sh.n_entries = meta[0];
    sh.n_aux = meta[1];
    sh.frozen = meta[2];
  }
  __syncthreads();

  // the first kPre row loads of the next group are issued into registers before the
  // current group is processed, so their global latency overlaps its compute. Positions
  // fit in int32 (checked by ott_flush); a row's ring slot is (base % cap + row) with one
  // conditional subtraction, since row < G <= cap.
  constexpr int kPre = 2;
  uint4 pk8[kPre], pv8[kPre];
  const int ring_end32 = (int)ring_end, in_first32 = (int)in_first;
#define OTT_ROW_SRC(BASE, BSLOT, ROW, COL, SK, SV)                                     \
  {                                                                                    \
    const int p_ = (BASE) + (ROW);                                                     \
    if (p_ < ring_end32) {                                                             \
      int s_ = (BSLOT) + (ROW);                                                        \
      s_ = s_ >= cap ? s_ - cap : s_;                                                  \
      const size_t off_ = ((size_t)u * cap + (size_t)s_) * d + (COL);                  \
      SK = c.pend_k + off_;                                                            \
      SV = c.pend_v + off_;                                                            \
    } else {                                                                           \
      const size_t off_ = (size_t)u * in_stride + (size_t)(p_ - in_first32) * d + (COL); \
      SK = in_k + off_;                                                                \
      SV = in_v + off_;                                                                \
    }                                                                                  \
  }
  int prow[kPre], pcol[kPre];  // this thread's (row, column) of prefetch slot it
#pragma unroll
  for (int it = 0; it < kPre; ++it) {
    const int e = tid * 8 + it * kFlushThreads * 8;
    prow[it] = e / d;
    pcol[it] = e % d;
  }
#define OTT_PREFETCH(BASE)                                              \
  {                                                                     \
    const int b_ = (int)(BASE), bs_ = b_ % cap;                         \
    _Pragma("unroll") for (int it = 0; it < kPre; ++it) {               \
      if (tid * 8 + it * kFlushThreads * 8 < G * d) {                   \
        const uint16_t *sk_, *sv_;                                      \
        OTT_ROW_SRC(b_, bs_, prow[it], pcol[it], sk_, sv_)              \
        pk8[it] = *reinterpret_cast<const uint4*>(sk_);                 \
        pv8[it] = *reinterpret_cast<const uint4*>(sv_);                 \
      }                                                                 \
    }                                                                   \
  }
  // 8-half vector loads need rows of whole 16-byte chunks; other head dims gather per element
  const bool vec = d % 8 == 0;
  if (n_groups > 0 && vec) OTT_PREFETCH(q0)

  for (int g = 0; g < n_groups; ++g) {
    const int64_t base = q0 + (int64_t)g * G;
    const int64_t gi = base / G;
    uint8_t* rec = record_ptr(c, u, gi);
    const int base32 = (int)base, bslot = base32 % cap;

    // ---- 1. gather the oldest G pending rows (cache.py:155-156), fp16 -> f32
    if (!vec) {
      for (int e = tid; e < G * d; e += kFlushThreads) {
        const uint16_t *srck, *srcv;
        OTT_ROW_SRC(base32, bslot, e / d, e % d, srck, srcv)
        sk[e] = *srck;
        sv[e] = *srcv;
      }
    }
#pragma unroll
    for (int it = 0; it < kPre; ++it) {
      const int e = tid * 8 + it * kFlushThreads * 8;
      if (vec && e < G * d) {
        *reinterpret_cast<uint4*>(sk + e) = pk8[it];
        *reinterpret_cast<uint4*>(sv + e) = pv8[it];
      }
    }
    for (int e = tid * 8 + kPre * kFlushThreads * 8; vec && e < G * d; e += kFlushThreads * 8) {
      uint4 k8, v8;
      {
        const uint16_t *srck, *srcv;
        OTT_ROW_SRC(base32, bslot, e / d, e % d, srck, srcv)
        k8 = *reinterpret_cast<const uint4*>(srck);
        v8 = *reinterpret_cast<const uint4*>(srcv);
      }
      *reinterpret_cast<uint4*>(sk + e) = k8;
      *reinterpret_cast<uint4*>(sv + e) = v8;
    }
    if (g + 1 < n_groups && vec) OTT_PREFETCH(base + G)
    if (tid < G) sel[tid] = 0;
    if (tid == 0) sh.any_selected = 0;
    __syncthreads();

    const bool active = N > 0 && !sh.frozen;  // cache.py:158 (block-uniform)
    if (active) {
      // ---- 2a. score_tokens: L1 norm of each key row in float64 (outlier.py:45-49)
      for (int i = warp; i < G; i += nwarps) {
        double s = 0.0;
        for (int col = lane; col < d; col += 32) s = __dadd_rn(s, fabs((double)h2f(sk[i * d + col])));
        s = warp_sum(s);
        if (lane == 0) score[i] = s;
      }
      __syncthreads();
      // ---- 2b. OutlierPool.update (outlier.py:84-117), rank-by-count.
      // items [0, N): current slots (pos < 0 = empty); [N, N+G): candidates.
      const int M = N + G;
      for (int t = tid; t < M; t += kFlushThreads) {
        if (t < N) {
          it_pos[t] = ppos[t];
          it_score[t] = pscore[t];
        } else {
          it_pos[t] = (int)(base + (t - N));
          it_score[t] = score[t - N];
        }
      }
      __syncthreads();
      for (int t = tid; t < M; t += kFlushThreads) {
        int r = -1;
        if (it_pos[t] >= 0) {
          const double s = it_score[t];
          const int p = it_pos[t];
          r = 0;
          for (int j = 0; j < M; ++j) {
            if (it_pos[j] < 0) continue;
            const double sj = it_score[j];
            r += (sj < s || (sj == s && it_pos[j] < p)) ? 1 : 0;  // _rank, outlier.py:52-54
          }
        }
        it_rank[t] = r;
      }
      __syncthreads();
      // evicted old entries -> aux in old reference order (= ascending rank),
      // free slots listed in ascending slot index.
      if (tid < N) {
        const int r = it_rank[tid];
        const bool evicted = r >= N;
        const bool is_free = r < 0 || evicted;
        int fidx = 0;
        for (int s = 0; s < tid; ++s) {
          const int rs = it_rank[s];
          fidx += (rs < 0 || rs >= N) ? 1 : 0;
        }
        if (is_free) free_slot[fidx] = tid;
        if (evicted) {
          int eidx = 0;
          for (int s = 0; s < N; ++s) eidx += (it_rank[s] >= N && it_rank[s] < r) ? 1 : 0;
          const int room = A - sh.n_aux;  // outlier.py:113-114
          if (eidx < room) {
            const int a = sh.n_aux + eidx;
            apos[a] = it_pos[tid];
            ascore[a] = it_score[tid];
          }
          const int p = it_pos[tid];
          atomicAnd(&pmask[p >> 5], ~(1u << (p & 31)));  // back to its shadow row
        }
      }
      __syncthreads();
      if (tid == 0) {
        int n_ev = 0, n_old = 0;
        for (int s = 0; s < N; ++s) {
          n_ev += it_rank[s] >= N ? 1 : 0;
          n_old += it_rank[s] >= 0 ? 1 : 0;
        }
        int n_wc = 0;
        for (int i = 0; i < G; ++i) n_wc += it_rank[N + i] < N ? 1 : 0;
        sh.n_evicted = n_ev;
        sh.n_win_cand = n_wc;
        sh.any_selected = n_wc > 0;
      }
      __syncthreads();
      // copy evicted rows into aux before their slots are reused
      {
        const int room = A - sh.n_aux;
        for (int s = warp; s < N; s += nwarps) {
          const int r = it_rank[s];
          if (r < N) continue;
          int eidx = 0;
          for (int t = 0; t < N; ++t) eidx += (it_rank[t] >= N && it_rank[t] < r) ? 1 : 0;
          if (eidx >= room) continue;
          const int a = sh.n_aux + eidx;
          for (int col = lane; col < d; col += 32) {
            ak[(size_t)a * d + col] = pk[(size_t)s * d + col];
            av[(size_t)a * d + col] = pv[(size_t)s * d + col];
          }
        }
      }
      __syncthreads();
      // winning candidates take free slots in candidate order
      for (int i = warp; i < G; i += nwarps) {
        const int r = it_rank[N + i];
        if (r >= N) continue;
        int widx = 0;
        for (int j = 0; j < i; ++j) widx += it_rank[N + j] < N ? 1 : 0;
        const int s = free_slot[widx];
        for (int col = lane; col < d; col += 32) {
          pk[(size_t)s * d + col] = sk[i * d + col];  // original row
          pv[(size_t)s * d + col] = sv[i * d + col];
        }
        if (lane == 0) {
          ppos[s] = (int)(base + i);
          pscore[s] = score[i];
          sel[i] = 1;
          const int p = (int)(base + i);
          atomicOr(&pmask[p >> 5], 1u << (p & 31));
          atomicOr(&smask[p >> 5], 1u << (p & 31));  // cache.py:173
        }
      }
      __syncthreads();
      if (tid == 0) {
        const int room = A - sh.n_aux;
        sh.n_aux += sh.n_evicted < room ? sh.n_evicted : room;
        int n_e = 0;
        for (int t = 0; t < M; ++t) n_e += (it_rank[t] >= 0 && it_rank[t] < N) ? 1 : 0;
        sh.n_entries = n_e;
        if (sh.n_aux >= A) sh.frozen = 1;  // outlier.py:115-116
      }
      // ---- 2c. substitute_means (outlier.py:120-142): column means over the
      // ORIGINAL G rows, float64 accumulate, cast to float32, then overwrite.
      if (sh.any_selected) {
        for (int col = tid; col < d; col += kFlushThreads) {
          double mk = 0.0, mv = 0.0;
          for (int i = 0; i < G; ++i) {
            mk = __dadd_rn(mk, (double)h2f(sk[i * d + col]));
            mv = __dadd_rn(mv, (double)h2f(sv[i * d + col]));
          }
          kmean[col] = __double2float_rn(__ddiv_rn(mk, (double)G));  // read in place of the sel rows
          vmean[col] = __double2float_rn(__ddiv_rn(mv, (double)G));
        }
      }
      __syncthreads();
    }

    const bool subst = active && sh.any_selected;  // block-uniform: kmean/vmean hold this group's means
    // ---- 3. quantize: K per channel (threads [0,d) of the first ceil(d/32) warps), V per
    // token (the remaining warps; d <= 128 leaves at least 4)
    const int kwarps = (d + 31) / 32;
    double* p64 = c.params64 ? c.params64 + ((size_t)u * c.max_groups + (size_t)gi) * 2 * (d + G) : nullptr;
    __half* ksh = reinterpret_cast<__half*>(rec + L.k_sh());
    __half* ksl = reinterpret_cast<__half*>(rec + L.k_sl());
    float* ke = reinterpret_cast<float*>(rec + L.k_e());
    float* vstep = reinterpret_cast<float*>(rec + L.v_step());
    float* vxmin = reinterpret_cast<float*>(rec + L.v_xmin());
    if (warp < kwarps) {
      const int col = tid;
      const int kshift = (c.bits == 1 && L.bits == 2) ? 1 : 0;
      float kst = 0.f;
      if (col < d) {
        // rows selected by the pool competition read the column mean (outlier.py:120-142)
        const float km = subst ? kmean[col] : 0.f;
        auto kx = [&](int i) { return (subst && sel[i]) ? km : h2f(sk[i * d + col]); };
        float fmn = kx(0), fmx = fmn;
        for (int i = 1; i < G; ++i) {
          const float x = kx(i);
          fmn = fminf(fmn, x);
          fmx = fmaxf(fmx, x);
        }
        const double mn = (double)fmn, mx = (double)fmx;
        double step;
        line_params(mn, mx, (double)levels, step);
        const double inv = step > 0.0 ? __drcp_rn(step) : 0.0;
        const FastLine fl = fast_line(fmn, fmx, step, inv, levels);
#pragma unroll 4
        for (int i = 0; i < G; ++i) {
          const float x = kx(i);
          bool slow;
          int code = quant_code_f32(x, fmn, fmx, levels, fl, slow);
          if (slow) code = quant_code_slow(x, fmn, fmx, mn, step, inv, levels, eps);
          kc[i * d + col] = (uint8_t)(code << kshift);
        }
        // decode-side encoding (ott_common.cuh): 2-bit: step = sh + sl, e = x_min - 4 u step;
        // other widths: float32 step and x_min. 1-bit K codes in 2-bit fields are stored
        // doubled with the step halved (exact), so the fp16 step halves cannot overflow
        const double kstep = kshift ? 0.5 * step : step;
        kst = (float)kstep;
        if (L.bits == 2 || k_tc4(L.bits, d) || k_tc8(L.bits, d)) {
          const __half sh = __double2half(kstep);
          const __half sl = __double2half(__dsub_rn(kstep, (double)__half2float(sh)));
          const int j = L.bits == 2 ? kpair_index(col, d) : (L.bits == 4 ? kpair4_index(col) : col);
          ksh[j] = sh;
          ksl[j] = sl;
          const double off = L.bits == 2 ? 4.0 * (double)kpair_u(col % 8) : (L.bits == 4 ? 64.0 : 1024.0);
          const float e = __double2float_rn(__dsub_rn(mn, __dmul_rn(off, kstep)));
          if (L.bits == 2) store_k_e2(rec, L, col, e);
          else ke[col] = e;
        } else {
          reinterpret_cast<float*>(ksh)[col] = __double2float_rn(step);
          ke[col] = __double2float_rn(mn);
        }
        if (p64) {
          p64[col] = mn;
          p64[d + col] = step;
        }
      }
      if (L.bits == 2 || L.bits == 4 || L.bits == 8) note_step_max(meta + 3, kst);
    }
    // d <= 128: the K warps and the (>= 4) V warps run side by side; d > 128: the K lines take
    // every warp, which then go on to the V lines
    const bool kv_par = nwarps - kwarps >= 4;
    if (!kv_par || warp >= kwarps) {
      // warp vw owns tokens vw + j nvw (j < 32 since G <= 128 and nvw >= 4): the warp reduces
      // each token's min/max, lane j keeps token j's and derives its line parameters (one
      // float64 division per lane instead of one per token), then the warp quantizes
      const int vw = kv_par ? warp - kwarps : warp, nvw = kv_par ? nwarps - kwarps : nwarps;
      float my_mn = 0.f, my_mx = 0.f;
      int n_my = 0;
      for (int i = vw; i < G; i += nvw, ++n_my) {
        // min/max of fp16-valued floats are exact in float32: reduce in float (1 shuffle per level)
        float fmn = 3.4e38f, fmx = -3.4e38f;
        const bool si = subst && sel[i];
        for (int col = lane; col < d; col += 32) {
          const float x = si ? vmean[col] : h2f(sv[i * d + col]);
          fmn = fminf(fmn, x);
          fmx = fmaxf(fmx, x);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          fmn = fminf(fmn, __shfl_xor_sync(0xffffffffu, fmn, o));
          fmx = fmaxf(fmx, __shfl_xor_sync(0xffffffffu, fmx, o));
        }
        if (lane == n_my) {
          my_mn = fmn;
          my_mx = fmx;
        }
      }
      double my_step = 0.0, my_inv = 0.0;
      FastLine my_fl;
      my_fl.ok = false;
      my_fl.inv32 = 0.f;
      my_fl.del = 0.f;
      if (lane < n_my) {
        const int i = vw + lane * nvw;
        const double mn = (double)my_mn;
        line_params(mn, (double)my_mx, (double)levels, my_step);
        my_inv = my_step > 0.0 ? __drcp_rn(my_step) : 0.0;
        my_fl = fast_line(my_mn, my_mx, my_step, my_inv, levels);
        vstep[i] = __double2float_rn(my_step);
        vxmin[i] = __double2float_rn(mn);
        if (p64) {
          p64[2 * d + i] = mn;
          p64[2 * d + G + i] = my_step;
        }
      }
      if (L.bits == 2 || L.bits == 4 || L.bits == 8) note_step_max(meta + 3, lane < n_my ? (float)my_step : 0.f);
      for (int j = 0; j < n_my; ++j) {
        const int i = vw + j * nvw;
        const float fmn = __shfl_sync(0xffffffffu, my_mn, j), fmx = __shfl_sync(0xffffffffu, my_mx, j);
        const double step = __shfl_sync(0xffffffffu, my_step, j), inv = __shfl_sync(0xffffffffu, my_inv, j);
        FastLine fl;
        fl.inv32 = __shfl_sync(0xffffffffu, my_fl.inv32, j);
        fl.ok = __shfl_sync(0xffffffffu, (int)my_fl.ok, j) != 0;
        fl.del = 4e-7f * (float)(levels + 1);
        const bool si = subst && sel[i];
#pragma unroll 4
        for (int col = lane; col < d; col += 32) {
          const float x = si ? vmean[col] : h2f(sv[i * d + col]);
          bool slow;
          int code = quant_code_f32(x, fmn, fmx, levels, fl, slow);
          if (slow) code = quant_code_slow(x, fmn, fmx, (double)fmn, step, inv, levels, eps);
          vc[i * d + col] = (uint8_t)code;
        }
      }
    }
    __syncthreads();

    // ---- 4. pack_codes (quant.py:241-256): element e=t*d+c at bits [b*e, b*e+b)
    {
      uint32_t* kw = reinterpret_cast<uint32_t*>(rec + L.k_codes());
      uint32_t* vw = reinterpret_cast<uint32_t*>(rec + L.v_codes());
      const int bits = L.bits;  // stored width (code_bits)
      const int n_codes = G * d;
      const int n_words = (n_codes * bits + 31) / 32;  // the tail of the last word stays 0
      for (int w = tid; w < 2 * n_words; w += kFlushThreads) {
        const bool isv = w >= n_words;
        const int ww = isv ? w - n_words : w;
        const uint8_t* src = isv ? vc : kc;
        uint32_t word = 0;
        if (bits == 2 && ww * 16 + 16 <= n_codes && (n_codes & 15) == 0) {  // 16 codes from one 16-byte load
          const uint4 b = *reinterpret_cast<const uint4*>(src + ww * 16);
          word = pack4x2(b.x) | (pack4x2(b.y) << 8) | (pack4x2(b.z) << 16) | (pack4x2(b.w) << 24);
        } else {  // codes overlapping stream bits [32 ww, 32 ww + 32); some straddle words
          const int e0 = (32 * ww) / bits, e1 = (32 * ww + 31) / bits;
          for (int e = e0; e <= e1 && e < n_codes; ++e) {
            const int sh = e * bits - 32 * ww;  // may be negative for the first code
            const uint64_t v = (uint64_t)src[e];
            word |= (uint32_t)(sh >= 0 ? (v << sh) : (v >> -sh));
          }
        }
        (isv ? vw : kw)[ww] = word;
      }
    }
    __syncthreads();
  }
#undef OTT_PREFETCH
#undef OTT_ROW_SRC
  if (tid == 0) {
    meta[0] = sh.n_entries;
    meta[1] = sh.n_aux;
    meta[2] = sh.frozen;
  }
}

// K1b: groups flushed after the unit's pool froze (or N = 0): no scoring, competition or
// substitution (cache.py:158), so every group is independent. One warp per group, no
// block barriers; 2-bit, d = 128, G = 32 (the tensor-core decode shapes).
//   * rows are staged in shared memory as fp16 with cp.async (V rows with their 16-byte
//     chunks XOR-swizzled by the row, so a lane-per-token read is bank-conflict free);
//   * K: lane l owns channels 4l..4l+3 (one code byte per token in pack_codes order),
//   * V: lane t owns token t (its eight 16-code words are built in registers);
//   * codes come from the same float32 fast path / float64 fallback as flush_kernel, so the
//     results are bit-identical.
// 16-byte global -> shared copy without a register round trip
// (unit, group) of a flat work item: 32-bit division when the item count allows (the 64-bit
// division routine is ~3x the instructions)
__device__ __forceinline__ void split_item(int64_t item, int64_t total, int n_groups, int& u, int& g) {
  if (total <= 0xffffffffLL) {
    const uint32_t it = (uint32_t)item, q = it / (uint32_t)n_groups;
    u = (int)q;
    g = (int)(it - q * (uint32_t)n_groups);
  } else {
    u = (int)(item / n_groups);
    g = (int)(item % n_groups);
  }
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gsrc) : "memory");
}
// The 32 rows of one tensor of a bulk-prefill group (g = its first row, d = 128) into smem rows
// (row r at r * 128 halves): lane = 16-byte chunk (lane & 15) of rows 2 it + (lane >> 4), V rows
// XOR-swizzled (chunk ^ (row & 15), and (2 it + hi) & 15 = (2 it & 15) ^ hi). The shared address
// is converted once and the global one advances by immediate offsets: two integer ops per copy
// instead of a generic-to-shared conversion and 64-bit address math each.
template <bool kSwizzle>
__device__ __forceinline__ void stage_rows_bulk(uint16_t* srows, const uint16_t* g, int lane) {
  constexpr int D = 128, G = 32;
  const int hi = lane >> 4, ch = lane & 15;
  const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(srows) + hi * D * 2;
  const uint32_t c16 = (kSwizzle ? (ch ^ hi) : ch) * 16;
  const char* gp = reinterpret_cast<const char*>(g + (size_t)hi * D + ch * 8);
#pragma unroll
  for (int it = 0; it < G / 2; ++it) {
    const uint32_t sa = s0 + it * 2 * D * 2 + (kSwizzle ? (c16 ^ ((2 * it & 15) * 16)) : c16);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gp + it * 2 * D * 2) : "memory");
  }
}

// K1a': score_tokens (outlier.py:45-49) for every token of a bulk flush in parallel, ahead of
// flush_scan_kernel (used when the pool is expected to stay active for many groups, N < A):
// one warp per group, lane t sums |k| of token t in float64 (exact) and leaves the 32 scores
// in the first 256 bytes of the group's record, which flush_frozen_kernel overwrites later.
__global__ void __launch_bounds__(128) flush_score_kernel(ott_cache_t c, int64_t q0, int n_groups, int64_t ring_end,
                                                          const uint16_t* __restrict__ in_k, int64_t in_stride,
                                                          int64_t in_first) {
  constexpr int D = 128, G = 32;
  const int lane = threadIdx.x & 31;
  const int64_t item = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (item >= (int64_t)c.n_units * n_groups) return;
  int u, g;
  split_item(item, (int64_t)c.n_units * n_groups, n_groups, u, g);
  if (c.pool_meta[(size_t)u * 4 + 2]) return;  // frozen: nothing will read the scores
  const int cap = G + c.residual;
  const int base = (int)(q0 + (int64_t)g * G);
  // Coalesced: load i brings rows 2i, 2i+1 (lane = 16-byte chunk ch of row 2i + hi), each lane
  // keeps one float64 partial per row pair, and a butterfly over the 16 lanes of each half
  // leaves lane (hi, ch) with the whole sum of row 2 ch + hi (exact in any order: fp16 magnitudes).
  const int hi = lane >> 4, ch = lane & 15;
  double part[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int p = base + 2 * i + hi;
    const uint16_t* row = p < (int)ring_end ? c.pend_k + ((size_t)u * cap + (size_t)(p % cap)) * D
                                            : in_k + (size_t)u * in_stride + (size_t)(p - (int)in_first) * D;
    const uint4 r = reinterpret_cast<const uint4*>(row)[ch];
    const __half2* h = reinterpret_cast<const __half2*>(&r);
    const float2 f0 = __half22float2(h[0]), f1 = __half22float2(h[1]), f2 = __half22float2(h[2]),
                 f3 = __half22float2(h[3]);
    part[i] = __dadd_rn(__dadd_rn(__dadd_rn(fabs((double)f0.x), fabs((double)f0.y)),
                                  __dadd_rn(fabs((double)f1.x), fabs((double)f1.y))),
                        __dadd_rn(__dadd_rn(fabs((double)f2.x), fabs((double)f2.y)),
                                  __dadd_rn(fabs((double)f3.x), fabs((double)f3.y))));
  }
#pragma unroll
  for (int o = 8; o >= 1; o >>= 1) {  // after step o, part[k] (k < o) holds row pair k + (ch & ~(o - 1))
    const bool upper = ch & o;
#pragma unroll
    for (int k = 0; k < o; ++k) {
      const double send = upper ? part[k] : part[k + o];
      const double keep = upper ? part[k + o] : part[k];
      part[k] = __dadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, o));
    }
  }
  const int t = 2 * ch + hi;  // this lane's token
  const double sc = part[0];
  double* rec = reinterpret_cast<double*>(record_ptr(c, u, base / G));
  rec[t] = sc;
  // the group's smallest score after them: the scan skips 32 groups at a time by these
  double m = sc;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) rec[32] = m;
}

// K1a: the sequential part of a bulk flush (cache.py:158-173 for every group in order):
// score_tokens, OutlierPool.update, the pool/aux rows and the pool/substitution bitmasks.
// One warp per unit; lane t scores token t of each group (or reads the score that
// flush_score_kernel left in the group's record, skipping 32 groups at a time by their
// minima while the pool is full); the competition is the same rank-by-count as flush_kernel
// (outlier.py:84-117). Substitution and quantization are left to flush_frozen_kernel (all
// groups in parallel). Stops when the pool freezes. d = 128, G = 32, N <= 128.
constexpr int kScanWarps = 1;  // one warp per block: a unit's scan is latency bound
constexpr int kScanStages = 4;  // K-row groups in flight per warp (cp.async ring)
struct ScanSmem {
  uint16_t rows[kScanWarps][kScanStages][32 * 128];  // chunk j of row t at (j ^ (t & 15))
  int slot_pos[kScanWarps][kMaxN];
  double slot_score[kScanWarps][kMaxN];
  int it_pos[kScanWarps][kMaxN + 32];
  double it_score[kScanWarps][kMaxN + 32];
  int it_rank[kScanWarps][kMaxN + 32];
  int free_slot[kScanWarps][kMaxN];
  int ev_slot[kScanWarps][kMaxN];  // aux index - n_aux -> evicted slot
  int win_cand[kScanWarps][32];    // winner number -> candidate index
};

__global__ void __launch_bounds__(32 * kScanWarps) flush_scan_kernel(ott_cache_t c, int64_t q0, int n_groups,
                                                                     int64_t ring_end, const uint16_t* __restrict__ in_k,
                                                                     const uint16_t* __restrict__ in_v,
                                                                     int64_t in_stride, int64_t in_first,
                                                                     bool prescored) {
  constexpr int D = 128, G = 32;
  extern __shared__ __align__(16) unsigned char smem[];
  ScanSmem& sm = *reinterpret_cast<ScanSmem*>(smem);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int u = blockIdx.x * kScanWarps + warp;
  if (u >= c.n_units) return;
  const int N = c.capacity, A = c.aux_capacity, M = N + G;
  const int cap = G + c.residual, ring_end32 = (int)ring_end, in_first32 = (int)in_first;
  int32_t* meta = c.pool_meta + (size_t)u * 4;
  int n_entries = meta[0], n_aux = meta[1], frozen = meta[2];
  if (N == 0 || frozen) return;
  int32_t* ppos = c.pool_pos + (size_t)u * N;
  double* pscore = c.pool_score + (size_t)u * N;
  uint16_t* pk = c.pool_k + (size_t)u * N * D;
  uint16_t* pv = c.pool_v + (size_t)u * N * D;
  int32_t* apos = c.aux_pos + (size_t)u * A;
  double* ascore = c.aux_score + (size_t)u * A;
  uint16_t* ak = c.aux_k + (size_t)u * A * D;
  uint16_t* av = c.aux_v + (size_t)u * A * D;
  uint32_t* pmask = c.pool_mask + (size_t)u * mask_words_per_unit(c);
  uint32_t* smask = c.subst_mask + (size_t)u * mask_words_per_unit(c);
  int* spos = sm.slot_pos[warp];
  double* sscore = sm.slot_score[warp];
  int* it_pos = sm.it_pos[warp];
  double* it_score = sm.it_score[warp];
  int* it_rank = sm.it_rank[warp];
  int* free_slot = sm.free_slot[warp];
  int* ev_slot = sm.ev_slot[warp];
  int* win_cand = sm.win_cand[warp];
  for (int s = lane; s < N; s += 32) {
    spos[s] = ppos[s];
    sscore[s] = pscore[s];
  }
  // largest entry score (valid when the pool is full; a candidate with an equal score has a
  // larger position, so it loses the tie)
  auto max_entry_score = [&]() {
    double m = -1.0;
    for (int t = lane; t < N; t += 32)
      if (spos[t] >= 0) m = fmax(m, sscore[t]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    return m;
  };
  const int q0i = (int)q0;
  const int bslot0 = q0i % cap;
  auto row_of = [&](int p, const uint16_t* ring, const uint16_t* in) -> const uint16_t* {
    if (p < ring_end32) {
      int sl = bslot0 + (p - q0i) % cap;
      sl = sl >= cap ? sl - cap : sl;
      return ring + ((size_t)u * cap + (size_t)sl) * D;
    }
    return in + (size_t)u * in_stride + (size_t)(p - in_first32) * D;
  };
  // K rows of group g -> stage g % kScanStages (one cp.async group per load; nothing for
  // pre-scored groups, whose scores are read from their records directly)
  auto load_group = [&](int g) {
    if (g < n_groups) {
      uint16_t* dst = sm.rows[warp][g % kScanStages];
      const int base = q0i + g * G, ch = lane & 15;
      if (!prescored) {
#pragma unroll 4
        for (int it = 0; it < G / 2; ++it) {
          const int row = 2 * it + (lane >> 4);
          cp_async16(dst + row * D + ((ch ^ (row & 15)) * 8), row_of(base + row, c.pend_k, in_k) + ch * 8);
        }
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
#pragma unroll
  for (int st = 0; st < kScanStages - 1; ++st) load_group(st);
  __syncwarp();
  double wmax = max_entry_score();
  int wbase = -32;  // pre-scored skip window (see below)
  double wmin = INFINITY;
  for (int g = 0; g < n_groups && !frozen; ++g) {
    if (prescored && n_entries == N) {
      // A full pool changes only for a group with a candidate below its largest entry
      // (outlier.py:102-117): find the next such group from the group minima, a window of 32
      // at a time (lane j holds group wbase + j; the window is reloaded only when passed).
      for (;;) {
        if (g >= wbase + 32) {
          wbase = g;
          const int gg = g + lane;
          wmin = gg < n_groups ? reinterpret_cast<const double*>(record_ptr(c, u, (q0i + gg * G) / G))[32] : INFINITY;
        }
        const uint32_t need = __ballot_sync(0xffffffffu, wmin < wmax) & ~((1u << (g - wbase)) - 1u);
        if (need) {
          g = wbase + __ffs(need) - 1;
          break;
        }
        g = wbase + 32;
        if (g >= n_groups) break;
      }
      if (g >= n_groups) break;
    }
    const int base = q0i + g * G;
    const uint16_t* srow = sm.rows[warp][g % kScanStages];
    if (!prescored) {
      load_group(g + kScanStages - 1);
      asm volatile("cp.async.wait_group %0;\n" ::"n"(kScanStages - 1) : "memory");
      __syncwarp();
    }
    // ---- score_tokens (outlier.py:45-49): L1 norm of key row `lane` in float64 (exact)
    double sc;
    if (prescored) {
      sc = reinterpret_cast<const double*>(record_ptr(c, u, base / G))[lane];
    } else {
      const uint4* kr = reinterpret_cast<const uint4*>(srow + lane * D);
      const int sw = lane & 15;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll 4
      for (int j = 0; j < D / 8; ++j) {
        const uint4 r = kr[j ^ sw];
        const __half2* h = reinterpret_cast<const __half2*>(&r);
        const float2 f0 = __half22float2(h[0]), f1 = __half22float2(h[1]), f2 = __half22float2(h[2]),
                     f3 = __half22float2(h[3]);
        a0 = __dadd_rn(a0, __dadd_rn(fabs((double)f0.x), fabs((double)f0.y)));
        a1 = __dadd_rn(a1, __dadd_rn(fabs((double)f1.x), fabs((double)f1.y)));
        a2 = __dadd_rn(a2, __dadd_rn(fabs((double)f2.x), fabs((double)f2.y)));
        a3 = __dadd_rn(a3, __dadd_rn(fabs((double)f3.x), fabs((double)f3.y)));
      }
      sc = __dadd_rn(__dadd_rn(a0, a1), __dadd_rn(a2, a3));  // exact: fp16 magnitudes fit 2^-24..2^16
    }
    // a full pool only changes if some candidate ranks below its largest entry (ties go to the
    // smaller position, and candidates come after every entry): otherwise update() selects
    // and evicts nothing (outlier.py:102-117)
    if (n_entries == N && !__any_sync(0xffffffffu, sc < wmax)) {
      __syncwarp();
      continue;
    }
    // ---- OutlierPool.update (outlier.py:84-117): items [0, N) slots, [N, N+G) candidates
    for (int t = lane; t < N; t += 32) {
      it_pos[t] = spos[t];
      it_score[t] = sscore[t];
    }
    it_pos[N + lane] = base + lane;
    it_score[N + lane] = sc;
    __syncwarp();
    for (int t = lane; t < M; t += 32) {
      int r = -1;
      if (it_pos[t] >= 0) {
        const double s0 = it_score[t];
        const int p0 = it_pos[t];
        r = 0;
        for (int j = 0; j < M; ++j) {
          const int pj = it_pos[j];
          if (pj < 0) continue;
          const double sj = it_score[j];
          r += (sj < s0 || (sj == s0 && pj < p0)) ? 1 : 0;  // _rank, outlier.py:52-54
        }
      }
      it_rank[t] = r;
    }
    __syncwarp();
    // evicted old entries -> aux in old-entry order (ascending rank); free slots ascending.
    // Ranks are distinct and an evicted entry's rank lies in [N, N + 32): one bit each, so an
    // entry's aux index is the number of evicted ranks below its own.
    const int room = A - n_aux;  // outlier.py:113-114
    uint32_t ev_bits = 0u;
    for (int s0 = 0; s0 < N; s0 += 32) {
      const int s = s0 + lane;
      const int r = s < N ? it_rank[s] : 0;
      ev_bits |= __reduce_or_sync(0xffffffffu, (s < N && r >= N) ? 1u << (r - N) : 0u);
    }
    const int n_ev = __popc(ev_bits);
    int n_free = 0;
    for (int s0 = 0; s0 < N; s0 += 32) {
      const int s = s0 + lane;
      const int r = s < N ? it_rank[s] : 0;
      const bool evicted = s < N && r >= N;
      const bool is_free = s < N && (r < 0 || r >= N);
      const uint32_t fb = __ballot_sync(0xffffffffu, is_free);
      if (is_free) free_slot[n_free + __popc(fb & ((1u << lane) - 1u))] = s;
      n_free += __popc(fb);
      if (evicted) {
        const int eidx = __popc(ev_bits & ((1u << (r - N)) - 1u));
        if (eidx < room) {
          apos[n_aux + eidx] = it_pos[s];
          ascore[n_aux + eidx] = it_score[s];
          ev_slot[eidx] = s;
        }
        const int p = it_pos[s];
        atomicAnd(&pmask[p >> 5], ~(1u << (p & 31)));  // back to its shadow row
      }
    }
    __syncwarp();
    // Row copies: lane = (K or V, 16-byte chunk) of one row; the loads of up to 8 rows are issued
    // before their stores, so a group's copies cost a few memory round trips, not one per row.
    // Evicted rows go into aux first, before their slots are reused.
    const int j16 = lane & 15;
    const int n_copy = n_ev < room ? n_ev : room;
    for (int r0 = 0; r0 < n_copy; r0 += 8) {
      uint4 buf[8];
#pragma unroll
      for (int m = 0; m < 8; ++m)
        if (r0 + m < n_copy) buf[m] = reinterpret_cast<const uint4*>((lane < 16 ? pk : pv) + (size_t)ev_slot[r0 + m] * D)[j16];
#pragma unroll
      for (int m = 0; m < 8; ++m)
        if (r0 + m < n_copy)
          reinterpret_cast<uint4*>((lane < 16 ? ak : av) + (size_t)(n_aux + r0 + m) * D)[j16] = buf[m];
    }
    __syncwarp();
    // winning candidates take the free slots in candidate order
    const bool win = it_rank[N + lane] < N;
    const uint32_t wins = __ballot_sync(0xffffffffu, win);
    const int n_win = __popc(wins);
    if (win) {
      const int widx = __popc(wins & ((1u << lane) - 1u));
      const int s = free_slot[widx];
      win_cand[widx] = lane;
      spos[s] = base + lane;
      sscore[s] = it_score[N + lane];
    }
    if (lane == 0 && wins) {  // positions base..base+31 share one mask word (base is 32-aligned)
      atomicOr(&pmask[base >> 5], wins);
      atomicOr(&smask[base >> 5], wins);  // cache.py:173
    }
    __syncwarp();
    for (int w0 = 0; w0 < n_win; w0 += 8) {
      uint4 buf[8];
#pragma unroll
      for (int m = 0; m < 8; ++m)
        if (w0 + m < n_win) {
          const int i = win_cand[w0 + m], p = base + i;
          buf[m] = lane >= 16   ? reinterpret_cast<const uint4*>(row_of(p, c.pend_v, in_v))[j16]
                   : prescored ? reinterpret_cast<const uint4*>(row_of(p, c.pend_k, in_k))[j16]
                               : reinterpret_cast<const uint4*>(srow + i * D)[j16 ^ (i & 15)];
        }
#pragma unroll
      for (int m = 0; m < 8; ++m)
        if (w0 + m < n_win)
          reinterpret_cast<uint4*>((lane < 16 ? pk : pv) + (size_t)free_slot[w0 + m] * D)[j16] = buf[m];
    }
    __syncwarp();
    n_aux += n_ev < room ? n_ev : room;
    int n_e = 0;
    for (int t = lane; t < M; t += 32) n_e += (it_rank[t] >= 0 && it_rank[t] < N) ? 1 : 0;
    n_entries = warp_sum(n_e);
    if (n_aux >= A) frozen = 1;  // outlier.py:115-116
    __syncwarp();  // stage g % kScanStages is reloaded next iteration
    wmax = max_entry_score();
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncwarp();
  for (int s = lane; s < N; s += 32) {
    ppos[s] = spos[s];
    pscore[s] = sscore[s];
  }
  if (lane == 0) {
    meta[0] = n_entries;
    meta[1] = n_aux;
    meta[2] = frozen;
  }
}

// fp16 neighbours (finite values; -0 and +0 are one value)
__device__ __forceinline__ uint16_t h_next(uint16_t b) {
  return b == 0x8000u || b == 0x0000u ? (uint16_t)0x0001u : ((b & 0x8000u) ? (uint16_t)(b - 1) : (uint16_t)(b + 1));
}
__device__ __forceinline__ uint16_t h_prev(uint16_t b) {
  return b == 0x8000u || b == 0x0000u ? (uint16_t)0x8001u : ((b & 0x8000u) ? (uint16_t)(b + 1) : (uint16_t)(b - 1));
}
__device__ __forceinline__ double h_val(uint16_t b) { return (double)__half2float(__ushort_as_half(b)); }

// Code thresholds of one line over fp16 inputs: t[k-1] = the smallest fp16 value x of the
// line's range with code(x) >= k (quant.py:91-102 incl. the max rule), so that
// code(x) = #{k : x >= t[k-1]} for every fp16 x in [x_min, x_max] (the code is monotone in x).
// With T = fl(x_min + fl(k step)) -- exactly the left side of the quant.py:97 check for c = k:
//   * x < T: code(x) < k (a code of k needs the check fl(k step + x_min) <= x to pass);
//   * x >= T: code(x) >= k iff fl((x - x_min) / step) >= k, which holds whenever x - T exceeds
//     margin = 1e-12 (|x_min| + levels step) (all float64 roundings involved are < 2^-50 of it).
// So t = the fp16 ceiling v of T, except when v - T <= margin: then the float64 quotient at v
// decides between v and the next fp16 value (false is returned, and quant_code is used per
// element, when 4 margin reaches the smallest fp16 spacing 2^-24). t[levels-1] = x_max: T_levels lies
// within float64 rounding below x_max (line_params) and x_max has code levels (quant.py:101).
// The tie case of code_thresholds: the fp16 ceiling v of T lies within the margin of T, so the
// float64 quotient at v decides: fl(d / step) >= k, d = v - x_min (exact: both are fp16 values).
// fl(q) >= k iff q >= k - delta_k, the midpoint below k (ties round to k, whose significand is
// even): delta_k = 2^(e - 53) for 2^e < k < 2^(e+1), 2^(e - 54) for k = 2^e. That is decided
// without the division as fma(-k, step, d) >= -delta_k step: d and k step are multiples of
// ulp(step) / 2 and d lies within (1 +- 1e-7) k step here, so d - k step is representable and the
// fma exact; delta_k step is a power-of-two scaling, exact. Common for fp16 lines (x_min + k step
// is an fp16 value whenever the range is a multiple of levels / gcd(k, levels) fp16 units).
__host__ __device__ constexpr double tie_delta(int k) {
  int e = 0;
  while ((2 << e) <= k) ++e;
  double d = 1.0;
  for (int i = 0; i < 53 + ((k & (k - 1)) == 0 ? 1 : 0) - e; ++i) d *= 0.5;
  return d;
}
__device__ __forceinline__ bool code_thresholds(uint16_t* t, float mnf, float mxf, double mn, double step, double inv,
                                                int levels, double eps) {
  (void)inv;
  (void)eps;
  const uint16_t mxb = __half_as_ushort(__float2half_rn(mxf));  // x_max is an fp16 value
  if (step == 0.0) {  // quant.py:91-92: every code 0 (no max rule)
#pragma unroll
    for (int k = 0; k < levels; ++k) t[k] = 0x7C00u;  // +inf
    return true;
  }
  const double margin = 1e-12 * (fabs(mn) + (double)levels * step);
  // fp16 values lie >= 2^-24 apart, so below this bound the value after a tie candidate is never
  // within 4 margin of it (lines with |x_min| + range beyond ~1.5e4 take the per-element path)
  const bool ok = 4.0 * margin < 0x1p-24;
#pragma unroll
  for (int k = 1; k < levels; ++k) {
    const double T = __dadd_rn(mn, __dmul_rn((double)k, step));
    uint16_t vb = __half_as_ushort(__float2half_ru(__double2float_ru(T)));  // smallest fp16 >= T (or +inf)
    const double dv = h_val(vb);
    // a tie candidate (dv - T <= margin; never for +inf): the float64 quotient at v decides,
    // branch-free (ties are common in fp16 lines, so a branch would diverge in most warps)
    const bool tie = __dsub_rn(dv, T) <= margin;
    const bool ge = __fma_rn(-(double)k, step, __dsub_rn(dv, mn)) >= -step * tie_delta(k);
    if (tie && !ge) vb = h_next(vb);
    if ((vb & 0x7C00u) == 0x7C00u || __half2float(__ushort_as_half(vb)) > mxf) vb = mxb;
    t[k - 1] = vb;
  }
  t[levels - 1] = mxb;
  return ok;
}

// 2-bit codes of two fp16 inputs as bit masks (16-bit all-ones / zero halves): with t1 <= t2 <= t3,
// code(x) = [x >= t1] + [x >= t2] + [x >= t3], so its high bit is b1 = [x >= t2] and its low bit
// b0 = [x >= (b1 ? t3 : t1)]: two mask compares and one select per two inputs
struct CodeMasks {
  uint32_t b0, b1;
};
__device__ __forceinline__ CodeMasks code_masks(__half2 x, const uint32_t* th) {
  const uint32_t b1 = __hge2_mask(x, *reinterpret_cast<const __half2*>(&th[1]));
  const uint32_t ts = (b1 & th[2]) | (~b1 & th[0]);
  return {__hge2_mask(x, *reinterpret_cast<const __half2*>(&ts)), b1};
}
// OR the two codes of m into acc: low-half input at bits LO, LO + 1, high-half input at HI, HI + 1
template <int LO, int HI>
__device__ __forceinline__ uint32_t put_codes(uint32_t acc, const CodeMasks& m) {
  constexpr uint32_t c0 = (1u << LO) | (1u << (16 + HI)), c1 = c0 << 1;
  return acc | (m.b0 & c0) | (m.b1 & c1);
}
// 4-bit (levels 15) / 3-bit (levels 7) codes of two fp16 inputs by binary search over the
// line's thresholds th[k - 1] = t_k (half2 words, monotone): each level is one mask compare
// against a threshold selected by the higher code bits (bitwise selects on the 0xFFFF masks).
// Returns the code bits as masks: b[0] = lowest.
__device__ __forceinline__ uint32_t sel_mask(uint32_t m, uint32_t a, uint32_t b) { return (m & a) | (~m & b); }
__device__ __forceinline__ uint32_t ge_mask(__half2 x, uint32_t t) {
  return __hge2_mask(x, *reinterpret_cast<const __half2*>(&t));
}
template <int kLevels>
__device__ __forceinline__ void nib_masks(__half2 x, const uint32_t* th, uint32_t (&b)[4]) {
  if constexpr (kLevels == 15) {
    b[3] = ge_mask(x, th[7]);
    b[2] = ge_mask(x, sel_mask(b[3], th[11], th[3]));
    b[1] = ge_mask(x, sel_mask(b[3], sel_mask(b[2], th[13], th[9]), sel_mask(b[2], th[5], th[1])));
    const uint32_t d0 = sel_mask(b[2], sel_mask(b[1], th[14], th[12]), sel_mask(b[1], th[10], th[8]));
    const uint32_t d1 = sel_mask(b[2], sel_mask(b[1], th[6], th[4]), sel_mask(b[1], th[2], th[0]));
    b[0] = ge_mask(x, sel_mask(b[3], d0, d1));
  } else {  // kLevels == 7
    b[3] = 0u;
    b[2] = ge_mask(x, th[3]);
    b[1] = ge_mask(x, sel_mask(b[2], th[5], th[1]));
    b[0] = ge_mask(x, sel_mask(b[2], sel_mask(b[1], th[6], th[4]), sel_mask(b[1], th[2], th[0])));
  }
}
// OR the 4-bit codes of m into acc: low-half input at bits LO..LO+3, high-half input at
// bits 16 + HI..16 + HI + 3 (fold with acc >> 16 afterwards)
template <int LO, int HI>
__device__ __forceinline__ uint32_t put_nibs(uint32_t acc, const uint32_t (&b)[4]) {
#pragma unroll
  for (int k = 0; k < 4; ++k) acc |= b[k] & ((1u << (LO + k)) | (1u << (16 + HI + k)));
  return acc;
}

// codes of two fp16 inputs against per-lane thresholds th[0..2]: code at bits 0-1 (low half)
// and 16-17 (high half). Each compare gives 1.0 or 0.0; 1024 + code is exact in fp16.
// the same as fp16 bits 1024 + code (bytes: code, 0x64, code', 0x64), unmasked
__device__ __forceinline__ uint32_t codes_h2_raw(__half2 x, const __half2* th) {
  const __half2 c = __hadd2(__hadd2(__hge2(x, th[0]), __hge2(x, th[1])), __hadd2(__hge2(x, th[2]), __float2half2_rn(1024.f)));
  return *reinterpret_cast<const uint32_t*>(&c);
}
// four codes from two raw pairs: one PRMT gathers the code bytes, pack4x2 squeezes them
__device__ __forceinline__ uint32_t codes4(uint32_t raw01, uint32_t raw23) { return pack4x2(__byte_perm(raw01, raw23, 0x6420)); }
__device__ __forceinline__ uint32_t codes_h2(__half2 x, const __half2* th) {
  const __half2 c = __hadd2(__hadd2(__hge2(x, th[0]), __hge2(x, th[1])), __hadd2(__hge2(x, th[2]), __float2half2_rn(1024.f)));
  return *reinterpret_cast<const uint32_t*>(&c) & 0x00030003u;
}

// V codes of token row vr (16-byte chunks swizzled by sw) with the per-element float64 recipe:
// the rare path of lines without exact fp16 thresholds, out of line (instruction cache)
__device__ __noinline__ void frozen_v_codes_slow(const uint4* vr, int sw, float fmn, float fmx, double mn, double step,
                                                 double inv, int levels, double eps, uint4* vcodes) {
  uint32_t w[8];
  for (int j = 0; j < 16; ++j) {
    const uint4 r = vr[j ^ sw];
    const __half2* h = reinterpret_cast<const __half2*>(&r);
    uint32_t bits = 0;
    for (int e = 0; e < 4; ++e) {
      const float2 f = __half22float2(h[e]);
      bits |= ((uint32_t)quant_code(f.x, fmn, fmx, mn, step, inv, levels, eps) << (4 * e)) |
              ((uint32_t)quant_code(f.y, fmn, fmx, mn, step, inv, levels, eps) << (4 * e + 2));
    }
    if (j & 1) w[j / 2] |= bits << 16;
    else w[j / 2] = bits;
  }
  vcodes[0] = make_uint4(w[0], w[1], w[2], w[3]);
  vcodes[1] = make_uint4(w[4], w[5], w[6], w[7]);
}

constexpr int kFrozenWarps = 4;
#ifndef OTT_FROZEN_PAIR  // 1: two warps per group in the 2-bit kernel (K rows / V rows), 8 KB of rows each
#define OTT_FROZEN_PAIR 1
#endif
struct FrozenSmem {
  uint16_t k[kFrozenWarps][32 * 128];
  uint16_t v[kFrozenWarps][32 * 128];
  float vmean[kFrozenWarps][128];  // V column means of a group with substituted rows
};
struct FrozenPairSmem {  // per warp: the K or the V rows of its group
  uint16_t rows[kFrozenWarps][32 * 128];
  float vmean[kFrozenWarps][128];
};

// Groups in which the pool competition selected tokens (cache.py:169-173): their rows are
// replaced by the column means of the ORIGINAL rows (outlier.py:120-142: float64 sums, which
// are exact for fp16 inputs, / G, rounded to float32) before quantization. The substituted
// values are float32, so these lines use the float32 fast path / float64 fallback per element
// instead of fp16 thresholds. `sel` bit t = token t substituted.
// out of line: substituted groups are rare, and inlined into both warp roles this path more
// than doubled the kernel (instruction-cache misses were its top stall)
__device__ __noinline__ void frozen_group_subst(uint8_t* rec, double* p64, const uint16_t* sk, const uint16_t* sv,
                                                float* vmean, uint32_t sel, int lane, int32_t* meta3, int part) {
  constexpr int D = 128, G = 32, kLevels = 3;
  const RecordLayout L(D, G, 2);
  const double eps = 1e-9 * (double)(kLevels + 1);
  const uint2* kr = reinterpret_cast<const uint2*>(sk) + lane;
  float kst_max = 0.f;
  float vst = 0.f;
  // ---- K: channels 4 lane .. +3
  if (part != 1) {
    double sum[4] = {0.0, 0.0, 0.0, 0.0};
    for (int t = 0; t < G; ++t) {
      const uint2 r = kr[t * (D / 4)];
      const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&r.x));
      const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&r.y));
      sum[0] = __dadd_rn(sum[0], (double)a.x);
      sum[1] = __dadd_rn(sum[1], (double)a.y);
      sum[2] = __dadd_rn(sum[2], (double)b.x);
      sum[3] = __dadd_rn(sum[3], (double)b.y);
    }
    float mean[4], fmn[4], fmx[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      mean[j] = __double2float_rn(__ddiv_rn(sum[j], (double)G));
      fmn[j] = 3.4e38f;
      fmx[j] = -3.4e38f;
    }
    auto kval = [&](int t, float (&x)[4]) {
      if ((sel >> t) & 1u) {
        x[0] = mean[0]; x[1] = mean[1]; x[2] = mean[2]; x[3] = mean[3];
      } else {
        const uint2 r = kr[t * (D / 4)];
        const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&r.x));
        const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&r.y));
        x[0] = a.x; x[1] = a.y; x[2] = b.x; x[3] = b.y;
      }
    };
    for (int t = 0; t < G; ++t) {
      float x[4];
      kval(t, x);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        fmn[j] = fminf(fmn[j], x[j]);
        fmx[j] = fmaxf(fmx[j], x[j]);
      }
    }
    double step[4], inv[4];
    FastLine fl[4];
    __half* ksh = reinterpret_cast<__half*>(rec + L.k_sh());
    __half* ksl = reinterpret_cast<__half*>(rec + L.k_sl());
    float ke[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = 4 * lane + j;
      const double mn = (double)fmn[j];
      line_params(mn, (double)fmx[j], (double)kLevels, step[j]);
      inv[j] = step[j] > 0.0 ? __drcp_rn(step[j]) : 0.0;
      fl[j] = fast_line(fmn[j], fmx[j], step[j], inv[j], kLevels);
      kst_max = fmaxf(kst_max, (float)step[j]);
      const __half sh = __double2half(step[j]);
      const __half sl = __double2half(__dsub_rn(step[j], (double)__half2float(sh)));
      ksh[kpair_index(col, D)] = sh;
      ksl[kpair_index(col, D)] = sl;
      ke[j] = __double2float_rn(__dsub_rn(mn, __dmul_rn(4.0 * (double)kpair_u(col % 8), step[j])));
      if (p64) {
        p64[col] = mn;
        p64[D + col] = step[j];
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) store_k_e2(rec, L, 4 * lane + j, ke[j]);
    uint8_t* kcodes = rec + L.k_codes() + lane;
    for (int t = 0; t < G; ++t) {
      float x[4];
      kval(t, x);
      uint32_t byte = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        bool slow;
        int code = quant_code_f32(x[j], fmn[j], fmx[j], kLevels, fl[j], slow);
        if (slow) code = quant_code_slow(x[j], fmn[j], fmx[j], (double)fmn[j], step[j], inv[j], kLevels, eps);
        byte |= (uint32_t)code << (2 * j);
      }
      kcodes[t * (D / 4)] = (uint8_t)byte;
    }
  }
  // ---- V column means: lane l sums channels 4l..4l+3 (chunk l/2, half l&1 of each swizzled row)
  if (part != 0) {
    double sum[4] = {0.0, 0.0, 0.0, 0.0};
    for (int t = 0; t < G; ++t) {
      const uint2 r = *reinterpret_cast<const uint2*>(sv + t * D + (((lane >> 1) ^ (t & 15)) * 8) + (lane & 1) * 4);
      const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&r.x));
      const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&r.y));
      sum[0] = __dadd_rn(sum[0], (double)a.x);
      sum[1] = __dadd_rn(sum[1], (double)a.y);
      sum[2] = __dadd_rn(sum[2], (double)b.x);
      sum[3] = __dadd_rn(sum[3], (double)b.y);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) vmean[4 * lane + j] = __double2float_rn(__ddiv_rn(sum[j], (double)G));
    __syncwarp();
  }
  // ---- V: token `lane`
  if (part != 0) {
    const int t = lane;
    const bool subst = (sel >> t) & 1u;
    const uint4* vr = reinterpret_cast<const uint4*>(sv + t * D);
    const int sw = t & 15;
    auto vval = [&](int j, float (&x)[8]) {  // channels 8j..8j+7
      if (subst) {
#pragma unroll
        for (int e = 0; e < 8; ++e) x[e] = vmean[8 * j + e];
      } else {
        const uint4 r = vr[j ^ sw];
        const __half2* h = reinterpret_cast<const __half2*>(&r);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __half22float2(h[e]);
          x[2 * e] = f.x;
          x[2 * e + 1] = f.y;
        }
      }
    };
    float fmn = 3.4e38f, fmx = -3.4e38f;
    for (int j = 0; j < D / 8; ++j) {
      float x[8];
      vval(j, x);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        fmn = fminf(fmn, x[e]);
        fmx = fmaxf(fmx, x[e]);
      }
    }
    const double mn = (double)fmn;
    double step;
    line_params(mn, (double)fmx, (double)kLevels, step);
    const double inv = step > 0.0 ? __drcp_rn(step) : 0.0;
    const FastLine fl = fast_line(fmn, fmx, step, inv, kLevels);
    vst = (float)step;
    reinterpret_cast<float*>(rec + L.v_step())[t] = __double2float_rn(step);
    reinterpret_cast<float*>(rec + L.v_xmin())[t] = __double2float_rn(mn);
    if (p64) {
      p64[2 * D + t] = mn;
      p64[2 * D + G + t] = step;
    }
    uint32_t w[D / 16];
#pragma unroll
    for (int j = 0; j < D / 8; ++j) {
      float x[8];
      vval(j, x);
      uint32_t bits = 0;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        bool slow;
        int code = quant_code_f32(x[e], fmn, fmx, kLevels, fl, slow);
        if (slow) code = quant_code_slow(x[e], fmn, fmx, mn, step, inv, kLevels, eps);
        bits |= (uint32_t)code << (2 * e);
      }
      if (j & 1) w[j / 2] |= bits << 16;
      else w[j / 2] = bits;
    }
    uint4* vcodes = reinterpret_cast<uint4*>(rec + L.v_codes() + t * (D / 4));
    vcodes[0] = make_uint4(w[0], w[1], w[2], w[3]);
    vcodes[1] = make_uint4(w[4], w[5], w[6], w[7]);
  }
  note_step_max(meta3, fmaxf(kst_max, vst));
}


__global__ void __launch_bounds__(32 * kFrozenWarps, 6) flush_frozen_kernel(ott_cache_t c, int64_t q0, int n_groups,
                                                                         int64_t ring_end,
                                                                         const uint16_t* __restrict__ in_k,
                                                                         const uint16_t* __restrict__ in_v,
                                                                         int64_t in_stride, int64_t in_first) {
  constexpr int D = 128, G = 32, kLevels = 3;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // OTT_FROZEN_PAIR: warp pairs share a group, the even warp quantizes K, the odd one V
  const int part = OTT_FROZEN_PAIR ? (warp & 1) : 2;  // 0 K, 1 V, 2 both
  const int64_t item = OTT_FROZEN_PAIR ? ((int64_t)blockIdx.x * kFrozenWarps + warp) >> 1
                                       : (int64_t)blockIdx.x * kFrozenWarps + warp;
  if (item >= (int64_t)c.n_units * n_groups) return;
  int u, g;
  split_item(item, (int64_t)c.n_units * n_groups, n_groups, u, g);
  const int cap = G + c.residual;
  const int base = (int)(q0 + (int64_t)g * G);
  const int64_t gi = base / G;
  uint8_t* rec = record_ptr(c, u, gi);
  const RecordLayout L(D, G, 2);
#if OTT_FROZEN_PAIR
  FrozenPairSmem& sm = *reinterpret_cast<FrozenPairSmem*>(smem);
  uint16_t* sk = sm.rows[warp];
  uint16_t* sv = sm.rows[warp];
#else
  FrozenSmem& sm = *reinterpret_cast<FrozenSmem*>(smem);
  uint16_t* sk = sm.k[warp];
  uint16_t* sv = sm.v[warp];
#endif
  // tokens of this group substituted by the pool competition (base is 32-aligned); loaded
  // before the rows so its latency overlaps theirs
  const uint32_t sel = c.subst_mask[(size_t)u * mask_words_per_unit(c) + (base >> 5)];

  // ---- stage the G rows (cache.py:155-156): lane = 16-byte chunk (lane & 15) of row pairs
  {
    const int bslot = base % cap, ring_end32 = (int)ring_end, in_first32 = (int)in_first;
    const int ch = lane & 15;
    if (base >= ring_end32) {  // bulk prefill: every row of the group comes from the input
      const size_t off0 = (size_t)u * in_stride + (size_t)(base - in_first32) * D;
      if (part != 1) stage_rows_bulk<false>(sk, in_k + off0, lane);
      if (part != 0) stage_rows_bulk<true>(sv, in_v + off0, lane);
    } else
#pragma unroll 4
    for (int it = 0; it < G / 2; ++it) {
      const int row = 2 * it + (lane >> 4);
      const int p = base + row;
      const uint16_t *pk, *pv;
      if (p < ring_end32) {
        int sl = bslot + row;
        sl = sl >= cap ? sl - cap : sl;
        const size_t off = ((size_t)u * cap + (size_t)sl) * D + ch * 8;
        pk = c.pend_k + off;
        pv = c.pend_v + off;
      } else {
        const size_t off = (size_t)u * in_stride + (size_t)(p - in_first32) * D + ch * 8;
        pk = in_k + off;
        pv = in_v + off;
      }
      if (part != 1) cp_async16(sk + row * D + ch * 8, pk);
      if (part != 0) cp_async16(sv + row * D + ((ch ^ (row & 15)) * 8), pv);
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncwarp();
  }
  double* p64 = c.params64 ? c.params64 + ((size_t)u * c.max_groups + (size_t)gi) * 2 * (D + G) : nullptr;
  const double eps = 1e-9 * (double)(kLevels + 1);
  int32_t* meta3 = c.pool_meta + (size_t)u * 4 + 3;
  if (OTT_FROZEN_SEL && sel) {
    if (OTT_FROZEN_SEL == 1) frozen_group_subst(rec, p64, sk, sv, sm.vmean[warp], sel, lane, meta3, part);
    return;
  }
  float kst_max = 0.f;
  float vst = 0.f;

  // ---- K: channels 4 lane .. 4 lane + 3, lines over the G tokens
  if (part != 1) {
    __half2 mn01 = __float2half2_rn(65504.f), mn23 = mn01, mx01 = __float2half2_rn(-65504.f), mx23 = mx01;
    const uint2* kr = reinterpret_cast<const uint2*>(sk) + lane;  // row stride D / 4 uint2
#pragma unroll 8
    for (int t = 0; t < G; ++t) {
      const uint2 r = kr[t * (D / 4)];
      const __half2 a = *reinterpret_cast<const __half2*>(&r.x), b = *reinterpret_cast<const __half2*>(&r.y);
      mn01 = __hmin2(mn01, a);
      mx01 = __hmax2(mx01, a);
      mn23 = __hmin2(mn23, b);
      mx23 = __hmax2(mx23, b);
    }
    float fmn[4], fmx[4];
    {
      const float2 a = __half22float2(mn01), b = __half22float2(mn23), x = __half22float2(mx01),
                   y = __half22float2(mx23);
      fmn[0] = a.x; fmn[1] = a.y; fmn[2] = b.x; fmn[3] = b.y;
      fmx[0] = x.x; fmx[1] = x.y; fmx[2] = y.x; fmx[3] = y.y;
    }
    double step[4], inv[4];
    uint16_t thr[4][kLevels];
    bool exact = true;  // all four lines have exact fp16 thresholds
    __half* ksh = reinterpret_cast<__half*>(rec + L.k_sh());
    __half* ksl = reinterpret_cast<__half*>(rec + L.k_sl());
    float ke[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = 4 * lane + j;
      const double mn = (double)fmn[j];
      line_params(mn, (double)fmx[j], (double)kLevels, step[j]);
      inv[j] = step[j] > 0.0 ? __drcp_rn(step[j]) : 0.0;
      exact &= code_thresholds(thr[j], fmn[j], fmx[j], mn, step[j], inv[j], kLevels, eps);
      kst_max = fmaxf(kst_max, (float)step[j]);
      const __half sh = __double2half(step[j]);
      const __half sl = __double2half(__dsub_rn(step[j], (double)__half2float(sh)));
      ksh[kpair_index(col, D)] = sh;
      ksl[kpair_index(col, D)] = sl;
      ke[j] = __double2float_rn(__dsub_rn(mn, __dmul_rn(4.0 * (double)kpair_u(col % 8), step[j])));
      if (p64) {
        p64[col] = mn;
        p64[D + col] = step[j];
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) store_k_e2(rec, L, 4 * lane + j, ke[j]);
    uint8_t* kcodes = rec + L.k_codes() + lane;  // byte (t d + 4 lane) / 4 holds channels 4 lane..+3 of token t
    if (exact) {
      uint32_t t01[kLevels], t23[kLevels];  // thresholds of channels (0, 1) and (2, 3) as half2 words
#pragma unroll
      for (int k = 0; k < kLevels; ++k) {
        t01[k] = (uint32_t)thr[0][k] | ((uint32_t)thr[1][k] << 16);
        t23[k] = (uint32_t)thr[2][k] | ((uint32_t)thr[3][k] << 16);
      }
#pragma unroll 4
      for (int t = 0; t < G; ++t) {
        const uint2 r = kr[t * (D / 4)];
        // channel j of the lane at bits 2j, 2j + 1 of the byte (pack order)
        uint32_t acc = put_codes<0, 2>(0u, code_masks(*reinterpret_cast<const __half2*>(&r.x), t01));
        acc = put_codes<4, 6>(acc, code_masks(*reinterpret_cast<const __half2*>(&r.y), t23));
        kcodes[t * (D / 4)] = (uint8_t)(acc | (acc >> 16));
      }
    } else {  // a line without exact thresholds (extreme range): the float64 recipe per element
      for (int t = 0; t < G; ++t) {
        const uint2 r = kr[t * (D / 4)];
        const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&r.x));
        const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&r.y));
        const float x[4] = {a.x, a.y, b.x, b.y};
        uint32_t byte = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          byte |= (uint32_t)quant_code_slow(x[j], fmn[j], fmx[j], (double)fmn[j], step[j], inv[j], kLevels, eps)
                  << (2 * j);
        kcodes[t * (D / 4)] = (uint8_t)byte;
      }
    }
  }

  // ---- V: token `lane`, line over the D channels (chunk j of the row at (j ^ (lane & 15)))
  if (part != 0) {
    const int t = lane;
    const uint4* vr = reinterpret_cast<const uint4*>(sv + t * D);
    const int sw = t & 15;
    __half2 mn2 = __float2half2_rn(65504.f), mx2 = __float2half2_rn(-65504.f);
#pragma unroll 4
    for (int j = 0; j < D / 8; ++j) {
      const uint4 r = vr[j ^ sw];
      const __half2* h = reinterpret_cast<const __half2*>(&r);
      mn2 = __hmin2(__hmin2(mn2, h[0]), __hmin2(h[1], __hmin2(h[2], h[3])));
      mx2 = __hmax2(__hmax2(mx2, h[0]), __hmax2(h[1], __hmax2(h[2], h[3])));
    }
    const float fmn = fminf(__low2float(mn2), __high2float(mn2));
    const float fmx = fmaxf(__low2float(mx2), __high2float(mx2));
    const double mn = (double)fmn;
    double step;
    line_params(mn, (double)fmx, (double)kLevels, step);
    const double inv = step > 0.0 ? __drcp_rn(step) : 0.0;
    uint16_t thr[kLevels];
    const bool exact = code_thresholds(thr, fmn, fmx, mn, step, inv, kLevels, eps);
    vst = (float)step;
    reinterpret_cast<float*>(rec + L.v_step())[t] = __double2float_rn(step);
    reinterpret_cast<float*>(rec + L.v_xmin())[t] = __double2float_rn(mn);
    if (p64) {
      p64[2 * D + t] = mn;
      p64[2 * D + G + t] = step;
    }
    uint32_t th[kLevels];
#pragma unroll
    for (int k = 0; k < kLevels; ++k) th[k] = (uint32_t)thr[k] * 0x00010001u;
    uint4* vcodes = reinterpret_cast<uint4*>(rec + L.v_codes() + t * (D / 4));
    if (exact) {
      uint32_t w[D / 16];
#pragma unroll
      for (int j = 0; j < D / 8; ++j) {  // chunk j = channels 8j..8j+7 -> half of word j / 2
        const uint4 r = vr[j ^ sw];
        const __half2* h = reinterpret_cast<const __half2*>(&r);
        // channels 8j + 2e (low half) and 8j + 2e + 1 (high half) at field bits 4e and 4e + 2
        uint32_t acc = put_codes<0, 2>(0u, code_masks(h[0], th));
        acc = put_codes<4, 6>(acc, code_masks(h[1], th));
        acc = put_codes<8, 10>(acc, code_masks(h[2], th));
        acc = put_codes<12, 14>(acc, code_masks(h[3], th));
        if (j & 1) w[j / 2] |= (acc + (acc << 16)) & 0xFFFF0000u;
        else w[j / 2] = (acc + (acc >> 16)) & 0xFFFFu;
      }
      vcodes[0] = make_uint4(w[0], w[1], w[2], w[3]);
      vcodes[1] = make_uint4(w[4], w[5], w[6], w[7]);
    } else {  // a line without exact thresholds: the float64 recipe per element, out of line
      frozen_v_codes_slow(vr, sw, fmn, fmx, mn, step, inv, kLevels, eps, vcodes);
    }
  }
  note_step_max(meta3, fmaxf(kst_max, vst));
}

// K1b for 4-bit codes (d = 128, G = 32): one warp per group after flush_scan_kernel, the same
// staging as flush_frozen_kernel; substituted groups (sel != 0) are handled inline (float64
// column sums of the original rows, float32 means, outlier.py:120-142). Codes take the float32
// fast path with the float64 recipe as fallback (levels = 15 would need 15 thresholds).
// kLevels = 7: 3-bit codes in the same 4-bit fields (code_bits). kBits = 2, kLevels = 1: 1-bit
// codes in 2-bit fields (K codes doubled, K step halved, K params in K2's pair order). kBits = 8: byte fields
// (8-bit codes, and 5..7-bit codes in 8-bit fields): K params in channel order with
// e = x_min - 1024 step, as K2-8 reads them.
template <int kLevels, int kBits>
__global__ void __launch_bounds__(32 * kFrozenWarps) flush_frozen4_kernel(ott_cache_t c, int64_t q0, int n_groups,
                                                                          int64_t ring_end,
                                                                          const uint16_t* __restrict__ in_k,
                                                                          const uint16_t* __restrict__ in_v,
                                                                          int64_t in_stride, int64_t in_first) {
  constexpr int D = 128, G = 32;
  constexpr int kShift = (kBits == 2 && kLevels == 1) ? 1 : 0;
  extern __shared__ __align__(16) unsigned char smem[];
  FrozenPairSmem& sm = *reinterpret_cast<FrozenPairSmem*>(smem);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // warp pairs share a group: the even warp stages and quantizes the K rows, the odd one V
  const int part = warp & 1;
  const int64_t item = ((int64_t)blockIdx.x * kFrozenWarps + warp) >> 1;
  if (item >= (int64_t)c.n_units * n_groups) return;
  int u, g;
  split_item(item, (int64_t)c.n_units * n_groups, n_groups, u, g);
  const int cap = G + c.residual;
  const int base = (int)(q0 + (int64_t)g * G);
  const int64_t gi = base / G;
  uint8_t* rec = record_ptr(c, u, gi);
  const RecordLayout L(D, G, kBits);
  uint16_t* sk = sm.rows[warp];
  uint16_t* sv = sm.rows[warp];
  const uint32_t sel = c.subst_mask[(size_t)u * mask_words_per_unit(c) + (base >> 5)];
  {
    const int bslot = base % cap, ring_end32 = (int)ring_end, in_first32 = (int)in_first;
    const int ch = lane & 15;
    if (base >= ring_end32) {  // bulk prefill: every row of the group comes from the input
      const size_t off0 = (size_t)u * in_stride + (size_t)(base - in_first32) * D;
      if (part == 0) stage_rows_bulk<false>(sk, in_k + off0, lane);
      else stage_rows_bulk<true>(sv, in_v + off0, lane);
    } else
#pragma unroll 4
    for (int it = 0; it < G / 2; ++it) {
      const int row = 2 * it + (lane >> 4);
      const int p = base + row;
      const uint16_t *pk, *pv;
      if (p < ring_end32) {
        int sl = bslot + row;
        sl = sl >= cap ? sl - cap : sl;
        const size_t off = ((size_t)u * cap + (size_t)sl) * D + ch * 8;
        pk = c.pend_k + off;
        pv = c.pend_v + off;
      } else {
        const size_t off = (size_t)u * in_stride + (size_t)(p - in_first32) * D + ch * 8;
        pk = in_k + off;
        pv = in_v + off;
      }
      if (part == 0) cp_async16(sk + row * D + ch * 8, pk);
      else cp_async16(sv + row * D + ((ch ^ (row & 15)) * 8), pv);
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncwarp();
  }
  double* p64 = c.params64 ? c.params64 + ((size_t)u * c.max_groups + (size_t)gi) * 2 * (D + G) : nullptr;
  const double eps = 1e-9 * (double)(kLevels + 1);
  int32_t* meta3 = c.pool_meta + (size_t)u * 4 + 3;
  float kst_max = 0.f, vst = 0.f;
  const uint2* kr = reinterpret_cast<const uint2*>(sk) + lane;
  // ---- K: channels 4 lane .. +3
  if (part == 0) {
    float mean[4] = {0.f, 0.f, 0.f, 0.f};
    if (sel) {
      double sum[4] = {0.0, 0.0, 0.0, 0.0};
      for (int t = 0; t < G; ++t) {
        const uint2 r = kr[t * (D / 4)];
        const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&r.x));
        const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&r.y));
        sum[0] = __dadd_rn(sum[0], (double)a.x);
        sum[1] = __dadd_rn(sum[1], (double)a.y);
        sum[2] = __dadd_rn(sum[2], (double)b.x);
        sum[3] = __dadd_rn(sum[3], (double)b.y);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) mean[j] = __double2float_rn(__ddiv_rn(sum[j], (double)G));
    }
    auto kval = [&](int t, float (&x)[4]) {
      if ((sel >> t) & 1u) {
        x[0] = mean[0]; x[1] = mean[1]; x[2] = mean[2]; x[3] = mean[3];
      } else {
        const uint2 r = kr[t * (D / 4)];
        const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&r.x));
        const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&r.y));
        x[0] = a.x; x[1] = a.y; x[2] = b.x; x[3] = b.y;
      }
    };
    float fmn[4] = {3.4e38f, 3.4e38f, 3.4e38f, 3.4e38f}, fmx[4] = {-3.4e38f, -3.4e38f, -3.4e38f, -3.4e38f};
    if (!sel) {  // fp16 rows only: packed min/max (as flush_frozen_kernel)
      __half2 mn01 = __float2half2_rn(65504.f), mn23 = mn01, mx01 = __float2half2_rn(-65504.f), mx23 = mx01;
#pragma unroll 8
      for (int t = 0; t < G; ++t) {
        const uint2 r = kr[t * (D / 4)];
        const __half2 a = *reinterpret_cast<const __half2*>(&r.x), b = *reinterpret_cast<const __half2*>(&r.y);
        mn01 = __hmin2(mn01, a);
        mx01 = __hmax2(mx01, a);
        mn23 = __hmin2(mn23, b);
        mx23 = __hmax2(mx23, b);
      }
      const float2 a = __half22float2(mn01), b = __half22float2(mn23), x = __half22float2(mx01),
                   y = __half22float2(mx23);
      fmn[0] = a.x; fmn[1] = a.y; fmn[2] = b.x; fmn[3] = b.y;
      fmx[0] = x.x; fmx[1] = x.y; fmx[2] = y.x; fmx[3] = y.y;
    } else {
      for (int t = 0; t < G; ++t) {
        float x[4];
        kval(t, x);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          fmn[j] = fminf(fmn[j], x[j]);
          fmx[j] = fmaxf(fmx[j], x[j]);
        }
      }
    }
    double step[4], inv[4];
    FastLine fl[4];
    __half* ksh = reinterpret_cast<__half*>(rec + L.k_sh());
    __half* ksl = reinterpret_cast<__half*>(rec + L.k_sl());
    float ke[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = 4 * lane + j;
      const double mn = (double)fmn[j];
      line_params(mn, (double)fmx[j], (double)kLevels, step[j]);
      inv[j] = step[j] > 0.0 ? __drcp_rn(step[j]) : 0.0;
      fl[j] = fast_line(fmn[j], fmx[j], step[j], inv[j], kLevels);
      // 1-bit codes in 2-bit fields: K codes doubled, step halved (exact; see flush_kernel)
      const double kstep = kShift ? 0.5 * step[j] : step[j];
      kst_max = fmaxf(kst_max, (float)kstep);
      const __half sh = __double2half(kstep);
      const __half sl = __double2half(__dsub_rn(kstep, (double)__half2float(sh)));
      const int kj = kBits == 2 ? kpair_index(col, D) : (kBits == 4 ? kpair4_index(col) : col);
      ksh[kj] = sh;
      ksl[kj] = sl;
      const double off = kBits == 2 ? 4.0 * (double)kpair_u(col % 8) : (kBits == 4 ? 64.0 : 1024.0);
      ke[j] = __double2float_rn(__dsub_rn(mn, __dmul_rn(off, kstep)));
      if (p64) {
        p64[col] = mn;
        p64[D + col] = step[j];
      }
    }
    if (kBits == 2) {
#pragma unroll
      for (int j = 0; j < 4; ++j) store_k_e2(rec, L, 4 * lane + j, ke[j]);
    } else {
      *reinterpret_cast<float4*>(rec + L.k_e() + 16 * lane) = make_float4(ke[0], ke[1], ke[2], ke[3]);
    }
    // channels 4 lane..+3 of token t: one byte of 2-bit fields, one uint16 of nibbles or one uint32 of bytes
    uint8_t* kcodes2 = rec + L.k_codes() + lane;
    uint16_t* kcodes4 = reinterpret_cast<uint16_t*>(rec + L.k_codes()) + lane;
    uint32_t* kcodes8 = reinterpret_cast<uint32_t*>(rec + L.k_codes()) + lane;
    bool done = false;
    if constexpr (kBits == 4 && (kLevels == 15 || kLevels == 7)) {
      if (!sel) {  // fp16 inputs: exact fp16 thresholds per line (code_thresholds), binary search
        uint16_t thr[4][kLevels];
        bool exact = true;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          exact &= code_thresholds(thr[j], fmn[j], fmx[j], (double)fmn[j], step[j], inv[j], kLevels, eps);
        if (exact) {
          uint32_t t01[kLevels], t23[kLevels];
#pragma unroll
          for (int k = 0; k < kLevels; ++k) {
            t01[k] = (uint32_t)thr[0][k] | ((uint32_t)thr[1][k] << 16);
            t23[k] = (uint32_t)thr[2][k] | ((uint32_t)thr[3][k] << 16);
          }
#pragma unroll 2
          for (int t = 0; t < G; ++t) {
            const uint2 r = kr[t * (D / 4)];
            uint32_t b[4];
            nib_masks<kLevels>(*reinterpret_cast<const __half2*>(&r.x), t01, b);
            uint32_t acc = put_nibs<0, 4>(0u, b);  // channels 4 lane, 4 lane + 1: nibbles 0, 1
            nib_masks<kLevels>(*reinterpret_cast<const __half2*>(&r.y), t23, b);
            acc = put_nibs<8, 12>(acc, b);         // channels 4 lane + 2, + 3: nibbles 2, 3
            kcodes4[t * (D / 4)] = (uint16_t)(acc | (acc >> 16));
          }
          done = true;
        }
      }
    }
    if (!done)
#pragma unroll 4
    for (int t = 0; t < G; ++t) {
      float x[4];
      kval(t, x);
      uint32_t h = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        bool slow;
        int code = quant_code_f32(x[j], fmn[j], fmx[j], kLevels, fl[j], slow);
        if (slow) code = quant_code_slow(x[j], fmn[j], fmx[j], (double)fmn[j], step[j], inv[j], kLevels, eps);
        h |= (uint32_t)(code << kShift) << (kBits * j);
      }
      if (kBits == 2) kcodes2[t * (D / 4)] = (uint8_t)h;
      else if (kBits == 4) kcodes4[t * (D / 4)] = (uint16_t)h;
      else kcodes8[t * (D / 4)] = h;
    }
  }
  // ---- V column means (substituted groups only): lane l sums channels 4l..4l+3
  if (part == 1 && sel) {
    double sum[4] = {0.0, 0.0, 0.0, 0.0};
    for (int t = 0; t < G; ++t) {
      const uint2 r = *reinterpret_cast<const uint2*>(sv + t * D + (((lane >> 1) ^ (t & 15)) * 8) + (lane & 1) * 4);
      const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&r.x));
      const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&r.y));
      sum[0] = __dadd_rn(sum[0], (double)a.x);
      sum[1] = __dadd_rn(sum[1], (double)a.y);
      sum[2] = __dadd_rn(sum[2], (double)b.x);
      sum[3] = __dadd_rn(sum[3], (double)b.y);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) sm.vmean[warp][4 * lane + j] = __double2float_rn(__ddiv_rn(sum[j], (double)G));
    __syncwarp();
  }
  // ---- V: token `lane`
  if (part == 1) {
    const int t = lane;
    const bool subst = (sel >> t) & 1u;
    const uint4* vr = reinterpret_cast<const uint4*>(sv + t * D);
    const int sw = t & 15;
    const float* vm = sm.vmean[warp];
    auto vval = [&](int j, float (&x)[8]) {  // channels 8j..8j+7
      if (subst) {
#pragma unroll
        for (int e = 0; e < 8; ++e) x[e] = vm[8 * j + e];
      } else {
        const uint4 r = vr[j ^ sw];
        const __half2* h = reinterpret_cast<const __half2*>(&r);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __half22float2(h[e]);
          x[2 * e] = f.x;
          x[2 * e + 1] = f.y;
        }
      }
    };
    float fmn = 3.4e38f, fmx = -3.4e38f;
    if (!subst) {  // fp16 row: packed min/max
      __half2 mn2 = __float2half2_rn(65504.f), mx2 = __float2half2_rn(-65504.f);
#pragma unroll 4
      for (int j = 0; j < D / 8; ++j) {
        const uint4 r = vr[j ^ sw];
        const __half2* h = reinterpret_cast<const __half2*>(&r);
        mn2 = __hmin2(__hmin2(mn2, h[0]), __hmin2(h[1], __hmin2(h[2], h[3])));
        mx2 = __hmax2(__hmax2(mx2, h[0]), __hmax2(h[1], __hmax2(h[2], h[3])));
      }
      fmn = fminf(__low2float(mn2), __high2float(mn2));
      fmx = fmaxf(__low2float(mx2), __high2float(mx2));
    } else {
      for (int j = 0; j < D / 8; ++j) {
        float x[8];
        vval(j, x);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          fmn = fminf(fmn, x[e]);
          fmx = fmaxf(fmx, x[e]);
        }
      }
    }
    const double mn = (double)fmn;
    double step;
    line_params(mn, (double)fmx, (double)kLevels, step);
    const double inv = step > 0.0 ? __drcp_rn(step) : 0.0;
    const FastLine fl = fast_line(fmn, fmx, step, inv, kLevels);
    vst = (float)step;
    reinterpret_cast<float*>(rec + L.v_step())[t] = __double2float_rn(step);
    reinterpret_cast<float*>(rec + L.v_xmin())[t] = __double2float_rn(mn);
    if (p64) {
      p64[2 * D + t] = mn;
      p64[2 * D + G + t] = step;
    }
    constexpr int kWords = D * kBits / 32;  // words of one token's V codes
    uint32_t w[kWords];
    if (kBits == 2) {
#pragma unroll
      for (int q = 0; q < kWords; ++q) w[q] = 0u;
    }
    bool vdone = false;
    if constexpr (kBits == 4 && (kLevels == 15 || kLevels == 7)) {
      if (!subst) {  // fp16 inputs: exact thresholds, binary search (see the K part)
        uint16_t thr[kLevels];
        if (code_thresholds(thr, fmn, fmx, mn, step, inv, kLevels, eps)) {
          uint32_t th[kLevels];
#pragma unroll
          for (int k = 0; k < kLevels; ++k) th[k] = (uint32_t)thr[k] * 0x00010001u;
#pragma unroll 2
          for (int j = 0; j < D / 8; ++j) {  // chunk j = channels 8j..8j+7 = nibbles of word j
            const uint4 r = vr[j ^ sw];
            const __half2* h = reinterpret_cast<const __half2*>(&r);
            uint32_t b[4];
            nib_masks<kLevels>(h[0], th, b);
            uint32_t lo = put_nibs<0, 4>(0u, b);
            nib_masks<kLevels>(h[1], th, b);
            lo = put_nibs<8, 12>(lo, b);
            nib_masks<kLevels>(h[2], th, b);
            uint32_t hi = put_nibs<0, 4>(0u, b);
            nib_masks<kLevels>(h[3], th, b);
            hi = put_nibs<8, 12>(hi, b);
            w[j] = ((lo | (lo >> 16)) & 0xFFFFu) | ((hi | (hi >> 16)) << 16);
          }
          vdone = true;
        }
      }
    }
    if (!vdone)
#pragma unroll
    for (int j = 0; j < D / 8; ++j) {  // chunk j = channels 8j..8j+7 = word j (nibbles) / 2j, 2j+1 (bytes)
      float x[8];
      vval(j, x);
      uint32_t bits[2] = {0u, 0u};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        bool slow;
        int code = quant_code_f32(x[e], fmn, fmx, kLevels, fl, slow);
        if (slow) code = quant_code_slow(x[e], fmn, fmx, mn, step, inv, kLevels, eps);
        if (kBits == 2) bits[0] |= (uint32_t)code << (2 * e);
        else if (kBits == 4) bits[0] |= (uint32_t)code << (4 * e);
        else bits[e >> 2] |= (uint32_t)code << (8 * (e & 3));
      }
      if (kBits == 2) {
        w[j >> 1] |= bits[0] << (16 * (j & 1));
      } else if (kBits == 4) {
        w[j] = bits[0];
      } else {
        w[2 * j] = bits[0];
        w[2 * j + 1] = bits[1];
      }
    }
    uint4* vcodes = reinterpret_cast<uint4*>(rec + L.v_codes() + t * (D * kBits / 8));
#pragma unroll
    for (int q = 0; q < kWords / 4; ++q) vcodes[q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
  }
  note_step_max(meta3, fmaxf(kst_max, vst));
}

// K4: ring write. One thread per 8 halves.
__global__ void ring_write_kernel(ott_cache_t c, const uint16_t* __restrict__ k, const uint16_t* __restrict__ v,
                                  int64_t in_stride, int64_t in_first, int64_t first_pos, int64_t n_rows,
                                  const int64_t* __restrict__ dev_counts) {
  if (dev_counts) {  // device-counter decode step: one row at position total_tokens
    first_pos = dev_counts[1];
    in_first = first_pos;
  }
  const int d = c.head_dim;
  const int cap = c.group_size + c.residual;
  if (d % 8) {  // head dims that are not whole 16-byte chunks: one thread per element
    const int64_t total = (int64_t)c.n_units * n_rows * d;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
      const int j = (int)(idx % d);
      const int64_t r = (idx / d) % n_rows;
      const int u = (int)(idx / ((int64_t)d * n_rows));
      const int64_t p = first_pos + r;
      const size_t src = (size_t)u * in_stride + (size_t)(p - in_first) * d + j;
      const size_t dst = ((size_t)u * cap + (size_t)(p % cap)) * d + j;
      c.pend_k[dst] = k[src];
      c.pend_v[dst] = v[src];
    }
    return;
  }
  const int vec_per_row = d / 8;
  const int64_t total = (int64_t)c.n_units * n_rows * vec_per_row;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(idx % vec_per_row);
    const int64_t r = (idx / vec_per_row) % n_rows;
    const int u = (int)(idx / (vec_per_row * n_rows));
    const int64_t p = first_pos + r;
    const size_t src = (size_t)u * in_stride + (size_t)(p - in_first) * d + j * 8;
    const size_t dst = ((size_t)u * cap + (size_t)(p % cap)) * d + j * 8;
    *reinterpret_cast<uint4*>(c.pend_k + dst) = *reinterpret_cast<const uint4*>(k + src);
    *reinterpret_cast<uint4*>(c.pend_v + dst) = *reinterpret_cast<const uint4*>(v + src);
  }
}

cudaError_t launch_flush(const ott_cache_t& c, int64_t q0, int n_groups, int64_t ring_end, const uint16_t* in_k,
                         const uint16_t* in_v, int64_t in_stride, int64_t in_first, cudaStream_t st,
                         const int64_t* dev_counts) {
  const size_t smem = flush_smem_bytes(c.head_dim, c.group_size, c.capacity);
  cudaError_t e = cudaFuncSetAttribute(flush_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  // host-triggered flushes at the tensor-core shapes (bulk prefill and decode flushes): the
  // sequential kernel runs only the pool competition (scoring, OutlierPool.update, masks,
  // pool/aux rows) group by group -- nothing once a unit's pool has frozen -- then
  // flush_frozen_kernel substitutes and quantizes all groups in parallel, a warp pair per group
  const bool split = OTT_FLUSH_SPLIT && !dev_counts && c.head_dim == 128 && c.group_size == 32;
  if (!split) {
    flush_kernel<<<c.n_units, kFlushThreads, smem, st>>>(c, q0, n_groups, ring_end, in_k, in_v, in_stride, in_first,
                                                           dev_counts);
    return cudaGetLastError();
  }
  // a pool that can absorb many evictions before freezing (N < A) stays active for long: score
  // all tokens in parallel first, so the sequential scan reads 256 B of scores per group
  const bool prescore = OTT_FLUSH_PRESCORE && c.capacity > 0 && c.capacity < c.aux_capacity;
  const int64_t n_items = (int64_t)c.n_units * n_groups;
  if (prescore) {
    flush_score_kernel<<<(unsigned)((n_items + 3) / 4), 128, 0, st>>>(c, q0, n_groups, ring_end, in_k, in_stride,
                                                                     in_first);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  e = cudaFuncSetAttribute(flush_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(ScanSmem));
  if (e != cudaSuccess) return e;
  flush_scan_kernel<<<(c.n_units + kScanWarps - 1) / kScanWarps, 32 * kScanWarps, sizeof(ScanSmem), st>>>(
      c, q0, n_groups, ring_end, in_k, in_v, in_stride, in_first, prescore);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int64_t items = (int64_t)c.n_units * n_groups;
  if (c.bits != 2) {  // 2-bit fields (1 bit), 4-bit fields (3, 4 bits) and byte fields (5..8 bits)
    auto kern = c.bits == 1   ? flush_frozen4_kernel<1, 2>
                : c.bits == 3 ? flush_frozen4_kernel<7, 4>
                : c.bits == 4 ? flush_frozen4_kernel<15, 4>
                : c.bits == 5 ? flush_frozen4_kernel<31, 8>
                : c.bits == 6 ? flush_frozen4_kernel<63, 8>
                : c.bits == 7 ? flush_frozen4_kernel<127, 8>
                              : flush_frozen4_kernel<255, 8>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(FrozenPairSmem));
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)((2 * items + kFrozenWarps - 1) / kFrozenWarps), 32 * kFrozenWarps, sizeof(FrozenPairSmem),
           st>>>(c, q0, n_groups, ring_end, in_k, in_v, in_stride, in_first);
    return cudaGetLastError();
  }
  const size_t fsm = OTT_FROZEN_PAIR ? sizeof(FrozenPairSmem) : sizeof(FrozenSmem);
  const int64_t warps = OTT_FROZEN_PAIR ? 2 * items : items;
  e = cudaFuncSetAttribute(flush_frozen_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm);
  if (e != cudaSuccess) return e;
  flush_frozen_kernel<<<(unsigned)((warps + kFrozenWarps - 1) / kFrozenWarps), 32 * kFrozenWarps, fsm, st>>>(
      c, q0, n_groups, ring_end, in_k, in_v, in_stride, in_first);
  return cudaGetLastError();
}

cudaError_t launch_ring_write(const ott_cache_t& c, const uint16_t* k, const uint16_t* v, int64_t in_stride,
                              int64_t in_first, int64_t first_pos, int64_t n_rows, cudaStream_t st,
                              const int64_t* dev_counts) {
  const int64_t total = (int64_t)c.n_units * n_rows * (c.head_dim % 8 ? c.head_dim : c.head_dim / 8);
  int blocks = (int)((total + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  ring_write_kernel<<<blocks, 256, 0, st>>>(c, k, v, in_stride, in_first, first_pos, n_rows, dev_counts);
  return cudaGetLastError();
}

}  // namespace ott
