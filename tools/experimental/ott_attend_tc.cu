// ott_attend_tc.cu — K2 for the 2-bit hot path (d = 128, G = 32): Q K^T on the 5th-generation
// tensor cores (tcgen05.mma, accumulator in TMEM), P V on the warp-level tensor cores.
//
// Reference semantics: attend_mixed (attention.py:79-92) over reconstructed_kv (62-76):
// quantized groups are dequantized as code * step + x_min (quant.py:105-111), positions in
// pool.entries are masked here and attended from the pool rows by the full-precision CTA
// (fp_body), softmax over all tiers (attend_full_precision, attention.py:35-59).
//
// Every warp is an independent pipeline over its own groups (no CTA-wide round trip):
//   1. TMA (one elected lane) streams the warp's group records into a 3-stage ring.
//   2. K side of group k+1, thread = token: the 2-bit K codes become fp16 1 + c 2^(2P-10)
//      (one LOP3 per pair, as in K2) and are stored into the warp's 32 TMEM lanes
//      (tcgen05.st 32x32b, the A operand); lane = (head, word pair) forms q' = q u step
//      as an exact fp16 hi/lo split into the warp's own B tile (16 rows: 8 hi, 8 lo; K-major
//      canonical layout) and the x_min bias sum_c q e. One elected lane issues 8
//      tcgen05.mma kind::f16 (M = 128, N = 16, K = 16) into the warp's own 16 TMEM columns
//      and commits to the warp's mbarrier. The MMA computes all 128 rows; only the warp's
//      32 lanes are read (the other rows are other warps' tokens against this warp's B).
//   3. Softmax of group k, thread = token: tcgen05.ld of its 16 logit columns, pool mask,
//      lazily rescaled online softmax (per warp), P' = 4 p v_step through shared memory
//      (ldmatrix.trans) into the B fragments of V^T P' (mma.sync m16n8k16, V codes as exact
//      fp16 subnormals, accumulators in registers).
// The MMA of group k+1 runs under the softmax and P V of group k.
#include "ott_attend.cuh"

namespace ott {

constexpr float kTcqMinit = -1e30f;  // finite initial running max (no -inf - -inf = NaN special cases)

namespace tcq {
constexpr int kWarps = 4;
constexpr int kThreads = 32 * kWarps;
constexpr int kStages = 3;                        // record stages per warp
constexpr int kRec = 3328;                        // record bytes at d = 128, G = 32
constexpr uint32_t kLBO = 128, kSBO = 16 * 128;   // B tile core-matrix strides (K, N), bytes
constexpr uint32_t kCols = 128;                   // TMEM: A at [0, 64) (f16 pairs), D of warp w at 64 + 16 w
constexpr uint32_t kIdesc = (1u << 4)             // D f32; A, B f16, both K-major
                            | ((uint32_t)(16 >> 3) << 17)    // N = 16
                            | ((uint32_t)(128 >> 4) << 24);  // M = 128
}  // namespace tcq

struct TcqSmem {
  alignas(256) uint8_t stage[tcq::kWarps][tcq::kStages][tcq::kRec];
  alignas(128) uint8_t bq[tcq::kWarps][2 * tcq::kSBO];  // q' rows: hi (heads 0-7), lo (heads 0-7)
  alignas(16) uint16_t pp[tcq::kWarps][32][8];          // P' [token][head]
  alignas(16) float4 qt[8][32];                          // q (fp32): [k][lane] = q[lane % 8][32 (lane / 8) + 4k ..]
  alignas(16) float bias[tcq::kWarps][2][8];             // scale * sum_c q e, per (warp, group parity, head)
  float mm[tcq::kWarps][8], ll[tcq::kWarps][8];
  alignas(8) uint64_t rbar[tcq::kWarps][tcq::kStages];
  alignas(8) uint64_t mbar[tcq::kWarps];
  uint32_t tmem_base;
};

__device__ __forceinline__ uint64_t tcq_bdesc(uint32_t saddr) {  // K-major, no swizzle (layout type 0), sm100 version bit
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(tcq::kLBO >> 4) << 16) |
         ((uint64_t)(tcq::kSBO >> 4) << 32) | (1ull << 46);
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}
// Two K code words (channels 16j .. 16j+31 of this lane's token) -> 16 fp16 pairs
// 1 + c 2^(2P-10) (pair m of a word from w << 6, w or w >> 6, see kq) stored to TMEM columns
// [taddr, taddr + 16). One asm block, so the results are produced directly in the registers
// tcgen05.st reads (no register moves).
__device__ __forceinline__ void tmem_unpack_st16(uint32_t taddr, uint32_t w0, uint32_t w1, uint32_t magic) {
#define OTT_KW(W, B)                                                   \
  "shl.b32 l6, " W ", 6;\n shr.b32 r6, " W ", 6;\n"                    \
  "lop3.b32 r" #B "0, l6, 0x00C000C0, %3, 0xEA;\n"                     \
  "lop3.b32 r" #B "1, l6, 0x03000300, %3, 0xEA;\n"                     \
  "lop3.b32 r" #B "2, " W ", 0x00300030, %3, 0xEA;\n"                  \
  "lop3.b32 r" #B "3, " W ", 0x00C000C0, %3, 0xEA;\n"                  \
  "lop3.b32 r" #B "4, " W ", 0x03000300, %3, 0xEA;\n"                  \
  "lop3.b32 r" #B "5, r6, 0x00300030, %3, 0xEA;\n"                     \
  "lop3.b32 r" #B "6, r6, 0x00C000C0, %3, 0xEA;\n"                     \
  "lop3.b32 r" #B "7, r6, 0x03000300, %3, 0xEA;\n"
  asm volatile(
      "{\n .reg .b32 l6, r6, ra0, ra1, ra2, ra3, ra4, ra5, ra6, ra7, rb0, rb1, rb2, rb3, rb4, rb5, rb6, rb7;\n"
      OTT_KW("%1", a) OTT_KW("%2", b)
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {ra0, ra1, ra2, ra3, ra4, ra5, ra6, ra7, rb0, rb1, rb2, rb3, rb4,"
      " rb5, rb6, rb7};\n}\n" ::"r"(taddr),
      "r"(w0), "r"(w1), "r"(magic)
      : "memory");
#undef OTT_KW
}
// The group's 8 Q K^T MMAs (k-step s: A columns 8s, B rows advanced by 2 core matrices) and
// the commit to the warp's mbarrier, in one asm block issued by one lane: the operands go to
// uniform registers once.
struct TcqDesc {  // loop-invariant Q K^T operands of one warp (kept in uniform registers)
  uint64_t b[8];   // B descriptors of the 8 k-steps
  uint32_t a[8];   // A (TMEM) columns of the 8 k-steps
  uint32_t d;      // D columns
};
__device__ __forceinline__ void tcq_issue_qk(const TcqDesc& q, uint32_t mbar) {
  // whole warp (converged): elect.sync picks the one issuing lane
  asm volatile(
      "{\n .reg .pred pe;\n"
      " elect.sync _|pe, 0xffffffff;\n"
      " @pe tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %9, %17, 0;\n"
      " @pe tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %10, %17, 1;\n"
      " @pe tcgen05.mma.cta_group::1.kind::f16 [%0], [%3], %11, %17, 1;\n"
      " @pe tcgen05.mma.cta_group::1.kind::f16 [%0], [%4], %12, %17, 1;\n"
      " @pe tcgen05.mma.cta_group::1.kind::f16 [%0], [%5], %13, %17, 1;\n"
      " @pe tcgen05.mma.cta_group::1.kind::f16 [%0], [%6], %14, %17, 1;\n"
      " @pe tcgen05.mma.cta_group::1.kind::f16 [%0], [%7], %15, %17, 1;\n"
      " @pe tcgen05.mma.cta_group::1.kind::f16 [%0], [%8], %16, %17, 1;\n"
      " @pe tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%18];\n}\n" ::"r"(q.d),
      "r"(q.a[0]), "r"(q.a[1]), "r"(q.a[2]), "r"(q.a[3]), "r"(q.a[4]), "r"(q.a[5]), "r"(q.a[6]), "r"(q.a[7]),
      "l"(q.b[0]), "l"(q.b[1]), "l"(q.b[2]), "l"(q.b[3]), "l"(q.b[4]), "l"(q.b[5]), "l"(q.b[6]), "l"(q.b[7]),
      "n"(tcq::kIdesc), "r"(mbar)
      : "memory");
}
// V code pairs as exact fp16 subnormals c 2^(2P-24) in place: pair m (channels m, m+8 of a
// code word) at mantissa position P = m for m <= 4 (AND only), P = m - 5 for m >= 5 (from
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
template <int I>
__device__ __forceinline__ float tcq_pick4(const float (&v)[8], int tig) {  // v[2 tig + I]
  return tig == 0 ? v[I] : (tig == 1 ? v[2 + I] : (tig == 2 ? v[4 + I] : v[6 + I]));
}

// K side of one group for warp w: A rows (this warp's 32 TMEM lanes), q' rows of B, bias;
// then one lane issues the group's Q K^T and commits to the warp's mbarrier.
template <int NR>
__device__ __forceinline__ void tcq_kside(TcqSmem& sm, int w, int lane, const uint8_t* rec, uint32_t a_lane,
                                          const TcqDesc& qd, uint32_t mbar, const __half2 (&q16)[2][8],
                                          uint32_t magic, float scale, int slot) {
  const RecordLayout L(128, 32);
  {  // A row = token `lane`: 8 code words -> 64 fp16 pairs, stored as two 32-column halves
    const uint4 c0 = *reinterpret_cast<const uint4*>(rec + swz(L.k_codes() + lane * 32));
    const uint4 c1 = *reinterpret_cast<const uint4*>(rec + swz(L.k_codes() + lane * 32 + 16));
    tmem_unpack_st16(a_lane, c0.x, c0.y, magic);
    tmem_unpack_st16(a_lane + 16, c0.z, c0.w, magic);
    tmem_unpack_st16(a_lane + 32, c1.x, c1.y, magic);
    tmem_unpack_st16(a_lane + 48, c1.z, c1.w, magic);
  }
  // q' rows: lane = (head h = lane % 8, word pair e4 = lane / 8: code words 2e4, 2e4+1 =
  // channels 32e4 .. 32e4+31). Lanes 8k..8k+7 write rows 0..7 of one core matrix:
  // 128 contiguous bytes per store phase, bank-conflict free.
  const int h = lane & 7, e4 = lane >> 3;
  float part = 0.f;
  if (h < NR) {
    float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};  // sum_c q_c e_c (FFMA2)
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float4 ev = *reinterpret_cast<const float4*>(rec + swz(L.k_e() + 128 * e4 + 16 * k));
      const float4 qv = sm.qt[k][lane];
      acc[0] = __ffma2_rn(make_float2(qv.x, qv.y), make_float2(ev.x, ev.y), acc[0]);
      acc[1] = __ffma2_rn(make_float2(qv.z, qv.w), make_float2(ev.z, ev.w), acc[1]);
    }
    part = (acc[0].x + acc[0].y) + (acc[1].x + acc[1].y);
    uint8_t* bq = &sm.bq[w][0];
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
      uint8_t* bh = bq + (2 * wd) * tcq::kLBO + h * 16;
      uint8_t* bl = bh + tcq::kSBO;
      *reinterpret_cast<uint4*>(bh) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<uint4*>(bh + tcq::kLBO) = make_uint4(hi[4], hi[5], hi[6], hi[7]);
      *reinterpret_cast<uint4*>(bl) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
      *reinterpret_cast<uint4*>(bl + tcq::kLBO) = make_uint4(lo[4], lo[5], lo[6], lo[7]);
    }
  }
  // reduce over the 4 word pairs (all lanes take part; idle heads carry 0)
  part += __shfl_xor_sync(0xffffffffu, part, 8);
  part += __shfl_xor_sync(0xffffffffu, part, 16);
  if (e4 == 0) sm.bias[w][slot][h] = part * scale;
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // B rows visible to the tensor core
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncwarp();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  tcq_issue_qk(qd, mbar);
  __syncwarp();
}

// Quantized-region partial for (unit blockIdx.x, split blockIdx.y < n_qsplits).
template <int NR>
__device__ void tcq_body(const AttnArgs& a, const Counts& n, const CUtensorMap* tmap, TcqSmem& sm) {
  constexpr int D = 128, G = 32, kS = tcq::kStages, kW = tcq::kWarps;
  const RecordLayout L(D, G);
  const ott_cache_t& c = a.c;
  const int u = blockIdx.x, split = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31;
  // warp-uniform in the compiler's eyes (shuffle from lane 0): the tcgen05 operands derived
  // from it live in uniform registers, so the MMA issue needs no per-lane waterfall
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int g = lane >> 2, tig = lane & 3;
  const int n_groups = (int)(n.q_tokens / G);
  const int per = (n_groups + a.n_qsplits - 1) / a.n_qsplits;
  const int g0 = split * per;
  const int g1 = min(n_groups, g0 + per);
  const int my_n = g1 > g0 + warp ? (g1 - g0 - warp + kW - 1) / kW : 0;
  const int64_t unit_rec = (int64_t)u * c.max_groups;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&sm.tmem_base)),
                 "n"(tcq::kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  const uint32_t rbar0 = (uint32_t)__cvta_generic_to_shared(&sm.rbar[warp][0]);
  const uint32_t stage0 = (uint32_t)__cvta_generic_to_shared(&sm.stage[warp][0][0]);
  const uint32_t mbar = (uint32_t)__cvta_generic_to_shared(&sm.mbar[warp]);
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kS; ++s) mbar_init(rbar0 + 8 * s, 1);
    mbar_init(mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
#pragma unroll
    for (int s = 0; s < kS; ++s)
      if (s < my_n) load_record<G>(stage0 + s * tcq::kRec, tmap, unit_rec + g0 + warp + s * kW, rbar0 + 8 * s);
  }
  for (int i = tid; i < 8 * 32; i += tcq::kThreads) {  // q table: [k][lane] = q[lane % 8][32 (lane / 8) + 4k ..]
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
  if (NR < 8)  // B rows of absent heads stay zero (their logit columns are never used)
    for (int i = tid; i < kW * 2 * (int)tcq::kSBO / 16; i += tcq::kThreads)
      reinterpret_cast<uint4*>(&sm.bq[0][0])[i] = make_uint4(0u, 0u, 0u, 0u);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = __shfl_sync(0xffffffffu, sm.tmem_base, 0);

  const uint32_t magic = a.k_magic;
  const float scale = a.scale_log2, scale4 = 4.f * a.scale_log2;
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
  const uint32_t a_lane = tmem + ((uint32_t)(32 * warp) << 16);          // A rows of this warp
  const uint32_t d_col = tmem + 64 + 16 * warp;                           // this warp's D columns
  const uint32_t d_lane = d_col + ((uint32_t)(32 * warp) << 16);
  const uint32_t b_s = (uint32_t)__cvta_generic_to_shared(&sm.bq[warp][0]);
  TcqDesc qd;
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    qd.b[s] = tcq_bdesc(b_s + s * 2 * tcq::kLBO);  // k-step s: 2 core matrices further along K
    qd.a[s] = tmem + 8 * s;                         // 16 fp16 = 8 TMEM columns per k-step
  }
  qd.d = d_col;
  const uint32_t pp_s = (uint32_t)__cvta_generic_to_shared(&sm.pp[warp][0][0]);
  const uint32_t lm_off = (uint32_t)(((lane & 7) + ((lane >> 3) & 1) * 8) * 32 + (lane >> 4) * 16);
  const uint32_t* pmask = c.pool_mask + (size_t)u * mask_words_per_unit(c);

  float o[8][4];
#pragma unroll
  for (int cm = 0; cm < 8; ++cm) o[cm][0] = o[cm][1] = o[cm][2] = o[cm][3] = 0.f;
  float m[8], l[8], vb[8];
#pragma unroll
  for (int h = 0; h < 8; ++h) {
    m[h] = kTcqMinit;
    l[h] = 0.f;
    vb[h] = 0.f;
  }

  if (my_n > 0) {
    mbar_wait(rbar0, 0u);
    tcq_kside<NR>(sm, warp, lane, &sm.stage[warp][0][0], a_lane, qd, mbar, q16, magic, scale, 0);
  }
#pragma unroll 1
  for (int k = 0; k < my_n; ++k) {
    const int gk = g0 + warp + k * kW;
    const uint32_t mword = __ldg(&pmask[gk]);
    // ---- logits of group k (thread = token: 8 hi columns, 8 lo columns)
    mbar_wait(mbar, (uint32_t)(k & 1));
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    uint32_t sv[16];
    tmem_ld16_nowait(d_lane, sv);
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    const int st = k % kS;
    const uint8_t* rec = &sm.stage[warp][st][0];
    const uint32_t rec_s = stage0 + st * tcq::kRec;
    const float4 b0 = *reinterpret_cast<const float4*>(&sm.bias[warp][k & 1][0]);
    const float4 b1 = *reinterpret_cast<const float4*>(&sm.bias[warp][k & 1][4]);
    const float bias[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    const bool pooled = (mword >> lane) & 1u;
    // x = logit - m (log2 units) with the running max folded into the per-group bias
    float bm[8], x[8];
#pragma unroll
    for (int h = 0; h < 8; ++h) bm[h] = bias[h] - m[h];
#pragma unroll
    for (int h = 0; h < 8; ++h)
      x[h] = (h < NR && !pooled)
                 ? fmaf(__uint_as_float(sv[h]), scale4, fmaf(__uint_as_float(sv[8 + h]), scale4, bm[h]))
                 : -INFINITY;
    // lazily rescaled online softmax: the warp's running max moves only when a logit
    // exceeds it by kLazy (p <= 2^kLazy keeps P' = 4 p step in fp16 range). m starts at a
    // finite -1e30, so the first group always takes this path.
    float dmax = x[0];
#pragma unroll
    for (int h = 1; h < NR; ++h) dmax = fmaxf(dmax, x[h]);
    if (__any_sync(0xffffffffu, dmax > kLazy)) {
      float corr[8];
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        corr[h] = 1.f;
        if (h < NR) {
          const float sh = (!pooled) ? fmaf(__uint_as_float(sv[h]), scale4, fmaf(__uint_as_float(sv[8 + h]), scale4, bias[h]))
                                     : -INFINITY;
          const float mnew = fmaxf(m[h], warp_max(sh));
          corr[h] = ex2(m[h] - mnew);
          m[h] = mnew;
          l[h] *= corr[h];
          vb[h] *= corr[h];
          x[h] = sh - mnew;
        }
      }
      const float c0 = tcq_pick4<0>(corr, tig), c1 = tcq_pick4<1>(corr, tig);
#pragma unroll
      for (int cm = 0; cm < 8; ++cm) {
        o[cm][0] *= c0;
        o[cm][1] *= c1;
        o[cm][2] *= c0;
        o[cm][3] *= c1;
      }
    }
    const float vs = *reinterpret_cast<const float*>(rec + swz(L.v_step() + 4 * lane));
    const float vx = *reinterpret_cast<const float*>(rec + swz(L.v_xmin() + 4 * lane));
    const float f = 4.f * vs;
    float pq[8];
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      pq[h] = 0.f;
      if (h < NR) {
        const float p = ex2(x[h]);
        l[h] += p;
        vb[h] = fmaf(p, vx, vb[h]);
        pq[h] = p * f;
      }
    }
    *reinterpret_cast<uint4*>(&sm.pp[warp][lane][0]) =
        make_uint4(pack_h2(pq[0], pq[1]), pack_h2(pq[2], pq[3]), pack_h2(pq[4], pq[5]), pack_h2(pq[6], pq[7]));
    // ---- K side of group k + 1 (the logits of group k are consumed): its Q K^T runs
    // under this group's P V
    if (k + 1 < my_n) {
      const int s1 = (k + 1) % kS;
      mbar_wait(rbar0 + 8 * s1, (uint32_t)(((k + 1) / kS) & 1));
      tcq_kside<NR>(sm, warp, lane, &sm.stage[warp][s1][0], a_lane, qd, mbar, q16, magic, scale, (k + 1) & 1);
    } else {
      __syncwarp();
    }
    uint32_t bq[4];
    ldsm_x4_t(bq, pp_s + lane * 16);
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const uint32_t bb0 = bq[2 * mt], bb1 = bq[2 * mt + 1];
      uint32_t vr[4];
      ldsm_x4_t(vr, rec_s + swz(L.v_codes() + mt * 16 * 32 + lm_off));
      const VSrc v0 = vsrc(vr[0]), v1 = vsrc(vr[1]), v2 = vsrc(vr[2]), v3 = vsrc(vr[3]);
#define OTT_PVQ(CM) mma16816(o[CM], vqt<CM>(v0), vqt<CM>(v2), vqt<CM>(v1), vqt<CM>(v3), bb0, bb1);
      OTT_PVQ(0) OTT_PVQ(1) OTT_PVQ(2) OTT_PVQ(3) OTT_PVQ(4) OTT_PVQ(5) OTT_PVQ(6) OTT_PVQ(7)
#undef OTT_PVQ
    }
    // ---- release this stage: prefetch the record of group k + kStages
    __syncwarp();
    if (lane == 0 && k + kS < my_n) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      load_record<G>(stage0 + st * tcq::kRec, tmap, unit_rec + g0 + warp + (k + kS) * kW, rbar0 + 8 * st);
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
      sm.mm[warp][h] = l[h] > 0.f ? m[h] : -INFINITY;  // no token seen: empty partial
      sm.ll[warp][h] = l[h];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();  // every warp is past its loop: stage memory is free, no MMA in flight
  {
    float* accw = reinterpret_cast<float*>(&sm.stage[warp][0][0]);  // [8 heads][128] natural channel order
    const float vb0 = tcq_pick4<0>(vb, tig), vb1 = tcq_pick4<1>(vb, tig);
#pragma unroll
    for (int cm = 0; cm < 8; ++cm) {
      const float f = (float)(1 << (22 - 2 * vpos(cm)));  // 2^(22-2P)
      accw[(2 * tig) * D + 8 * g + cm] = fmaf(o[cm][0], f, vb0);
      accw[(2 * tig + 1) * D + 8 * g + cm] = fmaf(o[cm][1], f, vb1);
      accw[(2 * tig) * D + 64 + 8 * g + cm] = fmaf(o[cm][2], f, vb0);
      accw[(2 * tig + 1) * D + 64 + 8 * g + cm] = fmaf(o[cm][3], f, vb1);
    }
  }
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(tcq::kCols));
  }
  for (int i = tid; i < NR * D; i += tcq::kThreads) {
    const int r = i / D, col = i % D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kW; ++w) M = fmaxf(M, sm.mm[w][r]);
    float Lsum = 0.f, A = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int w = 0; w < kW; ++w) {
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

template <int NR>
__global__ void __launch_bounds__(tcq::kThreads, 3)
    attend_tcq_kernel(const __grid_constant__ AttnArgs a, const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(256) unsigned char smem_raw[];
  allow_dependents();
  if ((int)blockIdx.y >= a.n_qsplits) {  // full-precision tiers: pool + pending
    const Counts n = counts_of(a);
    if (blockIdx.x == 0 && blockIdx.y == a.n_qsplits && threadIdx.x == 0)  // token counts for the combine's guard
      reinterpret_cast<int64_t*>(a.ws + (size_t)a.c.n_units * NR * a.n_splits * 130)[0] = n.q_tokens;
    fp_body<NR>(a, n, *reinterpret_cast<FpSmem*>(smem_raw));
  } else {
    tcq_body<NR>(a, counts_of(a), &tmap, *reinterpret_cast<TcqSmem*>(smem_raw));
  }
}

template <int NR>
static cudaError_t launch_tcq_t(const AttnArgs& a, cudaStream_t st) {
  CUtensorMap tmap;
  cudaError_t te = record_tensor_map(a.c, RecTma<32>::kBoxRows, RecTma<32>::kRows, &tmap);
  if (te != cudaSuccess) return te;
  const size_t smem = sizeof(TcqSmem) > sizeof(FpSmem) ? sizeof(TcqSmem) : sizeof(FpSmem);
  cudaError_t e = cudaFuncSetAttribute(attend_tcq_kernel<NR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  attend_tcq_kernel<NR><<<dim3(a.c.n_units, a.n_splits), tcq::kThreads, smem, st>>>(a, tmap);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_combine_tc128(a, NR, st);
}

cudaError_t launch_tcq(const AttnArgs& a, int n_rep, cudaStream_t st) {
  if (n_rep == 1) return launch_tcq_t<1>(a, st);
  if (n_rep == 2) return launch_tcq_t<2>(a, st);
  if (n_rep == 4) return launch_tcq_t<4>(a, st);
  if (n_rep == 8) return launch_tcq_t<8>(a, st);
  return cudaErrorInvalidValue;
}

}  // namespace ott
