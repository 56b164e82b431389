// ott_common.cuh — shared device helpers and layout math for the OTT kernels.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ott_b200.h"

namespace ott {

constexpr int kMaxD = 256;  // generic kernels; the tensor-core kernels take d = 128
constexpr int kMaxG = 128;
constexpr int kMaxN = 128;  // pool capacity supported by the flush kernel
constexpr int kMaxA = 1024;

// Code width stored in the record. At the tensor-core shapes the widths without a kernel of
// their own are stored in the next wider container (levels stay 2^bits - 1): 1-bit codes as
// 2-bit fields, 3-bit as 4-bit and 5..7-bit as 8-bit (d = 128, G in {32, 64, 128}), so they
// decode on the 2-, 4- and 8-bit tensor-core attention kernels.
__host__ __device__ constexpr int code_bits(int bits, int d, int G) {
  return (d != 128 || (G != 32 && G != 64 && G != 128)) ? bits
         : bits == 1                                     ? 2
         : bits == 3                                     ? 4
         : (bits >= 5 && bits <= 7)                      ? 8
                                                         : bits;
}

// Block record layout (see ott_b200.h). All offsets in bytes. `bits` is the stored code
// width (code_bits of the cache's bits).
//   width 2:      K codes | V codes | K sh[d] | K sl[d] | V step[G] | V x_min[G] | K e hi[d] | K e lo[d]
//   other widths: K codes | V codes | K sh[d] | K sl[d] | K e[d] (f32) | V step[G] | V x_min[G]
// At width 2 the K x_min term comes last so the decode kernels can stream a record's head
// (head_bytes) and fetch the e fields of 8 groups at once (batched bias, ott_attend.cu).
struct RecordLayout {
  int d, G, bits;
  __host__ __device__ RecordLayout(int d_, int G_, int bits_ = 2) : d(d_), G(G_), bits(code_bits(bits_, d_, G_)) {}
  // packed codes: ceil(G d bits / 8) bytes (quant.py:237-238), padded to 16 so every
  // field stays aligned (no padding at the tensor-core shapes d in {64, 128}, G % 32 == 0)
  __host__ __device__ int code_bytes() const { return ((G * d * bits + 7) / 8 + 15) & ~15; }
  __host__ __device__ int k_codes() const { return 0; }
  __host__ __device__ int v_codes() const { return code_bytes(); }
  __host__ __device__ int k_sh() const { return 2 * code_bytes(); }  // fp16 [d], pair order
  __host__ __device__ int k_sl() const { return k_sh() + 2 * d; }     // fp16 [d], pair order
  __host__ __device__ int v_step() const { return bits == 2 ? k_sl() + 2 * d : k_sl() + 6 * d; }
  __host__ __device__ int v_xmin() const { return v_step() + 4 * G; }
  // width 2: fp16 hi [d] then lo [d] (pair order) of e / u; other widths: f32 [d], channel order
  __host__ __device__ int k_e() const { return bits == 2 ? v_xmin() + 4 * G : k_sl() + 2 * d; }
  __host__ __device__ int head_bytes() const { return bits == 2 ? k_e() : bytes(); }  // before the e fields
  __host__ __device__ int bytes() const { return (v_step() + 8 * G + (bits == 2 ? 4 * d : 0) + 15) & ~15; }
};

constexpr float kEScale = 8.f;  // width-2 K e fields hold e / (kEScale u), see store_k_e2

// ---- K parameter encoding (tensor-core friendly; exact values live in params64).
// A 32-bit code word holds 16 channels of one token; the decode kernels extract
// code pairs (channel m, m+8) of a word in place at fp16 mantissa position P(m)
// (see ott_attend.cu), so the per-channel K step is stored split into two fp16
// values sh + sl (sh = fp16_rn(step64), sl = fp16_rn(step64 - sh)) in "pair
// order" (index 16*(c/16) + 2*(c%8) + (c%16)/8), and x_min is stored folded with
// that position scale: e = f32_rn(x_min64 - 4 * u(c) * step64), u(c) = 4^(4-P(c%8)).
// Dequantisation of channel c: k = code * step + x_min = code * step + e + 4 u step.
__host__ __device__ constexpr int kpair_pos(int m) { return m == 2 || m == 5 ? 2 : (m == 0 || m == 3 || m == 6 ? 3 : 4); }
__host__ __device__ constexpr float kpair_u(int m) { return kpair_pos(m) == 2 ? 16.f : (kpair_pos(m) == 3 ? 4.f : 1.f); }
// (pair order only when d % 16 == 0, where the tensor-core kernels read it; identity otherwise)
__host__ __device__ constexpr int kpair_index(int c, int d) {
  return d % 16 ? c : 16 * (c / 16) + 2 * (c % 8) + (c % 16) / 8;
}

__host__ __device__ inline size_t mask_words_per_unit(const ott_cache_t& c) {
  return ((size_t)c.max_groups * c.group_size + 31) / 32;  // one bit per quantized position
}

__host__ __device__ inline uint8_t* record_ptr(const ott_cache_t& c, int unit, int64_t group) {
  const RecordLayout L(c.head_dim, c.group_size, c.bits);
  return c.blocks + ((size_t)unit * c.max_groups + (size_t)group) * L.bytes();
}

__device__ __forceinline__ float h2f(uint16_t h) { return __half2float(__ushort_as_half(h)); }
// code of element e of a pack_codes stream (quant.py:241-256: element e at bits
// [e*bits, e*bits + bits), LSB first); a code spans at most two bytes for bits <= 8
__device__ __forceinline__ uint32_t code_at(const uint8_t* codes, int64_t e, int bits) {
  const int64_t b0 = e * bits;
  const uint32_t lo = codes[b0 >> 3];
  const uint32_t hi = ((b0 & 7) + bits > 8) ? codes[(b0 >> 3) + 1] : 0u;
  return ((lo | (hi << 8)) >> (b0 & 7)) & ((1u << bits) - 1u);
}
// 4-bit tensor-core encoding: a code word holds channels 8w..8w+7 (nibbles, LSB first); the
// unpack yields half2 pairs (8w+k, 8w+k+4), k = 0..3, every nibble at fp16 mantissa bits 4-7
// (value 1 + c/64, u = 64). K steps are stored in that pair order, e = x_min - 64 step.
__host__ __device__ constexpr int kpair4_index(int c) { return 8 * (c / 8) + 2 * (c % 4) + (c % 8) / 4; }
__host__ __device__ constexpr bool k_tc4(int bits, int d) { return bits == 4 && d % 8 == 0; }
// 8-bit tensor-core encoding: a byte per code; the unpack pairs consecutive channels
// (c, c+1) as fp16 1024 + code, so steps are stored in channel order and e = x_min - 1024 step.
__host__ __device__ constexpr bool k_tc8(int bits, int d) { return bits == 8 && d % 8 == 0; }

// float32 K step / x_min of channel c from the record. 2-bit and 4-bit records hold the
// tensor-core encodings (sh + sl halves in pair order, e = x_min - 4 u step resp. x_min - 64 step);
// other widths, whose steps can exceed the fp16 range (1 bit: up to 2 * 65504), hold float32
// step[d] in the sh/sl bytes and x_min in e.
__device__ __forceinline__ float k_step_of(const uint8_t* rec, const RecordLayout& L, int c) {
  if (L.bits != 2 && !k_tc4(L.bits, L.d) && !k_tc8(L.bits, L.d)) return reinterpret_cast<const float*>(rec + L.k_sh())[c];
  const int j = L.bits == 2 ? kpair_index(c, L.d) : (L.bits == 4 ? kpair4_index(c) : c);
  return h2f(reinterpret_cast<const uint16_t*>(rec + L.k_sh())[j]) + h2f(reinterpret_cast<const uint16_t*>(rec + L.k_sl())[j]);
}
__device__ __forceinline__ float k_xmin_of(const uint8_t* rec, const RecordLayout& L, int c, float step) {
  if (L.bits == 2) {  // e / (8 u) as fp16 hi + lo in pair order
    const int j = kpair_index(c, L.d);
    const uint16_t* eh = reinterpret_cast<const uint16_t*>(rec + L.k_e());
    const float u = kpair_u(c % 8);
    return fmaf(4.f * u, step, (h2f(eh[j]) + h2f(eh[L.d + j])) * (kEScale * u));
  }
  const float e = reinterpret_cast<const float*>(rec + L.k_e())[c];
  if (k_tc4(L.bits, L.d)) return fmaf(64.f, step, e);
  if (k_tc8(L.bits, L.d)) return fmaf(1024.f, step, e);
  return e;
}
__device__ __forceinline__ uint16_t f2h(float f) { return __half_as_ushort(__float2half_rn(f)); }
// Width-2 K x_min term of channel c: e = f32(x_min - 4 u step) (computed by the caller in
// float64), stored as t = e / (8 u) (exact) split into fp16 hi = fp16(t), lo = fp16(t - hi) in
// pair order: the decode kernels multiply it by q u (their Q K^T B operand) on tensor cores.
// |t| <= (65504 + 4 * 65504) / 8 for any fp16 input (1-bit steps included), so t never
// overflows fp16.
__device__ __forceinline__ void store_k_e2(uint8_t* rec, const RecordLayout& L, int c, float e) {
  const float t = e * (1.f / (kEScale * kpair_u(c % 8)));  // 8 u is a power of two: the same value as e / (8 u)
  const __half hi = __float2half_rn(t);
  const __half lo = __float2half_rn(t - __half2float(hi));
  uint16_t* eh = reinterpret_cast<uint16_t*>(rec + L.k_e());
  const int j = kpair_index(c, L.d);
  eh[j] = __half_as_ushort(hi);
  eh[L.d + j] = __half_as_ushort(lo);
}

// Largest K or V step of a unit's 2-bit groups (pool_meta[u][3], float bits, atomic max):
// the tensor-core attention scales its fp16 operands (q u step, 4 p v_step) by powers of two
// when this bound and |q| would overflow them (see step_scales in ott_attend.cu).
__device__ __forceinline__ void note_step_max(int32_t* meta3, float step) {  // whole warp
  float m = step;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(meta3, __float_as_int(m));
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_min_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace ott
