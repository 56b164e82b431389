// ott_common.cuh — shared device helpers and layout math for the OTT kernels.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ott_b200.h"

namespace ott {

constexpr int kMaxD = 128;
constexpr int kMaxG = 128;
constexpr int kMaxN = 128;  // pool capacity supported by the flush kernel
constexpr int kMaxA = 1024;

// Block record layout (see ott_b200.h). All offsets in bytes.
struct RecordLayout {
  int d, G;
  __host__ __device__ RecordLayout(int d_, int G_) : d(d_), G(G_) {}
  __host__ __device__ int code_bytes() const { return G * d / 4; }  // 2-bit codes
  __host__ __device__ int k_codes() const { return 0; }
  __host__ __device__ int v_codes() const { return code_bytes(); }
  __host__ __device__ int k_step() const { return 2 * code_bytes(); }
  __host__ __device__ int k_xmin() const { return k_step() + 4 * d; }
  __host__ __device__ int v_step() const { return k_xmin() + 4 * d; }
  __host__ __device__ int v_xmin() const { return v_step() + 4 * G; }
  __host__ __device__ int bytes() const { return v_xmin() + 4 * G; }
};

__host__ __device__ inline size_t mask_words_per_unit(const ott_cache_t& c) {
  return (size_t)c.max_groups * c.group_size / 32;
}

__host__ __device__ inline uint8_t* record_ptr(const ott_cache_t& c, int unit, int64_t group) {
  const RecordLayout L(c.head_dim, c.group_size);
  return c.blocks + ((size_t)unit * c.max_groups + (size_t)group) * L.bytes();
}

__device__ __forceinline__ float h2f(uint16_t h) { return __half2float(__ushort_as_half(h)); }
__device__ __forceinline__ uint16_t f2h(float f) { return __half_as_ushort(__float2half_rn(f)); }

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
