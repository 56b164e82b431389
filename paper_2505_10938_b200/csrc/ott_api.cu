// ott_api.cu — kernels behind the reference's standalone API objects that are not on the
// decode hot path: attend_full_precision (attention.py:35-59) and the OutlierPool.update
// competition (outlier.py:84-117). The hot path runs the same competition inside the flush
// kernels (ott_flush.cu) and the mixed-tier attention in ott_attend.cu.
#include "ott_common.cuh"

namespace ott {

constexpr int kExactThreads = 256;

__device__ __forceinline__ double block_reduce_d(double v, double* red, bool is_max) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double t = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmax(v, t) : v + t;
  }
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double r = red[0];
  for (int i = 1; i < kExactThreads / 32; ++i) r = is_max ? fmax(r, red[i]) : r + red[i];
  return r;
}

// One CTA per problem. scores[i] = f32(sum_j k[i][j] q[j]) / f32(sqrt(d)) (attention.py:52);
// weights = f32(exp(s - max) / sum) in float64 (tensor.py:45-57); out = weights V (float32).
__global__ void __launch_bounds__(kExactThreads) attend_exact_kernel(const float* __restrict__ q,
                                                                     const float* __restrict__ keys,
                                                                     const float* __restrict__ values, int n, int d,
                                                                     float* out, float* weights, float* scores) {
  __shared__ double red[kExactThreads / 32];
  const size_t b = blockIdx.x;
  const float* qb = q + b * d;
  const float* kb = keys + b * (size_t)n * d;
  const float* vb = values + b * (size_t)n * d;
  float* sb = scores + b * (size_t)n;
  float* wb = weights + b * (size_t)n;
  const float sqrt_d = (float)sqrt((double)d);
  double mx = -INFINITY;
  for (int i = threadIdx.x; i < n; i += kExactThreads) {
    float s = 0.f;
    for (int j = 0; j < d; ++j) s = fmaf(kb[(size_t)i * d + j], qb[j], s);
    s = __fdiv_rn(s, sqrt_d);
    sb[i] = s;
    mx = fmax(mx, (double)s);
  }
  mx = block_reduce_d(mx, red, true);
  double sum = 0.0;
  for (int i = threadIdx.x; i < n; i += kExactThreads) sum += exp((double)sb[i] - mx);
  sum = block_reduce_d(sum, red, false);
  for (int i = threadIdx.x; i < n; i += kExactThreads) wb[i] = (float)(exp((double)sb[i] - mx) / sum);
  __syncthreads();
  for (int j = threadIdx.x; j < d; j += kExactThreads) {
    float acc = 0.f;
    for (int i = 0; i < n; ++i) acc = fmaf(wb[i], vb[(size_t)i * d + j], acc);
    out[b * d + j] = acc;
  }
}

// rank of item i = #{j : (s_j, p_j) < (s_i, p_i)} (outlier.py:52-54, 102-103)
__global__ void pool_rank_kernel(const double* __restrict__ s, const int64_t* __restrict__ p, int n,
                                 int32_t* __restrict__ rank) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double si = s[i];
    const int64_t pi = p[i];
    int r = 0;
    for (int j = 0; j < n; ++j) r += (s[j] < si || (s[j] == si && p[j] < pi)) ? 1 : 0;
    rank[i] = r;
  }
}

// row_l1_norm (tensor.py:38-42): sum of |x| over a row in float64, one warp per row
__global__ void score_rows_kernel(const float* __restrict__ rows, int n, int d, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (int r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); r < n; r += gridDim.x * (blockDim.x / 32)) {
    double s = 0.0;
    for (int j = lane; j < d; j += 32) s += fabs((double)rows[(size_t)r * d + j]);
    s = warp_sum(s);
    if (lane == 0) out[r] = s;
  }
}

cudaError_t launch_score_rows(const float* rows, int n, int d, double* out, cudaStream_t st) {
  score_rows_kernel<<<(n + 7) / 8, 256, 0, st>>>(rows, n, d, out);
  return cudaGetLastError();
}

cudaError_t launch_attend_exact(const float* q, const float* keys, const float* values, int n, int d, int n_q,
                                float* out, float* weights, float* scores, cudaStream_t st) {
  attend_exact_kernel<<<n_q, kExactThreads, 0, st>>>(q, keys, values, n, d, out, weights, scores);
  return cudaGetLastError();
}

cudaError_t launch_pool_rank(const double* s, const int64_t* p, int n, int32_t* rank, cudaStream_t st) {
  pool_rank_kernel<<<(n + 127) / 128, 128, 0, st>>>(s, p, n, rank);
  return cudaGetLastError();
}

}  // namespace ott
