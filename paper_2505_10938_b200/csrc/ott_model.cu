// ott_model.cu — fused elementwise kernels for the config-1 decoder's decode step
// (model.py): RMSNorm, RoPE + q/k/v split, SiLU-gate. One launch each instead of
// ~8-15 torch elementwise kernels, so the CUDA-graph-captured decode step is
// dominated by its GEMMs and the OTT cache kernels. fp16 in/out, fp32 math.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ float h2f(uint16_t h) { return __half2float(__ushort_as_half(h)); }
__device__ __forceinline__ uint16_t f2h(float f) { return __half_as_ushort(__float2half_rn(f)); }

// y[r] = fp16(x[r] * rsqrt(mean(x[r]^2) + eps)) * w   (one CTA per row). The row stays in
// registers between the reduction and the scaling (up to kChunks 16-byte chunks per thread,
// dim <= 8 * kChunks * blockDim), and the weights are loaded before the reduction, so the
// kernel is one global round trip plus the block reduction (the decode step runs it with
// only B rows, so its latency is what counts).
constexpr int kNormChunks = 4;
__global__ void rmsnorm_kernel(const uint16_t* __restrict__ x, const uint16_t* __restrict__ w,
                               uint16_t* __restrict__ y, int dim, float eps) {
  const uint16_t* xr = x + (size_t)blockIdx.x * dim;
  uint16_t* yr = y + (size_t)blockIdx.x * dim;
  uint4 xv[kNormChunks], wv[kNormChunks];
  float ss = 0.f;
#pragma unroll
  for (int c = 0; c < kNormChunks; ++c) {
    const int i = (c * blockDim.x + threadIdx.x) * 8;
    if (i < dim) {
      xv[c] = *reinterpret_cast<const uint4*>(xr + i);
      wv[c] = *reinterpret_cast<const uint4*>(w + i);
    }
  }
#pragma unroll
  for (int c = 0; c < kNormChunks; ++c) {
    if ((c * blockDim.x + threadIdx.x) * 8 < dim) {
      const uint32_t u[4] = {xv[c].x, xv[c].y, xv[c].z, xv[c].w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&u[k]));
        ss = fmaf(f.x, f.x, fmaf(f.y, f.y, ss));
      }
    }
  }
  __shared__ float red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float t = (threadIdx.x & 31) < (blockDim.x >> 5) ? red[threadIdx.x & 31] : 0.f;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);  // every warp reduces the partials
  const float r = rsqrtf(t / (float)dim + eps);
#pragma unroll
  for (int c = 0; c < kNormChunks; ++c) {
    const int i = (c * blockDim.x + threadIdx.x) * 8;
    if (i < dim) {
      const uint32_t u[4] = {xv[c].x, xv[c].y, xv[c].z, xv[c].w}, gw[4] = {wv[c].x, wv[c].y, wv[c].z, wv[c].w};
      uint32_t o[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&u[k]));
        const __half2 n = __floats2half2_rn(f.x * r, f.y * r);
        const __half2 m = __hmul2(n, *reinterpret_cast<const __half2*>(&gw[k]));
        o[k] = *reinterpret_cast<const uint32_t*>(&m);
      }
      *reinterpret_cast<uint4*>(yr + i) = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
}

// qkv [B][(H + 2 Hkv) d] -> q [B][H][d], k [B][Hkv][d] rotated at position p
// (rotate-half RoPE with fp32 cos/sin tables [max_pos][d]), v [B][Hkv][d] copied.
__global__ void rope_qkv_kernel(const uint16_t* __restrict__ qkv, const float* __restrict__ cosT,
                                const float* __restrict__ sinT, const int64_t* __restrict__ pos_dev,
                                int64_t pos_host, uint16_t* __restrict__ q, uint16_t* __restrict__ k,
                                uint16_t* __restrict__ v, int H, int Hkv, int d) {
  const int b = blockIdx.y, head = blockIdx.x;  // head in [0, H + 2 Hkv)
  const int64_t p = pos_dev ? *pos_dev : pos_host;
  const uint16_t* src = qkv + ((size_t)b * (H + 2 * Hkv) + head) * d;
  const int half = d / 2;
  if (head >= H + Hkv) {  // v
    uint16_t* dst = v + ((size_t)b * Hkv + (head - H - Hkv)) * d;
    for (int i = threadIdx.x; i < d; i += blockDim.x) dst[i] = src[i];
    return;
  }
  uint16_t* dst = head < H ? q + ((size_t)b * H + head) * d : k + ((size_t)b * Hkv + (head - H)) * d;
  const float* c = cosT + (size_t)p * d;
  const float* s = sinT + (size_t)p * d;
  for (int i = threadIdx.x; i < half; i += blockDim.x) {  // the pair (i, i + half) per thread
    const float x0 = h2f(src[i]), x1 = h2f(src[i + half]);
    dst[i] = f2h(x0 * c[i] - x1 * s[i]);
    dst[i + half] = f2h(x1 * c[i + half] + x0 * s[i + half]);
  }
}

// out [rows][n] = fp16(silu(a) * b) with h [rows][2n] = (a | b)
__global__ void silu_mul_kernel(const uint16_t* __restrict__ h, uint16_t* __restrict__ out, int n) {
  const size_t row = blockIdx.y;
  const uint16_t* a = h + row * 2 * n;
  const uint16_t* bb = a + n;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) * 2; i < n; i += gridDim.x * blockDim.x * 2) {
    const float2 x = __half22float2(*reinterpret_cast<const __half2*>(a + i));
    const float2 y = __half22float2(*reinterpret_cast<const __half2*>(bb + i));
    const float s0 = x.x / (1.f + __expf(-x.x)), s1 = x.y / (1.f + __expf(-x.y));
    const __half2 r = __floats2half2_rn(s0 * y.x, s1 * y.y);
    *reinterpret_cast<__half2*>(out + row * n + i) = r;
  }
}

}  // namespace

extern "C" {

int ott_model_rmsnorm(const uint16_t* x, const uint16_t* w, uint16_t* y, int32_t rows, int32_t dim, float eps,
                      void* stream) {
  if (!x || !w || !y || rows < 1 || dim < 8 || dim % 8 || dim > 8 * kNormChunks * 1024) return 1;
  // one 16-byte chunk per thread where possible (dim / 8 threads, whole warps, <= 1024)
  int threads = (dim / 8 + 31) / 32 * 32;
  while (threads > 1024) threads = (threads / 2 + 31) / 32 * 32;
  rmsnorm_kernel<<<rows, threads, 0, (cudaStream_t)stream>>>(x, w, y, dim, eps);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

int ott_model_rope_qkv(const uint16_t* qkv, const float* cos_t, const float* sin_t, const int64_t* pos_dev,
                       int64_t pos_host, uint16_t* q, uint16_t* k, uint16_t* v, int32_t batch, int32_t n_heads,
                       int32_t n_kv_heads, int32_t head_dim, void* stream) {
  if (!qkv || !cos_t || !sin_t || !q || !k || !v || batch < 1 || head_dim % 2) return 1;
  dim3 grid(n_heads + 2 * n_kv_heads, batch);
  rope_qkv_kernel<<<grid, 64, 0, (cudaStream_t)stream>>>(qkv, cos_t, sin_t, pos_dev, pos_host, q, k, v, n_heads,
                                                         n_kv_heads, head_dim);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

int ott_model_silu_mul(const uint16_t* h, uint16_t* out, int32_t rows, int32_t n, void* stream) {
  if (!h || !out || rows < 1 || n % 2) return 1;
  const int blocks = (n / 2 + 255) / 256 < 16 ? (n / 2 + 255) / 256 : 16;
  silu_mul_kernel<<<dim3(blocks, rows), 256, 0, (cudaStream_t)stream>>>(h, out, n);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

}  // extern "C"
