// Does legacy mma.sync (HMMA.16816.F32) overlap with independent ALU work on B200?
// Per iteration: H independent HMMA (2 chains) + N independent LOP3 (8 chains); W warps per SM
// sub-partition (CTA = 4 W warps, one CTA per SM, 148 CTAs). Prints SM cycles per iteration per
// sub-partition: additive (H*cost + N) vs overlapped (max).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int H, int N>
__global__ void k(int iters, uint32_t seed, float* out, long long* cyc) {
  float c0[4] = {0, 0, 0, 0}, c1[4] = {0, 0, 0, 0};
  uint32_t a = seed ^ threadIdx.x, b = seed * 3u;
  uint32_t x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = seed + i * 77 + threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int h = 0; h < H; ++h) {
      float* c = (h & 1) ? c1 : c0;
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
          : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
          : "r"(a), "r"(a ^ 1u), "r"(a ^ 2u), "r"(a ^ 3u), "r"(b), "r"(b ^ 5u));
    }
#pragma unroll
    for (int n = 0; n < N; ++n) asm volatile("lop3.b32 %0, %0, %1, %2, 0x6a;\n" : "+r"(x[n & 7]) : "r"(a), "r"(b));
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = c0[0] + c0[1] + c1[2] + c1[3] + (float)(s & 1);
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

template <int H, int N>
void run(int w, int iters = 2048) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 8);
  k<H, N><<<148, 128 * w>>>(iters, 0x3c003c00u, out, cyc);
  k<H, N><<<148, 128 * w>>>(iters, 0x3c003c00u, out, cyc);
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double per = (double)c / iters;  // cycles per iteration (all W warps of a sub-partition)
  printf("HMMA=%d LOP3=%2d warps/SMSP=%d: %7.1f cyc/iter/SMSP  (%.2f cyc per HMMA, %.2f issue-slots of LOP3)\n", H, N,
         w, per, H ? per / (H * w) : 0.0, (double)N * w);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {1, 4}) {
    run<4, 0>(w);
    run<4, 8>(w);
    run<4, 16>(w);
    run<4, 32>(w);
    run<4, 64>(w);
    run<0, 32>(w);
  }
  return 0;
}
