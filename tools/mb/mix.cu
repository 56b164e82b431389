// Ideal (dependency-light) throughput of K2's per-group instruction mix on one SM sub-partition:
// per iteration H HMMA (4 accumulators), L LOP3, F HFMA2, S FFMA (8 independent chains each).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int H, int L, int F, int S>
__global__ void k(int iters, uint32_t seed, float* out, long long* cyc) {
  float c[4][4] = {};
  uint32_t a = seed ^ threadIdx.x, b = seed * 3u;
  uint32_t x[8], h[8];
  float f[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    x[i] = seed + i * 77 + threadIdx.x;
    h[i] = 0x3c003c00u + i;
    f[i] = (float)(threadIdx.x + i);
  }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < (H > L ? H : L); ++i) {
      if (i < H)
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
            : "+f"(c[i & 3][0]), "+f"(c[i & 3][1]), "+f"(c[i & 3][2]), "+f"(c[i & 3][3])
            : "r"(a), "r"(a ^ 1u), "r"(a ^ 2u), "r"(a ^ 3u), "r"(b), "r"(b ^ 5u));
#pragma unroll
      for (int j = 0; j < (L + H - 1) / (H > 0 ? H : 1) && (H > 0); ++j)
        if (i * ((L + H - 1) / H) + j < L) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;\n" : "+r"(x[(i * 3 + j) & 7]) : "r"(x[(i * 3 + j + 3) & 7]), "r"(a));
#pragma unroll
      for (int j = 0; j < (F + H - 1) / (H > 0 ? H : 1) && (H > 0); ++j)
        if (i * ((F + H - 1) / H) + j < F) asm volatile("fma.rn.f16x2 %0, %0, %1, %2;\n" : "+r"(h[(i * 3 + j) & 7]) : "r"(h[(i * 3 + j + 3) & 7]), "r"(b));
#pragma unroll
      for (int j = 0; j < (S + H - 1) / (H > 0 ? H : 1) && (H > 0); ++j)
        if (i * ((S + H - 1) / H) + j < S) asm volatile("fma.rn.f32 %0, %0, %1, %1;\n" : "+f"(f[(i * 3 + j) & 7]) : "f"(1.0001f));
    }
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t s = 0;
  float fs = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) { s ^= x[i] ^ h[i]; fs += f[i]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = c[0][0] + c[1][1] + c[2][2] + c[3][3] + (float)(s & 1) + fs;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

template <int H, int L, int F, int S>
void run(const char* name, int w = 4, int iters = 1024) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 8);
  k<H, L, F, S><<<148, 128 * w>>>(iters, 0x3c003c00u, out, cyc);
  k<H, L, F, S><<<148, 128 * w>>>(iters, 0x3c003c00u, out, cyc);
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-28s H=%2d L=%3d F=%2d S=%2d x%d warps/SMSP: %7.1f cyc/iter/SMSP\n", name, H, L, F, S, w, (double)c / iters);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<12, 0, 0, 0>("hmma only");
  run<12, 33, 0, 0>("hmma+lop3");
  run<12, 0, 12, 0>("hmma+hfma2");
  run<12, 0, 0, 8>("hmma+ffma");
  run<12, 33, 12, 8>("k2 mix / 4");
  run<12, 45, 12, 16>("k2 mix+ / 4");
  run<1, 33, 0, 0>("lop3 only (1 hmma)");
  run<1, 0, 32, 0>("hfma2 only (1 hmma)");
  run<1, 0, 0, 32>("ffma only (1 hmma)");
  run<1, 32, 32, 0>("lop3+hfma2 (1 hmma)");
  run<1, 32, 0, 32>("lop3+ffma (1 hmma)");
  return 0;
}
