// Overlap of two instruction classes on one B200 SM sub-partition (4 warps per SMSP): per
// iteration NA ops of class A interleaved with NB ops of class B (independent chains).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int K>
__device__ __forceinline__ void op(uint32_t& r, float& g, uint32_t o, float fo, float* c) {
  if (K == 0) asm volatile("lop3.b32 %0, %0, %1, 0x00ff00ff, 0x6a;\n" : "+r"(r) : "r"(o));
  if (K == 1) asm volatile("ex2.approx.ftz.f32 %0, %0;\n" : "+f"(g));
  if (K == 2) asm volatile("fma.rn.f32 %0, %0, %1, %1;\n" : "+f"(g) : "f"(fo));
  if (K == 3) asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %0;\n" : "+r"(r));
  if (K == 4)
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(o), "r"(o ^ 1u), "r"(o ^ 2u), "r"(o ^ 3u), "r"(o), "r"(o));
  if (K == 5) asm volatile("fma.rn.f16x2 %0, %0, %1, %1;\n" : "+r"(r) : "r"(o));
  if (K == 6) asm volatile("mad.lo.u32 %0, %0, %1, %1;\n" : "+r"(r) : "r"(o));
  if (K == 7)
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.f32.e4m3.e4m3.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(o), "r"(o ^ 1u), "r"(o ^ 2u), "r"(o ^ 3u), "r"(o), "r"(o));
  if (K == 8) {
    uint16_t t;
    asm volatile("cvt.rn.satfinite.e4m3x2.f16x2 %0, %1;\n" : "=h"(t) : "r"(r ^ o));
    r = r + t;
  }
}

template <int KA, int NA, int KB, int NB>
__global__ void k(int iters, uint32_t seed, uint32_t* out, long long* cyc) {
  uint32_t x[8], y[8];
  float f[8], h[8], c[4][4] = {};
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    x[i] = seed + i * 77 + threadIdx.x;
    y[i] = seed * 5 + i * 31 + threadIdx.x;
    f[i] = 0.001f * (float)(threadIdx.x + i);
    h[i] = -0.002f * (float)(threadIdx.x + i);
  }
  const uint32_t cst = seed | 0x11u;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    constexpr int N = NA > NB ? NA : NB;
#pragma unroll
    for (int n = 0; n < N; ++n) {
      if (n < NA) op<KA>(x[n & 7], f[n & 7], (KA == 4 || KA == 7) ? cst : x[(n + 3) & 7], 1.0001f, c[n & 3]);
      if (n < NB) op<KB>(y[n & 7], h[n & 7], (KB == 4 || KB == 7) ? cst : y[(n + 3) & 7], 0.9999f, c[(n + 2) & 3]);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= x[i] ^ y[i] ^ __float_as_uint(f[i] + h[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + (uint32_t)(c[0][0] + c[1][1] + c[2][2] + c[3][3]);
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

const char* nm[] = {"LOP3", "MUFU.EX2", "FFMA", "MOVM", "HMMA", "HFMA2", "IMAD", "QMMA", "CVT.E4M3"};
template <int KA, int NA, int KB, int NB>
void run(int iters = 512) {
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 8);
  k<KA, NA, KB, NB><<<148, 512>>>(iters, 0x3c003c00u, out, cyc);
  k<KA, NA, KB, NB><<<148, 512>>>(iters, 0x3c003c00u, out, cyc);
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%2d x %-9s + %2d x %-9s: %7.1f cycles per iteration per SMSP (4 warps)\n", NA, nm[KA], NB, nm[KB],
         (double)c / iters);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<7, 8, 0, 0>();
  run<4, 8, 0, 0>();
  run<7, 8, 2, 32>();
  run<7, 8, 0, 32>();
  run<7, 8, 4, 8>();
  run<8, 32, 0, 0>();
  run<8, 32, 2, 32>();
  run<8, 32, 0, 32>();
  return 0;
}
