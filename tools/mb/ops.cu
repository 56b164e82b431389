// Dispatch cost of single instruction classes on one B200 SM sub-partition (4 warps per SMSP,
// 8 independent chains per warp): cycles per warp-instruction.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define OPS 64
template <int KIND>
__global__ void k(int iters, uint32_t seed, uint32_t* out, long long* cyc) {
  uint32_t x[8];
  float f[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    x[i] = seed + i * 77 + threadIdx.x;
    f[i] = 0.001f * (float)(threadIdx.x + i);
  }
  const uint32_t seed4 = seed | 0x400000u;
  const unsigned short h4 = (unsigned short)(seed >> 20);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int n = 0; n < OPS; ++n) {
      uint32_t& r = x[n & 7];
      const uint32_t o = x[(n + 3) & 7];
      float& g = f[n & 7];
      if (KIND == 0) asm volatile("lop3.b32 %0, %0, %1, 0x00ff00ff, 0x6a;\n" : "+r"(r) : "r"(o));
      if (KIND == 1) asm volatile("shr.b32 %0, %0, 10;\n" : "+r"(r));
      if (KIND == 2) asm volatile("mul.hi.u32 %0, %0, %1;\n" : "+r"(r) : "r"(seed4));
      if (KIND == 3) asm volatile("mad.lo.u32 %0, %0, %1, %1;\n" : "+r"(r) : "r"(o));
      if (KIND == 4) asm volatile("prmt.b32 %0, %0, %1, 0x5410;\n" : "+r"(r) : "r"(o));
      if (KIND == 5) asm volatile("ex2.approx.ftz.f32 %0, %0;\n" : "+f"(g));
      if (KIND == 6) asm volatile("max.f32 %0, %0, %1;\n" : "+f"(g) : "f"(f[(n + 3) & 7]));
      if (KIND == 7) asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;\n" : "=r"(r) : "f"(g), "f"(f[(n + 3) & 7]));
      if (KIND == 8) asm volatile("add.u32 %0, %0, %1;\n" : "+r"(r) : "r"(o));
      if (KIND == 9) asm volatile("fma.rn.f32 %0, %0, %1, %1;\n" : "+f"(g) : "f"(f[(n + 3) & 7]));
      if (KIND == 10) asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %0;\n" : "+r"(r));
      if (KIND == 11) asm volatile("shf.r.clamp.b32 %0, %0, %1, 10;\n" : "+r"(r) : "r"(o));
      if (KIND == 12) asm volatile("and.b32 %0, %0, %1;\n" : "+r"(r) : "r"(o));
      if (KIND == 13) asm volatile("mul.rn.f16x2 %0, %0, %1;\n" : "+r"(r) : "r"(o));
      if (KIND == 14) asm volatile("add.rn.f32 %0, %0, %1;\n" : "+f"(g) : "f"(f[(n + 3) & 7]));
      if (KIND == 15) asm volatile("mul.wide.u16 %0, %1, %2;\n" : "=r"(r) : "h"((unsigned short)r), "h"(h4));
    }
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= x[i] ^ __float_as_uint(f[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

template <int KIND>
void run(const char* name, int iters = 512) {
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 8);
  k<KIND><<<148, 512>>>(iters, 0x3c003c00u, out, cyc);
  k<KIND><<<148, 512>>>(iters, 0x3c003c00u, out, cyc);
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-24s %.2f cycles per warp-instruction per SMSP\n", name, (double)c / iters / (OPS * 4));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<0>("LOP3");
  run<12>("AND (lop3)");
  run<1>("SHR (shf)");
  run<11>("SHF.R imm");
  run<2>("IMAD.HI (mul.hi)");
  run<3>("IMAD (mad.lo)");
  run<15>("mul.wide.u16");
  run<8>("IADD (add.u32)");
  run<4>("PRMT");
  run<5>("MUFU.EX2");
  run<6>("FMNMX");
  run<7>("F2FP pack f16x2");
  run<9>("FFMA");
  run<14>("FADD");
  run<13>("HMUL2");
  run<10>("MOVM");
  return 0;
}
