// Throughput of legacy mma.sync m16n8k32 s8/e4m3 on B200 vs m16n8k16 f16.
#include <cstdio>
#include <cstdint>
template <int KIND>
__global__ void k(float* out, int iters) {
  uint32_t a0 = threadIdx.x * 0x01010101u, a1 = a0 ^ 0x3c3c3c3cu, a2 = a0 + 7, a3 = a1 + 3;
  uint32_t b0 = 0x01010101u, b1 = 0x02020202u ^ threadIdx.x;
  int ci[4][4] = {};
  float cf[4][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (KIND == 0)
        asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+r"(ci[i][0]), "+r"(ci[i][1]), "+r"(ci[i][2]), "+r"(ci[i][3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      else
        asm volatile("mma.sync.aligned.m16n8k32.row.col.f32.e4m3.e4m3.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(cf[i][0]), "+f"(cf[i][1]), "+f"(cf[i][2]), "+f"(cf[i][3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  float s = 0;
  for (int i = 0; i < 4; ++i) s += ci[i][0] + ci[i][1] + ci[i][2] + ci[i][3] + cf[i][0] + cf[i][1] + cf[i][2] + cf[i][3];
  if (s == 1234.5f) out[0] = s;
}
template <int KIND>
void run(const char* name, int sms) {
  float* o; cudaMalloc(&o, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096, warps = 8;
  k<KIND><<<sms * 4, 32 * warps>>>(o, 16);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  k<KIND><<<sms * 4, 32 * warps>>>(o, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double n = (double)iters * 4 * sms * 4 * warps;
  printf("%s: %.1f G MMA/s (%.1f TOP/s)\n", name, n / ms / 1e6, n * 8192 / ms / 1e9);
  printf("  err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("imma m16n8k32 s8", sms); run<1>("fp8 m16n8k32 e4m3", sms);
  return 0;
}
