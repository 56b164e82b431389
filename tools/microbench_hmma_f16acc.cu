// Throughput of legacy mma.sync m16n8k16 with f32 vs f16 accumulators on B200.
#include <cstdio>
#include <cstdint>
template <int CH, bool F16>
__global__ void k(float* out, int iters) {
  uint32_t a0 = threadIdx.x * 0x00010001u, a1 = a0 ^ 0x3c003c00u, a2 = a0 + 7, a3 = a1 + 3;
  uint32_t b0 = 0x3c003c00u, b1 = 0x3c003c00u ^ threadIdx.x;
  float c[CH][4];
  uint32_t h[CH][2];
  for (int i = 0; i < CH; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.f; h[i][0] = h[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      if (F16)
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f16.f16.f16.f16 {%0,%1}, {%2,%3,%4,%5}, {%6,%7}, {%0,%1};"
                     : "+r"(h[i][0]), "+r"(h[i][1]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  float s = 0;
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3] + __uint_as_float(h[i][0]) + __uint_as_float(h[i][1]);
  if (s == 1234.5f) out[0] = s;
}
template <int CH, bool F16>
void run(const char* name, int sms) {
  float* o; cudaMalloc(&o, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096, warps = 8;
  k<CH, F16><<<sms * 4, 32 * warps>>>(o, 16);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  k<CH, F16><<<sms * 4, 32 * warps>>>(o, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double n = (double)iters * CH * sms * 4 * warps;
  printf("%s chains=%d: %.1f G HMMA/s (%.1f TFLOP/s)\n", name, CH, n / ms / 1e6, n * 4096 / ms / 1e9);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<1, false>("f32 acc", sms); run<4, false>("f32 acc", sms);
  run<1, true>("f16 acc", sms); run<4, true>("f16 acc", sms);
  return 0;
}
