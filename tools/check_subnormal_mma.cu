// Checks that mma.sync m16n8k16 f16 honours fp16 subnormal A inputs (no FTZ):
// A = c * 2^-16 encoded as raw bits (c << 8), B = 1.0 -> D = sum_k c * 2^-16.
#include <cstdio>
#include <cstdint>
__global__ void k(float* out) {
  const int lane = threadIdx.x;
  uint32_t a = (3u << 8) | (3u << 24);  // two halves, each 3 * 2^-16 (subnormal)
  uint32_t b = 0x3C003C00u;             // 1.0, 1.0
  float c[4] = {0, 0, 0, 0};
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a), "r"(a), "r"(a), "r"(a), "r"(b), "r"(b));
  out[lane] = c[0];
}
int main() {
  float* d; cudaMalloc(&d, 128);
  k<<<1, 32>>>(d);
  float h[32]; cudaMemcpy(h, d, 128, cudaMemcpyDeviceToHost);
  const double want = 16 * 3.0 / 65536.0;
  printf("subnormal mma: got %.9g want %.9g -> %s\n", h[0], want, h[0] == (float)want ? "OK" : "FTZ/MISMATCH");
  return h[0] == (float)want ? 0 : 1;
}
