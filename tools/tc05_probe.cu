// Feasibility probe for the tcgen05 Q K^T design (sm_100a):
//   A (M=128 token rows x K=128 fp16) written from registers into TMEM with
//   tcgen05.st 32x32b (one lane per thread), B (N=64 x K=128 fp16, K-major,
//   no-swizzle canonical layout) in shared memory, tcgen05.mma kind::f16 with A
//   from TMEM (the .ts form), fp32 D in TMEM, read back with tcgen05.ld.
// Checks the result against a host fp64 reference for three A encodings:
//   0: small integers, 1: 1 + c*2^(2P-10) (the decode kernel's K encoding),
//   2: fp16 subnormals c*2^-24 (V encoding candidate).
// Also times back-to-back M128 N64 K16 MMAs (throughput per SM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc05_probe tools/tc05_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <cuda_fp16.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int M = 128, N = 64, K = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// canonical K-major no-swizzle: core matrix (8 rows x 16 B) at (r/8)*SBO + (k/8)*LBO
constexpr uint32_t kLBO = 128, kSBO = (K / 8) * 128;
__host__ __device__ constexpr uint32_t b_off(int n, int k) { return (n / 8) * kSBO + (k / 8) * kLBO + (n % 8) * 16 + (k % 8) * 2; }

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((kLBO >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((kSBO >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (Blackwell)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}
__host__ __device__ constexpr uint32_t idesc(int m, int n) {
  return (1u << 4)                    // D f32
         | (0u << 7) | (0u << 10)     // A, B f16
         | (0u << 15) | (0u << 16)    // K-major both
         | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__global__ void probe(const uint16_t* A, const uint16_t* B, float* D, long long* cycles, int reps) {
  __shared__ alignas(128) uint8_t bs[N * K * 2];
  __shared__ alignas(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    *reinterpret_cast<uint16_t*>(bs + b_off(n, k)) = B[i];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tbase)), "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tbase;
  const uint32_t a_tm = tmem, d_tm = tmem + 64;
  // A row tid (lane tid): 64 columns of packed f16 pairs
  uint32_t r[64];
#pragma unroll
  for (int j = 0; j < 64; ++j) r[j] = (uint32_t)A[tid * K + 2 * j] | ((uint32_t)A[tid * K + 2 * j + 1] << 16);
  const uint32_t lane_addr = a_tm + ((uint32_t)(warp * 32) << 16);
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x64.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,"
      "%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63,%64};\n" ::"r"(lane_addr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]), "r"(r[32]), "r"(r[33]), "r"(r[34]), "r"(r[35]), "r"(r[36]),
      "r"(r[37]), "r"(r[38]), "r"(r[39]), "r"(r[40]), "r"(r[41]), "r"(r[42]), "r"(r[43]), "r"(r[44]), "r"(r[45]),
      "r"(r[46]), "r"(r[47]), "r"(r[48]), "r"(r[49]), "r"(r[50]), "r"(r[51]), "r"(r[52]), "r"(r[53]), "r"(r[54]),
      "r"(r[55]), "r"(r[56]), "r"(r[57]), "r"(r[58]), "r"(r[59]), "r"(r[60]), "r"(r[61]), "r"(r[62]), "r"(r[63]));
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  long long t0 = clock64();
  if (tid == 0) {
    const uint32_t id = idesc(M, N);
    const uint32_t b0 = smem_u32(bs);
    for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
      for (int s = 0; s < K / 16; ++s) {
        const uint64_t bd = sdesc(b0 + s * 2 * kLBO);
        const uint32_t acc = (s > 0) ? 1u : 0u;
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tm),
            "r"(a_tm + 8 * s), "l"(bd), "r"(id), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)));
  }
  __syncwarp();
  {
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done) : "r"(smem_u32(&bar)), "r"(0) : "memory");
  }
  long long t1 = clock64();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  uint32_t o[64];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,"
      "%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];\n"
      : "=r"(o[0]), "=r"(o[1]), "=r"(o[2]), "=r"(o[3]), "=r"(o[4]), "=r"(o[5]), "=r"(o[6]), "=r"(o[7]), "=r"(o[8]),
        "=r"(o[9]), "=r"(o[10]), "=r"(o[11]), "=r"(o[12]), "=r"(o[13]), "=r"(o[14]), "=r"(o[15]), "=r"(o[16]),
        "=r"(o[17]), "=r"(o[18]), "=r"(o[19]), "=r"(o[20]), "=r"(o[21]), "=r"(o[22]), "=r"(o[23]), "=r"(o[24]),
        "=r"(o[25]), "=r"(o[26]), "=r"(o[27]), "=r"(o[28]), "=r"(o[29]), "=r"(o[30]), "=r"(o[31]), "=r"(o[32]),
        "=r"(o[33]), "=r"(o[34]), "=r"(o[35]), "=r"(o[36]), "=r"(o[37]), "=r"(o[38]), "=r"(o[39]), "=r"(o[40]),
        "=r"(o[41]), "=r"(o[42]), "=r"(o[43]), "=r"(o[44]), "=r"(o[45]), "=r"(o[46]), "=r"(o[47]), "=r"(o[48]),
        "=r"(o[49]), "=r"(o[50]), "=r"(o[51]), "=r"(o[52]), "=r"(o[53]), "=r"(o[54]), "=r"(o[55]), "=r"(o[56]),
        "=r"(o[57]), "=r"(o[58]), "=r"(o[59]), "=r"(o[60]), "=r"(o[61]), "=r"(o[62]), "=r"(o[63])
      : "r"(d_tm + ((uint32_t)(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int j = 0; j < 64; ++j) D[tid * N + j] = __uint_as_float(o[j]);
  if (tid == 0) cycles[0] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(256));
}

// timing only: back-to-back MMAs into one accumulator, runtime shape and operand source
__global__ void timing(long long* cycles, uint32_t id, int reps, int ss) {
  __shared__ alignas(128) uint8_t bs[128 * K * 2];
  __shared__ alignas(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * K * 2 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(bs)[i] = 0x3C003C00u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tbase)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tbase;
  long long t0 = clock64();
  if (warp == 0) {  // warp-uniform issue loop; one elected lane issues each MMA
    const uint32_t b0 = smem_u32(bs);
    for (int rep = 0; rep < reps; ++rep) {
      const uint32_t dcol0 = tmem + 256;
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const uint64_t bd = sdesc(b0 + s * 2 * kLBO);
        const uint32_t acc = (ss & 2) ? (rep > 0 ? 1u : 0u) : ((s > 0) ? 1u : 0u);
        const uint32_t dcol = (ss & 2) ? dcol0 + (s & 3) * 64 : dcol0;
        if (ss & 1)
          asm volatile(
              "{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
              "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(dcol),
              "l"(bd), "l"(bd), "r"(id), "r"(acc));
        else
          asm volatile(
              "{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
              "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(dcol),
              "r"(tmem + 8 * s), "l"(bd), "r"(id), "r"(acc));
      }
    }
    asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(&bar)));
  }
  __syncwarp();
  {
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done) : "r"(smem_u32(&bar)), "r"(0) : "memory");
  }
  long long t1 = clock64();
  if (tid == 0) cycles[0] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(512));
}

// multi-CTA issue test: is MMA issue cost per warp (latency) or per SM (throughput)?
__global__ void timing3(long long* cycles, uint32_t id, int reps, int mode) {
  __shared__ alignas(128) uint8_t bs[64 * K * 2];
  __shared__ alignas(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 64 * K * 2 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(bs)[i] = 0x3C003C00u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tbase)), "n"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tbase;
  long long t0 = clock64();
  if (tid == 0) {
    const uint32_t b0 = smem_u32(bs);
    for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const uint64_t bd = sdesc(b0 + s * 2 * kLBO);
        const uint32_t acc = (s > 0) ? 1u : 0u;
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem + 64),
            "r"(tmem + 8 * s), "l"(bd), "r"(id), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)));
  }
  __syncwarp();
  {
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done) : "r"(smem_u32(&bar)), "r"(0) : "memory");
  }
  long long t1 = clock64();
  if (tid == 0) cycles[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(128));
}

// issue-cost test: descriptors precomputed outside the loop (uniform), 8 MMAs per iteration
template <int MODE>
__global__ void timing4(long long* cycles, uint32_t id, int reps) {
  __shared__ alignas(128) uint8_t bs[16 * K * 2];
  __shared__ alignas(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 16 * K * 2 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(bs)[i] = 0x3C003C00u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tbase)), "n"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tbase;
  long long t0 = clock64();
  if (tid == 0) {
    const uint32_t b0 = smem_u32(bs);
    const uint64_t d0 = sdesc(b0);
    for (int rep = 0; rep < reps; ++rep) {
      if (MODE == 0) {
        asm volatile(
            "{\n .reg .pred p, q;\n .reg .b64 d1, d2, d3, d4, d5, d6, d7;\n setp.ne.b32 p, %3, 0;\n setp.ne.b32 q, 1, 0;\n"
            "add.s64 d1, %2, 16;\n add.s64 d2, %2, 32;\n add.s64 d3, %2, 48;\n add.s64 d4, %2, 64;\n"
            "add.s64 d5, %2, 80;\n add.s64 d6, %2, 96;\n add.s64 d7, %2, 112;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %4, p;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%5], d1, %4, q;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%6], d2, %4, q;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%7], d3, %4, q;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%8], d4, %4, q;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%9], d5, %4, q;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%10], d6, %4, q;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%11], d7, %4, q;\n}\n" ::"r"(tmem + 64),
            "r"(tmem), "l"(d0), "r"(rep), "r"(id), "r"(tmem + 8), "r"(tmem + 16), "r"(tmem + 24), "r"(tmem + 32),
            "r"(tmem + 40), "r"(tmem + 48), "r"(tmem + 56));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)));
  }
  __syncwarp();
  {
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done) : "r"(smem_u32(&bar)), "r"(0) : "memory");
  }
  long long t1 = clock64();
  if (tid == 0) cycles[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(128));
}

static uint16_t h(float x) { __half v = __float2half_rn(x); uint16_t u; memcpy(&u, &v, 2); return u; }
static double hf(uint16_t u) { __half v; memcpy(&v, &u, 2); return (double)__half2float(v); }

int main() {
  uint16_t *hA = new uint16_t[M * K], *hB = new uint16_t[N * K];
  float* hD = new float[M * N];
  uint16_t *dA, *dB; float* dD; long long* dc;
  CK(cudaMalloc(&dA, M * K * 2)); CK(cudaMalloc(&dB, N * K * 2)); CK(cudaMalloc(&dD, M * N * 4)); CK(cudaMalloc(&dc, 8));
  uint32_t s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (s >> 8) & 0xFFFF; };
  int bad_total = 0;
  for (int enc = 0; enc < 3; ++enc) {
    for (int i = 0; i < M * K; ++i) {
      const int c = rnd() & 3, P = 2 + (rnd() % 3);
      if (enc == 0) hA[i] = h((float)c);
      else if (enc == 1) hA[i] = (uint16_t)(0x3C00u | ((uint32_t)c << (2 * P)));   // 1 + c*2^(2P-10)
      else hA[i] = (uint16_t)((uint32_t)c << (2 * (i % 3)));                       // subnormal c*2^(2p-24)
    }
    for (int i = 0; i < N * K; ++i) hB[i] = h(((int)(rnd() % 2001) - 1000) / 250.0f);
    CK(cudaMemcpy(dA, hA, M * K * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, hB, N * K * 2, cudaMemcpyHostToDevice));
    probe<<<1, 128>>>(dA, dB, dD, dc, 1);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(hD, dD, M * N * 4, cudaMemcpyDeviceToHost));
    double maxrel = 0; int bad = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0, mag = 0;
        for (int k = 0; k < K; ++k) { ref += hf(hA[m * K + k]) * hf(hB[n * K + k]); mag += fabs(hf(hA[m * K + k]) * hf(hB[n * K + k])); }
        const double err = fabs(hD[m * N + n] - ref) / (mag > 0 ? mag : 1);
        if (err > maxrel) maxrel = err;
        if (err > 1e-5) { if (bad < 3) printf("  enc %d m %d n %d: got %.9g ref %.9g\n", enc, m, n, hD[m * N + n], ref); ++bad; }
      }
    printf("encoding %d: max |err|/sum|terms| = %.3g, bad %d of %d\n", enc, maxrel, bad, M * N);
    bad_total += bad;
  }
  for (int reps : {64, 1024}) {
    probe<<<1, 128>>>(dA, dB, dD, dc, reps);
    CK(cudaDeviceSynchronize());
    long long cyc; CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
    printf("reps %d: %lld cycles for %d MMAs (M128 N64 K16, A in TMEM): %.2f cycles/MMA\n", reps, cyc, reps * 8,
           (double)cyc / (reps * 8));
  }
  for (int ss = 0; ss < 4; ++ss)
    for (int m : {64, 128})
      for (int n : {16, 64}) {
        if (m == 128 && n < 16) continue;
        CK(cudaFuncSetAttribute(timing, cudaFuncAttributeMaxDynamicSharedMemorySize, 0));
        timing<<<1, 128>>>(dc, idesc(m, n), 256, ss);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        long long cyc; CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
        printf("%s M%d N%d K16: %.2f cycles/MMA (%.0f FLOP/clk)\n", (ss & 1) ? ((ss & 2) ? "SS2" : "SS") : ((ss & 2) ? "TS2" : "TS"), m, n, (double)cyc / 2048,
               2.0 * m * n * 16 * 2048 / cyc);
      }
  {
    long long* dcy; CK(cudaMalloc(&dcy, 8 * 148 * 8));
    long long hc[148 * 8];
    for (int per : {1, 2, 4})
      for (int n : {16, 64}) {
        const int grid = 148 * per;
        timing3<<<grid, 128>>>(dcy, idesc(128, n), 512, 0);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(hc, dcy, 8 * grid, cudaMemcpyDeviceToHost));
        double avg = 0; for (int i = 0; i < grid; ++i) avg += hc[i]; avg /= grid;
        printf("timing3 %d CTA/SM M128 N%d: %.2f cycles per MMA per CTA\n", per, n, avg / (512 * 8));
      }
  }
  {
    long long* dcy; CK(cudaMalloc(&dcy, 8 * 148 * 8));
    long long hc[148 * 8];
    for (int per : {1, 4})
      for (int n : {16, 64}) {
        const int grid = 148 * per;
        timing4<0><<<grid, 128>>>(dcy, idesc(128, n), 512);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(hc, dcy, 8 * grid, cudaMemcpyDeviceToHost));
        double avg = 0; for (int i = 0; i < grid; ++i) avg += hc[i]; avg /= grid;
        printf("timing4 (8 MMAs per asm block) %d CTA/SM M128 N%d: %.2f cycles per MMA per CTA\n", per, n, avg / (512 * 8));
      }
  }
  printf(bad_total ? "PROBE FAILED\n" : "PROBE OK\n");
  return 0;
}
