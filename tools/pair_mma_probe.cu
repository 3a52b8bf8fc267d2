// pair_mma_probe.cu — can one kernel mix cta_group::2 and cta_group::1 tcgen05.mma, with each CTA's
// tensor memory allocated by a cta_group::1 tcgen05.alloc?  The shapes are GEMM2's in pair form
// (DESIGN.md §13): A = P^T (MN-major SW128, M = 128 Gaussians per CTA, K = 128 descriptor rows),
// B = one 64-feature half of Z per CTA (MN-major SW128, N = 64 per CTA, 128 in the pair).
//   1. the leader issues 8 x tcgen05.mma.cta_group::2 (M = 256, N = 128, K = 16) and commits with
//      multicast to both CTAs' barriers: CTA r's TMEM gets its own 128 rows x all 128 columns;
//   2. then each CTA issues 8 x tcgen05.mma.cta_group::1 (M = 128, N = 128) from its own SMEM into
//      another TMEM region.
// Small-integer operands make every product and sum exact; the host checks both results.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o pair_mma_probe tools/pair_mma_probe.cu && ./pair_mma_probe
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int M, int N) {  // kind::f16, f16 A/B, f32 D, both MN-major
  return (1u << 4) | (1u << 15) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// MN-major SW128 element offset (bytes): atom = mn / 64 (stride lbo), row = k (128 B), swizzled chunk
__device__ __forceinline__ uint32_t mn_off(int mn, int k, uint32_t lbo) {
  return (uint32_t)(mn / 64) * lbo + (uint32_t)k * 128u + ((uint32_t)(((mn % 64) / 8) ^ (k & 7)) << 4) + (uint32_t)(mn % 8) * 2u;
}
__host__ __device__ inline int aval(int r, int m, int k) { return ((m * 3 + k * 5 + r * 11) % 7) - 3; }
__host__ __device__ inline int bval(int n, int k) { return ((n * 7 + k * 3) % 5) - 2; }       // n global 0..127
__host__ __device__ inline int b2val(int r, int n, int k) { return ((n * 5 + k + r) % 9) - 4; }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) probe(float *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t *base = (uint8_t *)(((uintptr_t)smem + 1023) & ~(uintptr_t)1023);
  uint8_t *sA = base;              // 2 atoms x 16 KB: M = 128, K = 128
  uint8_t *sB = base + 32768;      // 1 atom: N = 64 (this CTA's half), K = 128
  uint8_t *sB2 = base + 49152;     // 2 atoms: N = 128 (cta_group::1 test)
  uint64_t *bar = (uint64_t *)(base + 81920);
  uint32_t *s_tmem = (uint32_t *)(base + 81920 + 64);
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < 128 * 128; e += 128) {
    const int mn = e % 128, k = e / 128;
    *(__half *)(sA + mn_off(mn, k, 16384)) = __int2half_rn(aval(rank, mn, k));
    *(__half *)(sB2 + mn_off(mn, k, 16384)) = __int2half_rn(b2val(rank, mn, k));
    if (mn < 64) *(__half *)(sB + mn_off(mn, k, 16384)) = __int2half_rn(bval(64 * rank + mn, k));
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(s_tmem)), "r"(512u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar[0])), "r"(1u));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar[1])), "r"(1u));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *s_tmem;
  auto wait = [&](uint64_t *b) {
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(
                     su32(b))
                 : "memory");
  };
  if (rank == 0 && tid == 0) {  // pair MMA: D (cols 0..127) = A(256 x 128) . B(128 x 128)
    for (int kk = 0; kk < 8; ++kk) {
      const uint64_t a = desc_sw128(su32(sA) + kk * 2048, 16384, 1024), b = desc_sw128(su32(sB) + kk * 2048, 16384, 1024);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem), "l"(a), "l"(b),
                   "r"(idesc(256, 128)), "r"(kk)
                   : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                     su32(&bar[0])),
                 "h"((uint16_t)3)
                 : "memory");
  }
  wait(&bar[0]);
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {  // per-CTA MMA: D2 (cols 256..383) = A(128 x 128) . B2(128 x 128)
    for (int kk = 0; kk < 8; ++kk) {
      const uint64_t a = desc_sw128(su32(sA) + kk * 2048, 16384, 1024), b = desc_sw128(su32(sB2) + kk * 2048, 16384, 1024);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem + 256), "l"(a), "l"(b),
                   "r"(idesc(128, 128)), "r"(kk)
                   : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[1]))
                 : "memory");
  }
  wait(&bar[1]);
  asm volatile("tcgen05.fence::after_thread_sync;");
  // read back: warp w = lanes 32w .. (rows), 128 columns of D and of D2
  for (int which = 0; which < 2; ++which) {
    for (int c0 = 0; c0 < 128; c0 += 8) {
      uint32_t r[8];
      const uint32_t ta = tmem + ((uint32_t)(32 * warp) << 16) + (which ? 256 : 0) + c0;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(ta));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int j = 0; j < 8; ++j)
        out[(((size_t)rank * 2 + which) * 128 + 32 * warp + lane) * 128 + c0 + j] = __uint_as_float(r[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
}

int main() {
  float *d_out;
  const size_t n = 2 * 2 * 128 * 128;
  cudaMalloc(&d_out, n * 4);
  cudaMemset(d_out, 0, n * 4);
  const int smem = 81920 + 1024 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<<<2, 128, smem>>>(d_out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("kernel error: %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<float> h(n);
  cudaMemcpy(h.data(), d_out, n * 4, cudaMemcpyDeviceToHost);
  long bad = 0, bad2 = 0;
  for (int r = 0; r < 2; ++r)
    for (int m = 0; m < 128; ++m)
      for (int c = 0; c < 128; ++c) {
        long ref = 0, ref2 = 0;
        for (int k = 0; k < 128; ++k) { ref += (long)aval(r, m, k) * bval(c, k); ref2 += (long)aval(r, m, k) * b2val(r, c, k); }
        if (h[(((size_t)r * 2 + 0) * 128 + m) * 128 + c] != (float)ref) ++bad;
        if (h[(((size_t)r * 2 + 1) * 128 + m) * 128 + c] != (float)ref2) ++bad2;
      }
  printf("pair cta_group::2 result mismatches: %ld / %d; per-CTA cta_group::1 mismatches: %ld / %d\n", bad, 2 * 128 * 128,
         bad2, 2 * 128 * 128);
  return (bad || bad2) ? 2 : 0;
}
