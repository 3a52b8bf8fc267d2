// m64_probe.cu — where does a cta_group::1 kind::f16 tcgen05.mma with M = 64 put its accumulator in
// tensor memory?  (a D <= 96 wide family would run GEMM2 for the packed second feature
// half as M = 64.)  A = 64 (M) x 128 (K) and B = 64 (N) x 128 (K), both MN-major SW128 in shared memory
// (GEMM2's operand form), small integers (exact); D read back from all 128 lanes x 64 columns and each
// lane matched against the reference rows.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o m64_probe tools/m64_probe.cu && ./m64_probe
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
__device__ __forceinline__ uint32_t mn_off(int mn, int k) {  // MN-major SW128, one 64-element atom column
  return (uint32_t)k * 128u + ((uint32_t)(((mn % 64) / 8) ^ (k & 7)) << 4) + (uint32_t)(mn % 8) * 2u;
}
// column k = 0 carries the row index (times an all-ones B column), so every row of D is distinct
__host__ __device__ inline int aval(int m, int k) { return k == 0 ? m : ((m * 3 + k * 5) % 7) - 3; }
__host__ __device__ inline int bval(int n, int k) { return k == 0 ? 1 : ((n * 7 + k * 3) % 5) - 2; }

__global__ void __launch_bounds__(128, 1) probe(float *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t *base = (uint8_t *)(((uintptr_t)smem + 1023) & ~(uintptr_t)1023);
  uint8_t *sA = base, *sB = base + 16384;
  uint64_t *bar = (uint64_t *)(base + 32768);
  uint32_t *s_tmem = (uint32_t *)(base + 32768 + 64);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < 64 * 128; e += 128) {
    const int mn = e % 64, k = e / 64;
    *(__half *)(sA + mn_off(mn, k)) = __int2half_rn(aval(mn, k));
    *(__half *)(sB + mn_off(mn, k)) = __int2half_rn(bval(mn, k));
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(s_tmem)), "r"(128u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar[0])), "r"(1u));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *s_tmem;
  // clear the 64 columns of all 128 lanes first (so untouched lanes read 0)
  {
    const uint32_t ta = tmem + ((uint32_t)(32 * warp) << 16);
    for (int c = 0; c < 64; ++c) asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(ta + c), "r"(0u));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    for (int kk = 0; kk < 8; ++kk) {
      const uint64_t a = desc_sw128(su32(sA) + kk * 2048, 8192, 1024), b = desc_sw128(su32(sB) + kk * 2048, 8192, 1024);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem), "l"(a), "l"(b),
                   "r"(idesc(64, 64)), "r"(kk)
                   : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[0]))
                 : "memory");
  }
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(
                   su32(&bar[0]))
               : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c0 = 0; c0 < 64; c0 += 8) {
    uint32_t r[8];
    const uint32_t ta = tmem + ((uint32_t)(32 * warp) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) out[(size_t)(32 * warp + lane) * 64 + c0 + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128u));
}

int main() {
  float *d_out;
  cudaMalloc(&d_out, 128 * 64 * 4);
  const int smem = 32768 + 1024 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<<<1, 128, smem>>>(d_out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("kernel error: %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<float> h(128 * 64);
  cudaMemcpy(h.data(), d_out, h.size() * 4, cudaMemcpyDeviceToHost);
  // which reference row m (if any) does lane l hold in its 64 columns?
  int matched = 0;
  for (int l = 0; l < 128; ++l) {
    int who = -1;
    bool zero = true;
    for (int c = 0; c < 64; ++c) zero = zero && h[(size_t)l * 64 + c] == 0.f;
    for (int m = 0; m < 64 && who < 0; ++m) {
      bool ok = true;
      for (int n = 0; n < 64 && ok; ++n) {
        long ref = 0;
        for (int k = 0; k < 128; ++k) ref += (long)aval(m, k) * bval(n, k);
        ok = h[(size_t)l * 64 + n] == (float)ref;
      }
      if (ok) who = m;
    }
    if (who >= 0) ++matched;
    printf("lane %3d: %s%d\n", l, who >= 0 ? "row " : (zero ? "zero " : "other "), who);
    if (who >= 0 && who != 16 * (l / 32) + (l % 32)) matched = -100000;  // expected: quarter q, lanes 0-15
  }
  printf("lanes holding a full reference row: %d (layout row m -> lane 32 (m / 16) + m %% 16: %s)\n", matched < 0 ? 0 : matched,
         matched == 64 ? "yes" : "no");
  return 0;
}
