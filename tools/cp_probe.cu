// cp_probe.cu — does tcgen05.cp.128x256b from a K-major SWIZZLE_128B shared-memory operand produce the
// tensor-memory A operand a TS tcgen05.mma expects?  (the wide family's split-feature
// prepass: Zr would be filled by tcgen05.cp instead of WORK-warp tcgen05.st.)
//   A: M = 128 rows x K = 128 fp16, K-major SW128 (two 64-element atoms, the layout k_stats' X/Z atoms
//      and W' use); B: N = 128 x K = 128, K-major SW128.
//   1. reference: SS-MMA D1 = A . B^T (8 k-steps of 16) from shared memory;
//   2. test: 8 x tcgen05.cp.128x256b, k-step kk's descriptor (start + 32 B within the atom, as the
//      UMMA k-advance) -> TMEM columns 8 kk .. 8 kk + 7, then TS-MMA D2 = A_tmem . B^T reading A at
//      column 8 kk per k-step (k_stats' `za + kk * 8`), issued by the same thread right behind the copies;
//   3. the copied columns read back with tcgen05.ld (column c of lane m = A[m][2c] | A[m][2c+1] << 16).
// Small-integer operands make every product and sum exact; the host checks all three.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o cp_probe tools/cp_probe.cu && ./cp_probe
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
__host__ __device__ constexpr uint32_t idesc_kk(int M, int N) {  // kind::f16, f16 A/B, f32 D, both K-major
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// K-major SW128 byte offset of element (row, k): atom k / 64 (16 KB), 128 B rows, swizzled 16 B chunks
__device__ __forceinline__ uint32_t k_off(int row, int k) {
  return (uint32_t)(k / 64) * 16384u + (uint32_t)row * 128u + ((uint32_t)(((k % 64) / 8) ^ (row & 7)) << 4) +
         (uint32_t)(k % 8) * 2u;
}
__host__ __device__ inline int aval(int m, int k) { return ((m * 3 + k * 5) % 7) - 3; }
__host__ __device__ inline int bval(int n, int k) { return ((n * 7 + k * 3) % 5) - 2; }

__global__ void __launch_bounds__(128, 1) probe(float *out, uint32_t *acols) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t *base = (uint8_t *)(((uintptr_t)smem + 1023) & ~(uintptr_t)1023);
  uint8_t *sA = base, *sB = base + 32768;
  uint64_t *bar = (uint64_t *)(base + 65536);
  uint32_t *s_tmem = (uint32_t *)(base + 65536 + 64);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < 128 * 128; e += 128) {
    const int r = e / 128, k = e % 128;
    *(__half *)(sA + k_off(r, k)) = __int2half_rn(aval(r, k));
    *(__half *)(sB + k_off(r, k)) = __int2half_rn(bval(r, k));
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(s_tmem)), "r"(512u));
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
  const uint32_t tmem = *s_tmem;  // columns: D1 0..127, D2 128..255, A copy 256..319
  if (tid == 0) {
    for (int kk = 0; kk < 8; ++kk) {  // 1. SS reference
      const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
      const uint64_t a = desc_sw128(su32(sA) + off, 16, 1024), b = desc_sw128(su32(sB) + off, 16, 1024);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem), "l"(a), "l"(b),
                   "r"(idesc_kk(128, 128)), "r"(kk)
                   : "memory");
    }
    for (int kk = 0; kk < 8; ++kk) {  // 2. copy A into TMEM, k-step by k-step
      const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
      asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tmem + 256 + 8 * kk),
                   "l"(desc_sw128(su32(sA) + off, 16, 1024))
                   : "memory");
    }
    for (int kk = 0; kk < 8; ++kk) {  //    TS-MMA from the copy
      const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
      const uint64_t b = desc_sw128(su32(sB) + off, 16, 1024);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem + 128),
                   "r"(tmem + 256 + 8 * kk), "l"(b), "r"(idesc_kk(128, 128)), "r"(kk)
                   : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[0]))
                 : "memory");
  }
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(
                   su32(&bar[0]))
               : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int which = 0; which < 3; ++which) {
    const int ncol = which < 2 ? 128 : 64;
    for (int c0 = 0; c0 < ncol; c0 += 8) {
      uint32_t r[8];
      const uint32_t ta = tmem + ((uint32_t)(32 * warp) << 16) + 128 * which + c0;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(ta));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int j = 0; j < 8; ++j) {
        const int m = 32 * warp + lane;
        if (which < 2) out[((size_t)which * 128 + m) * 128 + c0 + j] = __uint_as_float(r[j]);
        else acols[(size_t)m * 64 + c0 + j] = r[j];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
}

int main() {
  float *d_out;
  uint32_t *d_cols;
  cudaMalloc(&d_out, 2 * 128 * 128 * 4);
  cudaMalloc(&d_cols, 128 * 64 * 4);
  const int smem = 65536 + 1024 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<<<1, 128, smem>>>(d_out, d_cols);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("kernel error: %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<float> h(2 * 128 * 128);
  std::vector<uint32_t> c(128 * 64);
  cudaMemcpy(h.data(), d_out, h.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(c.data(), d_cols, c.size() * 4, cudaMemcpyDeviceToHost);
  long bad1 = 0, bad2 = 0, badc = 0;
  for (int m = 0; m < 128; ++m) {
    for (int n = 0; n < 128; ++n) {
      long ref = 0;
      for (int k = 0; k < 128; ++k) ref += (long)aval(m, k) * bval(n, k);
      if (h[(size_t)m * 128 + n] != (float)ref) ++bad1;
      if (h[(size_t)(128 + m) * 128 + n] != (float)ref) ++bad2;
    }
    for (int col = 0; col < 64; ++col) {
      const __half lo = __float2half((float)aval(m, 2 * col)), hi = __float2half((float)aval(m, 2 * col + 1));
      const uint32_t want = (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
      if (c[(size_t)m * 64 + col] != want) ++badc;
    }
  }
  printf("SS reference mismatches: %ld / 16384; TS-from-tcgen05.cp mismatches: %ld / 16384; copied A columns wrong: %ld / 8192\n",
         bad1, bad2, badc);
  return (bad1 || bad2 || badc) ? 2 : 0;
}
