// tools/signed_sqrt_check.cu — exhaustive check, over every finite fp32 bit pattern, that the
// finalize kernels' signed_sqrt (fv_common.cuh) equals copysignf(sqrtf(fabsf(x)), x) bit for bit.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1604_03498_b200/csrc -o /tmp/ssq \
//        tools/signed_sqrt_check.cu && /tmp/ssq
#include <cmath>
#include <cstdint>
#include <cstdio>

#include "fv_common.cuh"

__global__ void k(unsigned long long *bad, uint32_t base) {
  const uint32_t bits = base + blockIdx.x * blockDim.x + threadIdx.x;
  const float x = __uint_as_float(bits);
  if (!isfinite(x)) return;
  const float a = copysignf(sqrtf(fabsf(x)), x), b = gpufv::signed_sqrt(x);
  if (__float_as_uint(a) != __float_as_uint(b)) atomicAdd(bad, 1ull);
}

int main() {
  unsigned long long *d, h = 0;
  cudaMalloc(&d, 8);
  cudaMemset(d, 0, 8);
  for (uint64_t base = 0; base < (1ull << 32); base += (1ull << 30)) k<<<(1 << 30) / 256, 256>>>(d, (uint32_t)base);
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("signed_sqrt mismatches over all finite floats: %llu (%s)\n", h, cudaGetErrorString(cudaGetLastError()));
  return h != 0;
}
