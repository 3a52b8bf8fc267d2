// tools/tmem_probe.cu — microbenchmark of the tensor-memory and shared-memory ports on one B200 SM,
// to decide between k_stats designs: how long 128x128x16 kind::f16 UMMAs take with A
// from TMEM (TS) or shared memory (SS), alone and while 16 warps stream tcgen05.st / tcgen05.ld /
// st.shared traffic.  One CTA per SM, 576 threads (16 WORK warps + MMA warp + idle warp), like k_stats.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1604_03498_b200/csrc \
//        -o /tmp/tmem_probe tools/tmem_probe.cu -lcuda && /tmp/tmem_probe
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "ptx.cuh"

using namespace gpufv::ptx;

constexpr int kThreads = 576, kWork = 16;
constexpr int kSmem = 200 * 1024;

// mode bits: 1 = MMA TS, 2 = MMA SS, 4 = WORK tcgen05.st, 8 = WORK tcgen05.ld, 16 = WORK st.shared,
// 32 = WORK fp32 -> fp16x2 split (cvt.rn.f16x2.f32 + unpack + fadd2 + cvt: the P / feature split),
// 64 = WORK ex2.approx (MUFU), 128 = split with the hi part rounded by integer ops (no unpack),
// 256 = only the WORK warps NOT on the MMA warp's sub-partition (warp % 4 != 0) do the WORK traffic,
// 512 = split with the hi part from a Veltkamp split on the FMA pipe (c = a (2^13 + 1), hi = c - (c - a))
__global__ void __launch_bounds__(kThreads, 1) probe(int mode, int iters, long long *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sbase = (smem_u32(smem) + 1023u) & ~1023u;
  if (warp == 0) { tmem_alloc(&s_tmem, 512); tmem_relinquish(); }
  if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  long long t0 = clock64();
  if (warp == kWork) {
    if (lane == 0 && (mode & 3)) {
      const uint32_t idesc = idesc_f16_f32(128, 128, 0, 0);
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t bdesc = desc_sw128(sbase + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
          if (mode & 1) mma_f16_ts(tmem + 256, tmem + kk * 8, bdesc, idesc, 1u);
          else mma_f16_ss(tmem + 256, desc_sw128(sbase + 65536 + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024), bdesc,
                          idesc, 1u);
        }
      }
      mma_commit(&bar);
      mbar_wait(&bar, 0);
      if (blockIdx.x == 0) out[2] = clock64() - t0;  // MMA stream done
    }
  } else if (warp < kWork && !((mode & 256) && (warp & 3) == 0)) {
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    uint32_t r[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) r[i] = tid + i;
    const int witers = iters * 2;
    if (mode & 4) {
      for (int it = 0; it < witers; ++it) tmem_st32(tmem + 128 + lane_base + 32 * (warp >> 2), r);  // 32 cols
      tmem_st_wait();
    }
    if (mode & 8) {
      for (int it = 0; it < witers; ++it) {
        tmem_ld32(tmem + 384 + lane_base + 32 * (warp >> 2), r);
        tmem_ld_wait(r);
      }
    }
    if (mode & 16) {
      for (int it = 0; it < witers; ++it)
#pragma unroll
        for (int j = 0; j < 8; ++j) sts128(sbase + 131072 + ((warp * 8 + j) * 32 + lane) * 16 % 65536, r[j], r[j + 1], r[j + 2], r[j + 3]);
    }
    if (mode & 32) {
      float2 a = make_float2(__uint_as_float(r[0]) * 1e-30f + 0.37f, __uint_as_float(r[1]) * 1e-30f + 0.61f);
      uint32_t acc = 0;
      for (int it = 0; it < witers * 8; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          uint32_t hi, lo;
          split2_f16(a, hi, lo);
          acc ^= hi + lo;
          a.x += 1e-3f; a.y -= 1e-3f;
        }
      }
      r[0] = acc;
    }
    if (mode & 128) {
      float2 a = make_float2(__uint_as_float(r[0]) * 1e-30f + 0.37f, __uint_as_float(r[1]) * 1e-30f + 0.61f);
      uint32_t acc = 0;
      for (int it = 0; it < witers * 8; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float2 hf = make_float2(__uint_as_float((__float_as_uint(a.x) + 0x1000u) & 0xFFFFE000u),
                                        __uint_as_float((__float_as_uint(a.y) + 0x1000u) & 0xFFFFE000u));
          const __half2 h = __floats2half2_rn(hf.x, hf.y);
          const float2 d = __fadd2_rn(a, make_float2(-hf.x, -hf.y));
          const __half2 l = __floats2half2_rn(d.x, d.y);
          acc ^= *reinterpret_cast<const uint32_t *>(&h) + *reinterpret_cast<const uint32_t *>(&l);
          a.x += 1e-3f; a.y -= 1e-3f;
        }
      }
      r[0] = acc;
    }
    if (mode & 512) {
      float2 a = make_float2(__uint_as_float(r[0]) * 1e-30f + 0.37f, __uint_as_float(r[1]) * 1e-30f + 0.61f);
      uint32_t acc = 0;
      const float2 kSplit = make_float2(8193.f, 8193.f);
      for (int it = 0; it < witers * 8; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float2 c = __fmul2_rn(a, kSplit);
          const float2 hf = __fadd2_rn(c, __fadd2_rn(a, make_float2(-c.x, -c.y)));
          const __half2 h = __floats2half2_rn(hf.x, hf.y);
          const float2 d = __fadd2_rn(a, make_float2(-hf.x, -hf.y));
          const __half2 l = __floats2half2_rn(d.x, d.y);
          acc ^= *reinterpret_cast<const uint32_t *>(&h) + *reinterpret_cast<const uint32_t *>(&l);
          a.x += 1e-3f; a.y -= 1e-3f;
        }
      }
      r[0] = acc;
    }
    if (mode & 64) {
      float x = __uint_as_float(r[0]) * 1e-30f;
      for (int it = 0; it < witers * 8; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) x = ex2_approx(x) * -0.5f;
      }
      r[0] = __float_as_uint(x);
    }
    if (r[0] == 0xdeadbeef) out[1] = r[1];
    if (blockIdx.x == 0 && lane == 0) atomicMax(reinterpret_cast<unsigned long long *>(out + 3), (unsigned long long)(clock64() - t0));
  }
  tc_fence_before();
  __syncthreads();
  long long t1 = clock64();
  if (tid == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  long long *d;
  cudaMalloc(&d, 64);
  const int iters = 2000;
  struct { int mode; const char *name; } cases[] = {
      {1, "TS MMA alone"}, {2, "SS MMA alone"}, {4, "tcgen05.st alone"}, {8, "tcgen05.ld alone"},
      {16, "st.shared alone"}, {1 | 4, "TS MMA + tcgen05.st"}, {1 | 8, "TS MMA + tcgen05.ld"},
      {1 | 16, "TS MMA + st.shared"}, {2 | 4, "SS MMA + tcgen05.st"}, {2 | 16, "SS MMA + st.shared"},
      {2 | 8, "SS MMA + tcgen05.ld"}, {32, "fp16x2 split alone"}, {64, "ex2 alone"}, {1 | 32, "TS MMA + split"}, {128, "int-round split alone"},
      {1 | 128, "TS MMA + int-round split"}, {1 | 32 | 256, "TS MMA + split (not SMSP0)"},
      {1 | 128 | 256, "TS MMA + int split (not SMSP0)"}, {2 | 32, "SS MMA + split"}, {2 | 32 | 256, "SS MMA + split (not SMSP0)"},
      {512, "Veltkamp split alone"}, {1 | 512, "TS MMA + Veltkamp split"}};
  for (auto &c : cases) {
    probe<<<148, kThreads, kSmem>>>(c.mode, iters, d);  // warm-up
    cudaMemset(d, 0, 64);
    probe<<<148, kThreads, kSmem>>>(c.mode, iters, d);
    long long v[4] = {};
    if (cudaMemcpy(v, d, 32, cudaMemcpyDeviceToHost) != cudaSuccess) { printf("error %s\n", cudaGetErrorString(cudaGetLastError())); return 1; }
    const long long cyc = v[0], cmma = v[2], cwork = v[3];
    const double mma = (c.mode & 3) ? (double)iters * 8 : 0;
    const double wbytes = (c.mode & 4 || c.mode & 8) ? (double)iters * 2 * 16 * 32 * 32 * 4 : 0;  // per warp 4 KB per op
    const double sbytes = (c.mode & 16) ? (double)iters * 2 * 16 * 8 * 512 : 0;
    const double nsplit = (c.mode & (32 | 128 | 512)) ? (double)iters * 2 * 8 * 8 * 16 * 32 : 0;  // pairs split per SM
    const double nex2 = (c.mode & 64) ? (double)iters * 2 * 8 * 8 * 16 * 32 : 0;
    printf("%-24s %10lld cycles (mma %lld, work %lld)", c.name, cyc, cmma, cwork);
    if (mma) printf("  %6.1f cyc/UMMA", cmma / mma);
    if (wbytes) printf("  TMEM %6.1f B/clk", wbytes / cwork);
    if (sbytes) printf("  SMEM st %6.1f B/clk", sbytes / cwork);
    if (nsplit) printf("  split %6.2f pairs/clk", nsplit / cwork);
    if (nex2) printf("  ex2 %6.2f /clk", nex2 / cwork);
    printf("\n");
  }
  return 0;
}
