// k_embed.cuh — the step upstream of the FV path: raw 128-d dense-SIFT
// descriptors -> the encoder's M = m + 2 dims, "by lowering the dimension to m (m<128) with PCA and
// adding the normalized X and Y axis" (§3.1; SPEC embed S:201-203, no whitening):
//   X'_i = [ basis (d_i - mean) ; x_i / W_b ; y_i / H_b ; 0 ... ]   (row stride ldx = round_up(m+2, 4))
//
// A persistent tcgen05 kernel, computed transposed so that the PCA basis is the resident operand:
//   E^T[c, i] = sum_k basis[c, k] (d_ik - mean_k)
//   * A = basis (M = 128 output dims, rows >= m zero; K = 128) lives in tensor memory for the whole
//     kernel, split into tf32 hi | lo (each CTA converts it once in its prologue);
//   * B = one tile of 128 raw descriptors (N = 128, K-major): TMA brings it in four 32-dim boxes
//     (128B-swizzled, exactly the tf32 K-major operand layout) through a 6-stage ring; the WORK warps
//     subtract the mean and split each element in place into tf32 hi and a lo copy;
//   * 3 x TF32 split products (lo.hi + hi.lo + hi.hi per box, ~22 significant bits, fp32 accumulate)
//     into a double-buffered TMEM accumulator (lanes = output dims, columns = descriptors);
//   * epilogue: lane c of a warp writes dim c of 32 consecutive rows — each store instruction covers
//     128 contiguous bytes of one output row; lanes m, m + 1 write x/W, y/H, the rest of the row zero.
// kind::tf32 (not the fp16 split the encoder uses): raw SIFT values span any scale (0..0.5 or 0..255)
// and tf32 keeps the fp32 exponent range, so no operand scaling is needed; the tensor work (0.38 ms
// per 5.12 M rows at the tf32 rate) stays below the HBM time of the 512 B read + 4 ldx B written per
// descriptor, the kernel's bound.
#pragma once
#include <cuda.h>

#include "fv_common.cuh"
#include "ptx.cuh"

namespace gpufv {

constexpr int kEmbIn = 128;      // raw descriptor dims (SIFT: 8 orientations x 4 x 4 bins)
constexpr int kEmbMaxM = 126;    // M = m + 2 <= 128 (the encoder's D limit)
constexpr int kEmbStages = 5;    // ring of 32-dim boxes (a tile is 4 boxes)
constexpr int kEmbBox = 128 * 128;  // one box: 128 rows x 32 fp32 (128 B per row, SW128)
constexpr int kEmbXySlots = 8;      // ring of per-tile keypoint blocks (128 rows x 2 fp32 = 1 KB)
// roles: warp 0 MMA, warp 1 TMA, warps 2..9 EPILOGUE (TMEM lane quarter = warp % 4, descriptor half =
// (warp - 2) / 4; they also load the basis), warps 10..17 CONVERSION (mean subtraction + tf32 split)
constexpr int kEmbEpi = 8, kEmbConv = 8;
constexpr int kEmbThreads = (2 + kEmbEpi + kEmbConv) * 32;
// shared memory: stage s = [hi (in place of the TMA box) | lo], keypoint ring, mean, store staging, barriers
constexpr int kEmbSmHi = 0;
constexpr int kEmbSmLo = kEmbStages * kEmbBox;
constexpr int kEmbSmXy = 2 * kEmbStages * kEmbBox;
constexpr int kEmbSmOut = kEmbSmXy + kEmbXySlots * 1024;    // float[8 warps][32 rows][32 dims]: store staging
constexpr int kEmbSmMean = kEmbSmOut + kEmbEpi * 32 * 32 * 4;
constexpr int kEmbSmTileB = kEmbSmMean + kEmbIn * 4;       // int[8]: image of each tile's first row
constexpr int kEmbSmBar = kEmbSmTileB + 32;
constexpr int kEmbNumBars = 3 * kEmbStages + kEmbXySlots + 5;
constexpr int kEmbSmTmem = kEmbSmBar + kEmbNumBars * 8;
constexpr int kEmbSmemBytes = kEmbSmTmem + 16 + 1024;
static_assert(kEmbSmemBytes <= 232448, "shared memory budget (embed)");
// tensor memory: basis hi [0,128), basis lo [128,256), E^T double buffer [256,384), [384,512)
constexpr uint32_t kEmbTAhi = 0, kEmbTAlo = 128, kEmbTE = 256;

struct EmbedParams {
  const float *xy;               // n x 2 (pixels)
  const int64_t *offsets;        // batch + 1
  const float *wh;               // batch x 2 (image width, height)
  const float *mean;             // 128
  const float *basis;            // m x 128 (rows orthonormal)
  float *out;                    // n x ldx
  int64_t n;
  int batch, m, ldx;
};

namespace ptx {
// tf32 (round to nearest, ties away) in an fp32 container: the value the tensor core consumes
__device__ __forceinline__ float to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
// D[tmem] (+)= A[tmem] * B[smem], kind::tf32, warp-converged issue (one elected lane)
__device__ __forceinline__ void mma_tf32_ts_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(0u), "r"(0u), "r"(0u), "r"(0u)
      : "memory");
}
}  // namespace ptx

// kind::tf32 instruction descriptor: D f32, A/B tf32 (format 2), both K-major
__host__ __device__ constexpr uint32_t idesc_tf32_f32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

__global__ void __launch_bounds__(kEmbThreads, 1) k_embed(const __grid_constant__ CUtensorMap tmap_raw,
                                                          const __grid_constant__ CUtensorMap tmap_xy,
                                                          const __grid_constant__ CUtensorMap tmap_out,
                                                          const EmbedParams p) {
  using namespace ptx;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_base = smem_u32(smem_raw);
  const uint32_t sbase = (raw_base + 1023u) & ~1023u;
  uint8_t *smem = smem_raw + (sbase - raw_base);
  float *s_mean = reinterpret_cast<float *>(smem + kEmbSmMean);
  int *s_tileb = reinterpret_cast<int *>(smem + kEmbSmTileB);
  float *s_out = reinterpret_cast<float *>(smem + kEmbSmOut);
  const float2 *s_xy = reinterpret_cast<const float2 *>(smem + kEmbSmXy);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + kEmbSmBar);
  uint64_t *b_xfull = bars, *b_conv = bars + kEmbStages, *b_xempty = bars + 2 * kEmbStages;
  uint64_t *b_xyfull = bars + 3 * kEmbStages;
  uint64_t *b_efull = b_xyfull + kEmbXySlots, *b_eempty = b_efull + 2, *b_basis = b_efull + 4;
  uint32_t *s_tmem = reinterpret_cast<uint32_t *>(smem + kEmbSmTmem);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid < kEmbIn) s_mean[tid] = p.mean[tid];
  if (warp == 0) { tmem_alloc(s_tmem, kTmemCols); tmem_relinquish(); }
  if (tid == 32) {
    for (int s = 0; s < kEmbStages; ++s) {
      mbar_init(&b_xfull[s], 1);
      mbar_init(&b_conv[s], kEmbConv);
      mbar_init(&b_xempty[s], 1);
    }
    for (int s = 0; s < kEmbXySlots; ++s) mbar_init(&b_xyfull[s], 1);
    for (int e = 0; e < 2; ++e) { mbar_init(&b_efull[e], 1); mbar_init(&b_eempty[e], kEmbEpi); }
    mbar_init(b_basis, kEmbEpi);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  const int64_t ntiles = (p.n + 127) / 128;
  // local tiles of this CTA: blockIdx.x, + gridDim.x, ...
  const int nloc = (int)((ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x);

  if (warp == 1) {
    // ======================================================= TMA producer: 4 boxes + keypoints per tile
    // Ring distances: the producer runs at most 1.25 tiles ahead of the MMA (5 box stages) and the MMA
    // at most 2 tiles ahead of the epilogue (2 accumulators), so the 8-slot keypoint / image rings are
    // never overwritten before the epilogue has read them.
    if (lane == 0 && nloc > 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_raw)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_xy)) : "memory");
      for (int i = 0; i < nloc; ++i) {
        const int row0 = (int)(((int64_t)blockIdx.x + (int64_t)i * gridDim.x) * 128);
        {  // image of the tile's first row (last b with offsets[b] <= row0), published with the keypoints
          int lo = 0, hi = p.batch - 1;
          while (lo < hi) { const int mid = (lo + hi + 1) >> 1; if (p.offsets[mid] <= row0) lo = mid; else hi = mid - 1; }
          s_tileb[i & 7] = lo;
        }
        // keypoints of the tile's rows: floats [2 row0, 2 row0 + 256) of xy (past 2n read as zero)
        mbar_arrive_expect_tx(&b_xyfull[i & 7], 1024);
        asm volatile(
            "cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];" ::"r"(
                sbase + kEmbSmXy + (i & 7) * 1024),
            "l"(reinterpret_cast<uint64_t>(&tmap_xy)), "r"(2 * row0), "r"(smem_u32(&b_xyfull[i & 7]))
            : "memory");
        for (int b = 0; b < 4; ++b) {
          const int g = 4 * i + b, s = g % kEmbStages;
          if (g >= kEmbStages) mbar_wait(&b_xempty[s], ((g / kEmbStages) - 1) & 1);
          mbar_arrive_expect_tx(&b_xfull[s], kEmbBox);
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                  sbase + kEmbSmHi + s * kEmbBox),
              "l"(reinterpret_cast<uint64_t>(&tmap_raw)), "r"(32 * b), "r"(row0), "r"(smem_u32(&b_xfull[s]))
              : "memory");
        }
      }
    }
  } else if (warp == 0) {
    // ======================================================= MMA issuer (warp-converged)
    if (nloc > 0) {
      const uint32_t idesc = idesc_tf32_f32(128, 128);
      mbar_wait(b_basis, 0);
      tc_fence_after();
      for (int i = 0; i < nloc; ++i) {
        const int e = i & 1;
        if (i >= 2) mbar_wait(&b_eempty[e], ((i >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t dE = tmem + kEmbTE + 128 * e;
        for (int b = 0; b < 4; ++b) {
          const int g = 4 * i + b, s = g % kEmbStages;
          mbar_wait(&b_conv[s], (g / kEmbStages) & 1);
          tc_fence_after();
          const uint64_t dHi = desc_sw128(sbase + kEmbSmHi + s * kEmbBox, 16, 1024);
          const uint64_t dLo = desc_sw128(sbase + kEmbSmLo + s * kEmbBox, 16, 1024);
#pragma unroll
          for (int sp = 0; sp < 3; ++sp) {  // basis_lo.x_hi, basis_hi.x_lo, basis_hi.x_hi
            const uint32_t aT = tmem + (sp == 0 ? kEmbTAlo : kEmbTAhi) + 32 * b;
            const uint64_t dB = sp == 1 ? dLo : dHi;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)  // K = 8 tf32 = 32 bytes of the 128-byte row
              mma_tf32_ts_w(dE, aT + 8 * kk, dB + ((kk * 32) >> 4), idesc, (b | sp | kk) != 0);
          }
          mma_commit_w(&b_xempty[s]);  // the stage may be reloaded once these UMMAs have read it
        }
        mma_commit_w(&b_efull[e]);
      }
    }
  } else if (warp < 2 + kEmbEpi) {
    // ======================================================= EPILOGUE warps (two per TMEM lane quarter)
    const int q = warp & 3, ew = warp - 2, hh = ew >> 2;   // output dims 32 q .., descriptors 64 hh ..
    const uint32_t lane_base = (uint32_t)(32 * q) << 16;
    const int c = 32 * q + lane;
    {
      // basis -> tf32 hi | lo in TMEM: lane c = output dim, columns k (this warp: 64 hh .. 64 hh + 63)
#pragma unroll 1
      for (int kc = 2 * hh; kc < 2 * hh + 2; ++kc) {
        uint32_t hi[32], lo[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float v = c < p.m ? p.basis[(size_t)c * kEmbIn + 32 * kc + j] : 0.f;
          const float h = to_tf32(v);
          hi[j] = __float_as_uint(h);
          lo[j] = __float_as_uint(to_tf32(v - h));
        }
        tmem_st32(tmem + kEmbTAhi + lane_base + 32 * kc, hi);
        tmem_st32(tmem + kEmbTAlo + lane_base + 32 * kc, lo);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(b_basis);
    }
    const bool active = 32 * q < p.ldx;
    const bool xy_warp = 32 * q <= p.m + 1 && p.m < 32 * q + 32;  // this quarter holds dim m or m + 1
    float *stg = s_out + ew * 32 * 32;                            // this warp's 32 rows x 32 dims block
    const uint32_t stg_a = smem_u32(stg);
    for (int i = 0; i < nloc; ++i) {
      const int e = i & 1;
      const int64_t row0 = ((int64_t)blockIdx.x + (int64_t)i * gridDim.x) * 128;
      if (xy_warp) mbar_wait(&b_xyfull[i & 7], (i >> 3) & 1);
      mbar_wait(&b_efull[e], (i >> 1) & 1);
      tc_fence_after();
      if (active) {
#pragma unroll 1
        for (int ch = 0; ch < 2; ++ch) {
          const int j0 = 64 * hh + 32 * ch;
          uint32_t v[32];
          tmem_ld32(tmem + kEmbTE + 128 * e + lane_base + j0, v);
          // normalised keypoint of row j0 + lane: its image is found by walking forward from the image
          // of the tile's first row (usually 0-1 steps)
          float2 xn = make_float2(0.f, 0.f);
          if (xy_warp && row0 + j0 + lane < p.n) {
            const int64_t myrow = row0 + j0 + lane;
            int b = s_tileb[i & 7];
            while (p.offsets[b + 1] <= myrow) ++b;
            const float2 xy = s_xy[(i & 7) * 128 + j0 + lane];
            const float2 wh = reinterpret_cast<const float2 *>(p.wh)[b];
            xn = make_float2(xy.x / wh.x, xy.y / wh.y);
          }
          // the staging block is free once the previous chunk's TMA store has read it
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          __syncwarp();
          tmem_ld_wait(v);
#pragma unroll
          for (int j = 0; j < 32; ++j) stg[j * 32 + lane] = c < p.m ? __uint_as_float(v[j]) : 0.f;
          if (xy_warp) {
            __syncwarp();
            if (p.m >= 32 * q) stg[lane * 32 + (p.m - 32 * q)] = xn.x;
            if (p.m + 1 < 32 * q + 32) stg[lane * 32 + (p.m + 1 - 32 * q)] = xn.y;
          }
          fence_proxy_async_smem();
          __syncwarp();
          // one 32-row x 32-dim box to out (dims >= ldx and rows >= n are clipped by the tensor map)
          if (lane == 0) {
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                             reinterpret_cast<uint64_t>(&tmap_out)),
                         "r"(32 * q), "r"((int)(row0 + j0)), "r"(stg_a)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&b_eempty[e]);
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores complete
  } else {
    // ======================================================= CONVERSION warps
    const int ct = tid - 32 * (2 + kEmbEpi);   // 0..255
    const int crow = ct & 127, cg = ct >> 7;  // row, chunk group (16-byte chunks 4 cg .. 4 cg + 3)
    for (int i = 0; i < nloc; ++i) {
#pragma unroll 1
      for (int b = 0; b < 4; ++b) {
        const int g = 4 * i + b, s = g % kEmbStages;
        mbar_wait(&b_xfull[s], (g / kEmbStages) & 1);
        uint8_t *hib = smem + kEmbSmHi + s * kEmbBox;
        uint8_t *lob = smem + kEmbSmLo + s * kEmbBox;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          const int ch = 4 * cg + cc;
          const uint32_t o = crow * 128 + ((ch ^ (crow & 7)) << 4);
          float4 v = *reinterpret_cast<const float4 *>(hib + o);
          const float4 mu = *reinterpret_cast<const float4 *>(s_mean + 32 * b + 4 * ch);
          v.x -= mu.x; v.y -= mu.y; v.z -= mu.z; v.w -= mu.w;
          const float4 h = make_float4(to_tf32(v.x), to_tf32(v.y), to_tf32(v.z), to_tf32(v.w));
          const float4 l = make_float4(to_tf32(v.x - h.x), to_tf32(v.y - h.y), to_tf32(v.z - h.z), to_tf32(v.w - h.w));
          *reinterpret_cast<float4 *>(hib + o) = h;
          *reinterpret_cast<float4 *>(lob + o) = l;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&b_conv[s]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, kTmemCols);
}

}  // namespace gpufv
