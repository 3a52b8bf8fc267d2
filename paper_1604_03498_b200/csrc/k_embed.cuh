// k_embed.cuh — the step upstream of the FV path: raw 128-d dense-SIFT
// descriptors -> the encoder's M = m + 2 dims, "by lowering the dimension to m (m<128) with PCA and
// adding the normalized X and Y axis" (§3.1; SPEC embed S:201-203, no whitening):
//   X'_i = [ basis (d_i - mean) ; x_i / W_b ; y_i / H_b ; 0 ... ]   (row stride ldx = round_up(m+2, 4))
// A register-tiled fp32 SIMT GEMM (N x 128 . 128 x m, K = 128 is too short and the result feeds an
// fp32 path, so no tensor-core split): persistent blocks of 256 threads keep basis^T in shared
// memory and stream 64-row tiles; each thread owns 4 rows x 8 columns.
// Bound: fp32 FMA issue (10,240 FMA per descriptor at m = 80; 512 B read + 4 ldx B written).
#pragma once
#include "fv_common.cuh"

namespace gpufv {

constexpr int kEmbIn = 128;      // raw descriptor dims (SIFT: 8 orientations x 4 x 4 bins)
constexpr int kEmbRows = 64;     // rows per tile
constexpr int kEmbMaxM = 126;    // M = m + 2 <= 128 (the encoder's D limit)
constexpr int kEmbXStride = kEmbIn + 1;

struct EmbedParams {
  const float *raw;              // n x 128
  const float *xy;               // n x 2 (pixels)
  const int64_t *offsets;        // batch + 1
  const float *wh;               // batch x 2 (image width, height)
  const float *mean;             // 128
  const float *basis;            // m x 128 (rows orthonormal)
  float *out;                    // n x ldx
  int64_t n;
  int batch, m, mpad, ldx;
};

__global__ void __launch_bounds__(256) k_embed(const EmbedParams p) {
  extern __shared__ float emb_smem[];
  float *Bs = emb_smem;                           // [128][mpad]: Bs[k][c] = basis[c][k]
  float *Xs = emb_smem + kEmbIn * p.mpad;         // [64][129]: d - mean, row-major (padded)
  const int tid = threadIdx.x;
  const int cgroups = p.mpad / 8, nthr = 16 * cgroups;
  for (int e = tid; e < kEmbIn * p.mpad; e += 256) {
    const int c = e / kEmbIn, k = e - c * kEmbIn;  // coalesced over k in the basis
    Bs[k * p.mpad + c] = c < p.m ? p.basis[(size_t)c * kEmbIn + k] : 0.f;
  }
  const int rg = tid % 16, cg = tid / 16;  // rows rg + 16 i (i < 4; conflict-free Xs reads) x 8 columns
  const float4 *mean4 = reinterpret_cast<const float4 *>(p.mean);
  const int64_t ntiles = (p.n + kEmbRows - 1) / kEmbRows;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t r0 = t * kEmbRows;
    const int nr = (int)(p.n - r0 < kEmbRows ? p.n - r0 : kEmbRows);
    __syncthreads();  // Bs ready / previous tile consumed
    for (int e = tid; e < kEmbRows * (kEmbIn / 4); e += 256) {
      const int r = e / (kEmbIn / 4), k4 = e - r * (kEmbIn / 4);
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < nr) {
        v = __ldcs(reinterpret_cast<const float4 *>(p.raw + (size_t)(r0 + r) * kEmbIn) + k4);
        const float4 mu = mean4[k4];
        v.x -= mu.x; v.y -= mu.y; v.z -= mu.z; v.w -= mu.w;
      }
      float *xr = Xs + r * kEmbXStride + 4 * k4;
      xr[0] = v.x; xr[1] = v.y; xr[2] = v.z; xr[3] = v.w;
    }
    __syncthreads();
    if (tid < nthr) {
      float2 acc[4][4];  // packed fp32x2 accumulators: columns 8 cg + 2 c, + 1
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[i][c] = make_float2(0.f, 0.f);
      const float *xa = Xs + rg * kEmbXStride;
      const float *ba = Bs + 8 * cg;
#pragma unroll 4
      for (int k = 0; k < kEmbIn; ++k) {
        const float4 b0 = *reinterpret_cast<const float4 *>(ba + k * p.mpad);
        const float4 b1 = *reinterpret_cast<const float4 *>(ba + k * p.mpad + 4);
        const float2 bb[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w), make_float2(b1.x, b1.y),
                              make_float2(b1.z, b1.w)};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float x = xa[16 * i * kEmbXStride + k];
          const float2 xx = make_float2(x, x);
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[i][c] = __ffma2_rn(xx, bb[c], acc[i][c]);
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = rg + 16 * i;
        if (r >= nr) continue;
        float *o = p.out + (size_t)(r0 + r) * p.ldx + 8 * cg;
        if (8 * cg + 8 <= p.m) {
          reinterpret_cast<float4 *>(o)[0] = make_float4(acc[i][0].x, acc[i][0].y, acc[i][1].x, acc[i][1].y);
          reinterpret_cast<float4 *>(o)[1] = make_float4(acc[i][2].x, acc[i][2].y, acc[i][3].x, acc[i][3].y);
        } else {
#pragma unroll
          for (int c = 0; c < 8; ++c)
            if (8 * cg + c < p.m) o[c] = (c & 1) ? acc[i][c >> 1].y : acc[i][c >> 1].x;
        }
      }
    }
    // normalised keypoint coordinates and zero padding: columns m .. ldx-1
    for (int r = tid; r < nr; r += 256) {
      const int64_t row = r0 + r;
      int lo = 0, hi = p.batch - 1;  // image of this row: last b with offsets[b] <= row
      while (lo < hi) { const int mid = (lo + hi + 1) >> 1; if (p.offsets[mid] <= row) lo = mid; else hi = mid - 1; }
      const float2 xy = reinterpret_cast<const float2 *>(p.xy)[row];
      const float2 wh = reinterpret_cast<const float2 *>(p.wh)[lo];
      float *o = p.out + (size_t)row * p.ldx;
      o[p.m] = xy.x / wh.x;
      o[p.m + 1] = xy.y / wh.y;
      for (int c = p.m + 2; c < p.ldx; ++c) o[c] = 0.f;
    }
  }
}

}  // namespace gpufv
