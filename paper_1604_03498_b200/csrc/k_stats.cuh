// k_stats.cuh — steps a2-a6 of the hot path in one persistent kernel:
//   a2  X tile (128 descriptors) -> Z = [(x-c) 2^e, ((x-c) 2^e)^2] split into fp16 hi/lo (SMEM, SW128)
//   a3  GEMM1 on tcgen05:  L[i,j] = Z_i . W'_j  (3 x FP16 split: hi.hi + hi.lo + lo.hi, fp32 in TMEM)
//       -- the log-likelihood of Alg.1 l.4-5 in expanded form, log2 units --
//   a4  softmax epilogue:  gamma_ij = 2^(L_ij + b_j - m_i) / s_i, max/sum over the cluster's Gaussian
//       blocks exchanged through DSMEM (Alg.1 l.6-14); gamma <= tau zeroed (Alg.1 l.18,
//       P:177); rows past the image end masked to 0
//   a5  GEMM2 on tcgen05:  S'[f,j] += sum_i Z[i,f] P[i,j]  (P = gamma 2^14, 3 x FP16 split) — the
//       U/V accumulation of Alg.1 l.16-26 as moments, accumulated in TMEM across the
//       tiles of one image; S0_j = sum_i gamma_ij accumulated in registers
//   a6  at the end of each (cluster, image) segment: S' and S0 -> one partial slot in HBM (the
//       paper's "one copy of U and V for each block")
//
// Geometry: cluster of C = ceil(K/128) CTAs; CTA rank r owns Gaussians [128 r, 128 r + 128).  All
// CTAs of a cluster walk the same tiles.  Clusters own contiguous ranges of the global tile list
// (static schedule => deterministic).  256 threads; 1 CTA per SM (~214 KB SMEM, 512 TMEM columns).
#pragma once
#include "fv_common.cuh"
#include "ptx.cuh"

namespace gpufv {

struct StatsParams {
  const float *X;           // n_total x D
  const int64_t *offsets;   // batch + 1
  const int64_t *tile_start;// batch + 1 (k_schedule)
  const uint8_t *wimg;      // C x kWImgBytes prepared W' images
  const float *bias;        // Kp (log2 units; -1e30 for padded Gaussians)
  const float *xshift;      // kDP
  const float *xscale;      // kDP
  float *partials;          // nslots x (1 + kNF) x Kp
  float *gamma_out;         // optional N x K debug/test output (fv_posteriors)
  int batch, D, K, Kp;
  float threshold;          // <= 0: exact mode
  int gamma_mode;           // 0: none, 1: gamma, 2: raw L + b (log2 units)
};

__device__ __forceinline__ void warp_transpose_reduce32(float (&a)[32], int lane) {
  // After the call, a[0] on lane l holds sum over all lanes of the input a[l].
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const bool upper = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < off; ++i) {
      float send = upper ? a[i] : a[i + off];
      float keep = upper ? a[i + off] : a[i];
      a[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1) k_stats(const StatsParams p) {
  using namespace ptx;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_base = smem_u32(smem_raw);
  const uint32_t sbase = (raw_base + 1023u) & ~1023u;
  uint8_t *smem = smem_raw + (sbase - raw_base);

  const uint32_t sW = sbase + kSmW, sZ = sbase + kSmZ, sP = sbase + kSmP;
  float *s_bias = reinterpret_cast<float *>(smem + kSmBias);
  float *s_xshift = reinterpret_cast<float *>(smem + kSmXShift);
  float *s_xscale = reinterpret_cast<float *>(smem + kSmXScale);
  float *s_redm = reinterpret_cast<float *>(smem + kSmRedM);
  float *s_reds = reinterpret_cast<float *>(smem + kSmRedS);
  float2 *s_xchg = reinterpret_cast<float2 *>(smem + kSmXchg);
  float *s_s0red = reinterpret_cast<float *>(smem + kSmS0Red);
  uint64_t *s_bar = reinterpret_cast<uint64_t *>(smem + kSmBar);
  uint32_t *s_tmem = reinterpret_cast<uint32_t *>(smem + kSmTmemSlot);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_ctarank(), C = cluster_nctarank();
  const uint32_t cid = cluster_id_x(), ncl = nclusters_x();

  // ---------------- one-time setup: W' image of this rank, bias, feature shift/scale, TMEM, barriers
  {
    const uint4 *src = reinterpret_cast<const uint4 *>(p.wimg + (size_t)rank * kWImgBytes);
    uint4 *dst = reinterpret_cast<uint4 *>(smem + kSmW);
    for (int i = tid; i < kWImgBytes / 16; i += kThreads) dst[i] = __ldg(src + i);
    for (int i = tid; i < kG; i += kThreads) s_bias[i] = p.bias[rank * kG + i];
    if (tid < kDP) { s_xshift[tid] = p.xshift[tid]; s_xscale[tid] = p.xscale[tid]; }
  }
  if (warp == 0) { tmem_alloc(s_tmem, kTmemCols); tmem_relinquish(); }
  if (tid == 0) { mbar_init(&s_bar[0], 1); mbar_init(&s_bar[1], 1); fence_mbar_init(); }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  const uint32_t tL = tmem + kTmemL, tS = tmem + kTmemS, tStot = tmem + kTmemSTot;
  cluster_sync();  // every CTA of the cluster is resident before any DSMEM traffic

  const int64_t T = p.tile_start[p.batch];
  const int64_t t0 = (int64_t)cid * T / ncl, t1 = (int64_t)(cid + 1) * T / ncl;

  const int q = warp & 3, h = warp >> 2, row = 32 * q + lane;  // epilogue role: row, column half
  const uint32_t idesc1 = idesc_f16_f32(128, kG, 0, 0);         // A=Z K-major, B=W' K-major
  const uint32_t idesc2 = idesc_f16_f32(kNF, kG, 1, 1);         // A=Z^T MN-major, B=P MN-major
  const float thr = p.threshold;

  float s0acc[64];
#pragma unroll
  for (int j = 0; j < 64; ++j) s0acc[j] = 0.f;

  uint32_t ph1 = 0, ph2 = 0, xpar = 0;
  bool pending2 = false, seg_first = true, tot_valid = false;
  int chunk_tiles = 0;

  int b = 0;
  if (t0 < t1) {  // last b with tile_start[b] <= t0 (skips empty images)
    int lo = 0, hi = p.batch;
    while (lo < hi) { int mid = (lo + hi + 1) >> 1; if (p.tile_start[mid] <= t0) lo = mid; else hi = mid - 1; }
    b = lo;
  }

  for (int64_t t = t0; t < t1; ++t) {
    while (t >= p.tile_start[b + 1]) ++b;
    const int64_t img_lo = p.offsets[b], img_hi = p.offsets[b + 1];
    const int64_t row0 = img_lo + (t - p.tile_start[b]) * kTileM;
    const int nrows = (img_hi - row0 < kTileM) ? (int)(img_hi - row0) : kTileM;

    // previous GEMM2 still reads Z and P
    if (pending2) { mbar_wait(&s_bar[1], ph2); ph2 ^= 1; pending2 = false; }

    // ---------------- a2: Z tile (fp16 hi/lo, SW128 K-major rows)
#pragma unroll
    for (int it = 0; it < (kTileM * 8) / kThreads; ++it) {
      const int item = it * kThreads + tid;
      const int r = item >> 3, c = item & 7;  // row, 16-byte chunk (8 features)
      float x[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) x[e] = 0.f;
      if (r < nrows) {
        const float *xr = p.X + (row0 + r) * (int64_t)p.D;
        if (8 * c + 4 <= p.D) { float4 v = __ldg(reinterpret_cast<const float4 *>(xr + 8 * c)); x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w; }
        if (8 * c + 8 <= p.D) { float4 v = __ldg(reinterpret_cast<const float4 *>(xr + 8 * c + 4)); x[4] = v.x; x[5] = v.y; x[6] = v.z; x[7] = v.w; }
      }
      uint32_t lh[4], ll[4], qh[4], ql[4];
#pragma unroll
      for (int e = 0; e < 8; e += 2) {
        const int k = 8 * c + e;
        float a0 = (k < p.D && r < nrows) ? (x[e] - s_xshift[k]) * s_xscale[k] : 0.f;
        float a1 = (k + 1 < p.D && r < nrows) ? (x[e + 1] - s_xshift[k + 1]) * s_xscale[k + 1] : 0.f;
        split2_f16(a0, a1, lh[e >> 1], ll[e >> 1]);
        split2_f16(a0 * a0, a1 * a1, qh[e >> 1], ql[e >> 1]);
      }
      const uint32_t off = r * 128 + ((c ^ (r & 7)) << 4);
      sts128(sZ + off, lh[0], lh[1], lh[2], lh[3]);                              // hi, atom 0 (linear)
      sts128(sZ + kAtomBytes + off, qh[0], qh[1], qh[2], qh[3]);                 // hi, atom 1 (square)
      sts128(sZ + kOpBytes + off, ll[0], ll[1], ll[2], ll[3]);                   // lo, atom 0
      sts128(sZ + kOpBytes + kAtomBytes + off, ql[0], ql[1], ql[2], ql[3]);      // lo, atom 1
    }
    fence_proxy_async_smem();
    __syncthreads();

    // ---------------- a3: GEMM1 (one thread issues 3 x 8 UMMAs, K = 16 features each)
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        // Cross terms first, hi.hi last: the tensor-core accumulator truncates, so the big term
        // should meet as few accumulate steps as possible (emulation: 4.8e-6 -> 1.6e-6 gamma error).
        const uint32_t za = sZ + (s == 1 ? kOpBytes : 0);  // hi, lo, hi
        const uint32_t wb = sW + (s == 0 ? kOpBytes : 0);  // lo, hi, hi
#pragma unroll
        for (int kk = 0; kk < kNF / 16; ++kk) {
          const uint32_t off = (kk >> 2) * kAtomBytes + (kk & 3) * 32;
          mma_f16_ss(tL, desc_sw128(za + off, 16, 1024), desc_sw128(wb + off, 16, 1024), idesc1,
                     (s | kk) != 0);
        }
      }
      mma_commit(&s_bar[0]);
    }

    // ---------------- a4: softmax / threshold epilogue (thread = descriptor row, 64 Gaussians)
    mbar_wait(&s_bar[0], ph1);
    ph1 ^= 1;
    tc_fence_after();
    float v[64];
    {
      uint32_t r0[32], r1[32];
      const uint32_t ta = tL + ((uint32_t)(32 * q) << 16) + 64 * h;
      tmem_ld32(ta, r0);
      tmem_ld32(ta + 32, r1);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) { v[j] = __uint_as_float(r0[j]); v[32 + j] = __uint_as_float(r1[j]); }
    }
    float m = -3.0e38f;
#pragma unroll
    for (int j = 0; j < 64; ++j) { v[j] += s_bias[64 * h + j]; m = fmaxf(m, v[j]); }
    if (p.gamma_mode == 2 && row < nrows) {
      float *go = p.gamma_out + (row0 + row) * (int64_t)p.K;
#pragma unroll
      for (int j = 0; j < 64; ++j) { int gj = rank * kG + 64 * h + j; if (gj < p.K) go[gj] = v[j]; }
    }
    s_redm[h * kTileM + row] = m;
    __syncthreads();
    m = fmaxf(s_redm[row], s_redm[kTileM + row]);
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 64; ++j) { v[j] = ex2_approx(v[j] - m); s += v[j]; }
    s_reds[h * kTileM + row] = s;
    __syncthreads();
    s = s_reds[row] + s_reds[kTileM + row];
    float alpha;
    if (C > 1) {
      float2 *xb = s_xchg + xpar * (kMaxCluster * kTileM);
      if (h == 0) {
        const uint32_t my = smem_u32(&xb[rank * kTileM + row]);
        for (uint32_t r2 = 0; r2 < C; ++r2)
          if (r2 != rank) st_cluster_v2f32(mapa_shared(my, r2), m, s);
      }
      cluster_sync();
      float M = m;
      for (uint32_t r2 = 0; r2 < C; ++r2) if (r2 != rank) M = fmaxf(M, xb[r2 * kTileM + row].x);
      float S = s * ex2_approx(m - M);
      for (uint32_t r2 = 0; r2 < C; ++r2)
        if (r2 != rank) { float2 o = xb[r2 * kTileM + row]; S += o.y * ex2_approx(o.x - M); }
      alpha = ex2_approx(m - M) / S;
      xpar ^= 1;
    } else {
      alpha = 1.f / s;
    }
    if (row >= nrows) alpha = 0.f;  // rows past the image end contribute nothing
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      uint32_t hi[4], lo[4];
#pragma unroll
      for (int e = 0; e < 8; e += 2) {
        float g0 = v[8 * c + e] * alpha, g1 = v[8 * c + e + 1] * alpha;
        if (thr > 0.f) { g0 = (g0 > thr) ? g0 : 0.f; g1 = (g1 > thr) ? g1 : 0.f; }
        v[8 * c + e] = g0; v[8 * c + e + 1] = g1;
        s0acc[8 * c + e] += g0; s0acc[8 * c + e + 1] += g1;
        split2_f16(g0 * kPScale, g1 * kPScale, hi[e >> 1], lo[e >> 1]);
      }
      const uint32_t off = h * kAtomBytes + row * 128 + ((c ^ (row & 7)) << 4);
      sts128(sP + off, hi[0], hi[1], hi[2], hi[3]);
      sts128(sP + kOpBytes + off, lo[0], lo[1], lo[2], lo[3]);
    }
    if (p.gamma_mode == 1 && row < nrows) {
      float *go = p.gamma_out + (row0 + row) * (int64_t)p.K;
#pragma unroll
      for (int j = 0; j < 64; ++j) { int gj = rank * kG + 64 * h + j; if (gj < p.K) go[gj] = v[j]; }
    }
    tc_fence_before();
    fence_proxy_async_smem();
    __syncthreads();

    // ---------------- a5: GEMM2  S'[f, j] += sum_i Z[i, f] P[i, j]   (M = features, K = descriptors)
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int s2 = 0; s2 < 3; ++s2) {
        const uint32_t za = sZ + (s2 == 1 ? kOpBytes : 0);  // hi, lo, hi (cross terms first)
        const uint32_t pb = sP + (s2 == 0 ? kOpBytes : 0);  // lo, hi, hi
#pragma unroll
        for (int kk = 0; kk < kTileM / 16; ++kk) {
          const uint32_t off = kk * 2048;  // 16 rows x 128 B
          mma_f16_ss(tS, desc_sw128(za + off, kAtomBytes, 1024), desc_sw128(pb + off, kAtomBytes, 1024),
                     idesc2, (seg_first && s2 == 0 && kk == 0) ? 0u : 1u);
        }
      }
      mma_commit(&s_bar[1]);
    }
    pending2 = true;
    seg_first = false;
    ++chunk_tiles;

    // ---------------- a6: fold the GEMM2 chunk every kFoldTiles tiles; flush at the segment end
    const bool seg_end = (t + 1 == t1) || (t + 1 >= p.tile_start[b + 1]);
    if (seg_end || chunk_tiles == kFoldTiles) {
      mbar_wait(&s_bar[1], ph2); ph2 ^= 1; pending2 = false;
      tc_fence_after();
      // thread: lane = feature f = row, columns [64h, 64h + 64) in two halves of 32
      float *slot = p.partials + (size_t)(cid + b) * (1 + kNF) * p.Kp;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const uint32_t lane_col = ((uint32_t)(32 * q) << 16) + 64 * h + 32 * half;
        uint32_t ra[32], rt[32];
        tmem_ld32(tS + lane_col, ra);
        if (tot_valid) tmem_ld32(tStot + lane_col, rt);
        tmem_ld_wait();
        if (tot_valid) {
#pragma unroll
          for (int j = 0; j < 32; ++j) ra[j] = __float_as_uint(__uint_as_float(ra[j]) + __uint_as_float(rt[j]));
        }
        if (seg_end) {
          float4 *dst = reinterpret_cast<float4 *>(slot + (size_t)(1 + row) * p.Kp + rank * kG + 64 * h + 32 * half);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            dst[j] = make_float4(__uint_as_float(ra[4 * j]), __uint_as_float(ra[4 * j + 1]),
                                 __uint_as_float(ra[4 * j + 2]), __uint_as_float(ra[4 * j + 3]));
        } else {
          tmem_st32(tStot + lane_col, ra);
        }
      }
      if (!seg_end) tmem_st_wait();
      tot_valid = !seg_end;
      chunk_tiles = 0;
      seg_first = true;  // next GEMM2 starts a fresh chunk (accumulate = 0)
      if (seg_end) {  // S0: column sums of gamma over the 128 rows
        float a[32];
#pragma unroll
        for (int half = 0; half < 2; ++half) {
#pragma unroll
          for (int j = 0; j < 32; ++j) a[j] = s0acc[32 * half + j];
          warp_transpose_reduce32(a, lane);
          s_s0red[q * kG + 64 * h + 32 * half + lane] = a[0];
        }
#pragma unroll
        for (int j = 0; j < 64; ++j) s0acc[j] = 0.f;
      }
      tc_fence_before();
      __syncthreads();
      if (seg_end && tid < kG)
        slot[rank * kG + tid] = s_s0red[tid] + s_s0red[kG + tid] + s_s0red[2 * kG + tid] + s_s0red[3 * kG + tid];
    }
  }

  // ---------------- teardown
  if (pending2) { mbar_wait(&s_bar[1], ph2); }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) tmem_dealloc(tmem, kTmemCols);
}

}  // namespace gpufv
