// k_stats.cuh — steps a2-a6 of the hot path in one persistent, warp-specialised kernel.
//
//   a2  X tile (128 descriptors x 64 dims, TMA 2-D, 128B-swizzled, 2-stage ring) -> the features
//       Z = [(x-c) 2^e, ((x-c) 2^e)^2] split into fp16 hi/lo, written TWICE into tensor memory:
//         Zr  lanes = descriptors, K = features    (A operand of GEMM1)
//         Zt  lanes = features,    K = descriptors (A operand of GEMM2)
//   a3  GEMM1  L[i,j] = Zr_i . W'_j   (tcgen05 TS-MMA, 3 x FP16 split: hi.lo + lo.hi + hi.hi, fp32 TMEM)
//       = log2 of the Alg.1 l.4-5 log-likelihood in expanded form, up to the bias b_j
//   a4  softmax epilogue: gamma_ij = 2^(L_ij + b_j - m_i) / s_i with the row max/sum reduced over the
//       CTA's 4 column quarters and over the cluster's Gaussian blocks (DSMEM st.async exchange)
//       (Alg.1 l.6-14); gamma <= tau zeroed (Alg.1 l.18); rows past the image end
//       masked; P = gamma 2^14 split fp16 hi/lo into shared memory; S0_j = sum_i gamma_ij in registers
//   a5  GEMM2  S'[f,j] += sum_i Zt[f,i] P[i,j]  (TS-MMA, 3 x FP16 split) — the U/V accumulation of
//       Alg.1 l.16-26 as moments; restarted every kFold tiles (the tensor-core fp32
//       accumulator truncates)
//   a6  every kFold tiles and at each (cluster, image) segment end: S' -> an append-only partial slot
//       in HBM; S0 -> an S0 slot at the segment end (the paper's per-block U/V copies)
//
// Roles (576 threads = 18 warps, 1 CTA per SM, cluster of C = ceil(K/128) CTAs, rank r owns Gaussians
// [128 r, 128 r + 128)):
//   warps 0-15  WORK: warp w = (q = w%4, h = w/4) owns TMEM lanes 32q.. (tcgen05.ld/st lane rule) and
//               a quarter h of everything else: softmax over Gaussian columns 32h.., the Zr features of
//               dims 16h.., the Zt descriptors 32h.., the fold of S' columns 32h..
//   warp  16    MMA : one thread issues every tcgen05.mma / commit
//   warp  17    TMA : one thread issues the X tile loads (stage freed by Zt) + L2 prefetches 4 tiles ahead
// (Registers: a block's warps are spread over the 4 SM sub-partitions of 16K registers each, so
//  ceil(warps / 4) * regs_per_thread <= 512 (measured: 88 regs -> 640 threads, 104 -> 512); 18 warps
//  can use 96 registers.)
// Per local tile i, WORK warps run: Zr(i+1) | softmax(i) | wait G2(i-1) | [fold] | Zt(i) | P(i), and
// the MMA thread issues G1(0), then G1(i+1), G2(i) for i = 0..n-1; so the tensor pipe runs G2(i-1)
// while Zr(i+1) and softmax(i) are computed and G1(i+1) while Zt(i) and P(i) are written.
#pragma once
#include <cuda.h>

#include "fv_common.cuh"
#include "ptx.cuh"

namespace gpufv {

constexpr int kWarpsWork = 16;
constexpr int kWarpMma = kWarpsWork, kWarpTma = kWarpsWork + 1;
constexpr int kThreads2 = (kWarpTma + 1) * 32;  // 576
constexpr int kMaxC2 = 4;                        // K <= 512 in this kernel

// shared memory map (offsets from a 1024-aligned base)
constexpr int kS2W = 0;                              // W' hi | lo            64 KB
constexpr int kS2P = kS2W + 2 * kOpBytes;            // P hi | lo             64 KB
constexpr int kS2X = kS2P + 2 * kOpBytes;            // X stage[2] x 32 KB    64 KB
constexpr int kXStageBytes = 2 * 128 * 128;          // two 32-float x 128-row boxes
constexpr int kS2Bias = kS2X + 2 * kXStageBytes;     // float[128]
constexpr int kS2Cs = kS2Bias + kG * 4;              // float[64]  c_k 2^e_k
constexpr int kS2Sc = kS2Cs + kDP * 4;               // float[64]  2^e_k
constexpr int kS2Red = kS2Sc + kDP * 4;              // float[2][4][128] (max, sum) per column quarter
constexpr int kS2Xchg = kS2Red + 2 * 4 * kTileM * 4; // float2[2][kMaxC2][128]
constexpr int kS2S0 = kS2Xchg + 2 * kMaxC2 * kTileM * 8;  // float[4][128]
constexpr int kS2Bar = kS2S0 + 4 * kG * 4;           // uint64 barriers
constexpr int kNumBars = 16;
constexpr int kS2Tmem = kS2Bar + kNumBars * 8;
constexpr int kSmem2Bytes = kS2Tmem + 16 + 1024;
static_assert(kSmem2Bytes <= 232448, "shared memory budget");

// barrier slots
enum : int {
  B_XFULL0 = 0, B_XFULL1, B_XEMPTY0, B_XEMPTY1, B_ZR_FULL, B_ZT_FULL, B_G1_DONE, B_G2_DONE,
  B_L_EMPTY, B_P_FULL, B_FOLD_DONE, B_XCHG0, B_XCHG1
};

// tensor-memory columns
constexpr uint32_t kTZr = 0, kTZt = 128, kTL = 256, kTS = 384;

struct Stats2Params {
  const float *X;             // n_total x D (also behind the tensor map; used for L2 prefetch)
  const int64_t *offsets;     // batch + 1
  const int64_t *tile_start;  // batch + 1
  const uint8_t *wimg;        // C x kWImgBytes
  const float *bias;          // Kp
  const float *xshift, *xscale;
  float *slots;               // fold slots: nslots x kNF x Kp   (feature-major rows)
  float *s0slots;             // (ncl + batch) x Kp
  float *gamma_out;
  int batch, D, K, Kp;
  float threshold;
  int gamma_mode;
};

struct TileInfo {  // per local tile
  int64_t row0, t;
  int b, nrows;
  bool seg_last, chunk_first, fold;  // GEMM2 restarts at this tile; fold after this tile
};

// Walks the cluster's tile range [t0, t1) in order; every role keeps its own copy.
struct TileWalker {
  const Stats2Params *p;
  int64_t t, t1;
  int b;
  int seg_pos;  // index of t within its (cluster, image) segment
  __device__ void init(const Stats2Params &pp, int64_t t0_, int64_t t1_) {
    p = &pp; t = t0_; t1 = t1_; b = 0; seg_pos = 0;
    if (t0_ < t1_) {
      int lo = 0, hi = pp.batch;
      while (lo < hi) { int mid = (lo + hi + 1) >> 1; if (pp.tile_start[mid] <= t0_) lo = mid; else hi = mid - 1; }
      b = lo;
      while (t >= pp.tile_start[b + 1]) ++b;
    }
  }
  __device__ TileInfo info() const {
    TileInfo ti;
    ti.t = t;
    ti.b = b;
    const int64_t ib = p->tile_start[b];
    ti.row0 = p->offsets[b] + (t - ib) * kTileM;
    const int64_t rem = p->offsets[b + 1] - ti.row0;
    ti.nrows = rem < kTileM ? (int)rem : kTileM;
    ti.seg_last = (t + 1 == t1) || (t + 1 >= p->tile_start[b + 1]);
    ti.chunk_first = (seg_pos % kFold) == 0;
    ti.fold = ti.seg_last || ((seg_pos + 1) % kFold == 0);
    return ti;
  }
  __device__ void next() {
    const bool last = (t + 1 >= p->tile_start[b + 1]);
    ++t;
    if (last) { seg_pos = 0; if (t < t1) while (t >= p->tile_start[b + 1]) ++b; }
    else ++seg_pos;
  }
};

// 16-byte chunk c (4 floats) of row r in a 128B-swizzled 32-float box
__device__ __forceinline__ uint32_t xs_off(int r, int c) { return r * 128 + ((c ^ (r & 7)) << 4); }

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, int c0, int64_t c1, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"((int)c1), "r"(ptx::smem_u32(bar))
      : "memory");
}

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

__global__ void __launch_bounds__(kThreads2, 1) k_stats(const __grid_constant__ CUtensorMap tmap_x, const Stats2Params p) {
  using namespace ptx;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_base = smem_u32(smem_raw);
  const uint32_t sbase = (raw_base + 1023u) & ~1023u;
  uint8_t *smem = smem_raw + (sbase - raw_base);
  const uint32_t sW = sbase + kS2W, sP = sbase + kS2P, sX = sbase + kS2X;
  float *s_bias = reinterpret_cast<float *>(smem + kS2Bias);
  float *s_cs = reinterpret_cast<float *>(smem + kS2Cs);
  float *s_sc = reinterpret_cast<float *>(smem + kS2Sc);
  float *s_red = reinterpret_cast<float *>(smem + kS2Red);
  float2 *s_xchg = reinterpret_cast<float2 *>(smem + kS2Xchg);
  float *s_s0 = reinterpret_cast<float *>(smem + kS2S0);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + kS2Bar);
  uint32_t *s_tmem = reinterpret_cast<uint32_t *>(smem + kS2Tmem);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_ctarank(), C = cluster_nctarank();
  const int cid = (int)cluster_id_x(), ncl = (int)nclusters_x();

  // ---------------- setup
  {
    const uint4 *src = reinterpret_cast<const uint4 *>(p.wimg + (size_t)rank * kWImgBytes);
    uint4 *dst = reinterpret_cast<uint4 *>(smem + kS2W);
    for (int i = tid; i < kWImgBytes / 16; i += kThreads2) dst[i] = __ldg(src + i);
    for (int i = tid; i < kG; i += kThreads2) s_bias[i] = p.bias[rank * kG + i];
    if (tid < kDP) { s_sc[tid] = p.xscale[tid]; s_cs[tid] = p.xshift[tid] * p.xscale[tid]; }
  }
  if (warp == 0) { tmem_alloc(s_tmem, kTmemCols); tmem_relinquish(); }
  if (tid == 0) {
    mbar_init(&bars[B_XFULL0], 1); mbar_init(&bars[B_XFULL1], 1);
    mbar_init(&bars[B_XEMPTY0], kWarpsWork); mbar_init(&bars[B_XEMPTY1], kWarpsWork);
    mbar_init(&bars[B_ZR_FULL], kWarpsWork); mbar_init(&bars[B_ZT_FULL], kWarpsWork);
    mbar_init(&bars[B_G1_DONE], 1); mbar_init(&bars[B_G2_DONE], 1);
    mbar_init(&bars[B_L_EMPTY], kWarpsWork); mbar_init(&bars[B_P_FULL], kWarpsWork);
    mbar_init(&bars[B_FOLD_DONE], kWarpsWork);
    mbar_init(&bars[B_XCHG0], 1); mbar_init(&bars[B_XCHG1], 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  cluster_sync();

  const int64_t T = p.tile_start[p.batch];
  const int64_t t0 = (int64_t)cid * T / ncl, t1 = (int64_t)(cid + 1) * T / ncl;
  const int n = (int)(t1 - t0);
  TileWalker tw;
  tw.init(p, t0, t1);

  if (warp == kWarpTma) {
    // ======================================================= X producer (TMA)
    if (lane == 0 && n > 0) {
      const int Dv = p.D;
      TileWalker twp = tw;  // L2-prefetch walker, 4 tiles ahead
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_x)) : "memory");
      auto prefetch_l2 = [&](int i) {
        if (i >= n) return;
        const TileInfo ti = twp.info();
        twp.next();
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p.X + ti.row0 * Dv),
                     "r"((uint32_t)(ti.nrows * Dv * 4) & ~15u)
                     : "memory");
      };
      for (int i = 0; i < 4; ++i) prefetch_l2(i);
      for (int i = 0; i < n; ++i, tw.next()) {
        const TileInfo ti = tw.info();
        const int s = i & 1;
        if (i >= 2) {  // stage s is free once Zt(i-2) has been written by every WORK warp
          mbar_wait(&bars[B_XEMPTY0 + s], ((i >> 1) - 1) & 1);
          prefetch_l2(i + 2);
        }
        mbar_arrive_expect_tx(&bars[B_XFULL0 + s], kXStageBytes);
        tma_load_2d(sX + s * kXStageBytes, &tmap_x, 0, ti.row0, &bars[B_XFULL0 + s]);
        tma_load_2d(sX + s * kXStageBytes + 128 * 128, &tmap_x, 32, ti.row0, &bars[B_XFULL0 + s]);
      }
    }
  } else if (warp == kWarpMma) {
    // ======================================================= MMA issuer
    if (lane == 0 && n > 0) {
      const uint32_t idesc1 = idesc_f16_f32(128, kG, 0, 0);   // A = Zr (TMEM, K-major), B = W' K-major
      const uint32_t idesc2 = idesc_f16_f32(kNF, kG, 0, 1);   // A = Zt (TMEM, K-major), B = P MN-major
      uint32_t folds = 0;
      auto gemm1 = [&](int i) {
        mbar_wait(&bars[B_ZR_FULL], i & 1);
        if (i >= 1) mbar_wait(&bars[B_L_EMPTY], (i - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int s = 0; s < 3; ++s) {  // cross terms first, hi.hi last (truncating accumulator)
          const uint32_t za = tmem + kTZr + (s == 1 ? 64 : 0);   // hi, lo, hi
          const uint32_t wb = sW + (s == 0 ? kOpBytes : 0);      // lo, hi, hi
#pragma unroll
          for (int kk = 0; kk < kNF / 16; ++kk) {
            const uint32_t off = (kk >> 2) * kAtomBytes + (kk & 3) * 32;
            mma_f16_ts(tmem + kTL, za + kk * 8, desc_sw128(wb + off, 16, 1024), idesc1, (s | kk) != 0);
          }
        }
        mma_commit(&bars[B_G1_DONE]);
      };
      auto gemm2 = [&](int i, const TileInfo &ti) {
        mbar_wait(&bars[B_ZT_FULL], i & 1);
        mbar_wait(&bars[B_P_FULL], i & 1);
        if (ti.chunk_first && i > 0) { mbar_wait(&bars[B_FOLD_DONE], folds & 1); ++folds; }
        tc_fence_after();
#pragma unroll
        for (int s = 0; s < 3; ++s) {
          const uint32_t za = tmem + kTZt + (s == 1 ? 64 : 0);   // hi, lo, hi
          const uint32_t pb = sP + (s == 0 ? kOpBytes : 0);      // lo, hi, hi
#pragma unroll
          for (int kk = 0; kk < kTileM / 16; ++kk)
            mma_f16_ts(tmem + kTS, za + kk * 8, desc_sw128(pb + kk * 2048, kAtomBytes, 1024), idesc2,
                       (ti.chunk_first && s == 0 && kk == 0) ? 0u : 1u);
        }
        mma_commit(&bars[B_G2_DONE]);
      };
      gemm1(0);
      for (int i = 0; i < n; ++i, tw.next()) {
        const TileInfo ti = tw.info();
        if (i + 1 < n) gemm1(i + 1);
        gemm2(i, ti);
      }
    }
  } else {
    // ======================================================= WORK warps
    const int q = warp & 3, h = warp >> 2;  // TMEM lanes 32q.. ; quarter h
    const uint32_t lane_base = (uint32_t)(32 * q) << 16;
    const int row = 32 * q + lane;  // descriptor row of Zr / L / P; feature of Zt / S'
    const int D = p.D;
    const float thr = p.threshold * kPScale;
    float *red_m = s_red, *red_s = s_red + 4 * kTileM;

    // Zr quarter: row `row`, dims [16h, 16h+16) -> linear hi cols 8h.., quadratic hi cols 32+8h.., lo + 64
    auto conv_rows = [&](int i, const TileInfo &ti) {
      const int s = i & 1;
      mbar_wait(&bars[B_XFULL0 + s], (i >> 1) & 1);
      if (i >= 1) mbar_wait(&bars[B_G1_DONE], (i - 1) & 1);  // GEMM1(i-1) no longer reads Zr
      tc_fence_after();
      const uint8_t *xs = smem + kS2X + s * kXStageBytes + (h >> 1) * 16384;
      const bool valid = row < ti.nrows;
      uint32_t lh[8], ll[8], qh[8], ql[8];
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4) {
        const float4 v = *reinterpret_cast<const float4 *>(xs + xs_off(row, 4 * (h & 1) + c4));
        const float xv[4] = {v.x, v.y, v.z, v.w};
        float a[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int k = 16 * h + 4 * c4 + e;
          a[e] = (valid && k < D) ? fmaf(xv[e], s_sc[k], -s_cs[k]) : 0.f;
        }
        split2_f16(a[0], a[1], lh[2 * c4], ll[2 * c4]);
        split2_f16(a[2], a[3], lh[2 * c4 + 1], ll[2 * c4 + 1]);
        split2_f16(a[0] * a[0], a[1] * a[1], qh[2 * c4], ql[2 * c4]);
        split2_f16(a[2] * a[2], a[3] * a[3], qh[2 * c4 + 1], ql[2 * c4 + 1]);
      }
      tmem_st8(tmem + kTZr + lane_base + 8 * h, lh);
      tmem_st8(tmem + kTZr + lane_base + 32 + 8 * h, qh);
      tmem_st8(tmem + kTZr + lane_base + 64 + 8 * h, ll);
      tmem_st8(tmem + kTZr + lane_base + 96 + 8 * h, ql);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[B_ZR_FULL]);
    };
    // Zt quarter: feature f = row (k = f % 64, squared if f >= 64), descriptors [32h, 32h+32)
    auto conv_feats = [&](int i, const TileInfo &ti) {
      const int s = i & 1;
      const int k = row & 63;
      const uint8_t *xs = smem + kS2X + s * kXStageBytes + (k >> 5) * 16384;
      const bool sq = row >= 64, kval = k < D;
      const float sc = s_sc[k], cs = s_cs[k];
      const int kc = (k & 31) >> 2, ke = k & 3;
#pragma unroll
      for (int blk = 0; blk < 2; ++blk) {  // 16 descriptors -> 8 columns hi + 8 lo
        uint32_t hi[8], lo[8];
#pragma unroll
        for (int pr = 0; pr < 8; ++pr) {
          float a2[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = 32 * h + 16 * blk + 2 * pr + e;
            const float xv = *reinterpret_cast<const float *>(xs + xs_off(r, kc) + 4 * ke);
            const float a = (kval && r < ti.nrows) ? fmaf(xv, sc, -cs) : 0.f;
            a2[e] = sq ? a * a : a;
          }
          split2_f16(a2[0], a2[1], hi[pr], lo[pr]);
        }
        tmem_st8(tmem + kTZt + lane_base + 16 * h + 8 * blk, hi);
        tmem_st8(tmem + kTZt + lane_base + 64 + 16 * h + 8 * blk, lo);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) { mbar_arrive(&bars[B_ZT_FULL]); mbar_arrive(&bars[B_XEMPTY0 + s]); }
    };
    // fold quarter: S' (lane = feature `row`, Gaussian columns [32h, 32h+32)) -> append-only slot
    auto fold = [&](const TileInfo &ti, int64_t chunk_start) {
      float *dst = p.slots + (size_t)fold_slot(chunk_start, cid, ti.b) * kNF * p.Kp + (size_t)row * p.Kp + rank * kG +
                   32 * h;
      uint32_t v[32];
      tmem_ld32(tmem + kTS + lane_base + 32 * h, v);
      tmem_ld_wait();
      float4 *d4 = reinterpret_cast<float4 *>(dst);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        d4[j] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]), __uint_as_float(v[4 * j + 2]),
                            __uint_as_float(v[4 * j + 3]));
    };

    float s0acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) s0acc[j] = 0.f;
    TileWalker twr = tw;  // Zr walker, one tile ahead
    int64_t chunk_start = t0;
    TileInfo prev{};
    if (n > 0) { conv_rows(0, twr.info()); twr.next(); }
    for (int i = 0; i < n; ++i, tw.next()) {
      const TileInfo ti = tw.info();
      if (i + 1 < n) { conv_rows(i + 1, twr.info()); twr.next(); }

      // ---- softmax(i): L row quarter -> e = 2^(L + b - m), row sum, cluster combine
      mbar_wait(&bars[B_G1_DONE], i & 1);
      tc_fence_after();
      float v[32];
      {
        uint32_t rr[32];
        tmem_ld32(tmem + kTL + lane_base + 32 * h, rr);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(rr[j]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[B_L_EMPTY]);
      float m = -3.0e38f;
#pragma unroll
      for (int j = 0; j < 32; ++j) { v[j] += s_bias[32 * h + j]; m = fmaxf(m, v[j]); }
      if (p.gamma_mode == 2 && row < ti.nrows) {
        float *go = p.gamma_out + (ti.row0 + row) * (int64_t)p.K;
#pragma unroll
        for (int j = 0; j < 32; ++j) { int gj = rank * kG + 32 * h + j; if (gj < p.K) go[gj] = v[j]; }
      }
      red_m[h * kTileM + row] = m;
      named_bar_sync(1 + q, 128);
      m = fmaxf(fmaxf(red_m[row], red_m[kTileM + row]), fmaxf(red_m[2 * kTileM + row], red_m[3 * kTileM + row]));
      float s = 0.f;
#pragma unroll
      for (int j = 0; j < 32; ++j) { v[j] = ex2_approx(v[j] - m); s += v[j]; }
      red_s[h * kTileM + row] = s;
      named_bar_sync(1 + q, 128);
      s = (red_s[row] + red_s[kTileM + row]) + (red_s[2 * kTileM + row] + red_s[3 * kTileM + row]);
      float alpha;
      if (C > 1) {
        const int par = i & 1;
        float2 *xb = s_xchg + par * (kMaxC2 * kTileM);
        if (warp == 0 && lane == 0) mbar_arrive_expect_tx(&bars[B_XCHG0 + par], (C - 1) * kTileM * 8);
        if (h == 0) {
          const uint32_t my = smem_u32(&xb[rank * kTileM + row]);
          const uint32_t mybar = smem_u32(&bars[B_XCHG0 + par]);
          for (uint32_t r2 = 0; r2 < C; ++r2)
            if (r2 != rank) st_async_v2f32(mapa_shared(my, r2), m, s, mapa_shared(mybar, r2));
        }
        mbar_wait(&bars[B_XCHG0 + par], (i >> 1) & 1);
        float M = m;
        for (uint32_t r2 = 0; r2 < C; ++r2) if (r2 != rank) M = fmaxf(M, xb[r2 * kTileM + row].x);
        float S = s * ex2_approx(m - M);
        for (uint32_t r2 = 0; r2 < C; ++r2)
          if (r2 != rank) { const float2 o = xb[r2 * kTileM + row]; S += o.y * ex2_approx(o.x - M); }
        alpha = ex2_approx(m - M) / S;
      } else {
        alpha = 1.f / s;
      }
      if (row >= ti.nrows) alpha = 0.f;
      const float alpha_p = alpha * kPScale;  // P = gamma 2^14

      // ---- GEMM2(i-1) done: S' chunk complete (fold), Zt and P free
      if (i >= 1) {
        mbar_wait(&bars[B_G2_DONE], (i - 1) & 1);
        tc_fence_after();
        if (prev.fold) {
          fold(prev, chunk_start);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bars[B_FOLD_DONE]);
        }
      }
      if (ti.chunk_first) chunk_start = ti.t;
      conv_feats(i, ti);

      // ---- P(i) = gamma 2^14 (thresholded) -> fp16 hi/lo, S0 accumulation
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int e = 0; e < 8; e += 2) {
          float g0 = v[8 * c + e] * alpha_p, g1 = v[8 * c + e + 1] * alpha_p;
          if (thr > 0.f) { g0 = (g0 > thr) ? g0 : 0.f; g1 = (g1 > thr) ? g1 : 0.f; }
          v[8 * c + e] = g0; v[8 * c + e + 1] = g1;
          s0acc[8 * c + e] += g0; s0acc[8 * c + e + 1] += g1;
          split2_f16(g0, g1, hi[e >> 1], lo[e >> 1]);
        }
        const uint32_t off = (h >> 1) * kAtomBytes + row * 128 + (((4 * (h & 1) + c) ^ (row & 7)) << 4);
        sts128(sP + off, hi[0], hi[1], hi[2], hi[3]);
        sts128(sP + kOpBytes + off, lo[0], lo[1], lo[2], lo[3]);
      }
      if (p.gamma_mode == 1 && row < ti.nrows) {
        float *go = p.gamma_out + (ti.row0 + row) * (int64_t)p.K;
#pragma unroll
        for (int j = 0; j < 32; ++j) { int gj = rank * kG + 32 * h + j; if (gj < p.K) go[gj] = v[j] * (1.f / kPScale); }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[B_P_FULL]);
      if (ti.seg_last) {  // S0 of the segment (units of 2^14 gamma) -> s0 slot (cid + b)
        warp_transpose_reduce32(s0acc, lane);
        s_s0[q * kG + 32 * h + lane] = s0acc[0];
#pragma unroll
        for (int j = 0; j < 32; ++j) s0acc[j] = 0.f;
        named_bar_sync(5, kWarpsWork * 32);
        if (tid < kG)
          p.s0slots[(size_t)(cid + ti.b) * p.Kp + rank * kG + tid] =
              (s_s0[tid] + s_s0[kG + tid]) + (s_s0[2 * kG + tid] + s_s0[3 * kG + tid]);
        named_bar_sync(5, kWarpsWork * 32);
      }
      prev = ti;
    }
    if (n > 0) {  // last chunk
      mbar_wait(&bars[B_G2_DONE], (n - 1) & 1);
      tc_fence_after();
      fold(prev, chunk_start);
    }
  }

  // ---------------- teardown
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) tmem_dealloc(tmem, kTmemCols);
}

}  // namespace gpufv
