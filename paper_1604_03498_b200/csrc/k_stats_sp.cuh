// k_stats_sp.cuh — the thresholded (tau > 0) statistics path with Alg. 5's early termination
// ("early termination ... because there are many small
// posterior values", Alg.5): only the (descriptor, Gaussian) pairs with gamma > tau enter the
// first- and second-order sums, so instead of the dense GEMM2 over every pair the surviving pairs are
// accumulated on the CUDA cores.  Narrow family only (D <= 64, K <= 256, clusters of <= 2 CTAs).
//
// Steps a2-a4 are k_stats's (same TMA boxes, fp16 hi/lo feature split into TMEM, GEMM1 on tcgen05 with
// the 3-way split, online softmax with the cluster (m, s) exchange).  What replaces a5:
//   a4'  each WORK thread (one descriptor row x 32 Gaussians) writes gamma 2^14 of its 32 columns into
//        Gamma (shared, fp32, 128 rows x 128 Gaussians) and the survivor bits gamma > tau; a 32 x 32 bit
//        transpose across the warp turns them into per-Gaussian row masks (mask[j][q], bit r = row 32q+r)
//   a5'  warp w owns Gaussians 8w .. 8w+7 of this CTA, lane l the dims 2l, 2l+1: for each of its
//        Gaussians it walks the mask's set bits in ascending row order and adds gamma z, gamma z^2
//        (z = (x - c) 2^e from the fp32 X tile still resident in shared memory) into fp32 registers —
//        exactly the pairs Alg.1 l.18 / Alg.5 l.9 keep, summed in a fixed order (deterministic), with
//        round-to-nearest fp32 adds (no truncating tensor-core accumulator), S0_j alongside
//   a6   at chunk / segment ends the registers go to the same (cluster, image) segment slots k_stats
//        fills (feature-major rows, units gamma 2^14 x 2^e), so every finalize kernel is shared.
// The result equals the dense path's up to rounding (the same gamma, the same inclusion test); the
// work of a5' scales with the number of survivors (~7.5 of 256 per descriptor on the acceptance
// generator), not with K.
//
// Roles (576 threads): warp 0 MMA issuer (GEMM1 only), warp 1 TMA producer, warps 2..17 WORK.
// Shared memory: W' 64 KB, X ring of 2 tiles (2 x 2 boxes x 16 KB: a tile stays resident until its
// survivors are accumulated), Gamma 64 KB, masks 2 KB.  Tensor memory: Zr and L, both double-buffered
// (GEMM1(i+1) runs while the WORK warps finish tile i).
#pragma once
#include <cuda.h>

#include "fv_common.cuh"
#include "ptx.cuh"
#include "k_stats.cuh"

namespace gpufv {

// X tile: ONE unswizzled TMA box of 68 floats x 128 rows (columns D..67 read as zero), i.e. rows of
// 272 B: a warp reading one 16-byte chunk of 32 consecutive rows (the conversion) and a warp reading
// one whole row (the accumulation) are both bank-conflict free, and a row address is one IMAD
constexpr int kSpXLd = kDP + 4;                         // floats per X row in shared memory
constexpr int kSpXTile = kTileM * kSpXLd * 4;           // 34 KB (a multiple of 1 KB)
constexpr int kSpGLd = kG + 4;                          // floats per Gamma row (528 B: conflict-free STS.128)
constexpr int kSpW = 0;                                 // W' hi | lo            64 KB
constexpr int kSpX = kSpW + 2 * kOpBytes;               // X ring: 2 tiles       68 KB
constexpr int kSpG = kSpX + 2 * kSpXTile;               // Gamma [128][132] f32  66 KB
constexpr int kSpMask = kSpG + kTileM * kSpGLd * 4;     // uint32[128 Gaussians][4 row quarters]
constexpr int kSpList = kSpMask + kG * 16;              // uint8[16 warps][128]: survivor rows of one Gaussian
constexpr int kSpBias = kSpList + kWarpsWork * kTileM;  // float[128]
constexpr int kSpCs = kSpBias + kG * 4;                 // float[64]  -c_k 2^e_k
constexpr int kSpSc = kSpCs + kDP * 4;                  // float[64]  2^e_k
constexpr int kSpXchg = kSpSc + kDP * 4;                // float2[2][kMaxC2][4][128]
constexpr int kSpMeta = kSpXchg + 2 * kMaxC2 * 4 * kTileM * 8;
constexpr int kSpBar = kSpMeta + 128;
constexpr int kSpTmem = kSpBar + 16 * 8;
constexpr int kSmemSpBytes = kSpTmem + 16 + 1024;
static_assert(kSmemSpBytes <= 232448, "shared memory budget");

enum : int {
  S_XFULL0 = 0, S_XFULL1, S_XEMPTY0, S_XEMPTY1, S_ZR_FULL, S_G1D0, S_G1D1, S_LE0, S_LE1, S_XCHG0, S_XCHG1, S_W_FULL
};
constexpr uint32_t kSpTZr = 0, kSpTL = 256;            // TMEM: Zr[2] (cols 0..255), L[2] (256..511)
constexpr uint32_t kBarSpG = 6, kBarSpA = 7;           // named barriers: Gamma written / accumulated

// Features of dims k = 32 box + 8h .. +8 of one row from the padded X tile (row pitch kSpXLd floats);
// same arithmetic as zr_box (k_stats.cuh).
template <bool kMask>
__device__ __forceinline__ void zr_row(const float *xr, int box, int h, int D, bool valid, const float *s_sc,
                                       const float *s_ncs, uint32_t taddr) {
  using namespace ptx;
  uint32_t lh[4], ll[4], qh[4], ql[4];
  const int k0 = 32 * box + 8 * h;
#pragma unroll
  for (int c2 = 0; c2 < 2; ++c2) {
    const float4 v = *reinterpret_cast<const float4 *>(xr + k0 + 4 * c2);
    const float4 sc = *reinterpret_cast<const float4 *>(s_sc + k0 + 4 * c2);
    const float4 ncs = *reinterpret_cast<const float4 *>(s_ncs + k0 + 4 * c2);
    float2 a0 = __ffma2_rn(make_float2(v.x, v.y), make_float2(sc.x, sc.y), make_float2(ncs.x, ncs.y));
    float2 a1 = __ffma2_rn(make_float2(v.z, v.w), make_float2(sc.z, sc.w), make_float2(ncs.z, ncs.w));
    if (kMask) {
      const int kk = k0 + 4 * c2;
      if (!valid || kk >= D) a0.x = 0.f;
      if (!valid || kk + 1 >= D) a0.y = 0.f;
      if (!valid || kk + 2 >= D) a1.x = 0.f;
      if (!valid || kk + 3 >= D) a1.y = 0.f;
    }
    split2_f16(a0, lh[2 * c2], ll[2 * c2]);
    split2_f16(a1, lh[2 * c2 + 1], ll[2 * c2 + 1]);
    split2_f16(__fmul2_rn(a0, a0), qh[2 * c2], ql[2 * c2]);
    split2_f16(__fmul2_rn(a1, a1), qh[2 * c2 + 1], ql[2 * c2 + 1]);
  }
  tmem_st4(taddr + k0 / 2, lh);
  tmem_st4(taddr + 32 + k0 / 2, qh);
  tmem_st4(taddr + 64 + k0 / 2, ll);
  tmem_st4(taddr + 96 + k0 / 2, ql);
}

// 32 x 32 bit-matrix transpose across a warp: on entry bit c of lane r's word is M[r][c], on exit bit
// r of lane c's word is M[r][c].  Five butterfly stages (block swaps of the off-diagonal k x k blocks).
__device__ __forceinline__ uint32_t warp_bit_transpose(uint32_t w, int lane) {
  const uint32_t lo_cols[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const int k = 16 >> s;
    const uint32_t m = lo_cols[s];
    const uint32_t o = __shfl_xor_sync(0xffffffffu, w, k);
    w = (lane & k) ? ((w & ~m) | ((o >> k) & m)) : ((w & m) | ((o << k) & ~m));
  }
  return w;
}

template <bool kD64>
__global__ void __launch_bounds__(kThreads2, 1) k_stats_sp(const __grid_constant__ CUtensorMap tmap_x, const Stats2Params p) {
  using namespace ptx;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_base = smem_u32(smem_raw);
  const uint32_t sbase = (raw_base + 1023u) & ~1023u;
  uint8_t *smem = smem_raw + (sbase - raw_base);
  const uint32_t sW = sbase + kSpW, sX = sbase + kSpX, sG = sbase + kSpG;
  float *s_bias = reinterpret_cast<float *>(smem + kSpBias);
  float *s_ncs = reinterpret_cast<float *>(smem + kSpCs);
  float *s_sc = reinterpret_cast<float *>(smem + kSpSc);
  float2 *s_xchg = reinterpret_cast<float2 *>(smem + kSpXchg);
  uint32_t *s_mask = reinterpret_cast<uint32_t *>(smem + kSpMask);
  TileMeta *s_meta = reinterpret_cast<TileMeta *>(smem + kSpMeta);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + kSpBar);
  uint32_t *s_tmem = reinterpret_cast<uint32_t *>(smem + kSpTmem);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_ctarank(), C = cluster_nctarank();
  const int cid = (int)cluster_id_x(), ncl = (int)nclusters_x();

  // ---------------- setup
  for (int i = tid; i < kG; i += kThreads2) s_bias[i] = p.bias[rank * kG + i];
  if (tid < kDP) { s_sc[tid] = p.xscale[tid]; s_ncs[tid] = -(p.xshift[tid] * p.xscale[tid]); }
  if (warp == 0) { tmem_alloc(s_tmem, kTmemCols); tmem_relinquish(); }
  if (tid == 0) {
    mbar_init(&bars[S_XFULL0], 1); mbar_init(&bars[S_XFULL1], 1);
    mbar_init(&bars[S_XEMPTY0], 1); mbar_init(&bars[S_XEMPTY1], 1);
    mbar_init(&bars[S_ZR_FULL], kWarpsWork);
    mbar_init(&bars[S_G1D0], 1); mbar_init(&bars[S_G1D1], 1);
    mbar_init(&bars[S_LE0], kWarpsWork); mbar_init(&bars[S_LE1], kWarpsWork);
    mbar_init(&bars[S_XCHG0], 1); mbar_init(&bars[S_XCHG1], 1);
    mbar_init(&bars[S_W_FULL], 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(&bars[S_W_FULL], kWImgBytes);
    for (int c = 0; c < 4; ++c)
      bulk_g2s(sW + c * (kWImgBytes / 4), p.wimg + (size_t)rank * kWImgBytes + c * (kWImgBytes / 4), kWImgBytes / 4,
               &bars[S_W_FULL]);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  cluster_sync();
  griddep_launch_dependents();  // the finalize may start its prologue
  griddep_wait();               // k_schedule's tile prefix sums are complete and visible

  const int64_t T = p.tile_start[p.batch];
  const int t0 = (int)((int64_t)cid * T / ncl), t1 = (int)((int64_t)(cid + 1) * T / ncl);
  const int n = t1 - t0;

  if (warp == kWarpTma) {
    // ======================================================= tile walk + X producer (TMA)
    if (lane == 0 && n > 0) {
      const int Dv = p.ldx;
      TileWalker tw, twp;
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_x)) : "memory");
      tw.init(p, t0, t1);
      auto prefetch_l2 = [&](int i) {
        if (i >= n) return;
        const TileMeta m = twp.meta();
        twp.next();
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p.X + (size_t)m.row0 * Dv),
                     "r"((uint32_t)(m.nrows * Dv * 4) & ~15u)
                     : "memory");
      };
      for (int i = 0; i < n; ++i, tw.next()) {
        const TileMeta m = tw.meta();
        const int slot = i & 1;
        if (i >= 2) mbar_wait(&bars[S_XEMPTY0 + slot], ((i - 2) >> 1) & 1);  // tile i-2 accumulated
        s_meta[i & 3] = m;  // released to the WORK warps by the X_FULL phase completion
        mbar_arrive_expect_tx(&bars[S_XFULL0 + slot], kSpXTile);
        tma_load_2d(sX + slot * kSpXTile, &tmap_x, 0, m.row0, &bars[S_XFULL0 + slot]);
        if (i == 0) {  // L2 prefetch walker 4 tiles ahead (set up after the first loads are requested)
          twp.init(p, t0, t1);
          for (int k = 0; k < 4; ++k) prefetch_l2(k);
        }
        prefetch_l2(i + 4);
      }
    }
  } else if (warp == kWarpMma) {
    // ======================================================= MMA issuer: GEMM1 only
    if (n > 0) {
      const uint32_t idesc1 = idesc_f16_f32(128, kG, 0, 0);  // A = Zr (TMEM, K-major), B = W' K-major
      const uint64_t dW = desc_sw128(sW, 16, 1024);
      mbar_wait(&bars[S_W_FULL], 0);
      for (int i = 0; i < n; ++i) {
        TR(12);
        mbar_wait(&bars[S_ZR_FULL], i & 1);
        TR(13);
        if (i >= 2) mbar_wait(&bars[S_LE0 + (i & 1)], ((i - 2) >> 1) & 1);  // L[i % 2] read by softmax(i-2)
        tc_fence_after();
        const uint32_t zr = tmem + kSpTZr + 128 * (i & 1), dl = tmem + kSpTL + 128 * (i & 1);
#pragma unroll
        for (int s = 0; s < 3; ++s) {  // cross terms first, hi.hi last (truncating accumulator)
          const uint32_t za = zr + (s == 1 ? 64 : 0);   // hi, lo, hi
          const uint32_t wb = (s == 0 ? kOpBytes : 0);  // lo, hi, hi
#pragma unroll
          for (int kk = 0; kk < kNF / 16; ++kk) {
            const uint32_t off = wb + (kk >> 2) * kAtomBytes + (kk & 3) * 32;
            mma_f16_ts_w(dl, za + kk * 8, dW + (off >> 4), idesc1, (s | kk) != 0);
          }
        }
        mma_commit_w(&bars[S_G1D0 + (i & 1)]);
        TR(14);
      }
    }
  } else {
    // ======================================================= WORK warps
    const int ww = warp - kWarpWork0;       // WORK warp index 0..15
    const int q = warp & 3, h = ww >> 2;    // TMEM lanes 32q.. (physical warp % 4); Gaussian quarter h
    const uint32_t lane_base = (uint32_t)(32 * q) << 16;
    const int row = 32 * q + lane;          // descriptor row of the softmax
    const float thr = p.threshold * kPScale;

    auto xtile = [&](int i) { return reinterpret_cast<const float *>(smem + kSpX + (i & 1) * kSpXTile); };
    auto conv_box = [&](int i, int box) {  // Zr(i) box `box`: this warp's dims 32 box + 8h .. +8 of `row`
      const int nrows = s_meta[i & 3].nrows;
      const uint32_t ta = tmem + kSpTZr + 128 * (i & 1) + lane_base;
      const float *xr = xtile(i) + row * kSpXLd;
      if (!kD64 || nrows < kTileM) zr_row<true>(xr, box, h, p.D, row < nrows, s_sc, s_ncs, ta);
      else zr_row<false>(xr, box, h, kDP, true, s_sc, s_ncs, ta);
    };
    auto zr_done = [&]() {
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[S_ZR_FULL]);
    };

    // accumulation state (a5'): this warp's Gaussians jb .. jb+7, this lane's dims 2 lane, 2 lane + 1
    const int jb = 8 * ww;
    uint8_t *s_list = smem + kSpList + ww * kTileM;
    const float *s_gam = reinterpret_cast<const float *>(smem + kSpG);
    const float2 asc = make_float2(s_sc[2 * lane], s_sc[2 * lane + 1]);
    const float2 ancs = make_float2(s_ncs[2 * lane], s_ncs[2 * lane + 1]);
    float2 S1[8], S2[8];
    float s0 = 0.f;  // S0 of Gaussian jb + lane (lanes 0..7)
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) S1[jj] = S2[jj] = make_float2(0.f, 0.f);
    bool chunk_seg_first = true;

    if (n > 0) {
      mbar_wait(&bars[S_XFULL0], 0);
      conv_box(0, 0);
      conv_box(0, 1);
      zr_done();
    }
    for (int i = 0; i < n; ++i) {
      TRW(0);
      work_wait(&bars[S_G1D0 + (i & 1)], (i >> 1) & 1);  // L(i) ready
      TRW(1);
      float v[32];
      {
        uint32_t rr[32];
        tmem_ld32(tmem + kSpTL + 128 * (i & 1) + lane_base + 32 * h, rr);
        tmem_ld_wait(rr);
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(rr[j]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[S_LE0 + (i & 1)]);
      TRW(2);
      const TileMeta mt = s_meta[i & 3];
      float m = -3.0e38f;
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        const float4 bj = *reinterpret_cast<const float4 *>(s_bias + 32 * h + j);
        const float2 x0 = __fadd2_rn(make_float2(v[j], v[j + 1]), make_float2(bj.x, bj.y));
        const float2 x1 = __fadd2_rn(make_float2(v[j + 2], v[j + 3]), make_float2(bj.z, bj.w));
        v[j] = x0.x; v[j + 1] = x0.y; v[j + 2] = x1.x; v[j + 3] = x1.y;
        m = fmaxf(m, fmaxf(fmaxf(x0.x, x0.y), fmaxf(x1.x, x1.y)));
      }
      auto exp_local = [&]() {
        float2 sacc = make_float2(0.f, 0.f);
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const float2 d = __fadd2_rn(make_float2(v[j], v[j + 1]), make_float2(-m, -m));
          v[j] = ex2_approx(d.x); v[j + 1] = ex2_approx(d.y);
          sacc = __fadd2_rn(sacc, make_float2(v[j], v[j + 1]));
        }
        return sacc.x + sacc.y;
      };
      const int par = i & 1;
      float2 *xb = s_xchg + par * (kMaxC2 * 4 * kTileM);
      auto send = [&](float ssum) {
        if (C == 1) {
          xb[(rank * 4 + h) * kTileM + row] = make_float2(m, ssum);
          return;
        }
        if (ww == 0 && lane == 0) mbar_arrive_expect_tx(&bars[S_XCHG0 + par], C * 4 * kTileM * 8);
        const uint32_t my = smem_u32(&xb[(rank * 4 + h) * kTileM + row]);
        const uint32_t mybar = smem_u32(&bars[S_XCHG0 + par]);
        for (uint32_t r2 = 0; r2 < C; ++r2) st_async_v2f32(mapa_shared(my, r2), m, ssum, mapa_shared(mybar, r2));
      };
      if (i + 1 < n) {
        // tile i+1 (resident since tile i-1 was accumulated): box 0 inside the MUFU-bound exp loop,
        // box 1 behind the exchange send; then GEMM1(i+1) may start
        mbar_wait(&bars[S_XFULL0 + ((i + 1) & 1)], ((i + 1) >> 1) & 1);
        TRW(3);
        const float ssum = exp_local();
        conv_box(i + 1, 0);
        send(ssum);
        TRW(4);
        conv_box(i + 1, 1);
        zr_done();
        TRW(5);
      } else {
        send(exp_local());
      }
      if (C > 1) mbar_wait(&bars[S_XCHG0 + par], (i >> 1) & 1);
      else named_bar_sync(kBarXchgLocal, kWarpsWork * 32);
      TRW(6);
      float M = -3.0e38f, S = 0.f;
      {
        float2 o[kMaxC2 * 4];
#pragma unroll
        for (int e = 0; e < kMaxC2 * 4; ++e) {
          o[e] = make_float2(-3.0e38f, 0.f);
          if (e < (int)C * 4) { o[e] = xb[e * kTileM + row]; M = fmaxf(M, o[e].x); }
        }
#pragma unroll
        for (int e = 0; e < kMaxC2 * 4; ++e) S += o[e].y * ex2_approx(o[e].x - M);
      }
      float alpha_p = __fdividef(ex2_approx(m - M), S) * kPScale;
      if (row >= mt.nrows) alpha_p = 0.f;
      else if (!(S > 0.5f && S < 3.0e38f)) range_bad(p, mt.b, alpha_p, h == 0 && rank == 0);

      // ---- a4': Gamma row (gamma 2^14, all 32 columns) and the survivor bits gamma > tau (a NaN row
      // counts as surviving, so a flagged row reaches the statistics as NaN)
      TRW(7);
      uint32_t sbits = 0;
      {
        const float2 ap = make_float2(alpha_p, alpha_p);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float2 g0 = __fmul2_rn(make_float2(v[4 * c], v[4 * c + 1]), ap);
          const float2 g1 = __fmul2_rn(make_float2(v[4 * c + 2], v[4 * c + 3]), ap);
          sbits |= (!(g0.x <= thr) ? 1u : 0u) << (4 * c);
          sbits |= (!(g0.y <= thr) ? 1u : 0u) << (4 * c + 1);
          sbits |= (!(g1.x <= thr) ? 1u : 0u) << (4 * c + 2);
          sbits |= (!(g1.y <= thr) ? 1u : 0u) << (4 * c + 3);
          sts128(sG + (uint32_t)(row * kSpGLd + 32 * h + 4 * c) * 4u, __float_as_uint(g0.x), __float_as_uint(g0.y),
                 __float_as_uint(g1.x), __float_as_uint(g1.y));
        }
      }
      if (row >= mt.nrows) sbits = 0u;  // rows past the image end never enter the sums
      s_mask[(32 * h + lane) * 4 + q] = warp_bit_transpose(sbits, lane);  // Gaussian 32h + lane, rows 32q..
      TRW(8);
      named_bar_sync(kBarSpG, kWarpsWork * 32);
      TRW(9);

      // ---- a5': survivors of this warp's 8 Gaussians, rows ascending, into fp32 registers.  Per
      // Gaussian the warp first compacts the mask into a row list (lane l places rows 32q + l), then
      // takes the survivors four at a time (one 4-byte list load, all loads in flight before the math).
      {
        const float *xt = xtile(i) + 2 * lane;
        const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const int j = jb + jj;
          const bool mine = lane == jj;
          const uint4 mk = *reinterpret_cast<const uint4 *>(s_mask + j * 4);
          const uint32_t words[4] = {mk.x, mk.y, mk.z, mk.w};
          int cnt = 0;
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            const uint32_t w = words[qq];
            if ((w >> lane) & 1u) s_list[cnt + __popc(w & lt)] = (uint8_t)(32 * qq + lane);
            cnt += __popc(w);
          }
          __syncwarp();
          const float *gj = s_gam + j;
          for (int s4 = 0; s4 < cnt; s4 += 4) {
            const uint32_t rows4 = *reinterpret_cast<const uint32_t *>(s_list + s4);
            float g[4];
            float2 x[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {  // entries past cnt are stale rows (< 128): loaded, never used
              const int r = (rows4 >> (8 * k)) & 0x7f;
              g[k] = gj[r * kSpGLd];
              x[k] = *reinterpret_cast<const float2 *>(xt + r * kSpXLd);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              if (s4 + k < cnt) {  // warp-uniform
                const float2 z = __ffma2_rn(x[k], asc, ancs);
                const float2 t = __fmul2_rn(z, make_float2(g[k], g[k]));
                S1[jj] = __fadd2_rn(S1[jj], t);
                S2[jj] = __ffma2_rn(t, z, S2[jj]);
                if (mine) s0 += g[k];
              }
            }
          }
          __syncwarp();  // the list is rewritten for the next Gaussian
        }
      }
      TRW(10);
      named_bar_sync(kBarSpA, kWarpsWork * 32);  // Gamma, masks and X(i) are free
      TRW(11);
      if (ww == 0 && lane == 0) mbar_arrive(&bars[S_XEMPTY0 + (i & 1)]);

      // ---- a6: chunk end -> segment slot (first chunk stores, later chunks add, same thread, in order)
      if (mt.flags & 2) chunk_seg_first = (mt.flags & 8) != 0;
      if (mt.flags & 4) {
        float *base = p.slots + (size_t)seg_slot(cid, mt.b) * kNF * p.Kp + rank * kG + jb;
        const int fr[4] = {2 * lane, 2 * lane + 1, kDP + 2 * lane, kDP + 2 * lane + 1};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          float a[8];
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) a[jj] = u == 0 ? S1[jj].x : u == 1 ? S1[jj].y : u == 2 ? S2[jj].x : S2[jj].y;
          float *dst = base + (size_t)fr[u] * p.Kp;
          if (chunk_seg_first) {
            *reinterpret_cast<float4 *>(dst) = make_float4(a[0], a[1], a[2], a[3]);
            *reinterpret_cast<float4 *>(dst + 4) = make_float4(a[4], a[5], a[6], a[7]);
          } else {
            red_add_v4(dst, a[0], a[1], a[2], a[3]);
            red_add_v4(dst + 4, a[4], a[5], a[6], a[7]);
          }
        }
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) S1[jj] = S2[jj] = make_float2(0.f, 0.f);
      }
      if (mt.flags & 1) {  // segment end: S0 (units of 2^14 gamma) into row-group slot 0, zeros in 1..3
        p.s0slots[((size_t)seg_slot(cid, mt.b) * 4 + (lane >> 3)) * p.Kp + rank * kG + jb + (lane & 7)] =
            lane < 8 ? s0 : 0.f;
        s0 = 0.f;
      }
    }
  }

  // ---------------- teardown
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) tmem_dealloc(tmem, kTmemCols);
}

}  // namespace gpufv
