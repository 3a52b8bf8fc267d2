// k_stats_x.cuh — steps a2-a6 for D <= 64, K <= 256 with the log-likelihood computed TRANSPOSED
// (item 4): same method, numerics and outputs as k_stats, different operand placement.
//
//   GEMM1  L^T[g, i] = sum_f W'[g, f] Z[i, f]    A = W' resident in TMEM for the whole kernel
//                                               (lanes = Gaussians), B = Z(i) from shared memory
//   GEMM2  S'^T[g, f] += sum_i P^T[g, i] Z[i, f]  A = P^T written by the WORK warps in place of L^T,
//                                               B = the same Z(i) buffer (MN-major view)
//   Both are TS-MMAs (94-cycle UMMAs, profiles/r01g_tmem_smem_probe.txt); shared memory carries only Z
//   (written once per tile from the X boxes) and the X boxes — no P, no Zr, no Z copy.
//   Softmax across TMEM lanes: thread (lane = Gaussian g, warp column block h) holds L^T[g][32h ..+32];
//   the per-descriptor max over the warp's 32 Gaussians is one redux.sync.max.f32 per descriptor, the
//   sum a 32 x 32 butterfly transpose-reduce; (m, s) per descriptor then goes through the same 4C-pair
//   cluster exchange as k_stats (lane l of warp (q, h) carries descriptor 32h + l); S0_g is one register.
//
// TMEM: W' hi|lo (128 cols), L^T/P^T double buffer (2 x 128), S'^T (128).
// SMEM: Z double buffer (2 x 64 KB; the W' image is staged in it once at start), X tile (2 boxes,
// 32 KB), exchange, per-warp broadcast rows.
// Per local tile i the WORK warps run: wait G1(i) | L^T(i) | bias, max, exp | sum | send (m, s) |
// wait G2(i-1) [fold] | Z(i+1) from X(i+1) | wait exchange | combine | P^T(i), S0;
// the MMA thread issues G1(0), then per tile G1(i+1) (after Z(i+1)), G2(i) (after P^T(i)).
#pragma once
#include <cuda.h>

#include "fv_common.cuh"
#include "k_stats.cuh"
#include "ptx.cuh"

namespace gpufv {

constexpr int kX4Z = 0;                                    // Z[2]: hi | lo, 2 atoms each   128 KB
constexpr int kX4X = kX4Z + 2 * 2 * kOpBytes;             // X tile: box 0 | box 1          32 KB
constexpr int kX4Cs = kX4X + 2 * kXBoxBytes;              // float[64]  -c_k 2^e_k
constexpr int kX4Sc = kX4Cs + kDP * 4;                    // float[64]  2^e_k
constexpr int kX4Xchg = kX4Sc + kDP * 4;                  // float2[2 parity][kMaxC2][4][128]
constexpr int kX4Bc = kX4Xchg + 2 * kMaxC2 * 4 * kTileM * 8;  // float[16 warps][32]: broadcast rows
constexpr int kX4Meta = kX4Bc + kWarpsWork * 32 * 4;
constexpr int kX4Bar = kX4Meta + 128;
constexpr int kX4Tmem = kX4Bar + kNumBars * 8;
constexpr int kSmem4Bytes = kX4Tmem + 16 + 1024;
static_assert(kSmem4Bytes <= 232448, "shared memory budget (k_stats_x)");

enum : int {
  X_XFULL = 0, X_XEMPTY, X_ZFULL, X_G1_DONE, X_G2_DONE, X_P_FULL, X_FOLD_DONE, X_XCHG0, X_XCHG1, X_W_IMG, X_W_TMEM
};

constexpr uint32_t kX4W = 0, kX4LP = 128, kX4S = 384;  // TMEM columns

__device__ __forceinline__ float redux_max(float v) {
  float r;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}

template <bool kD64>
__global__ void __launch_bounds__(kThreads2, 1) k_stats_x(const __grid_constant__ CUtensorMap tmap_x, const Stats2Params p) {
  using namespace ptx;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_base = smem_u32(smem_raw);
  const uint32_t sbase = (raw_base + 1023u) & ~1023u;
  uint8_t *smem = smem_raw + (sbase - raw_base);
  const uint32_t sZ = sbase + kX4Z, sX = sbase + kX4X;
  float *s_ncs = reinterpret_cast<float *>(smem + kX4Cs);
  float *s_sc = reinterpret_cast<float *>(smem + kX4Sc);
  float2 *s_xchg = reinterpret_cast<float2 *>(smem + kX4Xchg);
  float *s_bc = reinterpret_cast<float *>(smem + kX4Bc);
  TileMeta *s_meta = reinterpret_cast<TileMeta *>(smem + kX4Meta);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + kX4Bar);
  uint32_t *s_tmem = reinterpret_cast<uint32_t *>(smem + kX4Tmem);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_ctarank(), C = cluster_nctarank();
  const int cid = (int)cluster_id_x(), ncl = (int)nclusters_x();

  if (tid < kDP) { s_sc[tid] = p.xscale[tid]; s_ncs[tid] = -(p.xshift[tid] * p.xscale[tid]); }
  if (warp == 0) { tmem_alloc(s_tmem, kTmemCols); tmem_relinquish(); }
  if (tid == 0) {
    mbar_init(&bars[X_XFULL], 1); mbar_init(&bars[X_XEMPTY], kWarpsWork);
    mbar_init(&bars[X_ZFULL], kWarpsWork);
    mbar_init(&bars[X_G1_DONE], 1); mbar_init(&bars[X_G2_DONE], 1);
    mbar_init(&bars[X_P_FULL], kWarpsWork); mbar_init(&bars[X_FOLD_DONE], kWarpsWork);
    mbar_init(&bars[X_XCHG0], 1); mbar_init(&bars[X_XCHG1], 1);
    mbar_init(&bars[X_W_IMG], 1); mbar_init(&bars[X_W_TMEM], kWarpsWork);
    fence_mbar_init();
    // this rank's W' image (64 KB, SW128 K-major [hi|lo][atom][128 rows][128 B]) staged in Z buffer 1
    mbar_arrive_expect_tx(&bars[X_W_IMG], kWImgBytes);
    for (int c = 0; c < 4; ++c)
      bulk_g2s(sZ + 2 * kOpBytes + c * (kWImgBytes / 4), p.wimg + (size_t)rank * kWImgBytes + c * (kWImgBytes / 4),
               kWImgBytes / 4, &bars[X_W_IMG]);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  cluster_sync();
  griddep_launch_dependents();
  griddep_wait();

  const int64_t T = p.tile_start[p.batch];
  const int t0 = (int)((int64_t)cid * T / ncl), t1 = (int)((int64_t)(cid + 1) * T / ncl);
  const int n = t1 - t0;

  if (warp == kWarpTma) {
    // ======================================================= tile walk + X producer (TMA)
    if (lane == 0 && n > 0) {
      const int Dv = p.ldx;
      TileWalker tw, twp;
      tw.init(p, t0, t1);
      twp.init(p, t0, t1);
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_x)) : "memory");
      auto prefetch_l2 = [&](int i) {
        if (i >= n) return;
        const TileMeta m = twp.meta();
        twp.next();
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p.X + (size_t)m.row0 * Dv),
                     "r"((uint32_t)(m.nrows * Dv * 4) & ~15u)
                     : "memory");
      };
      for (int i = 0; i < 4; ++i) prefetch_l2(i);
      for (int i = 0; i < n; ++i, tw.next()) {
        if (i >= 1) mbar_wait(&bars[X_XEMPTY], (i - 1) & 1);  // Z(i-1) converted from the X tile
        s_meta[i & 3] = tw.meta();
        mbar_arrive_expect_tx(&bars[X_XFULL], 2 * kXBoxBytes);
        tma_load_2d(sX, &tmap_x, 0, s_meta[i & 3].row0, &bars[X_XFULL]);
        tma_load_2d(sX + kXBoxBytes, &tmap_x, 32, s_meta[i & 3].row0, &bars[X_XFULL]);
        prefetch_l2(i + 4);
      }
    }
  } else if (warp == kWarpMma) {
    // ======================================================= MMA issuer
    if (lane == 0 && n > 0) {
      TileWalker tw;
      tw.init(p, t0, t1);
      const uint32_t idesc1 = idesc_f16_f32(kG, kTileM, 0, 0);  // A = W' (TMEM), B = Z K-major: L^T
      const uint32_t idesc2 = idesc_f16_f32(kG, kNF, 0, 1);     // A = P^T (TMEM), B = Z MN-major: S'^T
      uint32_t folds = 0;
      mbar_wait(&bars[X_W_TMEM], 0);
      auto gemm1 = [&](int i) {
        mbar_wait(&bars[X_ZFULL], i & 1);
        tc_fence_after();
        const uint32_t zb = sZ + (i & 1) * 2 * kOpBytes;
        const uint32_t dl = tmem + kX4LP + 128 * (i & 1);
#pragma unroll
        for (int s = 0; s < 3; ++s) {  // cross terms first, hi.hi last (truncating accumulator)
          const uint32_t wa = tmem + kX4W + (s == 1 ? 64 : 0);    // W' hi, lo, hi
          const uint32_t zz = zb + (s == 0 ? kOpBytes : 0);        // Z  lo, hi, hi
#pragma unroll
          for (int kk = 0; kk < kNF / 16; ++kk) {
            const uint32_t off = (kk >> 2) * kAtomBytes + (kk & 3) * 32;
            mma_f16_ts(dl, wa + kk * 8, desc_sw128(zz + off, 16, 1024), idesc1, (s | kk) != 0);
          }
        }
        mma_commit(&bars[X_G1_DONE]);
      };
      auto gemm2 = [&](int i, bool chunk_first) {
        mbar_wait(&bars[X_P_FULL], i & 1);
        if (chunk_first && i > 0) { mbar_wait(&bars[X_FOLD_DONE], folds & 1); ++folds; }
        tc_fence_after();
        const uint32_t zb = sZ + (i & 1) * 2 * kOpBytes;
        const uint32_t pa = tmem + kX4LP + 128 * (i & 1);
#pragma unroll
        for (int s = 0; s < 3; ++s) {
          const uint32_t a = pa + (s == 1 ? 64 : 0);              // P^T hi, lo, hi
          const uint32_t zz = zb + (s == 0 ? kOpBytes : 0);        // Z    lo, hi, hi
#pragma unroll
          for (int kk = 0; kk < kTileM / 16; ++kk)
            mma_f16_ts(tmem + kX4S, a + kk * 8, desc_sw128(zz + kk * 2048, kAtomBytes, 1024), idesc2,
                       (chunk_first && s == 0 && kk == 0) ? 0u : 1u);
        }
        mma_commit(&bars[X_G2_DONE]);
      };
      gemm1(0);
      for (int i = 0; i < n; ++i, tw.next()) {
        const bool chunk_first = (tw.meta().flags & 2) != 0;
        TR(13);
        if (i + 1 < n) gemm1(i + 1);
        TR(14);
        gemm2(i, chunk_first);
        TR(15);
      }
    }
  } else {
    // ======================================================= WORK warps
    const int q = warp & 3, h = warp >> 2;       // TMEM lanes 32q.. (Gaussians) ; descriptor block h
    const uint32_t lane_base = (uint32_t)(32 * q) << 16;
    const int g = 32 * q + lane;                 // CTA-local Gaussian of this thread
    const int gj = rank * kG + g;                // global Gaussian index
    const int D = kD64 ? kDP : p.D;
    const float thr = p.threshold * kPScale;
    const float bias = p.bias[gj];
    float *bc = s_bc + warp * 32;

    // one-time: W' image (staged in Z buffer 1) -> TMEM A operand (lane g: 64 hi + 64 lo columns,
    // column c = features 2c, 2c+1); warp (q, h) moves columns 16h .. 16h + 15 of hi and of lo
    mbar_wait(&bars[X_W_IMG], 0);
    {
      const uint8_t *wimg = smem + kX4Z + 2 * kOpBytes;
#pragma unroll
      for (int part = 0; part < 2; ++part) {  // hi, lo
        uint32_t w16[16];
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {      // 4 chunks of 8 features = 4 x 4 columns
          const int col = 16 * h + 4 * c4, f = 2 * col, atom = f / 64, chunk = (f & 63) >> 3;
          const uint4 v = *reinterpret_cast<const uint4 *>(wimg + part * kOpBytes + atom * kAtomBytes + sw_off(g, chunk));
          w16[4 * c4] = v.x; w16[4 * c4 + 1] = v.y; w16[4 * c4 + 2] = v.z; w16[4 * c4 + 3] = v.w;
        }
        tmem_st16(tmem + kX4W + lane_base + 64 * part + 16 * h, w16);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[X_W_TMEM]);
    }
    named_bar_sync(kBarXchgLocal + 1, kWarpsWork * 32);  // all W' reads done before Z buffer 1 is reused
    // Z(t) from the resident X tile: thread (row = 32 (warp & 3) + lane... ) converts like zr_box, but
    // stores the fp16 hi/lo words into the SW128 Z buffer [row][feature] (lin features 0..63 in atom 0,
    // quadratic in atom 1)
    const int zrow = 32 * q + lane;  // descriptor row converted by this thread (any mapping works)
    auto conv_z = [&](int t, int nrows) {
      const uint32_t zb = sZ + (t & 1) * 2 * kOpBytes;
#pragma unroll
      for (int box = 0; box < 2; ++box) {
        const uint8_t *xbox = smem + kX4X + box * kXBoxBytes;
        const int k0 = 32 * box + 8 * h;
        uint32_t lh[4], ll[4], qh[4], ql[4];
#pragma unroll
        for (int c2 = 0; c2 < 2; ++c2) {
          const float4 v = *reinterpret_cast<const float4 *>(xbox + sw_off(zrow, 2 * h + c2));
          const float4 sc = *reinterpret_cast<const float4 *>(s_sc + k0 + 4 * c2);
          const float4 ncs = *reinterpret_cast<const float4 *>(s_ncs + k0 + 4 * c2);
          float2 a0 = __ffma2_rn(make_float2(v.x, v.y), make_float2(sc.x, sc.y), make_float2(ncs.x, ncs.y));
          float2 a1 = __ffma2_rn(make_float2(v.z, v.w), make_float2(sc.z, sc.w), make_float2(ncs.z, ncs.w));
          if (!kD64 || nrows < kTileM) {
            const int kk = k0 + 4 * c2;
            const bool valid = zrow < nrows;
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
        const uint32_t o = sw_off(zrow, 4 * box + h);  // features k0 .. k0 + 7 of this row
        sts128(zb + o, lh[0], lh[1], lh[2], lh[3]);
        sts128(zb + kAtomBytes + o, qh[0], qh[1], qh[2], qh[3]);
        sts128(zb + kOpBytes + o, ll[0], ll[1], ll[2], ll[3]);
        sts128(zb + kOpBytes + kAtomBytes + o, ql[0], ql[1], ql[2], ql[3]);
      }
      fence_proxy_async_smem();  // generic-proxy Z stores -> visible to the tensor core
      __syncwarp();
      if (lane == 0) { mbar_arrive(&bars[X_XEMPTY]); mbar_arrive(&bars[X_ZFULL]); }
    };
    // S'^T quarter (lane = Gaussian g, columns = features 32h ..) -> slot rows f (feature-major)
    auto fold = [&](int b, bool first) {
      float *dst = p.slots + (size_t)seg_slot(cid, b) * kNF * p.Kp + (size_t)(32 * h) * p.Kp + gj;
      uint32_t v[32];
      tmem_ld32(tmem + kX4S + lane_base + 32 * h, v);
      tmem_ld_wait(v);
      if (first) {
#pragma unroll
        for (int f = 0; f < 32; ++f) dst[(size_t)f * p.Kp] = __uint_as_float(v[f]);
      } else {
#pragma unroll
        for (int f = 0; f < 32; ++f) atomicAdd(dst + (size_t)f * p.Kp, __uint_as_float(v[f]));
      }
    };

    float s0 = 0.f;
    int prev_b = 0;
    bool prev_fold = false, chunk_seg_first = true;
    if (n > 0) {
      mbar_wait(&bars[X_XFULL], 0);
      conv_z(0, s_meta[0].nrows);
    }
    for (int i = 0; i < n; ++i) {
      TRW(0);
      work_wait(&bars[X_G1_DONE], i & 1);
      TRW(1);
      const TileMeta mt = s_meta[i & 3];
      float v[32];
      {
        uint32_t rr[32];
        tmem_ld32(tmem + kX4LP + 128 * (i & 1) + lane_base + 32 * h, rr);
        tmem_ld_wait(rr);
#pragma unroll
        for (int c = 0; c < 32; ++c) v[c] = __uint_as_float(rr[c]) + bias;
      }
      if (p.gamma_mode == 2) {
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const int r = 32 * h + c;
          if (r < mt.nrows && gj < p.K) p.gamma_out[(size_t)(mt.row0 + r) * p.K + gj] = v[c];
        }
      }
      TRW(2);
      // per-descriptor max over the warp's Gaussians (redux), exponentials against it, lane c keeps m_c
      float my_m = -3.0e38f;
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        const float m = redux_max(v[c]);
        v[c] = ex2_approx(v[c] - m);
        if (lane == c) my_m = m;
      }
      TRW(5);
      // ---- GEMM2(i-1) done: S'^T chunk complete (fold), Z buffer (i+1) & 1 free
      if (i >= 1) {
        work_wait(&bars[X_G2_DONE], (i - 1) & 1);
        TRW(6);
        if (prev_fold) {
          fold(prev_b, chunk_seg_first);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bars[X_FOLD_DONE]);
        }
      }
      if (mt.flags & 2) chunk_seg_first = (mt.flags & 8) != 0;
      TRW(7);
      if (i + 1 < n) {
        mbar_wait(&bars[X_XFULL], (i + 1) & 1);
        TRW(8);
        conv_z(i + 1, s_meta[(i + 1) & 3].nrows);
      }
      TRW(9);
      TRW(3);
      // per-descriptor sums over the warp's Gaussians: lane l ends with s of descriptor 32h + l
      float my_s;
      {
        float t[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) t[c] = v[c];
        warp_transpose_reduce32(t, lane);
        my_s = t[0];
      }
      TRW(4);
      const int par = i & 1;
      float2 *xb = s_xchg + par * (kMaxC2 * 4 * kTileM);
      const int drow = 32 * h + lane;  // descriptor carried by this lane in the exchange
      if (C == 1) {
        xb[(rank * 4 + q) * kTileM + drow] = make_float2(my_m, my_s);
      } else {
        if (warp == 0 && lane == 0) mbar_arrive_expect_tx(&bars[X_XCHG0 + par], C * 4 * kTileM * 8);
        const uint32_t my = smem_u32(&xb[(rank * 4 + q) * kTileM + drow]);
        const uint32_t mybar = smem_u32(&bars[X_XCHG0 + par]);
        for (uint32_t r2 = 0; r2 < C; ++r2) st_async_v2f32(mapa_shared(my, r2), my_m, my_s, mapa_shared(mybar, r2));
      }
      // ---- exchange: (M, S) of descriptor drow over the 4C Gaussian blocks
      if (C > 1) mbar_wait(&bars[X_XCHG0 + par], (i >> 1) & 1);
      else named_bar_sync(kBarXchgLocal, kWarpsWork * 32);
      TRW(10);
      float M = -3.0e38f, S = 0.f;
      {
        float2 o[kMaxC2 * 4];
#pragma unroll
        for (int e = 0; e < kMaxC2 * 4; ++e) {
          o[e] = make_float2(-3.0e38f, 0.f);
          if (e < (int)C * 4) { o[e] = xb[e * kTileM + drow]; M = fmaxf(M, o[e].x); }
        }
#pragma unroll
        for (int e = 0; e < kMaxC2 * 4; ++e) S += o[e].y * ex2_approx(o[e].x - M);
      }
      if (p.loglik_out && q == 0 && rank == 0 && drow < mt.nrows) p.loglik_out[mt.row0 + drow] = M + log2f(S);
      float alpha = __fdividef(ex2_approx(my_m - M), S) * kPScale;
      if (drow >= mt.nrows) alpha = 0.f;
      bc[lane] = alpha;
      __syncwarp();
      // ---- P^T(i) = gamma 2^14 (thresholded) -> fp16 hi/lo pairs of descriptors, in place of L^T(i)
      uint32_t hi[16], lo[16];
#pragma unroll
      for (int c4 = 0; c4 < 8; ++c4) {
        const float4 a4 = *reinterpret_cast<const float4 *>(bc + 4 * c4);
        float2 g0 = __fmul2_rn(make_float2(v[4 * c4], v[4 * c4 + 1]), make_float2(a4.x, a4.y));
        float2 g1 = __fmul2_rn(make_float2(v[4 * c4 + 2], v[4 * c4 + 3]), make_float2(a4.z, a4.w));
        if (thr > 0.f) {
          g0 = __fmul2_rn(g0, make_float2(set_gt(g0.x, thr), set_gt(g0.y, thr)));
          g1 = __fmul2_rn(g1, make_float2(set_gt(g1.x, thr), set_gt(g1.y, thr)));
        }
        s0 += (g0.x + g0.y) + (g1.x + g1.y);
        if (p.gamma_mode == 1) {
          const float gg[4] = {g0.x, g0.y, g1.x, g1.y};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int r = 32 * h + 4 * c4 + e;
            if (r < mt.nrows && gj < p.K) p.gamma_out[(size_t)(mt.row0 + r) * p.K + gj] = gg[e] * (1.f / kPScale);
          }
        }
        split2_f16(g0, hi[2 * c4], lo[2 * c4]);
        split2_f16(g1, hi[2 * c4 + 1], lo[2 * c4 + 1]);
      }
      TRW(11);
      const uint32_t pt = tmem + kX4LP + 128 * (i & 1) + lane_base + 16 * h;
      tmem_st16(pt, hi);
      tmem_st16(pt + 64, lo);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[X_P_FULL]);
      TRW(12);
      if (mt.flags & 1) {  // segment end: S0 partial of Gaussian g over this warp's descriptor block h
        p.s0slots[((size_t)seg_slot(cid, mt.b) * 4 + h) * p.Kp + gj] = s0;
        s0 = 0.f;
      }
      prev_b = mt.b;
      prev_fold = (mt.flags & 4) != 0;
    }
    if (n > 0) {
      work_wait(&bars[X_G2_DONE], (n - 1) & 1);
      fold(prev_b, chunk_seg_first);
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) tmem_dealloc(tmem, kTmemCols);
}

}  // namespace gpufv
