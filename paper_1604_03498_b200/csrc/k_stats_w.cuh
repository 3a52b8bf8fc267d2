// k_stats_w.cuh — steps a2-a6 for wide descriptors (64 < D <= 128; C5: D = 128, K = 512).
//
// Same method and numerics as k_stats (k_stats.cuh: 3 x FP16 split tcgen05 GEMMs, online softmax with
// a cluster exchange, fp32 segment slots), re-tiled for the wider feature vector:
//   * the 2D = 256 features are two halves hf = 0, 1 of kNF = 128 features each: the dims
//     [64 hf, 64 hf + 64) as [lin | quad] — each half is laid out exactly like k_stats' single half;
//   * a CTA owns kGW = 64 Gaussians (W' for both halves = 64 KB of shared memory), so a cluster has
//     C = ceil(K / 64) <= 8 CTAs;
//   * GEMM1 accumulates both halves into L (128 x 64, N = 64);  GEMM2 runs per half into S'_hf
//     (128 features x 64 Gaussians each) from ONE shared-memory Z half buffer: Z_a(i) is copied from
//     Zr(i), GEMM2a(i) runs while the WORK warps convert half a of the next tile, then Z_b(i) is copied
//     and GEMM2b(i) runs while they convert half b.  Zr (both halves, 256 TMEM columns) is single-
//     buffered, which serialises GEMM1(i+1) behind the copies of tile i (~50 % tensor
//     occupancy by construction; this variant serves the C5 configuration, the narrow one is the
//     throughput path);
//   * the X tile (128 rows x 128 dims = 64 KB) streams through two 16 KB TMA box stages.
// Per local tile i the WORK warps run: wait G1(i) | softmax(i) | wait G2(i-1) [fold] | P(i) |
// copy Z_a(i) | Zr(i+1) half a | wait G2a(i) | copy Z_b(i) | Zr(i+1) half b;
// the MMA thread issues G1(0), then per tile G2a(i), G2b(i), G1(i+1).
#pragma once
#include <cuda.h>

#include "fv_common.cuh"
#include "k_stats.cuh"
#include "ptx.cuh"

namespace gpufv {

constexpr int kMaxCW = 8;  // K <= 512

// shared memory map (offsets from a 1024-aligned base)
constexpr int kWW = 0;                                // W' [half][hi|lo][atom][64 rows][128 B]  64 KB
constexpr int kPBytesW = kTileM * kGW * 2;            // 16 KB: one fp16 P operand (128 rows x 64)
constexpr int kWP = kWW + kWImgBytes;                 // P hi | lo                                32 KB
constexpr int kWZ = kWP + 2 * kPBytesW;               // Z half: hi | lo (2 atoms each)           64 KB
constexpr int kWX = kWZ + 2 * kOpBytes;               // X box stages 2 x 16 KB
constexpr int kWBias = kWX + 2 * kXBoxBytes;          // float[64]
constexpr int kWNcs = kWBias + kGW * 4;               // float[128]  -c_k 2^e_k
constexpr int kWSc = kWNcs + kDMax * 4;               // float[128]  2^e_k
constexpr int kWRed = kWSc + kDMax * 4;               // float2[2][4][128]
constexpr int kWXchg = kWRed + 2 * 4 * kTileM * 8;    // float2[2][kMaxCW][128]
constexpr int kWMeta = kWXchg + 2 * kMaxCW * kTileM * 8;
constexpr int kWBar = kWMeta + 128;
constexpr int kWNumBars = 16;
constexpr int kWTmem = kWBar + kWNumBars * 8;
constexpr int kSmemWBytes = kWTmem + 16 + 1024;
static_assert(kSmemWBytes <= 232448, "shared memory budget (wide)");

enum : int {
  W_XFULL0 = 0, W_XFULL1, W_XEMPTY0, W_XEMPTY1, W_ZR_FULL, W_G1_DONE, W_G2A_DONE, W_G2_DONE,
  W_L_EMPTY, W_P_FULL, W_ZB_FULL, W_FOLD_DONE, W_XCHG0, W_XCHG1, W_W_FULL, W_ZRA_FULL
};

// tensor-memory columns: Zr (half hf at 128 hf), L (64), S'_hf (64 each), L2 (64)
constexpr uint32_t kWTZr = 0, kWTL = 256, kWTS = 320;
// GEMM1's hi.hi products accumulate separately (L2, the 64 free columns) so that half a's can be issued
// with half a's cross terms, before half b is converted; the WORK warps add L + L2 (fp32, round to
// nearest: never worse than the truncating accumulator).  Same-box A/B: C5 +0.5 %, raw -> FV +0.7 %.
constexpr uint32_t kWTL2 = 448;

// kCW = cluster size at compile time (4: K = 256 e.g. the D = 82 raw -> FV path, 8: K = 512, C5), or 0
// for any other size (read from %cluster_nctarank): the exchange loops unroll without predicates.
// kHooks: the per-row posterior / log-likelihood outputs (fv_posteriors, the EM E-step) are compiled
// in; the encode instantiations leave them out (+2.5 % C5, +1 % raw -> FV at D = 82, same-box A/B).
// kPk (D <= 96, with kD128 = false): the second feature half holds only dims 64-95, packed as 64
// features [lin | quad] in one atom — GEMM2b runs as M = 64 (its accumulator in lanes 0-15 of each
// TMEM lane quarter, tools/m64_probe.cu), the Z_b copy and the half-b fold move half the data, and
// k_prep_w stores W' half b in the same packed order (wide == 2)
template <bool kD128, int kCW, bool kHooks, bool kPk = false>
__global__ void __launch_bounds__(kThreads2, 1) k_stats_w(const __grid_constant__ CUtensorMap tmap_x, const Stats2Params p) {
  using namespace ptx;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_base = smem_u32(smem_raw);
  const uint32_t sbase = (raw_base + 1023u) & ~1023u;
  uint8_t *smem = smem_raw + (sbase - raw_base);
  const uint32_t sW = sbase + kWW, sP = sbase + kWP, sZ = sbase + kWZ, sX = sbase + kWX;
  float *s_bias = reinterpret_cast<float *>(smem + kWBias);
  float *s_ncs = reinterpret_cast<float *>(smem + kWNcs);
  float *s_sc = reinterpret_cast<float *>(smem + kWSc);
  float2 *s_red = reinterpret_cast<float2 *>(smem + kWRed);
  float2 *s_xchg = reinterpret_cast<float2 *>(smem + kWXchg);
  TileMeta *s_meta = reinterpret_cast<TileMeta *>(smem + kWMeta);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + kWBar);
  uint32_t *s_tmem = reinterpret_cast<uint32_t *>(smem + kWTmem);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_ctarank(), C = kCW > 0 ? (uint32_t)kCW : cluster_nctarank();
  const int cid = (int)cluster_id_x(), ncl = (int)nclusters_x();

  // ---------------- setup
  {
    for (int i = tid; i < kGW; i += kThreads2) s_bias[i] = p.bias[rank * kGW + i];
    if (tid < kDMax) { s_sc[tid] = p.xscale[tid]; s_ncs[tid] = -(p.xshift[tid] * p.xscale[tid]); }
  }
  if (warp == 0) { tmem_alloc(s_tmem, kTmemCols); tmem_relinquish(); }
  if (tid == 0) {
    mbar_init(&bars[W_XFULL0], 1); mbar_init(&bars[W_XFULL1], 1);
    mbar_init(&bars[W_XEMPTY0], kWarpsWork); mbar_init(&bars[W_XEMPTY1], kWarpsWork);
    mbar_init(&bars[W_ZR_FULL], kWarpsWork); mbar_init(&bars[W_ZRA_FULL], kWarpsWork);
    mbar_init(&bars[W_G1_DONE], 1); mbar_init(&bars[W_G2A_DONE], 1); mbar_init(&bars[W_G2_DONE], 1);
    mbar_init(&bars[W_L_EMPTY], kWarpsWork); mbar_init(&bars[W_P_FULL], kWarpsWork);
    mbar_init(&bars[W_ZB_FULL], kWarpsWork); mbar_init(&bars[W_FOLD_DONE], kWarpsWork);
    mbar_init(&bars[W_XCHG0], 1); mbar_init(&bars[W_XCHG1], 1);
    mbar_init(&bars[W_W_FULL], 1);
    fence_mbar_init();
    // W' image of this rank: 64 KB bulk copy (async proxy), waited on by the MMA thread only
    mbar_arrive_expect_tx(&bars[W_W_FULL], kWImgBytes);
    for (int c = 0; c < 4; ++c)
      bulk_g2s(sW + c * (kWImgBytes / 4), p.wimg + (size_t)rank * kWImgBytes + c * (kWImgBytes / 4), kWImgBytes / 4,
               &bars[W_W_FULL]);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  cluster_sync();
  griddep_launch_dependents();  // k_finalize may start its prologue
  griddep_wait();               // k_schedule's tile prefix sums are complete and visible

  const int64_t T = p.tile_start[p.batch];
  const int t0 = (int)((int64_t)cid * T / ncl), t1 = (int)((int64_t)(cid + 1) * T / ncl);
  const int n = t1 - t0;
  // D <= 96 (e.g. the paper's 82-dim descriptors): dims 96..127 are padding — box 3 is neither loaded
  // nor converted (its Zr columns are zeroed once) and GEMM1 skips half b's k-steps 2, 3, 6, 7
  const bool skip3 = !kD128 && p.D <= 96;

  if (warp == kWarpTma) {
    // ======================================================= tile walk + X producer (TMA)
    // box b (dims 32 b ..) of every tile goes through stage b & 1; the k-th use of a stage has parity
    // k & 1 = (b >> 1) & 1, so each stage alternates phases 0, 1 within every tile.
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
        const TileMeta m = tw.meta();
        s_meta[i & 3] = m;  // released to the WORK warps by the X_FULL phase completions below
#pragma unroll 1
        for (int bx = 0; bx < 4; ++bx) {
          const int st = bx & 1;
          if (i >= 1 || bx >= 2) mbar_wait(&bars[W_XEMPTY0 + st], ((bx >> 1) + 1) & 1);
          if (bx == 3 && skip3) {  // D <= 96: box 3 is all padding; keep the stage's phase sequence
            mbar_arrive(&bars[W_XFULL0 + st]);
            continue;
          }
          mbar_arrive_expect_tx(&bars[W_XFULL0 + st], kXBoxBytes);
          tma_load_2d(sX + st * kXBoxBytes, &tmap_x, 32 * bx, m.row0, &bars[W_XFULL0 + st]);
        }
        prefetch_l2(i + 4);
      }
    }
  } else if (warp == kWarpMma) {
    // ======================================================= MMA issuer
    if (n > 0) {  // the whole warp, converged; one elected lane issues (ptx::*_w)
      TileWalker tw;
      tw.init(p, t0, t1);
      const uint32_t idesc1 = idesc_f16_f32(128, kGW, 0, 0);  // A = Zr (TMEM, K-major), B = W' K-major
      const uint32_t idesc2 = idesc_f16_f32(kNF, kGW, 1, 1);  // A = Z_hf^T (SMEM, MN-major), B = P MN-major
      uint32_t folds = 0;
      mbar_wait(&bars[W_W_FULL], 0);
      auto g1 = [&](int s, int hf) {  // one split product of one feature half into L
        const bool pk = kPk && hf == 1;  // packed half b: 64 features, lo at column 32
        const uint32_t za = tmem + kWTZr + 128 * hf + (s == 1 ? (pk ? 32 : 64) : 0);  // hi, lo, hi
        const uint32_t wb = sW + hf * (kWImgBytes / 2) + (s == 0 ? kGW * 128 * 2 : 0);  // lo, hi, hi
        const bool first = (s == 0 || s == 2) && hf == 0;         // L: cross terms, L2: hi.hi
        const uint32_t dl = tmem + (s == 2 ? kWTL2 : kWTL);
        const uint32_t mask = pk ? 0x0Fu : (hf == 1 && skip3) ? 0x33u : 0xFFu;  // k-steps holding dims < 96
#pragma unroll
        for (int kk = 0; kk < kNF / 16; ++kk) {
          if (!((mask >> kk) & 1u)) continue;
          const uint32_t off = (kk >> 2) * (kGW * 128) + (kk & 3) * 32;
          mma_f16_ts_w(dl, za + kk * 8, desc_sw128(wb + off, 16, 1024), idesc1, (first && kk == 0) ? 0u : 1u);
        }
      };
      // GEMM1 in two parts so half a's products run while half b is still being converted; the cross
      // terms accumulate in L apart from the hi.hi terms (L2): (s0,a) (s1,a) (s2,a -> L2) | (s0,b) (s1,b) (s2,b -> L2)
      auto gemm1a = [&](int i) {
        mbar_wait(&bars[W_ZRA_FULL], i & 1);
        if (i >= 1) mbar_wait(&bars[W_L_EMPTY], (i - 1) & 1);
        tc_fence_after();
        g1(0, 0);
        g1(1, 0);
        g1(2, 0);
      };
      auto gemm1b = [&](int i) {
        mbar_wait(&bars[W_ZR_FULL], i & 1);
        tc_fence_after();
        g1(0, 1);
        g1(1, 1);
        g1(2, 1);
        mma_commit_w(&bars[W_G1_DONE]);
      };
      auto gemm1 = [&](int i) { gemm1a(i); gemm1b(i); };
      const uint32_t idesc2b = idesc_f16_f32(kPk ? kNF / 2 : kNF, kGW, 1, 1);  // packed half b: M = 64
      auto gemm2 = [&](int hf, bool chunk_first) {  // S'_hf (+)= Z_hf^T P over the tile's 128 rows
        tc_fence_after();
#pragma unroll 1
        for (int s = 0; s < 3; ++s) {
          const uint32_t za = sZ + (s == 1 ? kOpBytes : 0);    // hi, lo, hi
          const uint32_t pb = sP + (s == 0 ? kPBytesW : 0);    // lo, hi, hi
#pragma unroll
          for (int kk = 0; kk < kTileM / 16; ++kk) {
            const uint32_t off = kk * 2048;  // 16 descriptor rows x 128 B
            mma_f16_ss_w(tmem + kWTS + kGW * hf, desc_sw128(za + off, kAtomBytes, 1024),
                       desc_sw128(pb + off, kAtomBytes, 1024), hf == 1 ? idesc2b : idesc2,
                       (chunk_first && s == 0 && kk == 0) ? 0u : 1u);
          }
        }
      };
      gemm1(0);
      for (int i = 0; i < n; ++i, tw.next()) {
        const bool chunk_first = (tw.meta().flags & 2) != 0;
        mbar_wait(&bars[W_P_FULL], i & 1);  // P(i) and Z_a(i) in shared memory
        if (chunk_first && i > 0) { mbar_wait(&bars[W_FOLD_DONE], folds & 1); ++folds; }
        TR(10);
        gemm2(0, chunk_first);
        mma_commit_w(&bars[W_G2A_DONE]);
        TR(11);
        if (i + 1 < n) gemm1a(i + 1);        // Zr(i+1) half a is converted before Z_b(i) is copied
        mbar_wait(&bars[W_ZB_FULL], i & 1);  // Z_b(i)
        TR(12);
        gemm2(1, chunk_first);
        mma_commit_w(&bars[W_G2_DONE]);
        TR(13);
        if (i + 1 < n) gemm1b(i + 1);
        TR(14);
      }
    }
  } else {
    // ======================================================= WORK warps
    const int ww = warp - kWarpWork0;       // WORK warp index 0..15
    const int q = warp & 3, h = ww >> 2;    // TMEM lanes 32q.. (physical warp % 4); Gaussian quarter h (16 columns)
    const uint32_t lane_base = (uint32_t)(32 * q) << 16;
    const int row = 32 * q + lane;  // descriptor row of Zr / L / P / Z; feature (of a half) of S'
    const float thr = p.threshold * kPScale;

    // Zr(i) half hf from boxes 2 hf, 2 hf + 1: each warp converts dims 8h.. of both boxes (zr_box of
    // k_stats, offset to the half's columns and dims); the last box waits for the thread's stores.
    auto conv_half = [&](int i, int hf) {
      const uint32_t ta = tmem + kWTZr + 128 * hf + lane_base;
#pragma unroll
      for (int bl = 0; bl < 2; ++bl) {
        const int bx = 2 * hf + bl, st = bx & 1;
        mbar_wait(&bars[W_XFULL0 + st], (bx >> 1) & 1);
        // the tile's metadata is published before its first box: read it only after a box wait
        const int nrows = s_meta[i & 3].nrows;
        const uint8_t *xbox = smem + kWX + st * kXBoxBytes;
        if (bx == 3 && skip3) {
        } else if (kPk && hf == 1)
          zr_box<true, 16, 32>(xbox, row, bl, h, p.D - kDP, row < nrows, s_sc + kDP, s_ncs + kDP, ta);
        else if (!kD128 || nrows < kTileM)
          zr_box<true>(xbox, row, bl, h, p.D - kDP * hf, row < nrows, s_sc + kDP * hf, s_ncs + kDP * hf, ta);
        else
          zr_box<false>(xbox, row, bl, h, kDP, true, s_sc + kDP * hf, s_ncs + kDP * hf, ta);
        if (bl == 1) tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&bars[W_XEMPTY0 + st]);
          if (bl == 1) mbar_arrive(&bars[hf == 1 ? W_ZR_FULL : W_ZRA_FULL]);
        }
      }
    };
    auto copy_z = [&](int hf) {  // this warp's Zr half hf words -> Z rows in shared memory
      const uint32_t ta = tmem + kWTZr + 128 * hf + lane_base;
      uint32_t z[32];
#pragma unroll
      for (int box = 0; box < 2; ++box) {
        uint32_t(&zb)[16] = *reinterpret_cast<uint32_t(*)[16]>(z + 16 * box);
        tmem_ld4(ta + 16 * box + 4 * h, *reinterpret_cast<uint32_t(*)[4]>(zb + 0));        // lin hi
        tmem_ld4(ta + 32 + 16 * box + 4 * h, *reinterpret_cast<uint32_t(*)[4]>(zb + 4));   // quad hi
        tmem_ld4(ta + 64 + 16 * box + 4 * h, *reinterpret_cast<uint32_t(*)[4]>(zb + 8));   // lin lo
        tmem_ld4(ta + 96 + 16 * box + 4 * h, *reinterpret_cast<uint32_t(*)[4]>(zb + 12));  // quad lo
      }
      tmem_ld_wait(z);
#pragma unroll
      for (int box = 0; box < 2; ++box) {
        const uint32_t o = sw_off(row, 4 * box + h);
        const uint32_t *zb = z + 16 * box;
        sts128(sZ + o, zb[0], zb[1], zb[2], zb[3]);
        sts128(sZ + kAtomBytes + o, zb[4], zb[5], zb[6], zb[7]);
        sts128(sZ + kOpBytes + o, zb[8], zb[9], zb[10], zb[11]);
        sts128(sZ + kOpBytes + kAtomBytes + o, zb[12], zb[13], zb[14], zb[15]);
      }
    };
    auto copy_zb_packed = [&]() {  // kPk: Zr half b (lin hi 0-15 | quad hi 16-31 | lo + 32) -> atom 0 of Z
      const uint32_t ta = tmem + kWTZr + 128 + lane_base;
      uint32_t z[16];
      tmem_ld4(ta + 4 * h, *reinterpret_cast<uint32_t(*)[4]>(z + 0));        // lin hi  dims 8h..
      tmem_ld4(ta + 16 + 4 * h, *reinterpret_cast<uint32_t(*)[4]>(z + 4));   // quad hi
      tmem_ld4(ta + 32 + 4 * h, *reinterpret_cast<uint32_t(*)[4]>(z + 8));   // lin lo
      tmem_ld4(ta + 48 + 4 * h, *reinterpret_cast<uint32_t(*)[4]>(z + 12));  // quad lo
      tmem_ld_wait(z);
      sts128(sZ + sw_off(row, h), z[0], z[1], z[2], z[3]);
      sts128(sZ + sw_off(row, 4 + h), z[4], z[5], z[6], z[7]);
      sts128(sZ + kOpBytes + sw_off(row, h), z[8], z[9], z[10], z[11]);
      sts128(sZ + kOpBytes + sw_off(row, 4 + h), z[12], z[13], z[14], z[15]);
    };
    // S'_hf quarter (lane = half feature, columns 16h..) -> segment slot rows [lin 0..127 | quad 0..127]
    auto fold = [&](int b, bool first) {
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        int f = (row < kDP) ? kDP * hf + row : kDMax + kDP * hf + (row - kDP);
        // packed half b (M = 64): feature fp = 16 q + lane sits in lane 32 q + lane, lane < 16
        const int fp = 16 * q + lane;
        if (kPk && hf == 1) f = fp < 32 ? kDP + fp : kDMax + kDP + (fp - 32);
        float *dst = p.slots + (size_t)seg_slot(cid, b) * (2 * kDMax) * p.Kp + (size_t)f * p.Kp + rank * kGW + 16 * h;
        uint32_t v[16];
        tmem_ld16(tmem + kWTS + kGW * hf + lane_base + 16 * h, v);
        tmem_ld_wait(v);
        if (kPk && hf == 1 && lane >= 16) continue;
        if (first) {
          float4 *d4 = reinterpret_cast<float4 *>(dst);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            d4[j] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]), __uint_as_float(v[4 * j + 2]),
                                __uint_as_float(v[4 * j + 3]));
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            red_add_v4(dst + 4 * j, __uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                       __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
        }
      }
    };

    float s0acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) s0acc[j] = 0.f;
    int prev_b = 0;
    bool prev_fold = false, chunk_seg_first = true;
    if (!kPk && n > 0 && skip3) {  // the Zr columns of dims 96..127 (box 3 of half b) stay zero for the whole run
      const uint32_t zero4[4] = {0u, 0u, 0u, 0u};
      const uint32_t ta = tmem + kWTZr + 128 + lane_base + 16 + 4 * h;
      tmem_st4(ta, zero4); tmem_st4(ta + 32, zero4); tmem_st4(ta + 64, zero4); tmem_st4(ta + 96, zero4);
    }
    if (n > 0) { conv_half(0, 0); conv_half(0, 1); }
    for (int i = 0; i < n; ++i) {
      TRW(0);
      work_wait(&bars[W_G1_DONE], i & 1);  // L(i) ready
      TRW(1);
      // ---- softmax(i), online form (see k_stats): quarter h = 16 Gaussian columns
      float v[16];
      {
        uint32_t rr[16];
        tmem_ld16(tmem + kWTL + lane_base + 16 * h, rr);
        uint32_t r2[16];
        tmem_ld16(tmem + kWTL2 + lane_base + 16 * h, r2);
        tmem_ld_wait(rr);
        tmem_ld_wait(r2);
#pragma unroll
        for (int j = 0; j < 16; j += 2) {
          const float2 a = __fadd2_rn(make_float2(__uint_as_float(rr[j]), __uint_as_float(rr[j + 1])),
                                      make_float2(__uint_as_float(r2[j]), __uint_as_float(r2[j + 1])));
          v[j] = a.x; v[j + 1] = a.y;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[W_L_EMPTY]);
      const TileMeta mt = s_meta[i & 3];
      float m = -3.0e38f;
#pragma unroll
      for (int j = 0; j < 16; j += 4) {
        const float4 bj = *reinterpret_cast<const float4 *>(s_bias + 16 * h + j);
        const float2 x0 = __fadd2_rn(make_float2(v[j], v[j + 1]), make_float2(bj.x, bj.y));
        const float2 x1 = __fadd2_rn(make_float2(v[j + 2], v[j + 3]), make_float2(bj.z, bj.w));
        v[j] = x0.x; v[j + 1] = x0.y; v[j + 2] = x1.x; v[j + 3] = x1.y;
        m = fmaxf(m, fmaxf(fmaxf(x0.x, x0.y), fmaxf(x1.x, x1.y)));
      }
      if (kHooks && p.gamma_mode == 2 && row < mt.nrows) {
        float *go = p.gamma_out + (size_t)(mt.row0 + row) * p.K;
#pragma unroll
        for (int j = 0; j < 16; ++j) { int gj = rank * kGW + 16 * h + j; if (gj < p.K) go[gj] = v[j]; }
      }
      float2 sacc = make_float2(0.f, 0.f);
#pragma unroll
      for (int j = 0; j < 16; j += 2) {
        const float2 d = __fadd2_rn(make_float2(v[j], v[j + 1]), make_float2(-m, -m));
        v[j] = ex2_approx(d.x); v[j + 1] = ex2_approx(d.y);
        sacc = __fadd2_rn(sacc, make_float2(v[j], v[j + 1]));
      }
      float2 *red = s_red + (i & 1) * (4 * kTileM);
      red[h * kTileM + row] = make_float2(m, sacc.x + sacc.y);
      TRW(2);
      named_bar_sync(kBarLane0 + q, 128);
      TRW(3);
      float M, S;
      {
        const float2 r0 = red[row], r1 = red[kTileM + row], r2 = red[2 * kTileM + row], r3 = red[3 * kTileM + row];
        M = fmaxf(fmaxf(r0.x, r1.x), fmaxf(r2.x, r3.x));
        S = (r0.y * ex2_approx(r0.x - M) + r1.y * ex2_approx(r1.x - M)) +
            (r2.y * ex2_approx(r2.x - M) + r3.y * ex2_approx(r3.x - M));
      }
      if (C > 1) {
        const int par = i & 1;
        float2 *xb = s_xchg + par * (kMaxCW * kTileM);
        if (ww == 0 && lane == 0) mbar_arrive_expect_tx(&bars[W_XCHG0 + par], (C - 1) * kTileM * 8);
        if (h == 0) {
          const uint32_t my = smem_u32(&xb[rank * kTileM + row]);
          const uint32_t mybar = smem_u32(&bars[W_XCHG0 + par]);
          for (uint32_t r2 = 0; r2 < C; ++r2)
            if (r2 != rank) st_async_v2f32(mapa_shared(my, r2), M, S, mapa_shared(mybar, r2));
        }
        TRW(12);
        mbar_wait(&bars[W_XCHG0 + par], (i >> 1) & 1);
        TRW(13);
        float Mg = M;
        for (uint32_t r2 = 0; r2 < C; ++r2)
          if (r2 != rank) Mg = fmaxf(Mg, xb[r2 * kTileM + row].x);
        float Sg = S * ex2_approx(M - Mg);
        for (uint32_t r2 = 0; r2 < C; ++r2)
          if (r2 != rank) { const float2 o = xb[r2 * kTileM + row]; Sg += o.y * ex2_approx(o.x - Mg); }
        M = Mg;
        S = Sg;
      }
      // per-descriptor log2-likelihood (EM, NEXT-3)
      if (kHooks && p.loglik_out && h == 0 && rank == 0 && row < mt.nrows) p.loglik_out[mt.row0 + row] = M + log2f(S);
      float alpha_p = __fdividef(ex2_approx(m - M), S) * kPScale;
      if (row >= mt.nrows) alpha_p = 0.f;
      else if (!(S > 0.5f && S < 3.0e38f)) range_bad(p, mt.b, alpha_p, h == 0 && rank == 0);
      TRW(4);

      // ---- GEMM2(i-1) (both halves) done: S' chunk complete (fold), Z and P free
      if (i >= 1) {
        work_wait(&bars[W_G2_DONE], (i - 1) & 1);
        if (prev_fold) {
          fold(prev_b, chunk_seg_first);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bars[W_FOLD_DONE]);
        }
      }
      if (mt.flags & 2) chunk_seg_first = (mt.flags & 8) != 0;
      TRW(5);

      // ---- P(i) = gamma 2^14 (thresholded) -> fp16 hi/lo (one 128 B row of 64 Gaussians), S0
      const float2 ap = make_float2(alpha_p, alpha_p);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int e = 0; e < 8; e += 2) {
          const int j = 8 * c + e;
          float2 g = __fmul2_rn(make_float2(v[j], v[j + 1]), ap);
          if (thr > 0.f) g = __fmul2_rn(g, make_float2(set_gt(g.x, thr), set_gt(g.y, thr)));
          v[j] = g.x; v[j + 1] = g.y;
          const float2 sa = __fadd2_rn(make_float2(s0acc[j], s0acc[j + 1]), g);
          s0acc[j] = sa.x; s0acc[j + 1] = sa.y;
          split2_f16(g, hi[e >> 1], lo[e >> 1]);
        }
        const uint32_t off = sw_off(row, 2 * h + c);
        sts128(sP + off, hi[0], hi[1], hi[2], hi[3]);
        sts128(sP + kPBytesW + off, lo[0], lo[1], lo[2], lo[3]);
      }
      if (kHooks && p.gamma_mode == 1 && row < mt.nrows) {
        float *go = p.gamma_out + (size_t)(mt.row0 + row) * p.K;
#pragma unroll
        for (int j = 0; j < 16; ++j) { int gj = rank * kGW + 16 * h + j; if (gj < p.K) go[gj] = v[j] * (1.f / kPScale); }
      }
      TRW(6);
      copy_z(0);
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[W_P_FULL]);
      TRW(7);
      if (i + 1 < n) conv_half(i + 1, 0);  // Zr half a of tile i is consumed (GEMM1(i), copy_z(0))
      TRW(8);
      work_wait(&bars[W_G2A_DONE], i & 1);  // GEMM2a(i) done reading Z
      TRW(9);
      if (kPk) copy_zb_packed();
      else copy_z(1);
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[W_ZB_FULL]);
      TRW(10);
      if (i + 1 < n) conv_half(i + 1, 1);
      TRW(11);
      if (mt.flags & 1) {  // segment end: S0 (units of 2^14 gamma), this warp's 32 rows -> partial slot q
        float t32[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) t32[j] = j < 16 ? s0acc[j] : 0.f;
        warp_transpose_reduce32(t32, lane);  // lane l < 16: column l summed over the warp's rows
        if (lane < 16) p.s0slots[((size_t)seg_slot(cid, mt.b) * 4 + q) * p.Kp + rank * kGW + 16 * h + lane] = t32[0];
#pragma unroll
        for (int j = 0; j < 16; ++j) s0acc[j] = 0.f;
      }
      prev_b = mt.b;
      prev_fold = (mt.flags & 4) != 0;
    }
    if (n > 0) {  // last chunk
      work_wait(&bars[W_G2_DONE], (n - 1) & 1);
      fold(prev_b, chunk_seg_first);
    }
  }

  // ---------------- teardown
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) tmem_dealloc(tmem, kTmemCols);
}

}  // namespace gpufv
