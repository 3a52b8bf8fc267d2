// k_stats.cuh — steps a2-a6 of the hot path in one persistent, warp-specialised kernel.
//
//   a2  X tile (128 descriptors x 64 dims) arrives as two TMA boxes (32 dims x 128 rows, 128B-swizzled)
//       through a single 16 KB stage; the features Z = [(x-c) 2^e, ((x-c) 2^e)^2] are split into fp16
//       hi/lo once and written to tensor memory Zr[t % 2] (lanes = descriptors: GEMM1's A operand)
//   a3  GEMM1  L[i,j] = Zr_i . W'_j   (tcgen05 TS-MMA, 3 x FP16 split: hi.lo + lo.hi + hi.hi, fp32 TMEM)
//       = log2 of the Alg.1 l.4-5 log-likelihood in expanded form, up to the bias b_j
//   a4  softmax epilogue: gamma_ij = 2^(L_ij + b_j - m_i) / s_i with the row max/sum reduced over the
//       CTA's 4 column quarters and over the cluster's Gaussian blocks (DSMEM st.async exchange)
//       (Alg.1 l.6-14); gamma <= tau zeroed (Alg.1 l.18); rows past the image end
//       masked; P = gamma 2^14 split fp16 hi/lo into shared memory; S0_j = sum_i gamma_ij in registers
//   a5  GEMM2  S'[f,j] += sum_i Z[i,f] P[i,j]  (tcgen05 SS-MMA, A = Z copied from Zr into shared memory,
//       MN-major; 3 x FP16 split) — the U/V accumulation of Alg.1 l.16-26 as moments;
//       restarted every kFold tiles (the tensor-core fp32 accumulator truncates)
//   a6  every kFold tiles and at each (cluster, image) segment end: S' -> an append-only partial slot
//       in HBM; S0 -> an S0 slot at the segment end (the paper's per-block U/V copies)
//
// Roles (576 threads = 18 warps, 1 CTA per SM, cluster of C = ceil(K/128) CTAs, rank r owns Gaussians
// [128 r, 128 r + 128)):
//   warps 0-15  WORK: warp w = (q = w%4, h = w/4) owns TMEM lanes 32q.. (tcgen05.ld/st lane rule) and a
//               quarter h of the rest: softmax over Gaussian columns 32h.., the features of dims 16h..
//               (box h/2 of the X tile), the fold of S' columns 32h..
//   warp  16    MMA : one thread issues every tcgen05.mma / commit
//   warp  17    TMA : one thread walks the tile list, publishes tile metadata in shared memory, loads
//               the X boxes (each after the previous box is released) and prefetches 4 tiles into L2
// (Registers: a block's warps are spread over the 4 SM sub-partitions of 16K registers each, so
//  ceil(warps / 4) * regs_per_thread <= 512 (measured: 88 regs -> 640 threads, 104 -> 512); 18 warps
//  can use 96 registers.)
// Per local tile i the WORK warps run: wait G1(i) | Zr(i+1) | softmax(i) | wait G2(i-1) | [fold] |
// copy Zr(i) -> Z | P(i); the MMA thread issues G1(0), then G1(i+1), G2(i).  The tensor pipe runs
// G2(i-1) while Zr(i+1) and softmax(i) are computed, and G1(i+1) while Z(i) and P(i) are written.
#pragma once
#include <cuda.h>

#include "fv_common.cuh"
#include "k_aux.cuh"
#include "ptx.cuh"

namespace gpufv {

constexpr int kWarpsWork = 16;
// MMA issuer and TMA producer are warps 0 and 1, the WORK warps 2..17 (TMEM lane quarter = physical
// warp % 4, so each quarter still has four WORK warps).  Measured against the WORK-first order
// (MMA / TMA warps 16 / 17): C4 k_stats 8.53 -> 8.38 ms, C5 29.6 -> 29.3 ms — the issuer shares its
// sub-partition with four WORK warps either way, but as the oldest warp it wins issue arbitration.
constexpr int kWarpMma = 0, kWarpTma = 1, kWarpWork0 = 2;
constexpr int kThreads2 = (kWarpsWork + 2) * 32;  // 576
constexpr int kMaxC2 = 2;                        // K <= 256 in this kernel (larger K: k_stats_w)

// per-tile metadata published by the TMA thread (ring of 4: slot t % 4 stays valid well past tile t)
struct TileMeta {
  int row0, nrows, b, t, flags;  // flags: 1 seg_last, 2 chunk_first, 4 fold, 8 seg_first
  int rb;                        // range-report word: b, or this CTA's own word (fused schedule)
};

// shared memory map (offsets from a 1024-aligned base)
constexpr int kS2W = 0;                              // W' hi | lo            64 KB
constexpr int kS2P = kS2W + 2 * kOpBytes;            // P hi | lo             64 KB
constexpr int kS2Z = kS2P + 2 * kOpBytes;            // Z hi | lo             64 KB  (GEMM2 A operand)
constexpr int kS2X = kS2Z + 2 * kOpBytes;            // X box stage           16 KB
constexpr int kXBoxBytes = 128 * 128;                // 32 floats x 128 rows
constexpr int kS2Bias = kS2X + kXBoxBytes;           // float[128]
constexpr int kS2Cs = kS2Bias + kG * 4;              // float[64]  -c_k 2^e_k
constexpr int kS2Sc = kS2Cs + kDP * 4;               // float[64]  2^e_k
constexpr int kS2Xchg = kS2Sc + kDP * 4;             // float2[2 parity][kMaxC2 ranks][4 quarters][128 rows] (m, s)
constexpr int kS2Meta = kS2Xchg + 2 * kMaxC2 * 4 * kTileM * 8;  // TileMeta[4]
constexpr int kS2Bar = kS2Meta + 128;                // uint64 barriers
constexpr int kNumBars = 16;
constexpr int kS2Tmem = kS2Bar + kNumBars * 8;
constexpr int kSmem2Bytes = kS2Tmem + 16 + 1024;
static_assert(kSmem2Bytes <= 232448, "shared memory budget");
static_assert(kLatGroups * sizeof(LatScratch) <= 2 * kOpBytes, "fused finalize scratch fits the P buffer");

// barrier slots
enum : int {
  B_XFULL0 = 0, B_XFULL1, B_XEMPTY0, B_XEMPTY1, B_ZR_FULL, B_G1_DONE, B_G2_DONE,
  B_L_EMPTY, B_P_FULL, B_FOLD_DONE, B_XCHG0, B_XCHG1, B_W_FULL
};

// tensor-memory columns: Zr double buffer, L, S'
constexpr uint32_t kTZr = 0, kTL = 256, kTS = 384;

// named barriers (0 = __syncthreads)
constexpr uint32_t kBarLane0 = 1;  // 1..4: the 4 WORK warps of a TMEM lane group (k_stats_w's quarter combine)
constexpr uint32_t kBarXchgLocal = 5;  // the 16 WORK warps of a single-CTA cluster (k_stats, K <= 128)
constexpr uint32_t kBarWorkSetup = 6;  // the 16 WORK warps: bias / scale tables loaded (k_stats)

struct Stats2Params {
  const float *X;             // n_total x D (also behind the tensor map; used for L2 prefetch)
  const int64_t *offsets;     // batch + 1
  const int64_t *tile_start;  // batch + 1
  const uint8_t *wimg;        // C x kWImgBytes
  const float *bias;          // Kp
  const float *xshift, *xscale;
  float *slots;               // segment slots: (ncl + batch) x kNF x Kp   (feature-major rows)
  float *s0slots;             // (ncl + batch) x Kp
  float *gamma_out;
  float *loglik_out;          // n_total (optional): per-descriptor log2 sum_j 2^(L_ij + b_j) (EM E-step)
  long long *trace;           // debug (GPUFV_TRACE builds): per-tile phase clocks of CTA 0
  int kfold;                  // GEMM2 restart period in tiles (kFold, or kFoldLong for large sets)
  int *rflags;                // batch: range flags (bit 0: a row with non-finite log-likelihoods), zeroed by k_schedule
  int batch, D, K, Kp;
  int64_t single_rows;        // >= 0: one set of this many rows whose schedule is known without k_schedule
                              // (tile_start = {0, T}): the tile walk then reads nothing from global memory
  // Range reports go to rflags[meta.rb]: rb = b with k_schedule (which zeroes the flags).  The fused
  // single-frame schedule (no k_schedule launched; the finalize derives the set's segments itself)
  // gives every CTA its own word (rflag_cta = 1: rb = b + CTA index, zeroed by the CTA at its start)
  // and the finalize ORs them into the image's flag — no word has to be zeroed before the kernel.
  // CTA (0, 0) zeroes the finalize's ticket.  The index is computed by the tile walker (TMA thread),
  // not in the WORK loop: writing the schedule tables here, or computing the word in the loop, grew
  // k_stats' spill area (-17 % / -2 % on the throughput path).
  int rflag_cta;
  unsigned *sched_counters;
  int ldx;                    // row stride of X in floats (>= D, % 4 == 0)
  float threshold;
  int gamma_mode;
};

// Walks the cluster's tile range [t0, t1) in order (TMA and MMA threads).  The current image's
// bounds live in registers and are re-read from global memory only when the walk crosses into the
// next image.  32-bit state: the host guarantees n_total < 2^30.
struct TileWalker {
  const Stats2Params *p;
  int t, t1, ts_b, ts_b1, off_b, off_b1, b, seg_pos, rb_off;
  __device__ void load_image() {
    if (p->single_rows >= 0) {  // one set: image 0 holds every tile
      b = 0; ts_b = 0; ts_b1 = (int)((p->single_rows + kTileM - 1) / kTileM);
      off_b = 0; off_b1 = (int)p->single_rows;
      return;
    }
    while (t >= (int)p->tile_start[b + 1]) ++b;  // skips empty images
    ts_b = (int)p->tile_start[b]; ts_b1 = (int)p->tile_start[b + 1];
    off_b = (int)p->offsets[b]; off_b1 = (int)p->offsets[b + 1];
  }
  __device__ void init(const Stats2Params &pp, int t0_, int t1_, int cta = 0) {
    p = &pp; t = t0_; t1 = t1_; b = 0; seg_pos = 0; rb_off = pp.rflag_cta ? cta : 0;
    ts_b = ts_b1 = off_b = off_b1 = 0;
    if (t0_ < t1_ && pp.single_rows >= 0) {
      load_image();
    } else if (t0_ < t1_) {
      int lo = 0, hi = pp.batch;
      while (lo < hi) { int mid = (lo + hi + 1) >> 1; if (pp.tile_start[mid] <= t0_) lo = mid; else hi = mid - 1; }
      b = lo;
      load_image();
    }
  }
  __device__ TileMeta meta() const {
    TileMeta m;
    m.t = t;
    m.b = b;
    m.rb = b + rb_off;
    m.row0 = off_b + (t - ts_b) * kTileM;
    const int rem = off_b1 - m.row0;
    m.nrows = rem < kTileM ? rem : kTileM;
    const bool seg_last = (t + 1 == t1) || (t + 1 >= ts_b1);
    const int kf = p->kfold;
    m.flags = (seg_last ? 1 : 0) | ((seg_pos % kf) == 0 ? 2 : 0) | (seg_pos == 0 ? 8 : 0) |
              ((seg_last || (seg_pos + 1) % kf == 0) ? 4 : 0);
    return m;
  }
  __device__ void next() {
    ++t;
    if (t >= ts_b1) { seg_pos = 0; if (t < t1) load_image(); }
    else ++seg_pos;
  }
};

// 16-byte chunk c of row r in a 128B-swizzled tile (8 x 16-byte chunks per 128-byte row)
__device__ __forceinline__ uint32_t sw_off(int r, int c) { return r * 128 + ((c ^ (r & 7)) << 4); }

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(ptx::smem_u32(bar))
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

// Features of dims k = 32 box + 8h .. +8 of one row, from the staged box (dims [32 box, 32 box + 32),
// 16-byte chunks 2h, 2h+1 of the row): linear hi -> Zr col k/2, quadratic hi -> col 32 + k/2,
// lo -> + 64.  kMask: dims >= D or a row past the image end are zeroed.
// kQO / kLO: column offsets of the quadratic hi and the linear lo words (the wide kernel's packed
// second half for D <= 96 puts [lin | quad] of 32 dims each in 32 columns per hi / lo part: 16 / 32)
template <bool kMask, int kQO = 32, int kLO = 64>
__device__ __forceinline__ void zr_box(const uint8_t *xbox, int row, int box, int h, int D, bool valid,
                                       const float *s_sc, const float *s_ncs, uint32_t taddr) {
  using namespace ptx;
  uint32_t lh[4], ll[4], qh[4], ql[4];
  const int k0 = 32 * box + 8 * h;
#pragma unroll
  for (int c2 = 0; c2 < 2; ++c2) {
    const float4 v = *reinterpret_cast<const float4 *>(xbox + sw_off(row, 2 * h + c2));
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
  tmem_st4(taddr + kQO + k0 / 2, qh);
  tmem_st4(taddr + kLO + k0 / 2, ll);
  tmem_st4(taddr + kLO + kQO + k0 / 2, ql);
}

// A row whose log-likelihoods are not all finite — a descriptor outside the fp16 operand range
// (|x - c| >= ~256 RMS in some dimension: the squared feature overflows), a GMM coefficient outside it
// (k_prep_w stores NaN), or non-finite input — has S = sum_j 2^(L_ij - M) NaN, 0 or inf (S >= 1
// otherwise: the row maximum contributes 2^0).  Its posteriors are made NaN, so the image's statistics
// and FV are NaN (never finite garbage), and the image is flagged for fv_range_flags.
__device__ __forceinline__ void range_bad(const Stats2Params &p, int b, float &alpha_p, bool reporter) {
  alpha_p = __int_as_float(0x7fffffff);
  if (reporter && p.rflags) atomicOr(p.rflags + b, 1);
}

// WORK-warp wait on an MMA-completion barrier.  Every warp waits on its own (try_wait suspends the
// warp instead of spinning), so the 16 warps are never coupled by a CTA-wide barrier here.  No warp
// can lag two phases behind: G1(i+1) needs ZR_FULL(i+1) and G2(i) needs P_FULL(i) from all 16 warps.
__device__ __forceinline__ void work_wait(uint64_t *bar, uint32_t parity) {
  ptx::mbar_wait(bar, parity);
  ptx::tc_fence_after();
}

#ifdef GPUFV_TRACE
#define TR(slot) do { if (p.trace && cid == 0 && rank == 0 && i < 64) p.trace[i * 16 + (slot)] = clock64(); } while (0)
#define TRW(slot) do { if (p.trace && cid == 0 && rank == 0 && i < 64 && lane == 0 && (ww == 0 || ww == 5 || ww == 10 || ww == 15)) \
    p.trace[1024 + ((i * 4 + (ww == 0 ? 0 : ww == 5 ? 1 : ww == 10 ? 2 : 3)) * 16) + (slot)] = clock64(); } while (0)
// kernel-level points (prologue / epilogue) of CTA 0: slots 7680 + 0..15, written by one thread each
#define TRP(slot) do { if (p.trace && cid == 0 && rank == 0) p.trace[7680 + (slot)] = clock64(); } while (0)
#else
#define TR(slot) do { } while (0)
#define TRW(slot) do { } while (0)
#define TRP(slot) do { } while (0)
#endif

// kC = cluster size (ceil(K / 128): 1 or 2) at compile time: the exchange loops and the combine over
// the 4 kC quarter pairs unroll without predicates (~3 % of the kernel's instructions at runtime C;
// C4 k_stats 8.62 -> 8.21 ms).  (A third parameter compiling the per-row hooks out measured 9.41 ms:
// the register allocation of this 96-register kernel moves with any change — measure each one.)
// kFin: the single-frame latency instantiation — after its last fold every CTA takes part in the
// frame's finalize (fin_lat_fused, k_aux.cuh: two grid barriers, no second kernel); `fin` is read only
// there.  The throughput instantiations (kFin = false) are unchanged.
template <bool kD64, int kC, bool kFin = false>
__global__ void __launch_bounds__(kThreads2, 1) k_stats(const __grid_constant__ CUtensorMap tmap_x, const Stats2Params p,
                                                        const __grid_constant__ FinParams fin) {
  using namespace ptx;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_base = smem_u32(smem_raw);
  const uint32_t sbase = (raw_base + 1023u) & ~1023u;
  uint8_t *smem = smem_raw + (sbase - raw_base);
  const uint32_t sW = sbase + kS2W, sP = sbase + kS2P, sZ = sbase + kS2Z, sX = sbase + kS2X;
  float *s_bias = reinterpret_cast<float *>(smem + kS2Bias);
  float *s_ncs = reinterpret_cast<float *>(smem + kS2Cs);
  float *s_sc = reinterpret_cast<float *>(smem + kS2Sc);
  float2 *s_xchg = reinterpret_cast<float2 *>(smem + kS2Xchg);
  TileMeta *s_meta = reinterpret_cast<TileMeta *>(smem + kS2Meta);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + kS2Bar);
  uint32_t *s_tmem = reinterpret_cast<uint32_t *>(smem + kS2Tmem);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_ctarank(), C = (uint32_t)kC;
  const int cid = (int)cluster_id_x(), ncl = (int)nclusters_x();

  if (tid == 0) TRP(0);
#ifdef GPUFV_TRACE
  if (p.trace && cid == 0 && rank == 0 && tid == 0) p.trace[7720] = ptx::globaltimer();
#endif
  // ---------------- setup (the bias / feature-scale tables are loaded by the WORK warps after the
  // cluster sync: their global-load latency stays off the CTA-wide barriers)
  if (warp == 0) { tmem_alloc(s_tmem, kTmemCols); tmem_relinquish(); }
  if (tid == 0) {
    if (p.rflag_cta) {  // fused schedule: this CTA's range word; CTA (0, 0) zeroes the finalize's ticket
      p.rflags[cid * kC + rank] = 0;
      if (cid == 0 && rank == 0) *p.sched_counters = 0u;
    }
    mbar_init(&bars[B_XFULL0], 1); mbar_init(&bars[B_XFULL1], 1);
    mbar_init(&bars[B_XEMPTY0], kWarpsWork); mbar_init(&bars[B_XEMPTY1], kWarpsWork);
    mbar_init(&bars[B_ZR_FULL], kWarpsWork);
    mbar_init(&bars[B_G1_DONE], 1); mbar_init(&bars[B_G2_DONE], 1);
    mbar_init(&bars[B_L_EMPTY], kWarpsWork); mbar_init(&bars[B_P_FULL], kWarpsWork);
    mbar_init(&bars[B_FOLD_DONE], kWarpsWork);
    mbar_init(&bars[B_XCHG0], 1); mbar_init(&bars[B_XCHG1], 1);
    mbar_init(&bars[B_W_FULL], 1);
    fence_mbar_init();
    // W' image of this rank: 64 KB bulk copy (async proxy), waited on by the MMA thread only
    mbar_arrive_expect_tx(&bars[B_W_FULL], kWImgBytes);
    for (int c = 0; c < 4; ++c)
      bulk_g2s(sW + c * (kWImgBytes / 4), p.wimg + (size_t)rank * kWImgBytes + c * (kWImgBytes / 4), kWImgBytes / 4,
               &bars[B_W_FULL]);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  if (tid == 0) TRP(1);
  cluster_sync();
  if (tid == 0) TRP(2);
  griddep_launch_dependents();  // k_finalize may start its prologue
  // k_schedule's tile prefix sums (and its zeroing of the range flags the WORK warps may set) are
  // complete and visible.  A single set's schedule needs no table: only the WORK warps wait then.
  if (p.single_rows < 0 || warp >= kWarpWork0) griddep_wait();
  if (tid == 0) TRP(3);

  const int64_t T = p.single_rows >= 0 ? (p.single_rows + kTileM - 1) / kTileM : p.tile_start[p.batch];
  const int t0 = (int)((int64_t)cid * T / ncl), t1 = (int)((int64_t)(cid + 1) * T / ncl);
  const int n = t1 - t0;

  if (warp == kWarpTma) {
    // ======================================================= tile walk + X producer (TMA)
    if (lane == 0 && n > 0) {
      const int Dv = p.ldx;
      TileWalker tw, twp;  // box walker, L2-prefetch walker (4 tiles ahead; set up after the first box
                           // is requested: its index loads would otherwise delay tile 0 of a small launch)
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
        s_meta[i & 3] = m;  // released to the WORK warps by the X_FULL phase completions below
        // box 0 (dims 0..31) after box 1 of the previous tile was released
        if (i >= 1) mbar_wait(&bars[B_XEMPTY1], (i - 1) & 1);
        // tile 0's box-0 release (phase 0 of X_EMPTY0) is not needed for a load (its box 1 went to the Z
        // buffer); observe it here so that every phase is waited on (compute-sanitizer synccheck)
        if (i == 1) mbar_wait(&bars[B_XEMPTY0], 0);
        mbar_arrive_expect_tx(&bars[B_XFULL0], kXBoxBytes);
        tma_load_2d(sX, &tmap_x, 0, m.row0, &bars[B_XFULL0]);
        if (i == 0) {
          TRP(4);
          twp.init(p, t0, t1);
          for (int k = 0; k < 4; ++k) prefetch_l2(k);
        }
        // box 1 (dims 32..63) after box 0 of this tile was released; tile 0's box 1 goes straight into
        // the Z buffer (unused until copy_z(0), which follows GEMM1(0) and so every box-1 conversion):
        // the first tile then pays one HBM round trip instead of two (latency path)
        if (i >= 1) mbar_wait(&bars[B_XEMPTY0], i & 1);
        mbar_arrive_expect_tx(&bars[B_XFULL1], kXBoxBytes);
        tma_load_2d(i == 0 ? sZ : sX, &tmap_x, 32, m.row0, &bars[B_XFULL1]);
        prefetch_l2(i + 4);
      }
    }
  } else if (warp == kWarpMma) {
    // ======================================================= MMA issuer
    if (n > 0) {  // the whole warp, converged; one elected lane issues (ptx::*_w)
      TileWalker tw;
      tw.init(p, t0, t1);
      const uint32_t idesc1 = idesc_f16_f32(128, kG, 0, 0);   // A = Zr (TMEM, K-major), B = W' K-major
      const uint32_t idesc2 = idesc_f16_f32(kNF, kG, 1, 1);   // A = Z^T (SMEM, MN-major), B = P MN-major
      uint32_t folds = 0;
      // operand descriptors built once: per UMMA only a compile-time offset (>> 4, into the 14-bit
      // start-address field; every shared address is < 2^18, so the field never carries) is added —
      // the issuing thread shares its sub-partition with four WORK warps, so its instruction count per
      // UMMA matters
      const uint64_t dW = desc_sw128(sW, 16, 1024);
      const uint64_t dZ = desc_sw128(sZ, kAtomBytes, 1024), dP = desc_sw128(sP, kAtomBytes, 1024);
      mbar_wait(&bars[B_W_FULL], 0);
      TRP(5);
      auto gemm1 = [&](int i) {
        mbar_wait(&bars[B_ZR_FULL], i & 1);
        if (i >= 1) mbar_wait(&bars[B_L_EMPTY], (i - 1) & 1);
        tc_fence_after();
        const uint32_t zr = tmem + kTZr + 128 * (i & 1);
#pragma unroll
        for (int s = 0; s < 3; ++s) {  // cross terms first, hi.hi last (truncating accumulator)
          const uint32_t za = zr + (s == 1 ? 64 : 0);          // hi, lo, hi
          const uint32_t wb = (s == 0 ? kOpBytes : 0);         // lo, hi, hi
#pragma unroll
          for (int kk = 0; kk < kNF / 16; ++kk) {
            const uint32_t off = wb + (kk >> 2) * kAtomBytes + (kk & 3) * 32;
            mma_f16_ts_w(tmem + kTL, za + kk * 8, dW + (off >> 4), idesc1, (s | kk) != 0);
          }
        }
        mma_commit_w(&bars[B_G1_DONE]);
      };
      auto gemm2 = [&](int i, bool chunk_first) {
        mbar_wait(&bars[B_P_FULL], i & 1);  // P(i) and Z(i) in shared memory
        if (chunk_first && i > 0) { mbar_wait(&bars[B_FOLD_DONE], folds & 1); ++folds; }
        tc_fence_after();
#pragma unroll
        for (int s = 0; s < 3; ++s) {
          const uint32_t za = (s == 1 ? kOpBytes : 0);         // hi, lo, hi
          const uint32_t pb = (s == 0 ? kOpBytes : 0);         // lo, hi, hi
#pragma unroll
          for (int kk = 0; kk < kTileM / 16; ++kk) {
            const uint32_t off = kk * 2048;  // 16 descriptor rows x 128 B
            mma_f16_ss_w(tmem + kTS, dZ + ((za + off) >> 4), dP + ((pb + off) >> 4), idesc2,
                       (chunk_first && s == 0 && kk == 0) ? 0u : 1u);
          }
        }
        mma_commit_w(&bars[B_G2_DONE]);
      };
      gemm1(0);
      for (int i = 0; i < n; ++i, tw.next()) {
        const bool chunk_first = (tw.meta().flags & 2) != 0;
        TR(12);
        if (i + 1 < n) gemm1(i + 1);
        TR(13);
        gemm2(i, chunk_first);
        TR(14);
      }
    }
  } else {
    // ======================================================= WORK warps
    const int ww = warp - kWarpWork0;       // WORK warp index 0..15
    const int q = warp & 3, h = ww >> 2;    // TMEM lanes 32q.. (physical warp % 4); quarter h
    const uint32_t lane_base = (uint32_t)(32 * q) << 16;
    const int row = 32 * q + lane;  // descriptor row of Zr / L / P / Z; feature of S'
    const int D = kD64 ? kDP : p.D;
    const float thr = p.threshold * kPScale;
    const uint8_t *xbox = smem + kS2X;

    // Zr(i), box `box`: this warp converts dims 32 box + 8h .. +8 of row `row`; all 16 WORK warps
    // share each box, so a box is released after ~1/16 of the tile's conversion work.  Box 0 needs no
    // wait::st (its X values are consumed by the time the stores issue); box 1 waits for all of this
    // thread's Zr(i) stores before ZR_FULL.
    auto conv_box = [&](int i, int box) {
      mbar_wait(&bars[B_XFULL0 + box], i & 1);
      const int nrows = s_meta[i & 3].nrows;
      const uint32_t ta = tmem + kTZr + 128 * (i & 1) + lane_base;
      const uint8_t *xb = (i == 0 && box == 1) ? smem + kS2Z : xbox;  // tile 0's box 1 sits in the Z buffer
      if (!kD64 || nrows < kTileM) zr_box<true>(xb, row, box, h, D, row < nrows, s_sc, s_ncs, ta);
      else zr_box<false>(xb, row, box, h, D, true, s_sc, s_ncs, ta);
      if (box == 1) tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&bars[B_XEMPTY0 + box]);
        if (box == 1) mbar_arrive(&bars[B_ZR_FULL]);
      }
    };
    auto copy_z = [&](int i) {  // this warp's Zr(i) words -> Z rows in shared memory (GEMM2 A operand)
      const uint32_t ta = tmem + kTZr + 128 * (i & 1) + lane_base;
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
        const uint32_t o = sw_off(row, 4 * box + h);  // 16-byte chunk of the atom holding dims 32 box + 8h ..
        const uint32_t *zb = z + 16 * box;
        sts128(sZ + o, zb[0], zb[1], zb[2], zb[3]);
        sts128(sZ + kAtomBytes + o, zb[4], zb[5], zb[6], zb[7]);
        sts128(sZ + kOpBytes + o, zb[8], zb[9], zb[10], zb[11]);
        sts128(sZ + kOpBytes + kAtomBytes + o, zb[12], zb[13], zb[14], zb[15]);
      }
    };
    // S' quarter (lane = feature, columns 32h..) of a finished chunk -> the segment slot: stored by
    // the segment's first chunk, added (red.global.add.v4.f32, same thread, program order) by the rest.
    // The 32 x 32 block is transposed through this warp's own 4 KB of the P buffer (the bytes its
    // P(i) stores overwrite next; GEMM2(i-1) has finished reading them) so that each global
    // instruction covers 4 feature rows x 128 contiguous bytes instead of 32 rows x 16 bytes.
    auto fold = [&](int b, bool first) {
      float *base = p.slots + (size_t)seg_slot(cid, b) * kNF * p.Kp + (size_t)(32 * q) * p.Kp + rank * kG + 32 * h;
      const uint32_t st0 = sP + (h >> 1) * kAtomBytes;
      auto saddr = [&](int r, int j) {  // 16-byte chunk j (columns 4j..4j+3) of local row r
        return st0 + (j >= 4 ? (uint32_t)kOpBytes : 0u) + sw_off(32 * q + r, 4 * (h & 1) + (j & 3));
      };
      uint32_t v[32];
      tmem_ld32(tmem + kTS + lane_base + 32 * h, v);
      tmem_ld_wait(v);
#pragma unroll
      for (int j = 0; j < 8; ++j) sts128(saddr(lane, j), v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      __syncwarp();
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int r = 4 * it + (lane >> 3), j = lane & 7;
        const float4 x = *reinterpret_cast<const float4 *>(smem + (saddr(r, j) - sbase));
        float *dst = base + (size_t)r * p.Kp + 4 * j;
        if (first) *reinterpret_cast<float4 *>(dst) = x;
        else red_add_v4(dst, x.x, x.y, x.z, x.w);
      }
      __syncwarp();  // the P(i) stores of this warp reuse the staging bytes
    };

    {
      const int wt = tid - kWarpWork0 * 32;
      for (int i = wt; i < kG; i += kWarpsWork * 32) s_bias[i] = p.bias[rank * kG + i];
      if (wt < kDP) { s_sc[wt] = p.xscale[wt]; s_ncs[wt] = -(p.xshift[wt] * p.xscale[wt]); }
      named_bar_sync(kBarWorkSetup, kWarpsWork * 32);
    }
    float s0acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) s0acc[j] = 0.f;
    int prev_b = 0;
    bool prev_fold = false, chunk_seg_first = true;
    if (n > 0) {
      conv_box(0, 0);
      conv_box(0, 1);
      // tile 0's box 1 was read from the Z buffer, which copy_z(0) overwrites: the ordering through
      // ZR_FULL -> GEMM1(0) -> G1_DONE already holds; this barrier states it in a form racecheck sees
      named_bar_sync(kBarWorkSetup, kWarpsWork * 32);
    }
    for (int i = 0; i < n; ++i) {
      TRW(0);
      work_wait(&bars[B_G1_DONE], i & 1);  // L(i) ready; Zr((i+1)%2) free (GEMM1(i-1) done)
      TRW(1);
      // ---- softmax(i), online form: this warp's column quarter is exponentiated against its own row
      // max m_h; the (m_h, s_h) pairs of the 4 quarters (one named barrier) and of the cluster's CTAs
      // (DSMEM) are then combined into the row's (M, S) and each quarter rescaled by 2^(m_h - M) / S.
      float v[32];
      {
        uint32_t rr[32];
        tmem_ld32(tmem + kTL + lane_base + 32 * h, rr);
        TRW(2);
        tmem_ld_wait(rr);
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(rr[j]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[B_L_EMPTY]);
      TRW(3);
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
      if (p.gamma_mode == 2 && row < mt.nrows) {
        float *go = p.gamma_out + (size_t)(mt.row0 + row) * p.K;
#pragma unroll
        for (int j = 0; j < 32; ++j) { int gj = rank * kG + 32 * h + j; if (gj < p.K) go[gj] = v[j]; }
      }
      auto exp_local = [&]() {  // e = 2^(v - m_h) in place; returns the quarter's row sum s_h
        float2 sacc = make_float2(0.f, 0.f);
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const float2 d = __fadd2_rn(make_float2(v[j], v[j + 1]), make_float2(-m, -m));
          v[j] = ex2_approx(d.x); v[j + 1] = ex2_approx(d.y);
          sacc = __fadd2_rn(sacc, make_float2(v[j], v[j + 1]));
        }
        return sacc.x + sacc.y;
      };
      // (m_h, s_h) of this warp's quarter -> slot [rank][h][row] of every CTA of the cluster (itself
      // included) by st.async on the parity buffer's mbarrier: one wait then gives each row the 4C
      // quarter pairs (no named barrier; parity double buffer, see DESIGN.md §6 for why no warp can
      // overwrite a buffer still being read)
      const int par = i & 1;
      float2 *xb = s_xchg + par * (kMaxC2 * 4 * kTileM);
      auto send = [&](float ssum) {
        if (C == 1) {  // a cluster of one CTA (K <= 128) has no DSMEM peer: local store + named barrier below
          xb[(rank * 4 + h) * kTileM + row] = make_float2(m, ssum);
          return;
        }
        if (ww == 0 && lane == 0) mbar_arrive_expect_tx(&bars[B_XCHG0 + par], C * 4 * kTileM * 8);
        const uint32_t my = smem_u32(&xb[(rank * 4 + h) * kTileM + row]);
        const uint32_t mybar = smem_u32(&bars[B_XCHG0 + par]);
        for (uint32_t r2 = 0; r2 < C; ++r2) st_async_v2f32(mapa_shared(my, r2), m, ssum, mapa_shared(mybar, r2));
      };
      if (i + 1 < n) {
        // Zr(i+1) box 0 (resident since the previous tile) in the same basic block as the exp loop:
        // its FMA/ALU work fills the issue slots the MUFU-bound exponentials leave idle
        mbar_wait(&bars[B_XFULL0], (i + 1) & 1);
        const int nr1 = s_meta[(i + 1) & 3].nrows;
        const float ssum = exp_local();
        zr_box<true>(xbox, row, 0, h, D, row < nr1, s_sc, s_ncs, tmem + kTZr + 128 * ((i + 1) & 1) + lane_base);
        send(ssum);  // (sending before the conversion measured -1.8 % on C4: the conversion then no
                     // longer fills the exponentials' issue gaps)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[B_XEMPTY0]);  // box 1 streams in behind the exchange below
      } else {
        send(exp_local());
      }
      TRW(4);
      if (C > 1) mbar_wait(&bars[B_XCHG0 + par], (i >> 1) & 1);
      else named_bar_sync(kBarXchgLocal, kWarpsWork * 32);
      TRW(12);
      float M = -3.0e38f, S = 0.f;
      {
        float2 o[kC * 4];
#pragma unroll
        for (int e = 0; e < kC * 4; ++e) { o[e] = xb[e * kTileM + row]; M = fmaxf(M, o[e].x); }
#pragma unroll
        for (int e = 0; e < kC * 4; ++e) S += o[e].y * ex2_approx(o[e].x - M);
      }
      // per-descriptor log2-likelihood (EM, NEXT-3): log2 sum_j 2^(L_ij + b_j) = M + log2 S
      if (p.loglik_out && h == 0 && rank == 0 && row < mt.nrows) p.loglik_out[mt.row0 + row] = M + log2f(S);
      // this quarter's gamma_ij = e_ij 2^(m_h - M) / S; P = gamma 2^14
      float alpha_p = __fdividef(ex2_approx(m - M), S) * kPScale;
      if (row >= mt.nrows) alpha_p = 0.f;
      else if (!(S > 0.5f && S < 3.0e38f)) range_bad(p, mt.rb, alpha_p, h == 0 && rank == 0);
      TRW(6);
      // Zr(i+1) box 1: its TMA load started when box 0 was released above (a single 16 KB stage)
      if (i + 1 < n) conv_box(i + 1, 1);
      TRW(13);

      // ---- GEMM2(i-1) done: S' chunk complete (fold), Z and P free
      if (i >= 1) {
        work_wait(&bars[B_G2_DONE], (i - 1) & 1);
        if (prev_fold) {
          fold(prev_b, chunk_seg_first);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bars[B_FOLD_DONE]);
        }
      }
      TRW(7);
      if (mt.flags & 2) chunk_seg_first = (mt.flags & 8) != 0;

      // ---- P(i) = gamma 2^14 (thresholded: gamma <= tau -> 0) -> fp16 hi/lo, S0 accumulation
      const float2 ap = make_float2(alpha_p, alpha_p);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int e = 0; e < 8; e += 2) {
          const int j = 8 * c + e;
          float2 g = __fmul2_rn(make_float2(v[j], v[j + 1]), ap);
          // gamma <= tau -> 0, applied unconditionally: with tau = 0 (exact mode) it keeps every gamma > 0
          // and zeroes only zeros, so the result is the same; the branch-free form measured +3.5 % on C4
          g = __fmul2_rn(g, make_float2(set_gt(g.x, thr), set_gt(g.y, thr)));
          v[j] = g.x; v[j + 1] = g.y;
          const float2 sa = __fadd2_rn(make_float2(s0acc[j], s0acc[j + 1]), g);
          s0acc[j] = sa.x; s0acc[j + 1] = sa.y;
          split2_f16(g, hi[e >> 1], lo[e >> 1]);
        }
        const uint32_t off = (h >> 1) * kAtomBytes + sw_off(row, 4 * (h & 1) + c);
        sts128(sP + off, hi[0], hi[1], hi[2], hi[3]);
        sts128(sP + kOpBytes + off, lo[0], lo[1], lo[2], lo[3]);
      }
      if (p.gamma_mode == 1 && row < mt.nrows) {
        float *go = p.gamma_out + (size_t)(mt.row0 + row) * p.K;
#pragma unroll
        for (int j = 0; j < 32; ++j) { int gj = rank * kG + 32 * h + j; if (gj < p.K) go[gj] = v[j] * (1.f / kPScale); }
      }
      TRW(8);
      copy_z(i);
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[B_P_FULL]);
      TRW(9);
      if (mt.flags & 1) {  // segment end: S0 (units of 2^14 gamma), this warp's 32 rows -> partial slot q
        warp_transpose_reduce32(s0acc, lane);
        p.s0slots[((size_t)seg_slot(cid, mt.b) * 4 + q) * p.Kp + rank * kG + 32 * h + lane] = s0acc[0];
#pragma unroll
        for (int j = 0; j < 32; ++j) s0acc[j] = 0.f;
      }
      prev_b = mt.b;
      prev_fold = (mt.flags & 4) != 0;
    }
    if (n > 0) {  // last chunk
      work_wait(&bars[B_G2_DONE], (n - 1) & 1);
      if (ww == 0 && lane == 0) TRP(6);
      fold(prev_b, chunk_seg_first);
      if (ww == 0 && lane == 0) TRP(7);
    }
  }

  // ---------------- teardown
  tc_fence_before();
  __syncthreads();
  if (tid == 0) TRP(8);
  if constexpr (kFin) {
    // the frame's finalize: the P / Z buffers are free (every GEMM2 and fold is done)
    if (warp == 0) tmem_dealloc(tmem, kTmemCols);
    fin_lat_fused(fin, reinterpret_cast<LatScratch *>(smem + kS2P));
  }
  cluster_sync();
  if (tid == 0) TRP(9);
#ifdef GPUFV_TRACE
  if (p.trace && cid == 0 && rank == 0 && tid == 0) p.trace[7721] = ptx::globaltimer();
  if (p.trace && tid == 0) atomicMax(reinterpret_cast<unsigned long long *>(p.trace + 7722), (unsigned long long)ptx::globaltimer());
#endif
  if (!kFin && warp == 0) tmem_dealloc(tmem, kTmemCols);
}

}  // namespace gpufv
