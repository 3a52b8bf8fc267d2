// k_aux.cuh — the small kernels around k_stats:
//   k_prep_shift, k_prep_bias, k_prep_bias_final, k_prep_w
//                            step a1: GMM -> prepared operands (Alg.1 l.1)
//   k_schedule               tile prefix sums from device offsets (ragged batches)
//   k_finalize               steps a6 (fixed-order fp64 slot reduction) + a7 (centring, VLFeat
//                            normalisation, P:449 / reading A9; the last block of each image applies
//                            the global L2 normalisation), also from fp64 stats (split path)
//   k_reduce_stats           a6 only -> fp64 sufficient statistics (descriptor-sharded path)

#pragma once
#include <cuda_fp16.h>
#include "fv_common.cuh"
#include "ptx.cuh"

namespace gpufv {

constexpr double kLog2e = 1.4426950408889634073599246810019;

__device__ __forceinline__ double gmm_var(const float *sigmas, size_t i, bool stddev) {
  double s = (double)sigmas[i];
  return stddev ? s * s : s;
}

// a1 (part 1): feature shift c_k = sum_j pi_j mu_jk / sum_j pi_j and power-of-two scale 2^e_k with
// e_k = -E where RMS_k = m 2^E (m in [0.5,1)), RMS_k^2 = sum_j pi_j (var_jk + mu_jk^2) / sum_j pi_j - c_k^2
// (one pass, fp64: only the exponent of RMS_k is used); the finalize's prior scales 1/sqrt(pi_j),
// 1/sqrt(2 pi_j) and inverse feature scales.  One block of 1024 threads: dimension k = tid % dstride
// (dstride = 64 or 128), Gaussian group tid / dstride, group partials summed in group order.
constexpr int kPrepThreads = 1024;
__global__ void __launch_bounds__(kPrepThreads) k_prep_shift(const float *w, const float *mu, const float *sg, int K,
                                                           int D, int Kp, int stddev, double *cshift, float *xshift,
                                                           float *xscale, double *pscale, double *xinv, int *gflag) {
  __shared__ double s_w[kPrepThreads], s_m[kPrepThreads], s_q[kPrepThreads];
  if (threadIdx.x == 0) {
    gflag[0] = 0;  // k_prep_w (later on the stream) sets bit 1 for an fp16 overflow
    gflag[2] = 0;  // gflag + 2, + 34: the fused finalize's grid-barrier counter and generation
    gflag[34] = 0;  // (separate 128-byte lines; self-resetting after the first use)
  }
  const int dstride = D <= kDP ? kDP : kDMax, ngrp = kPrepThreads / dstride;
  const int tid = threadIdx.x, k = tid % dstride, grp = tid / dstride;
  double ws = 0.0, am = 0.0, aq = 0.0;
  if (k < D) {
#pragma unroll 4
    for (int j = grp; j < K; j += ngrp) {
      const double wj = (double)w[j], m = (double)mu[(size_t)j * D + k];
      ws += wj;
      am += wj * m;
      aq += wj * (gmm_var(sg, (size_t)j * D + k, stddev) + m * m);
    }
  }
  s_w[tid] = ws; s_m[tid] = am; s_q[tid] = aq;
  __syncthreads();
  if (grp == 0) {
    double W = 0.0, M = 0.0, Q = 0.0;
    for (int g = 0; g < ngrp; ++g) { W += s_w[g * dstride + k]; M += s_m[g * dstride + k]; Q += s_q[g * dstride + k]; }
    double c = 0.0, sc = 1.0;
    if (k < D && W > 0.0) {
      c = M / W;
      const double r = sqrt(fmax(Q / W - c * c, 0.0));
      int E = 0;
      if (r > 0.0 && isfinite(r)) frexp(r, &E);
      sc = ldexp(1.0, -E);
    }
    cshift[k] = c;
    xshift[k] = (float)c;
    xscale[k] = (float)sc;
    xinv[k] = 1.0 / ((double)kPScale * sc);  // undoes P = gamma 2^14 and the feature scale (exact)
  }
  if (tid < kDMax && tid >= dstride) {  // dims past the tile family's width
    cshift[tid] = 0.0; xshift[tid] = 0.f; xscale[tid] = 1.f; xinv[tid] = 1.0 / (double)kPScale;
  }
  // finalize prior scales of the improved FV (reading A9): 1/sqrt(pi_j), 1/sqrt(2 pi_j)
  for (int j = tid; j < Kp; j += kPrepThreads) {
    pscale[j] = j < K ? 1.0 / sqrt((double)w[j]) : 0.0;
    pscale[Kp + j] = j < K ? 1.0 / sqrt(2.0 * (double)w[j]) : 0.0;
  }
}

// a1 (part 1b): per-Gaussian bias  b_j = ln pi_j - 1/2 sum_k ln var_jk - 1/2 sum_k (mu_jk - c_k)^2 / var_jk
// (natural log; the -D/2 ln 2pi constant is dropped, reading A2).  One block of 128 threads per
// Gaussian, one dimension per thread, fixed-order tree reduction.
__global__ void __launch_bounds__(kDMax) k_prep_bias(const float *w, const float *mu, const float *sg, int D,
                                                     int stddev, const double *cshift, double *bscratch) {
  __shared__ double s_red[kDMax];
  const int j = blockIdx.x, k = threadIdx.x;
  double t = 0.0;
  if (k < D) {
    const double v = gmm_var(sg, (size_t)j * D + k, stddev);
    const double d = (double)mu[(size_t)j * D + k] - cshift[k];
    t = log(v) + d * d / v;
  }
  s_red[k] = t;
  __syncthreads();
  for (int o = kDMax / 2; o > 0; o >>= 1) {
    if (k < o) s_red[k] += s_red[k + o];
    __syncthreads();
  }
  if (k == 0) bscratch[j] = log((double)w[j]) - 0.5 * s_red[0];
}

// a1 (part 1c): bias shift bmax = max_j b_j and the kernel's bias (b_j - bmax) log2 e (padded
// Gaussians: -1e30).  One block of 512 threads.
__global__ void __launch_bounds__(512) k_prep_bias_final(int K, int Kp, const double *bscratch, float *bias,
                                                         double *bmax_out) {
  __shared__ double s_red[512];
  const int tid = threadIdx.x;
  double bmax = -1e300;
  for (int j = tid; j < K; j += 512) bmax = fmax(bmax, bscratch[j]);
  s_red[tid] = bmax;
  __syncthreads();
  for (int o = 256; o > 0; o >>= 1) {
    if (tid < o) s_red[tid] = fmax(s_red[tid], s_red[tid + o]);
    __syncthreads();
  }
  bmax = s_red[0];
  if (tid == 0) *bmax_out = bmax;  // the bias shift (natural log units): log-likelihoods add it back
  for (int j = tid; j < Kp; j += 512) bias[j] = (j < K) ? (float)((bscratch[j] - bmax) * kLog2e) : -1.0e30f;
}

// a1 (part 2): W'_jf (log2 units, scaled by the feature exponents) split into fp16 hi/lo and stored
// as the exact SWIZZLE_128B K-major shared-memory image each CTA rank bulk-copies:
//   lin  feature of dim k:  W' =  log2e (mu_jk - c_k) / var_jk * 2^-e_k
//   quad feature of dim k:  W' = -log2e / (2 var_jk)          * 2^-2e_k
// Narrow (D <= 64, k_stats): 128 Gaussians per rank, features f = [lin 0..63 | quad 0..63], image =
//   [hi | lo] x 2 atoms (64 features) x 128 rows x 128 B.
// Wide (D <= 128, k_stats_w): 64 Gaussians per rank, two feature halves hf = 0, 1 of the dims
//   [64 hf, 64 hf + 64), each [lin | quad]; image = 2 halves x [hi | lo] x 2 atoms x 64 rows x 128 B.
// grid = Kp blocks (one Gaussian each), 2 dpad threads (one feature each).
// Also writes the finalize coefficients coef[3][kDMax][Kp] (a7, Eq. (6)-(7) of P:141-152 expanded about c):
//   coef[0][k][j] = mu_jk - c_k,  coef[1][k][j] = 1 / sqrt(var_jk),  coef[2][k][j] = 1 / var_jk
// (Gaussian-fastest so the finalize reads them coalesced; zero for padded j / k).
__global__ void k_prep_w(const float *mu, const float *sg, int K, int D, int stddev, const double *cshift,
                         const float *xscale, uint8_t *wimg, double *coef, int wide, int *gflag) {
  const int j = blockIdx.x, f = threadIdx.x, Kp = gridDim.x;
  int k, lin, off;
  if (!wide) {
    lin = f < kDP;
    k = f & (kDP - 1);
    const int rank = j / kG, row = j % kG, atom = f / 64, chunk = (f & 63) >> 3, e = f & 7;
    off = rank * kWImgBytes + atom * kAtomBytes + row * 128 + ((chunk ^ (row & 7)) << 4) + e * 2;
  } else {
    const int hf = f / kNF, fh = f % kNF;
    lin = fh < kDP;
    k = kDP * hf + (fh & (kDP - 1));
    // D <= 96 (packed second half, k_stats_w<.., kPk>): half b's 64 features [lin dims 64-95 | quad dims
    // 64-95] fill its first atom; the coefficients of dims 96-127 (zero) are not stored
    int pos = fh;
    if (wide == 2 && hf == 1) pos = (fh & 63) < 32 ? (lin ? fh : 32 + (fh - kDP)) : -1;
    const int rank = j / kGW, row = j % kGW;
    if (pos >= 0) {
      const int atom = pos / 64, chunk = (pos & 63) >> 3, e = pos & 7;
      off = rank * kWImgBytes + hf * (kWImgBytes / 2) + atom * (kGW * 128) + row * 128 + ((chunk ^ (row & 7)) << 4) + e * 2;
    } else {
      off = -1;
    }
  }
  const int lo_off = wide ? kGW * 128 * 2 : kOpBytes;  // lo half after the 2 hi atoms
  double wv = 0.0;
  if (j < K && k < D) {
    const double v = gmm_var(sg, (size_t)j * D + k, stddev);
    const double s = (double)xscale[k];
    const double mup = (double)mu[(size_t)j * D + k] - cshift[k];
    if (lin) wv = kLog2e * mup / v / s;
    else wv = -kLog2e / (2.0 * v) / (s * s);
    if (lin) {
      coef[(size_t)k * Kp + j] = mup;
      coef[(size_t)(kDMax + k) * Kp + j] = 1.0 / sqrt(v);
      coef[(size_t)(2 * kDMax + k) * Kp + j] = 1.0 / v;
    }
  } else if (lin) {
    coef[(size_t)k * Kp + j] = 0.0;
    coef[(size_t)(kDMax + k) * Kp + j] = 0.0;
    coef[(size_t)(2 * kDMax + k) * Kp + j] = 0.0;
  }
  float w32 = (float)wv;
  // a coefficient outside the fp16 range (a standard deviation below ~RMS/150 in some dimension, or a
  // non-finite / non-positive variance) cannot be split: it is stored as NaN, so every log-likelihood
  // of every row is NaN and each image is flagged by k_stats; the GMM itself is flagged here (bit 1)
  if (!(fabsf(w32) < 65504.f)) {
    w32 = __int_as_float(0x7fffffff);
    atomicOr(gflag, 2);
  }
  const __half hi = __float2half_rn(w32);
  const __half lo = __float2half_rn(w32 - __half2float(hi));
  if (off < 0) return;
  *reinterpret_cast<__half *>(wimg + off) = hi;
  *reinterpret_cast<__half *>(wimg + off + lo_off) = lo;
}

// fv_range_flags: flags_out[b] = rflags[b] | gflag (per-image range report of the last call).
__global__ void k_range_flags(const int *rflags, const int *gflag, int batch, int *flags_out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < batch) flags_out[b] = rflags[b] | *gflag;
}



// tile_start[0] = 0, tile_start[b+1] = sum_{b' <= b} ceil(N_b' / 128).  One block of 1024 threads.
// offsets == nullptr means a single set of n_single rows: {0, n_single} is written to off1 and used.
// Also the static split of the T tiles over the ncl clusters, for the finalize (no divisions there):
//   cstart[c] = c T / ncl (c = 0..ncl);  cown[2b], cown[2b+1] = first / last cluster owning a tile of
//   image b (last < first for an empty image).
// Also zeroes the finalize's per-image arrival counters (so no memset node separates k_stats from
// k_finalize in the stream) and lets k_stats start its prologue early (programmatic launch).
__global__ void k_schedule(const int64_t *offsets, int64_t *off1, int64_t n_single, int batch, int64_t *tile_start,
                           int ncl, int *cstart, int *cown, unsigned *counters, int *rflags, long long *trace) {
#ifdef GPUFV_TRACE
  if (trace && threadIdx.x == 0) trace[7723] = ptx::globaltimer();
#else
  (void)trace;
#endif
  __shared__ int64_t s_warp[32];
  __shared__ int64_t s_carry;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  ptx::griddep_launch_dependents();
  for (int b = tid; b < batch; b += 1024) { counters[b] = 0u; rflags[b] = 0; }
  if (!offsets) {
    if (tid == 0) {
      off1[0] = 0; off1[1] = n_single;
      tile_start[0] = 0; tile_start[1] = (n_single + kTileM - 1) / kTileM;
    }
  } else {
    if (tid == 0) { tile_start[0] = 0; s_carry = 0; }
    __syncthreads();
    for (int base = 0; base < batch; base += 1024) {
      const int b = base + tid;
      int64_t cnt = 0;
      if (b < batch) {
        int64_t n = offsets[b + 1] - offsets[b];
        cnt = n > 0 ? (n + kTileM - 1) / kTileM : 0;
      }
      int64_t x = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) { int64_t y = __shfl_up_sync(0xffffffffu, x, o); if (lane >= o) x += y; }
      if (lane == 31) s_warp[wid] = x;
      __syncthreads();
      if (wid == 0) {
        int64_t y = s_warp[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) { int64_t z = __shfl_up_sync(0xffffffffu, y, o); if (lane >= o) y += z; }
        s_warp[lane] = y;
      }
      __syncthreads();
      const int64_t incl = x + (wid > 0 ? s_warp[wid - 1] : 0) + s_carry;
      if (b < batch) tile_start[b + 1] = incl;
      __syncthreads();
      if (tid == 1023) s_carry = incl;
      __syncthreads();
    }
  }
  __syncthreads();
  const int64_t T = tile_start[batch];
  for (int c = tid; c <= ncl; c += 1024) cstart[c] = (int)((int64_t)c * T / ncl);
  for (int b = tid; b < batch; b += 1024) {
    const int64_t ft = tile_start[b], lt = tile_start[b + 1];
    int lo = 0, hi = -1;
    if (ft < lt) { lo = (int)tile_owner(ft, T, ncl); hi = (int)tile_owner(lt - 1, T, ncl); }
    cown[2 * b] = lo;
    cown[2 * b + 1] = hi;
  }
}

struct FinParams {
  const float *slots;         // segment slots from k_stats: (ncl + batch) x kNF x Kp (nullptr: stats)
  const float *s0slots;       // (ncl + batch) x 4 row groups x Kp
  const double *stats;        // batch x (1 + K(2D+1)) (nullptr when reading slots)
  const int64_t *offsets;     // batch + 1 (slots mode)
  const int64_t *tile_start;  // batch + 1 (slots mode)
  const int *cstart, *cown;   // k_schedule: cluster tile split (ncl + 1), per-image owner range (2 batch)
  const float *w;
  const double *coef;         // 3 x kDMax x Kp (k_prep_w)
  const float *xscale;
  const double *pscale;       // 2 x Kp: 1/sqrt(pi_j), 1/sqrt(2 pi_j) (k_prep_shift)
  const double *xinv;         // kDMax: 1 / (2^14 2^e_k) (k_prep_shift)
  float *out;                 // batch x 2KD
  double *stats_out;          // k_reduce_stats output
  double *norm2;              // batch x kFinMaxParts: each block's partial sum of squares (fixed slots)
  unsigned *counters;         // batch (zeroed before k_finalize): last-block ticket
  int batch, K, Kp, D, ncl, mode;
  int dpad;                   // 64 (k_stats) or 128 (k_stats_w): slot rows = [lin 0..dpad-1 | quad 0..dpad-1]
  int b_base;                 // first image of this launch (gridDim.y <= 65535 images per launch)
  // fused linear scoring (NEXT-4): scores[b][c] = svm_w[c] . fv_b + svm_b[c]; n_cls == 0: off
  const float *svm_w;         // n_cls x 2KD (same layout as one FV)
  const float *svm_b;         // n_cls (nullptr: zero bias)
  float *scores;              // batch x n_cls
  double *spart;              // batch x kFinMaxParts x n_cls: each block's partial dot products
  int n_cls;
  long long *trace;           // debug (GPUFV_TRACE builds): globaltimer points of block 0, slots 7700..
  // fused single-frame schedule (k_finalize_lat only): k_stats' per-CTA range words, ORed into rflags[0]
  const int *rflag_cta;
  int nflag;
  int *rflags;
  int64_t fused_n;            // >= 0: fused single set of fused_n rows (segments = clusters 0 .. ncl-1, N = fused_n)
  unsigned *gbar;             // fused finalize (k_stats<.., kFin>): grid-barrier {counter, generation}, prepared head
};

#ifdef GPUFV_TRACE
#define TRF(slot) do { if (p.trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0) \
    p.trace[7700 + (slot)] = ptx::globaltimer(); } while (0)
#else
#define TRF(slot) do { } while (0)
#endif

constexpr int kMaxCls = 32;     // classes of the fused linear scoring

constexpr int kFinJ = 32;       // Gaussians per finalize block
// partial-norm slots per image: k_finalize uses (K / 32) x (D / 64) <= 32 blocks, k_finalize_lat
// (K / 16) x (D / 16) <= 64
constexpr int kFinMaxParts = 64;
constexpr int kFinKI = kDP / 8; // dims per thread: k = kq + 8 i

// S0_j (gamma units) and S1_jk, S2_jk (about c, unscaled; k = kq + 8 i) of image b from the slots:
// a6, the fixed-order reduction over the image's (cluster) segments in ascending cluster order.
__device__ __forceinline__ void slot_sums(const FinParams &p, int b, int j, int kq, double &S0,
                                          double (&S1)[kFinKI], double (&S2)[kFinKI]) {
  S0 = 0.0;
#pragma unroll
  for (int i = 0; i < kFinKI; ++i) S1[i] = S2[i] = 0.0;
  const int ft = (int)p.tile_start[b], lt = (int)p.tile_start[b + 1];
  const int clo = p.cown[2 * b], chi = p.cown[2 * b + 1];
  for (int c = clo; c <= chi; ++c) {
    const int st = p.cstart[c], en = p.cstart[c + 1];
    const int s0 = st > ft ? st : ft, s1 = en < lt ? en : lt;
    if (s0 >= s1) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) S0 += (double)p.s0slots[((size_t)seg_slot(c, b) * 4 + q) * p.Kp + j];  // row groups
    {
      const float *sl = p.slots + (size_t)seg_slot(c, b) * 2 * p.dpad * p.Kp + j;
      float v1[kFinKI], v2[kFinKI];
#pragma unroll
      for (int i = 0; i < kFinKI; ++i) {
        const int k = kq + 8 * i;
        v1[i] = k < p.D ? __ldcs(sl + (size_t)k * p.Kp) : 0.f;          // streamed: read once
        v2[i] = k < p.D ? __ldcs(sl + (size_t)(p.dpad + k) * p.Kp) : 0.f;
      }
#pragma unroll
      for (int i = 0; i < kFinKI; ++i) { S1[i] += (double)v1[i]; S2[i] += (double)v2[i]; }
    }
  }
  S0 *= 1.0 / (double)kPScale;  // S0 was accumulated from P = gamma 2^14
#pragma unroll
  for (int i = 0; i < kFinKI; ++i) {
    const int k = kq + 8 * i;
    if (k < p.D) {
      const double xs = p.xinv[k];  // powers of two: exact
      S1[i] *= xs;
      S2[i] *= xs * xs * (double)kPScale;  // S2 carries 2^14 once and the feature scale twice
    }
  }
}

constexpr int kFinKR = 2;  // dims per thread (kr, kr + 32)

// a6 + a7 for one (32 Gaussians x 64 dims) tile of image b, computed by 256 threads (thread tid:
// Gaussians j0 + 4 jq .. +3, dims kr, kr + 32): U/V after the signed square root (or raw, mode 2) into
// sU/sV[j - j0][k - kb]; returns this thread's share of the squared norm (sum |U| + |V|).
__device__ __forceinline__ double fin_tile(const FinParams &p, int b, int j0, int kb, int tid, float (*sU)[kDP + 1],
                                           float (*sV)[kDP + 1]) {
  const int jq = tid & 7, kr = (tid >> 3) + kb;
  const int nj = min(kFinJ, p.K - j0), jb = j0 + 4 * jq;
  const int KD = p.K * p.D;
  double ss = 0.0;
  if (4 * jq < nj) {
    double N, S0[4], S1[kFinKR][4], S2[kFinKR][4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      S0[e] = 0.0;
#pragma unroll
      for (int r = 0; r < kFinKR; ++r) S1[r][e] = S2[r][e] = 0.0;
    }
    if (p.slots) {
      // a6: the image's (cluster) segments in ascending cluster order
      N = (double)(p.offsets[b + 1] - p.offsets[b]);
      const int ft = (int)p.tile_start[b], lt = (int)p.tile_start[b + 1];
      const int clo = p.cown[2 * b], chi = p.cown[2 * b + 1];
      // segments are taken two at a time with all their loads issued before either is accumulated
      // (a single image spread over many clusters would otherwise cost one L2 round trip per segment);
      // accumulation stays in ascending cluster order
      auto next_seg = [&](int &c) {  // next non-empty segment at or after c (-1: none); advances c
        for (; c <= chi; ++c) {
          const int st = p.cstart[c], en = p.cstart[c + 1];
          if ((st > ft ? st : ft) < (en < lt ? en : lt)) return c++;
        }
        return -1;
      };
      for (int c = clo; c <= chi;) {  // S0: 4 row-group partials per segment
        const int sa = next_seg(c), sb = next_seg(c);
        float4 s0[2][4];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int sg = u == 0 ? sa : sb;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            s0[u][q] = sg < 0 ? make_float4(0.f, 0.f, 0.f, 0.f)
                              : __ldcs(reinterpret_cast<const float4 *>(p.s0slots + ((size_t)seg_slot(sg, b) * 4 + q) * p.Kp + jb));
        }
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            S0[0] += (double)s0[u][q].x; S0[1] += (double)s0[u][q].y; S0[2] += (double)s0[u][q].z; S0[3] += (double)s0[u][q].w;
          }
      }
      for (int c = clo; c <= chi;) {  // S1, S2
        const int sa = next_seg(c), sb = next_seg(c);
        float4 v1[2][kFinKR], v2[2][kFinKR];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int sg = u == 0 ? sa : sb;
          const float *sl = p.slots + (size_t)seg_slot(sg < 0 ? 0 : sg, b) * 2 * p.dpad * p.Kp + jb;
#pragma unroll
          for (int r = 0; r < kFinKR; ++r) {
            const int k = kr + 32 * r;
            v1[u][r] = sg < 0 ? make_float4(0.f, 0.f, 0.f, 0.f) : __ldcs(reinterpret_cast<const float4 *>(sl + (size_t)k * p.Kp));
            v2[u][r] = sg < 0 ? make_float4(0.f, 0.f, 0.f, 0.f)
                              : __ldcs(reinterpret_cast<const float4 *>(sl + (size_t)(p.dpad + k) * p.Kp));
          }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int r = 0; r < kFinKR; ++r) {
            S1[r][0] += (double)v1[u][r].x; S1[r][1] += (double)v1[u][r].y; S1[r][2] += (double)v1[u][r].z; S1[r][3] += (double)v1[u][r].w;
            S2[r][0] += (double)v2[u][r].x; S2[r][1] += (double)v2[u][r].y; S2[r][2] += (double)v2[u][r].z; S2[r][3] += (double)v2[u][r].w;
          }
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) S0[e] *= 1.0 / (double)kPScale;  // S0 was accumulated from P = gamma 2^14
#pragma unroll
      for (int r = 0; r < kFinKR; ++r) {
        const int k = kr + 32 * r;
        const double xs = p.xinv[k];  // 1 / (2^14 2^e_k): powers of two, exact
#pragma unroll
        for (int e = 0; e < 4; ++e) { S1[r][e] *= xs; S2[r][e] *= xs * xs * (double)kPScale; }
      }
    } else {
      const double *st = p.stats + (size_t)b * (1 + (size_t)p.K * (2 * p.D + 1));
      N = st[0];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = jb + e;
        if (j >= p.K) continue;
        S0[e] = st[1 + j];
#pragma unroll
        for (int r = 0; r < kFinKR; ++r) {
          const int k = kr + 32 * r;
          if (k < p.D) {
            S1[r][e] = st[1 + p.K + (size_t)j * p.D + k];
            S2[r][e] = st[1 + p.K + (size_t)KD + (size_t)j * p.D + k];
          }
        }
      }
    }
    double fu[4], fv[4];
    const double invN = N > 0.0 ? 1.0 / N : 0.0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      fu[e] = fv[e] = 1.0;
      if (p.mode == 0 && N > 0.0 && jb + e < p.K) {
        fu[e] = invN * p.pscale[jb + e];           // 1 / (N sqrt(pi_j))
        fv[e] = invN * p.pscale[p.Kp + jb + e];    // 1 / (N sqrt(2 pi_j))
      }
    }
    const bool zero = (p.mode != 2) && !(N > 0.0);
#pragma unroll
    for (int r = 0; r < kFinKR; ++r) {
      const int k = kr + 32 * r;
      if (k >= p.D) continue;
      const double *cf = p.coef + (size_t)k * p.Kp + jb;
      const double2 m01 = *reinterpret_cast<const double2 *>(cf), m23 = *reinterpret_cast<const double2 *>(cf + 2);
      const double2 i01 = *reinterpret_cast<const double2 *>(cf + kDMax * p.Kp);
      const double2 i23 = *reinterpret_cast<const double2 *>(cf + kDMax * p.Kp + 2);
      const double2 v01 = *reinterpret_cast<const double2 *>(cf + 2 * kDMax * p.Kp);
      const double2 v23 = *reinterpret_cast<const double2 *>(cf + 2 * kDMax * p.Kp + 2);
      const double mup[4] = {m01.x, m01.y, m23.x, m23.y}, isd[4] = {i01.x, i01.y, i23.x, i23.y},
                   ivar[4] = {v01.x, v01.y, v23.x, v23.y};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (4 * jq + e >= nj) continue;
        double U = (S1[r][e] - mup[e] * S0[e]) * isd[e];                                       // sum gamma (x - mu)/sd
        double V = (S2[r][e] - 2.0 * mup[e] * S1[r][e] + mup[e] * mup[e] * S0[e]) * ivar[e] - S0[e];  // ((x-mu)^2/var - 1)
        float u, v;
        if (p.mode != 2) {
          U = zero ? 0.0 : U * fu[e];
          V = zero ? 0.0 : V * fv[e];
          ss += fabs(U) + fabs(V);  // = (signed sqrt)^2
          u = signed_sqrt((float)U);
          v = signed_sqrt((float)V);
        } else {
          u = (float)U;
          v = (float)V;
        }
        sU[4 * jq + e][k - kb] = u;
        sV[4 * jq + e][k - kb] = v;
      }
    }
  }
  return ss;
}

// fin_tile over a known segment range / list (slots mode): one round of loads per segment pair (S1
// and S2 of every thread; S0 of the tile's 32 Gaussians by the first warp, one Gaussian per lane — the
// other threads take it from shared memory sS0[j - s0base] instead of each re-summing it), the second
// segment of an odd pair skipped, no per-element bounds branches (columns j >= K are computed on
// padding and discarded).  Segment i is segs[i], or cfirst + i when segs == nullptr.  The 256 threads
// of the tile meet once on named barrier bar_id.  Per-accumulator summation order = fin_tile's:
// bitwise the same result.
template <int kSegs = 2>  // segments whose loads are in flight together
__device__ __forceinline__ double fin_tile_seg(const FinParams &p, int b, int j0, int kb, int tid, int bar_id, int bar_n,
                                               float (*sU)[kDP + 1], float (*sV)[kDP + 1], const int *segs,
                                               int cfirst, int nseg, double N, double *sS0, int s0base) {
  const int jq = tid & 7, kr = (tid >> 3) + kb;
  const int nj = min(kFinJ, p.K - j0), jb = j0 + 4 * jq;
  const size_t seg_stride = (size_t)2 * p.dpad * p.Kp;
  double S0l = 0.0, S0[4], S1[kFinKR][4], S2[kFinKR][4];
#pragma unroll
  for (int r = 0; r < kFinKR; ++r)
#pragma unroll
    for (int e = 0; e < 4; ++e) S1[r][e] = S2[r][e] = 0.0;
  TRF(8);
  for (int si = 0; si < nseg; si += kSegs) {
    int cs[kSegs];
    bool ok[kSegs];
    float4 v1[kSegs][kFinKR], v2[kSegs][kFinKR];
    float z0[kSegs][4];
#pragma unroll
    for (int u = 0; u < kSegs; ++u) {
      ok[u] = u == 0 || si + u < nseg;  // segment si is always valid
      cs[u] = ok[u] ? (segs ? segs[si + u] : cfirst + si + u) : cfirst;
      if (ok[u]) {
        const float *sl = p.slots + (size_t)seg_slot(cs[u], b) * seg_stride + jb;
#pragma unroll
        for (int r = 0; r < kFinKR; ++r) {
          const size_t k = (size_t)(kr + 32 * r) * p.Kp, k2 = k + (size_t)p.dpad * p.Kp;
          v1[u][r] = __ldcs(reinterpret_cast<const float4 *>(sl + k));
          v2[u][r] = __ldcs(reinterpret_cast<const float4 *>(sl + k2));
        }
      }
    }
    if (tid < 32) {  // S0 of Gaussian j0 + tid: 4 row-group partials per segment
#pragma unroll
      for (int u = 0; u < kSegs; ++u)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (ok[u]) z0[u][q] = __ldcs(p.s0slots + ((size_t)seg_slot(cs[u], b) * 4 + q) * p.Kp + j0 + tid);
#pragma unroll
      for (int u = 0; u < kSegs; ++u)
        if (ok[u])
#pragma unroll
          for (int q = 0; q < 4; ++q) S0l += (double)z0[u][q];
    }
#pragma unroll
    for (int u = 0; u < kSegs; ++u)
      if (ok[u])
#pragma unroll
        for (int r = 0; r < kFinKR; ++r) {
          S1[r][0] += (double)v1[u][r].x; S1[r][1] += (double)v1[u][r].y; S1[r][2] += (double)v1[u][r].z; S1[r][3] += (double)v1[u][r].w;
          S2[r][0] += (double)v2[u][r].x; S2[r][1] += (double)v2[u][r].y; S2[r][2] += (double)v2[u][r].z; S2[r][3] += (double)v2[u][r].w;
        }
  }
  TRF(5);
  if (tid < 32) sS0[j0 + tid - s0base] = S0l * (1.0 / (double)kPScale);  // S0 was accumulated from P = gamma 2^14
  ptx::named_bar_sync(bar_id, bar_n);  // the tile's S0
  TRF(6);
#pragma unroll
  for (int e = 0; e < 4; ++e) S0[e] = sS0[jb + e - s0base];
  double fu[4], fv[4];
  const double invN = N > 0.0 ? 1.0 / N : 0.0;
  const bool norm = p.mode == 0 && N > 0.0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    fu[e] = norm ? invN * p.pscale[jb + e] : 1.0;           // 1 / (N sqrt(pi_j))
    fv[e] = norm ? invN * p.pscale[p.Kp + jb + e] : 1.0;    // 1 / (N sqrt(2 pi_j))
  }
  const bool zero = (p.mode != 2) && !(N > 0.0);
  double ss = 0.0;
#pragma unroll
  for (int r = 0; r < kFinKR; ++r) {
    const int k = kr + 32 * r;
    if (k >= p.D) continue;
    const double xs = p.xinv[k];  // 1 / (2^14 2^e_k): powers of two, exact
    const double *cf = p.coef + (size_t)k * p.Kp + jb;
    const double2 m01 = *reinterpret_cast<const double2 *>(cf), m23 = *reinterpret_cast<const double2 *>(cf + 2);
    const double2 i01 = *reinterpret_cast<const double2 *>(cf + kDMax * p.Kp);
    const double2 i23 = *reinterpret_cast<const double2 *>(cf + kDMax * p.Kp + 2);
    const double2 v01 = *reinterpret_cast<const double2 *>(cf + 2 * kDMax * p.Kp);
    const double2 v23 = *reinterpret_cast<const double2 *>(cf + 2 * kDMax * p.Kp + 2);
    const double mup[4] = {m01.x, m01.y, m23.x, m23.y}, isd[4] = {i01.x, i01.y, i23.x, i23.y},
                 ivar[4] = {v01.x, v01.y, v23.x, v23.y};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const double s1 = S1[r][e] * xs, s2 = S2[r][e] * (xs * xs * (double)kPScale);
      double U = (s1 - mup[e] * S0[e]) * isd[e];                                      // sum gamma (x - mu)/sd
      double V = (s2 - 2.0 * mup[e] * s1 + mup[e] * mup[e] * S0[e]) * ivar[e] - S0[e];  // ((x-mu)^2/var - 1)
      float u, v;
      if (p.mode != 2) {
        U = zero ? 0.0 : U * fu[e];
        V = zero ? 0.0 : V * fv[e];
        if (4 * jq + e < nj) ss += fabs(U) + fabs(V);  // = (signed sqrt)^2
        u = signed_sqrt((float)U);
        v = signed_sqrt((float)V);
      } else {
        u = (float)U;
        v = (float)V;
      }
      sU[4 * jq + e][k - kb] = u;  // rows j >= K (padding) are never read
      sV[4 * jq + e][k - kb] = v;
    }
  }
  return ss;
}

// grid (ceil(K/32), batch), 256 threads.  Thread (jq = tid % 8, kr = tid / 8) owns Gaussians
// j0 + 4 jq .. +3 and dims kr, kr + 32: every slot / coefficient read is a 16-byte vector, coalesced
// over jq (the slots are feature-major rows of Kp Gaussians); U/V go through a shared-memory tile so
// the global stores are coalesced over (j, k).  The Eq. (6)-(7) combination runs in fp64; the signed
// square root (reading A9) in fp32 on the rounded value.  The L2 norm is accumulated with one
// atomic per block and the LAST block of each image (ticket) rescales it.
// Fused linear scoring (NEXT-4): each block also writes the dot products of its (pre-L2)
// U/V tile with the n_cls classifier rows into its own partial slot; the last block sums the slots in
// block order, divides by the image's norm and adds the bias (bitwise repeatable, no atomics).  With
// out == nullptr only the scores leave the kernel (the FV is never written to HBM).
// kSync (small launches, all blocks co-resident: the host uses it when the grid fits in one wave):
// every block of an image publishes its partial sum of squares, waits for its siblings and writes its
// tile once, already scaled — no serial rescale of the whole image by its last block (the latency
// path).  For large batches the last-block variant wins (waiting blocks would hold slots).
template <bool kScore, bool kSync>  // kScore = false: the plain encode (no scoring code compiled in)
__global__ void __launch_bounds__(256, 2) k_finalize(const FinParams p) {
  TRF(0);
  ptx::griddep_wait();  // k_stats (launched before us, programmatically) has completed
  TRF(1);
  __shared__ float sU[kFinJ][kDP + 1], sV[kFinJ][kDP + 1];
  __shared__ double s_red[8];
  __shared__ float s_dot[8][kMaxCls];
  __shared__ int s_last;
  const int b = p.b_base + (int)blockIdx.y, tid = threadIdx.x;
  const int j0 = blockIdx.x * kFinJ, nj = min(kFinJ, p.K - j0);
  const int kb = kDP * (int)blockIdx.z, nk = min(kDP, p.D - kb);  // this block's dims [kb, kb + nk)
  const int KD = p.K * p.D;
  double ss;
  if (p.slots && p.tile_start[p.batch] >= (int64_t)p.ncl) {  // every cluster non-empty: segments = cown range
    __shared__ double s_S0[kFinJ];
    const int lo = p.cown[2 * b], hi = p.cown[2 * b + 1];
    ss = fin_tile_seg(p, b, j0, kb, tid, 1, 256, sU, sV, nullptr, lo, hi - lo + 1,
                      (double)(p.offsets[b + 1] - p.offsets[b]), s_S0, j0);
  } else {
    ss = fin_tile(p, b, j0, kb, tid, sU, sV);
  }
  __syncthreads();
  TRF(2);
  const int part = blockIdx.z * gridDim.x + blockIdx.x, nparts = gridDim.x * gridDim.z;
  if (!kSync && (!kScore || p.out)) {
    float *o = p.out + (size_t)b * 2 * KD + (size_t)j0 * p.D + kb;
    for (int t = tid; t < nj * nk; t += 256) {
      const int r = t / nk, k = t - r * nk;
      o[(size_t)r * p.D + k] = sU[r][k];
      o[KD + (size_t)r * p.D + k] = sV[r][k];
    }
  }
  if (kScore) {
    // this thread's tile elements t = tid + 256 u (nj * nk <= 2048), classifier reads coalesced over t
    constexpr int kE = kFinJ * kDP / 256;
    float zu[kE], zv[kE];
    int wo[kE];
#pragma unroll
    for (int u = 0; u < kE; ++u) {
      const int t = tid + 256 * u, r = t / nk, k = t - r * nk;
      const bool ok = t < nj * nk;
      zu[u] = ok ? sU[r][k] : 0.f;
      zv[u] = ok ? sV[r][k] : 0.f;
      wo[u] = ok ? r * p.D + k : 0;
    }
    const float *wb = p.svm_w + (size_t)j0 * p.D + kb;
    for (int c = 0; c < p.n_cls; ++c) {
      const float *wc = wb + (size_t)c * 2 * KD;
      float a = 0.f;
#pragma unroll
      for (int u = 0; u < kE; ++u) {
        a = fmaf(zu[u], __ldg(wc + wo[u]), a);
        a = fmaf(zv[u], __ldg(wc + KD + wo[u]), a);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
      if ((tid & 31) == 0) s_dot[tid >> 5][c] = a;
    }
    __syncthreads();
    if (tid < p.n_cls) {
      double t = 0.0;
      for (int w = 0; w < 8; ++w) t += (double)s_dot[w][tid];
      p.spart[((size_t)b * kFinMaxParts + part) * p.n_cls + tid] = t;  // own slot: no atomics
      __threadfence();
    }
  }
  const bool l2 = p.mode != 2;
  if (kSync) {
    float sc = 1.f;
    if (l2 || kScore) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
      if ((tid & 31) == 0) s_red[tid >> 5] = ss;
      __syncthreads();
      if (tid == 0) {
        double tot = 0.0;
        for (int w = 0; w < 8; ++w) tot += s_red[w];
        p.norm2[(size_t)b * kFinMaxParts + part] = tot;  // own slot
      }
      __threadfence();  // this block's norm / score parts before its arrival
      __syncthreads();
      if (tid == 0) {
        unsigned *ctr = p.counters + b;
        atomicAdd(ctr, 1u);
        while (atomicAdd(ctr, 0u) < (unsigned)nparts) __nanosleep(32);
        __threadfence();
      }
      __syncthreads();
      TRF(3);
      double n2 = 0.0;  // fixed-order sum of the parts: the same bits in every block
      if (l2)
        for (int k = 0; k < nparts; ++k) n2 += __ldcg(p.norm2 + (size_t)b * kFinMaxParts + k);
      if (l2 && n2 > 0.0) sc = (float)(1.0 / sqrt(n2));
      if (kScore && part == 0 && tid < p.n_cls) {
        double d = 0.0;
        for (int k = 0; k < nparts; ++k) d += __ldcg(p.spart + ((size_t)b * kFinMaxParts + k) * p.n_cls + tid);
        const double inv = l2 ? (n2 > 0.0 ? 1.0 / sqrt(n2) : 0.0) : 1.0;
        p.scores[(size_t)b * p.n_cls + tid] = (float)(d * inv + (p.svm_b ? (double)p.svm_b[tid] : 0.0));
      }
    }
    if (!kScore || p.out) {
      float *o = p.out + (size_t)b * 2 * KD + (size_t)j0 * p.D + kb;
      for (int t = tid; t < nj * nk; t += 256) {
        const int r = t / nk, k = t - r * nk;
        o[(size_t)r * p.D + k] = sU[r][k] * sc;
        o[KD + (size_t)r * p.D + k] = sV[r][k] * sc;
      }
    }
    TRF(4);
    return;
  }
  if (!kScore && !l2) return;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
  if ((tid & 31) == 0) s_red[tid >> 5] = ss;
  __syncthreads();
  if (tid == 0) {
    double tot = 0.0;
    for (int w = 0; w < 8; ++w) tot += s_red[w];
    p.norm2[(size_t)b * kFinMaxParts + part] = tot;  // own slot: no atomics
    __threadfence();
    const unsigned ticket = atomicAdd(p.counters + b, 1u);  // only decides which block is last
    s_last = (ticket == nparts - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double n2 = 0.0;  // fixed-order sum of the parts: bitwise repeatable
  if (l2)
    for (int k = 0; k < nparts; ++k) n2 += __ldcg(p.norm2 + (size_t)b * kFinMaxParts + k);
  if (kScore && tid < p.n_cls) {  // scores of the normalised FV (an all-zero FV scores the bias)
    double d = 0.0;
    for (int k = 0; k < nparts; ++k) d += __ldcg(p.spart + ((size_t)b * kFinMaxParts + k) * p.n_cls + tid);
    const double inv = l2 ? (n2 > 0.0 ? 1.0 / sqrt(n2) : 0.0) : 1.0;
    p.scores[(size_t)b * p.n_cls + tid] = (float)(d * inv + (p.svm_b ? (double)p.svm_b[tid] : 0.0));
  }
  if (!l2 || (kScore && !p.out) || !(n2 > 0.0)) return;
  const float sc = (float)(1.0 / sqrt(n2));
  if ((2 * KD) % 4 != 0) {  // any D (the embedding path): scalar rescale
    float *o1 = p.out + (size_t)b * 2 * KD;
    for (int t = tid; t < 2 * KD; t += 256) o1[t] = __ldcg(o1 + t) * sc;
    return;
  }
  float4 *ob = reinterpret_cast<float4 *>(p.out + (size_t)b * 2 * KD);  // 2KD % 4 == 0
  const int n4 = (2 * KD) / 4;
  for (int t0 = 0; t0 < n4; t0 += 256 * 8) {  // 8 loads in flight per thread (the image is in L2)
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) { const int t = t0 + u * 256 + tid; if (t < n4) v[u] = __ldcg(ob + t); }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int t = t0 + u * 256 + tid;
      if (t < n4) { v[u].x *= sc; v[u].y *= sc; v[u].z *= sc; v[u].w *= sc; ob[t] = v[u]; }
    }
  }
}

// Whole-image finalize for large batches (D <= 64, K <= 256): persistent blocks of 512 threads take
// whole images; the two 256-thread groups compute the image's (32 x 64) tiles with fin_tile into a
// shared-memory copy of the image (2 x 256 x 65 floats), the block reduces the squared norm in a fixed
// order and writes the FV exactly once, already scaled — no per-image atomics, no last-block re-read
// of the image.  Scores (kScore) are taken from the same shared-memory image.
constexpr int kImgK = 256;
constexpr int kImgThreads = 512;
constexpr int kImgSmemBytes = 2 * kImgK * (kDP + 1) * 4;
constexpr int kImgMaxSeg = 160;  // segment list capacity per image (>= clusters of any launch)
template <bool kScore>
__global__ void __launch_bounds__(kImgThreads, 1) k_finalize_img(const FinParams p) {
  ptx::griddep_wait();  // k_stats (launched before us, programmatically) has completed
  extern __shared__ float fimg[];
  float(*iU)[kDP + 1] = reinterpret_cast<float(*)[kDP + 1]>(fimg);
  float(*iV)[kDP + 1] = reinterpret_cast<float(*)[kDP + 1]>(fimg + kImgK * (kDP + 1));
  __shared__ double s_red[kImgThreads / 32];
  __shared__ float s_dot[kImgThreads / 32][kMaxCls];
  const int tid = threadIdx.x, grp = tid >> 8, gt = tid & 255, lane = tid & 31, warp = tid >> 5;
  const int KD = p.K * p.D, ntiles = (p.K + kFinJ - 1) / kFinJ;
  const bool l2 = p.mode != 2;
  __shared__ int s_segs[kImgMaxSeg];
  __shared__ int s_nseg;
  __shared__ double s_S0[kImgK];
  // With every cluster non-empty (T >= ncl) the segments of image b are exactly clusters
  // cown[2b] .. cown[2b+1]: no scan.  That range and N of the images ahead of the current one are
  // kept in a ring (thread 0 reads image b + 2 gridDim.x while b is processed) so that at the top of
  // image b thread 0 can bulk-prefetch the next image's slots into L2 without waiting on any load.
  __shared__ __align__(8) int s_lh[3][2];
  __shared__ int64_t s_off[3][2];
  const bool direct = p.slots && p.tile_start[p.batch] >= (int64_t)p.ncl;
  const size_t seg_bytes = (size_t)2 * p.dpad * p.Kp * 4, s0_bytes = (size_t)4 * p.Kp * 4;
  auto info = [&](int bb, int slot) {  // thread 0 only: cown range and offsets of image bb, asynchronously
    if (bb < p.batch) {
      ptx::cp_async8(&s_lh[slot][0], p.cown + 2 * bb);
      ptx::cp_async8(&s_off[slot][0], p.offsets + bb);
      ptx::cp_async8(&s_off[slot][1], p.offsets + bb + 1);
    }
  };
  if (direct && tid == 0) { info(blockIdx.x, 0); info(blockIdx.x + gridDim.x, 1); ptx::cp_async_wait_all(); }
  __syncthreads();
  for (int b = blockIdx.x, it = 0; b < p.batch; b += gridDim.x, ++it) {
    const int cur = it % 3, nxt = (it + 1) % 3, far = (it + 2) % 3;
    if (direct && tid == 0) {
      if (b + (int)gridDim.x < p.batch)
        for (int c = s_lh[nxt][0]; c <= s_lh[nxt][1]; ++c) {  // the next image's segments -> L2
          const int64_t sl = seg_slot(c, b + gridDim.x);
          ptx::prefetch_l2_bulk(p.slots + sl * (seg_bytes / 4), (uint32_t)seg_bytes);
          ptx::prefetch_l2_bulk(p.s0slots + sl * (s0_bytes / 4), (uint32_t)s0_bytes);
        }
      info(b + 2 * gridDim.x, far);  // arrives while this image is processed
    }
    if (!direct && p.slots && tid == 0) {  // the image's non-empty (cluster) segments, once for all its tiles
      const int ft = (int)p.tile_start[b], lt = (int)p.tile_start[b + 1];
      const int clo = p.cown[2 * b], chi = p.cown[2 * b + 1];
      int ns = 0;
      for (int c = clo; c <= chi && ns < kImgMaxSeg; ++c) {
        const int st = p.cstart[c], en = p.cstart[c + 1];
        if ((st > ft ? st : ft) < (en < lt ? en : lt)) s_segs[ns++] = c;
      }
      s_nseg = ns;
    }
    if (!direct) __syncthreads();
    const bool use_list = p.slots && (direct || s_nseg < kImgMaxSeg);  // (a longer list falls back to the scan)
    const int cfirst = direct ? s_lh[cur][0] : 0, nseg = direct ? s_lh[cur][1] - s_lh[cur][0] + 1 : (p.slots ? s_nseg : 0);
    const double N = direct ? (double)(s_off[cur][1] - s_off[cur][0])
                            : (p.slots ? (double)(p.offsets[b + 1] - p.offsets[b]) : 0.0);
    double ss = 0.0;
    for (int t = grp; t < ntiles; t += kImgThreads / 256)
      ss += use_list ? fin_tile_seg(p, b, t * kFinJ, 0, gt, 1 + grp, 256, iU + t * kFinJ, iV + t * kFinJ,
                                    direct ? nullptr : s_segs, cfirst, nseg, N, s_S0, 0)
                     : fin_tile(p, b, t * kFinJ, 0, gt, iU + t * kFinJ, iV + t * kFinJ);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    if (lane == 0) s_red[warp] = ss;
    __syncthreads();
    double n2 = 0.0;  // fixed order: bitwise repeatable
    for (int w = 0; w < kImgThreads / 32; ++w) n2 += s_red[w];
    const float sc = (l2 && n2 > 0.0) ? (float)(1.0 / sqrt(n2)) : 1.f;
    // the image's (j, k) elements: row j by one warp, lanes over k (coalesced, no index division)
    if (kScore) {
      for (int c = 0; c < p.n_cls; ++c) {
        const float *wc = p.svm_w + (size_t)c * 2 * KD;
        float a = 0.f;
        for (int j = warp; j < p.K; j += kImgThreads / 32)
          for (int k = lane; k < p.D; k += 32) {
            const int e = j * p.D + k;
            a = fmaf(iU[j][k], __ldg(wc + e), a);
            a = fmaf(iV[j][k], __ldg(wc + KD + e), a);
          }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
        if (lane == 0) s_dot[warp][c] = a;
      }
      __syncthreads();
      if (tid < p.n_cls) {
        double d = 0.0;
        for (int w = 0; w < kImgThreads / 32; ++w) d += (double)s_dot[w][tid];
        const double inv = l2 ? (n2 > 0.0 ? 1.0 / sqrt(n2) : 0.0) : 1.0;
        p.scores[(size_t)b * p.n_cls + tid] = (float)(d * inv + (p.svm_b ? (double)p.svm_b[tid] : 0.0));
      }
    }
    if (!kScore || p.out) {
      float *o = p.out + (size_t)b * 2 * KD;
      if (p.D == kDP) {  // two rows per warp per step, no bounds checks on k
        for (int j = warp; j < p.K; j += 2 * (kImgThreads / 32)) {
          const int j2 = j + kImgThreads / 32;
          const float u0 = iU[j][lane] * sc, u1 = iU[j][lane + 32] * sc, v0 = iV[j][lane] * sc, v1 = iV[j][lane + 32] * sc;
          o[j * kDP + lane] = u0; o[j * kDP + lane + 32] = u1;
          o[KD + j * kDP + lane] = v0; o[KD + j * kDP + lane + 32] = v1;
          if (j2 < p.K) {
            const float a0 = iU[j2][lane] * sc, a1 = iU[j2][lane + 32] * sc, c0 = iV[j2][lane] * sc, c1 = iV[j2][lane + 32] * sc;
            o[j2 * kDP + lane] = a0; o[j2 * kDP + lane + 32] = a1;
            o[KD + j2 * kDP + lane] = c0; o[KD + j2 * kDP + lane + 32] = c1;
          }
        }
      } else {
        for (int j = warp; j < p.K; j += kImgThreads / 32)
          for (int k = lane; k < p.D; k += 32) {
            o[j * p.D + k] = iU[j][k] * sc;
            o[KD + j * p.D + k] = iV[j][k] * sc;
          }
      }
    }
    if (direct && tid == 0) ptx::cp_async_wait_all();
    __syncthreads();  // the next image overwrites the shared image, s_red, s_S0 and the segment list
  }
}

// Latency path (a handful of images, K <= 256, D <= 64, slots).  A single frame is spread over many
// clusters (one or a few tiles each, so k_stats finishes early), so its finalize reads many segments.
// That reduction is bound by how many L2 requests each SM keeps in flight, not by bandwidth (a 5,000-
// descriptor frame over 40 segments is 5 MB), so every load is a full 128-byte line: a block owns 32
// Gaussians x 8 dims, and a warp-wide float4 load covers 4 slot rows x 128 B (8 lanes per row; rows =
// (segment, feature) pairs).  Thread t (Gaussian group g = t % 8, row slot rs = t / 8) sums the rows
// rs, rs + 32, ... = one feature (S1 or S2 of one dim) over every other segment, all loads of a round
// in flight (kLatRows rows: 40 segments in one round); the two segment parities and the S0 partials
// are combined through shared memory in a fixed order.  Grid (K/32, batch, D/8) <= the SM count (one
// wave, every block co-resident): blocks publish their partial sum of squares, wait for their image's
// siblings and write their (32 x 8) sub-tile once, scaled (as k_finalize<.., kSync>).
constexpr int kLatThreads = 256;
constexpr int kLatJ = 32, kLatK = 8;   // Gaussians x dims per block
constexpr int kLatRows = 20;           // slot rows per thread per round of loads
__global__ void __launch_bounds__(kLatThreads) k_finalize_lat(const FinParams p) {
  ptx::griddep_wait();  // k_stats (launched before us, programmatically) has completed
  TRF(1);
  if (p.rflag_cta && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x < 32) {
    int fl = 0;  // fused schedule: the image's range flag from k_stats' per-CTA words (one warp: the
                 // loads are independent, a single thread would wait for each in turn)
    for (int c = threadIdx.x; c < p.nflag; c += 32) fl |= p.rflag_cta[c];
    fl = __reduce_or_sync(0xffffffffu, fl);
    if (threadIdx.x == 0) p.rflags[0] = fl;
  }
  __shared__ double s_part[2][2 * kLatK][kLatJ];  // [segment parity][feature][Gaussian]
  __shared__ double s_p0[kLatThreads / 8][kLatJ];  // S0 partials [row slot][Gaussian]
  __shared__ double s_S0[kLatJ];
  __shared__ double s_red[kLatThreads / 32];
  __shared__ int s_segs[kImgMaxSeg];
  __shared__ int s_nseg;
  const int b = p.b_base + (int)blockIdx.y, tid = threadIdx.x, lane = tid & 31;
  const int j0 = blockIdx.x * kLatJ, k0 = blockIdx.z * kLatK;
  const bool fused = p.fused_n >= 0;  // no k_schedule ran: a single set over every cluster
  const bool direct = fused || p.tile_start[p.batch] >= (int64_t)p.ncl;
  const int clo = fused ? 0 : p.cown[2 * b], chi = fused ? p.ncl - 1 : p.cown[2 * b + 1];
  if (!direct && tid == 0) {  // some cluster owns no tile: scan for the image's non-empty segments
    const int ft = (int)p.tile_start[b], lt = (int)p.tile_start[b + 1];
    int ns = 0;
    for (int c = clo; c <= chi && ns < kImgMaxSeg; ++c) {
      const int st = p.cstart[c], en = p.cstart[c + 1];
      if ((st > ft ? st : ft) < (en < lt ? en : lt)) s_segs[ns++] = c;
    }
    s_nseg = ns;
  }
  __syncthreads();
  const int nseg = direct ? chi - clo + 1 : s_nseg;
  auto seg = [&](int i) { return direct ? clo + i : s_segs[i]; };
  const size_t seg_stride = (size_t)2 * p.dpad * p.Kp;
  // this thread's output (j, k) and its coefficients: independent of the segments, in flight with them
  const int ok_ = tid & (kLatK - 1), oj = tid >> 3;  // 8 consecutive dims per 8 lanes (coalesced stores)
  const int j = j0 + oj, k = k0 + ok_;
  const bool valid = k < p.D && j < p.K;
  const double N = fused ? (double)p.fused_n : (double)(p.offsets[b + 1] - p.offsets[b]);
  double xs = 0.0, mup = 0.0, isd = 0.0, ivar = 0.0, psu = 0.0, psv = 0.0;
  if (valid) {
    xs = p.xinv[k];  // 1 / (2^14 2^e_k): powers of two, exact
    const double *cf = p.coef + (size_t)k * p.Kp + j;
    mup = cf[0]; isd = cf[kDMax * p.Kp]; ivar = cf[2 * kDMax * p.Kp];
    psu = p.pscale[j]; psv = p.pscale[p.Kp + j];
  }
  TRF(8);
  const int g = tid & 7, rs = tid >> 3;  // Gaussian group (4 Gaussians j0 + 4 g ..), row slot 0..31
  {
    // S1 / S2 rows: row r = 16 s + f (segment s, feature f = 2 (dim - k0) + {0: S1, 1: S2}); this
    // thread: f = rs % 16, segments rs / 16 + 2 u
    const int f = rs & 15, par = rs >> 4, kf = k0 + (f >> 1);
    const size_t frow = (size_t)((f & 1) ? p.dpad + kf : kf) * p.Kp + j0 + 4 * g;
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    if (kf < p.D) {
      for (int s0 = par; s0 < nseg; s0 += 2 * kLatRows) {
        float4 v[kLatRows];
#pragma unroll
        for (int u = 0; u < kLatRows; ++u) {
          const int si = s0 + 2 * u;
          v[u] = si < nseg ? __ldcs(reinterpret_cast<const float4 *>(p.slots + (size_t)seg_slot(seg(si), b) * seg_stride + frow))
                           : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < kLatRows; ++u) { a[0] += (double)v[u].x; a[1] += (double)v[u].y; a[2] += (double)v[u].z; a[3] += (double)v[u].w; }
      }
    }
    // S0 partials: pair v = 4 s + q (segment s, row group q); this thread: pairs rs + 32 u
    double z[4] = {0.0, 0.0, 0.0, 0.0};
    const int nv = 4 * nseg;
    for (int v0 = rs; v0 < nv; v0 += 32 * 8) {
      float4 w[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int v = v0 + 32 * u;
        w[u] = v < nv ? __ldcs(reinterpret_cast<const float4 *>(p.s0slots + ((size_t)seg_slot(seg(v >> 2), b) * 4 + (v & 3)) * p.Kp + j0 + 4 * g))
                      : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) { z[0] += (double)w[u].x; z[1] += (double)w[u].y; z[2] += (double)w[u].z; z[3] += (double)w[u].w; }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) { s_part[par][f][4 * g + e] = a[e]; s_p0[rs][4 * g + e] = z[e]; }
  }
  TRF(5);
  __syncthreads();
  if (tid < kLatJ) {  // S0 of Gaussian j0 + tid: the 32 row-slot partials in fixed order
    double S0 = 0.0;
    for (int r = 0; r < kLatThreads / 8; ++r) S0 += s_p0[r][tid];
    s_S0[tid] = S0 * (1.0 / (double)kPScale);  // S0 was accumulated from P = gamma 2^14
  }
  __syncthreads();
  TRF(6);
  float u = 0.f, v = 0.f;
  double ss = 0.0;
  if (valid) {
    const int fl = 2 * ok_;
    const double S0 = s_S0[oj];
    const double s1 = (s_part[0][fl][oj] + s_part[1][fl][oj]) * xs;
    const double s2 = (s_part[0][fl + 1][oj] + s_part[1][fl + 1][oj]) * (xs * xs * (double)kPScale);
    double U = (s1 - mup * S0) * isd;                                  // sum gamma (x - mu)/sd
    double V = (s2 - 2.0 * mup * s1 + mup * mup * S0) * ivar - S0;     // sum gamma ((x-mu)^2/var - 1)
    if (p.mode != 2) {
      const bool zero = !(N > 0.0);
      const double invN = zero ? 0.0 : 1.0 / N;
      if (p.mode == 0 && !zero) { U *= invN * psu; V *= invN * psv; }
      if (zero) U = V = 0.0;
      ss = fabs(U) + fabs(V);  // = (signed sqrt)^2
      u = signed_sqrt((float)U);
      v = signed_sqrt((float)V);
    } else {
      u = (float)U;
      v = (float)V;
    }
  }
  TRF(2);
  const int part = blockIdx.z * gridDim.x + blockIdx.x, nparts = gridDim.x * gridDim.z;
  float sc = 1.f;
  if (p.mode != 2) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    if (lane == 0) s_red[tid >> 5] = ss;
    __syncthreads();
    if (tid == 0) {
      double tot = 0.0;
      for (int w = 0; w < kLatThreads / 32; ++w) tot += s_red[w];
      p.norm2[(size_t)b * kFinMaxParts + part] = tot;  // own slot
      __threadfence();
      unsigned *ctr = p.counters + b;
      atomicAdd(ctr, 1u);
      while (atomicAdd(ctr, 0u) < (unsigned)nparts) __nanosleep(32);
      __threadfence();
    }
    __syncthreads();
    TRF(3);
    // fixed-order sum of the parts (the same bits in every block): lane l loads parts l, l + 32, then
    // a fixed xor tree
    double n2 = 0.0;
    for (int q = lane; q < nparts; q += 32) n2 += __ldcg(p.norm2 + (size_t)b * kFinMaxParts + q);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) n2 += __shfl_xor_sync(0xffffffffu, n2, off);
    if (n2 > 0.0) sc = (float)(1.0 / sqrt(n2));
  }
  if (valid) {
    const int KD = p.K * p.D;
    float *o = p.out + (size_t)b * 2 * KD + (size_t)j * p.D + k;
    o[0] = u * sc;
    o[KD] = v * sc;
  }
  TRF(4);
#ifdef GPUFV_TRACE
  if (p.trace && tid == 0) atomicMax(reinterpret_cast<unsigned long long *>(p.trace + 7724), (unsigned long long)ptx::globaltimer());
#endif
}

// ---------------------------------------------------------------------------------------------------
// Fused latency finalize: a single frame's a6 + a7 run by the stats kernel itself (k_stats<.., kFin>)
// after its last fold, instead of a k_finalize_lat launch behind it — no launch, no programmatic hand-
// off, and the coefficient loads overlap the grid barrier.  The arithmetic and its order are
// k_finalize_lat's (same segment split, same fp64 sums, same 64 norm parts), so the FVs are bitwise
// those of the two-kernel path (tests/test_gpu_parity.py).  The (K/32) x (D/8) "virtual blocks" of
// 256 threads are spread over the stats kernel's CTAs, two per CTA at a time (threads 0-511; a CTA
// may take several in turn when the frame has few clusters).  Two grid-wide barriers: every segment
// slot written; every partial norm published.  The stats grid is one co-resident wave (one CTA per
// SM, at most the occupancy query's cluster count; launched cooperatively).

// Grid-wide barrier on two words in the prepared GMM head (zeroed by k_prep_shift), called by one
// thread per CTA between __syncthreads.  Self-resetting: the last arrival zeroes the counter before it
// releases the next generation, so the words are back to {0, g + 1} after every use.
__device__ __forceinline__ void grid_barrier(unsigned *ctr, unsigned *gen, unsigned n) {
  unsigned g0, old;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g0) : "l"(gen) : "memory");
  // release: this CTA's writes (ordered before by the caller's __syncthreads) become visible with the
  // arrival; acquire: the last arrival sees every other CTA's writes before it releases the generation
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
  if (old == n - 1) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(ctr) : "memory");
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(gen), "r"(g0 + 1u) : "memory");
  } else {
    unsigned g;
    do {
      __nanosleep(20);
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(gen) : "memory");
    } while (g == g0);
  }
}

#ifndef GPUFV_FUSED_ROWS
#define GPUFV_FUSED_ROWS 10  // measured: 5,000 descriptors 29.0 -> 27.0 us, 8,000 31.0 -> 29.1 us (20: the loads spill)
#endif
struct LatScratch {  // one virtual block's shared memory (k_finalize_lat's __shared__ arrays)
  double part[2][2 * kLatK][kLatJ];
  double p0[kLatThreads / 8][kLatJ];
  double S0[kLatJ];
  double red[kLatThreads / 32];
  float dot[kLatThreads / 32][kMaxCls];  // fused scoring: per-warp partial dot products
};
constexpr int kLatGroups = 2;  // virtual blocks in flight per stats CTA (576 threads: 2 x 256)

// Virtual block vb = (bx, bz) of the single set: returns this thread's (unscaled) u, v and output
// offset, publishes the block's partial norm to norm2[vb].  gt = thread index in the group.
// kRows: slot rows per thread per round of loads.  The segments are summed in the same order for any
// kRows (each round continues the thread's chain si = par, par + 2, ...), so the result is bitwise
// k_finalize_lat's; inside the 96-register stats kernel fewer rows per round keep every load of a
// round in flight instead of spilling.
template <int kRows>
__device__ __forceinline__ void fin_lat_vblock(const FinParams &p, LatScratch &s, int vb, int gt, uint32_t bar,
                                               float &u, float &v, int64_t &oofs, bool &valid) {
  const int lat_x = (p.K + kLatJ - 1) / kLatJ;
  const int bx = vb % lat_x, bz = vb / lat_x, lane = gt & 31;
  const int j0 = bx * kLatJ, k0 = bz * kLatK, nseg = p.ncl;
  const size_t seg_stride = (size_t)2 * p.dpad * p.Kp;
  const int ok_ = gt & (kLatK - 1), oj = gt >> 3;
  const int j = j0 + oj, k = k0 + ok_;
  valid = k < p.D && j < p.K;
  const double N = (double)p.fused_n;
  double xs = 0.0, mup = 0.0, isd = 0.0, ivar = 0.0, psu = 0.0, psv = 0.0;
  if (valid) {
    xs = p.xinv[k];
    const double *cf = p.coef + (size_t)k * p.Kp + j;
    mup = cf[0]; isd = cf[kDMax * p.Kp]; ivar = cf[2 * kDMax * p.Kp];
    psu = p.pscale[j]; psv = p.pscale[p.Kp + j];
  }
  const int g = gt & 7, rs = gt >> 3;
  {
    const int f = rs & 15, par = rs >> 4, kf = k0 + (f >> 1);
    const size_t frow = (size_t)((f & 1) ? p.dpad + kf : kf) * p.Kp + j0 + 4 * g;
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    if (kf < p.D) {
      for (int s0 = par; s0 < nseg; s0 += 2 * kRows) {
        float4 w[kRows];
#pragma unroll
        for (int uu = 0; uu < kRows; ++uu) {
          const int si = s0 + 2 * uu;
          w[uu] = si < nseg ? __ldcg(reinterpret_cast<const float4 *>(p.slots + (size_t)seg_slot(si, 0) * seg_stride + frow))
                            : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int uu = 0; uu < kRows; ++uu) { a[0] += (double)w[uu].x; a[1] += (double)w[uu].y; a[2] += (double)w[uu].z; a[3] += (double)w[uu].w; }
      }
    }
    double z[4] = {0.0, 0.0, 0.0, 0.0};
    const int nv = 4 * nseg;
    for (int v0 = rs; v0 < nv; v0 += 32 * 8) {
      float4 w[8];
#pragma unroll
      for (int uu = 0; uu < 8; ++uu) {
        const int vv = v0 + 32 * uu;
        w[uu] = vv < nv ? __ldcg(reinterpret_cast<const float4 *>(p.s0slots + ((size_t)seg_slot(vv >> 2, 0) * 4 + (vv & 3)) * p.Kp + j0 + 4 * g))
                        : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int uu = 0; uu < 8; ++uu) { z[0] += (double)w[uu].x; z[1] += (double)w[uu].y; z[2] += (double)w[uu].z; z[3] += (double)w[uu].w; }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) { s.part[par][f][4 * g + e] = a[e]; s.p0[rs][4 * g + e] = z[e]; }
  }
  ptx::named_bar_sync(bar, kLatThreads);
  if (gt < kLatJ) {
    double S0 = 0.0;
    for (int r = 0; r < kLatThreads / 8; ++r) S0 += s.p0[r][gt];
    s.S0[gt] = S0 * (1.0 / (double)kPScale);
  }
  ptx::named_bar_sync(bar, kLatThreads);
  u = 0.f; v = 0.f;
  double ss = 0.0;
  if (valid) {
    const int fl = 2 * ok_;
    const double S0 = s.S0[oj];
    const double s1 = (s.part[0][fl][oj] + s.part[1][fl][oj]) * xs;
    const double s2 = (s.part[0][fl + 1][oj] + s.part[1][fl + 1][oj]) * (xs * xs * (double)kPScale);
    double U = (s1 - mup * S0) * isd;
    double V = (s2 - 2.0 * mup * s1 + mup * mup * S0) * ivar - S0;
    if (p.mode != 2) {
      const bool zero = !(N > 0.0);
      const double invN = zero ? 0.0 : 1.0 / N;
      if (p.mode == 0 && !zero) { U *= invN * psu; V *= invN * psv; }
      if (zero) U = V = 0.0;
      ss = fabs(U) + fabs(V);
      u = signed_sqrt((float)U);
      v = signed_sqrt((float)V);
    } else {
      u = (float)U;
      v = (float)V;
    }
  }
  oofs = (int64_t)j * p.D + k;
  if (p.n_cls > 0) {  // fused scoring (NEXT-4): this block's dot products with the classifier rows, on
                      // the FV before the L2 scale (k_finalize_img's order: U element, then V element)
    const int KD = p.K * p.D;
    for (int c = 0; c < p.n_cls; ++c) {
      float a = 0.f;
      if (valid) {
        const float *wc = p.svm_w + (size_t)c * 2 * KD;
        a = fmaf(u, __ldg(wc + oofs), a);
        a = fmaf(v, __ldg(wc + KD + oofs), a);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
      if (lane == 0) s.dot[gt >> 5][c] = a;
    }
  }
  if (p.mode != 2) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    if (lane == 0) s.red[gt >> 5] = ss;
  }
  if (p.mode != 2 || p.n_cls > 0) {
    ptx::named_bar_sync(bar, kLatThreads);
    if (p.mode != 2 && gt == 0) {
      double tot = 0.0;
      for (int w = 0; w < kLatThreads / 32; ++w) tot += s.red[w];
      p.norm2[vb] = tot;
    }
    if (gt < p.n_cls) {  // the block's partial per class, fixed warp order (bitwise repeatable)
      double d = 0.0;
      for (int w = 0; w < kLatThreads / 32; ++w) d += (double)s.dot[w][gt];
      p.spart[(size_t)vb * p.n_cls + gt] = d;
    }
  }
  ptx::named_bar_sync(bar, kLatThreads);  // the scratch is reused by the group's next virtual block
}

// Run by all threads of every CTA of the fused stats kernel after its last fold (tcgen05 work done).
constexpr uint32_t kBarFinGroup0 = 7;  // named barriers 7, 8: the two 256-thread groups
// (inlined: a __noinline__ version kept the tile loop's spills lower, 138 vs 266 bytes, but reached
// the kernel parameters and the shared scratch through generic pointers — 5,000 descriptors 27 -> 31 us)
__device__ __forceinline__ void fin_lat_fused(const FinParams &p, LatScratch *scr) {
  const int tid = threadIdx.x, cta = blockIdx.x, ncta = gridDim.x;
  const int lat_x = (p.K + kLatJ - 1) / kLatJ, lat_z = (p.D + kLatK - 1) / kLatK, nv = lat_x * lat_z;
  const int grp = tid / kLatThreads, gt = tid % kLatThreads;
  const bool active = grp < kLatGroups;
  const int KD = p.K * p.D;
#ifdef GPUFV_TRACE
#define TRFF(slot) do { if (p.trace && cta == 0 && tid == 0) p.trace[7700 + (slot)] = ptx::globaltimer(); } while (0)
#else
#define TRFF(slot) do { } while (0)
#endif
  TRFF(10);
  // barrier 1: every CTA's segment slots (stores / red.adds) and S0 slots are complete
  __syncthreads();
  if (tid == 0) grid_barrier(p.gbar, p.gbar + 32, (unsigned)ncta);
  __syncthreads();
  TRFF(11);
  if (cta == 0 && tid >= kLatGroups * kLatThreads && tid < kLatGroups * kLatThreads + 32) {
    // the image's range flag from the per-CTA words (k_finalize_lat's rule), by an otherwise idle warp
    const int l = tid & 31;
    int fl = 0;
    for (int c = l; c < p.nflag; c += 32) fl |= __ldcg(p.rflag_cta + c);
    fl = __reduce_or_sync(0xffffffffu, fl);
    if (l == 0) p.rflags[0] = fl;
  }
  // virtual blocks go to distinct CTAs first (the segment reads are bound by the L2 requests an SM
  // keeps in flight): vb = cta + ncta (grp + kLatGroups i)
  const int vb0 = cta + ncta * grp, vstep = kLatGroups * ncta;
  const int nmine = (active && vb0 < nv) ? (nv - 1 - vb0) / vstep + 1 : 0;
  float ku = 0.f, kv = 0.f;
  int64_t ko = 0;
  bool kval = false;
  for (int i = 0; i < nmine; ++i) {
    const int vb = vb0 + i * vstep;
    fin_lat_vblock<GPUFV_FUSED_ROWS>(p, scr[grp], vb, gt, kBarFinGroup0 + grp, ku, kv, ko, kval);
    // one virtual block: the values stay in registers until the norm is known; several: written
    // unscaled now and rescaled (re-read by the same thread) after the norm barrier
    if (p.out && kval && (nmine > 1 || p.mode == 2)) { p.out[ko] = ku; p.out[KD + ko] = kv; }
  }
  TRFF(12);
  if (p.mode == 2) return;  // (no scoring in this mode: the host keeps it on the two-kernel path)
  // barrier 2: every part's norm published; each thread sums the parts in the same fixed order
  __syncthreads();
  if (tid == 0) grid_barrier(p.gbar, p.gbar + 32, (unsigned)ncta);
  __syncthreads();
  TRFF(13);
  if (nmine == 0) return;
  const int lane = tid & 31;
  double n2 = 0.0;
  for (int q = lane; q < nv; q += 32) n2 += __ldcg(p.norm2 + q);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) n2 += __shfl_xor_sync(0xffffffffu, n2, off);
  const float sc = n2 > 0.0 ? (float)(1.0 / sqrt(n2)) : 1.f;
  if (p.n_cls > 0 && cta == 0 && tid < p.n_cls) {  // scores: the blocks' partials in block order
    double d = 0.0;
    for (int q = 0; q < nv; ++q) d += __ldcg(p.spart + (size_t)q * p.n_cls + tid);
    const double inv = n2 > 0.0 ? 1.0 / sqrt(n2) : 0.0;
    p.scores[tid] = (float)(d * inv + (p.svm_b ? (double)p.svm_b[tid] : 0.0));
  }
  if (!p.out) return;
  if (nmine == 1) {
    if (kval) { p.out[ko] = ku * sc; p.out[KD + ko] = kv * sc; }
    return;
  }
  for (int i = 0; i < nmine; ++i) {
    const int vb = vb0 + i * vstep, bx = vb % lat_x, bz = vb / lat_x;
    const int j = bx * kLatJ + (gt >> 3), k = bz * kLatK + (gt & (kLatK - 1));
    if (k < p.D && j < p.K) {
      float *o = p.out + (int64_t)j * p.D + k;
      o[0] = o[0] * sc;
      o[KD] = o[KD] * sc;
    }
  }
}

// a6 only: slots -> fp64 stats [N, S0, S1, S2] about c (reading A19).  Same grid as k_finalize.
__global__ void __launch_bounds__(256) k_reduce_stats(const FinParams p) {
  const int b = p.b_base + (int)blockIdx.y, tid = threadIdx.x, jj = tid & 31, kq = (tid >> 5) + kDP * (int)blockIdx.z;
  const int j = blockIdx.x * kFinJ + jj;
  if (j >= p.K) return;
  const int KD = p.K * p.D;
  double S0, S1[kFinKI], S2[kFinKI];
  slot_sums(p, b, j, kq, S0, S1, S2);
  double *st = p.stats_out + (size_t)b * (1 + (size_t)p.K * (2 * p.D + 1));
  if (blockIdx.x == 0 && blockIdx.z == 0 && tid == 0) st[0] = (double)(p.offsets[b + 1] - p.offsets[b]);
  if (kq == 0) st[1 + j] = S0;
#pragma unroll
  for (int i = 0; i < kFinKI; ++i) {
    const int k = kq + 8 * i;
    if (k < p.D) {
      st[1 + p.K + (size_t)j * p.D + k] = S1[i];
      st[1 + p.K + (size_t)KD + (size_t)j * p.D + k] = S2[i];
    }
  }
}

// ---------------------------------------------------------------- GMM EM (NEXT-3)
// Total log-likelihood of the E-step's descriptors under the input GMM (natural log):
//   LL = sum_i [ ln2 * ll2_i ] + N (bmax - D/2 ln 2 pi),
// ll2_i = log2 sum_j 2^(L_ij + b_j) from k_stats (b_j shifted by bmax and missing the -D/2 ln 2pi
// constant, which cancel in the posteriors, reading A2).  Fixed chunks per block summed in fp64 into
// the block's slot; the last block (ticket) sums the slots in block order: bitwise repeatable.
constexpr int kLLBlocks = 296;
__global__ void __launch_bounds__(256) k_loglik_reduce(const float *ll2, int64_t n, int D, const double *bmax,
                                                       double *parts, unsigned *ticket, double *out) {
  __shared__ double s_red[8];
  __shared__ int s_last;
  const int tid = threadIdx.x;
  const int64_t lo = (int64_t)blockIdx.x * n / gridDim.x, hi = (int64_t)(blockIdx.x + 1) * n / gridDim.x;
  double acc = 0.0;
  for (int64_t i = lo + tid; i < hi; i += 256) acc += (double)ll2[i];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((tid & 31) == 0) s_red[tid >> 5] = acc;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += s_red[w];
    parts[blockIdx.x] = t;
    __threadfence();
    s_last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last || tid != 0) return;
  __threadfence();
  double t = 0.0;
  for (unsigned b = 0; b < gridDim.x; ++b) t += __ldcg(parts + b);
  const double kLn2 = 0.69314718055994530941723212145818, kLn2Pi = 1.8378770664093454835606594728112;
  *out = kLn2 * t + (double)n * (*bmax - 0.5 * (double)D * kLn2Pi);
}

// M-step from the E-step statistics [N, S0 (K), S1 (KxD), S2 (KxD)] about c (reading A19):
//   mu_j = c + S1_j / S0_j,  var_j = S2_j / S0_j - (S1_j / S0_j)^2  (fp64; the moment form of the
//   oracle's two-pass definition), var <- max(var, max(floor_abs, floor_rel * var_k(X))) with
//   var_k(X) = sum_j S2_jk / N - (sum_j S1_jk / N)^2 (exact mode: sum_j gamma_ij = 1),
//   pi_j = max(S0_j / N, prior_floor) / sum;  S0_j == 0 keeps mu_j and var_j (reading A20).
// One block of 1024 threads (K(2D+1) <= 131,584 values).
__global__ void __launch_bounds__(1024) k_mstep(const double *st, int K, int D, const double *cshift, const float *w_old,
                                                const float *mu_old, const float *sg_old, int stddev, double floor_abs,
                                                double floor_rel, double prior_floor, float *w_new, float *mu_new,
                                                float *var_new) {
  __shared__ double s_floor[kDMax];
  __shared__ double s_red[32];
  __shared__ double s_a[1024], s_b[1024];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const double N = st[0];
  const double *S0 = st + 1, *S1 = st + 1 + K, *S2 = st + 1 + K + (size_t)K * D;
  (void)w_old;
  {  // global per-dimension moments from the statistics: dimension k = tid % dstride, Gaussian groups
     // tid / dstride (j = group + ngrp i), group partials summed in group order
    const int dstride = D <= kDP ? kDP : kDMax, ngrp = 1024 / dstride, k = tid % dstride, grp = tid / dstride;
    double a = 0.0, b = 0.0;
    if (k < D) {
#pragma unroll 4
      for (int j = grp; j < K; j += ngrp) { a += S1[(size_t)j * D + k]; b += S2[(size_t)j * D + k]; }
    }
    s_a[tid] = a; s_b[tid] = b;
    __syncthreads();
    if (grp == 0 && k < D) {
      double A = 0.0, B = 0.0;
      for (int g = 0; g < ngrp; ++g) { A += s_a[g * dstride + k]; B += s_b[g * dstride + k]; }
      const double m1 = N > 0.0 ? A / N : 0.0;
      const double gv = N > 0.0 ? B / N - m1 * m1 : 0.0;
      s_floor[k] = fmax(floor_abs, floor_rel * gv);
    }
  }
  double ps = 0.0;
  for (int j = tid; j < K; j += 1024) ps += fmax(N > 0.0 ? S0[j] / N : 0.0, prior_floor);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, off);
  if (lane == 0) s_red[wid] = ps;
  __syncthreads();
  double tot = 0.0;
  for (int w = 0; w < 32; ++w) tot += s_red[w];  // fixed order
  for (int j = tid; j < K; j += 1024) w_new[j] = (float)(fmax(N > 0.0 ? S0[j] / N : 0.0, prior_floor) / tot);
  for (int e = tid; e < K * D; e += 1024) {
    const int j = e / D, k = e - j * D;
    const double s0 = S0[j];
    double mu, var;
    if (s0 > 0.0) {
      const double m1 = S1[e] / s0;
      mu = cshift[k] + m1;
      var = S2[e] / s0 - m1 * m1;
    } else {
      mu = (double)mu_old[e];
      var = gmm_var(sg_old, e, stddev != 0);
    }
    mu_new[e] = (float)mu;
    var_new[e] = (float)fmax(var, s_floor[k]);
  }
}

}  // namespace gpufv
