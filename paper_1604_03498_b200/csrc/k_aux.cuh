// k_aux.cuh — the small kernels around k_stats:
//   k_prep_shift, k_prep_w   step a1: GMM -> prepared operands (Alg.1 l.1)
//   k_schedule               tile prefix sums from device offsets (ragged batches)
//   k_finalize               steps a6 (fixed-order fp64 slot reduction) + a7 (centring, VLFeat
//                            normalisation, P:449 / reading A9), also from fp64 stats (split path)
//   k_reduce_stats           a6 only -> fp64 sufficient statistics (descriptor-sharded path)
//   k_l2scale                global L2 normalisation of each image's FV
#pragma once
#include <cuda_fp16.h>
#include "fv_common.cuh"

namespace gpufv {

constexpr double kLog2e = 1.4426950408889634073599246810019;

__device__ __forceinline__ double gmm_var(const float *sigmas, size_t i, bool stddev) {
  double s = (double)sigmas[i];
  return stddev ? s * s : s;
}

// a1 (part 1): feature shift c_k = sum_j pi_j mu_jk / sum_j pi_j, power-of-two scale 2^e_k with
// e_k = -E where RMS_k = m 2^E (m in [0.5,1)), and the per-Gaussian bias
//   b_j = ln pi_j - 1/2 sum_k ln var_jk - 1/2 sum_k (mu_jk - c_k)^2 / var_jk    (minus max_j b_j)
// in log2 units.  One block of 256 threads.
__global__ void k_prep_shift(const float *w, const float *mu, const float *sg, int K, int D, int Kp,
                             int stddev, double *cshift, float *xshift, float *xscale, float *bias,
                             double *bscratch) {
  __shared__ double s_c[kDP];
  __shared__ double s_red[256];
  const int tid = threadIdx.x;
  if (tid < kDP) {
    double c = 0.0, sc = 1.0;
    if (tid < D) {
      double ws = 0.0, acc = 0.0;
      for (int j = 0; j < K; ++j) { ws += (double)w[j]; acc += (double)w[j] * (double)mu[(size_t)j * D + tid]; }
      c = acc / ws;
      double r = 0.0;
      for (int j = 0; j < K; ++j) {
        double d = (double)mu[(size_t)j * D + tid] - c;
        r += (double)w[j] * (gmm_var(sg, (size_t)j * D + tid, stddev) + d * d);
      }
      r = sqrt(r / ws);
      int E = 0;
      if (r > 0.0 && isfinite(r)) frexp(r, &E);
      sc = ldexp(1.0, -E);
    }
    s_c[tid] = c;
    cshift[tid] = c;
    xshift[tid] = (float)c;
    xscale[tid] = (float)sc;
  }
  __syncthreads();
  double bmax = -1e300;
  for (int j = tid; j < K; j += 256) {
    double ld = 0.0, q = 0.0;
    for (int k = 0; k < D; ++k) {
      double v = gmm_var(sg, (size_t)j * D + k, stddev);
      double d = (double)mu[(size_t)j * D + k] - s_c[k];
      ld += log(v);
      q += d * d / v;
    }
    double bj = log((double)w[j]) - 0.5 * ld - 0.5 * q;
    bscratch[j] = bj;
    bmax = fmax(bmax, bj);
  }
  s_red[tid] = bmax;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (tid < o) s_red[tid] = fmax(s_red[tid], s_red[tid + o]);
    __syncthreads();
  }
  bmax = s_red[0];
  for (int j = tid; j < Kp; j += 256)
    bias[j] = (j < K) ? (float)((bscratch[j] - bmax) * kLog2e) : -1.0e30f;
}

// a1 (part 2): W'_jf (log2 units, scaled by the feature exponents) split into fp16 hi/lo and stored
// as the exact SWIZZLE_128B K-major shared-memory image each CTA rank bulk-copies:
//   f <  64:  W'_jk      =  log2e (mu_jk - c_k) / var_jk * 2^-e_k
//   f >= 64:  W'_j,64+k  = -log2e / (2 var_jk)          * 2^-2e_k
// grid = Kp blocks (one Gaussian each), 128 threads (one feature each).
__global__ void k_prep_w(const float *mu, const float *sg, int K, int D, int stddev, const double *cshift,
                         const float *xscale, uint8_t *wimg) {
  const int j = blockIdx.x, f = threadIdx.x;
  const int k = f & (kDP - 1);
  double wv = 0.0;
  if (j < K && k < D) {
    const double v = gmm_var(sg, (size_t)j * D + k, stddev);
    const double s = (double)xscale[k];
    if (f < kDP) wv = kLog2e * ((double)mu[(size_t)j * D + k] - cshift[k]) / v / s;
    else wv = -kLog2e / (2.0 * v) / (s * s);
  }
  const float w32 = (float)wv;
  const __half hi = __float2half_rn(w32);
  const __half lo = __float2half_rn(w32 - __half2float(hi));
  const int rank = j / kG, row = j % kG, atom = f / 64, chunk = (f & 63) >> 3, e = f & 7;
  const size_t off = (size_t)rank * kWImgBytes + atom * kAtomBytes + row * 128 + ((chunk ^ (row & 7)) << 4) + e * 2;
  *reinterpret_cast<__half *>(wimg + off) = hi;
  *reinterpret_cast<__half *>(wimg + off + kOpBytes) = lo;
}

// tile_start[0] = 0, tile_start[b+1] = sum_{b' <= b} ceil(N_b' / 128).  One block of 1024 threads.
// offsets == nullptr means a single set of n_single rows: {0, n_single} is written to off1 and used.
__global__ void k_schedule(const int64_t *offsets, int64_t *off1, int64_t n_single, int batch, int64_t *tile_start) {
  __shared__ int64_t s_warp[32];
  __shared__ int64_t s_carry;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (!offsets) {
    if (tid == 0) {
      off1[0] = 0; off1[1] = n_single;
      tile_start[0] = 0; tile_start[1] = (n_single + kTileM - 1) / kTileM;
    }
    return;
  }
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

struct FinParams {
  const float *partials;      // from k_stats (nullptr when reading stats)
  const double *stats;        // batch x (1 + K(2D+1)) (nullptr when reading partials)
  const int64_t *offsets;     // batch + 1 (partials mode)
  const int64_t *tile_start;  // batch + 1 (partials mode)
  const float *w, *mu, *sg;
  const double *cshift;
  const float *xscale;
  float *out;                 // batch x 2KD
  double *stats_out;          // k_reduce_stats output
  double *norm2;              // batch
  int batch, K, Kp, D, ncl, stddev, mode;
};

// Owner cluster of global tile t under the static split [c T / ncl, (c+1) T / ncl).
__device__ __forceinline__ int64_t tile_owner(int64_t t, int64_t T, int64_t ncl) { return ((t + 1) * ncl - 1) / T; }

// Fixed-order (ascending cluster) fp64 reduction of image b's partial slots, unscaled.
__device__ __forceinline__ void slot_sums(const FinParams &p, int b, int j, int k, double &S0, double &S1, double &S2,
                                          double &N) {
  N = (double)(p.offsets[b + 1] - p.offsets[b]);
  S0 = S1 = S2 = 0.0;
  const int64_t T = p.tile_start[p.batch];
  const int64_t ft = p.tile_start[b], lt = p.tile_start[b + 1] - 1;
  if (ft > lt) return;
  const int64_t clo = tile_owner(ft, T, p.ncl), chi = tile_owner(lt, T, p.ncl);
  const size_t SL = (size_t)(1 + kNF) * p.Kp;
  for (int64_t c = clo; c <= chi; ++c) {
    if ((c * T) / p.ncl == ((c + 1) * T) / p.ncl) continue;  // cluster with an empty tile range wrote nothing
    const float *sl = p.partials + (size_t)(c + b) * SL;
    S0 += (double)sl[j];
    S1 += (double)sl[(size_t)(1 + k) * p.Kp + j];
    S2 += (double)sl[(size_t)(1 + kDP + k) * p.Kp + j];
  }
  const double xs = (double)p.xscale[k];
  // S0 is accumulated from gamma itself (registers), S1/S2 from gamma * 2^14 (GEMM2 operand)
  S1 /= (double)kPScale * xs;
  S2 /= (double)kPScale * xs * xs;
}

// grid (ceil(K*D/256), batch), 256 threads; thread -> (k, j) with j fastest (coalesced slot reads).
__global__ void k_finalize(const FinParams p) {
  __shared__ double s_red[256];
  const int b = blockIdx.y;
  const int pidx = blockIdx.x * blockDim.x + threadIdx.x;
  const int KD = p.K * p.D;
  double ss = 0.0;
  if (pidx < KD) {
    const int k = pidx / p.K, j = pidx - k * p.K;
    double S0, S1, S2, N;
    if (p.partials) {
      slot_sums(p, b, j, k, S0, S1, S2, N);
    } else {
      const double *st = p.stats + (size_t)b * (1 + (size_t)p.K * (2 * p.D + 1));
      N = st[0];
      S0 = st[1 + j];
      S1 = st[1 + p.K + (size_t)j * p.D + k];
      S2 = st[1 + p.K + (size_t)KD + (size_t)j * p.D + k];
    }
    const double var = gmm_var(p.sg, (size_t)j * p.D + k, p.stddev);
    const double mup = (double)p.mu[(size_t)j * p.D + k] - p.cshift[k];
    double U = (S1 - mup * S0) / sqrt(var);
    double V = (S2 - 2.0 * mup * S1 + mup * mup * S0) / var - S0;
    if (p.mode != 2) {
      if (N <= 0.0) { U = 0.0; V = 0.0; }
      if (p.mode == 0) {
        const double pj = (double)p.w[j];
        U /= N * sqrt(pj);
        V /= N * sqrt(2.0 * pj);
      }
      U = (U > 0.0) ? sqrt(U) : ((U < 0.0) ? -sqrt(-U) : 0.0);
      V = (V > 0.0) ? sqrt(V) : ((V < 0.0) ? -sqrt(-V) : 0.0);
      ss = U * U + V * V;
    }
    float *o = p.out + (size_t)b * 2 * KD;
    o[(size_t)j * p.D + k] = (float)U;
    o[(size_t)KD + (size_t)j * p.D + k] = (float)V;
  }
  if (p.mode == 2) return;
  s_red[threadIdx.x] = ss;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) s_red[threadIdx.x] += s_red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0 && s_red[0] != 0.0) atomicAdd(p.norm2 + b, s_red[0]);
}

// grid (ceil(2KD/1024), batch), 256 threads x float4.
__global__ void k_l2scale(float *out, const double *norm2, int KD2) {
  const int b = blockIdx.y;
  const double n2 = norm2[b];
  if (!(n2 > 0.0)) return;
  const float sc = (float)(1.0 / sqrt(n2));
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  float *o = out + (size_t)b * KD2;
  if (i + 3 < KD2) {
    float4 v = *reinterpret_cast<float4 *>(o + i);
    v.x *= sc; v.y *= sc; v.z *= sc; v.w *= sc;
    *reinterpret_cast<float4 *>(o + i) = v;
  } else {
    for (int t = i; t < KD2; ++t) o[t] *= sc;
  }
}

// a6 only: partial slots -> fp64 stats [N, S0, S1, S2] about c (reading A19).
__global__ void k_reduce_stats(const FinParams p) {
  const int b = blockIdx.y;
  const int pidx = blockIdx.x * blockDim.x + threadIdx.x;
  const int KD = p.K * p.D;
  if (pidx >= KD) return;
  const int k = pidx / p.K, j = pidx - k * p.K;
  double S0, S1, S2, N;
  slot_sums(p, b, j, k, S0, S1, S2, N);
  double *st = p.stats_out + (size_t)b * (1 + (size_t)p.K * (2 * p.D + 1));
  if (pidx == 0) st[0] = N;
  if (k == 0) st[1 + j] = S0;
  st[1 + p.K + (size_t)j * p.D + k] = S1;
  st[1 + p.K + (size_t)KD + (size_t)j * p.D + k] = S2;
}

}  // namespace gpufv
