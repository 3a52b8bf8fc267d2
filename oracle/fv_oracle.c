/*
 * fv_oracle.c — CPU double-precision ORACLE for Fisher-vector encoding (GPU-FV, arXiv 1604.03498).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (paper_1604_03498_b200/) may include,
 * link or call this file.  Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * `--impl reference`) use it.  It shares no code, header, table or constant with the CUDA path.
 *
 * It is deliberately plain and slow: IEEE double, round-to-nearest, no fast-math, `exp`/`log`/`sqrt`
 * from libm, loops in the order the paper writes them.  Citations: P:<line> = PAPER.md line,
 * S:<line> = SPEC.md line (the readings are listed in DESIGN.md §3, "Readings of the paper").
 *
 * Functions and what pins them (tests/test_oracle.py):
 *   fvo_posteriors   Alg.1 lines 2-15             pinned: K=1, symmetry, ratio closed form,
 *                                                              mpmath density brute force, invariants
 *   fvo_accumulate   Alg.1 lines 16-26            pinned: x=mu special case, K=1 moment
 *                                                              identity, tau cut-off, mpmath brute force
 *   fvo_normalize    "same encoding scheme as VLFeat"  pinned: unit norm, zero stays zero,
 *                    improved FV reading A9            K=1 x=mu closed form, duplication invariance
 *   fvo_stats        raw sufficient statistics about the       pinned: identities against fvo_accumulate
 *                    GMM-weighted mean c (A19)       (U = (S1-mu'S0)/sd etc.), mpmath brute force
 *   fvo_encode / fvo_encode_batched / fvo_stats_batched: compositions of the above (no new arithmetic).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Normalisation modes (reading A9). Same numeric values as the public header's flags,
 * restated here on purpose: the oracle does not include the product header. */
#define FVO_NORM_IMPROVED 0 /* U/(N sqrt(pi)), V/(N sqrt(2 pi)), signed sqrt, global L2 */
#define FVO_NORM_POWER_L2 1 /* signed sqrt, global L2 only                                 */
#define FVO_NORM_NONE 2     /* raw Alg.1 sums U, V                                           */

/* Block size of the paper's "one copy of U and V for each block" reduction (Alg.3).
 * Fixed (not thread-count dependent) so results do not depend on the number of OpenMP threads. */
#define FVO_BLOCK 4096

/* ---------------------------------------------------------------------------------------------
 * Phase 1 — posteriors.  Alg.1 lines 2-15, reading A2 for "distance"/"temp" and A3 for
 * the per-descriptor reset of maxPost and sum.
 *   l_ij   = ln pi_j - 1/2 sum_k ln var_jk - 1/2 sum_k (x_ik - mu_jk)^2 / var_jk      (direct form)
 *   maxPost = max_j l_ij ;  e_ij = exp(l_ij - maxPost) ;  sum = sum_j e_ij ;  gamma_ij = e_ij / sum
 * The -D/2 ln(2 pi) constant is included (it cancels; including it keeps l a true log-density).
 * --------------------------------------------------------------------------------------------- */
void fvo_posteriors(const double *X, int64_t N, int D, const double *priors, const double *means,
                    const double *vars, int K, double *gamma /* N x K */) {
  const double log2pi = log(2.0 * M_PI);
  for (int64_t i = 0; i < N; ++i) {
    const double *x = X + i * (int64_t)D;
    double *g = gamma + i * (int64_t)K;
    double maxPost = -INFINITY; /* reset per descriptor (A3) */
    for (int j = 0; j < K; ++j) {
      double t = 0.0; /* "t = distance(data[i], means_j, covariances_j)" (Alg.1 l.4) */
      double logdet = 0.0;
      for (int k = 0; k < D; ++k) {
        double d = x[k] - means[(int64_t)j * D + k];
        t += d * d / vars[(int64_t)j * D + k];
        logdet += log(vars[(int64_t)j * D + k]);
      }
      /* "Compute posteriors_{i,j} with temp" (Alg.1 l.5): log prior + Gaussian log-density */
      g[j] = log(priors[j]) - 0.5 * logdet - 0.5 * t - 0.5 * D * log2pi;
      if (g[j] > maxPost) maxPost = g[j]; /* Alg.1 l.6 */
    }
    double sum = 0.0; /* reset per descriptor (A3) */
    for (int j = 0; j < K; ++j) { /* Alg.1 l.8-11 */
      g[j] = exp(g[j] - maxPost);
      sum += g[j];
    }
    for (int j = 0; j < K; ++j) g[j] = g[j] / sum; /* Alg.1 l.12-14 */
  }
}

/* ---------------------------------------------------------------------------------------------
 * Phase 2 — accumulation, Alg.1 lines 16-26, literally:
 *   if gamma_ij > threshold:  U_jk += (x_ik - mu_jk) * sqrt(1/var_jk) * gamma_ij
 *                             V_jk += (((x_ik - mu_jk) * sqrt(1/var_jk))^2 - 1) * gamma_ij
 * threshold <= 0 means exact mode (every pair included; reading A5).  Strict '>' (A5).  No
 * renormalisation of thresholded posteriors (A6).  U, V are K x D, accumulated (+=), caller zeroes.
 * --------------------------------------------------------------------------------------------- */
void fvo_accumulate(const double *X, int64_t N, int D, const double *gamma, const double *means,
                    const double *vars, int K, double threshold, double *U, double *V) {
  for (int64_t i = 0; i < N; ++i) {
    const double *x = X + i * (int64_t)D;
    for (int j = 0; j < K; ++j) {
      double p = gamma[i * (int64_t)K + j];
      if (threshold > 0.0 && !(p > threshold)) continue; /* Alg.1 l.18 */
      for (int k = 0; k < D; ++k) {
        double isq = sqrt(1.0 / vars[(int64_t)j * D + k]); /* "sqrt(sigma^-1)", Alg.1 l.1 */
        double z = (x[k] - means[(int64_t)j * D + k]) * isq;
        U[(int64_t)j * D + k] += z * p;             /* Alg.1 l.20 */
        V[(int64_t)j * D + k] += (z * z - 1.0) * p; /* Alg.1 l.21 */
      }
    }
  }
}

/* ---------------------------------------------------------------------------------------------
 * Normalisation (reading A9: VLFeat "improved" FV):
 *   U_jk /= N sqrt(pi_j) ; V_jk /= N sqrt(2 pi_j) ; z <- sign(z) sqrt|z| ; z /= ||z||_2 (0 stays 0)
 * fv = [U (K x D row-major), V (K x D row-major)] (reading A8).  N = all descriptors (A10).
 * --------------------------------------------------------------------------------------------- */
void fvo_normalize(double *fv, int K, int D, int64_t N, const double *priors, int mode) {
  const int64_t KD = (int64_t)K * D;
  if (mode == FVO_NORM_NONE) return;
  if (N == 0) { /* empty image: all-zero FV, never NaN (A11) */
    for (int64_t t = 0; t < 2 * KD; ++t) fv[t] = 0.0;
    return;
  }
  if (mode == FVO_NORM_IMPROVED) {
    for (int j = 0; j < K; ++j)
      for (int k = 0; k < D; ++k) {
        fv[(int64_t)j * D + k] /= (double)N * sqrt(priors[j]);
        fv[KD + (int64_t)j * D + k] /= (double)N * sqrt(2.0 * priors[j]);
      }
  }
  double nrm2 = 0.0;
  for (int64_t t = 0; t < 2 * KD; ++t) {
    double z = fv[t];
    z = (z > 0.0) ? sqrt(z) : ((z < 0.0) ? -sqrt(-z) : 0.0); /* signed square root */
    fv[t] = z;
    nrm2 += z * z;
  }
  if (nrm2 > 0.0) {
    double nrm = sqrt(nrm2);
    for (int64_t t = 0; t < 2 * KD; ++t) fv[t] /= nrm;
  }
}

/* Encode one descriptor set: Phase 1, Phase 2 (in fixed blocks of FVO_BLOCK descriptors with one
 * U,V copy per block summed in block order — Alg.3), normalisation.  Returns 0, or -1 on
 * allocation failure.  gamma_out (N x K) is optional. */
int fvo_encode(const double *X, int64_t N, int D, const double *priors, const double *means,
               const double *vars, int K, double threshold, int mode, double *fv /* 2KD */,
               double *gamma_out) {
  const int64_t KD = (int64_t)K * D;
  double *g = (double *)malloc(sizeof(double) * (size_t)FVO_BLOCK * K);
  double *Ub = (double *)malloc(sizeof(double) * (size_t)KD);
  double *Vb = (double *)malloc(sizeof(double) * (size_t)KD);
  if (!g || !Ub || !Vb) { free(g); free(Ub); free(Vb); return -1; }
  for (int64_t t = 0; t < 2 * KD; ++t) fv[t] = 0.0;
  for (int64_t i0 = 0; i0 < N; i0 += FVO_BLOCK) {
    int64_t n = (N - i0 < FVO_BLOCK) ? (N - i0) : FVO_BLOCK;
    fvo_posteriors(X + i0 * D, n, D, priors, means, vars, K, g);
    if (gamma_out) memcpy(gamma_out + i0 * K, g, sizeof(double) * (size_t)(n * K));
    memset(Ub, 0, sizeof(double) * (size_t)KD);
    memset(Vb, 0, sizeof(double) * (size_t)KD);
    fvo_accumulate(X + i0 * D, n, D, g, means, vars, K, threshold, Ub, Vb);
    for (int64_t t = 0; t < KD; ++t) { fv[t] += Ub[t]; fv[KD + t] += Vb[t]; } /* block copies summed in order */
  }
  fvo_normalize(fv, K, D, N, priors, mode);
  free(g); free(Ub); free(Vb);
  return 0;
}

/* Batched: images are independent (offsets[b]..offsets[b+1]); OpenMP over images only, each image
 * computed by the same serial code, so the result does not depend on the thread count. */
int fvo_encode_batched(const double *X, const int64_t *offsets, int batch, int D, const double *priors,
                       const double *means, const double *vars, int K, double threshold, int mode,
                       double *out /* batch x 2KD */, int nthreads) {
  int err = 0;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1) reduction(| : err)
#endif
  for (int b = 0; b < batch; ++b) {
    int64_t n = offsets[b + 1] - offsets[b];
    err |= fvo_encode(X + offsets[b] * D, n, D, priors, means, vars, K, threshold, mode,
                      out + (int64_t)b * 2 * K * D, NULL) ? 1 : 0;
  }
  (void)nthreads;
  return err ? -1 : 0;
}

/* ---------------------------------------------------------------------------------------------
 * Sufficient statistics (reading A19) of one descriptor set about the GMM-weighted mean
 *   c_k = sum_j pi_j mu_jk / sum_j pi_j :
 *   stats = [ N, S0 (K), S1 (K x D), S2 (K x D) ]   with (only pairs with gamma_ij > threshold in
 *   thresholded mode)  S0_j = sum_i gamma_ij,  S1_jk = sum_i gamma_ij (x_ik - c_k),
 *   S2_jk = sum_i gamma_ij (x_ik - c_k)^2.
 * These are the quantities summed across GPUs in the descriptor-sharded path; the FV follows from
 * them by U = (S1 - mu' S0)/sd, V = (S2 - 2 mu' S1 + mu'^2 S0)/var - S0 with mu' = mu - c, which
 * tests/test_oracle.py checks against fvo_accumulate (the literal Alg.1 sums).
 * --------------------------------------------------------------------------------------------- */
int fvo_stats(const double *X, int64_t N, int D, const double *priors, const double *means,
              const double *vars, int K, double threshold, double *stats /* 1 + K(2D+1) */) {
  const int64_t KD = (int64_t)K * D;
  double *c = (double *)calloc((size_t)D, sizeof(double));
  double *g = (double *)malloc(sizeof(double) * (size_t)FVO_BLOCK * K);
  if (!c || !g) { free(c); free(g); return -1; }
  double wsum = 0.0;
  for (int j = 0; j < K; ++j) wsum += priors[j];
  for (int j = 0; j < K; ++j)
    for (int k = 0; k < D; ++k) c[k] += priors[j] * means[(int64_t)j * D + k];
  for (int k = 0; k < D; ++k) c[k] /= wsum;
  double *S0 = stats + 1, *S1 = stats + 1 + K, *S2 = stats + 1 + K + KD;
  memset(stats, 0, sizeof(double) * (size_t)(1 + K + 2 * KD));
  stats[0] = (double)N;
  for (int64_t i0 = 0; i0 < N; i0 += FVO_BLOCK) {
    int64_t n = (N - i0 < FVO_BLOCK) ? (N - i0) : FVO_BLOCK;
    fvo_posteriors(X + i0 * D, n, D, priors, means, vars, K, g);
    for (int64_t i = 0; i < n; ++i) {
      const double *x = X + (i0 + i) * D;
      for (int j = 0; j < K; ++j) {
        double p = g[i * K + j];
        if (threshold > 0.0 && !(p > threshold)) continue;
        S0[j] += p;
        for (int k = 0; k < D; ++k) {
          double d = x[k] - c[k];
          S1[(int64_t)j * D + k] += p * d;
          S2[(int64_t)j * D + k] += p * d * d;
        }
      }
    }
  }
  free(c); free(g);
  return 0;
}

int fvo_stats_batched(const double *X, const int64_t *offsets, int batch, int D, const double *priors,
                      const double *means, const double *vars, int K, double threshold,
                      double *stats /* batch x (1 + K(2D+1)) */, int nthreads) {
  int err = 0;
  const int64_t SL = 1 + (int64_t)K * (2 * D + 1);
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1) reduction(| : err)
#endif
  for (int b = 0; b < batch; ++b)
    err |= fvo_stats(X + offsets[b] * D, offsets[b + 1] - offsets[b], D, priors, means, vars, K,
                     threshold, stats + (int64_t)b * SL) ? 1 : 0;
  (void)nthreads;
  return err ? -1 : 0;
}

int fvo_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
