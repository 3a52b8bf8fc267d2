/*
 * gpufv.h — C ABI of the B200-native Fisher-vector encoder (GPU-FV, Ma et al., ICMR'16, arXiv 1604.03498).
 *
 * What is computed (PAPER.md = P:<line>; readings A1..A19 are listed in DESIGN.md §3):
 *   For an image with descriptors x_1..x_N (D dims) and a diagonal GMM (K components, priors pi_j,
 *   means mu_jk, variances var_jk — the paper's "covariances", reading A1):
 *     Phase 1, Alg.1 l.2-15:  l_ij = ln pi_j - 1/2 sum_k ln var_jk - 1/2 sum_k (x_ik-mu_jk)^2/var_jk
 *                                          gamma_ij = exp(l_ij - max_j l_ij) / sum_j exp(l_ij - max_j l_ij)
 *     Phase 2, Alg.1 l.16-26: for every (i,j) with gamma_ij > threshold (all pairs if threshold <= 0):
 *                                          U_jk += gamma_ij (x_ik-mu_jk)/sqrt(var_jk)
 *                                          V_jk += gamma_ij ((x_ik-mu_jk)^2/var_jk - 1)
 *     Normalisation, "same encoding scheme as VLFeat" (reading A9): U_jk /= N sqrt(pi_j),
 *       V_jk /= N sqrt(2 pi_j), z <- sign(z) sqrt|z|, z /= ||z||_2 (an all-zero vector stays zero).
 *   Output per image: 2*K*D floats, U block (K x D row-major, by Gaussian) then V block (reading A8).
 *
 * Conventions for every function below:
 *   - Array arguments are CUDA DEVICE pointers on the current device unless the name ends in _host.
 *     The library never allocates, frees or synchronises on the device paths; all work is enqueued
 *     asynchronously on `stream` (NULL = legacy default stream).  The caller owns every buffer.
 *   - fp32 in, fp32 out.  Sufficient statistics accumulate on the tensor cores in fp32 chunks of <= 16
 *     tiles that are added, in a fixed program order, into one fp32 slot per (cluster, image); slots are
 *     combined and normalised in fp64.  Results are deterministic (static schedule + fixed-order
 *     reductions): identical inputs give bitwise-identical outputs.
 *   - Limits: 1 <= K <= 512, 1 <= D <= 128, D % 4 == 0 (caller pads, reading A13), X 16-byte aligned.
 *     D <= 64 runs the narrow kernel (128 Gaussians per CTA); 64 < D <= 128 the wide one (64 per CTA).
 *   - Device data is not validated synchronously (that would need a kernel + sync): pi <= 0 gives NaN
 *     for the images it touches.  Inputs outside the fp16 operand range of the split contractions —
 *     descriptors with |x-c|/rms >= ~256 in some dimension (c, rms: GMM-weighted mean/RMS), components
 *     with a standard deviation below ~rms/150 in some dimension, var <= 0, non-finite X — make the
 *     affected images' outputs NaN (never finite garbage) and are reported per image by
 *     fv_range_flags().
 *   - Synchronous argument errors return a status; asynchronous CUDA errors are reported by the
 *     next call or by cudaGetLastError.  fv_last_error() returns a thread-local detail string.
 *   - Thread safety: reentrant; concurrent calls need distinct workspaces.
 */
#ifndef GPUFV_H
#define GPUFV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *fv_stream_t; /* == cudaStream_t */

typedef enum {
  FV_OK = 0,
  FV_ERR_ARG = 1,         /* null pointer, N/batch < 0, K < 1, D < 1, threshold NaN or >= 1, bad flags */
  FV_ERR_UNSUPPORTED = 2, /* K > 512, D > 128, D % 4 != 0, misaligned X, device is not sm_100     */
  FV_ERR_WORKSPACE = 3,   /* ws_bytes < fv_workspace_bytes(...) or ws misaligned (needs 1024 B)    */
  FV_ERR_CUDA = 4         /* a CUDA launch/runtime call failed (detail in fv_last_error())          */
} fv_status;

enum {
  FV_NORM_IMPROVED = 0,       /* default: 1/(N sqrt(pi)), 1/(N sqrt(2 pi)), signed sqrt, L2  (A9) */
  FV_NORM_POWER_L2 = 1,       /* signed sqrt + L2 only                                          */
  FV_NORM_NONE = 2,           /* raw Alg.1 sums U, V                                            */
  FV_NORM_MASK = 3,
  FV_SIGMA_IS_STDDEV = 1u << 4, /* `sigmas` are standard deviations (default: variances, A1)    */
  /* bit 5 is reserved: every path is deterministic (fixed-order reductions, no float atomics whose
     order varies), so there is no determinism flag */
  FV_PREPARED = 1u << 6,        /* `ws` already holds this GMM prepared by fv_gmm_prepare: skip a1 */
  FV_SPARSE_STATS = 1u << 7     /* threshold > 0, D <= 64, K <= 256: accumulate only the pairs gamma > tau
                                   on the CUDA cores (Alg. 5 early termination, round-to-nearest fp32 sums)
                                   instead of the dense tensor-core GEMM2; same result to rounding, slower
                                   on the acceptance generator */
};

/* Bytes of device workspace needed by the calls below for this problem size.  n_total = total
 * descriptors, batch = images per call.  With FV_HOST_IO_BYTES semantics the _host entry point also
 * needs room for the device copies of X, offsets and out: use fv_workspace_bytes_host. */
size_t fv_workspace_bytes(int64_t n_total, int batch, int K, int D, unsigned flags);
size_t fv_workspace_bytes_host(int64_t n_total, int batch, int K, int D, unsigned flags);

/* Step a1 (Alg.1 l.1 "Compute sqrt(sigma^-1)"; done "with a simple GPU kernel"):
 * prepares the GMM-derived operands (fp16 hi/lo split of [mu'/var, -1/(2 var)], log-prior+log-det
 * bias, feature shift c = sum_j pi_j mu_j / sum_j pi_j and power-of-two feature scales) into the head
 * of `ws`.  Later calls on the same ws may pass FV_PREPARED to skip it. */
fv_status fv_gmm_prepare(const float *weights /*K*/, const float *means /*KxD*/, const float *sigmas /*KxD*/,
                         int K, int D, unsigned flags, void *ws, size_t ws_bytes, fv_stream_t stream);

/* One descriptor set X (N x D row-major) -> out (2KD).  N == 0 gives an all-zero FV (A11).
 * Latency path (D <= 64, K <= 256, a frame small enough for one tile per cluster): ONE kernel launch —
 * the finalize runs inside the statistics kernel after a grid-wide barrier whose two words live in the
 * prepared head of `ws` (zeroed by the GMM preparation, back to zero after every call).  Its CTAs must
 * all be resident at once (at most the co-resident cluster count is launched; on a GPU shared with
 * other work the call waits for SMs to free up).  The same holds for one-image fv_encode_batched. */
fv_status fv_encode(const float *X, int64_t N, int D, const float *weights, const float *means,
                    const float *sigmas, int K, float threshold, unsigned flags, float *out,
                    void *ws, size_t ws_bytes, fv_stream_t stream);

/* A batch of independent images: X (n_total x D), image b = rows offsets[b]..offsets[b+1]-1
 * (`offsets`: device int64 array of batch+1 non-decreasing entries, offsets[0]=0, offsets[batch]=n_total)
 * -> out (batch x 2KD). */
fv_status fv_encode_batched(const float *X, const int64_t *offsets, int batch, int64_t n_total, int D,
                            const float *weights, const float *means, const float *sigmas, int K,
                            float threshold, unsigned flags, float *out, void *ws, size_t ws_bytes,
                            fv_stream_t stream);

/* Same as fv_encode_batched but X_host / offsets_host / out_host are HOST buffers (pinned for full
 * PCIe speed); the GMM arrays stay device pointers (a resident model).  The batch is processed in up to
 * 16 image chunks: the host->device copy of chunk k+1 and the device->host copy of chunk k-1 run on two
 * internal streams while chunk k is encoded on `stream`; the internal streams first wait for all work
 * already queued on `stream`, and the call synchronises all three before returning.  The two streams
 * and their events are created on the first host call of a (thread, device) and reused afterwards.
 * offsets_host is validated before any copy (offsets[0] == 0, non-decreasing, offsets[batch] ==
 * n_total; else FV_ERR_ARG).  Each chunk runs the device path on its own images, so
 * results equal fv_encode_batched's to rounding (same images, different static schedule) and are
 * bitwise repeatable across calls.  ws >= fv_workspace_bytes_host(...). */
fv_status fv_encode_batched_host(const float *X_host, const int64_t *offsets_host, int batch, int64_t n_total,
                                 int D, const float *weights, const float *means, const float *sigmas, int K,
                                 float threshold, unsigned flags, float *out_host, void *ws, size_t ws_bytes,
                                 fv_stream_t stream);

/* Fused linear scoring (the paper's video-monitoring application trains "a
 * classification model with liblinear" on per-frame FVs and predicts every frame):
 *   scores[b * n_cls + c] = sum_d svm_w[c * 2KD + d] * fv_b[d] + svm_b[c]
 * where fv_b is image b's FV exactly as fv_encode_batched would return it (same flags/normalisation).
 * svm_w: device, n_cls x 2KD fp32 (row c laid out like one FV: U block then V block); svm_b: device,
 * n_cls fp32 or NULL (zero bias); 1 <= n_cls <= 32 (else FV_ERR_ARG).  The dot products are taken in
 * the finalize kernel on the tile it has just computed (per-block partials in fixed slots, summed in
 * block order, scaled by the image's 1/||z||): bitwise repeatable.  `out` (batch x 2KD) may be NULL:
 * then the FVs never reach HBM and only batch x n_cls floats leave the kernel.
 * ws >= fv_workspace_bytes_scored(n_total, batch, K, D, n_cls, 0, flags). */
size_t fv_workspace_bytes_scored(int64_t n_total, int batch, int K, int D, int n_cls, int host_io, unsigned flags);
fv_status fv_encode_scored_batched(const float *X, const int64_t *offsets, int batch, int64_t n_total, int D,
                                   const float *weights, const float *means, const float *sigmas, int K,
                                   float threshold, unsigned flags, const float *svm_w, const float *svm_b, int n_cls,
                                   float *scores, float *out, void *ws, size_t ws_bytes, fv_stream_t stream);

/* Host-buffer variant for the monitoring stream: X_host / offsets_host in (pinned host), scores_host
 * (batch x n_cls) out; GMM and classifier stay device-resident.  Same chunked H2D / encode / D2H
 * pipeline as fv_encode_batched_host, but only the scores cross PCIe back.
 * ws >= fv_workspace_bytes_scored(n_total, batch, K, D, n_cls, 1, flags). */
fv_status fv_encode_scored_batched_host(const float *X_host, const int64_t *offsets_host, int batch, int64_t n_total,
                                        int D, const float *weights, const float *means, const float *sigmas, int K,
                                        float threshold, unsigned flags, const float *svm_w, const float *svm_b,
                                        int n_cls, float *scores_host, void *ws, size_t ws_bytes, fv_stream_t stream);

/* Split path for descriptor sharding (a2-a6 without a7).  stats: batch x (1 + K(2D+1)) doubles,
 *   stats[b] = [ N_b, S0 (K), S1 (K x D), S2 (K x D) ],
 *   S0_j = sum_i gamma_ij,  S1_jk = sum_i gamma_ij (x_ik - c_k),  S2_jk = sum_i gamma_ij (x_ik - c_k)^2,
 * summed over included pairs, about c = sum_j pi_j mu_j / sum_j pi_j (reading A19).  Statistics of
 * disjoint descriptor sets add (the NCCL all-reduce of the sharded path). */
fv_status fv_stats_batched(const float *X, const int64_t *offsets, int batch, int64_t n_total, int D,
                           const float *weights, const float *means, const float *sigmas, int K,
                           float threshold, unsigned flags, double *stats, void *ws, size_t ws_bytes,
                           fv_stream_t stream);

/* a7: stats (as above, possibly summed across GPUs) -> out (batch x 2KD):
 *   U = (S1 - mu' S0)/sqrt(var), V = (S2 - 2 mu' S1 + mu'^2 S0)/var - S0, mu' = mu - c, then the
 *   normalisation selected by flags.  Uses the prepared GMM in ws (runs a1 unless FV_PREPARED). */
fv_status fv_finalize(const double *stats, int batch, int D, const float *weights, const float *means,
                      const float *sigmas, int K, unsigned flags, float *out, void *ws, size_t ws_bytes,
                      fv_stream_t stream);

/* GMM training by EM on the GPU ("the GMM components trained beforehand",
 * P:141-142).  The E-step reuses the production path: exact posteriors (threshold 0) from the
 * GEMM1 + softmax kernel, sufficient statistics from GEMM2, plus each descriptor's log-likelihood.
 *
 * fv_gmm_estep: one descriptor set X (N x D) under the GMM (w, mu, sg) ->
 *   stats   (device, 1 + K(2D+1) doubles) = [N, S0 (K), S1 (K x D), S2 (K x D)] about c (as
 *           fv_stats_batched with threshold 0; they add across descriptor shards),
 *   loglik  (device, 1 double) = sum_i ln sum_j pi_j N(x_i; mu_j, diag var_j) (natural log, with the
 *           -(D/2) ln 2 pi constant; also additive across shards).
 * fv_gmm_mstep: stats (possibly summed over ranks) -> new parameters (device, fp32; variances
 *   whatever the sigma convention of the input), with SPEC train_gmm's floors:
 *     mu_j = c + S1_j/S0_j,  var_j = max(S2_j/S0_j - (S1_j/S0_j)^2, max(var_floor_abs, var_floor_rel * var_k(X))),
 *     pi_j = max(S0_j/N, prior_floor) / sum_l max(S0_l/N, prior_floor)
 *   where var_k(X) is the data's biased per-dimension variance (from the same statistics).  A component
 *   with S0_j == 0 keeps its mean and variance (reading A20).  The outputs may alias the inputs.
 *   Precision: the moment form about c turns the fp32 statistics' ~1e-7 relative error into an absolute
 *   variance error of ~1e-6 (|mu_j - c|^2 + var_j) (tests/test_gpu_em.py).
 *   Uses the prepared GMM (c) in ws: runs a1 unless FV_PREPARED.
 * fv_gmm_em_step: both on one device (stats kept in ws); loglik is the INPUT model's.
 * Floors must be finite and >= 0, prior_floor < 1 (else FV_ERR_ARG); EM needs N >= 1.
 * ws >= fv_workspace_bytes_em(N, K, D, flags). */
size_t fv_workspace_bytes_em(int64_t N, int K, int D, unsigned flags);
fv_status fv_gmm_estep(const float *X, int64_t N, int D, const float *weights, const float *means,
                       const float *sigmas, int K, unsigned flags, double *stats, double *loglik, void *ws,
                       size_t ws_bytes, fv_stream_t stream);
fv_status fv_gmm_mstep(const double *stats, int D, const float *weights, const float *means, const float *sigmas,
                       int K, unsigned flags, float var_floor_abs, float var_floor_rel, float prior_floor,
                       float *new_weights, float *new_means, float *new_vars, void *ws, size_t ws_bytes,
                       fv_stream_t stream);
fv_status fv_gmm_em_step(const float *X, int64_t N, int D, const float *weights, const float *means,
                         const float *sigmas, int K, unsigned flags, float var_floor_abs, float var_floor_rel,
                         float prior_floor, float *new_weights, float *new_means, float *new_vars, double *loglik,
                         void *ws, size_t ws_bytes, fv_stream_t stream);

/* PCA + normalised-xy embedding, the step upstream of the encoder ("by lowering
 * the dimension to m (m<128) with PCA and adding the normalized X and Y axis, a descriptor with
 * dimension M=m+2 is generated", §3.1; SPEC embed S:201-203; no whitening):
 *   X_out[i * ldx + c] = sum_k pca_basis[c * 128 + k] (raw[i * 128 + k] - pca_mean[k])   (c < m)
 *   X_out[i * ldx + m] = xy[2 i] / img_wh[2 b],  X_out[i * ldx + m + 1] = xy[2 i + 1] / img_wh[2 b + 1]
 *   X_out[i * ldx + c] = 0 for m + 2 <= c < ldx,
 * for descriptor i of image b (rows offsets[b] .. offsets[b+1]-1).  raw: device, n_total x 128 fp32
 * (16-byte aligned); xy: n_total x 2 keypoint pixel coordinates in the original image (16-byte
 * aligned); img_wh: batch x 2 (width, height; 8-byte aligned); pca_mean: 128 (16-byte aligned);
 * pca_basis: m x 128 row-major (rows orthonormal: not checked); 1 <= m <= 126; ldx >= m + 2,
 * ldx % 4 == 0.  Arithmetic (k_embed, tcgen05): d - mean in fp32, both operands split into tf32 hi + lo
 * (3 products, ~22 significant bits), fp32 tensor-core accumulation; |error| <= 1e-5 ||d - mean||.
 * Misaligned pointers: FV_ERR_UNSUPPORTED; asynchronous on `stream`, no allocation. */
fv_status fv_embed(const float *raw, const float *xy, const int64_t *offsets, int batch, int64_t n_total,
                   const float *img_wh, const float *pca_mean, const float *pca_basis, int m, float *X_out, int ldx,
                   fv_stream_t stream);

/* Raw descriptors to FVs in one call: fv_embed into the workspace (row stride round_up(m+2, 4)), then
 * the fv_encode_batched path with D = m + 2 (any D: the stride padding makes the rows TMA-aligned).
 * The GMM is K x (m + 2).  out: batch x 2K(m+2).  ws >= fv_workspace_bytes_embed(n_total, batch, K, m, flags). */
size_t fv_workspace_bytes_embed(int64_t n_total, int batch, int K, int m, unsigned flags);
fv_status fv_embed_encode_batched(const float *raw, const float *xy, const int64_t *offsets, int batch,
                                  int64_t n_total, const float *img_wh, const float *pca_mean,
                                  const float *pca_basis, int m, const float *weights, const float *means,
                                  const float *sigmas, int K, float threshold, unsigned flags, float *out,
                                  void *ws, size_t ws_bytes, fv_stream_t stream);

/* Test hook: posteriors gamma (N x K fp32) of one set, computed by the production kernel (same
 * GEMM + softmax path as fv_encode); entries <= threshold are zeroed when threshold > 0. */
fv_status fv_posteriors(const float *X, int64_t N, int D, const float *weights, const float *means,
                        const float *sigmas, int K, float threshold, unsigned flags, float *gamma,
                        void *ws, size_t ws_bytes, fv_stream_t stream);

/* Range report.  The contractions run on fp16 hi/lo split operands, so a descriptor with
 * |x_k - c_k| >= ~256 RMS_k in some dimension (c, RMS: the GMM-weighted mean and RMS of dimension k),
 * a component whose standard deviation in some dimension is below ~RMS_k/150, or non-finite input,
 * cannot be represented.  Such inputs are never turned into finite garbage: every row whose
 * log-likelihoods are not all finite gets NaN posteriors, so its image's statistics / FV / scores are
 * NaN, and the image is flagged.  After an fv_encode*, fv_stats_batched, fv_posteriors or E-step call
 * made with `ws`, this writes (stream-ordered, device int32 array of `batch` entries)
 *   flags_out[b] = bit 0: image b had a row with non-finite log-likelihoods;
 *                  bit 1: the prepared GMM has a coefficient outside the fp16 range (all images NaN).
 * n_total, batch, K, D are those of that call (they locate the flags in ws); 0 everywhere = in range. */
fv_status fv_range_flags(const void *ws, size_t ws_bytes, int64_t n_total, int batch, int K, int D,
                         int32_t *flags_out, fv_stream_t stream);

/* Profiling hook (bench accounting): when set, every k_stats launch made by this thread is bracketed
 * by cudaEventRecord(start/stop, stream) so the caller can time the dominant kernel alone with CUDA
 * events on the stream it runs on.  Pass NULL, NULL to disable.  (cudaEvent_t values.) */
void fv_profile_events(void *start_event, void *stop_event);

/* Debug hook: in libraries built with -DGPUFV_TRACE, CTA 0 of k_stats records per-tile phase clocks
 * (clock64) into dev_buf[64 x 16] (device memory, caller-owned); NULL disables.  No-op otherwise. */
void fv_debug_trace(long long *dev_buf);

/* Number of kernel launches the last successful call on this thread enqueued (for bench accounting). */
int fv_last_launch_count(void);

const char *fv_status_string(fv_status s);
const char *fv_last_error(void);
int fv_version(void); /* 100 * major + minor */

#ifdef __cplusplus
}
#endif
#endif /* GPUFV_H */
