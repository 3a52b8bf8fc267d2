/* examples/encode_c.c — the C ABI used from plain C (no PyTorch): one synthetic 5000-descriptor frame
 * encoded against a 256-component GMM with fv_encode, device memory from the CUDA runtime.
 *
 *   nvcc -o encode_c examples/encode_c.c -Iinclude -Lpaper_1604_03498_b200 -lgpufv \
 *        -Xlinker -rpath=$PWD/paper_1604_03498_b200 && ./encode_c [K D N]
 *
 * Prints the FV's L2 norm (1 for the improved FV), its first components and the status string; exits
 * non-zero on any error. */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "gpufv.h"

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "%s\n", cudaGetErrorString(e_)); return 2; } } while (0)

static double urand(unsigned long long *s) { /* xorshift64*: inputs only, no method arithmetic */
  *s ^= *s >> 12; *s ^= *s << 25; *s ^= *s >> 27;
  return (double)((*s * 2685821657736338717ULL) >> 11) / 9007199254740992.0;
}
static double nrand(unsigned long long *s) { return sqrt(-2.0 * log(urand(s) + 1e-300)) * cos(6.283185307179586 * urand(s)); }

int main(int argc, char **argv) {
  const int K = argc > 1 ? atoi(argv[1]) : 256, D = argc > 2 ? atoi(argv[2]) : 64;
  const long long N = argc > 3 ? atoll(argv[3]) : 5000;
  unsigned long long seed = 1604;
  float *w = malloc(K * sizeof(float)), *mu = malloc((size_t)K * D * sizeof(float)), *var = malloc((size_t)K * D * sizeof(float));
  float *X = malloc((size_t)N * D * sizeof(float)), *fv = malloc((size_t)2 * K * D * sizeof(float));
  double wsum = 0;
  for (int j = 0; j < K; ++j) { w[j] = (float)(0.5 + urand(&seed)); wsum += w[j]; }
  for (int j = 0; j < K; ++j) w[j] = (float)(w[j] / wsum);
  for (int j = 0; j < K; ++j)
    for (int k = 0; k < D; ++k) {
      const double s = 0.5 / sqrt(k + 1.0);
      mu[j * D + k] = (float)(s * 0.55 * nrand(&seed));
      var[j * D + k] = (float)(s * s * 0.7 * (0.5 + urand(&seed)));
    }
  for (long long i = 0; i < N; ++i) {
    const int j = (int)(urand(&seed) * K) % K;
    for (int k = 0; k < D; ++k) X[i * D + k] = (float)(mu[j * D + k] + sqrt(var[j * D + k]) * nrand(&seed));
  }
  float *dX, *dw, *dmu, *dvar, *dfv;
  void *ws_raw, *ws;
  const size_t wsb = fv_workspace_bytes(N, 1, K, D, 0);
  if (wsb == 0) { fprintf(stderr, "fv_workspace_bytes failed: %s\n", fv_last_error()); return 1; }
  CK(cudaMalloc((void **)&dX, (size_t)N * D * 4)); CK(cudaMalloc((void **)&dw, K * 4));
  CK(cudaMalloc((void **)&dmu, (size_t)K * D * 4)); CK(cudaMalloc((void **)&dvar, (size_t)K * D * 4));
  CK(cudaMalloc((void **)&dfv, (size_t)2 * K * D * 4)); CK(cudaMalloc(&ws_raw, wsb + 1024));
  ws = (void *)(((size_t)ws_raw + 1023) & ~(size_t)1023);  /* the workspace must be 1024-byte aligned */
  CK(cudaMemcpy(dX, X, (size_t)N * D * 4, cudaMemcpyHostToDevice)); CK(cudaMemcpy(dw, w, K * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dmu, mu, (size_t)K * D * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dvar, var, (size_t)K * D * 4, cudaMemcpyHostToDevice));
  fv_status st = fv_encode(dX, N, D, dw, dmu, dvar, K, 1e-6f, FV_NORM_IMPROVED, dfv, ws, wsb, NULL);
  if (st != FV_OK) { fprintf(stderr, "fv_encode: %s (%s)\n", fv_status_string(st), fv_last_error()); return 1; }
  CK(cudaMemcpy(fv, dfv, (size_t)2 * K * D * 4, cudaMemcpyDeviceToHost));
  double n2 = 0;
  for (int i = 0; i < 2 * K * D; ++i) n2 += (double)fv[i] * fv[i];
  printf("fv_encode: %s, %d launches, ||fv|| = %.6f, fv[0..3] = %.5f %.5f %.5f %.5f\n", fv_status_string(st),
         fv_last_launch_count(), sqrt(n2), fv[0], fv[1], fv[2], fv[3]);
  /* a synchronous argument error, reported without touching the device */
  st = fv_encode(dX, N, 6, dw, dmu, dvar, K, 0.f, 0, dfv, ws, wsb, NULL);
  printf("D=6: %s (%s)\n", fv_status_string(st), fv_last_error());
  cudaFree(dX); cudaFree(dw); cudaFree(dmu); cudaFree(dvar); cudaFree(dfv); cudaFree(ws_raw);
  free(w); free(mu); free(var); free(X); free(fv);
  return fabs(sqrt(n2) - 1.0) < 1e-4 && st == FV_ERR_UNSUPPORTED ? 0 : 1;
}
