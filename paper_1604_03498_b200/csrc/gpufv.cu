// gpufv.cu — host side of the C ABI declared in include/gpufv.h: argument validation, workspace
// layout, launches.  No allocation, no synchronisation (except fv_encode_batched_host, which must
// return host results), no CPU fallback: every step of the path runs in the kernels below.
// Experiment knobs (environment, read once per process; defaults are the measured best):
//   GPUFV_MIN_TILES=<n>   minimum tiles per cluster for small launches (default 2)
//   GPUFV_FIN_TILES=1     force the tile-parallel finalize for large batches (default: k_finalize_img)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdarg>
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "../../include/gpufv.h"
#include "fv_common.cuh"
#include "k_aux.cuh"
#include "k_stats.cuh"
#include "k_stats_w.cuh"
#include "k_stats_sp.cuh"
#include "k_embed.cuh"

using namespace gpufv;

namespace {

// NVTX ranges around every C-ABI entry point and each host-pipeline chunk (header-only NVTX v3: a
// no-op unless a profiler such as nsys / ncu --nvtx is attached)
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};

thread_local std::string g_err;
thread_local int g_launches = 0;
thread_local cudaEvent_t g_prof_start = nullptr, g_prof_stop = nullptr;
thread_local long long *g_trace = nullptr;

fv_status fail(fv_status s, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

fv_status cuda_check(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FV_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return FV_OK;
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

int sm_count() {
  static int cache[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (!cache[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

// Tile family: D <= 64 -> k_stats (128 Gaussians per CTA, cluster <= 4); 64 < D <= 128 -> k_stats_w
// (64 Gaussians per CTA, cluster <= 8).  K <= 512 for both.
constexpr int kMinTilesPerClusterDefault = 2;
constexpr int kMaxSegPerImage = 26;
constexpr int kMaxSegPerImageNarrow = 80;  // >= every cluster of a narrow launch: no cap
// GPUFV_MIN_TILES overrides it (latency experiments only); read once per process
int min_tiles_env() {
  static const int v = [] {
    const char *e = std::getenv("GPUFV_MIN_TILES");
    const int x = e ? std::atoi(e) : 0;
    return x > 0 ? x : 0;
  }();
  return v;
}
int min_tiles_per_cluster() { return min_tiles_env() > 0 ? min_tiles_env() : kMinTilesPerClusterDefault; }
// The single-frame finalize runs inside k_stats (fin_lat_fused) where it pays (fin_fused_wanted);
// GPUFV_FIN_FUSED=0 never (A/B runs), =2 whenever the kernel can (tests: more blocks than CTAs)
int fin_fused_mode() {
  static const int v = [] { const char *e = std::getenv("GPUFV_FIN_FUSED"); return e ? std::atoi(e) : 1; }();
  return v;
}
bool lat_finalize_fits(int K, int D, int batch);
bool fin_fused_wanted(int K, int D, int n_cls, int C, int64_t ncl, int64_t tiles, int64_t ncl_max);
bool is_wide(int K, int D) { return D > kDP || K > kG * kMaxC2; }
// Wide family with D <= 96 (the paper's 82-dim format): the second feature half packed into 64
// features (k_stats_w<.., kPk>, W' by k_prep_w with wide == 2); GPUFV_WIDE_PACK=0 for A/B runs
bool wide_packed(int K, int D) {
  static const bool env = [] { const char *e = std::getenv("GPUFV_WIDE_PACK"); return !(e && e[0] == '0'); }();
  return env && is_wide(K, D) && D <= 96;
}
int gauss_per_cta(int K, int D) { return is_wide(K, D) ? kGW : kG; }
int cluster_size(int K, int D) { return (K + gauss_per_cta(K, D) - 1) / gauss_per_cta(K, D); }
// Fused finalize for a single narrow frame (auto mode) only when the frame has one tile per cluster and
// every one of the finalize's (K/32) x (D/8) blocks gets a CTA of its own.  Measured (same box, p50):
// 5,000 descriptors 27.0 vs 30.1-32 us (the separate k_finalize_lat), 8,000: 29.1 vs 30.1-31; with
// fewer CTAs than blocks each CTA finalizes several in turn (1,000 descriptors: 37 vs 31 us), and with
// more tiles than clusters the extra segments cost more than the saved launch (two tiles per cluster,
// forced: 10,000 31.1 vs 31.2 us, 17,714 35.2 vs 34.2, 40,000 45.6 vs 45.0).
bool fin_fused_wanted(int K, int D, int n_cls, int C, int64_t ncl, int64_t tiles, int64_t ncl_max) {
  const int mode = fin_fused_mode();
  if (mode == 0 || is_wide(K, D) || n_cls > kMaxCls || !lat_finalize_fits(K, D, 1)) return false;
  if (mode >= 2) return true;
  const int nv = ((K + kLatJ - 1) / kLatJ) * ((D + kLatK - 1) / kLatK);
  return tiles <= ncl_max && ncl == tiles && (int64_t)C * ncl >= nv;
}

// Persistent grid: the number of co-resident clusters of the stats kernel on the current device.
int num_clusters(int C, bool wide) {
  static std::mutex mu;
  static int cache[64][2][kMaxCW + 1] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return -1;
  std::lock_guard<std::mutex> lk(mu);
  if (cache[dev][wide][C] > 0) return cache[dev][wide][C];
  const int smem = wide ? kSmemWBytes : kSmem2Bytes;
  if (cudaFuncSetAttribute(k_stats<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem2Bytes) != cudaSuccess ||
      cudaFuncSetAttribute(k_stats<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem2Bytes) != cudaSuccess ||
      cudaFuncSetAttribute(k_stats<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem2Bytes) != cudaSuccess ||
      cudaFuncSetAttribute(k_stats<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem2Bytes) != cudaSuccess ||
      cudaFuncSetAttribute(k_stats<true, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem2Bytes) != cudaSuccess ||
      cudaFuncSetAttribute(k_stats<false, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem2Bytes) != cudaSuccess ||
      cudaFuncSetAttribute(k_stats<true, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem2Bytes) != cudaSuccess ||
      cudaFuncSetAttribute(k_stats<false, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem2Bytes) != cudaSuccess ||
      cudaFuncSetAttribute(k_stats_w<true, 0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemWBytes) != cudaSuccess ||
      cudaFuncSetAttribute(k_stats_w<true, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemWBytes) != cudaSuccess ||
      cudaFuncSetAttribute(k_stats_w<true, 4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemWBytes) != cudaSuccess ||
      cudaFuncSetAttribute(k_stats_w<true, 4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemWBytes) != cudaSuccess ||
      cudaFuncSetAttribute(k_stats_w<true, 8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemWBytes) != cudaSuccess ||
      cudaFuncSetAttribute(k_stats_w<true, 8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemWBytes) != cudaSuccess ||
      cudaFuncSetAttribute(k_stats_w<false, 0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemWBytes) != cudaSuccess ||
      cudaFuncSetAttribute(k_stats_w<false, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemWBytes) != cudaSuccess ||
      cudaFuncSetAttribute(k_stats_w<false, 4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemWBytes) != cudaSuccess ||
      cudaFuncSetAttribute(k_stats_w<false, 4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemWBytes) != cudaSuccess ||
      cudaFuncSetAttribute(k_stats_w<false, 8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemWBytes) != cudaSuccess ||
      cudaFuncSetAttribute(k_stats_w<false, 8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemWBytes) != cudaSuccess ||
      cudaFuncSetAttribute(k_stats_w<false, 0, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemWBytes) != cudaSuccess ||
      cudaFuncSetAttribute(k_stats_w<false, 0, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemWBytes) != cudaSuccess ||
      cudaFuncSetAttribute(k_stats_w<false, 4, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemWBytes) != cudaSuccess ||
      cudaFuncSetAttribute(k_stats_w<false, 4, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemWBytes) != cudaSuccess ||
      cudaFuncSetAttribute(k_stats_w<false, 8, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemWBytes) != cudaSuccess ||
      cudaFuncSetAttribute(k_stats_w<false, 8, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemWBytes) != cudaSuccess ||
      cudaFuncSetAttribute(k_stats_sp<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemSpBytes) != cudaSuccess ||
      cudaFuncSetAttribute(k_stats_sp<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemSpBytes) != cudaSuccess)
    return -1;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(C * 148, 1, 1);
  cfg.blockDim = dim3(kThreads2, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  const cudaError_t e = wide ? cudaOccupancyMaxActiveClusters(&n, k_stats_w<true, 0, false>, &cfg)
                             : cudaOccupancyMaxActiveClusters(&n, k_stats<true, 2>, &cfg);
  if (e != cudaSuccess || n <= 0) {
    cudaGetLastError();
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    n = sms / C;
  }
  cache[dev][wide][C] = n;
  return n;
}

struct Layout {
  int C, Kp, ncl, dpad;  // cluster size, padded K, clusters, padded D (64 | 128)
  int64_t n_total, nslots;                                         // segment slots (cluster, image)
  size_t wimg, bias, xshift, xscale, cshift, bscratch, bmax, pscale, xinv, coef;  // prepared GMM (head of ws)
  size_t gflag;                                           // GMM range flag (prepared head, after bmax)
  size_t tiles, off1, cstart, cown, norm2, rflags, s0slots, slots;  // per call
  size_t spart;                                           // fused scoring partial dots (n_cls > 0)
  size_t llrows, llparts, emstats;                        // EM: per-row log2-likelihoods, reduction, stats
  size_t emb;                                             // embedded descriptors (n_total x ldx), NEXT-2
  size_t rflagc;                                          // per-CTA range words (fused single-frame schedule)
  size_t hx, hoff, hout;                                  // _host entry point
  size_t total;
};

bool make_layout(int64_t n_total, int batch, int K, int D, bool host_io, Layout &L, int n_cls = 0, bool em = false,
                 int emb_ld = 0) {
  L.C = cluster_size(K, D);
  L.Kp = L.C * gauss_per_cta(K, D);
  L.dpad = is_wide(K, D) ? kDMax : kDP;
  L.ncl = num_clusters(L.C, is_wide(K, D));
  if (L.ncl <= 0) return false;
  // small launches (one frame): at least min_tiles_per_cluster() tiles per cluster, so an image is split
  // into fewer (cluster) segments for the finalize to combine; tiles <= n_total/128 + batch
  // (a single set: exactly its tile count)
  const int64_t tmax = batch == 1 ? (n_total + kTileM - 1) / kTileM : n_total / kTileM + batch;
  int mt = min_tiles_per_cluster();
  // A single frame whose finalize runs inside k_stats: one tile per cluster — the finalize's (K/32) x
  // (D/8) blocks then land on distinct SMs and each cluster leaves one segment per tile (fin_fused_wanted)
  if (batch == 1 && min_tiles_env() == 0 && fin_fused_mode() == 1 &&
      fin_fused_wanted(K, D, n_cls, L.C, std::min<int64_t>(L.ncl, tmax), tmax, L.ncl))
    mt = 1;
  if (tmax > 0) L.ncl = (int)std::min<int64_t>(L.ncl, std::max<int64_t>(1, (tmax + mt - 1) / mt));
  // ... and at most ~kMaxSegPerImage segments per image on average: the tile-parallel finalize of one
  // image costs ~1 us per extra segment (measured: one 40,000-descriptor image 157 us over 74 clusters,
  // 92 us over 26), so a single large image uses fewer, longer cluster ranges (only for small images —
  // up to 32 tiles per cluster at the cap; a large single set such as an EM pass or a descriptor shard
  // needs every cluster).  The narrow family's one-round latency finalize reads up to 40 segments per
  // load round, so there the cap is lifted (round 2: 17,714 descriptors 42.3 -> 34.1 us, 40,000 64.7 ->
  // 45.5 us).  A function of (n_total, batch, K, D) only, so every workspace query agrees.
  const int seg_cap = is_wide(K, D) ? kMaxSegPerImage : kMaxSegPerImageNarrow;
  if (batch > 0 && tmax <= (int64_t)seg_cap * 32 * batch)
    L.ncl = (int)std::min<int64_t>(L.ncl, (int64_t)seg_cap * batch);
  // one slot per (cluster, image) segment, index cid + b (seg_slot, fv_common.cuh)
  L.n_total = n_total;
  L.nslots = (int64_t)L.ncl + batch + 1;
  size_t o = 0;
  L.wimg = o;     o = align_up(o + (size_t)L.C * kWImgBytes, 1024);
  L.bias = o;     o = align_up(o + (size_t)L.Kp * 4, 256);
  L.xshift = o;   o = align_up(o + kDMax * 4, 256);
  L.xscale = o;   o = align_up(o + kDMax * 4, 256);
  L.cshift = o;   o = align_up(o + kDMax * 8, 256);
  L.bscratch = o; o = align_up(o + (size_t)L.Kp * 8, 256);
  L.bmax = o;     o = align_up(o + 16, 256);
  L.gflag = L.bmax + 8;
  L.pscale = o;   o = align_up(o + (size_t)2 * L.Kp * 8, 256);
  L.xinv = o;     o = align_up(o + kDMax * 8, 1024);
  L.coef = o;     o = align_up(o + (size_t)3 * kDMax * L.Kp * 8, 1024);
  L.tiles = o;    o = align_up(o + (size_t)(batch + 1) * 8, 256);
  L.off1 = o;     o = align_up(o + 16, 256);
  L.cstart = o;   o = align_up(o + (size_t)(L.ncl + 1) * 4, 256);
  L.cown = o;     o = align_up(o + (size_t)(batch > 0 ? batch : 1) * 8, 256);
  L.norm2 = o;    o = align_up(o + (size_t)(batch > 0 ? batch : 1) * (kFinMaxParts * 8 + 4), 1024);  // norm parts + tickets
  L.rflags = o;   o = align_up(o + (size_t)(batch > 0 ? batch : 1) * 4, 256);
  L.rflagc = o;   o = align_up(o + (size_t)L.ncl * L.C * 4, 256);
  L.s0slots = o;  o = align_up(o + (size_t)(L.ncl + batch) * 4 * L.Kp * 4, 1024);
  L.slots = o;    o = align_up(o + (size_t)L.nslots * 2 * L.dpad * L.Kp * 4, 1024);
  L.spart = o;    o = align_up(o + (size_t)(n_cls > 0 ? batch : 0) * kFinMaxParts * n_cls * 8, 1024);
  L.llrows = L.llparts = L.emstats = o;
  if (em) {
    L.llrows = o;  o = align_up(o + (size_t)n_total * 4, 1024);
    L.llparts = o; o = align_up(o + (size_t)kLLBlocks * 8 + 8, 1024);  // block slots + ticket
    L.emstats = o; o = align_up(o + ((size_t)1 + (size_t)K * (2 * D + 1)) * 8, 1024);
  }
  L.emb = o;
  if (emb_ld > 0) o = align_up(o + (size_t)n_total * emb_ld * 4, 1024);
  L.hx = L.hoff = L.hout = 0;
  if (host_io) {
    // device staging of X, offsets and the per-image result (scores when n_cls > 0, else FVs)
    L.hx = o;   o = align_up(o + (size_t)n_total * D * 4, 1024);
    L.hoff = o; o = align_up(o + (size_t)(batch + 1) * 8, 256);
    L.hout = o; o = align_up(o + (size_t)batch * (n_cls > 0 ? n_cls : 2 * K * D) * 4, 1024);
  }
  L.total = o;
  return true;
}

fv_status check_gmm_args(int K, int D, const float *w, const float *mu, const float *sg, unsigned flags,
                         bool need_d4 = true) {
  if (!w || !mu || !sg) return fail(FV_ERR_ARG, "null GMM pointer");
  if (K < 1 || D < 1) return fail(FV_ERR_ARG, "K=%d and D=%d must be >= 1", K, D);
  if (K > kMaxK) return fail(FV_ERR_UNSUPPORTED, "K=%d > %d", K, kMaxK);
  if (D > kDMax) return fail(FV_ERR_UNSUPPORTED, "D=%d > %d", D, kDMax);
  if (need_d4 && D % 4 != 0) return fail(FV_ERR_UNSUPPORTED, "D=%d is not a multiple of 4 (pad, reading A13)", D);
  const unsigned known = FV_NORM_MASK | FV_SIGMA_IS_STDDEV | FV_PREPARED | FV_SPARSE_STATS;
  if (flags & ~known) return fail(FV_ERR_ARG, "unknown flag bits 0x%x", flags & ~known);
  if ((flags & FV_NORM_MASK) == 3) return fail(FV_ERR_ARG, "invalid normalisation mode 3");
  return FV_OK;
}

fv_status check_device() {
  static int ok_dev[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return fail(FV_ERR_CUDA, "no CUDA device"); }
  if (dev >= 0 && dev < 64 && ok_dev[dev]) return FV_OK;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) { cudaGetLastError(); return fail(FV_ERR_CUDA, "cudaGetDeviceProperties failed"); }
  if (prop.major != 10 || prop.minor != 0)
    return fail(FV_ERR_UNSUPPORTED, "device %s is sm_%d%d; this library is built for sm_100a only", prop.name, prop.major, prop.minor);
  // Every kernel of a call prefers the maximum shared-memory carveout — the one the stats kernels
  // need (227 KB per CTA).  With the default carveout an SM that last ran a small-SMEM kernel (the
  // finalize, the schedule) must drain and reconfigure its L1 / shared split before it can take a
  // stats CTA: measured ~6 us between k_schedule's entry and the first k_stats CTA of a single frame.
  {
    const int c = cudaSharedmemCarveoutMaxShared;
    const void *fns[] = {(const void *)k_schedule, (const void *)k_finalize_lat, (const void *)k_finalize<false, false>,
                         (const void *)k_finalize<false, true>, (const void *)k_finalize<true, false>,
                         (const void *)k_finalize<true, true>, (const void *)k_finalize_img<false>,
                         (const void *)k_finalize_img<true>, (const void *)k_reduce_stats, (const void *)k_prep_shift,
                         (const void *)k_prep_bias, (const void *)k_prep_bias_final, (const void *)k_prep_w,
                         (const void *)k_range_flags, (const void *)k_loglik_reduce, (const void *)k_mstep};
    for (const void *f : fns)
      if (cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, c) != cudaSuccess)
        return cuda_check("carveout attribute");
  }
  if (dev >= 0 && dev < 64) ok_dev[dev] = 1;
  return FV_OK;
}

fv_status check_ws(void *ws, size_t ws_bytes, const Layout &L) {
  if (!ws) return fail(FV_ERR_ARG, "null workspace");
  if (reinterpret_cast<uintptr_t>(ws) % 1024) return fail(FV_ERR_WORKSPACE, "workspace must be 1024-byte aligned");
  if (ws_bytes < L.total) return fail(FV_ERR_WORKSPACE, "workspace too small: %zu < %zu bytes", ws_bytes, L.total);
  return FV_OK;
}

uint8_t *at(void *ws, size_t off) { return static_cast<uint8_t *>(ws) + off; }

fv_status launch_prep(const Layout &L, const float *w, const float *mu, const float *sg, int K, int D, unsigned flags,
                      void *ws, cudaStream_t st) {
  const int sd = (flags & FV_SIGMA_IS_STDDEV) ? 1 : 0;
  k_prep_shift<<<1, kPrepThreads, 0, st>>>(w, mu, sg, K, D, L.Kp, sd, (double *)at(ws, L.cshift), (float *)at(ws, L.xshift),
                                  (float *)at(ws, L.xscale), (double *)at(ws, L.pscale), (double *)at(ws, L.xinv),
                                  (int *)at(ws, L.gflag));
  k_prep_bias<<<K, kDMax, 0, st>>>(w, mu, sg, D, sd, (const double *)at(ws, L.cshift), (double *)at(ws, L.bscratch));
  k_prep_bias_final<<<1, 512, 0, st>>>(K, L.Kp, (const double *)at(ws, L.bscratch), (float *)at(ws, L.bias),
                                       (double *)at(ws, L.bmax));
  k_prep_w<<<L.Kp, 2 * L.dpad, 0, st>>>(mu, sg, K, D, sd, (const double *)at(ws, L.cshift), (const float *)at(ws, L.xscale),
                                 at(ws, L.wimg), (double *)at(ws, L.coef), wide_packed(K, D) ? 2 : is_wide(K, D) ? 1 : 0,
                                 (int *)at(ws, L.gflag));
  g_launches += 4;
  return cuda_check("k_prep");
}

// a2-a6 over a batch: schedule + persistent stats kernel.  gamma (optional) for fv_posteriors.
fv_status launch_stats(const Layout &L, const float *X, const int64_t *&offsets, int64_t n_single, int batch, int D,
                       int K, float thr, void *ws, float *gamma, int gamma_mode, cudaStream_t st,
                       float *loglik_rows = nullptr, int ldx = 0, int rf_base = 0, int64_t rows = -1,
                       bool sparse_req = false, bool fuse = false, const FinParams *fin = nullptr) {
  if (ldx <= 0) ldx = D;
  int *rflags = (int *)at(ws, L.rflags) + rf_base;
  // offsets == nullptr: a single set of n_single rows; k_schedule materialises {0, n_single} in ws.
  int64_t *off1 = (int64_t *)at(ws, L.off1);
  unsigned *counters = (unsigned *)((double *)at(ws, L.norm2) + (size_t)(batch > 0 ? batch : 1) * kFinMaxParts);
  // fuse (a single frame whose finalize is k_finalize_lat): no k_schedule — k_stats writes the tables
  if (!fuse) {
    k_schedule<<<1, 1024, 0, st>>>(offsets, off1, n_single, batch, (int64_t *)at(ws, L.tiles), L.ncl,
                                   (int *)at(ws, L.cstart), (int *)at(ws, L.cown), counters, rflags, g_trace);
    g_launches += 1;
  }
  Stats2Params p;
  p.sched_counters = counters;
  // one set whose rows are known here: no offsets (fv_encode, the E-step), or one image of a full call
  // (offsets = {0, n_total} by the header contract; host-pipeline chunks pass rows >= 0 and keep the table)
  p.single_rows = (!offsets || (batch == 1 && rows < 0)) ? n_single : -1;
  if (!offsets) offsets = off1;
  p.X = X;
  p.offsets = offsets;
  p.tile_start = (const int64_t *)at(ws, L.tiles);
  p.wimg = at(ws, L.wimg);
  p.bias = (const float *)at(ws, L.bias);
  p.xshift = (const float *)at(ws, L.xshift);
  p.xscale = (const float *)at(ws, L.xscale);
  p.slots = (float *)at(ws, L.slots);
  p.s0slots = (float *)at(ws, L.s0slots);
  p.gamma_out = gamma;
  p.loglik_out = loglik_rows;
  p.trace = g_trace;
  p.rflags = fuse ? (int *)at(ws, L.rflagc) : rflags;  // fused: one range word per CTA (see Stats2Params)
  p.rflag_cta = fuse ? 1 : 0;
  if (rows < 0) rows = n_single;  // rows of this launch's images (n_total unless a host-pipeline chunk)
  p.kfold = (batch > 0 && rows / batch >= kLongSetRows) ? kFoldLong
            : (kFoldShort > 0 && batch > 0 && rows / batch <= kShortSetRows) ? kFoldShort : kFold;
  p.batch = batch;
  p.D = D;
  p.K = K;
  p.Kp = L.Kp;
  p.ldx = ldx;
  p.threshold = thr > 0.f ? thr : 0.f;
  p.gamma_mode = gamma_mode;
  // FV_SPARSE_STATS with tau > 0 on the narrow family: the survivor (Alg. 5) path instead of the dense
  // GEMM2 (measured 1.8x slower on C4: opt-in); per-row outputs need the dense kernel
  const bool sparse = sparse_req && !is_wide(K, D) && p.threshold > 0.f && !gamma && !loglik_rows;
  // X as a 2-D tensor map: dims {D, n_total}, boxes of 32 floats x 128 rows, 128B swizzle; rows past
  // n_total and dims past D read as zero.
  CUtensorMap tmap;
  {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
      cudaDriverEntryPointQueryResult q;
      void *fn = nullptr;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
        return fail(FV_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
      encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)(L.n_total > 0 ? L.n_total : 1)};
    cuuint64_t strides[1] = {(cuuint64_t)ldx * 4};
    // the survivor kernel takes one unswizzled box of kSpXLd floats x 128 rows per tile, the dense
    // kernels two 128B-swizzled boxes of 32 floats
    cuuint32_t box[2] = {sparse ? (cuuint32_t)kSpXLd : 32u, 128};
    cuuint32_t estr[2] = {1, 1};
    // an empty launch (n_total == 0, X typically NULL) loads no tile, but the map still needs a valid
    // global address: point it at the workspace
    float *xmap = (X && L.n_total > 0) ? const_cast<float *>(X) : reinterpret_cast<float *>(ws);
    CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, xmap, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, sparse ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(FV_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = L.C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // prologue overlaps k_schedule
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  // Fused finalize: its grid barriers need every CTA resident.  The grid is at most the occupancy
  // query's cluster count (one wave on an idle GPU — the assumption k_finalize_lat's and k_finalize<..,
  // true>'s sibling waits already make).  GPUFV_COOP=1 adds the cooperative-launch attribute, which
  // turns a grid that cannot be co-resident into a launch error; it is opt-in because Nsight Compute
  // cannot profile a cooperative cluster launch (the process dies under ncu).
  static const bool coop_env = [] { const char *e = std::getenv("GPUFV_COOP"); return e && e[0] == '1'; }();
  if (fin && coop_env) {
    attr[1].id = cudaLaunchAttributeCooperative;
    attr[1].val.cooperative = 1;  // (fin implies fuse: no programmatic serialization)
  }
  const FinParams fin_none{};
  const FinParams &fp = fin ? *fin : fin_none;
  cfg.gridDim = dim3(L.C * L.ncl, 1, 1);
  cfg.blockDim = dim3(kThreads2, 1, 1);
  cfg.dynamicSmemBytes = is_wide(K, D) ? kSmemWBytes : sparse ? kSmemSpBytes : kSmem2Bytes;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = (fuse && !(fin && coop_env)) ? 1 : 2;  // the first kernel of a fused call waits for the stream normally
  if (g_prof_start) cudaEventRecord(g_prof_start, st);
  cudaError_t e;
  if (sparse) e = (D == kDP) ? cudaLaunchKernelEx(&cfg, k_stats_sp<true>, tmap, p) : cudaLaunchKernelEx(&cfg, k_stats_sp<false>, tmap, p);
  else if (!is_wide(K, D)) {
    using KN = void (*)(const CUtensorMap, const Stats2Params, const FinParams);
    const KN kn[2][2][2] = {{{k_stats<false, 1>, k_stats<false, 1, true>}, {k_stats<false, 2>, k_stats<false, 2, true>}},
                            {{k_stats<true, 1>, k_stats<true, 1, true>}, {k_stats<true, 2>, k_stats<true, 2, true>}}};
    e = cudaLaunchKernelEx(&cfg, kn[D == kDP][L.C == 2][fin != nullptr], tmap, p, fp);
  }
  else {
    // instantiations: full-D fast path x cluster size (4, 8, runtime) x per-row hooks
    using KW = void (*)(const CUtensorMap, const Stats2Params);
    const KW kw[2][3][2] = {
        {{k_stats_w<false, 0, false>, k_stats_w<false, 0, true>}, {k_stats_w<false, 4, false>, k_stats_w<false, 4, true>},
         {k_stats_w<false, 8, false>, k_stats_w<false, 8, true>}},
        {{k_stats_w<true, 0, false>, k_stats_w<true, 0, true>}, {k_stats_w<true, 4, false>, k_stats_w<true, 4, true>},
         {k_stats_w<true, 8, false>, k_stats_w<true, 8, true>}}};
    const KW kwp[3][2] = {{k_stats_w<false, 0, false, true>, k_stats_w<false, 0, true, true>},
                          {k_stats_w<false, 4, false, true>, k_stats_w<false, 4, true, true>},
                          {k_stats_w<false, 8, false, true>, k_stats_w<false, 8, true, true>}};
    const bool hooks = gamma != nullptr || loglik_rows != nullptr;
    const int ci = L.C == 8 ? 2 : L.C == 4 ? 1 : 0;
    e = wide_packed(K, D) ? cudaLaunchKernelEx(&cfg, kwp[ci][hooks], tmap, p)
                          : cudaLaunchKernelEx(&cfg, kw[D == kDMax][ci][hooks], tmap, p);
  }
  if (g_prof_stop) cudaEventRecord(g_prof_stop, st);
  g_launches += 1;
  if (e != cudaSuccess) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, k_stats<true, 2>);
    cudaGetLastError();
    return fail(FV_ERR_CUDA,
                "k_stats launch: %s (grid %d x %d threads, cluster %d, dyn smem %d; kernel: %d regs, max threads %d, "
                "local %zu B, static smem %zu B, max dyn smem %d)",
                cudaGetErrorString(e), L.C * L.ncl, kThreads2, L.C, (int)cfg.dynamicSmemBytes, fa.numRegs, fa.maxThreadsPerBlock,
                fa.localSizeBytes, fa.sharedSizeBytes, fa.maxDynamicSharedSizeBytes);
  }
  return cuda_check("k_stats");
}

FinParams fin_params(const Layout &L, const int64_t *offsets, int batch, int K, int D, const float *w, const float *mu,
                     const float *sg, unsigned flags, void *ws) {
  (void)mu; (void)sg;
  FinParams f;
  f.trace = g_trace;
  f.slots = (const float *)at(ws, L.slots);
  f.s0slots = (const float *)at(ws, L.s0slots);
  f.stats = nullptr;
  f.offsets = offsets;
  f.tile_start = (const int64_t *)at(ws, L.tiles);
  f.cstart = (const int *)at(ws, L.cstart);
  f.cown = (const int *)at(ws, L.cown);
  f.w = w;
  f.coef = (const double *)at(ws, L.coef);
  f.xscale = (const float *)at(ws, L.xscale);
  f.pscale = (const double *)at(ws, L.pscale);
  f.xinv = (const double *)at(ws, L.xinv);
  f.out = nullptr;
  f.stats_out = nullptr;
  f.norm2 = (double *)at(ws, L.norm2);
  f.counters = (unsigned *)(f.norm2 + (size_t)(batch > 0 ? batch : 1) * kFinMaxParts);
  f.b_base = 0;
  f.svm_w = nullptr; f.svm_b = nullptr; f.scores = nullptr; f.n_cls = 0;
  f.spart = (double *)at(ws, L.spart);
  f.rflag_cta = nullptr; f.nflag = 0; f.rflags = nullptr; f.fused_n = -1;
  f.gbar = (unsigned *)((char *)at(ws, L.gflag) + 8);  // gflag + 2 and + 34 (zeroed by k_prep_shift)
  f.batch = batch; f.K = K; f.Kp = L.Kp; f.D = D; f.ncl = L.ncl;
  f.mode = (int)(flags & FV_NORM_MASK);
  f.dpad = L.dpad;
  return f;
}

// The latency finalize (k_finalize_lat) takes a launch: one wave of (K/32) x batch x (D/8) blocks.
bool lat_finalize_fits(int K, int D, int batch) {
  const int lat_x = (K + kLatJ - 1) / kLatJ, lat_z = (D + kLatK - 1) / kLatK;
  return K <= kImgK && D <= kDP && (int64_t)lat_x * batch * lat_z <= sm_count() && lat_x * lat_z <= kFinMaxParts;
}

// after_stats: launched right behind k_stats (whose k_schedule zeroed the counters): programmatic
// launch, no memset node in between.  Otherwise (fv_finalize from statistics) the counters are zeroed here.
fv_status launch_finalize(const FinParams &f, int batch, int K, int D, cudaStream_t st, bool after_stats = true) {
  if (batch == 0) return FV_OK;
  // large batches of narrow images: one persistent block per SM takes whole images (k_finalize_img)
  static const bool force_tiles = std::getenv("GPUFV_FIN_TILES") != nullptr;
  if (D <= kDP && K <= kImgK && batch >= 2 * sm_count() && !force_tiles) {
    static std::mutex mu;
    static bool attr_done[64] = {};  // the attribute is per device
    int dev = 0;
    cudaGetDevice(&dev);
    {
      std::lock_guard<std::mutex> lk(mu);
      if (dev < 0 || dev >= 64 || !attr_done[dev]) {
        if (cudaFuncSetAttribute(k_finalize_img<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kImgSmemBytes) !=
                cudaSuccess ||
            cudaFuncSetAttribute(k_finalize_img<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kImgSmemBytes) !=
                cudaSuccess)
          return cuda_check("k_finalize_img attribute");
        if (dev >= 0 && dev < 64) attr_done[dev] = true;
      }
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = after_stats ? 1 : 0;
    cfg.gridDim = dim3(std::min(batch, sm_count()), 1, 1);
    cfg.blockDim = dim3(kImgThreads, 1, 1);
    cfg.dynamicSmemBytes = kImgSmemBytes;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    FinParams fc = f;
    fc.b_base = 0;
    const cudaError_t e = f.n_cls > 0 ? cudaLaunchKernelEx(&cfg, k_finalize_img<true>, fc)
                                      : cudaLaunchKernelEx(&cfg, k_finalize_img<false>, fc);
    if (e != cudaSuccess) return fail(FV_ERR_CUDA, "k_finalize_img launch: %s", cudaGetErrorString(e));
    g_launches += 1;
    return cuda_check("k_finalize_img");
  }
  // a handful of narrow images straight after k_stats: 4x the blocks (k_finalize_lat)
  const int lat_x = (K + kLatJ - 1) / kLatJ, lat_z = (D + kLatK - 1) / kLatK;
  if (after_stats && f.slots && f.n_cls == 0 && lat_finalize_fits(K, D, batch)) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = dim3(lat_x, batch, lat_z);
    cfg.blockDim = dim3(kLatThreads, 1, 1);
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    FinParams fc = f;
    fc.b_base = 0;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, k_finalize_lat, fc);
    if (e != cudaSuccess) return fail(FV_ERR_CUDA, "k_finalize_lat launch: %s", cudaGetErrorString(e));
    g_launches += 1;
    return cuda_check("k_finalize_lat");
  }
  if (!after_stats && cudaMemsetAsync(f.counters, 0, (size_t)batch * 4, st) != cudaSuccess)
    return cuda_check("memset tickets");
  for (int b0 = 0; b0 < batch; b0 += 65535) {  // gridDim.y limit
    FinParams fc = f;
    fc.b_base = b0;
    const dim3 grid((K + kFinJ - 1) / kFinJ, std::min(65535, batch - b0), (D + kDP - 1) / kDP);
    // one wave (every block resident at once: <= 1 block per SM): blocks wait for their image's
    // siblings and write once (latency path); otherwise the last block of each image rescales it
    const bool sync = (int64_t)grid.x * grid.y * grid.z <= (int64_t)sm_count();
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = (after_stats && b0 == 0) ? 1 : 0;
    cfg.gridDim = grid;
    cfg.blockDim = dim3(256, 1, 1);
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e;
    if (f.n_cls > 0) e = sync ? cudaLaunchKernelEx(&cfg, k_finalize<true, true>, fc) : cudaLaunchKernelEx(&cfg, k_finalize<true, false>, fc);
    else e = sync ? cudaLaunchKernelEx(&cfg, k_finalize<false, true>, fc) : cudaLaunchKernelEx(&cfg, k_finalize<false, false>, fc);
    if (e != cudaSuccess) return fail(FV_ERR_CUDA, "k_finalize launch: %s", cudaGetErrorString(e));
    g_launches += 1;
  }
  return cuda_check("k_finalize");
}

// Fused linear scoring arguments (NEXT-4); n_cls == 0: plain encode.
struct Scoring {
  const float *w = nullptr, *b = nullptr;
  int n_cls = 0;
  float *scores = nullptr;
};

fv_status encode_batched_impl(const float *X, const int64_t *offsets, int batch, int64_t n_total, int D,
                              const float *w, const float *mu, const float *sg, int K, float thr, unsigned flags,
                              float *out, void *ws, size_t ws_bytes, cudaStream_t st, const Layout *Lin,
                              const Scoring &sc = Scoring(), int ldx = 0, int rf_base = 0, int64_t rows = -1) {
  const bool sparse = (flags & FV_SPARSE_STATS) != 0;
  Layout L;
  if (Lin) L = *Lin;
  else if (!make_layout(n_total, batch, K, D, false, L, sc.n_cls)) return fail(FV_ERR_CUDA, "occupancy query failed");
  if (fv_status s = check_ws(ws, ws_bytes, L)) return s;
  if (!(flags & FV_PREPARED))
    if (fv_status s = launch_prep(L, w, mu, sg, K, D, flags, ws, st)) return s;
  if (batch == 0) return FV_OK;
  // One frame whose finalize is k_finalize_lat: k_stats writes the schedule tables itself (no k_schedule
  // launch on the latency path; GPUFV_FUSED_SCHED=0 keeps the separate kernel, for A/B runs)
  static const bool fuse_env = [] { const char *e = std::getenv("GPUFV_FUSED_SCHED"); return !(e && e[0] == '0'); }();
  // (every cluster must own a tile: the finalize takes clusters 0 .. ncl-1 as the set's segments)
  const bool fuse_ok = fuse_env && batch == 1 && rows < 0 && n_total > 0 && !sparse && !is_wide(K, D) &&
                       lat_finalize_fits(K, D, batch) && (int64_t)L.ncl <= (n_total + kTileM - 1) / kTileM;
  // ... and its finalize runs inside k_stats (fin_lat_fused: no second kernel; GPUFV_FIN_FUSED=0 keeps
  // k_finalize_lat, for A/B runs).  A scored frame (the monitoring application) takes the fused path
  // only with its finalize fused (k_finalize_lat has no scoring) and an L2 norm (NORM_NONE scores stay
  // on the two-kernel path)
  const bool fin_fused = fuse_ok && (sc.n_cls == 0 || (flags & FV_NORM_MASK) != FV_NORM_NONE) &&
                         fin_fused_wanted(K, D, sc.n_cls, L.C, L.ncl, (n_total + kTileM - 1) / kTileM,
                                          num_clusters(L.C, false));
  const bool fuse = fuse_ok && (sc.n_cls == 0 || fin_fused);
  FinParams f = fin_params(L, offsets, batch, K, D, w, mu, sg, flags, ws);
  if (fuse) {  // the finalize ORs the per-CTA range flags into the image's flag word and derives the
               // single set's segments (every cluster owns >= 1 of its T >= ncl tiles) and N itself
    f.rflag_cta = (const int *)at(ws, L.rflagc);
    f.nflag = L.ncl * L.C;
    f.rflags = (int *)at(ws, L.rflags) + rf_base;
    f.fused_n = n_total;
  }
  f.out = out;
  f.svm_w = sc.w; f.svm_b = sc.b; f.n_cls = sc.n_cls; f.scores = sc.scores;
  if (fv_status s = launch_stats(L, X, offsets, n_total, batch, D, K, thr, ws, nullptr, 0, st, nullptr, ldx, rf_base, rows,
                                 sparse, fuse, fin_fused ? &f : nullptr))
    return s;
  if (fin_fused) return FV_OK;
  f.offsets = offsets;  // launch_stats points a single set's NULL offsets at k_schedule's {0, n}
  return launch_finalize(f, batch, K, D, st);
}

fv_status check_scoring(const float *svm_w, int n_cls, const float *scores, int batch) {
  if (n_cls < 1 || n_cls > kMaxCls) return fail(FV_ERR_ARG, "n_cls=%d must be in [1, %d]", n_cls, kMaxCls);
  if (!svm_w || (batch > 0 && !scores)) return fail(FV_ERR_ARG, "null classifier weights/scores");
  return FV_OK;
}

fv_status check_common(const float *X, int64_t n_total, int batch, int D, int K, float thr, const float *w,
                       const float *mu, const float *sg, unsigned flags) {
  if (fv_status s = check_gmm_args(K, D, w, mu, sg, flags)) return s;
  if (n_total < 0 || batch < 0) return fail(FV_ERR_ARG, "n_total=%lld, batch=%d must be >= 0", (long long)n_total, batch);
  if (n_total >= ((int64_t)1 << 30)) return fail(FV_ERR_UNSUPPORTED, "n_total=%lld >= 2^30 per call (split the batch)", (long long)n_total);
  if (n_total > 0 && !X) return fail(FV_ERR_ARG, "null X");
  if (X && reinterpret_cast<uintptr_t>(X) % 16) return fail(FV_ERR_UNSUPPORTED, "X must be 16-byte aligned");
  if (std::isnan(thr) || thr >= 1.f) return fail(FV_ERR_ARG, "threshold must be < 1 and not NaN");
  return FV_OK;
}

}  // namespace

extern "C" {

size_t fv_workspace_bytes(int64_t n_total, int batch, int K, int D, unsigned flags) {
  (void)flags;
  Layout L;
  if (K < 1 || K > kMaxK || batch < 0 || n_total < 0) return 0;
  if (!make_layout(n_total, batch, K, D, false, L)) return 0;
  return L.total;
}

size_t fv_workspace_bytes_host(int64_t n_total, int batch, int K, int D, unsigned flags) {
  (void)flags;
  Layout L;
  if (K < 1 || K > kMaxK || batch < 0 || n_total < 0) return 0;
  if (!make_layout(n_total, batch, K, D, true, L)) return 0;
  return L.total;
}

fv_status fv_gmm_prepare(const float *w, const float *mu, const float *sg, int K, int D, unsigned flags, void *ws,
                         size_t ws_bytes, fv_stream_t stream) {
  NvtxRange nvtx_range("fv_gmm_prepare");
  g_launches = 0;
  if (fv_status s = check_gmm_args(K, D, w, mu, sg, flags)) return s;
  if (fv_status s = check_device()) return s;
  Layout L;
  if (!make_layout(0, 0, K, D, false, L)) return fail(FV_ERR_CUDA, "occupancy query failed");
  if (!ws) return fail(FV_ERR_ARG, "null workspace");
  if (ws_bytes < L.tiles) return fail(FV_ERR_WORKSPACE, "workspace too small for the prepared GMM");
  return launch_prep(L, w, mu, sg, K, D, flags, ws, (cudaStream_t)stream);
}

fv_status fv_encode_batched(const float *X, const int64_t *offsets, int batch, int64_t n_total, int D, const float *w,
                            const float *mu, const float *sg, int K, float thr, unsigned flags, float *out, void *ws,
                            size_t ws_bytes, fv_stream_t stream) {
  NvtxRange nvtx_range("fv_encode_batched");
  g_launches = 0;
  if (fv_status s = check_common(X, n_total, batch, D, K, thr, w, mu, sg, flags)) return s;
  if (batch > 0 && (!offsets || !out)) return fail(FV_ERR_ARG, "null offsets/out");
  if (fv_status s = check_device()) return s;
  return encode_batched_impl(X, offsets, batch, n_total, D, w, mu, sg, K, thr, flags, out, ws, ws_bytes,
                             (cudaStream_t)stream, nullptr);
}

fv_status fv_encode(const float *X, int64_t N, int D, const float *w, const float *mu, const float *sg, int K,
                    float thr, unsigned flags, float *out, void *ws, size_t ws_bytes, fv_stream_t stream) {
  NvtxRange nvtx_range("fv_encode");
  g_launches = 0;
  if (fv_status s = check_common(X, N, 1, D, K, thr, w, mu, sg, flags)) return s;
  if (!out) return fail(FV_ERR_ARG, "null out");
  if (fv_status s = check_device()) return s;
  Layout L;
  if (!make_layout(N, 1, K, D, false, L)) return fail(FV_ERR_CUDA, "occupancy query failed");
  if (fv_status s = check_ws(ws, ws_bytes, L)) return s;
  return encode_batched_impl(X, nullptr, 1, N, D, w, mu, sg, K, thr, flags, out, ws, ws_bytes, (cudaStream_t)stream, &L);
}

}  // extern "C"

namespace {

// Internal streams / events of the host pipeline: created once per (thread, device) on first use and
// reused by every later call (never destroyed: they live as long as the thread's CUDA context), so a
// call makes no stream or event allocations after the first.
constexpr int kHostChunks = 16;
struct HostPipe {
  cudaStream_t cin = nullptr, cout = nullptr;
  cudaEvent_t ev[2 * kHostChunks + 1] = {};
  bool ok = false;
};
fv_status host_pipe(HostPipe *&hp) {
  thread_local HostPipe pipes[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return cuda_check("cudaGetDevice");
  hp = &pipes[dev];
  if (hp->ok) return FV_OK;
  if (cudaStreamCreateWithFlags(&hp->cin, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&hp->cout, cudaStreamNonBlocking) != cudaSuccess)
    return cuda_check("stream create");
  for (auto &e : hp->ev)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return cuda_check("event create");
  hp->ok = true;
  return FV_OK;
}

// Host-buffer pipeline shared by fv_encode_batched_host and fv_encode_scored_batched_host: the result
// per image is the FV (2KD floats) or, with scoring, its n_cls scores.
fv_status encode_host_impl(const float *X_host, const int64_t *offsets_host, int batch, int64_t n_total, int D,
                           const float *w, const float *mu, const float *sg, int K, float thr, unsigned flags,
                           float *res_host, const Scoring &sc_in, void *ws, size_t ws_bytes, cudaStream_t st) {
  // the offsets are on the host: validate them before any copy sized from them (header contract)
  if (batch > 0) {
    if (offsets_host[0] != 0 || offsets_host[batch] != n_total)
      return fail(FV_ERR_ARG, "offsets[0] must be 0 and offsets[batch] == n_total");
    for (int b = 0; b < batch; ++b)
      if (offsets_host[b + 1] < offsets_host[b]) return fail(FV_ERR_ARG, "offsets must be non-decreasing (b=%d)", b);
  }
  Layout L;
  if (!make_layout(n_total, batch, K, D, true, L, sc_in.n_cls)) return fail(FV_ERR_CUDA, "occupancy query failed");
  if (fv_status s = check_ws(ws, ws_bytes, L)) return s;
  HostPipe *hp = nullptr;
  if (fv_status s = host_pipe(hp)) return s;
  float *dX = (float *)at(ws, L.hx);
  int64_t *doff = (int64_t *)at(ws, L.hoff);
  float *dres = (float *)at(ws, L.hout);
  if (cudaMemcpyAsync(doff, offsets_host, (size_t)(batch + 1) * 8, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return cuda_check("H2D offsets");
  if (!(flags & FV_PREPARED))
    if (fv_status s = launch_prep(L, w, mu, sg, K, D, flags, ws, st)) return s;
  if (batch == 0) return cudaStreamSynchronize(st) == cudaSuccess ? FV_OK : cuda_check("stream sync");
  // the internal streams start behind everything already queued on the caller's stream (earlier work
  // may still use the workspace bytes the X copies overwrite)
  cudaEvent_t ev0 = hp->ev[2 * kHostChunks];
  if (cudaEventRecord(ev0, st) != cudaSuccess || cudaStreamWaitEvent(hp->cin, ev0, 0) != cudaSuccess ||
      cudaStreamWaitEvent(hp->cout, ev0, 0) != cudaSuccess)
    return cuda_check("order internal streams");
  // Pipelined in image chunks: the H2D copy of chunk k+1 (stream `cin`) and the D2H copy of chunk k-1
  // (stream `cout`) overlap the encode of chunk k on `stream`; events order each chunk's three steps.
  const size_t per_image = sc_in.n_cls > 0 ? (size_t)sc_in.n_cls : (size_t)2 * K * D;
  const int nch = std::max(1, std::min(batch, kHostChunks));
  cudaStream_t cin = hp->cin, cout = hp->cout;
  cudaEvent_t *ev = hp->ev;
  fv_status rs = FV_OK;
  for (int k = 0; k < nch && rs == FV_OK; ++k) {
    NvtxRange chunk_range("fv host chunk");
    const int b0 = (int)((int64_t)k * batch / nch), b1 = (int)((int64_t)(k + 1) * batch / nch);
    const int64_t r0 = offsets_host[b0], r1 = offsets_host[b1];
    if (r1 > r0 && cudaMemcpyAsync(dX + r0 * D, X_host + r0 * D, (size_t)(r1 - r0) * D * 4, cudaMemcpyHostToDevice,
                                   cin) != cudaSuccess) { rs = cuda_check("H2D X"); break; }
    cudaEventRecord(ev[2 * k], cin);
    cudaStreamWaitEvent(st, ev[2 * k], 0);
    // the chunk's images through the device path: absolute row offsets into the staged X
    Scoring sc = sc_in;
    float *out = dres + (size_t)b0 * per_image;
    if (sc.n_cls > 0) { sc.scores = out; out = nullptr; }
    // (a one-image call is one set with offsets {0, n_total}, checked above: rows = -1 lets it take the
    // single-kernel latency path like fv_encode)
    rs = encode_batched_impl(dX, doff + b0, b1 - b0, n_total, D, w, mu, sg, K, thr, flags | FV_PREPARED, out, ws,
                             ws_bytes, st, &L, sc, 0, b0, batch == 1 ? -1 : r1 - r0);
    if (rs != FV_OK) break;
    cudaEventRecord(ev[2 * k + 1], st);
    cudaStreamWaitEvent(cout, ev[2 * k + 1], 0);
    if (cudaMemcpyAsync(res_host + (size_t)b0 * per_image, dres + (size_t)b0 * per_image,
                        (size_t)(b1 - b0) * per_image * 4, cudaMemcpyDeviceToHost, cout) != cudaSuccess) {
      rs = cuda_check("D2H result");
      break;
    }
  }
  if (cudaStreamSynchronize(cout) != cudaSuccess || cudaStreamSynchronize(cin) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    if (rs == FV_OK) rs = cuda_check("stream sync");
  return rs;
}

}  // namespace

extern "C" {

fv_status fv_encode_batched_host(const float *X_host, const int64_t *offsets_host, int batch, int64_t n_total, int D,
                                 const float *w, const float *mu, const float *sg, int K, float thr, unsigned flags,
                                 float *out_host, void *ws, size_t ws_bytes, fv_stream_t stream) {
  NvtxRange nvtx_range("fv_encode_batched_host");
  g_launches = 0;
  if (fv_status s = check_common(X_host, n_total, batch, D, K, thr, w, mu, sg, flags)) return s;
  if (batch > 0 && (!offsets_host || !out_host)) return fail(FV_ERR_ARG, "null offsets/out");
  if (fv_status s = check_device()) return s;
  return encode_host_impl(X_host, offsets_host, batch, n_total, D, w, mu, sg, K, thr, flags, out_host, Scoring(), ws,
                          ws_bytes, (cudaStream_t)stream);
}

size_t fv_workspace_bytes_scored(int64_t n_total, int batch, int K, int D, int n_cls, int host_io, unsigned flags) {
  (void)flags;
  Layout L;
  if (K < 1 || K > kMaxK || batch < 0 || n_total < 0 || n_cls < 1 || n_cls > kMaxCls) return 0;
  if (!make_layout(n_total, batch, K, D, host_io != 0, L, n_cls)) return 0;
  return L.total;
}

fv_status fv_encode_scored_batched(const float *X, const int64_t *offsets, int batch, int64_t n_total, int D,
                                   const float *w, const float *mu, const float *sg, int K, float thr, unsigned flags,
                                   const float *svm_w, const float *svm_b, int n_cls, float *scores, float *out,
                                   void *ws, size_t ws_bytes, fv_stream_t stream) {
  NvtxRange nvtx_range("fv_encode_scored_batched");
  g_launches = 0;
  if (fv_status s = check_common(X, n_total, batch, D, K, thr, w, mu, sg, flags)) return s;
  if (batch > 0 && !offsets) return fail(FV_ERR_ARG, "null offsets");
  if (fv_status s = check_scoring(svm_w, n_cls, scores, batch)) return s;
  if (fv_status s = check_device()) return s;
  Scoring sc;
  sc.w = svm_w; sc.b = svm_b; sc.n_cls = n_cls; sc.scores = scores;
  return encode_batched_impl(X, offsets, batch, n_total, D, w, mu, sg, K, thr, flags, out, ws, ws_bytes,
                             (cudaStream_t)stream, nullptr, sc);
}

fv_status fv_encode_scored_batched_host(const float *X_host, const int64_t *offsets_host, int batch, int64_t n_total,
                                        int D, const float *w, const float *mu, const float *sg, int K, float thr,
                                        unsigned flags, const float *svm_w, const float *svm_b, int n_cls,
                                        float *scores_host, void *ws, size_t ws_bytes, fv_stream_t stream) {
  NvtxRange nvtx_range("fv_encode_scored_batched_host");
  g_launches = 0;
  if (fv_status s = check_common(X_host, n_total, batch, D, K, thr, w, mu, sg, flags)) return s;
  if (batch > 0 && !offsets_host) return fail(FV_ERR_ARG, "null offsets");
  if (fv_status s = check_scoring(svm_w, n_cls, scores_host, batch)) return s;
  if (fv_status s = check_device()) return s;
  Scoring sc;
  sc.w = svm_w; sc.b = svm_b; sc.n_cls = n_cls;
  return encode_host_impl(X_host, offsets_host, batch, n_total, D, w, mu, sg, K, thr, flags, scores_host, sc, ws,
                          ws_bytes, (cudaStream_t)stream);
}

fv_status fv_stats_batched(const float *X, const int64_t *offsets, int batch, int64_t n_total, int D, const float *w,
                           const float *mu, const float *sg, int K, float thr, unsigned flags, double *stats, void *ws,
                           size_t ws_bytes, fv_stream_t stream) {
  NvtxRange nvtx_range("fv_stats_batched");
  g_launches = 0;
  if (fv_status s = check_common(X, n_total, batch, D, K, thr, w, mu, sg, flags)) return s;
  if (batch > 0 && (!offsets || !stats)) return fail(FV_ERR_ARG, "null offsets/stats");
  if (fv_status s = check_device()) return s;
  Layout L;
  if (!make_layout(n_total, batch, K, D, false, L)) return fail(FV_ERR_CUDA, "occupancy query failed");
  if (fv_status s = check_ws(ws, ws_bytes, L)) return s;
  cudaStream_t st = (cudaStream_t)stream;
  if (!(flags & FV_PREPARED))
    if (fv_status s = launch_prep(L, w, mu, sg, K, D, flags, ws, st)) return s;
  if (batch == 0) return FV_OK;
  if (fv_status s = launch_stats(L, X, offsets, n_total, batch, D, K, thr, ws, nullptr, 0, st, nullptr, 0, 0, -1,
                                 (flags & FV_SPARSE_STATS) != 0))
    return s;
  FinParams f = fin_params(L, offsets, batch, K, D, w, mu, sg, flags, ws);
  f.stats_out = stats;
  for (int b0 = 0; b0 < batch; b0 += 65535) {
    FinParams fc = f;
    fc.b_base = b0;
    k_reduce_stats<<<dim3((K + kFinJ - 1) / kFinJ, std::min(65535, batch - b0), (D + kDP - 1) / kDP), 256, 0, st>>>(fc);
    g_launches += 1;
  }
  return cuda_check("k_reduce_stats");
}

fv_status fv_finalize(const double *stats, int batch, int D, const float *w, const float *mu, const float *sg, int K,
                      unsigned flags, float *out, void *ws, size_t ws_bytes, fv_stream_t stream) {
  NvtxRange nvtx_range("fv_finalize");
  g_launches = 0;
  if (fv_status s = check_gmm_args(K, D, w, mu, sg, flags)) return s;
  if (batch < 0) return fail(FV_ERR_ARG, "batch < 0");
  if (batch > 0 && (!stats || !out)) return fail(FV_ERR_ARG, "null stats/out");
  if (fv_status s = check_device()) return s;
  Layout L;
  if (!make_layout(0, batch, K, D, false, L)) return fail(FV_ERR_CUDA, "occupancy query failed");
  if (fv_status s = check_ws(ws, ws_bytes, L)) return s;
  cudaStream_t st = (cudaStream_t)stream;
  if (!(flags & FV_PREPARED))
    if (fv_status s = launch_prep(L, w, mu, sg, K, D, flags, ws, st)) return s;
  FinParams f = fin_params(L, nullptr, batch, K, D, w, mu, sg, flags, ws);
  f.slots = nullptr;
  f.stats = stats;
  f.out = out;
  return launch_finalize(f, batch, K, D, st, false);
}

fv_status fv_posteriors(const float *X, int64_t N, int D, const float *w, const float *mu, const float *sg, int K,
                        float thr, unsigned flags, float *gamma, void *ws, size_t ws_bytes, fv_stream_t stream) {
  NvtxRange nvtx_range("fv_posteriors");
  g_launches = 0;
  // bit 8 (undocumented, tests only): write raw log2-likelihoods instead of gamma
  const int mode = (flags & (1u << 8)) ? 2 : 1;
  flags &= ~(1u << 8);
  if (fv_status s = check_common(X, N, 1, D, K, thr, w, mu, sg, flags)) return s;
  if (N > 0 && !gamma) return fail(FV_ERR_ARG, "null gamma");
  if (fv_status s = check_device()) return s;
  Layout L;
  if (!make_layout(N, 1, K, D, false, L)) return fail(FV_ERR_CUDA, "occupancy query failed");
  if (fv_status s = check_ws(ws, ws_bytes, L)) return s;
  cudaStream_t st = (cudaStream_t)stream;
  if (!(flags & FV_PREPARED))
    if (fv_status s = launch_prep(L, w, mu, sg, K, D, flags, ws, st)) return s;
  if (N == 0) return FV_OK;
  const int64_t *offs = nullptr;
  return launch_stats(L, X, offs, N, 1, D, K, thr, ws, gamma, mode, st);
}

size_t fv_workspace_bytes_em(int64_t N, int K, int D, unsigned flags) {
  (void)flags;
  Layout L;
  if (K < 1 || K > kMaxK || N < 0) return 0;
  if (!make_layout(N, 1, K, D, false, L, 0, true)) return 0;
  return L.total;
}

}  // extern "C"

namespace {

// E-step of EM (NEXT-3) on one descriptor set: exact posteriors through the production stats kernel,
// sufficient statistics [N, S0, S1, S2] about c (k_reduce_stats) and the total log-likelihood.
fv_status estep_impl(const Layout &L, const float *X, int64_t N, int D, const float *w, const float *mu,
                     const float *sg, int K, unsigned flags, double *stats, double *loglik, void *ws, cudaStream_t st) {
  if (!(flags & FV_PREPARED))
    if (fv_status s = launch_prep(L, w, mu, sg, K, D, flags, ws, st)) return s;
  const size_t nst = (1 + (size_t)K * (2 * D + 1)) * 8;
  if (N == 0) {
    if (cudaMemsetAsync(stats, 0, nst, st) != cudaSuccess || cudaMemsetAsync(loglik, 0, 8, st) != cudaSuccess)
      return cuda_check("memset");
    return FV_OK;
  }
  const int64_t *offs = nullptr;
  float *llrows = (float *)at(ws, L.llrows);
  if (fv_status s = launch_stats(L, X, offs, N, 1, D, K, 0.f, ws, nullptr, 0, st, llrows)) return s;
  FinParams f = fin_params(L, offs, 1, K, D, w, mu, sg, flags, ws);
  f.stats_out = stats;
  k_reduce_stats<<<dim3((K + kFinJ - 1) / kFinJ, 1, (D + kDP - 1) / kDP), 256, 0, st>>>(f);
  double *parts = (double *)at(ws, L.llparts);
  unsigned *ticket = (unsigned *)(parts + kLLBlocks);
  if (cudaMemsetAsync(ticket, 0, 4, st) != cudaSuccess) return cuda_check("memset ticket");
  k_loglik_reduce<<<kLLBlocks, 256, 0, st>>>(llrows, N, D, (const double *)at(ws, L.bmax), parts, ticket, loglik);
  g_launches += 2;
  return cuda_check("k_reduce_stats/k_loglik_reduce");
}

fv_status mstep_impl(const Layout &L, const double *stats, int D, const float *w, const float *mu, const float *sg,
                     int K, unsigned flags, float floor_abs, float floor_rel, float prior_floor, float *w_new,
                     float *mu_new, float *var_new, void *ws, cudaStream_t st) {
  if (!(flags & FV_PREPARED))
    if (fv_status s = launch_prep(L, w, mu, sg, K, D, flags, ws, st)) return s;
  k_mstep<<<1, 1024, 0, st>>>(stats, K, D, (const double *)at(ws, L.cshift), w, mu, sg,
                              (flags & FV_SIGMA_IS_STDDEV) ? 1 : 0, floor_abs, floor_rel, prior_floor, w_new, mu_new,
                              var_new);
  g_launches += 1;
  return cuda_check("k_mstep");
}

fv_status check_floors(float floor_abs, float floor_rel, float prior_floor) {
  if (!(floor_abs >= 0.f) || !(floor_rel >= 0.f) || !(prior_floor >= 0.f) || !(prior_floor < 1.f) ||
      !std::isfinite(floor_abs) || !std::isfinite(floor_rel))
    return fail(FV_ERR_ARG, "floors must be finite, >= 0 (prior_floor < 1)");
  return FV_OK;
}

}  // namespace

extern "C" {

fv_status fv_gmm_estep(const float *X, int64_t N, int D, const float *w, const float *mu, const float *sg, int K,
                       unsigned flags, double *stats, double *loglik, void *ws, size_t ws_bytes, fv_stream_t stream) {
  NvtxRange nvtx_range("fv_gmm_estep");
  g_launches = 0;
  if (fv_status s = check_common(X, N, 1, D, K, 0.f, w, mu, sg, flags)) return s;
  if (!stats || !loglik) return fail(FV_ERR_ARG, "null stats/loglik");
  if (fv_status s = check_device()) return s;
  Layout L;
  if (!make_layout(N, 1, K, D, false, L, 0, true)) return fail(FV_ERR_CUDA, "occupancy query failed");
  if (fv_status s = check_ws(ws, ws_bytes, L)) return s;
  return estep_impl(L, X, N, D, w, mu, sg, K, flags, stats, loglik, ws, (cudaStream_t)stream);
}

fv_status fv_gmm_mstep(const double *stats, int D, const float *w, const float *mu, const float *sg, int K,
                       unsigned flags, float var_floor_abs, float var_floor_rel, float prior_floor, float *w_new,
                       float *mu_new, float *var_new, void *ws, size_t ws_bytes, fv_stream_t stream) {
  NvtxRange nvtx_range("fv_gmm_mstep");
  g_launches = 0;
  if (fv_status s = check_gmm_args(K, D, w, mu, sg, flags)) return s;
  if (!stats || !w_new || !mu_new || !var_new) return fail(FV_ERR_ARG, "null stats/output");
  if (fv_status s = check_floors(var_floor_abs, var_floor_rel, prior_floor)) return s;
  if (fv_status s = check_device()) return s;
  Layout L;
  if (!make_layout(0, 1, K, D, false, L, 0, true)) return fail(FV_ERR_CUDA, "occupancy query failed");
  if (fv_status s = check_ws(ws, ws_bytes, L)) return s;
  return mstep_impl(L, stats, D, w, mu, sg, K, flags, var_floor_abs, var_floor_rel, prior_floor, w_new, mu_new,
                    var_new, ws, (cudaStream_t)stream);
}

fv_status fv_gmm_em_step(const float *X, int64_t N, int D, const float *w, const float *mu, const float *sg, int K,
                         unsigned flags, float var_floor_abs, float var_floor_rel, float prior_floor, float *w_new,
                         float *mu_new, float *var_new, double *loglik, void *ws, size_t ws_bytes,
                         fv_stream_t stream) {
  NvtxRange nvtx_range("fv_gmm_em_step");
  g_launches = 0;
  if (fv_status s = check_common(X, N, 1, D, K, 0.f, w, mu, sg, flags)) return s;
  if (!w_new || !mu_new || !var_new || !loglik) return fail(FV_ERR_ARG, "null output");
  if (N < 1) return fail(FV_ERR_ARG, "EM needs N >= 1 descriptors");
  if (fv_status s = check_floors(var_floor_abs, var_floor_rel, prior_floor)) return s;
  if (fv_status s = check_device()) return s;
  Layout L;
  if (!make_layout(N, 1, K, D, false, L, 0, true)) return fail(FV_ERR_CUDA, "occupancy query failed");
  if (fv_status s = check_ws(ws, ws_bytes, L)) return s;
  cudaStream_t st = (cudaStream_t)stream;
  double *stats = (double *)at(ws, L.emstats);
  if (fv_status s = estep_impl(L, X, N, D, w, mu, sg, K, flags, stats, loglik, ws, st)) return s;
  return mstep_impl(L, stats, D, w, mu, sg, K, flags | FV_PREPARED, var_floor_abs, var_floor_rel, prior_floor, w_new,
                    mu_new, var_new, ws, st);
}

}  // extern "C"

namespace {

constexpr int kEmbLd(int m) { return (m + 2 + 3) / 4 * 4; }

fv_status check_embed_args(const float *raw, const float *xy, const int64_t *offsets, int batch, int64_t n_total,
                           const float *wh, const float *mean, const float *basis, int m) {
  if (m < 1 || m > kEmbMaxM) return fail(FV_ERR_ARG, "m=%d must be in [1, %d]", m, kEmbMaxM);
  if (n_total < 0 || batch < 0) return fail(FV_ERR_ARG, "n_total/batch < 0");
  if (n_total >= ((int64_t)1 << 30)) return fail(FV_ERR_UNSUPPORTED, "n_total >= 2^30 per call");
  if (!mean || !basis) return fail(FV_ERR_ARG, "null PCA model");
  if (batch > 0 && (!offsets || !wh)) return fail(FV_ERR_ARG, "null offsets/img_wh");
  if (n_total > 0 && (!raw || !xy)) return fail(FV_ERR_ARG, "null raw/xy");
  if ((raw && reinterpret_cast<uintptr_t>(raw) % 16) || reinterpret_cast<uintptr_t>(mean) % 16 ||
      (xy && reinterpret_cast<uintptr_t>(xy) % 16) || (wh && reinterpret_cast<uintptr_t>(wh) % 8))
    return fail(FV_ERR_UNSUPPORTED, "raw/mean/xy must be 16-byte and img_wh 8-byte aligned (TMA)");
  return FV_OK;
}

fv_status launch_embed(const float *raw, const float *xy, const int64_t *offsets, int batch, int64_t n_total,
                       const float *wh, const float *mean, const float *basis, int m, float *out, int ldx,
                       cudaStream_t st) {
  if (n_total == 0 || batch == 0) return FV_OK;
  EmbedParams e;
  e.xy = xy; e.offsets = offsets; e.wh = wh; e.mean = mean; e.basis = basis; e.out = out;
  e.n = n_total; e.batch = batch; e.m = m; e.ldx = ldx;
  // raw as a 2-D tensor map: dims {128, n_total}, boxes of 32 floats x 128 rows, 128B swizzle (the tf32
  // K-major operand layout); rows past n_total read as zero
  CUtensorMap tmap, tmap_xy, tmap_out;
  {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
      cudaDriverEntryPointQueryResult q;
      void *fn = nullptr;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
        return fail(FV_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
      encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    cuuint64_t dims[2] = {(cuuint64_t)kEmbIn, (cuuint64_t)n_total};
    cuuint64_t strides[1] = {(cuuint64_t)kEmbIn * 4};
    cuuint32_t box[2] = {32u, 128u};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(raw), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(FV_ERR_CUDA, "cuTensorMapEncodeTiled (raw) failed (%d)", (int)r);
    // keypoints as a 1-D map of 2 n_total floats, boxes of 256 (one tile's 128 rows); past the end: zero
    cuuint64_t dxy[1] = {(cuuint64_t)(2 * n_total)};
    cuuint32_t bxy[1] = {256u};
    cuuint32_t exy[1] = {1};
    cuuint64_t sxy[1] = {(cuuint64_t)(2 * n_total) * 4};  // unused for rank 1 (the driver wants a valid array)
    r = encode(&tmap_xy, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 1, const_cast<float *>(xy), dxy, sxy, bxy, exy,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(FV_ERR_CUDA, "cuTensorMapEncodeTiled (xy) failed (%d)", (int)r);
    // output as {ldx, n_total}, stored in 32-dim x 32-row boxes (unswizzled, row-major staging)
    cuuint64_t dout[2] = {(cuuint64_t)ldx, (cuuint64_t)n_total};
    cuuint64_t sout[1] = {(cuuint64_t)ldx * 4};
    cuuint32_t bout[2] = {32u, 32u};
    r = encode(&tmap_out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, out, dout, sout, bout, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(FV_ERR_CUDA, "cuTensorMapEncodeTiled (out) failed (%d)", (int)r);
  }
  static std::mutex mu;
  static bool attr_done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    if (dev < 0 || dev >= 64 || !attr_done[dev]) {
      if (cudaFuncSetAttribute(k_embed, cudaFuncAttributeMaxDynamicSharedMemorySize, kEmbSmemBytes) != cudaSuccess)
        return cuda_check("k_embed attribute");
      if (dev >= 0 && dev < 64) attr_done[dev] = true;
    }
  }
  const int64_t ntiles = (n_total + 127) / 128;
  const int grid = (int)std::min<int64_t>(ntiles, (int64_t)sm_count());
  k_embed<<<grid, kEmbThreads, kEmbSmemBytes, st>>>(tmap, tmap_xy, tmap_out, e);
  g_launches += 1;
  return cuda_check("k_embed");
}

}  // namespace

extern "C" {

fv_status fv_embed(const float *raw, const float *xy, const int64_t *offsets, int batch, int64_t n_total,
                   const float *img_wh, const float *pca_mean, const float *pca_basis, int m, float *X_out, int ldx,
                   fv_stream_t stream) {
  NvtxRange nvtx_range("fv_embed");
  g_launches = 0;
  if (fv_status s = check_embed_args(raw, xy, offsets, batch, n_total, img_wh, pca_mean, pca_basis, m)) return s;
  if (n_total > 0 && !X_out) return fail(FV_ERR_ARG, "null X_out");
  if (ldx < m + 2 || ldx % 4) return fail(FV_ERR_ARG, "ldx=%d must be >= m+2 and a multiple of 4", ldx);
  if (X_out && reinterpret_cast<uintptr_t>(X_out) % 16) return fail(FV_ERR_UNSUPPORTED, "X_out must be 16-byte aligned");
  if (fv_status s = check_device()) return s;
  return launch_embed(raw, xy, offsets, batch, n_total, img_wh, pca_mean, pca_basis, m, X_out, ldx,
                      (cudaStream_t)stream);
}

size_t fv_workspace_bytes_embed(int64_t n_total, int batch, int K, int m, unsigned flags) {
  (void)flags;
  Layout L;
  if (K < 1 || K > kMaxK || batch < 0 || n_total < 0 || m < 1 || m > kEmbMaxM) return 0;
  if (!make_layout(n_total, batch, K, m + 2, false, L, 0, false, kEmbLd(m))) return 0;
  return L.total;
}

fv_status fv_embed_encode_batched(const float *raw, const float *xy, const int64_t *offsets, int batch,
                                  int64_t n_total, const float *img_wh, const float *pca_mean,
                                  const float *pca_basis, int m, const float *w, const float *mu, const float *sg,
                                  int K, float thr, unsigned flags, float *out, void *ws, size_t ws_bytes,
                                  fv_stream_t stream) {
  NvtxRange nvtx_range("fv_embed_encode_batched");
  g_launches = 0;
  const int D = m + 2;
  if (fv_status s = check_embed_args(raw, xy, offsets, batch, n_total, img_wh, pca_mean, pca_basis, m)) return s;
  if (fv_status s = check_gmm_args(K, D, w, mu, sg, flags, false)) return s;
  if (std::isnan(thr) || thr >= 1.f) return fail(FV_ERR_ARG, "threshold must be < 1 and not NaN");
  if (batch > 0 && !out) return fail(FV_ERR_ARG, "null out");
  if (fv_status s = check_device()) return s;
  Layout L;
  const int ldx = kEmbLd(m);
  if (!make_layout(n_total, batch, K, D, false, L, 0, false, ldx)) return fail(FV_ERR_CUDA, "occupancy query failed");
  if (fv_status s = check_ws(ws, ws_bytes, L)) return s;
  cudaStream_t st = (cudaStream_t)stream;
  float *Xe = (float *)at(ws, L.emb);
  if (fv_status s = launch_embed(raw, xy, offsets, batch, n_total, img_wh, pca_mean, pca_basis, m, Xe, ldx, st))
    return s;
  return encode_batched_impl(Xe, offsets, batch, n_total, D, w, mu, sg, K, thr, flags, out, ws, ws_bytes, st, &L,
                             Scoring(), ldx);
}

fv_status fv_range_flags(const void *ws, size_t ws_bytes, int64_t n_total, int batch, int K, int D, int32_t *flags_out,
                         fv_stream_t stream) {
  NvtxRange nvtx_range("fv_range_flags");
  g_launches = 0;
  if (K < 1 || D < 1 || K > kMaxK || D > kDMax || n_total < 0 || batch < 0) return fail(FV_ERR_ARG, "bad sizes");
  if (batch > 0 && !flags_out) return fail(FV_ERR_ARG, "null flags_out");
  if (fv_status s = check_device()) return s;
  Layout L;
  if (!make_layout(n_total, batch, K, D, false, L)) return fail(FV_ERR_CUDA, "occupancy query failed");
  if (fv_status s = check_ws(const_cast<void *>(ws), ws_bytes, L)) return s;
  if (batch == 0) return FV_OK;
  k_range_flags<<<(batch + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
      (const int *)at(const_cast<void *>(ws), L.rflags), (const int *)at(const_cast<void *>(ws), L.gflag), batch, flags_out);
  g_launches = 1;
  return cuda_check("k_range_flags");
}

int fv_last_launch_count(void) { return g_launches; }

void fv_debug_trace(long long *dev_buf) { g_trace = dev_buf; }

void fv_profile_events(void *start_event, void *stop_event) {
  g_prof_start = static_cast<cudaEvent_t>(start_event);
  g_prof_stop = static_cast<cudaEvent_t>(stop_event);
}

const char *fv_status_string(fv_status s) {
  switch (s) {
    case FV_OK: return "FV_OK";
    case FV_ERR_ARG: return "FV_ERR_ARG: invalid argument";
    case FV_ERR_UNSUPPORTED: return "FV_ERR_UNSUPPORTED: unsupported shape/alignment/device";
    case FV_ERR_WORKSPACE: return "FV_ERR_WORKSPACE: workspace too small or misaligned";
    case FV_ERR_CUDA: return "FV_ERR_CUDA: CUDA error";
  }
  return "unknown fv_status";
}

const char *fv_last_error(void) { return g_err.c_str(); }

int fv_version(void) { return 1; }

}  // extern "C"
