"""ctypes wrapper around oracle/fv_oracle.c (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

Inputs are converted to float64 exactly (the GPU path receives the same float32 values), outputs are
float64 numpy arrays.  The library is built with plain ``gcc -O2 -fopenmp`` (no -ffast-math) on first
use, or by ``__graft_entry__.build()``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

NORM_IMPROVED = 0
NORM_POWER_L2 = 1
NORM_NONE = 2

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fv_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)


def build(force: bool = False) -> str:
    """Compile fv_oracle.c into oracle/liboracle.so (IEEE double, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared",
             "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            lib.fvo_posteriors.argtypes = [_dp, ctypes.c_int64, ctypes.c_int, _dp, _dp, _dp, ctypes.c_int, _dp]
            lib.fvo_posteriors.restype = None
            lib.fvo_accumulate.argtypes = [_dp, ctypes.c_int64, ctypes.c_int, _dp, _dp, _dp, ctypes.c_int,
                                           ctypes.c_double, _dp, _dp]
            lib.fvo_accumulate.restype = None
            lib.fvo_normalize.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_int64, _dp, ctypes.c_int]
            lib.fvo_normalize.restype = None
            lib.fvo_encode.argtypes = [_dp, ctypes.c_int64, ctypes.c_int, _dp, _dp, _dp, ctypes.c_int,
                                       ctypes.c_double, ctypes.c_int, _dp, _dp]
            lib.fvo_encode.restype = ctypes.c_int
            lib.fvo_encode_batched.argtypes = [_dp, _i64p, ctypes.c_int, ctypes.c_int, _dp, _dp, _dp,
                                               ctypes.c_int, ctypes.c_double, ctypes.c_int, _dp, ctypes.c_int]
            lib.fvo_encode_batched.restype = ctypes.c_int
            lib.fvo_stats.argtypes = [_dp, ctypes.c_int64, ctypes.c_int, _dp, _dp, _dp, ctypes.c_int,
                                      ctypes.c_double, _dp]
            lib.fvo_stats.restype = ctypes.c_int
            lib.fvo_stats_batched.argtypes = [_dp, _i64p, ctypes.c_int, ctypes.c_int, _dp, _dp, _dp,
                                              ctypes.c_int, ctypes.c_double, _dp, ctypes.c_int]
            lib.fvo_stats_batched.restype = ctypes.c_int
            lib.fvo_max_threads.argtypes = []
            lib.fvo_max_threads.restype = ctypes.c_int
            _lib = lib
    return _lib


def _d(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _gmm(priors, means, variances):
    w, m, v = _d(priors), _d(means), _d(variances)
    K = w.shape[0]
    assert m.ndim == 2 and m.shape[0] == K and v.shape == m.shape
    return w, m, v, K, m.shape[1]


def max_threads() -> int:
    return int(_load().fvo_max_threads())


def posteriors(X, priors, means, variances) -> np.ndarray:
    """Alg.1 lines 2-15: gamma (N x K) in double precision."""
    w, m, v, K, D = _gmm(priors, means, variances)
    X = _d(X).reshape(-1, D)
    g = np.empty((X.shape[0], K), dtype=np.float64)
    _load().fvo_posteriors(_p(X), X.shape[0], D, _p(w), _p(m), _p(v), K, _p(g))
    return g


def accumulate(X, gamma, means, variances, threshold: float = 0.0):
    """Alg.1 lines 16-26: raw (U, V), each K x D."""
    m, v = _d(means), _d(variances)
    K, D = m.shape
    X = _d(X).reshape(-1, D)
    g = _d(gamma).reshape(X.shape[0], K)
    U = np.zeros((K, D)); V = np.zeros((K, D))
    _load().fvo_accumulate(_p(X), X.shape[0], D, _p(g), _p(m), _p(v), K, float(threshold), _p(U), _p(V))
    return U, V


def normalize(fv, priors, N: int, mode: int = NORM_IMPROVED) -> np.ndarray:
    """Reading A9 on fv = [U, V] (length 2KD)."""
    w = _d(priors)
    K = w.shape[0]
    fv = _d(fv).copy().reshape(-1)
    D = fv.shape[0] // (2 * K)
    _load().fvo_normalize(_p(fv), K, D, int(N), _p(w), int(mode))
    return fv


def encode(X, priors, means, variances, threshold: float = 0.0, mode: int = NORM_IMPROVED,
           return_gamma: bool = False):
    """Full encode of one descriptor set -> FV (2KD,) [and gamma (N x K)]."""
    w, m, v, K, D = _gmm(priors, means, variances)
    X = _d(X).reshape(-1, D)
    fv = np.empty(2 * K * D)
    g = np.empty((X.shape[0], K)) if return_gamma else None
    rc = _load().fvo_encode(_p(X), X.shape[0], D, _p(w), _p(m), _p(v), K, float(threshold), int(mode),
                            _p(fv), _p(g) if g is not None else None)
    if rc != 0:
        raise MemoryError("fvo_encode failed")
    return (fv, g) if return_gamma else fv


def encode_batched(X, offsets, priors, means, variances, threshold: float = 0.0,
                   mode: int = NORM_IMPROVED, nthreads: int = 0) -> np.ndarray:
    """Independent images (CSR offsets, length batch+1) -> (batch, 2KD).  OpenMP over images."""
    w, m, v, K, D = _gmm(priors, means, variances)
    X = _d(X).reshape(-1, D)
    off = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
    B = off.shape[0] - 1
    assert off[0] == 0 and off[-1] == X.shape[0]
    out = np.empty((B, 2 * K * D))
    rc = _load().fvo_encode_batched(_p(X), off.ctypes.data_as(_i64p), B, D, _p(w), _p(m), _p(v), K,
                                    float(threshold), int(mode), _p(out), int(nthreads))
    if rc != 0:
        raise MemoryError("fvo_encode_batched failed")
    return out


def stats(X, priors, means, variances, threshold: float = 0.0) -> np.ndarray:
    """[N, S0 (K), S1 (KxD), S2 (KxD)] about c = sum_j pi_j mu_j / sum_j pi_j (reading A19)."""
    w, m, v, K, D = _gmm(priors, means, variances)
    X = _d(X).reshape(-1, D)
    s = np.empty(1 + K * (2 * D + 1))
    if _load().fvo_stats(_p(X), X.shape[0], D, _p(w), _p(m), _p(v), K, float(threshold), _p(s)) != 0:
        raise MemoryError("fvo_stats failed")
    return s


def stats_batched(X, offsets, priors, means, variances, threshold: float = 0.0, nthreads: int = 0):
    w, m, v, K, D = _gmm(priors, means, variances)
    X = _d(X).reshape(-1, D)
    off = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
    B = off.shape[0] - 1
    s = np.empty((B, 1 + K * (2 * D + 1)))
    rc = _load().fvo_stats_batched(_p(X), off.ctypes.data_as(_i64p), B, D, _p(w), _p(m), _p(v), K,
                                   float(threshold), _p(s), int(nthreads))
    if rc != 0:
        raise MemoryError("fvo_stats_batched failed")
    return s


def fv_from_stats(st, priors, means, variances, mode: int = NORM_IMPROVED) -> np.ndarray:
    """FV from summed statistics (the descriptor-sharded path's finalize, written plainly):
    U = (S1 - mu' S0)/sd, V = (S2 - 2 mu' S1 + mu'^2 S0)/var - S0, mu' = mu - c, then normalize."""
    w, m, v, K, D = _gmm(priors, means, variances)
    st = _d(st)
    N = int(round(st[0]))
    S0 = st[1:1 + K]
    S1 = st[1 + K:1 + K + K * D].reshape(K, D)
    S2 = st[1 + K + K * D:].reshape(K, D)
    c = (w[:, None] * m).sum(0) / w.sum()
    mp = m - c[None, :]
    U = (S1 - mp * S0[:, None]) / np.sqrt(v)
    V = (S2 - 2 * mp * S1 + mp * mp * S0[:, None]) / v - S0[:, None]
    return normalize(np.concatenate([U.ravel(), V.ravel()]), w, N, mode)


def score(fv, W, bias=None) -> np.ndarray:
    """Linear decision values of a linear classifier on Fisher vectors (the
    paper trains "a classification model with liblinear" on the frame FVs and predicts per frame,
    P:563-564):  s_bc = sum_d W_cd fv_bd + b_c, in double precision (one matmul).
    fv: (batch, 2KD) or (2KD,); W: (n_cls, 2KD); bias: (n_cls,) or None (zero)."""
    fv = _d(fv)
    W = _d(W)
    if W.ndim == 1:
        W = W[None]
    s = np.atleast_2d(fv) @ W.T
    if bias is not None:
        s = s + _d(bias)[None, :]
    return s if fv.ndim == 2 else s[0]


# ------------------------------------------------------------------ GMM EM training (NEXT-3)
# "the GMM components trained beforehand" — standard EM for a diagonal GMM,
# with SPEC's train_gmm floors: variance floor max(abs, rel * global per-dim variance), prior
# floor with renormalisation.  Plain numpy in float64; posteriors from the C oracle above.

def loglik_rows(X, priors, means, variances) -> np.ndarray:
    """Per-descriptor log-likelihood ln sum_j pi_j N(x_i; mu_j, diag var_j) (natural log, including the
    -(D/2) ln 2 pi constant): l_ij = ln pi_j - 1/2 sum_k ln(2 pi var_jk) - 1/2 sum_k (x_ik - mu_jk)^2 / var_jk
    (direct form, reading A2), then max + ln sum exp(l - max) per row (Alg.1 l.6-14's maxPost/sum)."""
    w, m, v, K, D = _gmm(priors, means, variances)
    X = _d(X).reshape(-1, D)
    L = np.empty((X.shape[0], K))
    for j in range(K):
        L[:, j] = (np.log(w[j]) - 0.5 * np.sum(np.log(2.0 * np.pi * v[j]))
                   - 0.5 * np.sum((X - m[j]) ** 2 / v[j], axis=1))
    mx = L.max(axis=1)
    return mx + np.log(np.exp(L - mx[:, None]).sum(axis=1))


def em_step(X, priors, means, variances, var_floor_abs: float = 1e-6, var_floor_rel: float = 1e-4,
            prior_floor: float = 1e-8):
    """One EM iteration.  Returns (priors', means', variances', LL) where LL = sum_i ln p(x_i) under the
    INPUT model.  E-step: gamma (Alg.1 Phase 1).  M-step (two-pass, plain definitions):
      N_j = sum_i gamma_ij;  mu_j = sum_i gamma_ij x_i / N_j;  var_jk = sum_i gamma_ij (x_ik - mu_jk)^2 / N_j
      var_jk <- max(var_jk, max(var_floor_abs, var_floor_rel * var_k(X)))   (var_k(X): biased, all rows)
      pi_j = max(N_j / N, prior_floor), then pi /= sum pi
    A component with N_j == 0 keeps its mean and (floored) variance (reading A20)."""
    w, m, v, K, D = _gmm(priors, means, variances)
    X = _d(X).reshape(-1, D)
    N = X.shape[0]
    g = posteriors(X, w, m, v)
    LL = float(loglik_rows(X, w, m, v).sum())
    Nj = g.sum(axis=0)
    mu = m.copy()
    var = v.copy()
    for j in range(K):
        if Nj[j] > 0:
            mu[j] = (g[:, j:j + 1] * X).sum(axis=0) / Nj[j]
            var[j] = (g[:, j:j + 1] * (X - mu[j]) ** 2).sum(axis=0) / Nj[j]
    gmean = X.sum(axis=0) / N
    gvar = ((X - gmean) ** 2).sum(axis=0) / N
    floor = np.maximum(var_floor_abs, var_floor_rel * gvar)
    var = np.maximum(var, floor[None, :])
    pi = np.maximum(Nj / N, prior_floor)
    pi = pi / pi.sum()
    return pi, mu, var, LL


# ------------------------------------------------------------------ PCA + xy embedding (NEXT-2)
def embed(raw, xy, offsets, wh, pca_mean, pca_basis) -> np.ndarray:
    """P:138 [§3.1]: "by lowering the dimension to m (m<128) with PCA and adding the normalized X and Y
    axis, a descriptor with dimension M=m+2 is generated" (SPEC embed S:201-203):
      row_i = [ basis (d_i - mean) ; x_i / W_b ; y_i / H_b ]   for descriptor i of image b,
    basis (m, 128), no whitening.  float64, (N, m + 2)."""
    raw, xy, wh = _d(raw), _d(xy), _d(wh)
    mean, B = _d(pca_mean), _d(pca_basis)
    off = np.asarray(offsets, dtype=np.int64)
    img = np.repeat(np.arange(len(off) - 1), np.diff(off))
    proj = (raw - mean[None, :]) @ B.T
    return np.concatenate([proj, xy / wh[img]], axis=1)


# ------------------------------------------------------------------ large single sets (C5, EM pool)
# Compositions for sets too large to convert to float64 in one piece.  They add no arithmetic: the
# statistics are sums over descriptors (reading A19), computed block by block with the same C code
# (fixed blocks of `block` rows, the paper's "one copy ... for each block" reduction, Alg.3)
# and summed in block order, so the result does not depend on the thread count.

def _block_ranges(N: int, block: int):
    return [(a, min(a + block, N)) for a in range(0, N, block)]


def stats_blocked(X, priors, means, variances, threshold: float = 0.0, block: int = 50_000,
                  nthreads: int = 0) -> np.ndarray:
    """stats() of one large set (any size, float32 X): [N, S0, S1, S2] about c, summed over fixed row
    blocks in order.  Equal to stats() up to fp64 summation order (tests/test_oracle.py)."""
    w, m, v, K, D = _gmm(priors, means, variances)
    N = X.shape[0]
    chunk = block * max(1, max_threads() if nthreads <= 0 else nthreads)
    total = np.zeros(1 + K * (2 * D + 1))
    for c0 in range(0, N, chunk):
        c1 = min(c0 + chunk, N)
        off = np.array([a for a, _ in _block_ranges(c1 - c0, block)] + [c1 - c0], dtype=np.int64)
        part = stats_batched(X[c0:c1], off, w, m, v, threshold=threshold, nthreads=nthreads)
        for row in part:  # block order
            total += row
    return total


def em_step_blocked(X, priors, means, variances, var_floor_abs: float = 1e-6, var_floor_rel: float = 1e-4,
                    prior_floor: float = 1e-8, block: int = 50_000, workers: int = 0):
    """em_step() for a large float32 set, in two passes over fixed row blocks (same definitions, each
    block's partial sums added in block order):
      pass 1: N_j = sum gamma_ij, sum_i gamma_ij x_i, sum_i x_i, LL = sum_i ln p(x_i)
      pass 2: sum_i gamma_ij (x_ik - mu_jk)^2 and sum_i (x_ik - mean_k)^2 about the pass-1 means.
    Posteriors come from the C oracle (fvo_posteriors) per block; blocks run on a thread pool (the C
    call and numpy release the GIL) and are combined in block order."""
    from concurrent.futures import ThreadPoolExecutor

    w, m, v, K, D = _gmm(priors, means, variances)
    N = X.shape[0]
    ranges = _block_ranges(N, block)
    workers = workers or max_threads()

    def p1(r):
        Xb = _d(X[r[0]:r[1]])
        g = posteriors(Xb, w, m, v)
        return g.sum(0), g.T @ Xb, Xb.sum(0), float(loglik_rows(Xb, w, m, v).sum())

    with ThreadPoolExecutor(max_workers=workers) as ex:
        parts = list(ex.map(p1, ranges))
    Nj = np.zeros(K); Sx = np.zeros((K, D)); xs = np.zeros(D); LL = 0.0
    for a, b, c, d in parts:
        Nj += a; Sx += b; xs += c; LL += d
    mu = m.copy()
    nz = Nj > 0
    mu[nz] = Sx[nz] / Nj[nz, None]
    gmean = xs / N

    def p2(r):
        Xb = _d(X[r[0]:r[1]])
        g = posteriors(Xb, w, m, v)
        sv = np.empty((K, D))
        for j in range(K):
            sv[j] = (g[:, j:j + 1] * (Xb - mu[j]) ** 2).sum(axis=0)
        return sv, ((Xb - gmean) ** 2).sum(axis=0)

    with ThreadPoolExecutor(max_workers=workers) as ex:
        parts = list(ex.map(p2, ranges))
    Sv = np.zeros((K, D)); gv = np.zeros(D)
    for a, b in parts:
        Sv += a; gv += b
    var = v.copy()
    var[nz] = Sv[nz] / Nj[nz, None]
    floor = np.maximum(var_floor_abs, var_floor_rel * gv / N)
    var = np.maximum(var, floor[None, :])
    pi = np.maximum(Nj / N, prior_floor)
    pi = pi / pi.sum()
    return pi, mu, var, LL
