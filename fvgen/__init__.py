"""Seeded synthetic inputs for GPU-FV tests and benchmarks (SURVEY.md §8(d) recipe).

This module holds NONE of the method's arithmetic (no log-likelihoods, posteriors, statistics or
normalisation); it only draws GMMs and descriptor sets.  It is the one module both the oracle side
(tests, bench cpu_baseline) and the CUDA side (tests, bench) use.  Everything is float32, row-major,
exactly what the C-ABI consumes; the oracle converts the same float32 values to double.

Recipe (post-PCA-like descriptors, P:138 / P:449):
  per-dimension spread     s_k = 0.5 (k+1)^(-1/2)                      (decaying PCA spectrum)
  priors                   pi ~ Dirichlet(2 * 1_K)
  means                    mu_jk = s_k sqrt(f) N(0,1)                  (f = between-cluster fraction)
  std-devs                 sd_jk = s_k sqrt(1-f) U(0.7, 1.3)           (variances = sd^2 go to the ABI)
  descriptors              c_i ~ Cat(pi), x_i = mu_{c_i} + sd_{c_i} * N(0, I); the first 5 % are
                           replaced by background N(0, diag s^2); then the rows are shuffled.
Acceptance set: f = 0.3.  Stress sets: f = 0.15 ("flat") and "peaked" (sd = s U(0.3, 0.7), mu = s N).
"""
from __future__ import annotations

import numpy as np

SEED_GMM = 1604


def spread(D: int) -> np.ndarray:
    return 0.5 * (np.arange(D, dtype=np.float64) + 1.0) ** -0.5


def make_gmm(K: int, D: int, seed: int = SEED_GMM, f: float = 0.3, kind: str = "acceptance"):
    """Return (priors[K], means[K,D], variances[K,D]) as float32 (variances = sigma^2, reading A1)."""
    rng = np.random.default_rng(seed)
    s = spread(D)
    pi = rng.dirichlet(2.0 * np.ones(K))
    if kind == "peaked":
        mu = s * rng.standard_normal((K, D))
        sd = s * rng.uniform(0.3, 0.7, (K, D))
    else:
        mu = s * np.sqrt(f) * rng.standard_normal((K, D))
        sd = s * np.sqrt(1.0 - f) * rng.uniform(0.7, 1.3, (K, D))
    pi = pi.astype(np.float32)
    # guarantee strictly positive float32 priors (Dirichlet draws can be tiny but never exactly 0)
    pi = np.maximum(pi, np.float32(1e-30))
    return pi, mu.astype(np.float32), (sd * sd).astype(np.float32)


def make_descriptors(gmm, N: int, seed: int, bg_frac: float = 0.05) -> np.ndarray:
    """N x D float32 descriptors drawn from the GMM (+ background), shuffled."""
    pi, mu, var = gmm
    K, D = mu.shape
    rng = np.random.default_rng(seed)
    if N == 0:
        return np.zeros((0, D), dtype=np.float32)
    p = pi.astype(np.float64)
    c = rng.choice(K, size=N, p=p / p.sum())
    sd = np.sqrt(var.astype(np.float64))
    x = mu[c].astype(np.float64) + sd[c] * rng.standard_normal((N, D))
    nb = int(round(bg_frac * N))
    if nb:
        x[:nb] = spread(D) * rng.standard_normal((nb, D))
    rng.shuffle(x, axis=0)
    return x.astype(np.float32)


def make_frames(gmm, frames: int, per_frame: int, seed: int, block: int = 64, bg_frac: float = 0.05,
                start: int = 0, total: int | None = None) -> np.ndarray:
    """Large streams (bench): frames x per_frame descriptors from the same recipe, drawn in float32
    blocks of `block` frames (one seeded generator per block, seeded by the block's first frame).
    Background rows are placed at random positions (each row with probability bg_frac) instead of
    first-then-shuffle; same distribution.

    `start` / `total` select frames [start, start + frames) of a stream of `total` frames (default
    start + frames): the rows are exactly those of make_frames(gmm, total, ...)[start*pf:(start+frames)*pf],
    so the ranks of a sharded run draw disjoint slices of one fixed set whatever the world size."""
    pi, mu, var = gmm
    K, D = mu.shape
    total = start + frames if total is None else int(total)
    assert 0 <= start and start + frames <= total
    cdf = np.cumsum(pi.astype(np.float64))
    cdf /= cdf[-1]
    sd = np.sqrt(var.astype(np.float64)).astype(np.float32)
    s = spread(D).astype(np.float32)
    X = np.empty((frames * per_frame, D), dtype=np.float32)

    def fill(g0):  # independent per block: same result for any thread count or slice
        rng = np.random.default_rng(seed + g0)
        nf = min(block, total - g0)
        n = nf * per_frame
        c = np.minimum(np.searchsorted(cdf, rng.random(n)), K - 1)
        z = rng.standard_normal((n, D), dtype=np.float32)
        bg = rng.random(n) < bg_frac
        a, b = max(g0, start), min(g0 + nf, start + frames)  # overlap with the requested frames
        whole = a == g0 and b == g0 + nf
        xb = X[(a - start) * per_frame:(b - start) * per_frame] if whole else np.empty((n, D), np.float32)
        np.multiply(sd[c], z, out=xb)
        xb += mu[c]
        xb[bg] = s * z[bg]
        if not whole:
            X[(a - start) * per_frame:(b - start) * per_frame] = xb[(a - g0) * per_frame:(b - g0) * per_frame]

    from concurrent.futures import ThreadPoolExecutor
    import os
    if frames == 0:
        return X
    first = (start // block) * block
    with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as ex:
        list(ex.map(fill, range(first, start + frames, block)))
    return X


def voc_counts(B: int, seed: int, mean: int = 20000) -> np.ndarray:
    """C3: ragged per-image descriptor counts round(mean * U(0.75, 1.25))."""
    rng = np.random.default_rng(seed)
    return np.round(mean * rng.uniform(0.75, 1.25, B)).astype(np.int64)


def make_batch(gmm, counts, seed_base: int):
    """Concatenate independently seeded images; returns (X[n_total, D] float32, offsets[B+1] int64)."""
    counts = np.asarray(counts, dtype=np.int64)
    D = gmm[1].shape[1]
    offsets = np.zeros(len(counts) + 1, dtype=np.int64)
    offsets[1:] = np.cumsum(counts)
    X = np.empty((int(offsets[-1]), D), dtype=np.float32)
    for b, n in enumerate(counts):
        X[offsets[b]:offsets[b + 1]] = make_descriptors(gmm, int(n), seed_base + b)
    return X, offsets


# Named configurations from BASELINE.json "configs".
CONFIGS = {
    "C1": dict(K=16, D=64, counts=[1000], seed_gmm=1604, seed_data=1605),
    "C2": dict(K=256, D=64, counts=[5000], seed_gmm=1604, seed_data=1604 + 1000),
    "C2_paper_geometry": dict(K=256, D=64, counts=[17714], seed_gmm=1604, seed_data=1604 + 1000),
    "C3": dict(K=256, D=64, B=256, mean=20000, seed_gmm=1604, seed_data=1604 + 10000),
    "C4": dict(K=256, D=64, frames=4096, per_frame=5000, seed_gmm=1604, seed_data=1604 + 20000),
    "C5": dict(K=512, D=128, counts=[10_000_000], seed_gmm=1605, seed_data=1605 + 1),
}


# ---------------------------------------------------------------- raw SIFT-shaped inputs (NEXT-2)
SIFT_DIM = 128


def make_pca(m: int, seed: int = 1604 + 50, in_dim: int = SIFT_DIM):
    """A PCA model (SPEC embed.PcaModel): mean (in_dim,) nonnegative SIFT-like, basis (m, in_dim) with
    orthonormal rows (QR of a seeded Gaussian matrix, sign-fixed).  float32."""
    rng = np.random.default_rng(seed)
    mean = np.abs(rng.normal(0.05, 0.03, in_dim))
    q, r = np.linalg.qr(rng.standard_normal((in_dim, m)))
    q = q * np.sign(np.diag(r))[None, :]
    return mean.astype(np.float32), np.ascontiguousarray(q.T).astype(np.float32)


def make_embedded_gmm(K: int, m: int, seed: int = SEED_GMM):
    """GMM over the embedded M = m + 2 dims: the first m from the acceptance recipe (make_gmm), the last
    two (normalised x, y in [0, 1]) with means U(0.2, 0.8) and std-devs U(0.15, 0.3)."""
    pi, mu, var = make_gmm(K, m, seed=seed)
    rng = np.random.default_rng(seed + 7)
    mxy = rng.uniform(0.2, 0.8, (K, 2))
    sxy = rng.uniform(0.15, 0.3, (K, 2))
    return (pi, np.concatenate([mu, mxy.astype(np.float32)], 1),
            np.concatenate([var, (sxy * sxy).astype(np.float32)], 1))


def make_raw_frames(gmm_m, pca, counts, seed: int, img_wh=(320, 240), resid: float = 0.01):
    """Raw 128-d descriptors whose PCA projection follows the m-dim GMM `gmm_m` (first m dims of an
    embedded GMM): raw = mean + basis^T y + resid * (noise orthogonal to the basis); keypoints uniform
    over a img_wh image.  Returns (raw (N, 128), xy (N, 2) pixels, offsets (B+1,), wh (B, 2)), float32."""
    mean, basis = pca
    m = basis.shape[0]
    pi, mu, var = gmm_m
    mu, var = mu[:, :m], var[:, :m]
    counts = np.asarray(counts, dtype=np.int64)
    off = np.zeros(len(counts) + 1, dtype=np.int64)
    off[1:] = np.cumsum(counts)
    Y = make_frames((pi, mu, var), 1, int(off[-1]), seed=seed) if off[-1] > 0 else np.zeros((0, m), np.float32)
    rng = np.random.default_rng(seed + 1)
    E = rng.standard_normal((Y.shape[0], basis.shape[1])).astype(np.float32)
    E -= (E @ basis.T) @ basis
    raw = (mean[None, :] + Y @ basis + resid * E).astype(np.float32)
    wh = np.tile(np.asarray(img_wh, np.float32), (len(counts), 1))
    xy = (rng.random((Y.shape[0], 2)) * np.repeat(wh, counts, axis=0)).astype(np.float32)
    return raw, xy, off, wh
