"""Randomised GPU parity sweep (seeded, reproducible): many (K, D, image-size mix, tau, normalisation,
sigma convention) combinations across both tile families, each against the fp64 oracle with the
north_star tolerances (FV 1e-4 relative L2; empty images all-zero; every FV finite).  Complements the
hand-picked cases in test_gpu_parity.py / test_gpu_wide.py with shapes nobody chose on purpose."""
import numpy as np
import pytest
import torch

import fvgen
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fv():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1604_03498_b200 as m
    return m


def _case(seed):
    rng = np.random.default_rng(seed)
    K = int(rng.choice([1, 2, 7, 16, 31, 64, 100, 128, 129, 200, 255, 256, 257, 384, 511, 512]))
    D = int(4 * rng.integers(1, 33))                      # 4 .. 128, multiples of 4
    counts = [int(c) for c in rng.choice([0, 1, 17, 127, 128, 129, 300, 1000, 2500], size=int(rng.integers(1, 5)))]
    if sum(counts) == 0:
        counts[0] = 64
    tau = float(rng.choice([0.0, 1e-6, 1e-3]))
    mode = int(rng.choice([0, 1, 2]))
    stddev = bool(rng.integers(0, 2))
    return K, D, counts, tau, mode, stddev


@pytest.mark.parametrize("seed", list(range(64)))
def test_random_shapes_match_oracle(fv, seed):
    K, D, counts, tau, mode, stddev = _case(7000 + seed)
    pi, mu, var = fvgen.make_gmm(K, D, seed=7100 + seed)
    X, off = fvgen.make_batch((pi, mu, var), counts, seed_base=7200 + 10 * seed)
    sg = np.sqrt(var).astype(np.float32) if stddev else var
    gmm = fv.GMM(pi, mu, sg, stddev=stddev)
    out = fv.encode_batched(torch.from_numpy(X).cuda(), torch.from_numpy(off).cuda(), gmm, threshold=tau,
                            mode=mode).cpu().numpy()
    ref = oracle.encode_batched(X, off, pi, mu, var, threshold=tau, mode=mode)
    assert np.all(np.isfinite(out))
    for b, n in enumerate(counts):
        if n == 0:
            assert np.all(out[b] == 0), f"empty image {b} not zero"
            continue
        nr = np.linalg.norm(ref[b])
        err = np.linalg.norm(out[b] - ref[b]) / (nr if nr > 0 else 1.0)
        assert err <= 1e-4, f"K={K} D={D} counts={counts} tau={tau} mode={mode} stddev={stddev} image {b}: {err:.2e}"


@pytest.mark.parametrize("seed", list(range(12)))
def test_random_stats_shards_and_scores(fv, seed):
    """Random shapes through the split path (statistics of two descriptor shards summed, then finalize)
    and the fused scoring, against the oracle on the whole set."""
    K, D, counts, tau, mode, _ = _case(8000 + seed)
    pi, mu, var = fvgen.make_gmm(K, D, seed=8100 + seed)
    n = max(2, sum(counts))
    X = fvgen.make_descriptors((pi, mu, var), n, seed=8200 + seed)
    gmm = fv.GMM(pi, mu, var)
    cut = n // 3
    s = sum(fv.stats_batched(torch.from_numpy(np.ascontiguousarray(part)).cuda(),
                             torch.tensor([0, part.shape[0]], dtype=torch.int64, device="cuda"), gmm, threshold=tau)
            for part in (X[:cut], X[cut:]))
    out = fv.finalize(s, gmm, mode=mode).cpu().numpy()[0]
    ref = oracle.encode(X, pi, mu, var, threshold=tau, mode=mode)
    assert np.linalg.norm(out - ref) / np.linalg.norm(ref) <= 1e-4
    W = np.random.default_rng(8300 + seed).standard_normal((3, 2 * K * D)).astype(np.float32)
    sc = fv.encode_scored_batched(torch.from_numpy(X).cuda(), torch.tensor([0, n], dtype=torch.int64, device="cuda"),
                                  gmm, torch.from_numpy(W).cuda(), threshold=tau, mode=mode).cpu().numpy()[0]
    sref = oracle.score(ref, W)
    assert np.all(np.abs(sc - sref) <= 1e-4 * np.linalg.norm(W, axis=1) * np.linalg.norm(ref) + 1e-6)


@pytest.mark.parametrize("seed", list(range(8)))
def test_random_em_steps(fv, seed):
    """Random GMM sizes: one EM step against the oracle (priors 1e-5, log-likelihood 2e-5 per
    descriptor)."""
    rng = np.random.default_rng(9000 + seed)
    K = int(rng.choice([1, 3, 16, 64, 130, 256, 300]))
    D = int(4 * rng.integers(1, 33))
    N = int(rng.choice([500, 2000, 5000]))
    g = fvgen.make_gmm(K, D, seed=9100 + seed)
    X = fvgen.make_descriptors(g, N, seed=9200 + seed)
    new, ll = fv.gmm_em_step(torch.from_numpy(X).cuda(), fv.GMM(*g))
    pi_r, mu_r, var_r, ll_r = oracle.em_step(X, *g)
    assert abs(float(ll.item()) - ll_r) <= 2e-5 * N
    assert np.abs(new.weights.cpu().numpy() - pi_r).max() <= 1e-5


@pytest.mark.parametrize("seed", list(range(16)))
def test_random_single_frames_match_oracle(fv, seed):
    """Random single frames through fv_encode on the latency path — sizes spanning the fused-finalize
    window (one tile per cluster, a CTA per finalize block) and its edges, narrow K / D, every mode, tau
    and sigma convention — against the oracle; a repeat on the same workspace is bitwise equal."""
    rng = np.random.default_rng(9000 + seed)
    K = int(rng.choice([16, 32, 64, 100, 128, 129, 200, 256]))
    D = int(4 * rng.integers(1, 17))                      # 4 .. 64
    N = int(rng.choice([1, 127, 128, 1000, 4096, 4097, 5000, 6400, 8191, 9472, 9473, 12000]))
    tau = float(rng.choice([0.0, 1e-6]))
    mode = int(rng.choice([0, 1, 2]))
    stddev = bool(rng.integers(0, 2))
    pi, mu, var = fvgen.make_gmm(K, D, seed=9100 + seed)
    X = fvgen.make_descriptors((pi, mu, var), N, seed=9200 + seed)
    gmm = fv.GMM(pi, mu, np.sqrt(var).astype(np.float32) if stddev else var, stddev=stddev)
    ws = fv.Workspace()
    Xd = torch.from_numpy(X).cuda()
    a = fv.encode(Xd, gmm, threshold=tau, mode=mode, ws=ws).cpu().numpy()
    b = fv.encode(Xd, gmm, threshold=tau, mode=mode, ws=ws, prepared=True).cpu().numpy()
    assert np.array_equal(a, b)
    ref = oracle.encode(X, pi, mu, var, threshold=tau, mode=mode)
    nr = np.linalg.norm(ref)
    err = np.linalg.norm(a - ref) / (nr if nr > 0 else 1.0)
    assert np.all(np.isfinite(a)) and err <= 1e-4, f"K={K} D={D} N={N} tau={tau} mode={mode} sd={stddev}: {err:.2e}"
