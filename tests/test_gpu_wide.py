"""GPU parity of the wide tile family (64 < D <= 128, K <= 512: k_stats_w) against the fp64 oracle,
with the tolerances of test_gpu_parity.py, plus the C5 configuration (one 10M x 128 set, K = 512) at
full size through the descriptor-sharded split path, checked by properties that hold at any size."""
import numpy as np
import pytest
import torch

import fvgen
import oracle

pytestmark = pytest.mark.gpu

GAMMA_ATOL = 1e-5
FV_RTOL = 1e-4
TAU = 1e-6


@pytest.fixture(scope="module")
def fv():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1604_03498_b200 as m
    return m


def rel_l2(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def case(K, D, N, seed=1605):
    gmm = fvgen.make_gmm(K, D, seed=seed)
    return gmm, fvgen.make_descriptors(gmm, N, seed=seed + 1)


@pytest.mark.parametrize("K,D,N", [(512, 128, 300), (64, 100, 257)])
def test_wide_raw_loglik_matches_oracle_up_to_constant(fv, K, D, N):
    gmm_np, X = case(K, D, N)
    L = fv.posteriors(dev(X), fv.GMM(*gmm_np), raw_loglik=True).cpu().numpy().astype(np.float64)
    pi, mu, var = (a.astype(np.float64) for a in gmm_np)
    ll = (np.log(pi)[None] - 0.5 * np.log(var).sum(1)[None]
          - 0.5 * (((X.astype(np.float64)[:, None, :] - mu[None]) ** 2) / var[None]).sum(2)) / np.log(2.0)
    d = L - ll
    dev_ = np.abs(d - np.median(d)) / (1e-3 + 1e-5 * np.abs(ll))
    assert dev_.max() < 1.0


@pytest.mark.parametrize("K,D,N", [(512, 128, 2000), (64, 128, 300), (100, 100, 257), (8, 68, 129), (1, 128, 40),
                                   (200, 96, 513)])
def test_wide_posteriors_exact(fv, K, D, N):
    gmm_np, X = case(K, D, N)
    g = fv.posteriors(dev(X), fv.GMM(*gmm_np)).cpu().numpy()
    ref = oracle.posteriors(X, *gmm_np)
    err = np.abs(g - ref)
    assert err.max() <= GAMMA_ATOL, f"max |gamma err| {err.max()}"
    np.testing.assert_allclose(g.sum(1), 1.0, atol=1e-4)


def test_wide_posteriors_thresholded(fv):
    gmm_np, X = case(512, 128, 2000)
    g = fv.posteriors(dev(X), fv.GMM(*gmm_np), threshold=TAU).cpu().numpy().astype(np.float64)
    ref = oracle.posteriors(X, *gmm_np)
    refz = np.where(ref > TAU, ref, 0.0)
    band = np.abs(ref - TAU) <= 1e-4 * TAU + 2e-9  # reading A16
    assert np.array_equal((g > 0)[~band], (refz > 0)[~band])
    assert np.abs(g - refz)[~band].max() <= GAMMA_ATOL


@pytest.mark.parametrize("K,D,N", [(512, 128, 3000), (64, 128, 1000), (300, 96, 777), (1, 128, 10), (512, 128, 129),
                                   (128, 72, 2500)])
@pytest.mark.parametrize("tau", [0.0, TAU])
def test_wide_encode_parity(fv, K, D, N, tau):
    gmm_np, X = case(K, D, N)
    out = fv.encode(dev(X), fv.GMM(*gmm_np), threshold=tau).cpu().numpy()
    ref = oracle.encode(X, *gmm_np, threshold=tau)
    assert rel_l2(out, ref) <= FV_RTOL
    assert abs(np.linalg.norm(out) - 1.0) < 1e-5


@pytest.mark.parametrize("mode", [1, 2])
def test_wide_encode_modes(fv, mode):
    gmm_np, X = case(512, 128, 1500)
    out = fv.encode(dev(X), fv.GMM(*gmm_np), threshold=TAU, mode=mode).cpu().numpy()
    assert rel_l2(out, oracle.encode(X, *gmm_np, threshold=TAU, mode=mode)) <= FV_RTOL


def test_wide_batched_ragged_with_empty_images(fv):
    gmm_np = fvgen.make_gmm(512, 128, seed=1605)
    counts = [0, 1, 127, 128, 129, 2100, 0, 300, 0]
    X, off = fvgen.make_batch(gmm_np, counts, seed_base=77)
    gmm = fv.GMM(*gmm_np)
    out = fv.encode_batched(dev(X), dev(off), gmm, threshold=TAU).cpu().numpy()
    again = fv.encode_batched(dev(X), dev(off), gmm, threshold=TAU).cpu().numpy()
    assert np.array_equal(out, again)
    ref = oracle.encode_batched(X, off, *gmm_np, threshold=TAU)
    for b, n in enumerate(counts):
        if n == 0:
            assert np.all(out[b] == 0)
        else:
            assert rel_l2(out[b], ref[b]) <= FV_RTOL, (b, n)


def test_wide_stats_finalize_and_shard_additivity(fv):
    """The C5 split path at a small size: fp64 statistics vs the oracle, finalize == encode, and the
    sum of two shards' statistics (the all-reduce) encodes the whole set."""
    gmm_np, X = case(512, 128, 4001)
    gmm = fv.GMM(*gmm_np)
    st = fv.stats_batched(dev(X), dev(np.array([0, 4001])), gmm, threshold=TAU)
    ref = oracle.stats(X, *gmm_np, threshold=TAU)
    s = st.cpu().numpy()[0]
    K = 512
    assert s[0] == 4001
    assert rel_l2(s[1:1 + K], ref[1:1 + K]) < 1e-5
    assert rel_l2(s[1 + K:], ref[1 + K:]) < 1e-5
    enc = fv.encode(dev(X), gmm, threshold=TAU).cpu().numpy()
    assert rel_l2(fv.finalize(st, gmm).cpu().numpy()[0], enc) < 1e-6
    halves = [fv.stats_batched(dev(X[a:b]), dev(np.array([0, b - a])), gmm, threshold=TAU) for a, b in
              [(0, 2000), (2000, 4001)]]
    out = fv.finalize(halves[0] + halves[1], gmm).cpu().numpy()[0]
    assert rel_l2(out, oracle.encode(X, *gmm_np, threshold=TAU)) <= FV_RTOL


@pytest.mark.slow
def test_c5_full_size_stats_invariants(fv):
    """C5 at full size (10M x 128, K = 512, exact mode) in one stats call (the launch shape the
    descriptor-sharded bench times on one GPU).  Invariants that hold at any size, from the
    definition of the statistics about c (reading A19) and sum_j gamma_ij = 1 (Alg.1 l.6-14):
      sum_j S0_j = N,  sum_j S1_jk = sum_i (x_ik - c_k) (to 1e-5 of sum_i |x_ik - c_k|),
      sum_j S2_jk = sum_i (x_ik - c_k)^2;
    plus a 20k-row sample checked element-wise against the oracle."""
    cfg = fvgen.CONFIGS["C5"]
    K, D, N = cfg["K"], cfg["D"], cfg["counts"][0]
    gmm_np = fvgen.make_gmm(K, D, seed=cfg["seed_gmm"])
    X = fvgen.make_frames(gmm_np, N // 5000, 5000, seed=cfg["seed_data"]).reshape(N, D)
    gmm = fv.GMM(*gmm_np)
    Xd = dev(X)
    st = fv.stats_batched(Xd, dev(np.array([0, N])), gmm).cpu().numpy()[0]
    pi, mu = gmm_np[0].astype(np.float64), gmm_np[1].astype(np.float64)
    c = (pi[:, None] * mu).sum(0) / pi.sum()
    Xc = Xd.double() - torch.from_numpy(c).cuda()
    s1 = Xc.sum(0).cpu().numpy()
    a1 = Xc.abs().sum(0).cpu().numpy()  # scale of the S1 sums (s1 itself nearly cancels)
    s2 = (Xc * Xc).sum(0).cpu().numpy()
    S0 = st[1:1 + K]
    S1 = st[1 + K:1 + K + K * D].reshape(K, D)
    S2 = st[1 + K + K * D:].reshape(K, D)
    assert st[0] == N
    assert abs(S0.sum() - N) / N < 1e-5
    assert np.all(np.abs(S1.sum(0) - s1) <= 1e-5 * a1)
    assert rel_l2(S2.sum(0), s2) < 1e-5
    sample = X[:20000]
    out = fv.encode(dev(sample), gmm).cpu().numpy()
    assert rel_l2(out, oracle.encode(sample, *gmm_np)) <= FV_RTOL
