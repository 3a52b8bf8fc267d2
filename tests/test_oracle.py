"""Pins for the CPU oracle (oracle/) against things other than itself (CPU only, no GPU).

Each test names the PAPER.md passage (P:line) or DESIGN.md reading it pins.  Kinds of pin:
closed forms and hand-derived worked examples (tests/golden/), invariants, special cases reducing to
textbook identities, and an independent 50-digit mpmath brute force that uses Gaussian DENSITIES
(not log-sum-exp) and literal Alg.1 loops.  Chosen so that a dropped term, wrong sign/index or
transposed operand in the oracle fails at least one of them.
"""
import json
import os

import numpy as np
import pytest
from mpmath import mp, mpf

import fvgen
import oracle

HERE = os.path.dirname(os.path.abspath(__file__))


# ---------------------------------------------------------------- independent mpmath brute force
def mp_encode(X, pi, mu, var, tau=0.0, mode=oracle.NORM_IMPROVED):
    """Literal Alg.1 in 50-digit arithmetic with densities: p_ij ∝ pi_j prod_k N(x_ik; mu_jk, var_jk)."""
    mp.dps = 50
    X = [[mpf(float(v)) for v in row] for row in np.asarray(X, dtype=np.float64)]
    pi = [mpf(float(v)) for v in pi]
    mu = [[mpf(float(v)) for v in row] for row in np.asarray(mu, dtype=np.float64)]
    var = [[mpf(float(v)) for v in row] for row in np.asarray(var, dtype=np.float64)]
    K, D, N = len(pi), len(mu[0]), len(X)
    G = []
    for x in X:
        dens = []
        for j in range(K):
            p = pi[j]
            for k in range(D):
                p *= mp.exp(-(x[k] - mu[j][k]) ** 2 / (2 * var[j][k])) / mp.sqrt(2 * mp.pi * var[j][k])
            dens.append(p)
        s = mp.fsum(dens)
        G.append([d / s for d in dens])
    U = [[mpf(0)] * D for _ in range(K)]
    V = [[mpf(0)] * D for _ in range(K)]
    for i in range(N):
        for j in range(K):
            if tau > 0 and not (G[i][j] > tau):
                continue
            for k in range(D):
                z = (X[i][k] - mu[j][k]) / mp.sqrt(var[j][k])
                U[j][k] += z * G[i][j]
                V[j][k] += (z * z - 1) * G[i][j]
    fv = [U[j][k] for j in range(K) for k in range(D)] + [V[j][k] for j in range(K) for k in range(D)]
    if mode != oracle.NORM_NONE:
        if N == 0:
            fv = [mpf(0)] * len(fv)
        else:
            if mode == oracle.NORM_IMPROVED:
                fv = [fv[t] / (N * mp.sqrt(pi[(t % (K * D)) // D] * (1 if t < K * D else 2)))
                      for t in range(len(fv))]
            fv = [mp.sign(z) * mp.sqrt(abs(z)) for z in fv]
            n = mp.sqrt(mp.fsum(z * z for z in fv))
            if n > 0:
                fv = [z / n for z in fv]
    return (np.array([[float(g) for g in row] for row in G]).reshape(N, K),
            np.array([float(v) for v in fv]))


def tiny_instance(seed, N=None, K=None, D=None):
    rng = np.random.default_rng(seed)
    N = N or int(rng.integers(1, 9))
    K = K or int(rng.integers(1, 5))
    D = D or int(rng.integers(1, 4))
    pi = rng.dirichlet(np.ones(K)).astype(np.float32)
    mu = rng.normal(0, 1, (K, D)).astype(np.float32)
    var = rng.uniform(0.3, 2.0, (K, D)).astype(np.float32)
    X = rng.normal(0, 1.2, (N, D)).astype(np.float32)
    return X, pi, mu, var


# ---------------------------------------------------------------- golden worked examples
def _golden():
    with open(os.path.join(HERE, "golden", "worked_examples.json")) as f:
        return json.load(f)["examples"]


@pytest.mark.parametrize("ex", _golden(), ids=lambda e: e["name"])
def test_golden_worked_examples(ex):
    """Hand-derived closed forms of Alg.1 + reading A9."""
    X = np.array(ex["X"]); pi = np.array(ex["priors"]); mu = np.array(ex["means"]); var = np.array(ex["vars"])
    tau = ex["threshold"]
    g = oracle.posteriors(X, pi, mu, var)
    np.testing.assert_allclose(g, np.array(ex["gamma"], dtype=np.float64), rtol=0, atol=1e-15)
    U, V = oracle.accumulate(X, g, mu, var, tau)
    np.testing.assert_allclose(U, np.array(ex["U_raw"]), rtol=0, atol=1e-15)
    np.testing.assert_allclose(V, np.array(ex["V_raw"]), rtol=0, atol=1e-15)
    if "fv_improved" in ex:
        fv = oracle.encode(X, pi, mu, var, tau, oracle.NORM_IMPROVED)
        np.testing.assert_allclose(fv, np.array(ex["fv_improved"]), rtol=0, atol=1e-15)


# ---------------------------------------------------------------- posteriors (Alg.1 l.2-15)
def test_single_gaussian_posterior_is_one():
    """K=1 => gamma == 1 exactly (Alg.1 l.12-14 divides e^0 by itself)."""
    X, pi, mu, var = tiny_instance(1, N=7, K=1, D=3)
    X = X * 100  # far from the mean: still exactly 1
    assert np.all(oracle.posteriors(X, pi, mu, var) == 1.0)


def test_posterior_ratio_closed_form_pins_logdet_and_prior():
    """K=2, same mean, x = mu: gamma1/gamma2 = (pi1/pi2) prod_k sqrt(var2k/var1k).
    Pins the -1/2 sum ln var term, the ln pi term and reading A1 (sigmas are variances): with
    std-devs the ratio would be prod var2/var1 instead."""
    pi = np.array([0.3, 0.7]); mu = np.array([[0.2, -1.0, 0.5]] * 2)
    var = np.array([[0.5, 2.0, 1.5], [1.1, 0.4, 3.0]])
    g = oracle.posteriors(mu[:1], pi, mu, var)[0]
    expect = (0.3 / 0.7) * np.prod(np.sqrt(var[1] / var[0]))
    assert g[0] / g[1] == pytest.approx(expect, rel=1e-14)


def test_posterior_symmetry_half():
    """Equal priors/variances, x equidistant from both means => 1/2."""
    rng = np.random.default_rng(3)
    D = 5
    a = rng.normal(size=D); b = rng.normal(size=D)
    var = np.ones((2, D)) * 0.7
    g = oracle.posteriors(((a + b) / 2)[None], [0.5, 0.5], np.stack([a, b]), var)
    np.testing.assert_allclose(g, 0.5, atol=1e-15)


def test_posteriors_match_mpmath_density_bruteforce():
    """Tiny instances (N<=8, K<=4, D<=3): log-sum-exp oracle == 50-digit density computation."""
    for seed in range(25):
        X, pi, mu, var = tiny_instance(100 + seed)
        g_ref, _ = mp_encode(X, pi, mu, var)
        g = oracle.posteriors(X, pi, mu, var)
        np.testing.assert_allclose(g, g_ref, rtol=1e-12, atol=1e-15)


def test_posterior_invariants_rowsum_argmax_permutations():
    """Row-stochastic, argmax of density, Gaussian permutation -> column permutation,
    descriptor permutation -> row permutation (north_star)."""
    gmm = fvgen.make_gmm(16, 8, seed=5)
    X = fvgen.make_descriptors(gmm, 300, seed=6)
    g = oracle.posteriors(X, *gmm)
    np.testing.assert_allclose(g.sum(1), 1.0, atol=1e-12)
    assert np.all(g >= 0) and np.all(g <= 1)
    # argmax against an independent numpy log-density
    pi, mu, var = (a.astype(np.float64) for a in gmm)
    ll = np.log(pi)[None] - 0.5 * np.log(var).sum(1)[None] - 0.5 * (
        ((X.astype(np.float64)[:, None, :] - mu[None]) ** 2) / var[None]).sum(2)
    assert np.array_equal(np.argmax(g, 1), np.argmax(ll, 1))
    perm = np.random.default_rng(0).permutation(16)
    g2 = oracle.posteriors(X, gmm[0][perm], gmm[1][perm], gmm[2][perm])
    np.testing.assert_allclose(g2, g[:, perm], rtol=1e-13, atol=1e-300)
    rp = np.random.default_rng(1).permutation(300)
    np.testing.assert_array_equal(oracle.posteriors(X[rp], *gmm), g[rp])


def test_posterior_shift_stability_far_descriptor():
    """A descriptor very far from every mean (huge negative log-likelihoods) still yields a valid row:
    the maxPost subtraction (Alg.1 l.9) keeps exp from underflowing to 0/0."""
    gmm = fvgen.make_gmm(8, 4, seed=9)
    X = np.full((1, 4), 50.0, dtype=np.float32)
    g = oracle.posteriors(X, *gmm)
    assert np.all(np.isfinite(g)) and g.sum() == pytest.approx(1.0, abs=1e-12)


# ---------------------------------------------------------------- accumulation (Alg.1 l.16-26)
def test_accumulate_matches_mpmath_literal_loops_and_encode():
    """Tiny instances: raw U,V and normalised FV vs the 50-digit literal Alg.1."""
    for seed in range(20):
        X, pi, mu, var = tiny_instance(200 + seed)
        for tau in (0.0, 0.05):
            _, fv_raw = mp_encode(X, pi, mu, var, tau, oracle.NORM_NONE)
            g = oracle.posteriors(X, pi, mu, var)
            U, V = oracle.accumulate(X, g, mu, var, tau)
            np.testing.assert_allclose(np.concatenate([U.ravel(), V.ravel()]), fv_raw, rtol=1e-11, atol=1e-13)
            for mode in (oracle.NORM_IMPROVED, oracle.NORM_POWER_L2):
                _, fv_ref = mp_encode(X, pi, mu, var, tau, mode)
                fv = oracle.encode(X, pi, mu, var, tau, mode)
                np.testing.assert_allclose(fv, fv_ref, rtol=1e-10, atol=1e-12)


def test_single_gaussian_moment_identity():
    """K=1 (gamma=1): U_k = N(xbar_k - mu_k)/sd_k, V_k = N[(s2_k + (xbar_k - mu_k)^2)/var_k - 1] with s2
    the biased sample variance — a textbook moment identity, independent of Alg.1's loop form."""
    rng = np.random.default_rng(11)
    N, D = 500, 6
    X = rng.normal(0.3, 1.7, (N, D))
    mu = rng.normal(size=(1, D)); var = rng.uniform(0.5, 2, (1, D))
    U, V = oracle.accumulate(X, np.ones((N, 1)), mu, var)
    xbar = X.mean(0); s2 = X.var(0)
    np.testing.assert_allclose(U[0], N * (xbar - mu[0]) / np.sqrt(var[0]), rtol=1e-10)
    np.testing.assert_allclose(V[0], N * ((s2 + (xbar - mu[0]) ** 2) / var[0] - 1), rtol=1e-10)


def test_descriptor_at_mean_gives_zero_U_and_minus_gamma_V():
    """x = mu_j => U_j = 0, V_j = -gamma_j per dimension."""
    gmm = fvgen.make_gmm(4, 5, seed=12)
    X = gmm[1][2:3].astype(np.float64)
    g = oracle.posteriors(X, *gmm)
    U, V = oracle.accumulate(X, g, gmm[1], gmm[2])
    np.testing.assert_allclose(U[2], 0.0, atol=1e-15)
    np.testing.assert_allclose(V[2], -g[0, 2], rtol=1e-14)


def test_threshold_semantics_linearity_and_monotonicity():
    """Alg.1 l.18 strict '>' (A5); linearity in gamma; raising tau only removes pairs."""
    gmm = fvgen.make_gmm(16, 8, seed=13)
    X = fvgen.make_descriptors(gmm, 200, seed=14)
    g = oracle.posteriors(X, *gmm)
    tau = 1e-3
    U_t, V_t = oracle.accumulate(X, g, gmm[1], gmm[2], tau)
    gz = np.where(g > tau, g, 0.0)
    U_z, V_z = oracle.accumulate(X, gz, gmm[1], gmm[2], 0.0)
    np.testing.assert_allclose(U_t, U_z, rtol=1e-13, atol=1e-14)
    np.testing.assert_allclose(V_t, V_z, rtol=1e-13, atol=1e-14)
    U2, V2 = oracle.accumulate(X, 2 * gz, gmm[1], gmm[2], 0.0)
    np.testing.assert_allclose(U2, 2 * U_z, rtol=1e-14, atol=1e-14)
    # all gamma <= tau  =>  zeros
    U0, V0 = oracle.accumulate(X, g, gmm[1], gmm[2], 0.9999999)
    cut = (g > 0.9999999)
    assert np.all(U0[~cut.any(0)] == 0) and np.all(V0[~cut.any(0)] == 0)


def test_permutation_invariances_of_fv():
    """Descriptor permutation leaves the FV unchanged; Gaussian permutation permutes U/V row blocks
    (north_star)."""
    gmm = fvgen.make_gmm(8, 4, seed=15)
    X = fvgen.make_descriptors(gmm, 777, seed=16)
    fv = oracle.encode(X, *gmm)
    rp = np.random.default_rng(2).permutation(777)
    np.testing.assert_allclose(oracle.encode(X[rp], *gmm), fv, rtol=1e-12, atol=1e-14)
    gp = np.random.default_rng(3).permutation(8)
    fvp = oracle.encode(X, gmm[0][gp], gmm[1][gp], gmm[2][gp])
    K, D = 8, 4
    U = fv[:K * D].reshape(K, D); V = fv[K * D:].reshape(K, D)
    np.testing.assert_allclose(fvp, np.concatenate([U[gp].ravel(), V[gp].ravel()]), rtol=1e-12, atol=1e-14)


# ---------------------------------------------------------------- normalisation (reading A9)
def test_normalisation_unit_norm_zero_and_duplication():
    """||z||=1 unless zero; zero stays zero; X u X gives the same FV (1/N cancels)."""
    gmm = fvgen.make_gmm(8, 6, seed=17)
    X = fvgen.make_descriptors(gmm, 300, seed=18)
    fv = oracle.encode(X, *gmm)
    assert np.linalg.norm(fv) == pytest.approx(1.0, abs=1e-12)
    np.testing.assert_allclose(oracle.encode(np.concatenate([X, X]), *gmm), fv, rtol=1e-11, atol=1e-13)
    z = oracle.normalize(np.zeros(2 * 8 * 6), gmm[0], 10)
    assert np.all(z == 0)
    e = oracle.encode(np.zeros((0, 6), np.float32), *gmm)
    assert np.all(e == 0) and np.all(np.isfinite(e))


def test_normalisation_closed_form_single_descriptor_at_mean():
    """K=1, one descriptor x=mu: U=0, V=-1 => FV = [0..0, -1/sqrt(D)..] (derived from A9)."""
    D = 7
    mu = np.random.default_rng(4).normal(size=(1, D))
    fv = oracle.encode(mu, [0.37], mu, np.ones((1, D)) * 0.4)
    np.testing.assert_allclose(fv[:D], 0.0, atol=1e-15)
    np.testing.assert_allclose(fv[D:], -1 / np.sqrt(D), rtol=1e-14)


def test_improved_prior_scaling_differs_from_power_l2():
    """The per-Gaussian 1/sqrt(pi_j) and the sqrt2 between U and V do not cancel through power+L2
    (reading A9 note): the two modes must differ on a generic instance."""
    gmm = fvgen.make_gmm(4, 3, seed=19)
    X = fvgen.make_descriptors(gmm, 50, seed=20)
    a = oracle.encode(X, *gmm, mode=oracle.NORM_IMPROVED)
    b = oracle.encode(X, *gmm, mode=oracle.NORM_POWER_L2)
    assert np.max(np.abs(a - b)) > 1e-3


# ---------------------------------------------------------------- sufficient statistics (A19)
@pytest.mark.parametrize("tau", [0.0, 1e-6, 1e-2])
def test_stats_reproduce_literal_alg1(tau):
    """fvo_stats (moments about c) + the algebraic centring reproduce fvo_accumulate's literal Alg.1
    sums — two independent code paths (P:179-180 algebra)."""
    gmm = fvgen.make_gmm(16, 8, seed=21)
    X = fvgen.make_descriptors(gmm, 1500, seed=22)
    st = oracle.stats(X, *gmm, threshold=tau)
    assert st[0] == 1500
    for mode in (oracle.NORM_NONE, oracle.NORM_IMPROVED):
        np.testing.assert_allclose(oracle.fv_from_stats(st, *gmm, mode=mode),
                                   oracle.encode(X, *gmm, threshold=tau, mode=mode), rtol=1e-9, atol=1e-11)
    # S0 equals the column sum of the (thresholded) posteriors
    g = oracle.posteriors(X, *gmm)
    g = np.where(g > tau, g, 0.0) if tau > 0 else g
    np.testing.assert_allclose(st[1:17], g.sum(0), rtol=1e-12)


def test_stats_are_additive_over_shards():
    """Descriptor sharding: stats of a union = sum of stats of the parts (the allreduce, §8(e))."""
    gmm = fvgen.make_gmm(8, 4, seed=23)
    X = fvgen.make_descriptors(gmm, 1000, seed=24)
    whole = oracle.stats(X, *gmm, threshold=1e-6)
    parts = sum(oracle.stats(X[a:b], *gmm, threshold=1e-6) for a, b in [(0, 333), (333, 800), (800, 1000)])
    np.testing.assert_allclose(parts, whole, rtol=1e-11, atol=1e-12)


def test_blocked_stats_equal_stats_on_one_set():
    """oracle.stats_blocked (the large-set goldens' writer) = stats() of the whole set: several row
    blocks, several per-call chunks, a ragged last block; exact and tau modes."""
    gmm = fvgen.make_gmm(16, 6, seed=31)
    X = fvgen.make_descriptors(gmm, 5003, seed=32)
    for tau in (0.0, 1e-6):
        whole = oracle.stats(X, *gmm, threshold=tau)
        blocked = oracle.stats_blocked(X, *gmm, threshold=tau, block=257, nthreads=3)
        np.testing.assert_allclose(blocked, whole, rtol=1e-11, atol=1e-11)
        assert blocked[0] == X.shape[0]


def test_blocked_em_step_equals_em_step():
    """oracle.em_step_blocked (two passes over row blocks, thread pool) = em_step() on the same set."""
    gmm = fvgen.make_gmm(6, 5, seed=33)
    X = fvgen.make_descriptors(gmm, 4001, seed=34)
    init = fvgen.make_gmm(6, 5, seed=35)
    a = oracle.em_step(X, *init)
    b = oracle.em_step_blocked(X, *init, block=300, workers=3)
    for x, y in zip(a[:3], b[:3]):
        np.testing.assert_allclose(y, x, rtol=1e-10, atol=1e-12)
    assert abs(a[3] - b[3]) <= 1e-9 * abs(a[3])


def test_batched_equals_per_image_and_thread_invariance():
    gmm = fvgen.make_gmm(8, 4, seed=25)
    X, off = fvgen.make_batch(gmm, [10, 0, 1, 300, 5000], seed_base=26)
    ref = np.stack([oracle.encode(X[off[b]:off[b + 1]], *gmm, 1e-6) for b in range(5)])
    for nt in (1, 3):
        out = oracle.encode_batched(X, off, *gmm, threshold=1e-6, nthreads=nt)
        np.testing.assert_array_equal(out, ref)
    assert np.all(ref[1] == 0)
    sb = oracle.stats_batched(X, off, *gmm, threshold=1e-6, nthreads=2)
    np.testing.assert_array_equal(sb[3], oracle.stats(X[off[3]:off[4]], *gmm, threshold=1e-6))


def test_generator_is_deterministic_and_shaped():
    gmm = fvgen.make_gmm(256, 64)
    assert gmm[0].dtype == np.float32 and gmm[1].shape == (256, 64) and np.all(gmm[2] > 0)
    a = fvgen.make_descriptors(gmm, 1000, 7); b = fvgen.make_descriptors(gmm, 1000, 7)
    assert np.array_equal(a, b) and a.shape == (1000, 64)


# ---------------------------------------------------------------- linear scoring (NEXT-4)
def test_score_closed_form_descriptor_at_mean():
    """K=1, one descriptor at mu: FV = [0..0, -1/sqrt(D)..] (A9), so the all-ones classifier scores
    -sqrt(D) + b and a U-only classifier scores b (closed forms; P:563-564 linear model)."""
    D = 6
    mu = np.random.default_rng(5).normal(size=(1, D))
    fv = oracle.encode(mu, [0.5], mu, np.ones((1, D)) * 0.3)
    W = np.stack([np.ones(2 * D), np.r_[np.ones(D), np.zeros(D)]])
    s = oracle.score(fv, W, [0.25, -1.5])
    np.testing.assert_allclose(s, [-np.sqrt(D) + 0.25, -1.5], rtol=1e-13, atol=1e-13)


def test_score_self_similarity_basis_and_linearity():
    """W = the (unit-norm) FVs themselves gives 1 on the diagonal (A9 unit norm); basis rows pick
    components; the score is linear in W and shifts by b (the plain definition, checked on a batch so
    a transposed W or a dropped bias fails)."""
    gmm = fvgen.make_gmm(8, 4, seed=31)
    X, off = fvgen.make_batch(gmm, [120, 80, 200], seed_base=32)
    F = oracle.encode_batched(X, off, *gmm)
    S = oracle.score(F, F)
    np.testing.assert_allclose(np.diag(S), 1.0, rtol=1e-12)
    assert np.all(np.abs(S - S.T) < 1e-12) and np.all(S <= 1 + 1e-12)
    idx = [0, 5, 2 * 8 * 4 - 1]
    E = np.eye(F.shape[1])[idx]
    np.testing.assert_array_equal(oracle.score(F, E, np.zeros(3)), F[:, idx])
    rng = np.random.default_rng(33)
    W1, W2 = rng.normal(size=(2, F.shape[1])), rng.normal(size=(2, F.shape[1]))
    b = np.array([0.5, -2.0])
    np.testing.assert_allclose(oracle.score(F, 2 * W1 - W2, b), 2 * oracle.score(F, W1) - oracle.score(F, W2) + b,
                               rtol=1e-12, atol=1e-12)
    assert oracle.score(F[1], W1).shape == (2,)


# ---------------------------------------------------------------- GMM EM (NEXT-3)
def test_loglik_matches_scipy_mixture_density():
    """ln p(x) against scipy's multivariate normal log-pdf (diagonal covariance) + logsumexp: a library
    path with its own normalising constants (pins the -(D/2) ln 2 pi, log-det and prior terms)."""
    from scipy.special import logsumexp
    from scipy.stats import multivariate_normal
    gmm = fvgen.make_gmm(5, 4, seed=41)
    X = fvgen.make_descriptors(gmm, 200, seed=42).astype(np.float64)
    pi, mu, var = (a.astype(np.float64) for a in gmm)
    comp = np.stack([np.log(pi[j]) + multivariate_normal(mu[j], np.diag(var[j])).logpdf(X) for j in range(5)], 1)
    np.testing.assert_allclose(oracle.loglik_rows(X, *gmm), logsumexp(comp, axis=1), rtol=1e-12, atol=1e-10)


def test_em_single_component_is_sample_mean_and_variance():
    """K=1: one M-step gives the sample mean and biased sample variance (numpy routines), pi = 1, and
    LL = sum of univariate normal log-pdfs (scipy) under the input model (SPEC train_gmm N=1 example)."""
    from scipy.stats import norm
    rng = np.random.default_rng(43)
    X = rng.normal(size=(500, 3)) * [1.0, 0.5, 2.0] + [0.3, -1.0, 4.0]
    mu0, var0 = np.array([[0.0, 0.0, 1.0]]), np.array([[2.0, 1.0, 3.0]])
    pi, mu, var, LL = oracle.em_step(X, [1.0], mu0, var0)
    np.testing.assert_allclose(pi, [1.0], rtol=0, atol=0)
    np.testing.assert_allclose(mu[0], X.mean(axis=0), rtol=1e-13)
    np.testing.assert_allclose(var[0], X.var(axis=0), rtol=1e-12)
    assert LL == pytest.approx(norm.logpdf(X, mu0[0], np.sqrt(var0[0])).sum(), rel=1e-13)


def test_em_mstep_equals_weighted_moments():
    """M-step = posterior-weighted mean / biased covariance diagonal (np.average, np.cov aweights) and
    pi = mean posterior — library routines on the oracle's own gamma."""
    gmm = fvgen.make_gmm(6, 5, seed=44)
    X = fvgen.make_descriptors(gmm, 800, seed=45).astype(np.float64)
    pi, mu, var, _ = oracle.em_step(X, *gmm, var_floor_abs=0.0, var_floor_rel=0.0, prior_floor=0.0)
    g = oracle.posteriors(X, *gmm)
    for j in range(6):
        np.testing.assert_allclose(mu[j], np.average(X, axis=0, weights=g[:, j]), rtol=1e-11, atol=1e-13)
        np.testing.assert_allclose(var[j], np.diag(np.cov(X.T, aweights=g[:, j], bias=True)), rtol=1e-10)
    np.testing.assert_allclose(pi, g.mean(axis=0), rtol=1e-12)
    assert pi.sum() == pytest.approx(1.0, abs=1e-14)


def test_em_monotone_loglik_and_separated_clusters():
    """EM never decreases the log-likelihood (SPEC: non-decreasing within 1e-8), and two well separated
    clusters are recovered from a perturbed start (means within 0.1 of the true centres)."""
    rng = np.random.default_rng(46)
    c = np.array([[-5.0, 0.0, 2.0], [5.0, 1.0, -2.0]])
    X = np.concatenate([c[0] + rng.normal(size=(400, 3)), c[1] + 0.5 * rng.normal(size=(600, 3))])
    pi, mu, var = np.array([0.5, 0.5]), c + [[1.0, -1.0, 0.5], [-1.0, 0.5, 1.0]], np.ones((2, 3)) * 4.0
    lls = []
    for _ in range(12):
        pi, mu, var, LL = oracle.em_step(X, pi, mu, var)
        lls.append(LL)
    assert all(b >= a - 1e-8 * abs(a) for a, b in zip(lls, lls[1:]))
    assert np.abs(mu - c).max() < 0.1
    np.testing.assert_allclose(pi, [0.4, 0.6], atol=1e-6)


def test_em_floors_and_component_permutation():
    """Variance floor (max(abs, rel * global var)) binds for a component sitting on duplicate points;
    the prior floor keeps a far component's weight at ~1e-8 after renormalisation; permuting the
    components permutes the result."""
    rng = np.random.default_rng(47)
    X = np.concatenate([np.tile([[1.0, 2.0]], (50, 1)), rng.normal(size=(300, 2))])
    mu0 = np.array([[1.0, 2.0], [0.0, 0.0], [1e3, 1e3]])
    var0 = np.array([[1e-4, 1e-4], [1.0, 1.0], [1.0, 1.0]])
    pi, mu, var, _ = oracle.em_step(X, [0.2, 0.7, 0.1], mu0, var0, var_floor_abs=1e-6, var_floor_rel=1e-3)
    gvar = X.var(axis=0)
    np.testing.assert_allclose(var[0], 1e-3 * gvar, rtol=1e-12)
    assert pi[2] == pytest.approx(1e-8 / (1 + 1e-8), rel=1e-6)
    perm = [2, 0, 1]
    pp, mp_, vp, LLp = oracle.em_step(X, np.array([0.2, 0.7, 0.1])[perm], mu0[perm], var0[perm],
                                      var_floor_abs=1e-6, var_floor_rel=1e-3)
    np.testing.assert_allclose(pp, pi[perm], rtol=1e-12)
    np.testing.assert_allclose(mp_, mu[perm], rtol=1e-12)
    np.testing.assert_allclose(vp, var[perm], rtol=1e-12)


# ---------------------------------------------------------------- PCA + xy embedding (NEXT-2)
def test_embed_closed_forms():
    """SPEC embed examples: d = mean -> first m coords zero; keypoint at the image centre -> (0.5, 0.5);
    a full orthonormal basis (m = 128) preserves ||d - mean|| (closed form); basis rows = unit vectors
    pick coordinates of d - mean; the two images use their own sizes."""
    mean, B = fvgen.make_pca(80, seed=3)
    raw = np.stack([mean, mean + 1.0]).astype(np.float32)
    xy = np.array([[160.0, 120.0], [50.0, 100.0]], np.float32)
    off = np.array([0, 1, 2])
    wh = np.array([[320.0, 240.0], [100.0, 400.0]], np.float32)
    E = oracle.embed(raw, xy, off, wh, mean, B)
    assert E.shape == (2, 82)
    np.testing.assert_allclose(E[0, :80], 0.0, atol=1e-12)
    np.testing.assert_allclose(E[0, 80:], [0.5, 0.5]); np.testing.assert_allclose(E[1, 80:], [0.5, 0.25])
    mf, Bf = fvgen.make_pca(128, seed=4)
    d = np.random.default_rng(5).normal(size=(7, 128))
    Ef = oracle.embed(d, np.zeros((7, 2)), [0, 7], [[1.0, 1.0]], mf, Bf)
    np.testing.assert_allclose(np.linalg.norm(Ef[:, :128], axis=1), np.linalg.norm(d - mf, axis=1), rtol=1e-6)
    I = np.eye(128)[[3, 0, 127]]
    Ei = oracle.embed(d, np.zeros((7, 2)), [0, 7], [[1.0, 1.0]], np.zeros(128), I)
    np.testing.assert_array_equal(Ei[:, :3], d[:, [3, 0, 127]])


def test_embed_is_linear_and_generator_is_consistent():
    """Projection is linear (SPEC invariant); the raw generator's descriptors project back to the
    m-dim GMM sample up to the small orthogonal residual."""
    mean, B = fvgen.make_pca(80, seed=6)
    rng = np.random.default_rng(7)
    d1, d2 = rng.normal(size=(2, 5, 128))
    z = np.zeros((5, 2))
    a = 0.3
    np.testing.assert_allclose(oracle.embed(a * d1 + (1 - a) * d2, z, [0, 5], [[1, 1]], mean, B)[:, :80],
                               a * oracle.embed(d1, z, [0, 5], [[1, 1]], mean, B)[:, :80]
                               + (1 - a) * oracle.embed(d2, z, [0, 5], [[1, 1]], mean, B)[:, :80], atol=1e-12)
    gmm = fvgen.make_embedded_gmm(8, 80, seed=8)
    raw, xy, off, wh = fvgen.make_raw_frames(gmm, (mean, B), [300, 200], seed=9)
    E = oracle.embed(raw, xy, off, wh, mean, B)
    assert E.shape == (500, 82) and np.all((E[:, 80:] >= 0) & (E[:, 80:] <= 1))
    assert np.abs(E[:, :80]).max() < 5.0
