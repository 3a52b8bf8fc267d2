"""GPU parity of the fused linear scoring (the paper's monitoring application
scores every frame's FV with a liblinear model) against oracle.score on the fp64
oracle's FVs.  Tolerance: the FV is within 1e-4 relative L2 of the oracle (north_star), so by
Cauchy-Schwarz |s_gpu - s_oracle| <= 1e-4 ||W_c|| ||fv|| (= ||W_c|| for unit-norm FVs); the test uses
that bound.  The fused dot must also agree with scoring the FV the same call returns (to fp32
summation error, 1e-5 ||W_c||)."""
import numpy as np
import pytest
import torch

import fvgen
import oracle

pytestmark = pytest.mark.gpu

FV_RTOL = 1e-4


@pytest.fixture(scope="module")
def fv():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1604_03498_b200 as m
    return m


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def classifier(n_cls, dim, seed):
    rng = np.random.default_rng(seed)
    W = rng.standard_normal((n_cls, dim)).astype(np.float32)
    b = rng.uniform(-1, 1, n_cls).astype(np.float32)
    return W, b


def check_scores(s_gpu, F_ref, W, b, mode=oracle.NORM_IMPROVED):
    ref = oracle.score(F_ref, W, b)
    wn = np.linalg.norm(W.astype(np.float64), axis=1)[None, :]
    fn = np.linalg.norm(F_ref, axis=1)[:, None]
    err = np.abs(s_gpu.astype(np.float64) - ref)
    bound = FV_RTOL * wn * np.maximum(fn, 1e-30) + 1e-6
    assert np.all(err <= bound), f"max err/bound {np.max(err / bound)}"


@pytest.mark.parametrize("tau", [0.0, 1e-6])
@pytest.mark.parametrize("mode", [oracle.NORM_IMPROVED, oracle.NORM_POWER_L2, oracle.NORM_NONE])
def test_scores_match_oracle_ragged_batch(fv, tau, mode):
    K, D = 256, 64
    gmm_np = fvgen.make_gmm(K, D, seed=1604)
    X, off = fvgen.make_batch(gmm_np, [700, 0, 129, 2000, 1, 385], seed_base=4100)
    W, b = classifier(3, 2 * K * D, seed=4200)
    gmm = fv.GMM(*gmm_np)
    s, F = fv.encode_scored_batched(dev(X), dev(off), gmm, dev(W), dev(b), threshold=tau, mode=mode, return_fv=True)
    s, F = s.cpu().numpy(), F.cpu().numpy()
    F_ref = oracle.encode_batched(X, off, *gmm_np, threshold=tau, mode=mode)
    check_scores(s, F_ref, W, b, mode)
    # the fused dot equals scoring the FV this call returned
    own = oracle.score(F.astype(np.float64), W, b)
    wn = np.linalg.norm(W.astype(np.float64), axis=1)[None, :] * np.maximum(np.linalg.norm(F, axis=1)[:, None], 1e-30)
    assert np.all(np.abs(s - own) <= 1e-5 * wn + 1e-6)
    # empty image scores exactly the bias
    np.testing.assert_array_equal(s[1], b)
    # the scores-only call (FVs never written) is bitwise identical
    s2 = fv.encode_scored_batched(dev(X), dev(off), gmm, dev(W), dev(b), threshold=tau, mode=mode).cpu().numpy()
    np.testing.assert_array_equal(s2, s)
    # and the FV equals the plain encode's
    F3 = fv.encode_batched(dev(X), dev(off), gmm, threshold=tau, mode=mode).cpu().numpy()
    np.testing.assert_array_equal(F3, F)


def test_scores_wide_family_max_classes_and_no_bias(fv):
    K, D = 320, 96  # wide kernel, finalize grid z = 2
    gmm_np = fvgen.make_gmm(K, D, seed=1605)
    X, off = fvgen.make_batch(gmm_np, [900, 257, 64], seed_base=4300)
    W, _ = classifier(fv.MAX_CLASSES, 2 * K * D, seed=4400)
    gmm = fv.GMM(*gmm_np)
    s = fv.encode_scored_batched(dev(X), dev(off), gmm, dev(W), None, threshold=1e-6).cpu().numpy()
    F_ref = oracle.encode_batched(X, off, *gmm_np, threshold=1e-6)
    check_scores(s, F_ref, W, np.zeros(fv.MAX_CLASSES, np.float32))


def test_scores_c4_frames_and_host_pipeline(fv):
    """C4-shaped frames (5000 descriptors, K=256, D=64, tau=1e-6): device and host entry points against
    the oracle; the host pipeline (chunked) agrees with the device call to rounding."""
    K, D = 256, 64
    gmm_np = fvgen.make_gmm(K, D, seed=1604)
    X, off = fvgen.make_batch(gmm_np, [5000] * 6, seed_base=1604 + 20000)
    W, b = classifier(2, 2 * K * D, seed=4500)
    gmm = fv.GMM(*gmm_np)
    s_dev = fv.encode_scored_batched(dev(X), dev(off), gmm, dev(W), dev(b), threshold=1e-6).cpu().numpy()
    s_host = fv.encode_scored_batched_host(torch.from_numpy(X).pin_memory(), torch.from_numpy(off), gmm, dev(W),
                                           dev(b), threshold=1e-6).numpy()
    F_ref = oracle.encode_batched(X, off, *gmm_np, threshold=1e-6)
    check_scores(s_dev, F_ref, W, b)
    check_scores(s_host, F_ref, W, b)
    np.testing.assert_allclose(s_host, s_dev, rtol=0, atol=1e-5 * np.linalg.norm(W, axis=1).max())


def test_scores_self_similarity(fv):
    """Classifier rows = the oracle's own FVs: the diagonal scores are ||fv||^2 = 1 up to the FV error."""
    K, D = 64, 32
    gmm_np = fvgen.make_gmm(K, D, seed=77)
    X, off = fvgen.make_batch(gmm_np, [400, 1500, 900], seed_base=78)
    F_ref = oracle.encode_batched(X, off, *gmm_np)
    gmm = fv.GMM(*gmm_np)
    s = fv.encode_scored_batched(dev(X), dev(off), gmm, dev(F_ref.astype(np.float32))).cpu().numpy()
    np.testing.assert_allclose(np.diag(s), 1.0, atol=2e-4)


@pytest.mark.parametrize("n_cls", [1, 32])
@pytest.mark.parametrize("tau,mode", [(0.0, oracle.NORM_IMPROVED), (1e-6, oracle.NORM_IMPROVED),
                                      (1e-6, oracle.NORM_POWER_L2), (1e-6, oracle.NORM_NONE)])
def test_single_frame_scores_latency_path(fv, n_cls, tau, mode):
    """One monitoring frame (5,000 descriptors, the real-time use of P:563-564): the scores come out of
    the single-kernel latency path (the finalize and the dot products inside k_stats; NORM_NONE stays on
    the two-kernel path) within the Cauchy-Schwarz bound of the oracle; the returned FV is bitwise the
    plain encode's; a scores-only call (no FV written) gives the same scores bitwise."""
    K, D = 256, 64
    gmm_np = fvgen.make_gmm(K, D, seed=1604)
    X, off = fvgen.make_batch(gmm_np, [5000], seed_base=4700 + n_cls)
    W, b = classifier(n_cls, 2 * K * D, seed=4800 + n_cls)
    gmm = fv.GMM(*gmm_np)
    s, F = fv.encode_scored_batched(dev(X), dev(off), gmm, dev(W), dev(b), threshold=tau, mode=mode, return_fv=True)
    s, F = s.cpu().numpy(), F.cpu().numpy()
    F_ref = oracle.encode_batched(X, off, *gmm_np, threshold=tau, mode=mode)
    check_scores(s, F_ref, W, b, mode)
    F2 = fv.encode_batched(dev(X), dev(off), gmm, threshold=tau, mode=mode).cpu().numpy()
    np.testing.assert_array_equal(F2, F)
    s2 = fv.encode_scored_batched(dev(X), dev(off), gmm, dev(W), dev(b), threshold=tau, mode=mode).cpu().numpy()
    np.testing.assert_array_equal(s2, s)
