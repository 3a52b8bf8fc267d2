"""Full-size parity of the large single sets against expected values the fp64 oracle wrote
(tests/golden/make_large_golden.py: oracle.stats_blocked / oracle.em_step_blocked over the same seeded
fvgen sets).  Alg.1 l.16-26 as sufficient statistics (reading A19); NEXT-3's EM step
(PAPER.md:141-142).

  C5 (BASELINE configs[4]): 10,000,000 x 128, K = 512, exact — one fv_stats_batched call over the whole
     set (the launch shape bench.py --workload c5 times on one GPU), per-Gaussian S0 / S1 / S2 and the
     finalized FV element-wise against the oracle's.
  5.12 M x 64, K = 256 (the bench's EM pool): statistics in exact and tau = 1e-6 modes, the FV, and one
     EM step.

Before comparing, each test checks it regenerated the golden's input (per-column sums and a row-sample
hash stored with the expected values)."""
import hashlib
import os

import numpy as np
import pytest
import torch

import fvgen
import oracle

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
FV_RTOL = 1e-4          # north_star: normalised FV within 1e-4 relative L2
STATS_RTOL = 1e-5       # S1 / S2 blocks, relative L2 (fp32 chunk sums, fp64 segment reduction)
S0_RTOL = 1e-5          # every Gaussian's S0, relative


@pytest.fixture(scope="module")
def fv():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1604_03498_b200 as m
    return m


def rel_l2(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def load(name):
    path = os.path.join(HERE, "golden", name)
    if not os.path.exists(path):
        pytest.skip(f"{path} missing (python tests/golden/make_large_golden.py)")
    return np.load(path)


def check_same_input(X, Xd, g):
    assert hashlib.sha256(np.ascontiguousarray(X[::9973]).tobytes()).hexdigest() == str(g["sha"])
    np.testing.assert_allclose(Xd.double().sum(0).cpu().numpy(), g["colsum"], rtol=0, atol=1e-6 * X.shape[0])


def compare_stats(st, ref, K, D, label):
    S0, S1, S2 = st[1:1 + K], st[1 + K:1 + K + K * D], st[1 + K + K * D:]
    R0, R1, R2 = ref[1:1 + K], ref[1 + K:1 + K + K * D], ref[1 + K + K * D:]
    e0 = float(np.max(np.abs(S0 - R0) / np.maximum(R0, 1e-300)))
    e1, e2 = rel_l2(S1, R1), rel_l2(S2, R2)
    print(f"{label}: S0 max rel {e0:.2e}  S1 rel-L2 {e1:.2e}  S2 rel-L2 {e2:.2e}")
    assert st[0] == ref[0]
    assert e0 <= S0_RTOL and e1 <= STATS_RTOL and e2 <= STATS_RTOL
    return e0, e1, e2


@pytest.mark.slow
def test_c5_full_size_against_oracle(fv):
    g = load("large_c5.npz")
    K, D = int(g["K"]), int(g["D"])
    gmm_np = fvgen.make_gmm(K, D, seed=int(g["seed_gmm"]))
    X = fvgen.make_frames(gmm_np, int(g["frames"]), int(g["per_frame"]), seed=int(g["seed_data"]))
    N = X.shape[0]
    Xd = torch.from_numpy(X).cuda()
    check_same_input(X, Xd, g)
    del X
    gmm = fv.GMM(*gmm_np)
    st = fv.stats_batched(Xd, torch.tensor([0, N], dtype=torch.int64, device="cuda"), gmm)
    out = fv.finalize(st, gmm).cpu().numpy()[0]
    ref = g["stats"]
    compare_stats(st.cpu().numpy()[0], ref, K, D, "C5")
    ref_fv = oracle.fv_from_stats(ref, *gmm_np)
    err = rel_l2(out, ref_fv)
    print(f"C5 FV rel-L2 vs oracle: {err:.3e}")
    assert err <= FV_RTOL
    # the U and V blocks separately (V carries the S2 - ... - S0 cancellation)
    KD = K * D
    assert rel_l2(out[:KD], ref_fv[:KD]) <= FV_RTOL and rel_l2(out[KD:], ref_fv[KD:]) <= FV_RTOL


@pytest.mark.slow
@pytest.mark.parametrize("mode", ["exact", "tau"])
def test_pool64_full_size_against_oracle(fv, mode):
    g = load("large_pool64.npz")
    K, D = int(g["K"]), int(g["D"])
    gmm_np = fvgen.make_gmm(K, D, seed=int(g["seed_gmm"]))
    X = fvgen.make_frames(gmm_np, int(g["frames"]), int(g["per_frame"]), seed=int(g["seed_data"]))
    N = X.shape[0]
    Xd = torch.from_numpy(X).cuda()
    check_same_input(X, Xd, g)
    tau = 1e-6 if mode == "tau" else 0.0
    gmm = fv.GMM(*gmm_np)
    st = fv.stats_batched(Xd, torch.tensor([0, N], dtype=torch.int64, device="cuda"), gmm, threshold=tau)
    ref = g["stats_tau" if mode == "tau" else "stats_exact"]
    compare_stats(st.cpu().numpy()[0], ref, K, D, f"pool64 {mode}")
    out = fv.finalize(st, gmm).cpu().numpy()[0]
    err = rel_l2(out, oracle.fv_from_stats(ref, *gmm_np))
    print(f"pool64 {mode} FV rel-L2 vs oracle: {err:.3e}")
    assert err <= FV_RTOL
    # the one-call encode of the same set (k_stats -> k_finalize) agrees as well
    enc = fv.encode(Xd, gmm, threshold=tau).cpu().numpy()
    assert rel_l2(enc, oracle.fv_from_stats(ref, *gmm_np)) <= FV_RTOL


@pytest.mark.slow
def test_pool64_em_step_full_size_against_oracle(fv):
    """One EM iteration over the 5.12 M-row pool (bench.py --workload em, rank 0) from the seed-1704 GMM:
    priors within 1e-5 relative (S0 / N), means within 1e-5 standard deviations, variances within 1e-5
    relative, log-likelihood within 1e-5 nats per descriptor."""
    g = load("large_pool64.npz")
    K, D = int(g["K"]), int(g["D"])
    gmm_np = fvgen.make_gmm(K, D, seed=int(g["seed_gmm"]))
    X = fvgen.make_frames(gmm_np, int(g["frames"]), int(g["per_frame"]), seed=int(g["seed_data"]))
    N = X.shape[0]
    Xd = torch.from_numpy(X).cuda()
    check_same_input(X, Xd, g)
    init = fv.GMM(*fvgen.make_gmm(K, D, seed=int(g["seed_init"])))
    new, ll = fv.gmm_em_step(Xd, init)
    pi, mu, var = (t.cpu().double().numpy() for t in (new.weights, new.means, new.sigmas))
    e_pi = (np.abs(pi - g["em_pi"]) / g["em_pi"]).max()
    e_mu = (np.abs(mu - g["em_mu"]) / np.sqrt(g["em_var"])).max()
    e_var = (np.abs(var - g["em_var"]) / g["em_var"]).max()
    e_ll = abs(float(ll.item()) - float(g["em_ll"])) / N
    print(f"EM full size: pi rel {e_pi:.2e}  mu/sd {e_mu:.2e}  var rel {e_var:.2e}  ll/N {e_ll:.2e}")
    assert e_pi <= 1e-5 and e_mu <= 1e-5 and e_var <= 1e-5 and e_ll <= 1e-5
