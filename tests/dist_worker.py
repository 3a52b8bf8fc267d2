"""Worker for tests/test_dist.py: one gloo rank (RANK/WORLD_SIZE/MASTER_* from the environment).
Runs the dist orchestration with oracle-injected compute steps and saves results to $OUT_DIR."""
import importlib.util
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import fvgen  # noqa: E402
import oracle  # noqa: E402

spec = importlib.util.spec_from_file_location("fvdist", os.path.join(ROOT, "paper_1604_03498_b200", "dist.py"))
fvd = importlib.util.module_from_spec(spec)
spec.loader.exec_module(fvd)

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo", rank=rank, world_size=world)
gmm = fvgen.make_gmm(16, 8, seed=31)
X = fvgen.make_descriptors(gmm, 2001, seed=32)
lo, hi = fvd.shard_ranges(X.shape[0], world)[rank]
res = {}
for det in (False, True):
    fv = fvd.encode_descriptor_sharded(
        X[lo:hi], gmm, threshold=1e-6,
        stats_fn=lambda Xs: torch.from_numpy(oracle.stats(Xs, *gmm, threshold=1e-6)),
        finalize_fn=lambda st: torch.from_numpy(oracle.fv_from_stats(st.numpy()[0], *gmm)),
        deterministic=det)
    res[f"desc_{det}"] = fv.numpy()
Xb, off = fvgen.make_batch(gmm, [10, 300, 0, 77, 5], seed_base=33)
out = fvd.encode_frames_sharded(
    Xb, off, gmm, encode_fn=lambda Xs, o: torch.from_numpy(oracle.encode_batched(Xs, o.numpy(), *gmm, threshold=1e-6)),
    gather=True)
res["frames"] = out.numpy()


def mstep_from_stats(st):
    """Test-local M-step in the statistics' moment form (about c), to compare against the oracle's
    two-pass em_step on the whole set."""
    pi, mu, var = (a.astype(np.float64) for a in gmm)
    K, D = mu.shape
    st = st.numpy()
    N, S0 = st[0], st[1:1 + K]
    S1 = st[1 + K:1 + K + K * D].reshape(K, D)
    S2 = st[1 + K + K * D:].reshape(K, D)
    c = (pi[:, None] * mu).sum(0) / pi.sum()
    m1 = S1 / S0[:, None]
    gvar = S2.sum(0) / N - (S1.sum(0) / N) ** 2
    v = np.maximum(S2 / S0[:, None] - m1 ** 2, np.maximum(1e-6, 1e-4 * gvar)[None])
    w = np.maximum(S0 / N, 1e-8)
    return w / w.sum(), c + m1, v


for det in (False, True):
    new, ll = fvd.em_step_sharded(
        X[lo:hi], gmm,
        estep_fn=lambda Xs: (torch.from_numpy(oracle.stats(Xs, *gmm)),
                             torch.tensor([oracle.loglik_rows(Xs, *gmm).sum()], dtype=torch.float64)),
        mstep_fn=mstep_from_stats, deterministic=det)
    res[f"em_pi_{det}"], res[f"em_mu_{det}"], res[f"em_var_{det}"] = new
    res[f"em_ll_{det}"] = np.array([ll])
rng = np.random.default_rng(34)
W = rng.standard_normal((3, 2 * 16 * 8))
sc = fvd.score_frames_sharded(
    Xb, off, gmm, W,
    score_fn=lambda Xs, o: torch.from_numpy(oracle.score(oracle.encode_batched(Xs, o.numpy(), *gmm, threshold=1e-6), W)))
res["scores"] = sc.numpy()
np.savez(os.path.join(os.environ["OUT_DIR"], f"rank{rank}.npz"), **res)
dist.destroy_process_group()
