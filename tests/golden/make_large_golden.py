"""Writes the full-size expected values in tests/golden/large_*.npz (run once, on a CPU host).

Calls only oracle/ (the arithmetic) and fvgen/ (the seeded inputs), as DESIGN.md §2 requires for
stored expected values:
  large_c5.npz      C5 (BASELINE configs[4]): 10,000,000 x 128, K = 512, exact mode —
                    oracle.stats_blocked -> [N, S0, S1, S2] about c (reading A19; Alg.1 l.16-26,
                    PAPER.md:175-184, as sufficient statistics).
  large_pool64.npz  the bench's 5.12 M-row D = 64 pool (rank-0 EM pool of bench.py --workload em),
                    K = 256: statistics in exact and tau = 1e-6 modes under the generating GMM, and one
                    oracle.em_step_blocked from the EM init GMM (seed 1704; NEXT-3).
Each file also stores a fingerprint of the generated X (per-column fp64 sums and a sha256 of every
9973rd row) so a test on another host can confirm it regenerated the same set before comparing.

  python tests/golden/make_large_golden.py [c5|pool64|all]      (C5 ~20 min on 8 cores)
"""
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import fvgen  # noqa: E402
import oracle  # noqa: E402

C5 = dict(K=512, D=128, frames=2000, per_frame=5000, seed_gmm=1605, seed_data=1606)
POOL = dict(K=256, D=64, frames=1024, per_frame=5000, seed_gmm=1604, seed_data=1604 + 30000, seed_init=1704)


def fingerprint(X):
    colsum = X.astype(np.float64).sum(axis=0)
    h = hashlib.sha256(np.ascontiguousarray(X[::9973]).tobytes()).hexdigest()
    return colsum, h


def c5_data():
    g = fvgen.make_gmm(C5["K"], C5["D"], seed=C5["seed_gmm"])
    X = fvgen.make_frames(g, C5["frames"], C5["per_frame"], seed=C5["seed_data"])
    return g, X


def pool_data():
    g = fvgen.make_gmm(POOL["K"], POOL["D"], seed=POOL["seed_gmm"])
    X = fvgen.make_frames(g, POOL["frames"], POOL["per_frame"], seed=POOL["seed_data"])
    return g, X


def main(which):
    if which in ("c5", "all"):
        t = time.time()
        g, X = c5_data()
        cs, h = fingerprint(X)
        st = oracle.stats_blocked(X, *g)
        np.savez_compressed(os.path.join(HERE, "large_c5.npz"), stats=st, fv=oracle.fv_from_stats(st, *g),
                            colsum=cs, sha=h, **{k: v for k, v in C5.items()})
        print("c5", time.time() - t, flush=True)
    if which in ("pool64", "all"):
        t = time.time()
        g, X = pool_data()
        cs, h = fingerprint(X)
        st0 = oracle.stats_blocked(X, *g)
        st1 = oracle.stats_blocked(X, *g, threshold=1e-6)
        init = fvgen.make_gmm(POOL["K"], POOL["D"], seed=POOL["seed_init"])
        pi, mu, var, ll = oracle.em_step_blocked(X, *init)
        np.savez_compressed(os.path.join(HERE, "large_pool64.npz"), stats_exact=st0, stats_tau=st1,
                            fv_exact=oracle.fv_from_stats(st0, *g), fv_tau=oracle.fv_from_stats(st1, *g),
                            em_pi=pi, em_mu=mu, em_var=var, em_ll=ll, colsum=cs, sha=h,
                            **{k: v for k, v in POOL.items()})
        print("pool64", time.time() - t, flush=True)


def add_fv():
    """Adds the oracle's FVs (oracle.fv_from_stats of the stored statistics) to files written before
    they were stored."""
    for name, cfg, keys in (("large_c5.npz", C5, [("stats", "fv")]),
                            ("large_pool64.npz", POOL, [("stats_exact", "fv_exact"), ("stats_tau", "fv_tau")])):
        path = os.path.join(HERE, name)
        if not os.path.exists(path):
            continue
        d = dict(np.load(path))
        g = fvgen.make_gmm(cfg["K"], cfg["D"], seed=cfg["seed_gmm"])
        for sk, fk in keys:
            d[fk] = oracle.fv_from_stats(d[sk], *g)
        np.savez_compressed(path, **d)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "addfv":
        add_fv()
        sys.exit(0)
    main(sys.argv[1] if len(sys.argv) > 1 else "all")
