"""Small calls of every C-ABI entry point (run under compute-sanitizer by tests/test_c_example.py):
batched encode with ragged/empty images, host pipeline, stats + finalize, posteriors, fused scoring,
EM step, PCA+xy embedding + encode.  Exits non-zero if any result is non-finite."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import fvgen  # noqa: E402
import paper_1604_03498_b200 as fv  # noqa: E402

dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
outs = []
for K, D in ((256, 64), (96, 128), (16, 36)):
    g_np = fvgen.make_gmm(K, D, seed=5)
    X, off = fvgen.make_batch(g_np, [300, 0, 129, 1], seed_base=6)
    g = fv.GMM(*g_np)
    outs.append(fv.encode_batched(dev(X), dev(off), g, threshold=1e-6))
    outs.append(fv.encode_batched_host(torch.from_numpy(X).pin_memory(), torch.from_numpy(off), g).cuda())
    st = fv.stats_batched(dev(X), dev(off), g)
    outs.append(fv.finalize(st, g))
    outs.append(fv.posteriors(dev(X[:200]), g, threshold=1e-6))
    W = dev(np.random.default_rng(7).standard_normal((3, 2 * K * D)).astype(np.float32))
    outs.append(fv.encode_scored_batched(dev(X), dev(off), g, W, threshold=1e-6))
    new, ll = fv.gmm_em_step(dev(X), g)
    outs += [new.weights, new.means, new.sigmas, ll]
m = 30
mean, B = fvgen.make_pca(m, seed=8)
ge = fvgen.make_embedded_gmm(32, m, seed=9)
raw, xy, off, wh = fvgen.make_raw_frames(ge, (mean, B), [500, 0, 77], seed=10)
outs.append(fv.embed_encode_batched(dev(raw), dev(xy), dev(off), dev(wh), dev(mean), dev(B), fv.GMM(*ge)))
torch.cuda.synchronize()
bad = [i for i, t in enumerate(outs) if not torch.isfinite(t.float()).all()]
print("entry points ok" if not bad else f"non-finite outputs: {bad}")
sys.exit(1 if bad else 0)
