"""Single-frame scored latency (the monitoring application: one 5,000-descriptor frame -> n_cls
scores, FV not written, prepared GMM), CUDA events, p50 of 50 calls.  PROBE_N, PROBE_CLS override the shape."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import fvgen  # noqa: E402
import paper_1604_03498_b200 as fv  # noqa: E402

N = int(os.environ.get("PROBE_N", "5000"))
C = int(os.environ.get("PROBE_CLS", "1"))
gmm_np = fvgen.make_gmm(256, 64, seed=1604)
X = torch.from_numpy(fvgen.make_descriptors(gmm_np, N, seed=2604)).cuda()
off = torch.tensor([0, N], dtype=torch.int64, device="cuda")
W = torch.from_numpy(np.random.default_rng(1).standard_normal((C, 2 * 256 * 64)).astype(np.float32)).cuda()
gmm = fv.GMM(*gmm_np)
ws = fv.Workspace()
fv.encode_scored_batched(X, off, gmm, W, None, threshold=1e-6, ws=ws)  # sizes ws
fv.gmm_prepare(gmm, ws)
for _ in range(5):
    fv.encode_scored_batched(X, off, gmm, W, None, threshold=1e-6, ws=ws, prepared=True)
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(50)]
for a, b in ev:
    a.record(); fv.encode_scored_batched(X, off, gmm, W, None, threshold=1e-6, ws=ws, prepared=True); b.record()
torch.cuda.synchronize()
us = sorted(1e3 * a.elapsed_time(b) for a, b in ev)
print(f"scored frame N={N} n_cls={C}: p50 {us[25]:.1f} us, min {us[0]:.1f} us")
