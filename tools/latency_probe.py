"""Single-frame latency probe (C2 shape: one 5000-descriptor frame, K=256, D=64, tau=1e-6): runs the
prepared fv_encode a few times so `ncu --metrics gpu__time_duration.sum` can list per-kernel
durations (serialised by ncu) next to the CUDA-event latency printed here."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import fvgen  # noqa: E402
import paper_1604_03498_b200 as fv  # noqa: E402

N = int(os.environ.get("PROBE_N", "5000"))
gmm_np = fvgen.make_gmm(256, 64, seed=1604)
X = torch.from_numpy(fvgen.make_descriptors(gmm_np, N, seed=1604 + 1000)).cuda()
gmm = fv.GMM(*gmm_np)
ws = fv.Workspace()
ws.ensure(fv.workspace_bytes(N, 1, 256, 64))
fv.gmm_prepare(gmm, ws)
out = torch.empty(2 * 256 * 64, device="cuda")
reps = int(os.environ.get("PROBE_REPS", "5"))
for _ in range(reps):
    fv.encode(X, gmm, threshold=1e-6, ws=ws, prepared=True, out=out)
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(50)]
for a, b in ev:
    a.record(); fv.encode(X, gmm, threshold=1e-6, ws=ws, prepared=True, out=out); b.record()
torch.cuda.synchronize()
us = sorted(1e3 * a.elapsed_time(b) for a, b in ev)
# the stats kernel alone (library hook brackets each k_stats launch with these events)
kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(50)]
for a, b in kev:
    a.record(); b.record()
for a, b in kev:
    fv.profile_events(a, b)
    fv.encode(X, gmm, threshold=1e-6, ws=ws, prepared=True, out=out)
fv.profile_events(None, None)
torch.cuda.synchronize()
ks = sorted(1e3 * a.elapsed_time(b) for a, b in kev)
# without FV_PREPARED: the GMM preparation (step a1) runs inside every call
ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(50)]
for a, b in ev2:
    a.record(); fv.encode(X, gmm, threshold=1e-6, ws=ws, prepared=False, out=out); b.record()
torch.cuda.synchronize()
up = sorted(1e3 * a.elapsed_time(b) for a, b in ev2)
print(f"N={N}: p50 {us[25]:.1f} us, min {us[0]:.1f} us; k_stats p50 {ks[25]:.1f} us; unprepared call p50 {up[25]:.1f} us")
