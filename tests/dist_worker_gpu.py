"""Worker for tests/test_gpu_dist.py: one rank of a 2-process gloo group sharing the one GPU, running
paper_1604_03498_b200.dist with its DEFAULT compute steps (the CUDA library: fv_stats_batched,
fv_finalize, fv_encode_batched, fv_gmm_estep / fv_gmm_mstep, fv_encode_scored_batched) on CUDA tensors.
Results are compared with the oracle on the whole set; errors are written to $OUT_DIR/rank<r>.json."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import fvgen  # noqa: E402
import oracle  # noqa: E402
import paper_1604_03498_b200 as fv  # noqa: E402
from paper_1604_03498_b200 import dist as fvd  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("gloo", rank=rank, world_size=world)


def rel(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


res = {}
TAU = 1e-6
# descriptor sharding (C5's path) on both tile families, all-reduce and the deterministic all-gather
for K, D, N in ((512, 128, 6001), (256, 64, 9003)):
    g_np = fvgen.make_gmm(K, D, seed=51)
    X = fvgen.make_descriptors(g_np, N, seed=52)
    lo, hi = fvd.shard_ranges(N, world)[rank]
    gmm = fv.GMM(*g_np)
    ref = oracle.encode(X, *g_np, threshold=TAU)
    ref_st = oracle.stats(X, *g_np, threshold=TAU)
    for det in (False, True):
        out, st = fvd.encode_descriptor_sharded(torch.from_numpy(X[lo:hi]).cuda(), gmm, threshold=TAU,
                                                deterministic=det, return_stats=True)
        res[f"desc_K{K}_D{D}_det{int(det)}_fv"] = rel(out.cpu().numpy(), ref)
        s = st.cpu().numpy()[0]
        res[f"desc_K{K}_D{D}_det{int(det)}_N"] = float(s[0])
        res[f"desc_K{K}_D{D}_det{int(det)}_stats"] = rel(s[1:], ref_st[1:])
# frame sharding (C3/C4's path): whole-stream X and rank-local rows, gathered in frame order
g_np = fvgen.make_gmm(256, 64, seed=53)
Xb, off = fvgen.make_batch(g_np, [10, 3000, 0, 777, 5, 2500, 128], seed_base=54)
gmm = fv.GMM(*g_np)
ref = oracle.encode_batched(Xb, off, *g_np, threshold=TAU)
out = fvd.encode_frames_sharded(torch.from_numpy(Xb).cuda(), off, gmm, threshold=TAU, gather=True).cpu().numpy()
res["frames_full"] = max(rel(out[b], ref[b]) for b in range(len(off) - 1) if off[b + 1] > off[b])
res["frames_empty_zero"] = float(np.abs(out[2]).max())
shard = fvd.FrameShard(off, rank, world, device="cuda")
Xl = torch.from_numpy(Xb[shard.r0:shard.r1]).cuda()
out = fvd.encode_frames_sharded(Xl, None, gmm, threshold=TAU, gather=True, shard=shard, rows_local=True).cpu().numpy()
res["frames_local"] = max(rel(out[b], ref[b]) for b in range(len(off) - 1) if off[b + 1] > off[b])
# frame-sharded fused scoring (NEXT-4)
W = np.random.default_rng(55).standard_normal((3, 2 * 256 * 64)).astype(np.float32)
sc = fvd.score_frames_sharded(torch.from_numpy(Xb).cuda(), off, gmm, torch.from_numpy(W).cuda(), threshold=TAU)
sref = oracle.score(ref, W)
fvn = np.linalg.norm(ref, axis=1)
res["scores"] = float(np.max(np.abs(sc.cpu().numpy() - sref) / (np.linalg.norm(W, axis=1)[None, :] * np.maximum(fvn[:, None], 1))))
# descriptor-sharded EM (NEXT-3)
g_np = fvgen.make_gmm(64, 32, seed=56)
X = fvgen.make_descriptors(g_np, 8000, seed=57)
init = fvgen.make_gmm(64, 32, seed=58)
lo, hi = fvd.shard_ranges(X.shape[0], world)[rank]
new, ll = fvd.em_step_sharded(torch.from_numpy(X[lo:hi]).cuda(), fv.GMM(*init))
pi_r, mu_r, var_r, ll_r = oracle.em_step(X, *init)
res["em_pi"] = float(np.abs(new.weights.cpu().numpy() - pi_r).max())
res["em_mu_over_sd"] = float((np.abs(new.means.cpu().numpy() - mu_r) / np.sqrt(var_r)).max())
res["em_var_rel"] = float((np.abs(new.sigmas.cpu().numpy() - var_r) / var_r).max())
res["em_ll_per_desc"] = abs(ll - ll_r) / X.shape[0]
with open(os.path.join(os.environ["OUT_DIR"], f"rank{rank}.json"), "w") as f:
    json.dump(res, f)
dist.destroy_process_group()
