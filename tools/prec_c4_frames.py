import sys, numpy as np, torch
sys.path.insert(0, '.')
import fvgen, oracle, paper_1604_03498_b200 as fv
cfg = fvgen.CONFIGS["C4"]
gmm_np = fvgen.make_gmm(cfg["K"], cfg["D"], seed=cfg["seed_gmm"])
F, P = 512, cfg["per_frame"]
X = fvgen.make_frames(gmm_np, F, P, seed=cfg["seed_data"])
off = np.arange(F + 1, dtype=np.int64) * P
out = fv.encode_batched(torch.from_numpy(X).cuda(), torch.from_numpy(off).cuda(), fv.GMM(*gmm_np), threshold=1e-6).cpu().numpy()
idx = list(range(0, F, 37))
ref = oracle.encode_batched(np.concatenate([X[f*P:(f+1)*P] for f in idx]), np.arange(len(idx)+1, dtype=np.int64)*P, *gmm_np, threshold=1e-6)
err = [np.linalg.norm(out[f]-ref[i])/np.linalg.norm(ref[i]) for i, f in enumerate(idx)]
print("max rel-L2 over", len(idx), "frames:", max(err), "mean", np.mean(err))
