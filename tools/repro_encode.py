import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import fvgen, oracle, paper_1604_03498_b200 as fv
def run(K, D, N, tau):
    gmm_np = fvgen.make_gmm(K, D, seed=1604)
    X = fvgen.make_descriptors(gmm_np, N, seed=1605)
    out = fv.encode(torch.from_numpy(X).cuda(), fv.GMM(*gmm_np), threshold=tau).cpu().numpy()
    ref = oracle.encode(X, *gmm_np, threshold=tau)
    print(K, D, N, tau, np.linalg.norm(out - ref) / np.linalg.norm(ref), flush=True)
for args in [tuple(map(float, a.split(","))) for a in sys.argv[1:]]:
    run(int(args[0]), int(args[1]), int(args[2]), args[3])
