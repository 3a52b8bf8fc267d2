"""The multi-GPU orchestration (paper_1604_03498_b200.dist) with the REAL CUDA compute steps: two gloo
ranks as separate processes sharing the one GPU, CUDA tensors, default stats / finalize / encode / EM /
scoring entry points, compared with the oracle on the whole set (north_star's descriptor sharding with an
all-reduce of the sufficient statistics, and frame sharding).  NCCL itself needs one GPU per rank, so
the NCCL transport is exercised only by bench.py --gpus N on a multi-GPU box."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def results(tmp_path_factory):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out_dir = str(tmp_path_factory.mktemp("gpudist"))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   OUT_DIR=out_dir, OMP_NUM_THREADS="4")
        procs.append(subprocess.Popen([sys.executable, os.path.join(HERE, "dist_worker_gpu.py")], env=env))
    for p in procs:
        assert p.wait(timeout=900) == 0
    return [json.load(open(os.path.join(out_dir, f"rank{r}.json"))) for r in range(2)]


def test_descriptor_sharded_cuda_path_matches_oracle(results):
    for res in results:
        for K, D, N in ((512, 128, 6001), (256, 64, 9003)):
            for det in (0, 1):
                key = f"desc_K{K}_D{D}_det{det}"
                assert res[key + "_N"] == N
                assert res[key + "_fv"] <= 1e-4, (key, res[key + "_fv"])
                assert res[key + "_stats"] <= 1e-5, (key, res[key + "_stats"])
    # every rank finalises the same all-reduced statistics
    assert results[0]["desc_K512_D128_det1_fv"] == results[1]["desc_K512_D128_det1_fv"]


def test_frame_sharded_cuda_path_matches_oracle(results):
    for res in results:
        assert res["frames_full"] <= 1e-4 and res["frames_local"] <= 1e-4
        assert res["frames_empty_zero"] == 0.0
        assert res["scores"] <= 1e-4


def test_sharded_em_cuda_path_matches_oracle(results):
    for res in results:
        assert res["em_pi"] <= 1e-7 and res["em_mu_over_sd"] <= 1e-4
        assert res["em_var_rel"] <= 1e-4 and res["em_ll_per_desc"] <= 2e-5


def test_bench_two_ranks_sharing_one_gpu(tmp_path):
    """The N > 1 bench harness end to end on a one-GPU box: `bench.py --gpus 2` launches two ranks
    itself (torch.distributed.run on 127.0.0.1); GPUFV_BENCH_SHARE_GPU=1 puts both on GPU 0 with gloo
    collectives (NCCL refuses two ranks on one device).  Frame sharding, the self-checks, the max-over-
    ranks timing and the single JSON line of rank 0 all run; the numbers mean nothing here."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, GPUFV_BENCH_SHARE_GPU="1")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--frames", "256", "--steps", "3",
                        "--warmup", "3", "--e2e-steps", "0", "--cpu-seconds", "0", "--no-latency", "--no-legs",
                        "--score-steps", "0"], env=env, capture_output=True, text=True, timeout=900, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["steps"] == 3
