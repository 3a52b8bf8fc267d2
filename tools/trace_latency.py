"""Single-frame timeline of k_stats CTA 0 (GPUFV_TRACE build, clock64 cycles from kernel entry):
prologue (setup, cluster sync, programmatic-launch wait, first TMA, W' image arrival), each tile's
WORK-warp slot 0 (L(i) ready) and the epilogue (last GEMM2 done, fold, teardown).  One C2-shaped
frame (N descriptors, default 5000; K=256, D=64, tau=1e-6).

  python tools/trace_latency.py            (GPU box; PROBE_N=17714 for the paper geometry)"""
import ctypes
import os
import subprocess
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import fvgen  # noqa: E402

lib_path = "/tmp/libgpufv_trace_lat.so"
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-DGPUFV_TRACE",
                       "-Xcompiler", "-fPIC", "-shared", "-o", lib_path,
                       os.path.join(ROOT, "paper_1604_03498_b200", "csrc", "gpufv.cu")])
lib = ctypes.CDLL(lib_path)
vp = ctypes.c_void_p
lib.fv_workspace_bytes.restype = ctypes.c_size_t
lib.fv_workspace_bytes.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_uint]
lib.fv_encode_batched.argtypes = [vp, vp, ctypes.c_int, ctypes.c_int64, ctypes.c_int, vp, vp, vp, ctypes.c_int,
                                  ctypes.c_float, ctypes.c_uint, vp, vp, ctypes.c_size_t, vp]
lib.fv_debug_trace.argtypes = [vp]
N = int(os.environ.get("PROBE_N", "5000"))
K, D = 256, 64
gmm = fvgen.make_gmm(K, D, seed=1604)
X = torch.from_numpy(fvgen.make_descriptors(gmm, N, seed=1604 + 1000)).cuda()
off = torch.tensor([0, N], dtype=torch.int64, device="cuda")
w, m, v = (torch.from_numpy(a).cuda() for a in gmm)
nb = lib.fv_workspace_bytes(N, 1, K, D, 0)
ws = torch.empty(nb + 1024, dtype=torch.uint8, device="cuda")
wsp = (ws.data_ptr() + 1023) // 1024 * 1024
out = torch.empty(1, 2 * K * D, device="cuda")
tr = torch.zeros(8192, dtype=torch.int64, device="cuda")
args = lambda flags: (vp(X.data_ptr()), vp(off.data_ptr()), 1, N, D, vp(w.data_ptr()), vp(m.data_ptr()),
                      vp(v.data_ptr()), K, ctypes.c_float(1e-6), flags, vp(out.data_ptr()), vp(wsp), nb, None)
assert lib.fv_encode_batched(*args(0)) == 0
for _ in range(5):
    assert lib.fv_encode_batched(*args(1 << 6)) == 0  # FV_PREPARED (bit 6)
torch.cuda.synchronize()
lib.fv_debug_trace(vp(tr.data_ptr()))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
assert lib.fv_encode_batched(*args(1 << 6)) == 0
e1.record()
torch.cuda.synchronize()
print(f"CUDA events around the traced call: {1e3 * e0.elapsed_time(e1):.1f} us")
t = tr.cpu().numpy()
P = t[7680:7696]
t0 = P[0]
names = ["entry", "setup done (__syncthreads)", "cluster_sync", "griddep_wait (k_schedule done)",
         "first X box TMA issued", "W' image in SMEM (MMA thread)", "last GEMM2 done (WORK warp 0)",
         "last fold stored", "teardown __syncthreads", "teardown cluster_sync"]
print(f"N={N}: k_stats CTA 0 timeline, cycles from kernel entry")
for k, name in enumerate(names):
    if P[k]:
        print(f"  P{k} {name:34s} {P[k] - t0:8d}")
work = t[1024:1024 + 64 * 4 * 16].reshape(64, 4, 16)
for i in range(64):
    if work[i, 0, 0]:
        print(f"  tile {i}: WORK slot 0 (L ready) {work[i, 0, 0] - t0:8d}   P write done (slot 9) {work[i, 0, 9] - t0:8d}")
G = t[7700:7725]
g0 = G[20]
print("global timeline (ns from k_stats CTA 0 entry, %globaltimer):")
for k, name in [(20, "k_stats CTA 0 entry"), (21, "k_stats CTA 0 end"), (22, "k_stats last CTA end"),
                (0, "k_finalize block 0 entry"), (1, "k_finalize griddep_wait returned"),
                (8, "k_finalize segment loop start"), (5, "k_finalize segment loads summed"),
                (6, "k_finalize S0 barrier passed"), (2, "k_finalize tile computed"), (3, "k_finalize image norm known (all blocks)"),
                (4, "k_finalize block 0 end"),
                (10, "fused finalize: CTA 0 enters"), (11, "fused finalize: barrier 1 passed"),
                (12, "fused finalize: CTA 0 blocks computed"), (13, "fused finalize: barrier 2 passed")]:
    if G[k]:
        print(f"  {name:42s} {G[k] - g0:8d}")
if G[23]:
    print(f"  {'k_schedule entry':42s} {G[23] - g0:8d}")
if G[24]:
    print(f"  {'k_finalize last block end':42s} {G[24] - g0:8d}")
