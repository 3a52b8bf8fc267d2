"""Per-tile phase clocks of CTA 0 (GPUFV_TRACE build): compiles a trace variant of the library to
/tmp, runs one C4-shaped batched encode (FRAMES frames x 5000, K=256, D=64, tau=1e-6) through it,
and prints the mean cycle offsets of each trace slot relative to slot 0 of the same tile (WORK warps
0/5/10/15) and of the MMA thread's issue points, over tiles 8..63.

  python tools/trace_tiles.py            (GPU box; TRACE_NVCC_FLAGS adds nvcc flags, e.g. -DGPUFV_KFOLD=...)"""
import ctypes
import os
import subprocess
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import fvgen  # noqa: E402

lib_path = "/tmp/libgpufv_trace.so"
extra = os.environ.get("TRACE_NVCC_FLAGS", "").split()
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-DGPUFV_TRACE", *extra,
                       "-Xcompiler", "-fPIC", "-shared", "-o", lib_path,
                       os.path.join(ROOT, "paper_1604_03498_b200", "csrc", "gpufv.cu")])
lib = ctypes.CDLL(lib_path)
vp = ctypes.c_void_p
lib.fv_workspace_bytes.restype = ctypes.c_size_t
lib.fv_workspace_bytes.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_uint]
lib.fv_encode_batched.argtypes = [vp, vp, ctypes.c_int, ctypes.c_int64, ctypes.c_int, vp, vp, vp, ctypes.c_int,
                                  ctypes.c_float, ctypes.c_uint, vp, vp, ctypes.c_size_t, vp]
lib.fv_debug_trace.argtypes = [vp]
F = int(os.environ.get("FRAMES", "512"))
K, D = int(os.environ.get("TRACE_K", "256")), int(os.environ.get("TRACE_D", "64"))
TAU = float(os.environ.get("TRACE_TAU", "1e-6"))
gmm = fvgen.make_gmm(K, D, seed=1604)
X = torch.from_numpy(fvgen.make_frames(gmm, F, 5000, seed=1604 + 20000)).cuda()
off = torch.arange(F + 1, dtype=torch.int64, device="cuda") * 5000
w, m, v = (torch.from_numpy(a).cuda() for a in gmm)
nb = lib.fv_workspace_bytes(X.shape[0], F, K, D, 0)
ws = torch.empty(nb + 1024, dtype=torch.uint8, device="cuda")
wsp = (ws.data_ptr() + 1023) // 1024 * 1024
out = torch.empty(F, 2 * K * D, device="cuda")
tr = torch.zeros(8192, dtype=torch.int64, device="cuda")
args = lambda: (vp(X.data_ptr()), vp(off.data_ptr()), F, X.shape[0], D, vp(w.data_ptr()), vp(m.data_ptr()),
                vp(v.data_ptr()), K, ctypes.c_float(TAU), 0, vp(out.data_ptr()), vp(wsp), nb, None)
assert lib.fv_encode_batched(*args()) == 0
lib.fv_debug_trace(vp(tr.data_ptr()))
assert lib.fv_encode_batched(*args()) == 0
torch.cuda.synchronize()
t = tr.cpu().numpy()
mma = t[:1024].reshape(64, 16)
work = t[1024:1024 + 64 * 4 * 16].reshape(64, 4, 16)
tiles = range(8, 64)
base = work[:, 0, 0]
period = np.diff(base[8:64]).mean()
print(f"tile period (warp 0, slot 0 -> next tile): {period:.0f} cycles")
for s in range(16):
    vals = [work[i, w_, s] - base[i] for i in tiles for w_ in range(4) if work[i, w_, s] > 0]
    if vals:
        print(f"WORK slot {s:2d}: mean {np.mean(vals):7.0f}  (warps 0/5/10/15 min {np.min(vals):6.0f} max {np.max(vals):6.0f})")
for s in range(16):
    vals = [mma[i, s] - base[i] for i in tiles if mma[i, s] > 0]
    if vals:
        print(f"MMA  slot {s:2d}: mean {np.mean(vals):7.0f}")
