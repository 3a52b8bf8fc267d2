"""B200-native Fisher-vector encoder (GPU-FV, arXiv 1604.03498) — thin Python binding.

Every call marshals torch CUDA tensors into the C ABI of ``libgpufv.so`` (include/gpufv.h) and
enqueues on the current torch CUDA stream.  All arithmetic runs in the library's sm_100a kernels;
there is NO CPU fallback: if the shared library is missing this module raises on import.
PyTorch is used only for device memory, streams and (in ``dist``) process groups.
"""
from __future__ import annotations

import ctypes
import os

import torch

__all__ = [
    "NORM_IMPROVED", "NORM_POWER_L2", "NORM_NONE", "SIGMA_IS_STDDEV", "PREPARED", "SPARSE_STATS",
    "GMM", "Workspace", "lib", "lib_path", "workspace_bytes", "gmm_prepare", "encode", "encode_batched",
    "encode_batched_host", "stats_batched", "finalize", "posteriors", "last_launch_count", "profile_events",
    "encode_scored_batched", "encode_scored_batched_host", "MAX_CLASSES", "gmm_estep", "gmm_mstep", "gmm_em_step",
    "gmm_fit", "embed", "embed_encode_batched", "FVError", "range_flags",
]

NORM_IMPROVED = 0
NORM_POWER_L2 = 1
NORM_NONE = 2
SIGMA_IS_STDDEV = 1 << 4
PREPARED = 1 << 6
SPARSE_STATS = 1 << 7  # threshold > 0: survivor (Alg. 5) accumulation instead of the dense tensor-core GEMM2
_RAW_LOGLIK = 1 << 8
MAX_CLASSES = 32  # test hook of fv_posteriors: raw log2-likelihoods instead of gamma

_HERE = os.path.dirname(os.path.abspath(__file__))
lib_path = os.path.join(_HERE, "libgpufv.so")

if not os.path.exists(lib_path):
    raise ImportError(
        f"{lib_path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(there is no CPU fallback)")

lib = ctypes.CDLL(lib_path)

_c = ctypes
_vp, _i64, _i32, _f32, _u32, _sz = _c.c_void_p, _c.c_int64, _c.c_int, _c.c_float, _c.c_uint, _c.c_size_t

lib.fv_workspace_bytes.argtypes = [_i64, _i32, _i32, _i32, _u32]
lib.fv_workspace_bytes.restype = _sz
lib.fv_workspace_bytes_host.argtypes = [_i64, _i32, _i32, _i32, _u32]
lib.fv_workspace_bytes_host.restype = _sz
lib.fv_gmm_prepare.argtypes = [_vp, _vp, _vp, _i32, _i32, _u32, _vp, _sz, _vp]
lib.fv_encode.argtypes = [_vp, _i64, _i32, _vp, _vp, _vp, _i32, _f32, _u32, _vp, _vp, _sz, _vp]
lib.fv_encode_batched.argtypes = [_vp, _vp, _i32, _i64, _i32, _vp, _vp, _vp, _i32, _f32, _u32, _vp, _vp, _sz, _vp]
lib.fv_encode_batched_host.argtypes = lib.fv_encode_batched.argtypes
lib.fv_stats_batched.argtypes = [_vp, _vp, _i32, _i64, _i32, _vp, _vp, _vp, _i32, _f32, _u32, _vp, _vp, _sz, _vp]
lib.fv_finalize.argtypes = [_vp, _i32, _i32, _vp, _vp, _vp, _i32, _u32, _vp, _vp, _sz, _vp]
lib.fv_posteriors.argtypes = [_vp, _i64, _i32, _vp, _vp, _vp, _i32, _f32, _u32, _vp, _vp, _sz, _vp]
lib.fv_workspace_bytes_scored.argtypes = [_i64, _i32, _i32, _i32, _i32, _i32, _u32]
lib.fv_workspace_bytes_scored.restype = _sz
lib.fv_encode_scored_batched.argtypes = [_vp, _vp, _i32, _i64, _i32, _vp, _vp, _vp, _i32, _f32, _u32, _vp, _vp, _i32,
                                         _vp, _vp, _vp, _sz, _vp]
lib.fv_encode_scored_batched_host.argtypes = [_vp, _vp, _i32, _i64, _i32, _vp, _vp, _vp, _i32, _f32, _u32, _vp, _vp,
                                              _i32, _vp, _vp, _sz, _vp]
lib.fv_workspace_bytes_em.argtypes = [_i64, _i32, _i32, _u32]
lib.fv_workspace_bytes_em.restype = _sz
lib.fv_gmm_estep.argtypes = [_vp, _i64, _i32, _vp, _vp, _vp, _i32, _u32, _vp, _vp, _vp, _sz, _vp]
lib.fv_gmm_mstep.argtypes = [_vp, _i32, _vp, _vp, _vp, _i32, _u32, _f32, _f32, _f32, _vp, _vp, _vp, _vp, _sz, _vp]
lib.fv_gmm_em_step.argtypes = [_vp, _i64, _i32, _vp, _vp, _vp, _i32, _u32, _f32, _f32, _f32, _vp, _vp, _vp, _vp, _vp,
                               _sz, _vp]
lib.fv_embed.argtypes = [_vp, _vp, _vp, _i32, _i64, _vp, _vp, _vp, _i32, _vp, _i32, _vp]
lib.fv_workspace_bytes_embed.argtypes = [_i64, _i32, _i32, _i32, _u32]
lib.fv_workspace_bytes_embed.restype = _sz
lib.fv_embed_encode_batched.argtypes = [_vp, _vp, _vp, _i32, _i64, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _i32, _f32, _u32,
                                        _vp, _vp, _sz, _vp]
for _fn in ("fv_gmm_estep", "fv_gmm_mstep", "fv_gmm_em_step", "fv_embed", "fv_embed_encode_batched"):
    getattr(lib, _fn).restype = _i32
for _fn in ("fv_gmm_prepare", "fv_encode", "fv_encode_batched", "fv_encode_batched_host", "fv_stats_batched",
            "fv_finalize", "fv_posteriors", "fv_encode_scored_batched", "fv_encode_scored_batched_host"):
    getattr(lib, _fn).restype = _i32
lib.fv_status_string.argtypes = [_i32]
lib.fv_status_string.restype = _c.c_char_p
lib.fv_last_error.argtypes = []
lib.fv_last_error.restype = _c.c_char_p
lib.fv_last_launch_count.argtypes = []
lib.fv_last_launch_count.restype = _i32
lib.fv_version.restype = _i32
lib.fv_range_flags.argtypes = [_vp, _sz, _i64, _i32, _i32, _i32, _vp, _vp]
lib.fv_range_flags.restype = _i32
lib.fv_profile_events.argtypes = [_vp, _vp]
lib.fv_profile_events.restype = None


class FVError(RuntimeError):
    def __init__(self, status: int):
        self.status = status
        super().__init__(f"{lib.fv_status_string(status).decode()}: {lib.fv_last_error().decode()}")


def _check(status: int):
    if status != 0:
        raise FVError(status)


def _stream():
    return _c.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t):
    return _c.c_void_p(t.data_ptr()) if t is not None else None


def last_launch_count() -> int:
    return int(lib.fv_last_launch_count())


def profile_events(start=None, stop=None):
    """Bracket every k_stats launch of this thread with these torch.cuda.Event objects (None: off)."""
    lib.fv_profile_events(_c.c_void_p(start.cuda_event) if start is not None else None,
                          _c.c_void_p(stop.cuda_event) if stop is not None else None)


class GMM:
    """Device-resident diagonal GMM: weights (K), means (K x D), sigmas (K x D; variances unless
    ``stddev``), all float32 contiguous CUDA tensors."""

    def __init__(self, weights, means, sigmas, stddev: bool = False, device=None):
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.weights = torch.as_tensor(weights, dtype=torch.float32).to(dev).contiguous()
        self.means = torch.as_tensor(means, dtype=torch.float32).to(dev).contiguous()
        self.sigmas = torch.as_tensor(sigmas, dtype=torch.float32).to(dev).contiguous()
        self.K, self.D = self.means.shape
        self.flags = SIGMA_IS_STDDEV if stddev else 0

    def ptrs(self):
        return _ptr(self.weights), _ptr(self.means), _ptr(self.sigmas)


def workspace_bytes(n_total: int, batch: int, K: int, D: int, flags: int = 0, host_io: bool = False) -> int:
    fn = lib.fv_workspace_bytes_host if host_io else lib.fv_workspace_bytes
    n = int(fn(int(n_total), int(batch), int(K), int(D), int(flags)))
    if n == 0:
        raise FVError(1)
    return n


class Workspace:
    """A growable 1024-byte-aligned device buffer (torch caching allocator); holds the prepared GMM
    at its head, so reuse one Workspace per GMM and pass prepared=True after gmm_prepare."""

    def __init__(self, nbytes: int = 0, device=None):
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self._buf = None
        self.nbytes = 0
        self.ptr = 0
        if nbytes:
            self.ensure(nbytes)

    def ensure(self, nbytes: int):
        if nbytes > self.nbytes:
            # growing invalidates a prepared GMM; callers re-prepare (encode(prepared=False))
            self._buf = torch.empty(nbytes + 1024, dtype=torch.uint8, device=self.device)
            base = self._buf.data_ptr()
            self.ptr = (base + 1023) // 1024 * 1024
            self.nbytes = nbytes
            self.generation = getattr(self, "generation", 0) + 1
        return self

    def args(self):
        return _c.c_void_p(self.ptr), _c.c_size_t(self.nbytes)


def _ws(ws, need, device):
    if ws is None:
        ws = Workspace(device=device)
    gen = getattr(ws, "generation", 0)
    ws.ensure(need)
    return ws, getattr(ws, "generation", 0) != gen


def _mode_flags(gmm: GMM, mode: int, prepared: bool) -> int:
    return int(mode) | gmm.flags | (PREPARED if prepared else 0)


def gmm_prepare(gmm: GMM, ws: Workspace):
    """Step a1 once per GMM (Alg.1 l.1): later calls may pass prepared=True."""
    ws.ensure(workspace_bytes(0, 1, gmm.K, gmm.D))
    w, m, s = gmm.ptrs()
    _check(lib.fv_gmm_prepare(w, m, s, gmm.K, gmm.D, gmm.flags, *ws.args(), _stream()))


def _check_X(X, D):
    if not (X.is_cuda and X.dtype == torch.float32 and X.is_contiguous() and X.dim() == 2 and X.shape[1] == D):
        raise ValueError(f"X must be a contiguous float32 CUDA tensor of shape (N, {D})")


def _check_offsets(offsets, X=None):
    """offsets: contiguous int64 CUDA tensor (batch + 1,) on X's device (a host tensor would be handed to
    the kernels as a device pointer)."""
    if not (offsets.is_cuda and offsets.dtype == torch.int64 and offsets.is_contiguous() and offsets.dim() == 1
            and offsets.shape[0] >= 1):
        raise ValueError("offsets must be a contiguous 1-D int64 CUDA tensor of batch + 1 entries")
    if X is not None and offsets.device != X.device:
        raise ValueError("offsets and X must be on the same device")


def encode(X, gmm: GMM, threshold: float = 0.0, mode: int = NORM_IMPROVED, ws: Workspace | None = None,
           prepared: bool = False, out=None):
    """One descriptor set (N x D) -> FV (2KD,)."""
    _check_X(X, gmm.D)
    ws, grown = _ws(ws, workspace_bytes(X.shape[0], 1, gmm.K, gmm.D), X.device)
    prepared = prepared and not grown
    if out is None:
        out = torch.empty(2 * gmm.K * gmm.D, dtype=torch.float32, device=X.device)
    w, m, s = gmm.ptrs()
    _check(lib.fv_encode(_ptr(X), X.shape[0], gmm.D, w, m, s, gmm.K, float(threshold),
                         _mode_flags(gmm, mode, prepared), _ptr(out), *ws.args(), _stream()))
    return out


def encode_batched(X, offsets, gmm: GMM, threshold: float = 0.0, mode: int = NORM_IMPROVED,
                   ws: Workspace | None = None, prepared: bool = False, out=None):
    """Independent images: X (n_total x D), offsets (batch+1, int64 CUDA) -> (batch, 2KD)."""
    _check_X(X, gmm.D)
    _check_offsets(offsets, X)
    B = offsets.shape[0] - 1
    ws, grown = _ws(ws, workspace_bytes(X.shape[0], B, gmm.K, gmm.D), X.device)
    prepared = prepared and not grown
    if out is None:
        out = torch.empty(B, 2 * gmm.K * gmm.D, dtype=torch.float32, device=X.device)
    w, m, s = gmm.ptrs()
    _check(lib.fv_encode_batched(_ptr(X), _ptr(offsets), B, X.shape[0], gmm.D, w, m, s, gmm.K, float(threshold),
                                 _mode_flags(gmm, mode, prepared), _ptr(out), *ws.args(), _stream()))
    return out


def encode_batched_host(X_host, offsets_host, gmm: GMM, threshold: float = 0.0, mode: int = NORM_IMPROVED,
                        ws: Workspace | None = None, prepared: bool = False, out_host=None):
    """Host buffers in and out (pinned CPU tensors for full PCIe speed); the GMM stays on the GPU.
    The H2D copy, encode and D2H copy all happen inside the library call, which returns when the
    host result is ready."""
    assert X_host.device.type == "cpu" and X_host.dtype == torch.float32 and X_host.is_contiguous()
    assert offsets_host.device.type == "cpu" and offsets_host.dtype == torch.int64
    B = offsets_host.shape[0] - 1
    ws, grown = _ws(ws, workspace_bytes(X_host.shape[0], B, gmm.K, gmm.D, host_io=True), gmm.means.device)
    prepared = prepared and not grown
    if out_host is None:
        out_host = torch.empty(B, 2 * gmm.K * gmm.D, dtype=torch.float32, pin_memory=True)
    w, m, s = gmm.ptrs()
    _check(lib.fv_encode_batched_host(_ptr(X_host), _ptr(offsets_host), B, X_host.shape[0], gmm.D, w, m, s, gmm.K,
                                      float(threshold), _mode_flags(gmm, mode, prepared), _ptr(out_host),
                                      *ws.args(), _stream()))
    return out_host


def stats_batched(X, offsets, gmm: GMM, threshold: float = 0.0, ws: Workspace | None = None,
                  prepared: bool = False, out=None, sparse: bool = False):
    """Sufficient statistics (batch, 1 + K(2D+1)) float64 about c (reading A19); they add across
    disjoint descriptor shards."""
    _check_X(X, gmm.D)
    _check_offsets(offsets, X)
    B = offsets.shape[0] - 1
    ws, grown = _ws(ws, workspace_bytes(X.shape[0], B, gmm.K, gmm.D), X.device)
    prepared = prepared and not grown
    if out is None:
        out = torch.empty(B, 1 + gmm.K * (2 * gmm.D + 1), dtype=torch.float64, device=X.device)
    w, m, s = gmm.ptrs()
    _check(lib.fv_stats_batched(_ptr(X), _ptr(offsets), B, X.shape[0], gmm.D, w, m, s, gmm.K, float(threshold),
                                _mode_flags(gmm, SPARSE_STATS if sparse else 0, prepared), _ptr(out), *ws.args(),
                                _stream()))
    return out


def finalize(stats, gmm: GMM, mode: int = NORM_IMPROVED, ws: Workspace | None = None, prepared: bool = False,
             out=None):
    """Statistics (batch, 1 + K(2D+1)) float64 -> FVs (batch, 2KD)."""
    assert stats.is_cuda and stats.dtype == torch.float64 and stats.is_contiguous()
    st = stats.reshape(-1, 1 + gmm.K * (2 * gmm.D + 1))
    B = st.shape[0]
    ws, grown = _ws(ws, workspace_bytes(0, B, gmm.K, gmm.D), stats.device)
    prepared = prepared and not grown
    if out is None:
        out = torch.empty(B, 2 * gmm.K * gmm.D, dtype=torch.float32, device=stats.device)
    w, m, s = gmm.ptrs()
    _check(lib.fv_finalize(_ptr(st), B, gmm.D, w, m, s, gmm.K, _mode_flags(gmm, mode, prepared), _ptr(out),
                           *ws.args(), _stream()))
    return out


def posteriors(X, gmm: GMM, threshold: float = 0.0, raw_loglik: bool = False, ws: Workspace | None = None):
    """Test hook: gamma (N x K) from the production kernel; raw_loglik returns log2-likelihoods
    (+ per-Gaussian bias, shifted by a per-GMM constant) instead."""
    _check_X(X, gmm.D)
    ws, _ = _ws(ws, workspace_bytes(X.shape[0], 1, gmm.K, gmm.D), X.device)
    g = torch.empty(X.shape[0], gmm.K, dtype=torch.float32, device=X.device)
    w, m, s = gmm.ptrs()
    flags = gmm.flags | (_RAW_LOGLIK if raw_loglik else 0)
    _check(lib.fv_posteriors(_ptr(X), X.shape[0], gmm.D, w, m, s, gmm.K, float(threshold), flags, _ptr(g),
                             *ws.args(), _stream()))
    return g


def range_flags(ws: Workspace, n_total: int, batch: int, gmm: GMM):
    """Per-image range report (int32, batch) of the last encode / stats / posteriors / E-step call made with
    ``ws`` on (n_total descriptors, batch images, gmm): bit 0 = the image had a row with non-finite
    log-likelihoods (a descriptor outside the fp16 operand range or non-finite input), bit 1 = the GMM has
    a coefficient outside the fp16 range.  Flagged images' outputs are NaN (include/gpufv.h)."""
    flags = torch.empty(max(int(batch), 0), dtype=torch.int32, device=ws.device)
    _check(lib.fv_range_flags(*ws.args(), int(n_total), int(batch), gmm.K, gmm.D, _ptr(flags), _stream()))
    return flags


def _classifier(svm_w, svm_b, gmm: GMM):
    dim = 2 * gmm.K * gmm.D
    if not (svm_w.is_cuda and svm_w.dtype == torch.float32 and svm_w.is_contiguous()):
        raise ValueError("svm_w must be a contiguous float32 CUDA tensor (n_cls, 2KD)")
    W = svm_w.reshape(-1, dim)
    if svm_b is not None and not (svm_b.is_cuda and svm_b.dtype == torch.float32 and svm_b.numel() == W.shape[0]):
        raise ValueError("svm_b must be a float32 CUDA tensor (n_cls,)")
    return W, W.shape[0]


def encode_scored_batched(X, offsets, gmm: GMM, svm_w, svm_b=None, threshold: float = 0.0,
                          mode: int = NORM_IMPROVED, ws: Workspace | None = None, prepared: bool = False,
                          out=None, return_fv: bool = False):
    """Fused linear scoring (NEXT-4): scores (batch, n_cls) = FV . svm_w^T + svm_b, taken in
    the finalize kernel.  With return_fv (or an ``out`` tensor) the FVs are also written and returned
    as (scores, fv); otherwise they never reach HBM."""
    _check_X(X, gmm.D)
    _check_offsets(offsets, X)
    W, n_cls = _classifier(svm_w, svm_b, gmm)
    B = offsets.shape[0] - 1
    need = int(lib.fv_workspace_bytes_scored(X.shape[0], B, gmm.K, gmm.D, n_cls, 0, 0))
    if need == 0:
        raise FVError(1)
    ws, grown = _ws(ws, need, X.device)
    prepared = prepared and not grown
    scores = torch.empty(B, n_cls, dtype=torch.float32, device=X.device)
    if out is None and return_fv:
        out = torch.empty(B, 2 * gmm.K * gmm.D, dtype=torch.float32, device=X.device)
    w, m, s = gmm.ptrs()
    _check(lib.fv_encode_scored_batched(_ptr(X), _ptr(offsets), B, X.shape[0], gmm.D, w, m, s, gmm.K,
                                        float(threshold), _mode_flags(gmm, mode, prepared), _ptr(W), _ptr(svm_b),
                                        n_cls, _ptr(scores), _ptr(out), *ws.args(), _stream()))
    return (scores, out) if out is not None else scores


def encode_scored_batched_host(X_host, offsets_host, gmm: GMM, svm_w, svm_b=None, threshold: float = 0.0,
                               mode: int = NORM_IMPROVED, ws: Workspace | None = None, prepared: bool = False,
                               scores_host=None):
    """Monitoring-stream entry point: pinned host descriptors in, host scores (batch, n_cls) out; the
    GMM and the classifier stay on the GPU and only the scores cross PCIe back."""
    assert X_host.device.type == "cpu" and X_host.dtype == torch.float32 and X_host.is_contiguous()
    assert offsets_host.device.type == "cpu" and offsets_host.dtype == torch.int64
    W, n_cls = _classifier(svm_w, svm_b, gmm)
    B = offsets_host.shape[0] - 1
    need = int(lib.fv_workspace_bytes_scored(X_host.shape[0], B, gmm.K, gmm.D, n_cls, 1, 0))
    if need == 0:
        raise FVError(1)
    ws, grown = _ws(ws, need, gmm.means.device)
    prepared = prepared and not grown
    if scores_host is None:
        scores_host = torch.empty(B, n_cls, dtype=torch.float32, pin_memory=True)
    w, m, s = gmm.ptrs()
    _check(lib.fv_encode_scored_batched_host(_ptr(X_host), _ptr(offsets_host), B, X_host.shape[0], gmm.D, w, m, s,
                                             gmm.K, float(threshold), _mode_flags(gmm, mode, prepared), _ptr(W),
                                             _ptr(svm_b), n_cls, _ptr(scores_host), *ws.args(), _stream()))
    return scores_host


# ------------------------------------------------------------------ GMM EM training (NEXT-3)
def _em_ws(ws, N, gmm, device):
    need = int(lib.fv_workspace_bytes_em(int(N), gmm.K, gmm.D, 0))
    if need == 0:
        raise FVError(1)
    return _ws(ws, need, device)[0]


def gmm_estep(X, gmm: GMM, ws: Workspace | None = None):
    """E-step: (stats (1 + K(2D+1),) float64 about c, loglik (1,) float64) of X under gmm;
    both add across descriptor shards."""
    _check_X(X, gmm.D)
    ws = _em_ws(ws, X.shape[0], gmm, X.device)
    st = torch.empty(1 + gmm.K * (2 * gmm.D + 1), dtype=torch.float64, device=X.device)
    ll = torch.empty(1, dtype=torch.float64, device=X.device)
    w, m, s = gmm.ptrs()
    _check(lib.fv_gmm_estep(_ptr(X), X.shape[0], gmm.D, w, m, s, gmm.K, gmm.flags, _ptr(st), _ptr(ll), *ws.args(),
                            _stream()))
    return st, ll


def gmm_mstep(stats, gmm: GMM, var_floor_abs: float = 1e-6, var_floor_rel: float = 1e-4,
              prior_floor: float = 1e-8, ws: Workspace | None = None) -> GMM:
    """M-step from (possibly all-reduced) E-step statistics -> a new GMM (variances)."""
    assert stats.is_cuda and stats.dtype == torch.float64 and stats.is_contiguous()
    ws = _em_ws(ws, 0, gmm, stats.device)
    new = GMM(torch.empty_like(gmm.weights), torch.empty_like(gmm.means), torch.empty_like(gmm.sigmas),
              device=gmm.means.device)
    w, m, s = gmm.ptrs()
    _check(lib.fv_gmm_mstep(_ptr(stats), gmm.D, w, m, s, gmm.K, gmm.flags, float(var_floor_abs), float(var_floor_rel),
                            float(prior_floor), *new.ptrs(), *ws.args(), _stream()))
    return new


def gmm_em_step(X, gmm: GMM, var_floor_abs: float = 1e-6, var_floor_rel: float = 1e-4, prior_floor: float = 1e-8,
                ws: Workspace | None = None, out: GMM | None = None):
    """One EM iteration on one device -> (new GMM, loglik of X under the INPUT gmm as a (1,) float64
    tensor).  ``out`` may be ``gmm`` itself (in-place update)."""
    _check_X(X, gmm.D)
    ws = _em_ws(ws, X.shape[0], gmm, X.device)
    if out is None:
        out = GMM(torch.empty_like(gmm.weights), torch.empty_like(gmm.means), torch.empty_like(gmm.sigmas),
                  device=gmm.means.device)
    ll = torch.empty(1, dtype=torch.float64, device=X.device)
    w, m, s = gmm.ptrs()
    _check(lib.fv_gmm_em_step(_ptr(X), X.shape[0], gmm.D, w, m, s, gmm.K, gmm.flags, float(var_floor_abs),
                              float(var_floor_rel), float(prior_floor), *out.ptrs(), _ptr(ll), *ws.args(), _stream()))
    out.flags = 0  # the M-step writes variances
    return out, ll


def gmm_fit(X, init: GMM, max_iters: int = 100, tol: float = 1e-6, **floors):
    """EM from ``init`` until the relative log-likelihood improvement is < tol (SPEC train_gmm S:255) or
    max_iters.  Returns (GMM, [loglik per iteration]).  Host loop only; every step runs in the kernels
    (one device sync per iteration to read the log-likelihood)."""
    ws = Workspace(device=X.device)
    cur, hist = init, []
    for _ in range(max_iters):
        nxt, ll = gmm_em_step(X, cur, ws=ws, **floors)
        hist.append(float(ll.item()))
        cur = nxt
        if len(hist) > 1 and abs(hist[-1] - hist[-2]) <= tol * abs(hist[-2]):
            break
    return cur, hist


# ------------------------------------------------------------------ PCA + xy embedding (NEXT-2)
def _check_embed_inputs(raw, xy, offsets, img_wh, pca_mean, pca_basis):
    for name, t, cols in (("raw", raw, 128), ("xy", xy, 2), ("img_wh", img_wh, 2)):
        if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous() and t.dim() == 2 and t.shape[1] == cols):
            raise ValueError(f"{name} must be a contiguous float32 CUDA tensor (*, {cols})")
    _check_offsets(offsets, raw)
    for name, t in (("pca_mean", pca_mean), ("pca_basis", pca_basis)):
        if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous() and t.device == raw.device):
            raise ValueError(f"{name} must be a contiguous float32 CUDA tensor on raw's device")
    if not (pca_basis.dim() == 2 and pca_basis.shape[1] == 128 and pca_mean.numel() == 128):
        raise ValueError("pca_mean must have 128 entries and pca_basis shape (m, 128)")
    return pca_basis.shape[0]


def embed(raw, xy, offsets, img_wh, pca_mean, pca_basis, ldx: int | None = None):
    """Raw SIFT (N, 128) + keypoints (N, 2) -> (N, ldx) float32 = [PCA (m), x/W, y/H, 0 pad]."""
    m = _check_embed_inputs(raw, xy, offsets, img_wh, pca_mean, pca_basis)
    ldx = ldx or (m + 2 + 3) // 4 * 4
    out = torch.empty(raw.shape[0], ldx, dtype=torch.float32, device=raw.device)
    _check(lib.fv_embed(_ptr(raw), _ptr(xy), _ptr(offsets), offsets.shape[0] - 1, raw.shape[0], _ptr(img_wh),
                        _ptr(pca_mean), _ptr(pca_basis), m, _ptr(out), ldx, _stream()))
    return out


def embed_encode_batched(raw, xy, offsets, img_wh, pca_mean, pca_basis, gmm: GMM, threshold: float = 0.0,
                         mode: int = NORM_IMPROVED, ws: Workspace | None = None, out=None):
    """Raw descriptors -> FVs (batch, 2K(m+2)) in one call; gmm is K x (m+2)."""
    m = _check_embed_inputs(raw, xy, offsets, img_wh, pca_mean, pca_basis)
    if gmm.D != m + 2:
        raise ValueError(f"GMM dimension {gmm.D} != m + 2 = {m + 2}")
    B = offsets.shape[0] - 1
    need = int(lib.fv_workspace_bytes_embed(raw.shape[0], B, gmm.K, m, 0))
    if need == 0:
        raise FVError(1)
    ws, _ = _ws(ws, need, raw.device)
    if out is None:
        out = torch.empty(B, 2 * gmm.K * gmm.D, dtype=torch.float32, device=raw.device)
    w, mu, s = gmm.ptrs()
    _check(lib.fv_embed_encode_batched(_ptr(raw), _ptr(xy), _ptr(offsets), B, raw.shape[0], _ptr(img_wh),
                                       _ptr(pca_mean), _ptr(pca_basis), m, w, mu, s, gmm.K, float(threshold),
                                       _mode_flags(gmm, mode, False), _ptr(out), *ws.args(), _stream()))
    return out
