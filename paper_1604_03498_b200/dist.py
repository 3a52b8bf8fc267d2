"""Multi-GPU partitioning of the FV hot path (one process per GPU, torch.distributed).

Two strategies:

* Image/frame sharding (C3 batches, C4 streams): images are independent, so each rank encodes its own
  share and there is no collective on the data path.  `shard_ranges` gives contiguous frame blocks;
  `partition_images` balances ragged images (longest-processing-time greedy, deterministic).
* Descriptor sharding (C5: one huge set): each rank computes the fp64 sufficient statistics
  [N, S0, S1, S2] of its contiguous descriptor shard (`fv_stats_batched`), the statistics are summed
  with one `all_reduce` (NCCL over NVLink on B200; they add exactly because they are sums over
  descriptors — reading A19), and every rank runs `fv_finalize`.  `deterministic=True` replaces the
  all-reduce by an all-gather and a fixed-order sum (bitwise repeatable across runs).

The compute steps are injectable (`stats_fn`, `finalize_fn`, `encode_fn`) so the orchestration can be
tested with world_size 2 on CPU over gloo; by default they are the CUDA library's entry points.
"""
from __future__ import annotations

import heapq

import torch
import torch.distributed as dist


def shard_ranges(n: int, world: int):
    """Contiguous [lo, hi) ranges of n items over `world` ranks (sizes differ by at most 1)."""
    return [(r * n // world, (r + 1) * n // world) for r in range(world)]


def partition_images(counts, world: int):
    """Longest-processing-time greedy assignment of images (by descriptor count) to ranks.
    Returns one ascending index list per rank; ties broken by image index (deterministic)."""
    heap = [(0, r) for r in range(world)]
    parts = [[] for _ in range(world)]
    for b in sorted(range(len(counts)), key=lambda i: (-int(counts[i]), i)):
        load, r = heapq.heappop(heap)
        parts[r].append(b)
        heapq.heappush(heap, (load + int(counts[b]), r))
    return [sorted(p) for p in parts]


def _all_gather(parts, t, group):
    """all_gather; gloo has no CUDA all_gather, so CUDA tensors go through host copies there (tests run two
    gloo ranks on one GPU; NCCL gathers device tensors directly)."""
    if t.is_cuda and dist.get_backend(group) == "gloo":
        host = [torch.empty(p.shape, dtype=p.dtype) for p in parts]
        dist.all_gather(host, t.cpu(), group=group)
        for p, h in zip(parts, host):
            p.copy_(h)
    else:
        dist.all_gather(parts, t, group=group)


def _rank_world(group):
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


class FrameShard:
    """This rank's share of a frame stream of B frames (CSR `offsets`, host): frames [lo, hi) =
    shard_ranges(B, world)[rank], rows [r0, r1), and the frame offsets rebased to r0, built once as a
    tensor on `device` (so a timed step makes no host->device copy)."""

    def __init__(self, offsets, rank: int, world: int, device=None):
        import numpy as np

        off = np.asarray(offsets, dtype=np.int64)
        self.B = off.shape[0] - 1
        self.rank, self.world = rank, world
        self.lo, self.hi = shard_ranges(self.B, world)[rank]
        self.r0, self.r1 = int(off[self.lo]), int(off[self.hi])
        self.sizes = [b - a for a, b in shard_ranges(self.B, world)]
        self.local_offsets = torch.from_numpy(off[self.lo:self.hi + 1] - self.r0)
        if device is not None:
            self.local_offsets = self.local_offsets.to(device)


def encode_frames_sharded(X, offsets, gmm, threshold: float = 0.0, mode: int = 0, group=None, encode_fn=None,
                          gather: bool = False, shard: FrameShard | None = None, rows_local: bool = False):
    """Frame-sharded encode: rank r encodes frames shard_ranges(B, world)[r].  X / offsets describe the
    whole stream (offsets on the host), or, with rows_local=True, X holds only this rank's rows
    [r0, r1) (each rank keeps just its own frames resident).  `shard` (a FrameShard) may be passed
    instead of offsets to reuse a plan across steps.  Returns this rank's FVs, or all FVs in frame order
    when gather=True (an all_gather outside the hot path)."""
    rank, world = _rank_world(group)
    if shard is None:
        shard = FrameShard(offsets, rank, world)
    Xs = X if rows_local else X[shard.r0:shard.r1]
    if encode_fn is None:
        from . import encode_batched as _enc

        def encode_fn(Xs, offs):
            return _enc(Xs, offs.to(Xs.device), gmm, threshold=threshold, mode=mode)
    out = encode_fn(Xs, shard.local_offsets)
    if not gather or world == 1:
        return out
    mx = max(shard.sizes)  # all_gather needs equal shapes: pad to the largest shard, trim after
    padded = out.new_zeros((mx, out.shape[1]))
    padded[:out.shape[0]] = out
    buf = [out.new_zeros((mx, out.shape[1])) for _ in shard.sizes]
    _all_gather(buf, padded, group)
    return torch.cat([t[:s] for t, s in zip(buf, shard.sizes)], 0)


def encode_descriptor_sharded(X_shard, gmm, threshold: float = 0.0, mode: int = 0, group=None, stats_fn=None,
                              finalize_fn=None, deterministic: bool = False, return_stats: bool = False):
    """One descriptor set sharded over ranks: X_shard is this rank's contiguous rows.  Returns the
    (identical on every rank) normalised FV of the whole set, shape (2KD,) — and, with return_stats, the
    all-reduced statistics [N, S0, S1, S2] (1, 1 + K(2D+1)) as well."""
    rank, world = _rank_world(group)
    if stats_fn is None:
        from . import stats_batched as _stats

        def stats_fn(Xs):
            offs = torch.tensor([0, Xs.shape[0]], dtype=torch.int64, device=Xs.device)
            return _stats(Xs, offs, gmm, threshold=threshold)
    if finalize_fn is None:
        from . import finalize as _fin

        def finalize_fn(st):
            return _fin(st, gmm, mode=mode)
    st = stats_fn(X_shard).reshape(1, -1)  # [N, S0, S1, S2] (a6)
    if st.dtype != torch.float64:
        st = st.to(torch.float64)
    if world > 1:
        if deterministic:
            parts = [torch.empty_like(st) for _ in range(world)]
            _all_gather(parts, st, group)
            st = parts[0].clone()
            for t in parts[1:]:
                st += t  # fixed rank order
        else:
            dist.all_reduce(st, op=dist.ReduceOp.SUM, group=group)  # a8
    fv = finalize_fn(st).reshape(-1)
    return (fv, st) if return_stats else fv


def em_step_sharded(X_shard, gmm, group=None, estep_fn=None, mstep_fn=None, deterministic: bool = False,
                    **floors):
    """One EM iteration (NEXT-3) over a descriptor set sharded by rows across ranks: every rank runs the
    E-step on its shard (sufficient statistics [N, S0, S1, S2] about c and the log-likelihood sum), the
    1 + K(2D+1) + 1 fp64 values are summed with one all_reduce (they add across shards, reading A19),
    and every rank runs the same M-step.  Returns (new GMM, total log-likelihood under the input GMM)."""
    rank, world = _rank_world(group)
    if estep_fn is None:
        from . import gmm_estep as _estep

        def estep_fn(Xs):
            return _estep(Xs, gmm)
    if mstep_fn is None:
        from . import gmm_mstep as _mstep

        def mstep_fn(st):
            return _mstep(st, gmm, **floors)
    st, ll = estep_fn(X_shard)
    buf = torch.cat([st.reshape(-1).to(torch.float64), ll.reshape(-1).to(torch.float64)])
    if world > 1:
        if deterministic:
            parts = [torch.empty_like(buf) for _ in range(world)]
            _all_gather(parts, buf, group)
            buf = parts[0].clone()
            for t in parts[1:]:
                buf += t  # fixed rank order
        else:
            dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return mstep_fn(buf[:-1].contiguous()), float(buf[-1].item())


def score_frames_sharded(X, offsets, gmm, svm_w, svm_b=None, threshold: float = 0.0, mode: int = 0, group=None,
                         score_fn=None, gather: bool = True, shard: FrameShard | None = None, rows_local: bool = False):
    """Frame-sharded monitoring (NEXT-4): rank r scores frames shard_ranges(B, world)[r] with
    the classifier fused into the finalize (no FV leaves the GPU); only the (frames, n_cls) scores are
    all-gathered (4 B per frame and class instead of 2KD floats).  X / shard / rows_local as in
    encode_frames_sharded."""
    rank, world = _rank_world(group)
    if shard is None:
        shard = FrameShard(offsets, rank, world)
    Xs = X if rows_local else X[shard.r0:shard.r1]
    if score_fn is None:
        from . import encode_scored_batched as _sc

        def score_fn(Xs, offs):
            return _sc(Xs, offs.to(Xs.device), gmm, svm_w, svm_b, threshold=threshold, mode=mode)
    s = score_fn(Xs, shard.local_offsets)
    if not gather or world == 1:
        return s
    mx = max(shard.sizes)
    padded = s.new_zeros((mx, s.shape[1]))
    padded[:s.shape[0]] = s
    buf = [s.new_zeros((mx, s.shape[1])) for _ in shard.sizes]
    _all_gather(buf, padded, group)
    return torch.cat([t[:n] for t, n in zip(buf, shard.sizes)], 0)
