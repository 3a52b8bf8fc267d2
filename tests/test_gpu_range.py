"""The fp16 operand domain and empty inputs (include/gpufv.h "Range report").

The split contractions represent features and GMM coefficients as fp16 hi/lo pairs.  Inputs outside
that range must never come back as finite garbage: either the result is correct (within the north_star
tolerance against the oracle), or the image's output is NaN AND fv_range_flags reports it.  Alg.1's
distance is defined for any input (Alg.1 l.4-5), so both outcomes are checked against
the oracle's direct-form result."""
import numpy as np
import pytest
import torch

import fvgen
import oracle

pytestmark = pytest.mark.gpu

FV_RTOL = 1e-4


@pytest.fixture(scope="module")
def fv():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1604_03498_b200 as m
    return m


def rel_l2(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def rms_and_c(gmm_np):
    pi, mu, var = (a.astype(np.float64) for a in gmm_np)
    w = pi / pi.sum()
    c = (w[:, None] * mu).sum(0)
    rms = np.sqrt((w[:, None] * (var + mu * mu)).sum(0) - c * c)
    return rms, c


def encode_with_flags(fv, X, off, gmm_np, tau, K=None):
    gmm = fv.GMM(*gmm_np)
    ws = fv.Workspace()
    out = fv.encode_batched(dev(X), dev(off), gmm, threshold=tau, ws=ws).cpu().numpy()
    flags = fv.range_flags(ws, X.shape[0], len(off) - 1, gmm).cpu().numpy()
    return out, flags


def either_correct_or_reported(out, flags, ref):
    for b in range(len(flags)):
        if flags[b]:
            assert np.all(np.isnan(out[b])), f"image {b} flagged but not NaN"
        else:
            assert np.all(np.isfinite(out[b])), f"image {b} not finite and not flagged"
            assert rel_l2(out[b], ref[b]) <= FV_RTOL, (b, rel_l2(out[b], ref[b]))


@pytest.mark.parametrize("K,D", [(256, 64), (512, 128)])
@pytest.mark.parametrize("tau", [0.0, 1e-6])
def test_outlier_descriptor_far_outside_range_is_reported(fv, K, D, tau):
    """One descriptor at 2000 RMS in one dimension of image 1 (the squared feature overflows fp16): image
    1 is NaN and flagged, images 0 and 2 are unaffected and match the oracle."""
    gmm_np = fvgen.make_gmm(K, D, seed=31)
    X, off = fvgen.make_batch(gmm_np, [700, 900, 300], seed_base=32)
    rms, c = rms_and_c(gmm_np)
    X[off[1] + 17, 3] = np.float32(c[3] + 2000 * rms[3])
    out, flags = encode_with_flags(fv, X, off, gmm_np, tau)
    assert list(flags) == [0, 1, 0]
    assert np.all(np.isnan(out[1]))
    ref = oracle.encode_batched(X, off, *gmm_np, threshold=tau)
    for b in (0, 2):
        assert rel_l2(out[b], ref[b]) <= FV_RTOL


@pytest.mark.parametrize("k_rms", [100.0, 300.0, 600.0])
def test_outlier_descriptor_either_correct_or_reported(fv, k_rms):
    """Outliers at 100 / 300 / 600 RMS (the limit is 256-512 RMS, depending on where RMS falls between
    powers of two): within range the FV matches the oracle, beyond it the image is NaN and flagged."""
    gmm_np = fvgen.make_gmm(256, 64, seed=33)
    X, off = fvgen.make_batch(gmm_np, [2000, 2000], seed_base=34)
    rms, c = rms_and_c(gmm_np)
    for k in (0, 20, 63):
        X[off[1] + 5 + k, k] = np.float32(c[k] - k_rms * rms[k])
    out, flags = encode_with_flags(fv, X, off, gmm_np, 0.0)
    ref = oracle.encode_batched(X, off, *gmm_np)
    assert flags[0] == 0
    either_correct_or_reported(out, flags, ref)
    if k_rms <= 100:
        assert flags[1] == 0
    if k_rms >= 600:
        assert flags[1] == 1


@pytest.mark.parametrize("shrink", [50.0, 200.0, 1000.0])
def test_narrow_component_either_correct_or_reported(fv, shrink):
    """One component whose standard deviation in one dimension is RMS/shrink (its -1/(2 var) coefficient
    leaves the fp16 range beyond ~RMS/150): correct, or every image NaN with the GMM bit set."""
    pi, mu, var = (a.copy() for a in fvgen.make_gmm(256, 64, seed=35))
    rms, c = rms_and_c((pi, mu, var))
    var[7, 11] = np.float32((rms[11] / shrink) ** 2)
    X, off = fvgen.make_batch((pi, mu, var), [1500, 800], seed_base=36)
    out, flags = encode_with_flags(fv, X, off, (pi, mu, var), 0.0)
    ref = oracle.encode_batched(X, off, pi, mu, var)
    either_correct_or_reported(out, flags, ref)
    if shrink >= 1000:
        assert np.all(flags & 2)
    if shrink <= 50:
        assert not np.any(flags)


def test_nonfinite_descriptor_is_reported(fv):
    gmm_np = fvgen.make_gmm(128, 32, seed=37)
    X, off = fvgen.make_batch(gmm_np, [300, 300, 300], seed_base=38)
    X[off[2] + 3, 5] = np.nan
    X[off[0] + 1, 0] = np.inf
    out, flags = encode_with_flags(fv, X, off, gmm_np, 1e-6)
    assert list(flags) == [1, 0, 1]
    assert np.all(np.isnan(out[0])) and np.all(np.isnan(out[2]))
    assert rel_l2(out[1], oracle.encode(X[off[1]:off[2]], *gmm_np, threshold=1e-6)) <= FV_RTOL


def test_flags_follow_the_host_pipeline_chunks(fv):
    """fv_encode_batched_host runs the batch in chunks; the flags land at the batch's image indices."""
    gmm_np = fvgen.make_gmm(256, 64, seed=39)
    counts = [400] * 40
    X, off = fvgen.make_batch(gmm_np, counts, seed_base=40)
    rms, c = rms_and_c(gmm_np)
    for b in (3, 26, 39):
        X[off[b] + 9, 2] = np.float32(c[2] + 5000 * rms[2])
    gmm = fv.GMM(*gmm_np)
    ws = fv.Workspace()
    out = fv.encode_batched_host(torch.from_numpy(X).pin_memory(), torch.from_numpy(off), gmm, ws=ws).numpy()
    flags = fv.range_flags(ws, X.shape[0], len(counts), gmm).cpu().numpy()
    assert sorted(np.nonzero(flags)[0].tolist()) == [3, 26, 39]
    assert np.all(np.isnan(out[[3, 26, 39]]))
    ok = [b for b in range(40) if b not in (3, 26, 39)]
    assert np.all(np.isfinite(out[ok]))


def test_in_range_inputs_are_never_flagged(fv):
    """The acceptance and both stress generators stay in range."""
    for kind, f in (("acceptance", 0.3), ("acceptance", 0.15), ("peaked", 0.3)):
        gmm_np = fvgen.make_gmm(256, 64, seed=41, f=f, kind=kind)
        X, off = fvgen.make_batch(gmm_np, [3000, 1000], seed_base=42)
        out, flags = encode_with_flags(fv, X, off, gmm_np, 1e-6)
        assert not np.any(flags) and np.all(np.isfinite(out)), kind


# ------------------------------------------------------------------ empty inputs (reading A11)
def test_empty_set_and_all_empty_batch(fv):
    """N = 0 (X may be a NULL pointer) gives an all-zero FV; a batch whose images are all empty gives
    all-zero FVs; stats of an empty shard are zero with N = 0 (the descriptor-sharded path)."""
    for K, D in ((256, 64), (512, 128)):
        gmm = fv.GMM(*fvgen.make_gmm(K, D, seed=43))
        X0 = torch.empty(0, D, dtype=torch.float32, device="cuda")
        assert torch.count_nonzero(fv.encode(X0, gmm)).item() == 0
        off = torch.zeros(4, dtype=torch.int64, device="cuda")
        out = fv.encode_batched(X0, off, gmm, threshold=1e-6)
        assert out.shape == (3, 2 * K * D) and torch.count_nonzero(out).item() == 0
        st = fv.stats_batched(X0, torch.zeros(2, dtype=torch.int64, device="cuda"), gmm)
        assert torch.count_nonzero(st).item() == 0
        assert torch.count_nonzero(fv.finalize(st, gmm)).item() == 0


def test_binding_rejects_host_offsets(fv):
    gmm = fv.GMM(*fvgen.make_gmm(16, 8, seed=44))
    X = torch.zeros(10, 8, device="cuda")
    with pytest.raises(ValueError):
        fv.stats_batched(X, torch.tensor([0, 10]), gmm)
    with pytest.raises(ValueError):
        fv.encode_scored_batched(X, torch.tensor([0, 10]), gmm, torch.zeros(1, 2 * 16 * 8, device="cuda"))


@pytest.mark.parametrize("K", [256, 100])
def test_single_frame_fused_schedule_reports_range(fv, K):
    """A single frame takes the fused schedule (no k_schedule: per-CTA flag words ORed by the finalize).
    An outlier row makes the frame NaN and flagged; the next call on the same workspace with clean data
    clears the flag (the words are written unconditionally, nothing relies on prior zeroing)."""
    gmm_np = fvgen.make_gmm(K, 64, seed=43)
    X, off = fvgen.make_batch(gmm_np, [5000], seed_base=44)
    rms, c = rms_and_c(gmm_np)
    bad = X.copy()
    bad[4321, 7] = np.float32(c[7] + 2000 * rms[7])
    gmm = fv.GMM(*gmm_np)
    ws = fv.Workspace()
    out = fv.encode(dev(bad), gmm, threshold=1e-6, ws=ws).cpu().numpy()
    assert np.all(np.isnan(out))
    assert list(fv.range_flags(ws, 5000, 1, gmm).cpu().numpy()) == [1]
    out = fv.encode(dev(X), gmm, threshold=1e-6, ws=ws).cpu().numpy()
    assert list(fv.range_flags(ws, 5000, 1, gmm).cpu().numpy()) == [0]
    assert rel_l2(out, oracle.encode(X, *gmm_np, threshold=1e-6)) <= FV_RTOL
