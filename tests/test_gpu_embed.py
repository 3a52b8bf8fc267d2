"""GPU parity of the PCA + xy embedding and of the raw-descriptor
-> FV path (embed + encode at D = m + 2 = 82, the paper's descriptor format) against the fp64
oracle (oracle.embed, then oracle.encode on the oracle's embedding).

Tolerances: k_embed (tcgen05, kind::tf32) splits both operands into tf32 hi + lo (relative
representation error <= 2^-21 per element) and accumulates 48 UMMAs in fp32, so |err| <= (3 * 2^-21 +
48 * 2^-23) * sum_k |b_ck (d_k - mean_k)| <= 1e-5 ||d - mean|| (Cauchy-Schwarz, orthonormal rows); the
FV bound is north_star's 1e-4 relative L2 (the embedding moves the encoder input by ~1e-7 relative)."""
import numpy as np
import pytest
import torch

import fvgen
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fv():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1604_03498_b200 as m
    return m


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("m,counts", [(80, [5000, 1, 0, 333]), (62, [1000, 2049]), (7, [130, 64])])
def test_embed_matches_oracle(fv, m, counts):
    mean, B = fvgen.make_pca(m, seed=11)
    gmm = fvgen.make_embedded_gmm(16, m, seed=12)
    raw, xy, off, wh = fvgen.make_raw_frames(gmm, (mean, B), counts, seed=13, img_wh=(320, 240))
    wh[-1] = [640, 480]
    E = fv.embed(dev(raw), dev(xy), dev(off), dev(wh), dev(mean), dev(B)).cpu().numpy()
    ref = oracle.embed(raw, xy, off, wh, mean, B)
    ld = (m + 2 + 3) // 4 * 4
    assert E.shape == (raw.shape[0], ld)
    bound = 1e-5 * np.linalg.norm(raw.astype(np.float64) - mean, axis=1)[:, None] + 1e-30
    assert np.all(np.abs(E[:, :m] - ref[:, :m]) <= bound)
    np.testing.assert_allclose(E[:, m:m + 2], ref[:, m:], rtol=1e-7)
    assert np.all(E[:, m + 2:] == 0)


@pytest.mark.parametrize("scale", [255.0, 1.0 / 512])
def test_embed_any_input_scale(fv, scale):
    """Unnormalised (0..255) and tiny SIFT values: the tf32 split keeps the fp32 exponent range, so the
    relative bound holds at any scale (an fp16 split would overflow or go subnormal); ragged tail."""
    m = 80
    mean, B = fvgen.make_pca(m, seed=14)
    gmm = fvgen.make_embedded_gmm(16, m, seed=15)
    raw, xy, off, wh = fvgen.make_raw_frames(gmm, (mean, B), [4001, 130], seed=16)
    raw = (raw * scale).astype(np.float32)
    mean = (mean * scale).astype(np.float32)
    E = fv.embed(dev(raw), dev(xy), dev(off), dev(wh), dev(mean), dev(B)).cpu().numpy()
    ref = oracle.embed(raw, xy, off, wh, mean, B)
    bound = 1e-5 * np.linalg.norm(raw.astype(np.float64) - mean, axis=1)[:, None] + 1e-30
    assert np.all(np.abs(E[:, :m] - ref[:, :m]) <= bound)
    np.testing.assert_allclose(E[:, m:m + 2], ref[:, m:], rtol=1e-7)


@pytest.mark.parametrize("tau", [0.0, 1e-6])
def test_raw_to_fv_d82_matches_oracle(fv, tau):
    """One 320x240 frame of 5000 raw descriptors + a 700-descriptor image, K=256, m=80 -> D=82 (wide
    kernel, D not a multiple of 4 through the padded row stride)."""
    m, K = 80, 256
    mean, B = fvgen.make_pca(m, seed=21)
    gmm_np = fvgen.make_embedded_gmm(K, m, seed=22)
    raw, xy, off, wh = fvgen.make_raw_frames(gmm_np, (mean, B), [5000, 700], seed=23)
    gmm = fv.GMM(*gmm_np)
    out = fv.embed_encode_batched(dev(raw), dev(xy), dev(off), dev(wh), dev(mean), dev(B), gmm,
                                  threshold=tau).cpu().numpy()
    E = oracle.embed(raw, xy, off, wh, mean, B)
    ref = oracle.encode_batched(E, off, *gmm_np, threshold=tau)
    rel = np.linalg.norm(out - ref, axis=1) / np.linalg.norm(ref, axis=1)
    print(f"D=82 tau={tau}: rel-L2 {rel}")
    assert out.shape == (2, 2 * K * 82) and np.all(rel < 1e-4)


def test_raw_to_fv_narrow_d64(fv):
    """m = 62 -> D = 64: the narrow kernel behind the embedding."""
    m, K = 62, 128
    mean, B = fvgen.make_pca(m, seed=31)
    gmm_np = fvgen.make_embedded_gmm(K, m, seed=32)
    raw, xy, off, wh = fvgen.make_raw_frames(gmm_np, (mean, B), [3000, 2500], seed=33)
    out = fv.embed_encode_batched(dev(raw), dev(xy), dev(off), dev(wh), dev(mean), dev(B), fv.GMM(*gmm_np),
                                  threshold=1e-6).cpu().numpy()
    ref = oracle.encode_batched(oracle.embed(raw, xy, off, wh, mean, B), off, *gmm_np, threshold=1e-6)
    rel = np.linalg.norm(out - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert np.all(rel < 1e-4)


@pytest.mark.parametrize("m,K", [(41, 33), (30, 256), (100, 64)])
def test_raw_to_fv_odd_dims(fv, m, K):
    """D = m + 2 not a multiple of 4 (43, 102) and odd K: the padded row stride carries the encoder, the
    finalize rescales a 2KD that is not a multiple of 4 (scalar path); narrow (D <= 64) and wide."""
    mean, B = fvgen.make_pca(m, seed=41)
    gmm_np = fvgen.make_embedded_gmm(K, m, seed=42)
    raw, xy, off, wh = fvgen.make_raw_frames(gmm_np, (mean, B), [1500, 0, 777, 2100], seed=43)
    out = fv.embed_encode_batched(dev(raw), dev(xy), dev(off), dev(wh), dev(mean), dev(B), fv.GMM(*gmm_np),
                                  threshold=1e-6).cpu().numpy()
    ref = oracle.encode_batched(oracle.embed(raw, xy, off, wh, mean, B), off, *gmm_np, threshold=1e-6)
    assert np.all(out[1] == 0)
    for b in (0, 2, 3):
        assert np.linalg.norm(out[b] - ref[b]) / np.linalg.norm(ref[b]) < 1e-4


def test_embed_many_small_images_per_tile(fv):
    """Hundreds of 0..9-descriptor images (several images in every 128-row tile, empty ones between):
    each row's keypoint is normalised by its own image's size (the epilogue's walk from the tile's
    first image)."""
    m = 30
    mean, B = fvgen.make_pca(m, seed=17)
    gmm = fvgen.make_embedded_gmm(8, m, seed=18)
    rng = np.random.default_rng(19)
    counts = [int(c) for c in rng.integers(0, 10, size=400)]
    raw, xy, off, wh = fvgen.make_raw_frames(gmm, (mean, B), counts, seed=20)
    wh = (wh * rng.uniform(0.5, 2.0, size=wh.shape)).astype(np.float32)  # a different size per image
    E = fv.embed(dev(raw), dev(xy), dev(off), dev(wh), dev(mean), dev(B)).cpu().numpy()
    ref = oracle.embed(raw, xy, off, wh, mean, B)
    np.testing.assert_allclose(E[:, m:m + 2], ref[:, m:], rtol=1e-7)
    bound = 1e-5 * np.linalg.norm(raw.astype(np.float64) - mean, axis=1)[:, None] + 1e-30
    assert np.all(np.abs(E[:, :m] - ref[:, :m]) <= bound)
