"""NEXT-4 GPU parity: fh_coreset_build / fh_coreset_emit (through the C ABI)
against the coreset oracle (oracle/coreset.py) on the same seeded volumes.
Bars: masks, counts, FBB and occupancy bits bit-exact; sample coordinates
bit-exact float32 (Eqs. 1-2 then (q+1)/2 is (i-lo)/(hi-lo) rounded once on
both sides, R25); labels bit-exact.  -m gpu."""
import numpy as np
import pytest
import torch

from oracle import coreset as C
import workloads as W

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2507_03836_b200 import fhash as fh


def f32(x):
    return float(np.float32(x))


def run(vol, kind, p0, p1=0.0):
    v = torch.from_numpy(np.ascontiguousarray(vol)).cuda()
    cs = fh.Coreset(v, kind, f32(p0), f32(p1))
    coords, values = cs.emit()
    return cs, coords.cpu().numpy(), values.cpu().numpy()


def check_against_oracle(vol, kind, p0, p1=0.0):
    cs, coords, values = run(vol, kind, p0, p1)
    # the oracle compares against the same float32 thresholds
    try:
        samples, fbb, occ = C.build_coreset(vol, kind, f32(p0), f32(p1))
    except C.FeatureNotFound:
        assert cs.count == 0 and cs.fbb is None       # the paper's feature-not-found case
        assert not cs.occupancy.any()
        return cs
    assert cs.count == len(samples)
    assert cs.fbb == fbb
    u, lab = C.samples_unit_f32(samples)
    assert np.array_equal(coords.view(np.uint32), u.view(np.uint32))
    assert np.array_equal(values, lab)
    occ_gpu = cs.occupancy.cpu().numpy().view(np.uint32)
    for k in range(vol.shape[0]):
        assert np.array_equal(occ_gpu[k], occ[k])
    return cs


def rand_vol(seed, n=3, shape=(6, 7, 9)):
    return np.random.default_rng(seed).random((n,) + shape).astype(np.float32)


@pytest.mark.parametrize("kind,p0,p1", [(C.INTERVAL, 0.45, 0.5), (C.SEGMENTATION, 0.93, 0.0),
                                        (C.ISOSURFACE, 0.97, 0.002), (C.ISOSURFACE, 0.5, 0.0)])
@pytest.mark.parametrize("shape", [(6, 7, 9), (2, 2, 2), (5, 3, 33), (17, 9, 4), (9, 9, 2), (2, 9, 9),
                                   # X = 97..128: Wx = 4 (the 4-words-per-thread dilation); X = 130: Wx = 5
                                   # (one word per thread); 9x9x100 / 5x5x5: std5 occupancy with 8 words per
                                   # thread / a 2-word bitmap (ragged tail); 3x4x128: non-std5 rows path
                                   # 3x3x129: Wc = 4 cell words, Wx = 5 vertex words (the carry word)
                                   # Y % 4 == 0 with Wx in {4, 8} (3x8x256, 2x12x100)
                                   (9, 9, 100), (4, 5, 130), (3, 4, 128), (5, 5, 5), (3, 3, 129),
                                   (3, 8, 256), (2, 12, 100)])
def test_coreset_parity(kind, p0, p1, shape):
    check_against_oracle(rand_vol(kind * 7 + shape[0], 3, shape), kind, p0, p1)


def test_coreset_single_frame_and_ramp_example():
    """n = 1 (t = 0 for every sample) and S:154's isosurface ramp."""
    check_against_oracle(rand_vol(3, 1, (5, 6, 7)), C.SEGMENTATION, 0.8)
    ramp = np.array([0, 0.25, 0.5, 0.75, 1.0], np.float32)
    vol = np.broadcast_to(ramp, (2, 2, 2, 5)).copy()
    check_against_oracle(vol, C.ISOSURFACE, 0.5, 0.0)


def test_coreset_feature_not_found_and_everything():
    vol = rand_vol(4)
    cs, _, _ = run(vol, C.INTERVAL, 2.0, 3.0)
    assert cs.count == 0 and cs.fbb is None
    n, Z, Y, X = vol.shape
    cs = check_against_oracle(vol, C.INTERVAL, -1.0, 2.0)
    assert cs.count == n * X * Y * Z and cs.fbb == ((0, 0, 0), (X - 1, Y - 1, Z - 1))


def test_coreset_moving_gaussian_oracle():
    """S:203's moving-Gaussian case at 4 x 20^3 against the oracle."""
    n, S = 4, 20
    z, y, x = np.meshgrid(*(np.arange(S) / (S - 1),) * 3, indexing="ij")
    vol = np.stack([np.exp(-((x - 0.25 - 0.15 * k) ** 2 + (y - 0.5) ** 2 + (z - 0.5) ** 2) / (2 * 0.08 ** 2))
                    for k in range(n)]).astype(np.float32)
    cs = check_against_oracle(vol, C.SEGMENTATION, 0.5)
    assert 0 < cs.count < n * S ** 3


def test_coreset_full_size_properties():
    """The bench's shape (cfg3 field: 8 key frames of the 256^3 Gaussian-blob
    volume, segmentation at 0.5): the mask count equals a vectorised dense
    scan of the dilated predicate; every emitted sample's vertex is inside
    the FBB, its label is the volume value, and it lies within one vertex of
    a feature vertex; samples are in frame-major row-major order."""
    blobs = W.gaussian_blob_params(W.rng(0))
    field = fh.field_gaussian_blobs(256, 32, blobs)
    keys = field[::4].contiguous()                     # 8 key frames
    cs = fh.Coreset(keys, C.SEGMENTATION, 0.5)
    coords, values = cs.emit()
    vol = keys.cpu().numpy()
    n, Z, Y, X = vol.shape
    f = vol >= np.float32(0.5)
    d = np.zeros_like(f)
    fp = np.pad(f, ((0, 0), (1, 1), (1, 1), (1, 1)))
    for c in range(3):
        for b in range(3):
            for a in range(3):
                d |= fp[:, c:c + Z, b:b + Y, a:a + X]
    assert cs.count == int(d.sum())
    (lo, hi) = cs.fbb
    kk, zz, yy, xx = np.nonzero(d)
    assert (xx.min(), yy.min(), zz.min()) == lo and (xx.max(), yy.max(), zz.max()) == hi
    c = coords.cpu().numpy().astype(np.float64)
    v = values.cpu().numpy()
    idx = np.random.default_rng(0).choice(cs.count, 4096, replace=False)
    for i in idx:
        k = int(round(c[i, 3] * (n - 1)))
        x, y, z = (int(round(lo[a] + c[i, a] * (hi[a] - lo[a]))) for a in range(3))
        assert d[k, z, y, x] and v[i] == vol[k, z, y, x]
    # order: (k, z, y, x) non-decreasing
    key = np.round(c[:, 3] * (n - 1)) * 1e12 + np.round(c[:, 2] * (hi[2] - lo[2])) * 1e8 + \
        np.round(c[:, 1] * (hi[1] - lo[1])) * 1e4 + np.round(c[:, 0] * (hi[0] - lo[0]))
    assert np.all(np.diff(key) > 0)
