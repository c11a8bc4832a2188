"""Pins of the coreset-selection oracle (NEXT-4; oracle/coreset.py) against
what the paper and the mathematics fix -- worked examples (SPEC S:139-219,
each cited), closed forms of Eqs. 1-2, invariants, and a brute-force
per-vertex predicate scan written independently of the oracle (dense numpy
arrays instead of the oracle's hash-set pipeline).  CPU only."""
import itertools

import numpy as np
import pytest

from oracle import coreset as C


# ------------------------------------------------------------ extraction
def test_extract_interval_trivial():
    """constant-0 frame, interval [0.4, 0.6] -> empty; constant
    0.5 -> every vertex."""
    z = np.zeros((3, 4, 5), np.float32)
    assert C.extract_feature(z, C.INTERVAL, 0.4, 0.6) == set()
    h = np.full((3, 4, 5), 0.5, np.float32)
    assert len(C.extract_feature(h, C.INTERVAL, 0.4, 0.6)) == 60


def test_extract_isosurface_ramp_example():
    """a ramp 0, .25, .5, .75, 1 along x with isovalue 0.5, eps 0 ->
    the vertex of value 0.5 plus the corners of the straddling cells (values
    0.25 and 0.75); here on a 5x2x2 grid (constant along y, z)."""
    ramp = np.array([0, 0.25, 0.5, 0.75, 1.0], np.float32)
    vol = np.broadcast_to(ramp, (2, 2, 5)).copy()
    f = C.extract_feature(vol, C.ISOSURFACE, 0.5, 0.0)
    assert sorted({x for (x, _, _) in f}) == [1, 2, 3]
    assert len(f) == 3 * 4


def test_extract_segmentation_threshold():
    v = np.arange(24, dtype=np.float32).reshape(2, 3, 4) / 23.0
    f = C.extract_feature(v, C.SEGMENTATION, 0.5)
    assert f == {(x, y, z) for z in range(2) for y in range(3) for x in range(4) if v[z, y, x] >= 0.5}


# ------------------------------------------------------------ dilation
def test_dilation_examples():
    """empty -> empty; an interior vertex -> 27; a grid corner
    -> 8 (clamped neighbourhood)."""
    dims = (5, 5, 5)
    assert C.dilate_feature(set(), dims) == set()
    assert len(C.dilate_feature({(2, 2, 2)}, dims)) == 27
    assert len(C.dilate_feature({(0, 0, 0)}, dims)) == 8
    assert len(C.dilate_feature({(4, 2, 2)}, dims)) == 18   # face vertex: 2 x 3 x 3
    assert len(C.dilate_feature({(4, 0, 2)}, dims)) == 12   # edge vertex: 2 x 2 x 3


# ------------------------------------------------------------ Morton / occupancy
def part1by2(v: int) -> int:
    """Standard 3-way bit spread (magic-number form, independent of the
    oracle's per-bit loop)."""
    v &= 0x1FFFFF
    v = (v | (v << 32)) & 0x1F00000000FFFF
    v = (v | (v << 16)) & 0x1F0000FF0000FF
    v = (v | (v << 8)) & 0x100F00F00F00F00F
    v = (v | (v << 4)) & 0x10C30C30C30C30C3
    v = (v | (v << 2)) & 0x1249249249249249
    return v


def test_morton_standard_on_cubic_grids():
    """R24 equals the standard interleave (x in bit 0) on cubic power-of-two
    grids: S:179-180 (0,0,0) -> 0, (1,1,1) -> 7; (3,0,2) -> bits x0,x1,z1 =
    1 + 8 + 32 = 41 (SPEC's printed 37 contradicts its own x-in-bit-0 rule;
    DESIGN.md R24)."""
    bits = [5, 5, 5]
    assert C.morton_encode(0, 0, 0, bits) == 0
    assert C.morton_encode(1, 1, 1, bits) == 7
    assert C.morton_encode(3, 0, 2, bits) == 41
    g = np.random.default_rng(0)
    for _ in range(500):
        x, y, z = (int(a) for a in g.integers(0, 32, 3))
        assert C.morton_encode(x, y, z, bits) == part1by2(x) | part1by2(y) << 1 | part1by2(z) << 2


@pytest.mark.parametrize("cells", [(5, 3, 2), (8, 8, 1), (1, 1, 1), (7, 16, 3), (33, 2, 5)])
def test_morton_bijective_rectangular(cells):
    bits = C.morton_bits(cells)
    idx = {C.morton_encode(x, y, z, bits) for z in range(2 ** bits[2]) for y in range(2 ** bits[1])
           for x in range(2 ** bits[0])}
    assert idx == set(range(1 << sum(bits)))


def test_occupancy_examples():
    """empty -> all zero; all vertices -> every cell set; a single
    vertex (1,1,1) of a 3^3-vertex grid -> exactly its 8 incident cells."""
    dims = (3, 3, 3)
    assert not C.build_occupancy(set(), dims).any()
    allv = {(x, y, z) for x in range(3) for y in range(3) for z in range(3)}
    w = C.build_occupancy(allv, dims)
    assert int(sum(bin(int(a)).count("1") for a in w)) == 8
    w = C.build_occupancy({(1, 1, 1)}, dims)
    assert int(sum(bin(int(a)).count("1") for a in w)) == 8
    dims = (6, 4, 3)   # rectangular: 5 x 3 x 2 cells
    allv = {(x, y, z) for x in range(6) for y in range(4) for z in range(3)}
    w = C.build_occupancy(allv, dims)
    assert int(sum(bin(int(a)).count("1") for a in w)) == 30


# ------------------------------------------------------------ FBB, Eqs. 1-2
def test_fuse_fbb_examples():
    """S:186-188 plus the empty and single-vertex cases."""
    dims = (10, 10, 10)
    b = ((1, 2, 3), (4, 5, 6))
    assert C.fuse_fbb([b], dims) == b
    assert C.fuse_fbb([((0, 1, 1), (4, 2, 2)), ((2, 0, 1), (6, 2, 3))], dims) == ((0, 0, 1), (6, 2, 3))
    assert C.fuse_fbb([((0, 0, 0), (9, 9, 9)), b], dims) == ((0, 0, 0), (9, 9, 9))
    assert C.fuse_fbb([None, ((3, 9, 2), (3, 9, 5))], dims) == ((3, 8, 2), (4, 9, 5))
    with pytest.raises(C.FeatureNotFound):
        C.fuse_fbb([None, None], dims)


def test_eqs_1_2_closed_forms():
    """the FBB centroid -> 0, the min corner -> -1, the max
    corner -> +1, halfway between centroid and max on x -> 0.5."""
    dims = (21, 11, 9)
    fbb = ((4, 2, 0), (16, 8, 8))
    assert C.to_fbb_coords((10, 5, 4), fbb, dims) == pytest.approx((0, 0, 0), abs=1e-12)
    assert C.to_fbb_coords((4, 2, 0), fbb, dims) == pytest.approx((-1, -1, -1), abs=1e-12)
    assert C.to_fbb_coords((16, 8, 8), fbb, dims) == pytest.approx((1, 1, 1), abs=1e-12)
    assert C.to_fbb_coords((13, 5, 4), fbb, dims) == pytest.approx((0.5, 0, 0), abs=1e-12)
    with pytest.raises(AssertionError):
        C.to_fbb_coords((3, 5, 4), fbb, dims)


# ------------------------------------------------------------ brute force
def brute_force(vol, kind, p0, p1=0.0):
    """Independent scan: per vertex feature predicate on dense arrays, then a
    3x3x3 sliding max (np.pad + shifts) for the dilation; FBB from the
    dilated masks; samples in frame-major row-major order."""
    n, Z, Y, X = vol.shape
    v = vol.astype(np.float64)
    masks = []
    for k in range(n):
        a = v[k]
        if kind == C.INTERVAL:
            f = (a >= p0) & (a <= p1)
        elif kind == C.SEGMENTATION:
            f = a >= p0
        else:
            f = np.abs(a - p0) <= p1
            cmin = np.full((Z - 1, Y - 1, X - 1), np.inf)
            cmax = np.full((Z - 1, Y - 1, X - 1), -np.inf)
            for c, b, e in itertools.product((0, 1), repeat=3):
                s = a[c:Z - 1 + c, b:Y - 1 + b, e:X - 1 + e]
                cmin, cmax = np.minimum(cmin, s), np.maximum(cmax, s)
            st = (cmin <= p0) & (p0 <= cmax)
            for c, b, e in itertools.product((0, 1), repeat=3):
                f[c:Z - 1 + c, b:Y - 1 + b, e:X - 1 + e] |= st
        fp = np.pad(f, 1)
        d = np.zeros_like(f)
        for c, b, e in itertools.product((0, 1, 2), repeat=3):
            d |= fp[c:c + Z, b:b + Y, e:e + X]
        masks.append(d)
    return masks


def random_volume(seed, n=3, shape=(6, 7, 9)):
    g = np.random.default_rng(seed)
    return g.random((n,) + shape).astype(np.float32)


@pytest.mark.parametrize("kind,p0,p1", [(C.INTERVAL, 0.45, 0.5), (C.SEGMENTATION, 0.93, 0.0),
                                        (C.ISOSURFACE, 0.97, 0.002)])
def test_build_coreset_equals_brute_force(kind, p0, p1):
    """build_coreset equals a brute-force per-(frame, vertex) scan of
    the dilated-feature predicate; Eq. 3 union, FBB = the padded range of all
    dilated masks, coordinates per Eqs. 1-2, t per R25."""
    vol = random_volume(kind)
    n, Z, Y, X = vol.shape
    samples, fbb, occ = C.build_coreset(vol, kind, p0, p1)
    masks = brute_force(vol, kind, p0, p1)
    exp = []
    for k in range(n):
        for z, y, x in zip(*np.nonzero(masks[k])):
            exp.append((k, int(x), int(y), int(z)))
    assert len(samples) == len(exp)
    allm = np.any(np.stack(masks), axis=0)
    zs, ys, xs = np.nonzero(allm)
    lo, hi = [xs.min(), ys.min(), zs.min()], [xs.max(), ys.max(), zs.max()]
    for a, D in enumerate((X, Y, Z)):
        if lo[a] == hi[a]:
            hi[a], lo[a] = (hi[a] + 1, lo[a]) if hi[a] + 1 < D else (hi[a], lo[a] - 1)
    assert fbb == (tuple(int(a) for a in lo), tuple(int(a) for a in hi))
    for (q, val), (k, x, y, z) in zip(samples, exp):
        t = -1 + 2 * k / (n - 1)
        xyz = [-1 + 2 * (c - lo[a]) / (hi[a] - lo[a]) for a, c in enumerate((x, y, z))]
        assert q == pytest.approx((t, *xyz), abs=1e-12)
        assert val == vol[k, z, y, x]


def test_invariants_and_degenerate_specs():
    """f in d and every cell meeting f has its 8 corners in d;
    b_k inside the FBB; coordinates in [-1,1]^4.  A spec that matches
    nothing raises FeatureNotFound; one that matches everything gives
    n X Y Z samples and the full FBB."""
    vol = random_volume(5)
    n, Z, Y, X = vol.shape
    dims = (X, Y, Z)
    f = C.extract_feature(vol[0], C.INTERVAL, 0.3, 0.4)
    d = C.dilate_feature(f, dims)
    assert f <= d
    for (x, y, z) in f:
        for cx, cy, cz in itertools.product((x - 1, x), (y - 1, y), (z - 1, z)):
            if 0 <= cx < X - 1 and 0 <= cy < Y - 1 and 0 <= cz < Z - 1:
                for a, b, c in itertools.product((0, 1), repeat=3):
                    assert (cx + a, cy + b, cz + c) in d
    samples, fbb, _ = C.build_coreset(vol, C.INTERVAL, 0.3, 0.4)
    assert all(-1 - 1e-12 <= c <= 1 + 1e-12 for q, _ in samples for c in q)
    with pytest.raises(C.FeatureNotFound):
        C.build_coreset(vol, C.INTERVAL, 2.0, 3.0)
    samples, fbb, occ = C.build_coreset(vol, C.INTERVAL, -1.0, 2.0)
    assert len(samples) == n * X * Y * Z
    assert fbb == ((0, 0, 0), (X - 1, Y - 1, Z - 1))


def test_moving_gaussian_coreset_is_small_and_covers_sweep():
    """a moving Gaussian with a segmentation threshold gives a coreset
    strictly smaller than n x the full vertex count, and the FBB covers the
    blob's swept extent."""
    n, S = 4, 12
    z, y, x = np.meshgrid(*(np.arange(S) / (S - 1),) * 3, indexing="ij")
    vol = np.stack([np.exp(-((x - 0.25 - 0.15 * k) ** 2 + (y - 0.5) ** 2 + (z - 0.5) ** 2) / (2 * 0.08 ** 2))
                    for k in range(n)]).astype(np.float32)
    samples, fbb, occ = C.build_coreset(vol, C.SEGMENTATION, 0.5)
    assert 0 < len(samples) < n * S ** 3
    for k in range(n):
        cx = int(round((0.25 + 0.15 * k) * (S - 1)))
        assert fbb[0][0] <= cx <= fbb[1][0]
    u, v = C.samples_unit_f32(samples)
    assert u.dtype == np.float32 and np.all((u >= 0) & (u <= 1))
