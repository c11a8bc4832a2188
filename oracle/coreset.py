"""CPU ORACLE of the feature-based coreset selection (NEXT-4) -- TEST
INFRASTRUCTURE ONLY (see oracle/__init__.py for who may import it).

Follows PAPER.md §3.1 "Feature-Based Coreset Selection" (Fig. 1)
step by step, in the paper's order and notation, on small volumes:

  1. Feature Extraction   f_k = the feature's vertex set in key frame k
  2. Feature Dilation     d_k = f_k plus neighbouring vertices, built with a
                          hash-based dictionary (a Python set) as the paper
                          does; occupancy grid of the cells d_k
                          touches, stored as bits at the voxel's Morton index
                          
  3. Bounding Box and Temporal Fusion: b_k = range of d_k, FBB = minimal
                          superset of all b_k
  4. Position Translation and Scaling: Eq. 1 (subtract the FBB centroid),
                          Eq. 2 (times 2 / Size^FBB) -> [-1, 1]
  5. Time Step Concatenation: d_k^t = ([t, x, y, z], v) pairs, Coreset =
                          union over k of d_k^t, Eq. 3

Readings where the paper is silent:
  R22 feature kinds (the paper names spatial / temporal / 4D features with
      "specific feature extraction methods"): interval  lo <= v <= hi;
      isosurface  |v - iso| <= eps, plus the 8 corners of every cell whose
      corner values straddle iso (min <= iso <= max); segmentation  v >= thr
      (connected-component filtering with minimum size 1, i.e. none).
  R23 "neighboring vertices": the 26-neighbourhood (3x3x3 cube,
      clamped at the volume boundary) -- enough for the 8-corner
      interpolation of every cell that touches f_k.
  R24 occupancy grid: one bit per CELL (X-1)(Y-1)(Z-1), set iff any of its 8
      corners is in d_k ("set to 1 if d_k intersects with the voxel");
      bit position = Morton index of the cell with bits interleaved from the
      least significant end (x, y, z at every bit position j while the axis
      has more than j bits, b_a = ceil(log2 cells_a)) -- the standard 3-way
      interleave (x in bit 0) on a cubic power-of-two grid, and a bijection
      onto [0, 2^(b_x+b_y+b_z)) on a rectangular one.
  R25 normalised coordinates ("x, y, and z ... normalized to range
      [-1, 1]"): vertex i of an axis with S vertices sits at -1 + 2 i/(S-1);
      Size^FBB and Origin^FBB are taken in those units; an FBB axis of a
      single vertex is padded to two (hi+1, or lo-1 at the upper boundary).
      Key frame k of n gets t = -1 + 2 k/(n-1) (0 when n = 1).
  R26 sample order: frame-major, then vertex z, y, x (row-major, x fastest);
      the coreset is a set, the order only fixes the output layout.
The library's encoder domain is [0, 1] (R2), so `to_unit()` maps the
[-1, 1] coordinates q of Eqs. 1-2 to (q + 1) / 2.

Every function here is pinned in tests/test_oracle_coreset.py against
closed forms, worked examples and a brute-force predicate scan that does not
use these functions.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np

INTERVAL, ISOSURFACE, SEGMENTATION = 0, 1, 2


class FeatureNotFound(ValueError):
    """No key frame contains the feature (no FBB can be formed)."""


# ------------------------------------------------------------ 1. extraction
def extract_feature(frame: np.ndarray, kind: int, p0: float, p1: float = 0.0) -> set:
    """f_k as a set of (x, y, z) vertices (R22).  frame is [Z][Y][X].
    interval: p0 = lo, p1 = hi; isosurface: p0 = iso, p1 = eps;
    segmentation: p0 = threshold."""
    Z, Y, X = frame.shape
    f = set()
    v = frame.astype(np.float64)
    if kind == INTERVAL:
        for z in range(Z):
            for y in range(Y):
                for x in range(X):
                    if p0 <= v[z, y, x] <= p1:
                        f.add((x, y, z))
    elif kind == SEGMENTATION:
        for z in range(Z):
            for y in range(Y):
                for x in range(X):
                    if v[z, y, x] >= p0:
                        f.add((x, y, z))
    elif kind == ISOSURFACE:
        iso, eps = p0, p1
        for z in range(Z):
            for y in range(Y):
                for x in range(X):
                    if abs(v[z, y, x] - iso) <= eps:
                        f.add((x, y, z))
        for z in range(Z - 1):
            for y in range(Y - 1):
                for x in range(X - 1):
                    corners = [(x + a, y + b, z + c) for c in (0, 1) for b in (0, 1) for a in (0, 1)]
                    vals = [v[cz, cy, cx] for (cx, cy, cz) in corners]
                    if min(vals) <= iso <= max(vals):
                        f.update(corners)
    else:
        raise ValueError("unknown feature kind")
    return f


# ------------------------------------------------------------ 2. dilation
def dilate_feature(f: set, dims: Tuple[int, int, int]) -> set:
    """d_k = f_k plus the 26 neighbours of each member, clamped (R23), in a
    hash-based dictionary."""
    X, Y, Z = dims
    d = set()
    for (x, y, z) in f:
        for c in (-1, 0, 1):
            for b in (-1, 0, 1):
                for a in (-1, 0, 1):
                    u = (x + a, y + b, z + c)
                    if 0 <= u[0] < X and 0 <= u[1] < Y and 0 <= u[2] < Z:
                        d.add(u)
    return d


def morton_bits(cells: Sequence[int]) -> List[int]:
    """b_a = bits to index cells_a (>= 0) per axis (R24)."""
    return [max(0, int(c - 1).bit_length()) for c in cells]


def morton_encode(x: int, y: int, z: int, bits: Sequence[int]) -> int:
    """R24 interleave: for j = 0, 1, ...: bit j of x, y, z (each axis while
    it has more than j bits), packed from bit 0 upwards."""
    v = (x, y, z)
    out, pos = 0, 0
    for j in range(max(bits) if bits else 0):
        for a in range(3):
            if bits[a] > j:
                out |= ((v[a] >> j) & 1) << pos
                pos += 1
    return out


def build_occupancy(d: set, dims: Tuple[int, int, int]) -> np.ndarray:
    """Occupancy bits of the cells touched by d_k (R24), as uint32 words
    (bit i of word w = Morton index 32 w + i)."""
    X, Y, Z = dims
    cells = (X - 1, Y - 1, Z - 1)
    bits = morton_bits(cells)
    nbits = 1 << sum(bits)
    words = np.zeros((nbits + 31) // 32, dtype=np.uint32)
    for z in range(Z - 1):
        for y in range(Y - 1):
            for x in range(X - 1):
                hit = any((x + a, y + b, z + c) in d for c in (0, 1) for b in (0, 1) for a in (0, 1))
                if hit:
                    m = morton_encode(x, y, z, bits)
                    words[m >> 5] |= np.uint32(1 << (m & 31))
    return words


# ------------------------------------------------------------ 3. boxes, FBB
def bounding_box(d: set) -> Tuple[Tuple[int, int, int], Tuple[int, int, int]] | None:
    """b_k: the range of d_k on x, y, z (None if d_k is empty)."""
    if not d:
        return None
    xs, ys, zs = zip(*d)
    return (min(xs), min(ys), min(zs)), (max(xs), max(ys), max(zs))


def fuse_fbb(boxes: Sequence, dims: Tuple[int, int, int]):
    """FBB = the minimal superset of every b_k; single-vertex axes are
    padded to two vertices (R25).  Raises FeatureNotFound if all are empty."""
    boxes = [b for b in boxes if b is not None]
    if not boxes:
        raise FeatureNotFound("no key frame contains the feature")
    lo = [min(b[0][a] for b in boxes) for a in range(3)]
    hi = [max(b[1][a] for b in boxes) for a in range(3)]
    for a in range(3):
        if hi[a] == lo[a]:
            if hi[a] + 1 < dims[a]:
                hi[a] += 1
            else:
                lo[a] -= 1
    return tuple(lo), tuple(hi)


def normalized(i: int, S: int) -> float:
    """Vertex i of an S-vertex axis in the paper's [-1, 1] units (R25)."""
    return -1.0 + 2.0 * i / (S - 1)


def to_fbb_coords(v: Tuple[int, int, int], fbb, dims) -> Tuple[float, float, float]:
    """Eq. 1 (translate by the FBB centroid) then Eq. 2 (scale by
    2 / Size^FBB), fp64, in normalised units."""
    lo, hi = fbb
    out = []
    for a in range(3):
        assert lo[a] <= v[a] <= hi[a], "vertex outside the FBB"
        nlo, nhi = normalized(lo[a], dims[a]), normalized(hi[a], dims[a])
        origin = 0.5 * (nlo + nhi)           # centroid of the FBB
        size = nhi - nlo                     # Size^FBB
        q = normalized(v[a], dims[a]) - origin           # Eq. 1
        q = q * (2.0 / size)                              # Eq. 2
        out.append(q)
    return tuple(out)


def to_unit(q: float) -> float:
    """[-1, 1] (paper) -> [0, 1] (encoder ABI domain, R2)."""
    return (q + 1.0) / 2.0


# ------------------------------------------------------------ 5. coreset
def build_coreset(vol: np.ndarray, kind: int, p0: float, p1: float = 0.0):
    """vol [n][Z][Y][X] of the n key frames (already normalised values).
    Returns (samples, fbb, occupancy): samples = list of ((t, x, y, z) in
    [-1,1], v) in R26 order; fbb = ((lo), (hi)) vertex indices; occupancy =
    per-frame uint32 word arrays."""
    n, Z, Y, X = vol.shape
    dims = (X, Y, Z)
    ds, boxes, occ = [], [], []
    for k in range(n):
        f = extract_feature(vol[k], kind, p0, p1)
        d = dilate_feature(f, dims)
        ds.append(d)
        occ.append(build_occupancy(d, dims))
        boxes.append(bounding_box(d))
    fbb = fuse_fbb(boxes, dims)
    samples = []
    for k in range(n):
        t = 0.0 if n == 1 else -1.0 + 2.0 * k / (n - 1)
        for (x, y, z) in sorted(ds[k], key=lambda u: (u[2], u[1], u[0])):
            q = to_fbb_coords((x, y, z), fbb, dims)
            samples.append(((t,) + q, float(vol[k, z, y, x])))   # d_k^t, Eq. 3 union
    return samples, fbb, occ


def samples_unit_f32(samples) -> Tuple[np.ndarray, np.ndarray]:
    """Samples as the library lays them out: float32 [M][4] coordinates
    (x, y, z, t) in [0, 1] (R2 order, P:79's [t,x,y,z] permuted) and float32
    labels [M]."""
    c = np.array([[to_unit(q[1]), to_unit(q[2]), to_unit(q[3]), to_unit(q[0])] for q, _ in samples],
                 dtype=np.float64).reshape(-1, 4)
    v = np.array([s[1] for s in samples], dtype=np.float64)
    return c.astype(np.float32), v.astype(np.float32)
