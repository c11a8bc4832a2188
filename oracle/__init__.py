"""CPU ORACLE for the F-Hash encode and train step -- TEST INFRASTRUCTURE.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import this package.  It shares no code with the
CUDA path (`paper_2507_03836_b200/`) and never imports it.

  * fhash_oracle.c  -- level builder (Eqs. 4-9), cell location, the 16
                       corner indices, fp64 forward / backward, stats.
  * train.py        -- MLP forward/backward, MSE, Adam in fp64 numpy.
  * coreset.py      -- NEXT-4 feature-based coreset selection (§3.1, Eqs.
                       1-3): extraction, dilation, occupancy bits, FBB,
                       Eqs. 1-2 coordinates, the Eq. 3 union.

Parity-pin status of each function is listed in DESIGN.md §4.  The capped
(hashed) level index (reading R5: the paper never caps) is pinned by values
worked out by hand from its definition (tests/golden/r5_hash.json), the
x-adjacency property and brute-force statistics.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fhash_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

GCC_FLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *GCC_FLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        u32p = ctypes.POINTER(ctypes.c_uint32)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        i32p = ctypes.POINTER(ctypes.c_int32)
        f32p = ctypes.POINTER(ctypes.c_float)
        f64p = ctypes.POINTER(ctypes.c_double)
        L.fho_fold_schedule.argtypes = [u32p, ctypes.c_uint32, ctypes.c_uint32, u32p, ctypes.c_int]
        L.fho_fold_schedule.restype = ctypes.c_int
        L.fho_build_levels.argtypes = [u32p, ctypes.c_int, ctypes.c_uint64, u64p, u64p, i32p, u64p]
        L.fho_build_levels.restype = ctypes.c_uint64
        L.fho_fhash.argtypes = [u32p] + [ctypes.c_uint64] * 4
        L.fho_fhash.restype = ctypes.c_uint64
        L.fho_brick_index.argtypes = [u32p] + [ctypes.c_uint64] * 4
        L.fho_brick_index.restype = ctypes.c_uint64
        L.fho_spatial_hash.argtypes = [ctypes.c_uint32] * 4 + [ctypes.c_uint64]
        L.fho_spatial_hash.restype = ctypes.c_uint64
        common = [u32p, i32p, u64p, u64p, ctypes.c_int]
        L.fho_encode_indices.argtypes = common + [f32p, ctypes.c_int64, u32p, f64p]
        L.fho_encode_indices.restype = ctypes.c_int64
        L.fho_encode_fwd.argtypes = common + [ctypes.c_int, f32p, ctypes.c_int64, f64p, f64p, f64p]
        L.fho_encode_fwd.restype = None
        L.fho_encode_bwd.argtypes = common + [ctypes.c_int, f32p, ctypes.c_int64, f64p, f64p, f64p]
        L.fho_encode_bwd.restype = None
        L.fho_level_stats.argtypes = [u32p, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, u64p, u64p]
        L.fho_level_stats.restype = ctypes.c_int
        mcommon = [u32p, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint64]
        L.fho_mhe_indices.argtypes = mcommon + [f32p, ctypes.c_int64, u32p, f64p]
        L.fho_mhe_indices.restype = ctypes.c_int64
        L.fho_mhe_fwd.argtypes = mcommon + [ctypes.c_int, f32p, ctypes.c_int64, f64p, f64p, f64p]
        L.fho_mhe_fwd.restype = None
        L.fho_mhe_bwd.argtypes = mcommon + [ctypes.c_int, f32p, ctypes.c_int64, f64p, f64p, f64p]
        L.fho_mhe_bwd.restype = None
        L.fho_mhe_level_stats.argtypes = [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64, u64p, u64p]
        L.fho_mhe_level_stats.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _c(a, dtype) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=dtype)


def fold_schedule(S_xyz: Sequence[int], n_t: int, fold: int, max_L: int = 64):
    """Eqs. 4-8, paper order (level 1 = native first).
    Returns a list of (Rx, Ry, Rz, Rt)."""
    S = _c(S_xyz, np.uint32)
    out = np.zeros((max_L, 4), np.uint32)
    L = lib().fho_fold_schedule(_p(S, ctypes.c_uint32), n_t, fold, _p(out, ctypes.c_uint32), max_L)
    if L < 0:
        raise ValueError(f"fold_schedule: bad arguments ({L})")
    return [tuple(int(v) for v in row) for row in out[:L]]


class Levels:
    """Oracle level table (a1).  res: [L][4] (x,y,z,t) vertex counts."""

    def __init__(self, res: Sequence[Sequence[int]], cap: int = 0, lin: int = 0):
        """lin: 0 = Eq. 9 row-major; 1 = brick (tiled Z-order) order
        of the bijective levels (NEXT-2, reading R21)."""
        self.res = _c(res, np.uint32).reshape(-1, 4)
        self.L = self.res.shape[0]
        self.cap = int(cap)
        self.corners = np.zeros(self.L, np.uint64)
        self.tsize = np.zeros(self.L, np.uint64)
        self.hashed = np.zeros(self.L, np.int32)
        self.offset = np.zeros(self.L, np.uint64)
        tot = lib().fho_build_levels(_p(self.res, ctypes.c_uint32), self.L, self.cap,
                                     _p(self.corners, ctypes.c_uint64), _p(self.tsize, ctypes.c_uint64),
                                     _p(self.hashed, ctypes.c_int32), _p(self.offset, ctypes.c_uint64))
        if tot == 0:
            raise ValueError("build_levels: bad arguments")
        self.total = int(tot)
        if lin == 1:   # mode code 2 in the C oracle = brick order on bijective levels
            self.hashed[self.hashed == 0] = 2

    def param_count(self, F: int) -> int:
        return self.total * F

    def _common(self):
        return (_p(self.res, ctypes.c_uint32), _p(self.hashed, ctypes.c_int32),
                _p(self.tsize, ctypes.c_uint64), _p(self.offset, ctypes.c_uint64), self.L)

    def indices(self, coords: np.ndarray, want_w: bool = True) -> Tuple[np.ndarray, Optional[np.ndarray], int]:
        """Oracle-I: (idx [N][L][16] uint32, W [N][L][16] fp64, #clamped samples)."""
        c = _c(coords, np.float32).reshape(-1, 4)
        N = c.shape[0]
        idx = np.zeros((N, self.L, 16), np.uint32)
        W = np.zeros((N, self.L, 16), np.float64) if want_w else None
        nbad = lib().fho_encode_indices(*self._common(), _p(c, ctypes.c_float), N,
                                        _p(idx, ctypes.c_uint32),
                                        _p(W, ctypes.c_double) if want_w else None)
        return idx, W, int(nbad)

    def forward(self, coords: np.ndarray, table: np.ndarray, want_abs: bool = False):
        """Oracle-F: out [N][L*F] fp64 (and sum_c W_c|E_c| when want_abs)."""
        c = _c(coords, np.float32).reshape(-1, 4)
        t = _c(table, np.float64)
        F = t.shape[1]
        assert t.shape[0] == self.total
        N = c.shape[0]
        out = np.zeros((N, self.L * F), np.float64)
        ab = np.zeros_like(out) if want_abs else None
        lib().fho_encode_fwd(*self._common(), F, _p(c, ctypes.c_float), N, _p(t, ctypes.c_double),
                             _p(out, ctypes.c_double), _p(ab, ctypes.c_double) if want_abs else None)
        return (out, ab) if want_abs else out

    def backward(self, coords: np.ndarray, dout: np.ndarray, F: int, want_abs: bool = False):
        """Oracle-B: G [sum T][F] fp64 (and A = sum |W g| when want_abs)."""
        c = _c(coords, np.float32).reshape(-1, 4)
        g = _c(dout, np.float64)
        N = c.shape[0]
        assert g.shape == (N, self.L * F)
        G = np.zeros((self.total, F), np.float64)
        A = np.zeros_like(G) if want_abs else None
        lib().fho_encode_bwd(*self._common(), F, _p(c, ctypes.c_float), N, _p(g, ctypes.c_double),
                             _p(G, ctypes.c_double), _p(A, ctypes.c_double) if want_abs else None)
        return (G, A) if want_abs else G

    def level_stats(self, l: int, max_vertices: int = 1 << 26):
        """Oracle-S: (distinct buckets, collisions, utilisation)."""
        r = _c(self.res[l], np.uint32)
        d = np.zeros(1, np.uint64)
        col = np.zeros(1, np.uint64)
        rc = lib().fho_level_stats(_p(r, ctypes.c_uint32), int(self.hashed[l]), int(self.tsize[l]),
                                   max_vertices, _p(d, ctypes.c_uint64), _p(col, ctypes.c_uint64))
        if rc != 0:
            raise ValueError(f"level_stats rc={rc}")
        return int(d[0]), int(col[0]), float(d[0]) / float(self.tsize[l])


class MHELevels:
    """NEXT-3 oracle: the MHE baseline (one 3D hash encoder per key frame,
    fixed T per level; Fig. 4).  res: vertices per
    spatial axis per level."""

    def __init__(self, res: Sequence[int], n_frames: int, T: int):
        self.res = _c(res, np.uint32)
        self.L, self.n_frames, self.T = len(self.res), int(n_frames), int(T)
        self.total = self.L * self.n_frames * self.T

    def param_count(self, F: int) -> int:
        return self.total * F

    def _common(self):
        return (_p(self.res, ctypes.c_uint32), self.L, self.n_frames, self.T)

    def indices(self, coords, want_w=True):
        c = _c(coords, np.float32).reshape(-1, 4)
        N = c.shape[0]
        idx = np.zeros((N, self.L, 8), np.uint32)
        W = np.zeros((N, self.L, 8), np.float64) if want_w else None
        nb = lib().fho_mhe_indices(*self._common(), _p(c, ctypes.c_float), N, _p(idx, ctypes.c_uint32),
                                   _p(W, ctypes.c_double) if want_w else None)
        return idx, W, int(nb)

    def forward(self, coords, table, want_abs=False):
        c = _c(coords, np.float32).reshape(-1, 4)
        t = _c(table, np.float64)
        F = t.shape[1]
        assert t.shape[0] == self.total
        N = c.shape[0]
        out = np.zeros((N, self.L * F))
        ab = np.zeros_like(out) if want_abs else None
        lib().fho_mhe_fwd(*self._common(), F, _p(c, ctypes.c_float), N, _p(t, ctypes.c_double),
                          _p(out, ctypes.c_double), _p(ab, ctypes.c_double) if want_abs else None)
        return (out, ab) if want_abs else out

    def backward(self, coords, dout, F, want_abs=False):
        c = _c(coords, np.float32).reshape(-1, 4)
        g = _c(dout, np.float64)
        N = c.shape[0]
        G = np.zeros((self.total, F))
        A = np.zeros_like(G) if want_abs else None
        lib().fho_mhe_bwd(*self._common(), F, _p(c, ctypes.c_float), N, _p(g, ctypes.c_double),
                          _p(G, ctypes.c_double), _p(A, ctypes.c_double) if want_abs else None)
        return (G, A) if want_abs else G

    def level_stats(self, l: int, max_vertices: int = 1 << 27):
        d = np.zeros(1, np.uint64)
        col = np.zeros(1, np.uint64)
        rc = lib().fho_mhe_level_stats(int(self.res[l]), self.T, max_vertices, _p(d, ctypes.c_uint64),
                                       _p(col, ctypes.c_uint64))
        if rc != 0:
            raise ValueError(f"mhe level_stats rc={rc}")
        return int(d[0]), int(col[0]), float(d[0]) / float(self.T)


def fhash(res4: Sequence[int], x: int, y: int, z: int, t: int) -> int:
    """Eq. 9 for one corner; res4 = (Rx, Ry, Rz, Rt)."""
    r = _c(res4, np.uint32)
    return int(lib().fho_fhash(_p(r, ctypes.c_uint32), x, y, z, t))


def brick_index(res4: Sequence[int], x: int, y: int, z: int, t: int) -> int:
    """NEXT-2 brick (tiled Z-order) linearization of one vertex (R21)."""
    r = _c(res4, np.uint32)
    return int(lib().fho_brick_index(_p(r, ctypes.c_uint32), x, y, z, t))


def spatial_hash(X: int, Y: int, Z: int, T: int, tsize: int) -> int:
    return int(lib().fho_spatial_hash(X, Y, Z, T, tsize))
