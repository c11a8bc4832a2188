"""Seeded synthetic workloads shared by the tests, `bench.py` and `smoke()`.

This module holds ONLY inputs: level-resolution lists, caps, batch sizes and
seeded random arrays.  It contains none of the method's arithmetic (no cell
location, no F-Hash, no interpolation), so the CPU oracle (`oracle/`) and the
CUDA path (`paper_2507_03836_b200/`) can both be fed from it without sharing
any computation.  Neither of those two packages imports this module; the
callers pass the arrays in.

Recipes follow SURVEY.md §8(d) (BASELINE.json `configs`):
  * one numpy PCG64(seed) generator per case, draw order = tables, then
    coordinates, then upstream gradients;
  * coordinates `rng.random((N, 4), dtype=float32)` (always < 1, never
    rounded up to 1.0), layout [N][4] = (x, y, z, t) in the ABI domain [0,1];
  * tables U(-1e-4, 1e-4) (paper P:233 "uniform initialization", range from
    BASELINE.json cfg1 / SPEC S:398), packed level-major [sum_l T_l][F];
  * upstream gradients N(0, 1) float32, [N][L*F].
The paper's datasets (Combustion, Argon Bubble, Supernova; PAPER.md
Table `tab:datasets`) are not available; these synthetic inputs
stand in for them (DESIGN.md §"Inputs").
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Sequence, Tuple

import numpy as np

Res = Tuple[int, int, int, int]  # vertices per axis (x, y, z, t)


def geometric(lo: float, hi: float, L: int) -> List[int]:
    """R_l = floor(lo * (hi/lo)^(l/(L-1)) + 0.5) in fp64 (SURVEY.md §8(d)
    "Resolution rule for geometric lists"; round, not floor)."""
    if L == 1:
        return [int(lo)]
    return [int(math.floor(lo * (hi / lo) ** (l / (L - 1)) + 0.5)) for l in range(L)]


@dataclasses.dataclass(frozen=True)
class EncoderConfig:
    name: str
    levels: Tuple[Res, ...]     # coarse -> fine, the order handed to build_levels
    F: int
    cap: int                    # 0 = uncapped (pure MPHF); else power of two
    table_dtype: str            # "f32" | "f16"

    @property
    def L(self) -> int:
        return len(self.levels)


def cfg1_levels() -> Tuple[Res, ...]:
    # BASELINE.json configs[0]: spatial 4,8,12,16; temporal 2,3,4,5.
    return tuple((s, s, s, t) for s, t in zip((4, 8, 12, 16), (2, 3, 4, 5)))


def cfg2_levels() -> Tuple[Res, ...]:
    # BASELINE.json configs[1]: spatial geometric 16..512 (growth 2^(1/3)),
    # temporal 2..64, L = 16.
    rs = geometric(16, 512, 16)
    rt = geometric(2, 64, 16)
    return tuple((s, s, s, t) for s, t in zip(rs, rt))


def cfg4_levels() -> Tuple[Res, ...]:
    # per-axis geometric from (16,16,16,2) to the
    # native (640,256,256,100), L = 16 (paper's per-axis independence).
    rx = geometric(16, 640, 16)
    ry = geometric(16, 256, 16)
    rt = geometric(2, 100, 16)
    return tuple((x, y, y, t) for x, y, t in zip(rx, ry, rt))


CFG1 = EncoderConfig("cfg1", cfg1_levels(), F=2, cap=0, table_dtype="f32")
CFG1H = EncoderConfig("cfg1h", cfg1_levels(), F=2, cap=1 << 11, table_dtype="f32")
CFG2 = EncoderConfig("cfg2", cfg2_levels(), F=2, cap=1 << 19, table_dtype="f32")
CFG3 = EncoderConfig("cfg3", cfg2_levels(), F=2, cap=1 << 19, table_dtype="f16")
CFG4 = EncoderConfig("cfg4", cfg4_levels(), F=4, cap=1 << 22, table_dtype="f16")

N_CFG1 = 4096
N_CFG2 = 1 << 20
N_CFG3 = 1 << 18
N_CFG4 = 1 << 22


def table_sizes(levels: Sequence[Res], cap: int) -> List[int]:
    """Bucket count per level as the harness needs it to size buffers:
    the corner count, or the cap when the corner count exceeds it.  (This is
    buffer sizing, not index arithmetic; the library and the oracle each
    compute their own and the tests compare them.)"""
    out = []
    for r in levels:
        c = r[0] * r[1] * r[2] * r[3]
        out.append(cap if (cap and c > cap) else c)
    return out


def rng(seed: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def draw_table(g: np.random.Generator, n_entries: int, F: int, dtype: str = "f32") -> np.ndarray:
    t = g.uniform(-1e-4, 1e-4, size=(n_entries, F)).astype(np.float32)
    if dtype == "f16":
        t = t.astype(np.float16)
    return t


def draw_coords(g: np.random.Generator, N: int) -> np.ndarray:
    return g.random((N, 4), dtype=np.float32)


def draw_grads(g: np.random.Generator, N: int, width: int) -> np.ndarray:
    return g.standard_normal((N, width), dtype=np.float32)


@dataclasses.dataclass
class EncodeCase:
    cfg: EncoderConfig
    table: np.ndarray      # [sum T][F] float32 or float16
    coords: np.ndarray     # [N][4] float32
    dout: np.ndarray       # [N][L*F] float32


def encode_case(cfg: EncoderConfig, N: int, seed: int = 0,
                coords: Optional[np.ndarray] = None) -> EncodeCase:
    g = rng(seed)
    n_entries = sum(table_sizes(cfg.levels, cfg.cap))
    table = draw_table(g, n_entries, cfg.F, cfg.table_dtype)
    c = draw_coords(g, N) if coords is None else coords
    dout = draw_grads(g, N, cfg.L * cfg.F)
    return EncodeCase(cfg, table, c, dout)


def edge_coords() -> np.ndarray:
    """Hand-picked coordinates on the domain edges and on lattice vertices
    (values exactly 0, 1, 0.5, and tiny/near-one floats).  Used for the edge
    cases of the parity tests."""
    vals = np.array([0.0, 1.0, 0.5, 0.25, 1e-7, np.nextafter(np.float32(1), np.float32(0)),
                     1.0 / 3.0, 2.0 / 3.0], dtype=np.float32)
    pts = []
    for a in vals:
        for b in vals[:4]:
            pts.append((a, b, vals[(len(pts) * 3) % len(vals)], b))
    return np.array(pts, dtype=np.float32)


def bad_coords() -> np.ndarray:
    """Out-of-domain and NaN coordinates (clamped, flagged as FH_E_DOMAIN)."""
    return np.array([[-0.5, 0.5, 0.5, 0.5], [0.5, 1.5, 0.5, 0.5],
                     [np.nan, 0.5, 0.5, 0.5], [0.5, 0.5, 0.5, np.inf]], dtype=np.float32)


# ---------------------------------------------------------------- train step
@dataclasses.dataclass(frozen=True)
class MLPConfig:
    widths: Tuple[int, ...]   # e.g. (32, 64, 64, 1): input, hidden..., output


MLP3 = MLPConfig((32, 64, 64, 1))   # BASELINE.json configs[2]
MLP4 = MLPConfig((64, 64, 64, 1))   # BASELINE.json configs[3]


def draw_mlp(g: np.random.Generator, m: MLPConfig) -> List[Tuple[np.ndarray, np.ndarray]]:
    """nn.Linear default init U(+-1/sqrt(fan_in)) for weights and biases
    (SURVEY.md §8(c) D14).  Weight layout [out][in] row-major."""
    layers = []
    for fi, fo in zip(m.widths[:-1], m.widths[1:]):
        b = 1.0 / math.sqrt(fi)
        W = g.uniform(-b, b, size=(fo, fi)).astype(np.float32)
        bias = g.uniform(-b, b, size=(fo,)).astype(np.float32)
        layers.append((W, bias))
    return layers


def gaussian_blob_params(g: np.random.Generator, blobs: int = 8) -> np.ndarray:
    """[blobs][7] = (sigma, c0x, c0y, c0z, vx, vy, vz): sigma ~ U(0.05, 0.15),
    c0 ~ U(0.2, 0.8)^3, v ~ U(-0.3, 0.3)^3."""
    sig = g.uniform(0.05, 0.15, size=blobs)
    c0 = g.uniform(0.2, 0.8, size=(blobs, 3))
    v = g.uniform(-0.3, 0.3, size=(blobs, 3))
    return np.concatenate([sig[:, None], c0, v], axis=1).astype(np.float32)


def gaussian_blobs_field(g: np.random.Generator, S: int = 256, T: int = 32, blobs: int = 8,
                         dtype=np.float32) -> np.ndarray:
    """BASELINE.json configs[2] field: sum of 8 Gaussian blobs moving
    linearly in time + 0.1 sin(8 pi x) sin(8 pi y), min-max normalised to
    [0,1] (paper P:372 normalises values to [0,1]).  Layout [t][z][y][x].
    Generated in chunks of time steps on the host (float32)."""
    sig = g.uniform(0.05, 0.15, size=blobs)
    c0 = g.uniform(0.2, 0.8, size=(blobs, 3))
    v = g.uniform(-0.3, 0.3, size=(blobs, 3))
    ax = np.arange(S, dtype=np.float64) / (S - 1)
    out = np.empty((T, S, S, S), dtype=dtype)
    sx = np.sin(8 * np.pi * ax)
    noise = 0.1 * (sx[None, :] * sx[:, None])  # [y][x]
    for ti in range(T):
        tau = ti / (T - 1) if T > 1 else 0.0
        f = np.broadcast_to(noise[None], (S, S, S)).astype(np.float64).copy()
        for i in range(blobs):
            c = c0[i] + v[i] * tau
            gx = np.exp(-((ax - c[0]) ** 2) / (2 * sig[i] ** 2))
            gy = np.exp(-((ax - c[1]) ** 2) / (2 * sig[i] ** 2))
            gz = np.exp(-((ax - c[2]) ** 2) / (2 * sig[i] ** 2))
            f += gz[:, None, None] * gy[None, :, None] * gx[None, None, :]
        out[ti] = f
    lo, hi = float(out.min()), float(out.max())
    out -= lo
    out /= (hi - lo)
    return out
