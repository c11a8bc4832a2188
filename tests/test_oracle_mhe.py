"""Pins for the NEXT-3 MHE baseline oracle (oracle.MHELevels).  CPU only.

The paper's MHE parameter counts (Table tab:convergence_time_and_encoding_
parameter, MHE column: 120.0 M at P:619, 252.0 M at P:645, 1120.0 M at
P:671) fix the table layout T x L x F x key frames; Fig. 4 and
S:327/S:337 fix the collision / bucket-waste behaviour; trilinear
interpolation fixes the rest (vertex exactness, multilinear reproduction,
partition of unity, adjoint, finite differences)."""
import numpy as np
import pytest

import oracle
import workloads as W


@pytest.mark.parametrize("T_log,L,n,printed,cite", [(20, 6, 10, 120.0, "P:619"), (21, 7, 9, 252.0, "P:645"),
                                                   (23, 7, 10, 1120.0, "P:671")])
def test_mhe_parameter_counts_table3(T_log, L, n, printed, cite):
    m = oracle.MHELevels([16] * L, n, 1 << T_log)
    assert m.param_count(2) / 2 ** 20 == pytest.approx(printed, abs=0.05), cite


def test_mhe_collisions_and_bucket_waste():
    """S:327 pigeonhole: R^3 > T -> collisions; R^3 < T -> utilisation
    < 1 (bucket waste, Fig. 4); direct levels are collision-free."""
    m = oracle.MHELevels([8, 16, 40], 2, 4096)
    d, col, util = m.level_stats(0)     # 512 vertices in 4096 buckets
    assert col == 0 and util == 512 / 4096
    d, col, util = m.level_stats(1)     # 4096 vertices == T: direct, full
    assert col == 0 and util == 1.0
    d, col, util = m.level_stats(2)     # 64000 vertices > T: hashed
    assert col == 64000 - d > 0 and util <= 1.0


def test_mhe_partition_of_unity_frames_and_constant():
    m = oracle.MHELevels([5, 9, 40], 4, 1 << 10)
    c = W.draw_coords(W.rng(1), 500)
    idx, Wt, nb = m.indices(c)
    assert nb == 0 and np.all(Wt >= 0) and np.max(np.abs(Wt.sum(-1) - 1)) < 1e-14
    # frame = nearest key frame of t (R20): entries of level l live in [l*n*T + k*T, +T)
    k = np.clip(np.floor(c[:, 3] * np.float32(3) + np.float32(0.5)), 0, 3).astype(np.int64)
    for l in range(3):
        lo = l * 4 * 1024 + k * 1024
        assert np.all((idx[:, l, :] >= lo[:, None]) & (idx[:, l, :] < lo[:, None] + 1024))
    out = m.forward(c, np.full((m.total, 2), -0.3))
    assert np.max(np.abs(out + 0.3)) < 1e-15


def test_mhe_vertex_exact_and_trilinear_reproduction():
    R = 9   # direct level (729 <= T)
    m = oracle.MHELevels([R], 3, 1024)
    tab = np.zeros((m.total, 1))
    for k in range(3):
        for z in range(R):
            for y in range(R):
                for x in range(R):
                    tab[k * 1024 + x + R * (y + R * z), 0] = (x / 8) * (y / 8) * (z / 8) + k
    g = np.random.default_rng(2)
    c = np.concatenate([g.random((400, 3)), np.repeat([[0.0], [0.5], [1.0]], [150, 150, 100], axis=0)], 1)
    c = c.astype(np.float32)
    out = m.forward(c, tab)[:, 0]
    kk = np.array([0] * 150 + [1] * 150 + [2] * 100)
    assert np.max(np.abs(out - (np.prod(c[:, :3].astype(np.float64), 1) + kk))) < 1e-6
    v = np.array([[0.25, 0.5, 0.875, 0.5]], np.float32)   # vertex (2, 4, 7), frame 1
    assert m.forward(v, tab)[0, 0] == tab[1024 + 2 + 9 * (4 + 9 * 7), 0]


def test_mhe_backward_adjoint_and_finite_differences():
    m = oracle.MHELevels([4, 7, 30], 2, 256)
    g = np.random.default_rng(3)
    c = W.draw_coords(W.rng(4), 200)
    E = g.standard_normal((m.total, 2))
    up = g.standard_normal((200, 6))
    G = m.backward(c, up, 2)
    assert abs(np.sum(up * m.forward(c, E)) - np.sum(G * E)) < 1e-10
    nz = np.argwhere(G != 0)[:20]
    for j, f in nz:
        Ep, Em = E.copy(), E.copy()
        Ep[j, f] += 1e-3
        Em[j, f] -= 1e-3
        fd = (np.sum(up * m.forward(c, Ep)) - np.sum(up * m.forward(c, Em))) / 2e-3
        assert abs(fd - G[j, f]) <= 1e-5 * max(1e-3, abs(G[j, f]))
