"""Pins for the CPU oracle (oracle/) against what the paper and mathematics
fix -- NOT against itself.  CPU only (-m "not gpu").

Each test names the passage it pins.  A plausible mistake in the oracle
(dropped term, wrong sign/index, transposed operand, off-by-one cell) fails
at least one of: SPEC worked values, Table-3 parameter counts, brute-force
bijectivity, partition of unity, lattice exactness, multilinear
reproduction, finite differences, adjoint identity.
"""
import json
import os

import numpy as np
import pytest

import oracle
import workloads as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ------------------------------------------------------------ a1 fold schedule
@pytest.mark.parametrize("ex", gold("spec_examples.json")["configure_levels"])
def test_fold_schedule_spec_examples(ex):
    """S:282-284 worked examples of Eqs. 4-8."""
    lv = oracle.fold_schedule(ex["S"], ex["n"], ex["fold"])
    assert len(lv) == ex["Ls"]
    assert [r[0] for r in lv] == ex["x"]
    assert [r[1] for r in lv] == ex["y"]
    assert [r[2] for r in lv] == ex["z"]
    if "t" in ex:
        assert [r[3] for r in lv] == ex["t"]


@pytest.mark.parametrize("row", gold("paper_table3.json")["rows"])
def test_table3_parameter_counts(row):
    """Table tab:convergence_time_and_encoding_parameter:
    F-Hash parameter counts in mebi, printed to one decimal."""
    lv = oracle.fold_schedule(row["S"], row["n"], row["fold"])
    levels = oracle.Levels(lv, cap=0)
    mi = levels.param_count(row["F"]) / 2 ** 20
    assert abs(mi - row["printed_Mi"]) / row["printed_Mi"] < 1e-3, mi
    # R1: reading Res as the CELL count would give 27.75 / 121.41 Mi
    cells = sum((r[0] + 1) * (r[1] + 1) * (r[2] + 1) * (r[3] + 1) for r in lv) * row["F"] / 2 ** 20
    assert abs(cells - row["printed_Mi"]) / row["printed_Mi"] > 0.1


def test_fold_schedule_monotone_decay_random():
    """Res^l <= max(ceil(Res^{l-1}/f), 2); level 1 = native (Eq. 4);
    last level <= f on every axis (ceil(S/f^(L_s-1)) <= f since f^L_s >= S,
    Eq. 5) and axes that reached f earlier are padded with Tail = 2 (Eq. 8);
    L_s = max_a ceil(log_f S_a) (Eqs. 5-6)."""
    g = np.random.default_rng(1)
    for _ in range(200):
        S = [int(v) for v in g.integers(2, 300, size=3)]
        n = int(g.integers(2, 40))
        f = int(g.integers(2, 7))
        lv = oracle.fold_schedule(S, n, f)
        assert list(lv[0]) == S + [n]
        import math
        Ls = max(max(1, math.ceil(math.log(v) / math.log(f) - 1e-12)) for v in S + [n])
        assert len(lv) == Ls
        assert all(v <= f for v in lv[-1]) or Ls == 1
        for a in range(4):
            col = [r[a] for r in lv]
            first_le_f = next(i for i, v in enumerate(col) if v <= f)
            assert all(v == 2 for v in col[first_le_f + 1:])
        for a in range(4):
            for l in range(1, len(lv)):
                assert lv[l][a] <= max(-(-lv[l - 1][a] // f), 2)
                assert lv[l][a] >= 2


# ------------------------------------------------------------ a4 F-Hash, Eq. 9
@pytest.mark.parametrize("ex", gold("spec_examples.json")["fhash"])
def test_fhash_spec_examples(ex):
    t, x, y, z = ex["res_txyz"]
    ct, cx, cy, cz = ex["corner_txyz"]
    assert oracle.fhash((x, y, z, t), cx, cy, cz, ct) == ex["index"]


def test_fhash_permutation_2345():
    """a (2,3,4,5) grid enumerates to a permutation of 0..119."""
    ex = gold("spec_examples.json")["fhash_permutation"]
    r = ex["res"]
    got = sorted(oracle.fhash(r, x, y, z, t) for t in range(r[3]) for z in range(r[2])
                 for y in range(r[1]) for x in range(r[0]))
    assert got == list(range(ex["count"]))


@pytest.mark.parametrize("cfg", [W.CFG1])
def test_bijective_levels_full_utilisation(cfg):
    """P:174 'bijective MPHF without collision and bucket waste': brute force
    over every vertex of every cfg1 level (128+1536+6912+20480 entries)."""
    lv = oracle.Levels(cfg.levels, cfg.cap)
    assert list(lv.tsize) == [128, 1536, 6912, 20480]
    assert lv.param_count(cfg.F) == 58112
    for l in range(lv.L):
        d, col, util = lv.level_stats(l)
        assert col == 0 and util == 1.0 and d == int(lv.tsize[l])


def test_bijectivity_random_fold_schedules():
    """bijectivity on random (S, n, fold) draws, brute force."""
    g = np.random.default_rng(7)
    for _ in range(200):
        S = [int(v) for v in g.integers(2, 14, size=3)]
        lvs = oracle.fold_schedule(S, int(g.integers(2, 8)), int(g.integers(2, 5)))
        lv = oracle.Levels(lvs, 0)
        for l in range(lv.L):
            d, col, util = lv.level_stats(l)
            assert col == 0 and util == 1.0


def test_brick_linearization_bijective_and_local():
    """NEXT-2 (P:174 'Morton and Z-order ... with preserved locality'):
    the brick order is a bijection onto [0, C) on every cfg1 level and on
    ragged shapes (brute force), equals Eq. 9 when every axis fits one brick,
    and keeps the 16 corners of a cell closer than Eq. 9 does."""
    for r in [(4, 8, 12, 2), (8, 8, 8, 3), (12, 12, 12, 4), (16, 16, 16, 5), (5, 7, 9, 3), (2, 2, 2, 2),
              (13, 3, 6, 7), (17, 1 + 1, 11, 5)]:
        got = sorted(oracle.brick_index(r, x, y, z, t) for t in range(r[3]) for z in range(r[2])
                     for y in range(r[1]) for x in range(r[0]))
        assert got == list(range(r[0] * r[1] * r[2] * r[3])), r
        lv = oracle.Levels([r], lin=1)
        d, col, util = lv.level_stats(0)
        assert col == 0 and util == 1.0
    r = (2, 2, 2, 2)   # one brick: identical to Eq. 9
    for t in range(2):
        for z in range(2):
            for y in range(2):
                for x in range(2):
                    assert oracle.brick_index(r, x, y, z, t) == oracle.fhash(r, x, y, z, t)
    # the brick of a cell at even coordinates holds exactly its 16 corners, in
    # Morton (Z-order) bit order x, y, z, t of the lowest bit
    r = (6, 4, 4, 4)
    base = oracle.brick_index(r, 2, 2, 2, 2)
    assert [oracle.brick_index(r, 2 + (c & 1), 2 + (c >> 1 & 1), 2 + (c >> 2 & 1), 2 + (c >> 3 & 1)) - base
            for c in range(16)] == list(range(16))
    r = (64, 64, 64, 8)
    lines = []
    for lin in (0, 1):
        lv = oracle.Levels([r], lin=lin)
        idx, _, _ = lv.indices(W.draw_coords(W.rng(3), 2000), want_w=False)
        # distinct 128-byte lines (16 entries of 8 B) touched by a cell's 16 corners
        lines.append(np.mean([len(set((row // 16).tolist())) for row in idx[:, 0, :]]))
    assert lines[1] < 0.65 * lines[0], lines


def test_capped_levels_hash_stats():
    """R5 capped levels: T_l = cap, every bucket index < T_l, pigeonhole
    collisions and utilisation < 1 possible; the bijective levels
    of the same encoder stay collision-free."""
    lv = oracle.Levels(W.CFG1H.levels, W.CFG1H.cap)
    assert list(lv.hashed) == [0, 0, 1, 1]
    assert list(lv.tsize) == [128, 1536, 2048, 2048]
    assert lv.total == 5760
    for l in range(lv.L):
        d, col, util = lv.level_stats(l)
        if lv.hashed[l]:
            assert col == int(lv.corners[l]) - d > 0
            assert 0.5 < util <= 1.0
        else:
            assert col == 0 and util == 1.0


def test_hash_reduces_to_x_when_yzt_zero():
    """R5 with Y=Z=T=0 the XOR hash is X*1 mod T (prime 1 on x)."""
    for X in [0, 1, 5, 2047, 2048, 123456]:
        assert oracle.spatial_hash(X, 0, 0, 0, 2048) == X % 2048
    # uint32 wrap-around: Y*2654435761 mod 2^32
    assert oracle.spatial_hash(0, 3, 0, 0, 1 << 32) == (3 * 2654435761) % (1 << 32)


def test_hash_hand_computed_golden():
    """R5 against values worked out by hand (tests/golden/r5_hash.json, the
    arithmetic written beside each): every term non-zero, Z/T swapped (a
    swapped or mistyped z or t prime fails), each prime alone, and the
    uint32 wrap of X + (...)."""
    g = gold("r5_hash.json")
    for c in g["cases"]:
        assert oracle.spatial_hash(c["X"], c["Y"], c["Z"], c["T"], c["tsize"]) == c["bucket"], c["what"]


def test_hash_pipeline_golden():
    """Steps 1-3 end to end on a capped cfg1h level: cell location (R2),
    corner order (R3) and R5 plus the level offset, against the hand-worked
    indices in tests/golden/r5_hash.json."""
    p = gold("r5_hash.json")["pipeline"]
    lv = oracle.Levels([tuple(r) for r in p["levels"]], p["cap"])
    idx, _, bad = lv.indices(np.array([p["coord"]], np.float32), want_w=False)
    assert bad == 0
    for c in p["corners"]:
        assert int(idx[0, p["level"], c["c"]]) == c["index"], c


def test_hash_x_neighbours_adjacent():
    """R5 (x additive): the x-neighbour of a capped-level vertex is the next
    bucket (mod T_l) -- the property the pair layout relies on (DESIGN.md
    §8.1) -- while y, z, t neighbours scatter."""
    g = W.rng(5)
    T = 1 << 11
    for _ in range(200):
        X, Y, Z, Tt = (int(v) for v in g.integers(0, 5000, 4))
        h = oracle.spatial_hash(X, Y, Z, Tt, T)
        assert oracle.spatial_hash(X + 1, Y, Z, Tt, T) == (h + 1) % T
    far = sum(abs(oracle.spatial_hash(7, y + 1, 3, 2, T) - oracle.spatial_hash(7, y, 3, 2, T)) > 16 for y in range(100))
    assert far > 80


def test_cfg2_cfg4_table_sizes():
    """SURVEY.md Appendix A per-level tables (independently computed)."""
    lv2 = oracle.Levels(W.CFG2.levels, W.CFG2.cap)
    assert lv2.total == 6297307
    assert list(lv2.hashed) == [0] * 5 + [1] * 11
    assert int(lv2.corners[15]) == 8589934592
    lv4 = oracle.Levels(W.CFG4.levels, W.CFG4.cap)
    assert lv4.total == 39916734
    assert list(lv4.hashed) == [0] * 8 + [1] * 8


# ------------------------------------------------- a2/a3/a6 weights, forward
def test_time_bracket_spec_examples():
    """S:301-302 on the ABI domain [0,1] (R2: q -> (q+1)/2)."""
    for ex in gold("spec_examples.json")["time_bracket"]:
        lv = oracle.Levels([(2, 2, 2, ex["Rt"])])
        idx, Wt, _ = lv.indices(np.array([[0.3, 0.3, 0.3, ex["t01"]]], np.float32))
        w_next = Wt[0, 0, 8:].sum()          # corners with b_t = 1 (R3)
        assert w_next == pytest.approx(ex["w"], abs=1e-7)
        # i_t: the b_t = 0 corner with bx=by=bz=0 is Eq. 9 at t = i_t
        assert idx[0, 0, 0] == ex["i"] * 8


def test_centre_example_7_5():
    """Res=(2,2,2,2), F=1, E = own F-Hash index, query at centre -> 7.5.
    Also pins the corner order R3: with all R=2, idx_c == c."""
    lv = oracle.Levels([(2, 2, 2, 2)])
    table = np.arange(16, dtype=np.float64)[:, None]
    ctr = np.array([[0.5, 0.5, 0.5, 0.5]], np.float32)
    assert lv.forward(ctr, table)[0, 0] == 7.5
    idx, _, _ = lv.indices(ctr)
    assert list(idx[0, 0]) == list(range(16))


def test_partition_of_unity_and_weight_range():
    """sum_c W_c = 1, W_c in [0,1], for random points and levels."""
    case = W.encode_case(W.CFG1H, 2000, seed=3)
    lv = oracle.Levels(W.CFG1H.levels, W.CFG1H.cap)
    _, Wt, nbad = lv.indices(case.coords)
    assert nbad == 0
    assert np.all(Wt >= 0) and np.all(Wt <= 1)
    assert np.max(np.abs(Wt.sum(-1) - 1.0)) < 1e-14


def test_constant_table_constant_output():
    """constant table -> constant output, any point, any level."""
    lv = oracle.Levels(W.CFG1H.levels, W.CFG1H.cap)
    c = W.draw_coords(W.rng(5), 500)
    out = lv.forward(c, np.full((lv.total, 2), 0.37))
    assert np.max(np.abs(out - 0.37)) < 1e-15


def _vertex_coords(R, k):
    return np.float32(k / (R - 1))


def test_lattice_points_exact():
    """S:310 / S:344: at a lattice vertex the encode returns that vertex's
    embedding exactly (all weight on one corner).  R-1 powers of two so that
    k/(R-1) is exact in fp32."""
    res = [(5, 9, 3, 2), (9, 5, 17, 3), (17, 3, 5, 5)]
    lv = oracle.Levels(res)
    g = np.random.default_rng(11)
    table = g.uniform(-1, 1, size=(lv.total, 2))
    for l, r in enumerate(res):
        for _ in range(50):
            v = [int(g.integers(0, r[a])) for a in range(4)]
            p = np.array([[_vertex_coords(r[a], v[a]) for a in range(4)]], np.float32)
            out = lv.forward(p, table)
            e = table[int(lv.offset[l]) + oracle.fhash(r, *v)]
            assert np.array_equal(out[0, 2 * l:2 * l + 2], e)
            _, Wt, _ = lv.indices(p)
            assert sorted(Wt[0, l])[-1] == 1.0 and np.sum(Wt[0, l] != 0) == 1


def test_multilinear_reproduction():
    """Multilinear interpolation reproduces multilinear functions exactly:
    with E(v) = prod_a v_a/(R_a-1) (feature 0) and prod_a (1 - v_a/(R_a-1))
    (feature 1) on a bijective level, the encode equals p_x p_y p_z p_t and
    prod (1-p_a) up to the fp32 rounding of s = p (R-1) (R2)."""
    res = [(4, 7, 5, 3), (13, 6, 9, 4), (16, 16, 16, 5)]
    lv = oracle.Levels(res)
    table = np.zeros((lv.total, 2))
    for l, r in enumerate(res):
        for t in range(r[3]):
            for z in range(r[2]):
                for y in range(r[1]):
                    for x in range(r[0]):
                        u = [x / (r[0] - 1), y / (r[1] - 1), z / (r[2] - 1), t / (r[3] - 1)]
                        j = int(lv.offset[l]) + x + r[0] * (y + r[1] * (z + r[2] * t))
                        table[j, 0] = np.prod(u)
                        table[j, 1] = np.prod([1 - v for v in u])
    c = W.draw_coords(W.rng(2), 3000).astype(np.float64)
    out = lv.forward(c.astype(np.float32), table)
    for l in range(len(res)):
        exp0 = np.prod(c, axis=1)
        exp1 = np.prod(1 - c, axis=1)
        assert np.max(np.abs(out[:, 2 * l] - exp0)) < 1e-6
        assert np.max(np.abs(out[:, 2 * l + 1] - exp1)) < 1e-6


def test_continuity_across_faces():
    """approaching a shared cell face from both sides converges."""
    r = (9, 7, 6, 4)
    lv = oracle.Levels([r])
    table = np.random.default_rng(4).uniform(-1, 1, size=(lv.total, 2))
    base = np.array([0.31, 0.47, 0.73, 0.61], np.float32)
    for a in range(4):
        k = 3 if r[a] > 4 else 1
        for eps in [1e-6, 1e-7]:
            lo = base.copy()
            hi = base.copy()
            lo[a] = np.float32(k / (r[a] - 1) - eps)
            hi[a] = np.float32(k / (r[a] - 1) + eps)
            o = lv.forward(np.stack([lo, hi]), table)
            assert np.max(np.abs(o[0] - o[1])) < 50 * eps


def test_out_of_domain_clamped_and_counted():
    """R2: coordinates outside [0,1] (or NaN) are clamped and counted."""
    lv = oracle.Levels(W.CFG1.levels)
    bad = W.bad_coords()
    _, _, nbad = lv.indices(bad)
    assert nbad == len(bad)
    clamped = np.nan_to_num(np.clip(bad, 0, 1), nan=0.0, posinf=1.0)
    table = np.random.default_rng(0).uniform(-1, 1, size=(lv.total, 2))
    assert np.array_equal(lv.forward(bad, table), lv.forward(clamped, table))


# ------------------------------------------------------------- a10 backward
def test_backward_adjoint_identity():
    """<g, F(E)> = <F^T(g), E> for random E and g (fp64)."""
    case = W.encode_case(W.CFG1H, 1500, seed=9)
    lv = oracle.Levels(W.CFG1H.levels, W.CFG1H.cap)
    E = np.random.default_rng(1).standard_normal((lv.total, 2))
    out = lv.forward(case.coords, E)
    G = lv.backward(case.coords, case.dout, 2)
    lhs = float(np.sum(case.dout.astype(np.float64) * out))
    rhs = float(np.sum(G * E))
    assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(lhs))


def test_backward_finite_differences():
    """S:320 / S:347: central finite differences of L(E) = <g, F(E)> in fp64
    match the analytic gradient within 1e-5 relative."""
    case = W.encode_case(W.CFG1H, 64, seed=12)
    lv = oracle.Levels(W.CFG1H.levels, W.CFG1H.cap)
    E = np.random.default_rng(3).standard_normal((lv.total, 2))
    g = case.dout.astype(np.float64)
    G = lv.backward(case.coords, g, 2)
    touched = np.argwhere(G != 0)
    pick = touched[np.random.default_rng(5).choice(len(touched), 60, replace=False)]
    h = 1e-3
    for j, f in pick:
        Ep = E.copy(); Ep[j, f] += h
        Em = E.copy(); Em[j, f] -= h
        fd = (np.sum(g * lv.forward(case.coords, Ep)) - np.sum(g * lv.forward(case.coords, Em))) / (2 * h)
        assert abs(fd - G[j, f]) <= 1e-5 * max(1e-3, abs(G[j, f]))


def test_backward_lattice_point_single_entry_and_zero_upstream():
    """zero upstream -> zero grads; a lattice point puts the whole
    gradient on one entry per level."""
    r = (5, 9, 3, 2)
    lv = oracle.Levels([r])
    p = np.array([[0.25, 0.5, 1.0, 0.0]], np.float32)
    G = lv.backward(p, np.array([[1.5, -2.0]]), 2)
    nz = np.argwhere(G != 0)
    assert len(nz) == 2 and nz[0, 0] == nz[1, 0]
    assert nz[0, 0] == oracle.fhash(r, 1, 4, 2, 0)
    assert G[nz[0, 0], 0] == 1.5 and G[nz[0, 0], 1] == -2.0
    assert not np.any(lv.backward(p, np.zeros((1, 2)), 2))
