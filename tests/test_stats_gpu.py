"""encoding_stats on the GPU (fh_level_stats, the collision
/ bucket-waste contrast of Fig. 4) against the oracle's
exhaustive Oracle-S (oracle.Levels.level_stats, MHELevels.level_stats):
distinct buckets, collisions and utilisation must agree EXACTLY (integer
work).  -m gpu."""
import pytest
import torch

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2507_03836_b200 import fhash as fh

ORACLE_MAX = 1 << 24   # levels the oracle brute-forces in well under a second


def _fhash_levels(levels, cap, lin):
    enc = fh.Encoder(levels, 2, "f32", cap, lin=lin)
    ref = oracle.Levels(levels, cap, lin=1 if lin == fh.FH_LIN_BRICK else 0)
    return enc, ref


@pytest.mark.parametrize("cfg", [W.CFG1, W.CFG1H, W.CFG2], ids=lambda c: c.name)
@pytest.mark.parametrize("lin", ["eq9", "brick"])
def test_fhash_level_stats_match_oracle(cfg, lin):
    enc, ref = _fhash_levels(cfg.levels, cfg.cap, fh.FH_LIN_BRICK if lin == "brick" else fh.FH_LIN_EQ9)
    checked = 0
    for l in range(enc.L):
        info = enc.level_info(l)
        if info["corners"] > ORACLE_MAX:
            continue
        got = enc.level_stats(l)
        exp = ref.level_stats(l, max_vertices=ORACLE_MAX)
        assert got[0] == exp[0] and got[1] == exp[1], (l, got, exp)
        assert got[2] == pytest.approx(exp[2], rel=0, abs=1e-15)
        if not info["hashed"]:   # Eq. 9 / brick are bijections: no collision, no waste
            assert got == (info["corners"], 0, 1.0)
        checked += 1
    assert checked >= 3


def test_fhash_capped_levels_large():
    """cfg2's capped levels (up to ~8.6e9 vertices into T = 2^19): exact
    agreement with the oracle's brute force up to 2^29 vertices per level
    (a few seconds of CPU); beyond, distinct + collisions = C, distinct <= T."""
    enc = fh.Encoder(W.CFG2.levels, 2, "f32", W.CFG2.cap)
    ref = oracle.Levels(W.CFG2.levels, W.CFG2.cap)
    hashed = [l for l in range(enc.L) if enc.level_info(l)["hashed"]]
    assert hashed
    for l in hashed:
        info = enc.level_info(l)
        d, c, u = enc.level_stats(l)
        assert d + c == info["corners"] and d <= info["table_size"]
        if info["corners"] <= (1 << 29):
            exp = ref.level_stats(l, max_vertices=1 << 29)
            assert (d, c) == exp[:2], (l, (d, c), exp)


def test_paper_shape_fold2_is_collision_free():
    """The paper's central claim (Eq. 9): the fold-2 Combustion
    schedule (8 levels, no cap) is collision-free with zero bucket waste on
    every level, the largest level included (far beyond the oracle's
    brute-force size)."""
    levels = oracle.fold_schedule((200, 110, 54), 10, 2)
    enc = fh.Encoder(levels, 2, "f32", 0)
    for l in range(enc.L):
        info = enc.level_info(l)
        assert enc.level_stats(l) == (info["corners"], 0, 1.0)


@pytest.mark.parametrize("res,T", [([4, 9, 17, 33, 65], 1 << 12), ([16, 30, 60, 120], 1 << 14),
                                   ([5, 50, 200], 1 << 20)])
def test_mhe_level_stats_match_oracle(res, T):
    enc = fh.MHEEncoder(res, 2, T, 3, "f32")
    ref = oracle.MHELevels(res, 3, T)
    for l in range(len(res)):
        got = enc.level_stats(l)
        exp = ref.level_stats(l)
        assert got[0] == exp[0] and got[1] == exp[1], (l, got, exp)
        R = res[l]
        if R ** 3 <= T:   # direct-indexed: no collisions, waste = T - R^3 (Fig. 4)
            assert got[:2] == (R ** 3, 0)


def test_mhe_paper_shape_waste_and_collisions():
    """Paper-scale MHE (T = 2^20, 6 geometric levels 16..512): the
    coarse levels waste buckets (R^3 < T), the fine ones collide."""
    res = W.geometric(16, 512, 6)
    enc = fh.MHEEncoder(res, 2, 1 << 20, 10, "f32")
    st = [enc.level_stats(l) for l in range(len(res))]
    assert st[0][2] < 0.01 and st[0][1] == 0
    assert st[-1][1] > 0 and st[-1][0] <= (1 << 20)
