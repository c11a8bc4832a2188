"""C-ABI library: loads, exports every symbol include/fhash.h declares, and
its host-only logic (a1 level builder, validation) matches the pins.
CPU only -- no compute call needs a GPU here."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import workloads as W
from paper_2507_03836_b200 import fhash as fh

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    import glob
    src = "".join(open(f).read() for f in sorted(glob.glob(os.path.join(ROOT, "include", "*.h"))))
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fh_[a-z_0-9]+)\s*\(", src)))


def test_library_loads_and_exports_header_symbols():
    L = fh.lib()
    syms = header_symbols()
    assert len(syms) >= 15
    assert sorted(fh.EXPORTS) == syms
    for s in syms:
        assert hasattr(L, s), s
    assert b"sm_100a" in L.fh_version()


def test_library_is_sm100a_cubin():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump -lelf {fh.LIB_PATH}").read()
    assert "sm_100a" in out


def test_fold_schedule_spec_examples_through_abi():
    """S:282-284 through the C ABI (host code)."""
    assert fh.fold_schedule((4, 8, 2), 2, 2) == [(4, 8, 2, 2), (2, 4, 2, 2), (2, 2, 2, 2)]
    assert fh.fold_schedule((2, 2, 2), 2, 2) == [(2, 2, 2, 2)]
    lv = fh.fold_schedule((80, 83, 204), 9, 2)
    assert [r[2] for r in lv] == [204, 102, 51, 26, 13, 7, 4, 2]
    assert [r[3] for r in lv] == [9, 5, 3, 2, 2, 2, 2, 2]


def test_fold_schedule_matches_oracle_random():
    import numpy as np
    g = np.random.default_rng(3)
    for _ in range(300):
        S = [int(v) for v in g.integers(2, 1000, size=3)]
        n, f = int(g.integers(2, 200)), int(g.integers(2, 9))
        assert fh.fold_schedule(S, n, f) == oracle.fold_schedule(S, n, f)


@pytest.mark.parametrize("cfg", [W.CFG1, W.CFG1H, W.CFG2, W.CFG3, W.CFG4], ids=lambda c: c.name)
def test_build_levels_matches_oracle(cfg):
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    ref = oracle.Levels(cfg.levels, cfg.cap)
    assert enc.entries == ref.total
    assert enc.param_count == ref.total * cfg.F
    for l in range(cfg.L):
        I = enc.level_info(l)
        assert I["res"] == tuple(int(v) for v in ref.res[l])
        assert I["corners"] == int(ref.corners[l])
        assert I["table_size"] == int(ref.tsize[l])
        assert I["hashed"] == bool(ref.hashed[l])
        assert I["offset"] == int(ref.offset[l])


def test_table3_param_count_through_abi():
    """P:619 Combustion-Seg 24.2 Mi; P:671 Supernova-Seg 107.7 Mi (fold 2, F 2)."""
    for S, printed in (((200, 110, 54), 24.2), ((156, 183, 185), 107.7)):
        enc = fh.Encoder(fh.fold_schedule(S, 10, 2), 2)
        assert abs(enc.param_count / 2 ** 20 - printed) / printed < 1e-3


@pytest.mark.parametrize("kw,status", [
    (dict(levels=[], F=2), fh.FH_E_ARG),
    (dict(levels=[(4, 4, 4, 2)], F=3), fh.FH_E_ARG),
    (dict(levels=[(4, 1, 4, 2)], F=2), fh.FH_E_ARG),
    (dict(levels=[(4, 4, 4, 2)], F=2, cap=1000), fh.FH_E_ARG),
    (dict(levels=[(4, 4, 4, 2)] * 33, F=2), fh.FH_E_ARG),
    (dict(levels=[(4096, 4096, 4096, 16)], F=2), fh.FH_E_RANGE),
    (dict(levels=[(1024, 1024, 1024, 2)], F=2), fh.FH_E_RANGE),             # sum T F = 2^32 exactly
    (dict(levels=[(1024, 1024, 1023, 2), (128, 128, 128, 2)], F=2), fh.FH_E_RANGE),   # crosses 2^32 at level 1
    (dict(levels=[(4, 4, 4, 2)], F=2, cap=1 << 32), fh.FH_E_RANGE),           # cap above 2^31
    (dict(levels=[(1 << 25, 2, 2, 2)], F=1), fh.FH_E_ARG),
])
def test_build_levels_errors(kw, status):
    with pytest.raises(fh.FHashError) as ei:
        fh.Encoder(**kw)
    assert ei.value.status == status


def test_fold_schedule_errors():
    with pytest.raises(fh.FHashError) as ei:
        fh.fold_schedule((1, 4, 4), 2, 2)
    assert ei.value.status == fh.FH_E_ARG
    with pytest.raises(fh.FHashError):
        fh.fold_schedule((4, 4, 4), 2, 1)


def test_arm_pace_alg1():
    """Alg. 1: N_s = max(min(N_r / N_a, 64), 1); 0 when no ray alive."""
    assert fh.arm_pace(1000, 1000) == 1
    assert fh.arm_pace(1000, 1) == 64
    assert fh.arm_pace(100, 3) == 33
    assert fh.arm_pace(100, 200) == 1
    assert fh.arm_pace(100, 0) == 0


def test_encode_argument_errors_are_host_side():
    """Argument validation happens before any device work: NULL/misaligned
    pointers and bad dtypes are rejected synchronously (no GPU needed)."""
    enc = fh.Encoder(W.CFG1.levels, 2)
    L = fh.lib()
    assert L.fh_encode_fwd(enc.handle, None, 10, None, None, 0, None) == fh.FH_E_ARG
    assert L.fh_encode_fwd(enc.handle, 16, 10, 16, 16, 7, None) == fh.FH_E_ARG   # dtype
    assert L.fh_encode_fwd(enc.handle, 8, 10, 16, 16, 0, None) == fh.FH_E_ARG    # misaligned coords
    assert L.fh_encode_bwd(enc.handle, 16, -1, 16, 16, None) == fh.FH_E_ARG
    assert L.fh_encode_fwd(None, 16, 10, 16, 16, 0, None) == fh.FH_E_ARG
    assert b"NULL" in L.fh_last_error()
    # N = 0 is a no-op
    assert L.fh_encode_fwd(enc.handle, 16, 0, 16, 16, 0, None) == fh.FH_OK
    # fh_encode_bwd_ex: unknown flags, misaligned dout
    assert L.fh_encode_bwd_ex(enc.handle, 16, 10, 16, 16, 0x80, None) == fh.FH_E_ARG
    assert L.fh_encode_bwd_ex(enc.handle, 16, 10, 4, 16, 1, None) == fh.FH_E_ARG
    # FH_BWD_DOUT_LEVEL_MAJOR: accepted by F-Hash encoders (the call then fails
    # only on the missing device here), rejected host-side by the MHE baseline
    lm = 2
    assert L.fh_encode_bwd_ex(enc.handle, 16, 10, 16, 16, lm | 1, None) != fh.FH_E_ARG
    mhe = fh.MHEEncoder([4, 8, 12, 16], 2, 1 << 10, 5)
    assert L.fh_encode_bwd_ex(mhe.handle, 16, 10, 16, 16, lm, None) == fh.FH_E_ARG
    assert b"MHE" in L.fh_last_error()
    # the trainer's dL/d(enc) layout query: NULL trainer -> -1
    assert fh._train_lib().fh_train_dx_layout(None) == -1
    # fh_level_stats: NULL pointers, level out of range, workspace query
    assert L.fh_level_stats(enc.handle, 0, None, 0, None, None) == fh.FH_E_ARG
    assert L.fh_level_stats(enc.handle, 99, 256, 1 << 20, 256, None) == fh.FH_E_ARG
    assert L.fh_level_stats_workspace_size(enc.handle, 0) >= (128 + 31) // 32 * 4
    assert L.fh_level_stats_workspace_size(enc.handle, 99) == 0
    assert L.fh_level_stats(enc.handle, 0, 256, 4, 256, None) == fh.FH_E_ARG   # workspace too small


def test_host_only_encoder_reports_state_error():
    """Without a CUDA device (this CPU container) fh_build_levels still
    builds the host plan (level queries, scratch sizing) but makes no device
    state, and a valid encode call returns FH_E_STATE rather than faulting."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("host-only behaviour")
    enc = fh.Encoder(W.CFG2.levels, 2, cap=W.CFG2.cap)
    assert enc.scratch_size() > 0
    L = fh.lib()
    assert L.fh_encode_fwd(enc.handle, 16, 10, 256, 256, 0, None) == fh.FH_E_STATE
    assert b"without a CUDA device" in L.fh_last_error()
    assert L.fh_encode_bwd(enc.handle, 16, 10, 256, 256, None) == fh.FH_E_STATE


def test_build_levels_lin_brick_info_and_errors():
    """NEXT-2 through the ABI: the brick linearization keeps the table sizes
    and packing of Eq. 9 (a bijection onto [0, C_l)), is reported per level,
    leaves hashed levels alone, and rejects unknown values."""
    cfg = W.CFG1H
    a = fh.Encoder(cfg.levels, 2, cap=cfg.cap)
    b = fh.Encoder(cfg.levels, 2, cap=cfg.cap, lin=fh.FH_LIN_BRICK)
    assert a.entries == b.entries
    for l in range(cfg.L):
        ia, ib = a.level_info(l), b.level_info(l)
        assert ia["table_size"] == ib["table_size"] and ia["offset"] == ib["offset"]
        assert ia["lin"] == 0
        assert ib["lin"] == (0 if ib["hashed"] else fh.FH_LIN_BRICK)
    with pytest.raises(fh.FHashError) as e:
        fh.Encoder(cfg.levels, 2, lin=7)
    assert e.value.status == fh.FH_E_ARG


def test_coreset_host_helpers_match_oracle():
    """NEXT-4 host helpers: fh_morton_cell equals the oracle's R24 interleave
    on cubic and rectangular grids; fh_occupancy_words = 2^(sum b_a) bits in
    words; workspace sizing rejects degenerate / oversized volumes."""
    from oracle import coreset as C
    for dims in [(33, 33, 33), (6, 4, 3), (641, 257, 257), (2, 2, 2), (9, 130, 5)]:
        cells = [d - 1 for d in dims]
        bits = C.morton_bits(cells)
        g = np.random.default_rng(sum(dims))
        for _ in range(200):
            x, y, z = (int(g.integers(0, c)) for c in cells)
            assert fh.morton_cell(dims, x, y, z) == C.morton_encode(x, y, z, bits)
        assert fh.occupancy_words(dims) == ((1 << sum(bits)) + 31) // 32
        assert fh.morton_cell(dims, cells[0], 0, 0) == 2 ** 64 - 1
    L = fh._coreset_lib()
    dims = (ctypes.c_uint32 * 3)(1, 4, 4)
    assert L.fh_coreset_workspace_size(dims, 2) == 0
    dims = (ctypes.c_uint32 * 3)(2048, 2048, 1024)
    assert L.fh_coreset_workspace_size(dims, 1) == 0
