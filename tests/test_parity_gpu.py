"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on
the same seeded inputs, element by element.  -m gpu.

Bars (from BASELINE.json north_star and SURVEY.md §8(c)):
  indices     bit-exact (uint32), all N*L*16
  weights     |w_gpu - W| <= 1e-6 * W + 1e-12   (fp32 4-factor product)
  forward     |gpu - oracle| <= 1e-6 * sum_c W_c |E_c| + 1e-30
  backward    |gpu - oracle| <= 1e-5 * sum |W_c g|; untouched entries exactly 0
  bf16 out    within half a bf16 ulp of the oracle + the forward bound
"""
import re

import numpy as np
import pytest
import torch

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2507_03836_b200 import fhash as fh


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def run_fwd(enc, case, out_dtype="f32"):
    out = enc.fwd(dev(case.coords), dev(case.table), out_dtype=out_dtype)
    st = enc.status_sync()
    return out.float().cpu().numpy().astype(np.float64), st


def run_bwd(enc, case):
    dtable = torch.zeros((enc.entries, enc.F), dtype=torch.float32, device="cuda")
    enc.bwd(dev(case.coords), dev(case.dout), dtable)
    st = enc.status_sync()
    return dtable.cpu().numpy().astype(np.float64), st


def kernel_names(fn):
    """Names of the CUDA kernels fn() launches (CUPTI through torch.profiler):
    proves which launch path a test exercised."""
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    return [e.name for e in prof.events() if e.device_type.name == "CUDA"]


def check_fwd(got, ref, absref, rel=1e-6):
    err = np.abs(got - ref)
    bound = rel * absref + 1e-30
    bad = err > bound
    assert not bad.any(), f"{bad.sum()} fwd mismatches; worst ratio {np.max(err / bound):.3g}"


def check_bwd(got, G, A, rel=1e-5):
    untouched = A == 0
    assert np.all(got[untouched] == 0.0), "untouched entries must be exactly zero"
    err = np.abs(got - G)
    bound = rel * A
    bad = (err > bound) & ~untouched
    assert not bad.any(), f"{bad.sum()} bwd mismatches; worst ratio {np.max(err[~untouched] / bound[~untouched]):.3g}"


CFGS = [W.CFG1, W.CFG1H]


@pytest.mark.parametrize("cfg", CFGS, ids=lambda c: c.name)
@pytest.mark.parametrize("N", [4096, 4096 + 37, 1, 255])
def test_indices_bit_exact(cfg, N):
    case = W.encode_case(cfg, N, seed=0)
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    ref = oracle.Levels(cfg.levels, cfg.cap)
    idx, w = enc.indices(dev(case.coords))
    assert enc.status_sync() == fh.FH_OK
    ridx, rW, _ = ref.indices(case.coords)
    assert np.array_equal(idx.cpu().numpy().view(np.uint32), ridx)
    wg = w.cpu().numpy().astype(np.float64)
    assert np.all(np.abs(wg - rW) <= 1e-6 * rW + 1e-12)


def test_indices_hand_computed_golden():
    """The kernels' corner indices on the hand-worked R5 case
    (tests/golden/r5_hash.json "pipeline"): not only equal to the oracle,
    equal to the arithmetic written out in the golden file."""
    import json
    import os
    p = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "r5_hash.json")))["pipeline"]
    enc = fh.Encoder([tuple(r) for r in p["levels"]], 2, "f32", p["cap"])
    idx, _ = enc.indices(dev(np.array([p["coord"]], np.float32)))
    got = idx.cpu().numpy().view(np.uint32)
    for c in p["corners"]:
        assert int(got[0, p["level"], c["c"]]) == c["index"], c


@pytest.mark.parametrize("cfg", CFGS, ids=lambda c: c.name)
@pytest.mark.parametrize("N", [4096, 4096 + 37, 1])
def test_forward_parity(cfg, N):
    case = W.encode_case(cfg, N, seed=0)
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    ref = oracle.Levels(cfg.levels, cfg.cap)
    got, st = run_fwd(enc, case)
    assert st == fh.FH_OK
    r, ab = ref.forward(case.coords, case.table, want_abs=True)
    check_fwd(got, r, ab)


@pytest.mark.parametrize("cfg", CFGS, ids=lambda c: c.name)
@pytest.mark.parametrize("N", [4096, 4096 + 37, 1])
def test_backward_parity(cfg, N):
    case = W.encode_case(cfg, N, seed=0)
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    ref = oracle.Levels(cfg.levels, cfg.cap)
    got, st = run_bwd(enc, case)
    assert st == fh.FH_OK
    G, A = ref.backward(case.coords, case.dout, cfg.F, want_abs=True)
    check_bwd(got, G, A)


@pytest.mark.parametrize("shift", ["0", "1", "2", "3"])
@pytest.mark.parametrize("F,tdt", [(1, "f32"), (2, "f32"), (2, "f16"), (4, "f16"), (1, "f16")])
def test_shifted_pairs_modes(shift, F, tdt, monkeypatch):
    """DESIGN.md §8.1 shifted pairs: FH_PAIR_SHIFT 0 (off), 1 (backward
    scratch, default), 3 (also the shifted table copy in the forward) give
    oracle-exact results on Eq. 9 and capped (R5) levels (2: forward only);
    the scratch is
    re-zeroed by the merge, so a second backward accumulates exactly."""
    monkeypatch.setenv("FH_PAIR_SHIFT", shift)
    cfg = W.EncoderConfig("shift", W.CFG1H.levels, F=F, cap=W.CFG1H.cap, table_dtype=tdt)
    case = W.encode_case(cfg, 8192 + 5, seed=21)
    enc = fh.Encoder(cfg.levels, F, tdt, cfg.cap)
    ref = oracle.Levels(cfg.levels, cfg.cap)
    got, st = run_fwd(enc, case)
    assert st == fh.FH_OK
    r, ab = ref.forward(case.coords, case.table, want_abs=True)
    check_fwd(got, r, ab)
    dtable = torch.zeros((enc.entries, F), dtype=torch.float32, device="cuda")
    c, g = dev(case.coords), dev(case.dout)
    enc.bwd(c, g, dtable)
    enc.bwd(c, g, dtable)
    assert enc.status_sync() == fh.FH_OK
    G, A = ref.backward(case.coords, case.dout, F, want_abs=True)
    check_bwd(dtable.cpu().numpy().astype(np.float64), 2 * G, 2 * A)


@pytest.mark.parametrize("cfg", [W.CFG1, W.CFG1H], ids=lambda c: c.name)
@pytest.mark.parametrize("N", [0, 1, 4096 + 37])
def test_backward_overwrite(cfg, N):
    """fh_encode_bwd_ex(FH_BWD_OVERWRITE): dtable = the gradient whatever it
    held before (every level group, the shared-memory small levels and the
    shifted scratch included); N = 0 leaves it all zero."""
    case = W.encode_case(cfg, max(N, 1), seed=3)
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    ref = oracle.Levels(cfg.levels, cfg.cap)
    dtable = torch.full((enc.entries, cfg.F), 7.0, device="cuda")
    c, g = dev(case.coords[:N]), dev(case.dout[:N])
    enc.bwd(c, g, dtable, overwrite=True)
    assert enc.status_sync() == fh.FH_OK
    if N == 0:
        assert torch.count_nonzero(dtable).item() == 0
        return
    G, A = ref.backward(case.coords[:N], case.dout[:N], cfg.F, want_abs=True)
    check_bwd(dtable.cpu().numpy().astype(np.float64), G, A)
    # fh_encode_fwd_bwd(zero_dtable=1) is the same overwrite
    dtable.fill_(-3.0)
    out = torch.empty((N, enc.L * cfg.F), device="cuda")
    enc.fwd_bwd(c, dev(case.table), out, g, dtable, zero_dtable=True)
    assert enc.status_sync() == fh.FH_OK
    check_bwd(dtable.cpu().numpy().astype(np.float64), G, A)


@pytest.mark.parametrize("F", [1, 2, 4, 8])
@pytest.mark.parametrize("tdt", ["f32", "f16"])
def test_feature_widths_and_dtypes(F, tdt):
    cfg = W.EncoderConfig("f", W.cfg1_levels(), F=F, cap=1 << 11, table_dtype=tdt)
    case = W.encode_case(cfg, 3001, seed=F)
    enc = fh.Encoder(cfg.levels, F, tdt, cfg.cap)
    ref = oracle.Levels(cfg.levels, cfg.cap)
    got, _ = run_fwd(enc, case)
    r, ab = ref.forward(case.coords, case.table.astype(np.float64), want_abs=True)
    check_fwd(got, r, ab)
    gb, _ = run_bwd(enc, case)
    G, A = ref.backward(case.coords, case.dout, F, want_abs=True)
    check_bwd(gb, G, A)


@pytest.mark.parametrize("tdt", ["f32", "f16"])
def test_bf16_output(tdt):
    """R13: bf16 encoder output = RNE(fp32 blend); within half a bf16 ulp of
    the oracle plus the fp32 forward bound."""
    cfg = W.EncoderConfig("b", W.cfg1_levels(), F=2, cap=1 << 11, table_dtype=tdt)
    case = W.encode_case(cfg, 4096, seed=5)
    enc = fh.Encoder(cfg.levels, 2, tdt, cfg.cap)
    ref = oracle.Levels(cfg.levels, cfg.cap)
    got, _ = run_fwd(enc, case, out_dtype="bf16")
    r, ab = ref.forward(case.coords, case.table.astype(np.float64), want_abs=True)
    half_ulp = np.ldexp(1.0, np.frexp(np.abs(r))[1] - 9)
    assert np.all(np.abs(got - r) <= half_ulp + 2e-6 * ab + 1e-30)


def test_edge_and_lattice_coordinates():
    """Domain edges (0, 1, next-below-1) and lattice vertices."""
    cfg = W.CFG1H
    coords = W.edge_coords()
    case = W.encode_case(cfg, len(coords), seed=1, coords=coords)
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    ref = oracle.Levels(cfg.levels, cfg.cap)
    idx, _ = enc.indices(dev(coords))
    assert enc.status_sync() == fh.FH_OK
    assert np.array_equal(idx.cpu().numpy().view(np.uint32), ref.indices(coords)[0])
    got, _ = run_fwd(enc, case)
    r, ab = ref.forward(coords, case.table, want_abs=True)
    check_fwd(got, r, ab)
    gb, _ = run_bwd(enc, case)
    G, A = ref.backward(coords, case.dout, cfg.F, want_abs=True)
    check_bwd(gb, G, A)


def test_out_of_domain_flagged_and_clamped():
    cfg = W.CFG1
    bad = W.bad_coords()
    case = W.encode_case(cfg, len(bad), seed=2, coords=bad)
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    ref = oracle.Levels(cfg.levels, cfg.cap)
    got, st = run_fwd(enc, case)
    assert st == fh.FH_E_DOMAIN
    assert enc.status_sync() == fh.FH_OK  # flag cleared by the read
    r, ab = ref.forward(bad, case.table, want_abs=True)
    check_fwd(got, r, ab)
    gb, st = run_bwd(enc, case)
    assert st == fh.FH_E_DOMAIN
    G, A = ref.backward(bad, case.dout, cfg.F, want_abs=True)
    check_bwd(gb, G, A)


def test_empty_batch_is_noop():
    enc = fh.Encoder(W.CFG1.levels, 2)
    c = torch.empty((0, 4), device="cuda")
    out = enc.fwd(c, torch.zeros((enc.entries, 2), device="cuda"))
    assert out.shape == (0, 8)
    assert enc.status_sync() == fh.FH_OK


def test_single_level_extremes():
    """Degenerate resolutions: all-2 level (one cell), a long thin level,
    and 32 levels (the maximum)."""
    levels = [(2, 2, 2, 2), (1000, 2, 2, 2), (2, 2, 2, 1000)] + [(3, 4, 5, 2)] * 29
    cfg = W.EncoderConfig("x", tuple(levels), F=2, cap=0, table_dtype="f32")
    case = W.encode_case(cfg, 777, seed=4)
    enc = fh.Encoder(levels, 2)
    ref = oracle.Levels(levels)
    idx, _ = enc.indices(dev(case.coords))
    assert np.array_equal(idx.cpu().numpy().view(np.uint32), ref.indices(case.coords)[0])
    got, _ = run_fwd(enc, case)
    r, ab = ref.forward(case.coords, case.table, want_abs=True)
    check_fwd(got, r, ab)


# ------------------------------------------ NEXT-2: brick linearization (R21)
BRICK_LEVELS = [W.cfg1_levels(), ((5, 7, 9, 3), (13, 3, 6, 7), (2, 2, 2, 2), (17, 2, 11, 5)),
                tuple(oracle.fold_schedule((200, 110, 54), 10, 2)[3:])]


@pytest.mark.parametrize("levels", BRICK_LEVELS, ids=["cfg1", "ragged", "fold2-tail"])
@pytest.mark.parametrize("cap", [0, 1 << 11])
def test_brick_indices_forward_backward(levels, cap):
    """FH_LIN_BRICK: indices bit-exact against the oracle's brick order
    (Levels(lin=1)) on even, odd and degenerate shapes with and without
    capped levels; forward and backward within the bars."""
    cfg = W.EncoderConfig("brick", tuple(levels), F=2, cap=cap, table_dtype="f32")
    case = W.encode_case(cfg, 4096 + 37, seed=11)
    enc = fh.Encoder(cfg.levels, 2, "f32", cap, lin=fh.FH_LIN_BRICK)
    ref = oracle.Levels(cfg.levels, cap, lin=1)
    idx, w = enc.indices(dev(case.coords))
    assert enc.status_sync() == fh.FH_OK
    ridx, rW, _ = ref.indices(case.coords)
    assert np.array_equal(idx.cpu().numpy().view(np.uint32), ridx)
    got, _ = run_fwd(enc, case)
    r, ab = ref.forward(case.coords, case.table, want_abs=True)
    check_fwd(got, r, ab)
    gb, _ = run_bwd(enc, case)
    G, A = ref.backward(case.coords, case.dout, 2, want_abs=True)
    check_bwd(gb, G, A)


def test_brick_edges():
    """Brick order at the domain edges / lattice points."""
    cfg = W.EncoderConfig("brick", W.cfg1_levels(), F=2, cap=0, table_dtype="f32")
    coords = np.concatenate([W.edge_coords(), W.draw_coords(W.rng(12), 6000)])
    case = W.encode_case(cfg, len(coords), seed=12, coords=coords)
    enc = fh.Encoder(cfg.levels, 2, lin=fh.FH_LIN_BRICK)
    ref = oracle.Levels(cfg.levels, 0, lin=1)
    idx, _ = enc.indices(dev(coords))
    assert np.array_equal(idx.cpu().numpy().view(np.uint32), ref.indices(coords)[0])
    c, t, g = dev(case.coords), dev(case.table), dev(case.dout)
    a = enc.fwd(c, t)
    r, ab = ref.forward(coords, case.table, want_abs=True)
    check_fwd(a.cpu().numpy().astype(np.float64), r, ab)
    dt = torch.zeros((enc.entries, 2), device="cuda")
    enc.bwd(c, g, dt)
    G, A = ref.backward(coords, case.dout, 2, want_abs=True)
    check_bwd(dt.cpu().numpy().astype(np.float64), G, A)


def test_brick_cfg2_full_size():
    """cfg2 (levels 0-4 bijective -> brick order, 5-15 hashed) at the bench
    size: forward on every row and backward on every entry vs the oracle."""
    cfg = W.CFG2
    case = W.encode_case(cfg, W.N_CFG2, seed=3)
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap, lin=fh.FH_LIN_BRICK)
    ref = oracle.Levels(cfg.levels, cfg.cap, lin=1)
    got, st = run_fwd(enc, case)
    assert st == fh.FH_OK
    r, ab = ref.forward(case.coords, case.table, want_abs=True)
    check_fwd(got, r, ab)
    del r, ab, got
    gb, _ = run_bwd(enc, case)
    G, A = ref.backward(case.coords, case.dout, cfg.F, want_abs=True)
    check_bwd(gb, G, A)


# ----------------------------------------------- full size (bench launch cfg)
def test_cfg2_full_size_parity():
    """BASELINE.json configs[1] at full size (2^20 points, 16 levels), the
    launch configuration bench.py times: forward on every row, backward on
    every entry, indices on a 64k-row sample."""
    cfg = W.CFG2
    case = W.encode_case(cfg, W.N_CFG2, seed=0)
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    ref = oracle.Levels(cfg.levels, cfg.cap)
    sub = case.coords[::16]
    idx, _ = enc.indices(dev(sub), want_w=False)
    assert np.array_equal(idx.cpu().numpy().view(np.uint32), ref.indices(sub, want_w=False)[0])
    got, st = run_fwd(enc, case)
    assert st == fh.FH_OK
    r, ab = ref.forward(case.coords, case.table, want_abs=True)
    check_fwd(got, r, ab)
    del r, ab, got
    gb, _ = run_bwd(enc, case)
    G, A = ref.backward(case.coords, case.dout, cfg.F, want_abs=True)
    check_bwd(gb, G, A)


def test_cfg4_sampled_rows_and_adjoint():
    """BASELINE.json configs[3] shapes (2^22 points, F=4, fp16 tables capped
    at 2^22): forward on sampled rows vs the oracle, and the adjoint identity
    <g, fwd(E)> = <bwd(g), E> at full size."""
    cfg = W.CFG4
    g = W.rng(0)
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    table = W.draw_table(g, enc.entries, cfg.F, "f16")
    coords = W.draw_coords(g, W.N_CFG4)
    ref = oracle.Levels(cfg.levels, cfg.cap)
    c_d, t_d = dev(coords), dev(table)
    out = enc.fwd(c_d, t_d)
    rows = np.random.default_rng(1).choice(W.N_CFG4, 1 << 15, replace=False)
    r, ab = ref.forward(coords[rows], table.astype(np.float64), want_abs=True)
    check_fwd(out[torch.from_numpy(rows).cuda()].cpu().numpy().astype(np.float64), r, ab)
    dout = torch.randn(out.shape, device="cuda", generator=torch.Generator("cuda").manual_seed(0))
    dtab = torch.zeros((enc.entries, cfg.F), device="cuda")
    enc.bwd(c_d, dout, dtab)
    assert enc.status_sync() == fh.FH_OK
    lhs = torch.sum(dout.double() * out.double()).item()
    rhs = torch.sum(dtab.double() * t_d.double()).item()
    scale = torch.sum(dout.double().abs() * out.double().abs()).item()
    assert abs(lhs - rhs) <= 1e-5 * scale


def test_cfg4_full_size_backward_every_entry():
    """BASELINE.json configs[3] (2^22 points, L=16, F=4, fp16 tables capped
    at 2^22: 40 M entries, 609 MiB of fp32 gradients, the HBM regime) in the
    launch configuration bench.py times (FH_BWD_OVERWRITE into a NaN-filled
    buffer, L2-sized level groups): the backward on EVERY entry against
    Oracle-B -- the dominant kernel of the train step."""
    cfg = W.CFG4
    g = W.rng(40)
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    coords = W.draw_coords(g, W.N_CFG4)
    dout = g.standard_normal((W.N_CFG4, cfg.L * cfg.F), dtype=np.float32)
    c_d, g_d = dev(coords), dev(dout)
    dt = torch.full((enc.entries, cfg.F), float("nan"), device="cuda")
    enc.bwd(c_d, g_d, dt, overwrite=True)
    assert enc.status_sync() == fh.FH_OK
    got = dt.cpu().numpy()
    # the same gradient from a level-major dout (FH_BWD_DOUT_LEVEL_MAJOR, the
    # trainer's dL/d(enc) layout for F >= 4)
    g_lm = g_d.view(W.N_CFG4, cfg.L, cfg.F).permute(1, 0, 2).contiguous()
    del g_d
    dt.fill_(float("nan"))
    enc.bwd(c_d, g_lm, dt, overwrite=True, level_major=True)
    assert enc.status_sync() == fh.FH_OK
    got_lm = dt.cpu().numpy()
    del dt, c_d, g_lm
    G, A = oracle.Levels(cfg.levels, cfg.cap).backward(coords, dout, cfg.F, want_abs=True)
    del dout
    check_bwd(got.astype(np.float64), G, A)
    check_bwd(got_lm.astype(np.float64), G, A)


def test_combustion_fold2_full_size_every_entry():
    """The paper's own encoder: Combustion-Seg, pure MPHF (Eq. 9; no
    cap), fold 2 (Eqs. 4-8; 24.2 Mi parameters), F = 2 fp32, at
    the paper's batch of 2^21 -- forward on every row and backward on
    every entry against the oracle.  This one launch sequence runs the
    entry-range passes of the 95 MB finest level, the 64-copy replicated pass
    of the 4900-entry level and the shared-memory few-cell launches
    (CTA copies and lane-private tiny levels) together; the launch list
    proves each ran."""
    levels = tuple(oracle.fold_schedule((200, 110, 54), 10, 2))
    cfg = W.EncoderConfig("pc", levels, F=2, cap=0, table_dtype="f32")
    N = 1 << 21
    case = W.encode_case(cfg, N, seed=41)
    enc = fh.Encoder(levels, 2)
    assert enc.param_count == 25374176
    ref = oracle.Levels(levels)
    c, t, g = dev(case.coords), dev(case.table), dev(case.dout)
    out = enc.fwd(c, t)
    dt = torch.full((enc.entries, 2), float("nan"), device="cuda")
    enc.bwd(c, g, dt, overwrite=True)               # first pass on the stream: scratch attached
    dt.fill_(float("nan"))
    names = kernel_names(lambda: enc.bwd(c, g, dt, overwrite=True))
    assert any("bwd_kernel<2, true>" in n for n in names), "entry-range passes"
    assert any("rep_reduce_kernel" in n for n in names), "replicated pass"
    assert sum("bwd_small_kernel" in n for n in names) >= 2, "CTA-copy and lane-private launches"
    assert enc.status_sync() == fh.FH_OK
    got = out.cpu().numpy().astype(np.float64)
    r, ab = ref.forward(case.coords, case.table, want_abs=True)
    check_fwd(got, r, ab)
    del r, ab, got
    G, A = ref.backward(case.coords, case.dout, 2, want_abs=True)
    check_bwd(dt.cpu().numpy().astype(np.float64), G, A)


# ------------------------------------------------------ closed forms on GPU
def test_constant_table_and_multilinear_on_gpu():
    """Closed forms, no oracle: constant table -> constant output;
    multilinear table -> p_x p_y p_z p_t."""
    levels = [(4, 7, 5, 3), (13, 6, 9, 4)]
    enc = fh.Encoder(levels, 2)
    coords = W.draw_coords(W.rng(8), 5000)
    c = dev(coords)
    out = enc.fwd(c, torch.full((enc.entries, 2), 0.25, device="cuda")).cpu().numpy()
    assert np.all(out == 0.25)
    tab = np.zeros((enc.entries, 2), np.float32)
    off = 0
    for r in levels:
        for t in range(r[3]):
            for z in range(r[2]):
                for y in range(r[1]):
                    for x in range(r[0]):
                        j = off + x + r[0] * (y + r[1] * (z + r[2] * t))
                        tab[j, 0] = (x / (r[0] - 1)) * (y / (r[1] - 1)) * (z / (r[2] - 1)) * (t / (r[3] - 1))
        off += r[0] * r[1] * r[2] * r[3]
    out = enc.fwd(c, dev(tab)).cpu().numpy().astype(np.float64)
    exp = np.prod(coords.astype(np.float64), axis=1)
    assert np.max(np.abs(out[:, 0] - exp)) < 2e-6
    assert np.max(np.abs(out[:, 2] - exp)) < 2e-6


def test_concurrent_streams_share_one_encoder():
    """The shifted-pair scratch is per (encoder, stream): two
    full-size passes of ONE encoder on two streams at once, different data,
    each equal to the oracle on its own inputs (sampled rows / adjoint at
    cfg2 size would not see a scratch race between the streams; an exact
    check needs oracle-sized inputs, so cfg1h at a batch large enough to use
    the scratch on every level)."""
    cfg = W.CFG1H
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    ref = oracle.Levels(cfg.levels, cfg.cap)
    cases = [W.encode_case(cfg, 40000 + k, seed=40 + k) for k in range(2)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs, dts = [], []
    torch.cuda.synchronize()
    for case, st in zip(cases, streams):
        with torch.cuda.stream(st):
            c, t, g = dev(case.coords), dev(case.table), dev(case.dout)
            o = torch.empty((c.shape[0], enc.L * cfg.F), device="cuda")
            d = torch.full((enc.entries, cfg.F), 5.0, device="cuda")
            for _ in range(3):   # repeated passes keep both streams busy together
                enc.fwd(c, t, o, stream=st)
                enc.bwd(c, g, d, stream=st, overwrite=True)
            outs.append(o)
            dts.append(d)
    torch.cuda.synchronize()
    assert enc.status_sync() == fh.FH_OK
    for case, o, d in zip(cases, outs, dts):
        r, ab = ref.forward(case.coords, case.table, want_abs=True)
        check_fwd(o.cpu().numpy().astype(np.float64), r, ab)
        G, A = ref.backward(case.coords, case.dout, cfg.F, want_abs=True)
        check_bwd(d.cpu().numpy().astype(np.float64), G, A)


def test_kernel_launch_counter():
    """fh_kernel_launches counts the library's kernels: a cfg1h fwd + bwd
    issues at least one forward and one backward launch, and nothing is
    counted for an empty batch."""
    cfg = W.CFG1H
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    case = W.encode_case(cfg, 5000, seed=2)
    c, t, g = dev(case.coords), dev(case.table), dev(case.dout)
    d = torch.zeros((enc.entries, cfg.F), device="cuda")
    n0 = fh.kernel_launches()
    enc.fwd(c[:0], t, torch.empty((0, enc.L * cfg.F), device="cuda"))
    enc.bwd(c[:0], g[:0], d)
    assert fh.kernel_launches() == n0
    enc.fwd(c, t)
    n1 = fh.kernel_launches()
    enc.bwd(c, g, d)
    n2 = fh.kernel_launches()
    torch.cuda.synchronize()
    assert n1 - n0 >= 1 and n2 - n1 >= 1


def test_step_host_end_to_end():
    """fh_encode_step_host (the bench's e2e path): H2D of coords / dout from
    pinned host buffers, fwd, bwd overwriting a dtable that held garbage,
    D2H of out and dtable -- host results equal the oracle."""
    cfg = W.CFG1H
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    ref = oracle.Levels(cfg.levels, cfg.cap)
    case = W.encode_case(cfg, 3000 + 7, seed=9)
    N, LF = case.coords.shape[0], enc.L * cfg.F
    coords_h = torch.from_numpy(np.ascontiguousarray(case.coords)).pin_memory()
    dout_h = torch.from_numpy(np.ascontiguousarray(case.dout)).pin_memory()
    out_h = torch.empty((N, LF)).pin_memory()
    dt_h = torch.empty((enc.entries, cfg.F)).pin_memory()
    table = dev(case.table)
    cd, gd = torch.empty((N, 4), device="cuda"), torch.empty((N, LF), device="cuda")
    od = torch.empty((N, LF), device="cuda")
    dd = torch.full((enc.entries, cfg.F), float("nan"), device="cuda")
    st = torch.cuda.Stream()
    enc.step_host(coords_h, dout_h, table, cd, gd, od, dd, out_h, dt_h, st)
    st.synchronize()
    assert enc.status_sync(st) == fh.FH_OK
    r, ab = ref.forward(case.coords, case.table, want_abs=True)
    check_fwd(out_h.numpy().astype(np.float64), r, ab)
    G, A = ref.backward(case.coords, case.dout, cfg.F, want_abs=True)
    check_bwd(dt_h.numpy().astype(np.float64), G, A)


@pytest.mark.parametrize("F,lm", [(1, False), (2, False), (2, True), (4, True)])
@pytest.mark.parametrize("split", ["0", "1"])
def test_backward_entry_range_passes(split, F, lm, monkeypatch):
    """A level whose gradients exceed the backward group budget is reduced
    in entry-range passes (FH_BWD_SPLIT, default on for F <= 2; F = 4 keeps
    one pass: cfg4 with a level-major dout and FH_BWD_OVERWRITE, the train
    step's form, 5.36 ms in one pass vs 5.47 in two): forced with a tiny
    budget (FH_BWD_GROUP_MB) on cfg1h, results equal the oracle."""
    monkeypatch.setenv("FH_BWD_SPLIT", split)
    monkeypatch.setenv("FH_BWD_GROUP_MB", "0.002")   # 2 KB: every level alone, all but level 0 split
    monkeypatch.setenv("FH_SMALL_MAX_T", "0")        # no level in the shared-memory pass
    cfg = W.EncoderConfig("split", W.CFG1H.levels, F=F, cap=W.CFG1H.cap, table_dtype="f32")
    N = 6000 + 3
    case = W.encode_case(cfg, N, seed=17)
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    ref = oracle.Levels(cfg.levels, cfg.cap)
    c, g = dev(case.coords), dev(case.dout)
    if lm:
        g = g.view(N, cfg.L, F).permute(1, 0, 2).contiguous()
    dt = torch.zeros((enc.entries, F), device="cuda")
    names = kernel_names(lambda: enc.bwd(c, g, dt, level_major=lm))
    st = enc.status_sync()
    got = dt.cpu().numpy().astype(np.float64)
    ranged = any(re.search(r"bwd_kernel<\d+, (true|1)>", n) for n in names)
    assert ranged == (split == "1" and F <= 2), names
    assert st == fh.FH_OK
    G, A = ref.backward(case.coords, case.dout, cfg.F, want_abs=True)
    check_bwd(got, G, A)


@pytest.mark.parametrize("levels,cap,F", [([(1024, 1024, 1023, 2), (4, 4, 4, 2)], 0, 2),
                                          ([(2048, 2048, 1024, 2), (5, 3, 4, 2)], 1 << 31, 1)],
                         ids=["eq9-2^31-entries", "hash-cap-2^31"])
def test_maximum_table_size(levels, cap, F):
    """Maximum sizes (sum T_l * F just below 2^32, the uint32 index range of
    the ABI): a bijective level of 2^31 - 2^21 entries at F = 2, and a level
    capped at 2^31 (R5 hash) at F = 1, each followed by a small level whose
    offset is near the top of the range.  Indices bit-exact against the
    oracle; partition of unity (constant table -> output 1); backward by the
    adjoint identity <g, fwd(t)> = <bwd(g), t> (the oracle cannot hold the
    17 GB tables in fp64)."""
    enc = fh.Encoder(levels, F, "f32", cap)
    ref = oracle.Levels(levels, cap)
    assert enc.entries == ref.total and enc.entries * F < (1 << 32)
    g = W.rng(77)
    coords = np.concatenate([W.draw_coords(g, 4000), W.edge_coords()]).astype(np.float32)
    c = dev(coords)
    idx, _ = enc.indices(c)
    assert enc.status_sync() == fh.FH_OK
    assert np.array_equal(idx.cpu().numpy().view(np.uint32), ref.indices(coords, want_w=False)[0])
    gen = torch.Generator("cuda").manual_seed(5)
    table = torch.ones((enc.entries, F), device="cuda")
    out = enc.fwd(c, table)
    assert torch.allclose(out, torch.ones_like(out), rtol=0, atol=1e-6)
    table.uniform_(-1.0, 1.0, generator=gen)
    out = enc.fwd(c, table)
    dout = torch.randn(out.shape, device="cuda", generator=gen)
    dt = torch.zeros_like(table)
    enc.bwd(c, dout, dt)
    assert enc.status_sync() == fh.FH_OK
    lhs = torch.sum(dout.double() * out.double()).item()
    rhs = 0.0
    step = 1 << 26
    for a in range(0, enc.entries, step):
        rhs += torch.sum(dt[a:a + step].double() * table[a:a + step].double()).item()
    scale = torch.sum(dout.abs().double()).item()
    assert abs(lhs - rhs) <= 1e-5 * scale, (lhs, rhs, scale)
    # the small last level, placed at the top of the index range, exactly:
    # the oracle of that level alone sees the same corners (level-local)
    last = ref.L - 1
    off, T = int(ref.offset[last]), int(ref.tsize[last])
    sub = oracle.Levels([levels[last]], cap)
    G, A = sub.backward(coords, dout[:, last * F:(last + 1) * F].cpu().numpy(), F, want_abs=True)
    check_bwd(dt[off:off + T].cpu().numpy().astype(np.float64), G, A)
    del table, dt
    torch.cuda.empty_cache()


def test_encode_makes_no_device_allocations():
    """SURVEY.md §8(b) ownership: after fh_build_levels (which makes the
    16-byte status word) no encode call allocates device memory -- large
    fwd / bwd passes without scratch (no shifted pairs) and with caller
    scratch leave the device's free memory unchanged."""
    cfg = W.CFG2
    N = 1 << 18
    g = torch.Generator("cuda").manual_seed(1)
    c = torch.rand((N, 4), device="cuda", generator=g)
    warm = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    t = torch.zeros((warm.entries, cfg.F), device="cuda")
    out = torch.empty((N, cfg.L * cfg.F), device="cuda")
    dout = torch.randn((N, cfg.L * cfg.F), device="cuda", generator=g)
    dt = torch.empty_like(t)
    warm.fwd(c, t, out)
    warm.bwd(c, dout, dt, overwrite=True)             # loads every kernel module
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap, auto_scratch=False)
    buf = torch.empty(enc.scratch_size(), dtype=torch.uint8, device="cuda")
    s2 = torch.cuda.Stream()
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    enc.fwd(c, t, out)
    enc.bwd(c, dout, dt, overwrite=True)
    enc.attach_scratch(buf, s2)
    enc.fwd(c, t, out, stream=s2)
    enc.bwd(c, dout, dt, stream=s2, overwrite=True)
    torch.cuda.synchronize()
    assert torch.cuda.mem_get_info()[0] == free0
    assert enc.status_sync() == fh.FH_OK


def test_caller_owned_scratch():
    """fh_encoder_attach_scratch: the shifted-pair scratch in caller-owned
    memory (the caller owns every device buffer); results
    equal the oracle; detach works; MHE encoders refuse."""
    cfg = W.CFG1H
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    ref = oracle.Levels(cfg.levels, cfg.cap)
    n = enc.scratch_size()
    assert n >= enc.entries * cfg.F * 4
    buf = torch.empty(n, dtype=torch.uint8, device="cuda")
    st = torch.cuda.Stream()
    enc.attach_scratch(buf, st)
    case = W.encode_case(cfg, 20000, seed=23)
    with torch.cuda.stream(st):
        c, t, g = dev(case.coords), dev(case.table), dev(case.dout)
        out = enc.fwd(c, t, stream=st)
        d = torch.full((enc.entries, cfg.F), 3.0, device="cuda")
        enc.bwd(c, g, d, stream=st, overwrite=True)
    st.synchronize()
    assert enc.status_sync(st) == fh.FH_OK
    r, ab = ref.forward(case.coords, case.table, want_abs=True)
    check_fwd(out.cpu().numpy().astype(np.float64), r, ab)
    G, A = ref.backward(case.coords, case.dout, cfg.F, want_abs=True)
    check_bwd(d.cpu().numpy().astype(np.float64), G, A)
    enc.attach_scratch(None, st)
    with pytest.raises(fh.FHashError):
        enc.attach_scratch(buf[: n // 2], st)          # too small
    mhe = fh.MHEEncoder([8, 16], 2, 1 << 10, 2, "f32")
    assert mhe.scratch_size() == 0
    with pytest.raises(fh.FHashError):
        mhe.attach_scratch(buf, st)


@pytest.mark.parametrize("rep", ["0", "8191"])
def test_backward_replicated_pass(rep, monkeypatch):
    """A contended mid-size level (2048 < T < 8192 entries, >= 4096 updates
    per entry) is reduced in a pass of its own into 64 replicated copies
    summed afterwards (FH_REP_MAX_T; 0 disables): equal to the oracle, at an
    ODD level offset (81: the copies start at the even entry below it so the
    pairs keep their 16-byte alignment).  The launch list proves which path
    ran (rep_reduce_kernel)."""
    monkeypatch.setenv("FH_REP_MAX_T", rep)
    levels = [(3, 3, 3, 3), (9, 9, 9, 9)]           # offset of level 1 = 81 (odd), T = 6561
    cfg = W.EncoderConfig("rep", tuple(levels), F=2, cap=0, table_dtype="f32")
    N = 1 << 21                                     # 16 N / T = 5114 updates per entry
    case = W.encode_case(cfg, N, seed=31)
    enc = fh.Encoder(levels, 2)
    ref = oracle.Levels(levels)
    c, g = dev(case.coords), dev(case.dout)
    dt = torch.zeros((enc.entries, 2), device="cuda")
    enc.bwd(c, g, dt)                               # attaches the scratch (first pass on the stream)
    dt.zero_()
    names = kernel_names(lambda: enc.bwd(c, g, dt))
    assert any("rep_reduce_kernel" in n for n in names) == (rep != "0"), names
    assert enc.status_sync() == fh.FH_OK
    G, A = ref.backward(case.coords, case.dout, 2, want_abs=True)
    check_bwd(dt.cpu().numpy().astype(np.float64), G, A)


def test_backward_f1_adjacent_odd_levels():
    """F = 1 with two adjacent mid-size levels at an odd boundary (6561):
    no shifted scratch or replicated copies for F = 1 (their merge works in
    16-byte float pairs that would straddle the boundary); equal to the
    oracle, a second pass accumulates exactly."""
    levels = [(9, 9, 9, 9), (16, 16, 16, 16)]
    cfg = W.EncoderConfig("f1", tuple(levels), F=1, cap=0, table_dtype="f32")
    case = W.encode_case(cfg, 100000, seed=32)
    enc = fh.Encoder(levels, 1)
    ref = oracle.Levels(levels)
    c, g = dev(case.coords), dev(case.dout)
    dt = torch.zeros((enc.entries, 1), device="cuda")
    enc.bwd(c, g, dt)
    enc.bwd(c, g, dt)
    assert enc.status_sync() == fh.FH_OK
    G, A = ref.backward(case.coords, case.dout, 1, want_abs=True)
    check_bwd(dt.cpu().numpy().astype(np.float64), 2 * G, 2 * A)


@pytest.mark.parametrize("tdt", ["f32", "f16"])
def test_forward_shifted_copy_odd_run_start(tdt):
    """The forward's shifted table copy when a run of shifted levels starts
    at an ODD offset: a large unshifted level (129^3 x 5, 10.7 M entries,
    beyond the copy budget) followed by a small one at offset 10,733,445.
    The scratch is filled with NaN first, so a slot the copy misses shows
    up; samples at the first cells of level 1 read the pair (b, b + 1)."""
    levels = [(129, 129, 129, 5), (65, 65, 65, 3)]
    cfg = W.EncoderConfig("oddrun", tuple(levels), F=2, cap=0, table_dtype=tdt)
    enc = fh.Encoder(levels, 2, tdt, 0, auto_scratch=False)
    assert enc.level_info(1)["offset"] % 2 == 1
    g = W.rng(33)
    corner = np.array([[0.0, 0.0, 0.0, 0.0], [1e-3, 1e-3, 1e-3, 1e-3], [0.01, 0.0, 0.0, 0.2]], np.float32)
    coords = np.concatenate([np.repeat(corner, 50, axis=0), W.draw_coords(g, 1 << 17)]).astype(np.float32)
    case = W.encode_case(cfg, len(coords), seed=33, coords=coords)
    buf = torch.full((enc.scratch_size() // 4,), float("nan"), device="cuda").view(torch.uint8)
    enc.attach_scratch(buf)
    c, t = dev(case.coords), dev(case.table)
    out = enc.fwd(c, t)
    assert enc.status_sync() == fh.FH_OK
    r, ab = oracle.Levels(levels).forward(case.coords, case.table, want_abs=True)
    check_fwd(out.cpu().numpy().astype(np.float64), r, ab)


def test_host_threads_share_one_encoder():
    """Two host threads drive one encoder on their own streams at the same
    time (ctypes releases the GIL): the per-stream scratch attach is
    serialised by the encoder's lock; both results equal the oracle."""
    import threading
    cfg = W.CFG1H
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    ref = oracle.Levels(cfg.levels, cfg.cap)
    cases = [W.encode_case(cfg, 30000 + k, seed=60 + k) for k in range(2)]
    results, errors = [None, None], []

    def run(k):
        try:
            st = torch.cuda.Stream()
            case = cases[k]
            with torch.cuda.stream(st):
                c, t, g = dev(case.coords), dev(case.table), dev(case.dout)
                o = enc.fwd(c, t, stream=st)
                d = torch.zeros((enc.entries, cfg.F), device="cuda")
                enc.bwd(c, g, d, stream=st, overwrite=True)
            st.synchronize()
            results[k] = (o.cpu().numpy().astype(np.float64), d.cpu().numpy().astype(np.float64))
        except Exception as ex:   # surfaced below
            errors.append(ex)

    threads = [threading.Thread(target=run, args=(k,)) for k in range(2)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
    assert enc.status_sync() == fh.FH_OK
    for case, (o, d) in zip(cases, results):
        r, ab = ref.forward(case.coords, case.table, want_abs=True)
        check_fwd(o, r, ab)
        G, A = ref.backward(case.coords, case.dout, cfg.F, want_abs=True)
        check_bwd(d, G, A)


@pytest.mark.parametrize("F", [1, 2, 4, 8])
def test_few_cell_levels_backward(F):
    """The coarse end of a fold schedule (the Combustion fold-2 tail: 728,
    112, 32 and 16 entries) in the shared-memory backward paths -- CTA /
    per-warp copies and one lane-private launch per tiny level -- for every
    F; equal to the oracle at a batch large enough that every entry takes
    thousands of contributions."""
    levels = [(13, 7, 4, 2), (7, 4, 2, 2), (4, 2, 2, 2), (2, 2, 2, 2)]
    cfg = W.EncoderConfig("tail", tuple(levels), F=F, cap=0, table_dtype="f32")
    case = W.encode_case(cfg, 200000, seed=44)
    enc = fh.Encoder(levels, F)
    ref = oracle.Levels(levels)
    got, st = run_bwd(enc, case)
    assert st == fh.FH_OK
    G, A = ref.backward(case.coords, case.dout, F, want_abs=True)
    check_bwd(got, G, A)


@pytest.mark.parametrize("F", [1, 2, 4, 8])
def test_backward_level_major_dout(F):
    """FH_BWD_DOUT_LEVEL_MAJOR: dout as [L][N][F] gives the oracle's
    gradient through every backward path -- the few-cell levels in shared
    memory, an L2 level group, a capped (hashed) level -- and accumulates
    (+=) like the row-major form; the overwrite flag combines with it."""
    levels = [(2, 2, 2, 2), (13, 7, 4, 2), (33, 33, 33, 5), (64, 64, 64, 8)]
    cfg = W.EncoderConfig("lm", tuple(levels), F=F, cap=1 << 16, table_dtype="f32")
    N = 60000 + 37
    case = W.encode_case(cfg, N, seed=45)
    enc = fh.Encoder(levels, F, "f32", 1 << 16)
    ref = oracle.Levels(levels, 1 << 16)
    c = dev(case.coords)
    g_lm = dev(case.dout).view(N, cfg.L, F).permute(1, 0, 2).contiguous()
    dt = torch.full((enc.entries, F), float("nan"), device="cuda")
    enc.bwd(c, g_lm, dt, overwrite=True, level_major=True)
    enc.bwd(c, g_lm, dt, level_major=True)
    assert enc.status_sync() == fh.FH_OK
    G, A = ref.backward(case.coords, case.dout, F, want_abs=True)
    check_bwd(dt.cpu().numpy().astype(np.float64), 2 * G, 2 * A)


@pytest.mark.parametrize("F", [4, 8])
@pytest.mark.parametrize("attach", [True, False])
def test_backward_inpass_replicas(F, attach):
    """F >= 4: a contended level (6561 entries, ~2560 updates each at 2^20
    samples) reduces into in-pass replicated copies of the scratch (CTA b ->
    copy b % R, then rep_reduce_kernel adds them into dtable); equal to the
    oracle on every entry, accumulating (+=) like the direct form.  Without
    a scratch attached the same call runs without copies, same result."""
    levels = [(9, 9, 9, 9), (16, 16, 16, 16), (33, 33, 33, 5)]
    cfg = W.EncoderConfig("inrep", tuple(levels), F=F, cap=0, table_dtype="f32")
    N = (1 << 20) + 5
    case = W.encode_case(cfg, N, seed=46)
    enc = fh.Encoder(levels, F, "f32", 0, auto_scratch=attach)
    ref = oracle.Levels(levels)
    c, g = dev(case.coords), dev(case.dout)
    g_lm = g.view(N, cfg.L, F).permute(1, 0, 2).contiguous()
    dt = torch.full((enc.entries, F), float("nan"), device="cuda")
    names = kernel_names(lambda: enc.bwd(c, g_lm, dt, overwrite=True, level_major=True))
    assert any("rep_reduce_kernel" in n for n in names) == attach, names
    enc.bwd(c, g, dt)
    assert enc.status_sync() == fh.FH_OK
    G, A = ref.backward(case.coords, case.dout, F, want_abs=True)
    check_bwd(dt.cpu().numpy().astype(np.float64), 2 * G, 2 * A)
