"""Randomised parity sweep (-m gpu): random encoder configurations through
the C ABI against the oracle -- levels, per-axis resolutions (2..40),
capped / uncapped, F in {1,2,4,8}, fp32 / fp16 tables, Eq. 9 / brick order,
ragged batch sizes.  Same bars as tests/test_parity_gpu.py."""
import numpy as np
import pytest
import torch

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2507_03836_b200 import fhash as fh


def random_case(seed):
    g = np.random.default_rng(1000 + seed)
    L = int(g.integers(1, 9))
    levels = tuple(tuple(int(r) for r in g.integers(2, 41, 4)) for _ in range(L))
    F = int(g.choice([1, 2, 4, 8]))
    tdt = str(g.choice(["f32", "f16"]))
    cap = int(g.choice([0, 1 << 8, 1 << 11, 1 << 14]))
    lin = int(g.integers(0, 2))
    N = int(g.integers(1, 6000))
    return W.EncoderConfig(f"r{seed}", levels, F=F, cap=cap, table_dtype=tdt), lin, N


@pytest.mark.parametrize("seed", range(64))
def test_random_encoder_parity(seed):
    cfg, lin, N = random_case(seed)
    case = W.encode_case(cfg, N, seed=seed)
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap, lin=lin)
    ref = oracle.Levels(cfg.levels, cfg.cap, lin=lin)
    c = torch.from_numpy(case.coords).cuda()
    t = torch.from_numpy(case.table).cuda()
    g = torch.from_numpy(case.dout).cuda()
    idx, _ = enc.indices(c, want_w=False)
    ridx, _, _ = ref.indices(case.coords, want_w=False)
    assert np.array_equal(idx.cpu().numpy().view(np.uint32), ridx)
    out = enc.fwd(c, t)
    r, ab = ref.forward(case.coords, case.table.astype(np.float64), want_abs=True)
    got = out.cpu().numpy().astype(np.float64)
    assert np.all(np.abs(got - r) <= 1e-6 * ab + 1e-30)
    G, A = ref.backward(case.coords, case.dout, cfg.F, want_abs=True)
    dt = torch.zeros((enc.entries, cfg.F), device="cuda")
    enc.bwd(c, g, dt)
    gb = dt.cpu().numpy().astype(np.float64)
    assert np.all(gb[A == 0] == 0)
    assert np.all(np.abs(gb - G) <= 1e-5 * A)
    assert enc.status_sync() == fh.FH_OK


def random_large_case(seed):
    """Larger batches than random_case, so the N-dependent backward paths
    (shifted gradient pairs, replicated copies of contended levels, the
    few-cell shared-memory levels, the fused merges between level groups)
    all take part; coarse levels included on purpose."""
    g = np.random.default_rng(5000 + seed)
    L = int(g.integers(2, 9))
    lv = [tuple(int(r) for r in g.integers(2, 6, 4)) for _ in range(L // 2)]          # few-cell levels
    lv += [tuple(int(r) for r in g.integers(6, 41, 4)) for _ in range(L - L // 2)]   # larger / capped levels
    order = g.permutation(L)
    levels = tuple(lv[i] for i in order)
    F = int(g.choice([1, 2, 4]))
    cap = int(g.choice([0, 1 << 11, 1 << 14]))
    N = int(g.integers(100000, 300000))
    return W.EncoderConfig(f"R{seed}", levels, F=F, cap=cap, table_dtype="f32"), N


@pytest.mark.parametrize("seed", range(16))
def test_random_large_batch_backward(seed):
    cfg, N = random_large_case(seed)
    case = W.encode_case(cfg, N, seed=seed)
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    ref = oracle.Levels(cfg.levels, cfg.cap)
    c = torch.from_numpy(case.coords).cuda()
    g = torch.from_numpy(case.dout).cuda()
    G, A = ref.backward(case.coords, case.dout, cfg.F, want_abs=True)
    for overwrite in (False, True):
        dt = torch.full((enc.entries, cfg.F), 0.0 if not overwrite else 7.0, device="cuda")
        enc.bwd(c, g, dt, overwrite=overwrite)
        gb = dt.cpu().numpy().astype(np.float64)
        assert np.all(gb[A == 0] == 0)
        assert np.all(np.abs(gb - G) <= 1e-5 * A)
    assert enc.status_sync() == fh.FH_OK
