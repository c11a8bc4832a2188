"""NEXT-3 GPU parity: the MHE baseline encoder kernels against the oracle
(oracle.MHELevels).  Same bars as the F-Hash encode.  -m gpu."""
import numpy as np
import pytest
import torch

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2507_03836_b200 import fhash as fh

from test_parity_gpu import check_bwd, check_fwd, dev  # noqa: E402


@pytest.mark.parametrize("res,T,n,F,tdt,N", [([8, 16, 40], 4096, 4, 2, "f32", 4133),
                                             ([4, 9, 17, 33, 65], 1 << 12, 10, 2, "f16", 3001),
                                             ([16, 30, 60, 120], 1 << 14, 3, 4, "f32", 2000),
                                             ([5, 50], 1 << 10, 1, 1, "f32", 777)])
def test_mhe_indices_fwd_bwd(res, T, n, F, tdt, N):
    g = W.rng(len(res) * 7 + F)
    enc = fh.MHEEncoder(res, F, T, n, tdt)
    ref = oracle.MHELevels(res, n, T)
    assert enc.entries == ref.total and enc.param_count == ref.param_count(F)
    table = W.draw_table(g, enc.entries, F, tdt)
    coords = np.concatenate([W.draw_coords(g, N - 8), W.edge_coords()[:8]]).astype(np.float32)
    dout = W.draw_grads(g, N, len(res) * F)
    c = dev(coords)
    idx, w = enc.indices(c)
    assert enc.status_sync() == fh.FH_OK
    ridx, rW, _ = ref.indices(coords)
    assert np.array_equal(idx.cpu().numpy().view(np.uint32), ridx)
    assert np.all(np.abs(w.cpu().numpy() - rW) <= 1e-6 * rW + 1e-12)
    out = enc.fwd(c, dev(table)).cpu().numpy().astype(np.float64)
    r, ab = ref.forward(coords, table.astype(np.float64), want_abs=True)
    check_fwd(out, r, ab)
    dt = torch.zeros((enc.entries, F), device="cuda")
    enc.bwd(c, dev(dout), dt)
    G, A = ref.backward(coords, dout, F, want_abs=True)
    check_bwd(dt.cpu().numpy().astype(np.float64), G, A)


def test_mhe_paper_sized_encoder_adjoint():
    """Paper-scale MHE (T = 2^20, 6 levels, 10 key frames, F = 2; the
    Combustion MHE column of Table 3): adjoint identity at 2^20
    points."""
    res = W.geometric(16, 512, 6)
    enc = fh.MHEEncoder(res, 2, 1 << 20, 10, "f32")
    assert enc.param_count / 2 ** 20 == pytest.approx(120.0, abs=0.05)
    gen = torch.Generator("cuda").manual_seed(0)
    c = torch.rand((1 << 20, 4), device="cuda", generator=gen)
    t = (torch.rand((enc.entries, 2), device="cuda", generator=gen) - 0.5) * 2e-4
    out = enc.fwd(c, t)
    g = torch.randn(out.shape, device="cuda", generator=gen)
    dt = torch.zeros_like(t)
    enc.bwd(c, g, dt)
    lhs = torch.sum(g.double() * out.double()).item()
    rhs = torch.sum(dt.double() * t.double()).item()
    assert abs(lhs - rhs) <= 1e-5 * torch.sum(g.double().abs() * out.double().abs()).item()


def test_mhe_backward_overwrite():
    """fh_encode_bwd_ex(FH_BWD_OVERWRITE) on an MHE encoder: the dtable held
    garbage, the result equals the oracle's gradient."""
    res, T, n, F = [8, 16, 40], 4096, 4, 2
    g = W.rng(5)
    enc = fh.MHEEncoder(res, F, T, n, "f32")
    ref = oracle.MHELevels(res, n, T)
    coords = W.draw_coords(g, 3001).astype(np.float32)
    dout = W.draw_grads(g, 3001, len(res) * F)
    dt = torch.full((enc.entries, F), 9.0, device="cuda")
    enc.bwd(dev(coords), dev(dout), dt, overwrite=True)
    assert enc.status_sync() == fh.FH_OK
    G, A = ref.backward(coords, dout, F, want_abs=True)
    check_bwd(dt.cpu().numpy().astype(np.float64), G, A)
