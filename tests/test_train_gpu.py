"""GPU parity of the train step (a8 MLP fwd/bwd on tcgen05, a9 MSE, a10
encode bwd of dL/d(enc), a11 Adam) against Oracle-T.  -m gpu.

Following SURVEY.md §8(c), the MLP oracle is fed the GPU's own bf16 encoder
output (so a bf16 rounding flip in the encode does not propagate), and the
encode backward is checked with the GPU's own dL/d(enc) as upstream.
Tolerances: loss 1e-3 relative; every MLP gradient element
and every dL/d(enc) element within 1e-2 of its own sum of |contributions|
plus the ReLU-ambiguity term (oracle.train.mlp_backward_bounds: bf16
operands, fp32 accumulation in a different order, occasional one-ulp bf16
flips of h / dz); table grads 1e-5 * sum|W g|; Adam elementwise 1e-6
relative (+ lr-scaled floor).
"""
import numpy as np
import pytest
import torch

import oracle
from oracle import train as T
import workloads as W

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2507_03836_b200 import fhash as fh


def small_cfg(F, L, tdt="f16", cap=1 << 12):
    levels = tuple((s, s, s, t) for s, t in zip(W.geometric(4, 24, L), W.geometric(2, 6, L)))
    return W.EncoderConfig(f"t{L}x{F}", levels, F=F, cap=cap, table_dtype=tdt)


def make(cfg, N, seed=0, max_batch=None):
    g = W.rng(seed)
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    table = W.draw_table(g, enc.entries, cfg.F, "f32")
    layers = W.draw_mlp(g, W.MLPConfig((cfg.L * cfg.F, 64, 64, 1)))
    coords = W.draw_coords(g, N)
    target = g.random(N, dtype=np.float32)
    tr = fh.Trainer(enc, table, layers, max_batch or N)
    return enc, tr, coords, target


@pytest.mark.parametrize("F,L,N", [(4, 4, 1000), (2, 16, 1000), (4, 16, 777), (2, 16, 128), (4, 12, 3000)])
def test_mlp_fwd_bwd_parity(F, L, N):
    cfg = small_cfg(F, L)
    enc, tr, coords, target = make(cfg, N, seed=F * 100 + L)
    check_fwd_bwd(cfg, tr, coords, target, N)


def test_train_fwd_bwd_cfg3_full_size():
    """bench.py's train_step launch configuration (BASELINE.json configs[2]:
    cfg3 encoder, L=16 F=2 fp16 tables cap 2^19, MLP 32-64-64-1, batch 2^18):
    2048 tiles, so every TMEM slot accumulates several tiles' weight
    gradients before its partial row and the reduce kernel -- the small cases
    above give each slot at most one tile.  Same bars as above."""
    cfg, N = W.CFG3, W.N_CFG3
    g = W.rng(33)
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    table = W.draw_table(g, enc.entries, cfg.F, "f32")
    layers = W.draw_mlp(g, W.MLP3)
    coords = W.draw_coords(g, N)
    target = g.random(N, dtype=np.float32)
    tr = fh.Trainer(enc, table, layers, N)
    assert (N + 127) // 128 > 2 * torch.cuda.get_device_properties(0).multi_processor_count
    check_fwd_bwd(cfg, tr, coords, target, N)


def test_train_fwd_bwd_cfg5_shape_multi_tile():
    """The K0 = 64 kernel bench.py's cfg5 leg runs (BASELINE.json configs[3]
    encoder: L=16 F=4 fp16 tables cap 2^22, MLP 64-64-64-1) at 2^20 samples
    (8192 tiles, ~28 per slot): loss, MLP gradients, dL/d(enc) and the table
    gradient (every entry of the 160 M-parameter table, through the cfg4
    backward's L2 level groups) against the oracle."""
    cfg, N = W.CFG4, 1 << 20
    g = W.rng(44)
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    table = W.draw_table(g, enc.entries, cfg.F, "f32")
    layers = W.draw_mlp(g, W.MLP4)
    coords = W.draw_coords(g, N)
    target = g.random(N, dtype=np.float32)
    tr = fh.Trainer(enc, table, layers, N)
    del table
    check_fwd_bwd(cfg, tr, coords, target, N)


@pytest.mark.parametrize("F,L,N", [(2, 16, 1), (4, 16, 129), (2, 8, 255), (4, 4, 7), (4, 16, 1), (4, 8, 8)])
def test_mlp_fwd_bwd_ragged_tiles(F, L, N):
    """Tile edges of the TMA paths: one sample, one full tile + one row, a
    tile short of one row, fewer rows than one 8-row group (the X tensor map
    zero-fills row groups past N; rows past N inside the last group are
    zeroed by the kernel; the dX tensor map clips rows past N)."""
    cfg = small_cfg(F, L)
    enc, tr, coords, target = make(cfg, N, seed=F * 10 + N)
    check_fwd_bwd(cfg, tr, coords, target, N)


@pytest.mark.parametrize("F,L", [(2, 16), (4, 8)])
def test_mlp_fwd_bwd_after_a_larger_batch(F, L):
    """A trainer's workspace keeps the previous call's encoder output and dX
    rows past the current N: a small batch after a large one must not read
    them (per-launch tensor maps sized to N), and its dX rows past N are
    left alone (F = 4: the level-major dX, [L][N][F] packed for this N, ends
    at N K0 floats; nothing past it is written)."""
    cfg = small_cfg(F, L)
    g = W.rng(77)
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    tr = fh.Trainer(enc, W.draw_table(g, enc.entries, cfg.F, "f32"), W.draw_mlp(g, W.MLPConfig((L * F, 64, 64, 1))), 5000)
    big = W.draw_coords(g, 5000)
    tr.fwd_bwd(torch.from_numpy(big).cuda(), torch.from_numpy(g.random(5000, dtype=np.float32)).cuda())
    torch.cuda.synchronize()
    raw_big = tr.dx_raw(5000).clone()
    N = 301
    coords = W.draw_coords(g, N)
    target = g.random(N, dtype=np.float32)
    check_fwd_bwd(cfg, tr, coords, target, N)
    # rows past N (also those inside the last 128-row tile) are clipped by the dX store
    K0 = L * F
    assert torch.equal(tr.dx_raw(5000)[N * K0:], raw_big[N * K0:])


def check_fwd_bwd(cfg, tr, coords, target, N, table_grad=True):
    c, t = torch.from_numpy(coords).cuda(), torch.from_numpy(target).cuda()
    assert tr.dx_layout() == (cfg.F if cfg.F >= 4 else 0)   # level-major dL/d(enc) for F >= 4
    n_global = N + 17  # exercise the 1/N_global scaling
    loss = tr.fwd_bwd(c, t, n_global)
    assert tr.status() == fh.FH_OK
    x0 = tr.enc_out(N).float().cpu().numpy().astype(np.float64)
    master = tr.mlp_master.cpu().numpy().astype(np.float64)
    K0 = cfg.L * cfg.F
    o = 0
    layers = []
    for fi, fo in ((K0, 64), (64, 64), (64, 1)):
        Wt = master[o:o + fi * fo].reshape(fo, fi); o += fi * fo
        b = master[o:o + fo]; o += fo
        layers.append((Wt, b))
    y, cache = T.mlp_forward(x0, layers)
    tg = target.astype(np.float64)
    ref_loss, dy = T.mse_loss(y, tg, n_global)
    grads, dx0 = T.mlp_backward(dy, layers, cache)
    bounds, A_dx, U_dx = T.mlp_backward_bounds(layers, cache, tg, n_global)
    assert abs(loss.item() - ref_loss) <= 1e-3 * abs(ref_loss)
    g = tr.mlp_grad.cpu().numpy().astype(np.float64)
    o = 0
    for k, ((dW, db), (AW, Ab, UW, Ub)) in enumerate(zip(grads, bounds)):
        for ref, A, U in ((dW.ravel(), AW.ravel(), UW.ravel()), (db.ravel(), Ab.ravel(), Ub.ravel())):
            got = g[o:o + ref.size]; o += ref.size
            err, tol = np.abs(got - ref), 1e-2 * A + U + 1e-30
            assert np.all(err <= tol), (k, int(np.sum(err > tol)), float(np.max(err / tol)))
    dx = tr.dx(N).cpu().numpy().astype(np.float64)
    err, tol = np.abs(dx - dx0), 1e-2 * A_dx + U_dx + 1e-30
    assert np.all(err <= tol), (int(np.sum(err > tol)), float(np.max(err / tol)))
    if not table_grad:
        return
    # encode bwd of the GPU's own dL/d(enc), against Oracle-B (strict)
    ref = oracle.Levels(cfg.levels, cfg.cap)
    G, A = ref.backward(coords, dx, cfg.F, want_abs=True)
    got = tr.table_grad.cpu().numpy().astype(np.float64)
    assert np.all(got[A == 0] == 0)
    assert np.all(np.abs(got - G) <= 1e-5 * A)


def test_encoder_output_is_bf16_of_forward():
    cfg = small_cfg(2, 16)
    enc, tr, coords, target = make(cfg, 500, seed=3)
    tr.fwd_bwd(torch.from_numpy(coords).cuda(), torch.from_numpy(target).cuda())
    x0 = tr.enc_out(500).float().cpu().numpy().astype(np.float64)
    ref = oracle.Levels(cfg.levels, cfg.cap)
    r, ab = ref.forward(coords, tr.table_shadow.float().cpu().numpy().astype(np.float64), want_abs=True)
    half_ulp = np.ldexp(1.0, np.frexp(np.abs(r))[1] - 9)
    assert np.all(np.abs(x0 - r) <= half_ulp + 2e-6 * ab + 1e-30)


def test_adam_parity_and_shadows():
    cfg = small_cfg(4, 8)
    enc, tr, coords, target = make(cfg, 256, seed=5)
    g = torch.Generator("cuda").manual_seed(1)
    p0 = (tr.table_master.clone(), tr.mlp_master.clone())
    for step in (1, 2, 3):
        gr = torch.randn(tr.grads.shape, device="cuda", generator=g) * 0.1
        tr.grads.copy_(gr)
        before = [x.clone().cpu().numpy().astype(np.float64) for x in
                  (tr.table_master, tr.table_m, tr.table_v, tr.mlp_master, tr.mlp_m, tr.mlp_v)]
        grn = gr.cpu().numpy().astype(np.float64)
        tr.apply()
        torch.cuda.synchronize()
        assert tr.step_count == step
        nt_pad = (tr.n_table + 3) // 4 * 4
        for (p, m, v), gseg, (pg, mg, vg) in (
                ((before[0].ravel(), before[1], before[2]), grn[:tr.n_table],
                 (tr.table_master, tr.table_m, tr.table_v)),
                ((before[3], before[4], before[5]), grn[nt_pad:], (tr.mlp_master, tr.mlp_m, tr.mlp_v))):
            rp, rm, rv = T.adam_step(p, gseg, m, v, step)
            gp = pg.cpu().numpy().ravel().astype(np.float64)
            assert np.all(np.abs(gp - rp) <= 1e-6 * (np.abs(rp) + 0.01))
            # m = b1 m + (1-b1) g cancels: bound by the magnitude of its terms
            assert np.all(np.abs(mg.cpu().numpy() - rm) <= 1e-6 * (0.9 * np.abs(m) + 0.1 * np.abs(gseg)) + 1e-12)
            assert np.allclose(vg.cpu().numpy(), rv, rtol=1e-6, atol=1e-15)
        assert torch.equal(tr.table_shadow, tr.table_master.half())
        assert torch.equal(tr.mlp_shadow, tr.mlp_master.bfloat16())
    assert not torch.equal(p0[0], tr.table_master)


def test_fp32_table_training_adam():
    """FH_F32 tables (no fp16 shadow: the kernels read the fp32 master
    directly): a full train step runs, Adam matches the oracle on every table
    parameter and writes no shadow."""
    cfg = small_cfg(2, 8, tdt="f32")
    enc, tr, coords, target = make(cfg, 900, seed=21)
    assert tr.table_shadow is None
    c, t = torch.from_numpy(coords).cuda(), torch.from_numpy(target).cuda()
    loss = tr.fwd_bwd(c, t)
    assert tr.status() == fh.FH_OK and torch.isfinite(loss).all()
    g = tr.grads.clone().cpu().numpy().astype(np.float64)
    before = [x.clone().cpu().numpy().astype(np.float64) for x in (tr.table_master, tr.table_m, tr.table_v)]
    tr.apply()
    torch.cuda.synchronize()
    rp, _, _ = T.adam_step(before[0].ravel(), g[:tr.n_table], before[1], before[2], 1)
    gp = tr.table_master.cpu().numpy().ravel().astype(np.float64)
    assert np.all(np.abs(gp - rp) <= 1e-6 * (np.abs(rp) + 0.01))
    loss2 = tr.step(c, t)   # the next step reads the updated fp32 master
    assert tr.status() == fh.FH_OK and torch.isfinite(loss2).all()


def test_sharded_apply_matches_full_apply():
    """fh_train_apply_sharded over [0, n) equals fh_train_apply; over a
    sub-range it touches only that range of the table state."""
    from paper_2507_03836_b200 import dp
    cfg = small_cfg(4, 8)
    trs = []
    for _ in range(2):
        enc, tr, coords, target = make(cfg, 700, seed=11)
        trs.append((enc, tr))
    c, t = torch.from_numpy(coords).cuda(), torch.from_numpy(target).cuda()
    (_, a), (_, b) = trs
    sdp = dp.ShardedDP(b)   # no process group: world 1, shard = whole table
    for _ in range(2):
        # identical gradients on both (the encode bwd's atomics are unordered)
        a.fwd_bwd(c, t, 700)
        b.grads.copy_(a.grads)
        a.apply()
        sdp.reduce()
        sdp.apply()
        sdp.gather()
    torch.cuda.synchronize()
    assert torch.equal(a.table_master, b.table_master)
    assert torch.equal(a.table_shadow, b.table_shadow)
    assert torch.equal(a.mlp_master, b.mlp_master)
    # partial range
    b.fwd_bwd(c, t, 700)
    before = b.table_master.clone().view(-1)
    shard = b.grads[:b.n_table].clone()
    lo, hi = 64, 64 + 400
    b.apply_sharded(lo, hi, shard[lo:hi].contiguous())
    torch.cuda.synchronize()
    after = b.table_master.view(-1)
    assert torch.equal(after[:lo], before[:lo]) and torch.equal(after[hi:], before[hi:])
    assert not torch.equal(after[lo:hi], before[lo:hi])


@pytest.mark.parametrize("F,L,N,tdt", [(2, 16, 1000, "f16"), (4, 16, 3001, "f16"), (4, 4, 130, "f16"),
                                        (1, 16, 200, "f16"), (8, 8, 500, "f32"), (2, 24, 700, "f32"),
                                        (2, 16, 1, "f16")])
def test_infer_forward_parity(F, L, N, tdt):
    """NEXT-1: fh_infer (ONE fused launch: encode fwd into the shared-memory
    X tile + tcgen05 MLP forward) equals Oracle-T's forward on the GPU's own
    bf16 encoding (which the fused kernel recomputes bit-identically), and
    reproduces the train step's loss."""
    cfg = small_cfg(F, L, tdt)
    enc, tr, coords, target = make(cfg, N, seed=21 + F + L)
    check_infer(cfg, tr, coords, target, N)


def test_infer_cfg3_full_size():
    """fh_infer at bench.py's cfg3 inference launch (2^18 samples, the cfg3
    encoder and MLP 32-64-64-1), same bars."""
    cfg, N = W.CFG3, W.N_CFG3
    g = W.rng(55)
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    tr = fh.Trainer(enc, W.draw_table(g, enc.entries, cfg.F, "f32"), W.draw_mlp(g, W.MLP3), N)
    check_infer(cfg, tr, W.draw_coords(g, N), g.random(N, dtype=np.float32), N)


def test_infer_cfg4_shape_many_tiles():
    """fh_infer with the cfg4 encoder (F = 4 fp16, K0 = 64: the two-group
    full-tile kernel) at 2^17 samples -- every CTA loops over several tiles
    and all four X buffers rotate -- same bars."""
    cfg, N = W.CFG4, 1 << 17
    g = W.rng(56)
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    tr = fh.Trainer(enc, W.draw_table(g, enc.entries, cfg.F, "f32"), W.draw_mlp(g, W.MLP4), N)
    check_infer(cfg, tr, W.draw_coords(g, N), g.random(N, dtype=np.float32), N)


def test_infer_two_phase_large_batch_hbm_tables():
    """A large batch over tables beyond the forward's L2 budget (cfg4: 305
    MiB fp16) takes fh_encode_fwd's L2-sized level groups into the workspace
    and then the fused kernel's MLP-only mode (fh_infer_workspace_size > 0):
    same bars against Oracle-T."""
    import ctypes
    cfg, N = W.CFG4, 1 << 18
    g = W.rng(57)
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    tr = fh.Trainer(enc, W.draw_table(g, enc.entries, cfg.F, "f32"), W.draw_mlp(g, W.MLP4), N)
    L = fh._train_lib()
    assert int(L.fh_infer_workspace_size(enc.handle, ctypes.byref(tr.desc), N)) >= N * 64 * 2
    check_infer(cfg, tr, W.draw_coords(g, N), g.random(N, dtype=np.float32), N, one_launch=False)


def check_infer(cfg, tr, coords, target, N, one_launch=True):
    c, t = torch.from_numpy(coords).cuda(), torch.from_numpy(target).cuda()
    loss = tr.fwd_bwd(c, t, N).item()
    x0 = tr.enc_out(N).float().cpu().numpy().astype(np.float64)
    torch.cuda.synchronize()
    l0 = fh.kernel_launches()
    y = tr.infer(c).cpu().numpy().astype(np.float64)
    if one_launch:
        assert fh.kernel_launches() - l0 == 1      # NEXT-1 fused: encode + MLP in one launch
    assert tr.status() == fh.FH_OK
    master = tr.mlp_master.cpu().numpy().astype(np.float64)
    K0, o, layers = cfg.L * cfg.F, 0, []
    for fi, fo in ((K0, 64), (64, 64), (64, 1)):
        Wt = master[o:o + fi * fo].reshape(fo, fi); o += fi * fo
        layers.append((Wt, master[o:o + fo])); o += fo
    yr, _ = T.mlp_forward(x0, layers)
    assert np.max(np.abs(y - yr)) <= 1e-3 * max(1.0, np.max(np.abs(yr)))
    assert abs(np.mean((y - target) ** 2) - loss) <= 1e-4 * loss


def test_zero_lr_leaves_parameters():
    cfg = small_cfg(2, 8)
    g = W.rng(0)
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    tr = fh.Trainer(enc, W.draw_table(g, enc.entries, 2), W.draw_mlp(g, W.MLPConfig((16, 64, 64, 1))), 512, lr=0.0)
    p0 = tr.mlp_master.clone(), tr.table_master.clone()
    c = torch.rand(512, 4, device="cuda")
    tr.step(c, torch.rand(512, device="cuda"))
    torch.cuda.synchronize()
    assert torch.equal(p0[0], tr.mlp_master) and torch.equal(p0[1], tr.table_master)


def test_training_reduces_loss_on_moving_gaussians():
    """End-to-end sanity (not parity): the cfg3 field recipe at 32^3 x 8,
    training on random voxels reduces the MSE by > 10x in 200 steps."""
    field = torch.from_numpy(W.gaussian_blobs_field(W.rng(0), S=32, T=8)).cuda()
    levels = tuple((s, s, s, t) for s, t in zip(W.geometric(4, 32, 8), W.geometric(2, 8, 8)))
    enc = fh.Encoder(levels, 4, "f16", 1 << 14)
    g = W.rng(1)
    tr = fh.Trainer(enc, W.draw_table(g, enc.entries, 4), W.draw_mlp(g, W.MLPConfig((32, 64, 64, 1))), 1 << 14)
    gen = torch.Generator("cuda").manual_seed(0)
    losses = []
    for it in range(200):
        idx = torch.randint(0, field.numel(), (1 << 14,), device="cuda", generator=gen)
        x = idx % 32; y = (idx // 32) % 32; z = (idx // 1024) % 32; t = idx // 32768
        coords = torch.stack([x / 31.0, y / 31.0, z / 31.0, t / 7.0], 1).float().contiguous()
        target = field.view(-1)[idx].contiguous()
        losses.append(tr.step(coords, target).item())
    assert tr.status() == fh.FH_OK
    assert np.mean(losses[-10:]) < 0.1 * np.mean(losses[:5]), (losses[:5], losses[-10:])


def test_divergence_flag():
    cfg = small_cfg(2, 8)
    enc, tr, coords, target = make(cfg, 300, seed=9)
    target[5] = np.inf
    tr.fwd_bwd(torch.from_numpy(coords).cuda(), torch.from_numpy(target).cuda())
    assert tr.status() == fh.FH_E_DIVERGED
    assert tr.status() == fh.FH_OK


def test_bwd_launch_ranges_events_and_apply_ranges():
    """The backward launches' ranges partition the table; the caller's
    events are recorded by fh_train_fwd_bwd; fh_train_apply_ranges over
    ranges covering the table (aligned chunks + unaligned tails, in any
    order) is bit-identical to fh_train_apply."""
    from paper_2507_03836_b200 import dp
    cfg = small_cfg(2, 16, cap=1 << 10)
    trs = [make(cfg, 1500, seed=31) for _ in range(2)]
    (_, ta, coords, target), (_, tb, _, _) = trs
    launches = ta.bwd_launch_ranges()
    cover = np.zeros(ta.n_table, np.int64)
    for rngs in launches:
        for b, e in rngs:
            cover[b:e] += 1
    assert np.all(cover == 1) and len(launches) >= 1
    evs = [torch.cuda.Event() for _ in launches]
    for ev in evs:
        ev.record()
    ta.set_bwd_events(evs)
    c, t = torch.from_numpy(coords).cuda(), torch.from_numpy(target).cuda()
    mains, tails = dp.overlap_plan(launches, 3, 0)
    for step in range(3):
        ta.fwd_bwd(c, t)
        tb.grads.copy_(ta.grads)      # same gradients (atomics make two runs differ in fp32 order)
        torch.cuda.synchronize()
        assert all(ev.query() for ev in evs)
        ranges = [(a, a + m) for (_, a, m) in mains][::-1] + tails   # any order
        ta.apply_ranges(ranges, [ta.grads[b:e] for b, e in ranges])
        tb.apply()
        torch.cuda.synchronize()
        assert torch.equal(ta.table_master, tb.table_master)
        assert torch.equal(ta.table_shadow, tb.table_shadow)
        assert torch.equal(ta.mlp_master, tb.mlp_master)
    assert ta.step_count == tb.step_count == 3
    ta.set_bwd_events([])


def test_overlapped_dp_single_rank_equals_plain_step():
    """OverlappedShardedDP without a process group (one rank) takes exactly
    the plain train step."""
    from paper_2507_03836_b200 import dp
    cfg = small_cfg(4, 16, cap=1 << 11)
    (_, ta, coords, target), (_, tb, _, _) = [make(cfg, 2000, seed=41) for _ in range(2)]
    odp = dp.OverlappedShardedDP(ta)
    c, t = torch.from_numpy(coords).cuda(), torch.from_numpy(target).cuda()
    for _ in range(3):
        ta.fwd_bwd(c, t, 2000)
        tb.grads.copy_(ta.grads)      # same gradients (atomics make two runs differ in fp32 order)
        odp.reduce_and_apply()
        tb.apply()
        torch.cuda.synchronize()
        assert torch.equal(ta.table_master, tb.table_master)
        assert torch.equal(ta.table_shadow, tb.table_shadow)
        assert torch.equal(ta.mlp_master, tb.mlp_master)
    loss = odp.step(c, t, 2000)        # the composed step runs too
    assert ta.status() == fh.FH_OK and torch.isfinite(loss).all()


def test_fwd_bwd_zero_samples_records_events_after_zeroing():
    """A rank with no samples (N_local = 0, n_global > 0): fh_train_fwd_bwd
    zeroes the gradients and records the caller's per-launch events AFTER
    the zeroing, so a communication stream that waits on them reads zeros
    (not the previous step's gradients)."""
    cfg = small_cfg(2, 16, cap=1 << 10)
    enc, tr, coords, target = make(cfg, 500, seed=37)
    launches = tr.bwd_launch_ranges()
    evs = [torch.cuda.Event() for _ in launches]
    for ev in evs:
        ev.record()
    tr.set_bwd_events(evs)
    tr.fwd_bwd(torch.from_numpy(coords).cuda(), torch.from_numpy(target).cuda())
    torch.cuda.synchronize()
    tr.grads[:tr.n_table].fill_(float("nan"))            # stale: must be overwritten before the events
    torch.cuda.synchronize()
    main = torch.cuda.Stream()
    comm = torch.cuda.Stream()
    empty = torch.empty((0, 4), device="cuda")
    with torch.cuda.stream(main):
        torch.cuda._sleep(2_000_000)                      # keep the zeroing late on its stream
        tr.fwd_bwd(empty, torch.empty((0,), device="cuda"), 1000, stream=main)
    seen = []
    with torch.cuda.stream(comm):
        for ev in evs:
            comm.wait_event(ev)
        seen.append(tr.grads[:tr.n_table].clone())
    torch.cuda.synchronize()
    assert torch.all(seen[0] == 0)
    assert torch.all(tr.table_grad == 0)
    tr.set_bwd_events([])


def test_apply_peers_sums_ranks_and_broadcasts():
    """fh_train_apply_peers with W = 3 'ranks' simulated by local buffers:
    the update uses the rank-ordered SUM of the three gradient buffers
    (bit-identical to Adam on the summed gradient), broadcast ranges land in
    all three shadow buffers, replicated ranges only in the local one, and
    the MLP uses the summed MLP gradients."""
    cfg = small_cfg(2, 16, cap=1 << 10)
    (_, ta, coords, target), (_, tb, _, _) = [make(cfg, 1500, seed=51) for _ in range(2)]
    c, t = torch.from_numpy(coords).cuda(), torch.from_numpy(target).cuda()
    ta.fwd_bwd(c, t)
    g = torch.Generator("cuda").manual_seed(5)
    peers = [ta.grads] + [torch.randn(ta.grads.shape, device="cuda", generator=g) * 0.01 for _ in range(2)]
    shadows = [ta.shadow_flat] + [torch.zeros_like(ta.shadow_flat) for _ in range(2)]
    total = (peers[0] + peers[1]) + peers[2]
    nt = ta.n_table
    half = (nt // 2) // 4 * 4
    bcast_rng, local_rng = [(0, half)], [(half, nt)]
    ta.apply_peers([p.data_ptr() for p in peers], [s.data_ptr() for s in shadows],
                   [p[ta.nt_pad:].data_ptr() for p in peers], bcast_rng + local_rng, [1, 0], True, True)
    tb.grads.copy_(total)
    tb.apply()
    torch.cuda.synchronize()
    assert torch.equal(ta.table_master, tb.table_master)
    assert torch.equal(ta.mlp_master, tb.mlp_master)
    assert torch.equal(ta.table_shadow, tb.table_shadow)
    for s in shadows[1:]:
        assert torch.equal(s[:half], ta.shadow_flat[:half])
        assert torch.all(s[half:nt] == 0)
    assert ta.step_count == 1


def test_apply_multicast_nvls_single_gpu():
    """fh_train_apply_multicast (multimem.ld_reduce +
    Adam + multimem.st) on a real NVLS multicast object spanning this one
    GPU (tests/mc_alloc.py: cuMemCreate memory bound to a one-device
    multicast object): the reduction over one rank is the buffer itself, so
    the update must equal plain Adam bit for bit; broadcast ranges reach the
    shadow through the multicast address (f16x2 multimem.st), replicated
    ranges through the local one; vector and pair (unaligned) paths."""
    import mc_alloc
    ok, why = mc_alloc.multicast_supported()
    if not ok:
        pytest.skip(why)
    cfg = small_cfg(2, 16, cap=1 << 10)
    mca = mc_alloc.McAllocator()
    g = W.rng(61)
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    table = W.draw_table(g, enc.entries, cfg.F, "f32")
    layers = W.draw_mlp(g, W.MLPConfig((32, 64, 64, 1)))
    ta = fh.Trainer(enc, table, layers, 1500, alloc=mca)
    tb = fh.Trainer(enc, table, layers, 1500)
    coords = torch.from_numpy(W.draw_coords(g, 1500)).cuda()
    target = torch.from_numpy(g.random(1500, dtype=np.float32)).cuda()
    for step in range(2):
        ta.fwd_bwd(coords, target)
        tb.grads.copy_(ta.grads)
        nt = ta.n_table
        half = (nt // 2) // 4 * 4
        odd = half + 6            # a broadcast range off the 4-element grid: pair path
        rngs = [(0, half), (half, odd), (odd, nt)]
        ta.apply_multicast(mca.mc(ta.grads), mca.mc(ta.shadow_flat), mca.mc(ta.grads) + ta.nt_pad * 4,
                           rngs, [1, 1, 0], True, True)
        tb.apply()
        torch.cuda.synchronize()
        assert torch.equal(ta.table_master, tb.table_master)
        assert torch.equal(ta.mlp_master, tb.mlp_master)
        assert torch.equal(ta.table_shadow, tb.table_shadow)
    assert ta.step_count == 2
    # broadcast ranges must be whole fp16 pairs
    with pytest.raises(fh.FHashError):
        ta.apply_multicast(mca.mc(ta.grads), mca.mc(ta.shadow_flat), mca.mc(ta.grads) + ta.nt_pad * 4,
                           [(1, 5)], [1], False, True)


def test_apply_multicast_argument_checks():
    """fh_train_apply_multicast's host-side checks (run without a multicast
    object: every call here fails before any launch)."""
    cfg = small_cfg(2, 16, cap=1 << 10)
    enc, tr, _, _ = make(cfg, 300, seed=63)
    g = tr.grads.data_ptr()
    sh = tr.shadow_flat.data_ptr()
    nt = tr.n_table
    bad = [
        (0, sh, g, [(0, 4)], [1], False),                 # NULL grad address
        (g, 0, g, [(0, 4)], [1], False),                  # NULL shadow address
        (g + 4, sh, g, [(0, 4)], [1], False),             # grad not 16-byte aligned
        (g, sh + 2, g, [(0, 4)], [1], False),             # shadow not 8-byte aligned
        (g, sh, g, [(1, 5)], [1], False),                 # broadcast range not in fp16 pairs
        (g, sh, g, [(0, nt + 2)], [1], False),            # range outside the table
        (g, sh, 0, [(0, 4)], [1], True),                  # with_mlp and a NULL MLP address
    ]
    for (mg, ms, mm, rngs, bc, with_mlp) in bad:
        with pytest.raises(fh.FHashError):
            tr.apply_multicast(mg, ms, mm, rngs, bc, with_mlp, True)
    assert tr.step_count == 0
    # an fp32-table trainer has no fp16 shadow to broadcast
    cfg32 = small_cfg(2, 16, tdt="f32", cap=1 << 10)
    _, tr32, _, _ = make(cfg32, 300, seed=64)
    with pytest.raises(fh.FHashError):
        tr32.apply_multicast(tr32.grads.data_ptr(), tr32.grads.data_ptr(), tr32.grads.data_ptr(), [(0, 4)], [1],
                             False, True)


def test_multicast_sharded_dp_single_rank():
    """dp.MulticastShardedDP (per backward launch: this rank's chunk through
    fh_train_apply_multicast, tails + MLP at the end) on a 1-rank NCCL group
    with a one-device multicast object: equal to the plain step, bit for bit."""
    import mc_alloc
    import torch.distributed as dist
    from paper_2507_03836_b200 import dp
    ok, why = mc_alloc.multicast_supported()
    if not ok:
        pytest.skip(why)
    import os
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29581")
    created = not dist.is_initialized()
    if created:
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        cfg = small_cfg(2, 16, cap=1 << 10)
        mca = mc_alloc.McAllocator()
        g = W.rng(62)
        enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
        table = W.draw_table(g, enc.entries, cfg.F, "f32")
        layers = W.draw_mlp(g, W.MLPConfig((32, 64, 64, 1)))
        ta = fh.Trainer(enc, table, layers, 3000, alloc=mca)
        tb = fh.Trainer(enc, table, layers, 3000)
        sdp = dp.MulticastShardedDP(ta, mc=(mca.mc(ta.grads), mca.mc(ta.shadow_flat)), barrier=lambda: None)
        for k in range(3):
            coords = torch.from_numpy(W.draw_coords(W.rng(100 + k), 3000)).cuda()
            target = torch.from_numpy(W.rng(200 + k).random(3000, dtype=np.float32)).cuda()
            sdp.step(coords, target, 3000)
            tb.fwd_bwd(coords, target)
            tb.apply()
        torch.cuda.synchronize()
        assert torch.equal(ta.table_master, tb.table_master)
        assert torch.equal(ta.mlp_master, tb.mlp_master)
        assert torch.equal(ta.table_shadow, tb.table_shadow)
    finally:
        if created:
            dist.destroy_process_group()


def test_peer_sharded_dp_single_rank():
    """dp.PeerShardedDP on a 1-rank NCCL group with torch symmetric memory:
    the fused kernel path equals the plain step (same gradients)."""
    import os
    import torch.distributed as dist
    from paper_2507_03836_b200 import dp
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = "29561"
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        cfg = small_cfg(4, 16, cap=1 << 11)
        g = W.rng(61)
        enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
        table = W.draw_table(g, enc.entries, cfg.F, "f32")
        layers = W.draw_mlp(g, W.MLPConfig((cfg.L * cfg.F, 64, 64, 1)))
        coords = W.draw_coords(g, 2000)
        target = g.random(2000, dtype=np.float32)
        ta = fh.Trainer(enc, table, layers, 2000, alloc=dp.symm_alloc)
        tb = fh.Trainer(enc, table, layers, 2000)
        pdp = dp.PeerShardedDP(ta)
        c, t = torch.from_numpy(coords).cuda(), torch.from_numpy(target).cuda()
        for _ in range(3):
            ta.fwd_bwd(c, t)
            tb.grads.copy_(ta.grads)
            pdp.reduce_and_apply()
            tb.apply()
            torch.cuda.synchronize()
            assert torch.equal(ta.table_master, tb.table_master)
            assert torch.equal(ta.table_shadow, tb.table_shadow)
            assert torch.equal(ta.mlp_master, tb.mlp_master)
        loss = pdp.step(c, t, 2000)
        assert ta.status() == fh.FH_OK and torch.isfinite(loss).all()
    finally:
        dist.destroy_process_group()


def test_overlapped_dp_nccl_single_rank_collective_path():
    """dp.OverlappedShardedDP with its collective path forced on a 1-rank
    NCCL group: reduce-scatters queued on the communication stream behind
    the backward launches' events, the tails + MLP all-reduce, Adam over the
    owned ranges and the shadow all-gathers -- bit-identical to the plain
    step (same gradients; NCCL over one rank is a copy).  Exercises the
    stream / event plumbing the multi-GPU bench uses."""
    import os
    import torch.distributed as dist
    from paper_2507_03836_b200 import dp
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = "29563"
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        cfg = small_cfg(4, 16, cap=1 << 11)
        g = W.rng(62)
        enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
        table = W.draw_table(g, enc.entries, cfg.F, "f32")
        layers = W.draw_mlp(g, W.MLPConfig((cfg.L * cfg.F, 64, 64, 1)))
        coords = W.draw_coords(g, 3000)
        target = g.random(3000, dtype=np.float32)
        ta = fh.Trainer(enc, table, layers, 3000)
        tb = fh.Trainer(enc, table, layers, 3000)
        odp = dp.OverlappedShardedDP(ta, force_collectives=True)
        assert odp.force
        c, t = torch.from_numpy(coords).cuda(), torch.from_numpy(target).cuda()
        for _ in range(3):
            ta.fwd_bwd(c, t)
            tb.grads.copy_(ta.grads)
            odp.reduce_and_apply()
            tb.apply()
            torch.cuda.synchronize()
            assert torch.equal(ta.table_master, tb.table_master)
            assert torch.equal(ta.table_shadow, tb.table_shadow)
            assert torch.equal(ta.mlp_master, tb.mlp_master)
        loss = odp.step(c, t, 3000)
        torch.cuda.synchronize()
        assert ta.status() == fh.FH_OK and torch.isfinite(loss).all()
    finally:
        dist.destroy_process_group()


def test_fwd_bwd_overwrites_gradients():
    """fh_train_fwd_bwd OVERWRITES the grad buffers (include/fhash.h): a
    trainer whose grads hold NaN before the call ends with the same
    gradients as one whose grads were zero (up to the reduction order of the
    atomics), table and MLP parts; N = 0 leaves them all zero."""
    cfg = small_cfg(2, 8, cap=1 << 11)
    _, ta, coords, target = make(cfg, 3000, seed=41)
    _, tb, _, _ = make(cfg, 3000, seed=41)
    c, t = torch.from_numpy(coords).cuda(), torch.from_numpy(target).cuda()
    ta.grads.fill_(float("nan"))
    tb.grads.zero_()
    ta.fwd_bwd(c, t)
    tb.fwd_bwd(c, t)
    torch.cuda.synchronize()
    nt = ta.n_table   # (the padding between the table and MLP parts is never written)
    for ga, gb in ((ta.grads[:nt], tb.grads[:nt]), (ta.mlp_grad, tb.mlp_grad)):
        assert torch.isfinite(ga).all()
        assert torch.allclose(ga, gb, rtol=1e-5, atol=1e-6 * gb.abs().max().item())
    ta.grads.fill_(float("nan"))
    ta.fwd_bwd(c[:0], t[:0], 3000)
    torch.cuda.synchronize()
    assert torch.count_nonzero(ta.grads[:ta.n_table]).item() == 0
    assert torch.count_nonzero(ta.mlp_grad).item() == 0


def test_fused_nccl_dp_step_equals_plain_step():
    """The fused data-parallel form (fh_trainer_set_comm, SURVEY.md §8(b)
    nccl_comm): the library's own NCCL reduce-scatter of every backward
    level group (overlapped through per-group events), the tails + MLP
    all-reduce, ONE Adam over the rank's chunks + tails, and the in-place
    fp16 all-gather.  On a 1-rank communicator it must be exactly Adam on
    the step's gradient: a twin trainer fed the same gradients (copied from
    the DP trainer, whose grad buffers still hold them) and stepped with the
    plain fh_train_apply ends bit-identical after every step (the atomics of
    two independent fwd_bwd runs would differ in the last bits)."""
    cfg = small_cfg(4, 12)
    g = W.rng(70)
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    table = W.draw_table(g, enc.entries, cfg.F, "f32")
    layers = W.draw_mlp(g, W.MLPConfig((cfg.L * cfg.F, 64, 64, 1)))
    N = 3000
    a = fh.Trainer(enc, table, layers, N)
    b = fh.Trainer(enc, table, layers, N)
    comm = fh.NcclComm(fh.nccl_unique_id(), 1, 0)
    b.set_comm(comm)
    for k in range(3):
        c = torch.from_numpy(W.draw_coords(g, N)).cuda()
        t = torch.from_numpy(g.random(N, dtype=np.float32)).cuda()
        b.step(c, t)
        a.grads.copy_(b.grads)
        a.apply()
        torch.cuda.synchronize()
        assert torch.equal(a.table_shadow, b.table_shadow), k
        assert torch.equal(a.table_master, b.table_master), k
        assert torch.equal(a.mlp_master, b.mlp_master) and torch.equal(a.mlp_shadow, b.mlp_shadow), k
    assert b.status() == fh.FH_OK and a.step_count == b.step_count == 3
    b.set_comm(None)
    comm.destroy()


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_fused_dp_plan_matches_overlap_plan(world):
    """The library's gradient partition for the fused DP form is the one
    dp.overlap_plan defines (tested on CPU with gloo at world 2): its
    workspace = this rank's shards (sum m / W) + tails + MLP, 256-aligned."""
    from paper_2507_03836_b200 import dp
    cfg = W.CFG3
    g = W.rng(71)
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    tr = fh.Trainer(enc, W.draw_table(g, enc.entries, cfg.F, "f32"), W.draw_mlp(g, W.MLP3), 1024)
    mains, tails = dp.overlap_plan(tr.bwd_launch_ranges(), world, 0)
    shard = sum(m // world for (_, _, m) in mains)
    tail = sum(e - b for b, e in tails) + tr.n_mlp
    up = lambda v: (v + 255) // 256 * 256
    assert int(fh._train_lib().fh_trainer_dp_workspace_size(tr._h, world)) == up(4 * shard) + up(4 * tail)
