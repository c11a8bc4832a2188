"""Pins for Oracle-T (oracle/train.py): MLP, MSE, Adam.  CPU only."""
import numpy as np
import torch

from oracle import train as T
import workloads as W


def _tiny(seed=0, widths=(6, 5, 4, 1)):
    g = np.random.default_rng(seed)
    layers = [(g.standard_normal((o, i)), g.standard_normal(o)) for i, o in zip(widths[:-1], widths[1:])]
    x = g.standard_normal((7, widths[0]))
    t = g.standard_normal(7)
    return layers, x, t


def _loss(layers, x, t, n_global):
    y, _ = T.mlp_forward(x, layers, emulate_bf16=False)
    return T.mse_loss(y, t, n_global)[0]


def test_mlp_finite_differences():
    """S:420 / S:460: analytic grads of every parameter and of the input
    match central differences (fp64, no bf16 emulation) within 1e-5 rel."""
    layers, x, t = _tiny()
    n_global = 11
    y, cache = T.mlp_forward(x, layers, emulate_bf16=False)
    _, dy = T.mse_loss(y, t, n_global)
    grads, dx = T.mlp_backward(dy, layers, cache, emulate_bf16=False)
    h = 1e-6
    for k, (Wk, bk) in enumerate(layers):
        for arr, gk in ((Wk, grads[k][0]), (bk, grads[k][1])):
            for j in range(arr.size):
                old = arr.flat[j]
                arr.flat[j] = old + h; lp = _loss(layers, x, t, n_global)
                arr.flat[j] = old - h; lm = _loss(layers, x, t, n_global)
                arr.flat[j] = old
                fd = (lp - lm) / (2 * h)
                assert abs(fd - gk.flat[j]) <= 1e-5 * max(1e-2, abs(fd))
    for j in range(x.size):
        old = x.flat[j]
        x.flat[j] = old + h; lp = _loss(layers, x, t, n_global)
        x.flat[j] = old - h; lm = _loss(layers, x, t, n_global)
        x.flat[j] = old
        assert abs((lp - lm) / (2 * h) - dx.flat[j]) <= 1e-5 * max(1e-2, abs(dx.flat[j]))


def test_targets_equal_forward_zero_loss_and_grads():
    """targets = forward(model) -> loss 0 and all gradients 0."""
    layers, x, _ = _tiny(1)
    y, cache = T.mlp_forward(x, layers)
    loss, dy = T.mse_loss(y, y, 7)
    grads, dx = T.mlp_backward(dy, layers, cache)
    assert loss == 0.0 and not np.any(dx)
    assert all(not np.any(a) and not np.any(b) for a, b in grads)


def test_zero_weights_bias_only():
    """zero weights -> the output is the last bias."""
    layers, x, _ = _tiny(2)
    z = [(np.zeros_like(Wk), np.zeros_like(bk)) for Wk, bk in layers]
    z[-1] = (z[-1][0], np.array([0.625]))
    y, _ = T.mlp_forward(x, z)
    assert np.all(y == 0.625)


def test_bf16_round_matches_library_and_ties_to_even():
    """bf16 RNE: 1+2^-8 -> 1 (tie, even), 1+3*2^-8 -> 1+2^-6 (tie, even);
    and equal to torch's float32 -> bfloat16 conversion on random values."""
    assert T.bf16_round(np.array([1 + 2 ** -8]))[0] == 1.0
    assert T.bf16_round(np.array([1 + 3 * 2 ** -8]))[0] == 1 + 2 ** -6
    x = np.random.default_rng(0).standard_normal(10000).astype(np.float32) * 7
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(T.bf16_round(x), ref)


def test_adam_first_step_closed_form_and_lr0():
    """Adam step 1: m_hat = g, v_hat = g^2 -> delta = -lr g / (|g| + eps);
    lr = 0 leaves parameters unchanged."""
    g = np.random.default_rng(4).standard_normal(1000)
    p0 = np.random.default_rng(5).standard_normal(1000)
    p, m, v = T.adam_step(p0, g, np.zeros(1000), np.zeros(1000), 1, lr=0.01)
    assert np.allclose(p - p0, -0.01 * g / (np.abs(g) + 1e-8), rtol=1e-12, atol=0)
    p2, _, _ = T.adam_step(p0, g, m, v, 2, lr=0.0)
    assert np.array_equal(p2, p0)


def test_adam_constant_gradient_fixed_step():
    """With a constant gradient g the bias-corrected moments stay g and g^2,
    so every step moves by -lr * g / (|g| + eps)."""
    g = np.array([0.3, -2.0, 1e-3])
    p = np.zeros(3); m = np.zeros(3); v = np.zeros(3)
    for s in range(1, 6):
        p_old = p
        p, m, v = T.adam_step(p, g, m, v, s, lr=0.01)
        assert np.allclose(p - p_old, -0.01 * g / (np.abs(g) + 1e-8), rtol=1e-10)


def test_mlp_init_shapes():
    layers = W.draw_mlp(W.rng(0), W.MLP3)
    assert [l[0].shape for l in layers] == [(64, 32), (64, 64), (1, 64)]
    assert sum(l[0].size + l[1].size for l in layers) == 6337


def _mlp_case(seed, N=512, widths=(32, 64, 64, 1)):
    g = np.random.default_rng(seed)
    layers = W.draw_mlp(g, W.MLPConfig(widths))
    x = g.uniform(-1e-2, 1e-2, (N, widths[0]))           # encoder outputs are small
    t = g.random(N)
    return layers, x, t


def test_bf16_oracle_within_bf16_distance_of_fp64():
    """The bf16-emulating Oracle-T (R13 rounding points) against the
    unrounded fp64 MLP -- whose formulas the finite-difference pin fixes:
    every gradient element within 2^-5 (about four bf16 roundings of 2^-8
    in a chain) of its sum of |contributions| plus the ReLU-ambiguity term,
    and the loss within 1e-2 relative.  So the emulation is a precision
    reading, not a different computation."""
    for seed in range(4):
        layers, x, t = _mlp_case(seed)
        y64, c64 = T.mlp_forward(x, layers, emulate_bf16=False)
        yb, cb = T.mlp_forward(x, layers, emulate_bf16=True)
        l64, dy64 = T.mse_loss(y64, t, 1000)
        lb, dyb = T.mse_loss(yb, t, 1000)
        assert abs(lb - l64) <= 1e-2 * l64
        g64, dx64 = T.mlp_backward(dy64, layers, c64, emulate_bf16=False)
        gb, dxb = T.mlp_backward(dyb, layers, cb, emulate_bf16=True)
        bounds, A_dx, U_dx = T.mlp_backward_bounds(layers, c64, t, 1000)
        for (dW, db), (dWb, dbb), (AW, Ab, UW, Ub) in zip(g64, gb, bounds):
            assert np.all(np.abs(dWb - dW) <= 2 ** -5 * AW + UW + 1e-300)
            assert np.all(np.abs(dbb - db) <= 2 ** -5 * Ab + Ub + 1e-300)
        assert np.all(np.abs(dxb - dx64) <= 2 ** -5 * A_dx + U_dx + 1e-300)


def test_backward_bounds_are_sums_of_abs_contributions():
    """mlp_backward_bounds on a one-hidden-layer net with no ambiguous units:
    A equals the textbook sums of |contributions| written out by loops."""
    g = np.random.default_rng(9)
    W1, b1 = g.standard_normal((3, 2)), np.abs(g.standard_normal(3)) + 5.0   # z1 > 0 everywhere
    W2, b2 = g.standard_normal((1, 3)), g.standard_normal(1)
    x = g.uniform(0, 0.1, (4, 2))
    layers = [(W1, b1), (W2, b2)]
    t = g.random(4)
    y, cache = T.mlp_forward(x, layers, emulate_bf16=False)
    bounds, A_dx, U_dx = T.mlp_backward_bounds(layers, cache, t, 4)
    # forward abs scales written out: S1[n,i] = sum_j |W1 x| + |b1|, Sy = sum_i |W2 S1| + |b2|
    S1 = [[sum(abs(W1[i, j] * x[n, j]) for j in range(2)) + abs(b1[i]) for i in range(3)] for n in range(4)]
    Sy = [sum(abs(W2[0, i]) * S1[n][i] for i in range(3)) + abs(b2[0]) for n in range(4)]
    Ady = [2.0 * (Sy[n] + abs(t[n])) / 4 for n in range(4)]
    for i in range(3):
        assert np.isclose(bounds[1][0][0, i], sum(Ady[n] * S1[n][i] for n in range(4)))
        for j in range(2):
            want = sum(Ady[n] * abs(W2[0, i]) * abs(x[n, j]) for n in range(4))
            assert np.isclose(bounds[0][0][i, j], want)
    for n in range(4):
        for j in range(2):
            assert np.isclose(A_dx[n, j], sum(Ady[n] * abs(W2[0, i]) * abs(W1[i, j]) for i in range(3)))
    assert not np.any(U_dx) and not np.any(bounds[0][2])
