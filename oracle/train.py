"""Oracle-T: the small-MLP train step around the encoder -- TEST INFRASTRUCTURE.

fp64 numpy, plain matrix products, no blocking or fusion.  Only tests/,
smoke() and bench.py's CPU legs may import it.  Shares no code with the CUDA
path.

Readings:
  R12  Adam, lr 0.01, beta = (0.9, 0.999), eps = 1e-8, bias
       correction; loss = MSE over the GLOBAL batch,
       dL/dy = 2 (y - target) / N_global.  Dense Adam: every parameter, every
       step.
  R13  precision points of the GPU train path, emulated here by rounding to
       bf16 (round-to-nearest-even) exactly where the GPU rounds: the encoder
       output x0, the bf16 shadow of every weight matrix, the hidden
       activations h1, h2 after ReLU, and the back-propagated dz2, dz1 that
       feed the tensor-core GEMMs.  Everything else is fp64 here (fp32 on the
       GPU).
  R15  ReLU hidden layers, identity output, biases present, widths e.g.
       32 -> 64 -> 64 -> 1 (BASELINE.json configs[2]).

Pins (tests/test_oracle_train.py): central finite differences of the fp64
(unrounded) MLP, targets = forward -> zero loss and zero grads, zero
weights -> bias-only output, Adam first-step closed form
-lr * g / (|g| + eps), lr = 0 -> unchanged, and the bf16-emulating
oracle within bf16 distance (the mlp_backward_bounds bar) of the unrounded
fp64 one -- the emulated rounding points are a precision reading (R13), not
a change of the mathematics.

Tolerance companion (mlp_backward_bounds): for every gradient element the
sum of the absolute values of its contributions (like Oracle-B's A), and an
extra term for ReLU units whose pre-activation is within rounding distance
of 0 (their derivative, 0 or 1, is decided by rounding order).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round to the nearest bf16 (ties to even) via fp32, returned as fp64.
    (fp32 -> bf16 is what the GPU's cvt.rn.bf16.f32 does.)"""
    f = np.ascontiguousarray(np.asarray(x, dtype=np.float64).astype(np.float32))
    b = f.view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return b.astype(np.uint32).view(np.float32).astype(np.float64)


def _id(x):
    return np.asarray(x, dtype=np.float64)


def mlp_forward(x0: np.ndarray, layers: Sequence[Tuple[np.ndarray, np.ndarray]], emulate_bf16: bool = True):
    """Forward of the MLP: z_k = W_k a_{k-1} + b_k; a_k = ReLU(z_k) for
    hidden layers, y = z_last.  Rows are samples; W is [out][in].
    Returns (y [N], cache)."""
    r = bf16_round if emulate_bf16 else _id
    a = r(x0)
    acts = [a]
    zs = []
    n_layers = len(layers)
    for k, (W, b) in enumerate(layers):
        Wk = r(W)
        z = a @ Wk.T + _id(b)[None, :]
        zs.append(z)
        if k < n_layers - 1:
            a = r(np.maximum(z, 0.0))
            acts.append(a)
    y = zs[-1][:, 0]
    return y, (acts, zs)


def mse_loss(y: np.ndarray, target: np.ndarray, n_global: int):
    """MSE over the global batch (R12): loss = sum (y - t)^2 / N_global and
    dL/dy = 2 (y - t) / N_global."""
    d = _id(y) - _id(target)
    return float(np.sum(d * d) / n_global), 2.0 * d / n_global


def mlp_backward(dy: np.ndarray, layers, cache, emulate_bf16: bool = True):
    """Analytic backward.  Returns (grads [(dW, db)...], dx0 [N][in]).
    dz_k rounded to bf16 before it is used as a GEMM operand (R13) except
    for the last layer's dy (the GPU keeps it in fp32 and uses CUDA cores
    for the 64 -> 1 layer)."""
    r = bf16_round if emulate_bf16 else _id
    acts, zs = cache
    n_layers = len(layers)
    grads: List[Tuple[np.ndarray, np.ndarray]] = [None] * n_layers  # type: ignore
    dz = _id(dy)[:, None]  # [N][1]
    dx0 = None
    for k in range(n_layers - 1, -1, -1):
        W, _ = layers[k]
        Wk = r(W)
        a_prev = acts[k]
        dz_op = dz if k == n_layers - 1 else r(dz)
        dW = dz_op.T @ a_prev
        db = dz_op.sum(axis=0)   # R13: the bias gradient sums the same (rounded) dz the GEMMs use
        grads[k] = (dW, db)
        da = dz_op @ Wk
        if k > 0:
            dz = da * (zs[k - 1] > 0.0)
        else:
            dx0 = da
    return grads, dx0


def mlp_backward_bounds(layers, cache, target: np.ndarray, n_global: int, tau: float = 2.0 ** -8):
    """Per-element tolerance companions of mse_loss + mlp_backward, by plain
    propagation of absolute values through the same formulas:
      A  -- running sum of |contributions|: forward abs scales
            S_0 = |a_0|, S_k = (S_{k-1} |W_k|^T + |b_k|) masked by the ReLU,
            S_y = S_{last} |W|^T + |b|; dL/dy's companion 2 (S_y + |t|) / N;
            backward A_dz -> A_dW = A_dz^T S_{k-1}, A_db = sum A_dz,
            A_da = A_dz |W_k|, masked by ReLU'.  A rounding error relative to
            each summed term (bf16 operands, fp32 order) stays within c * A.
      U  -- ambiguity of the ReLU derivative: a unit with
            |z| <= tau * S (pre-activation within tau of its own abs scale;
            tau = one bf16 ulp covers an operand flip upstream) may take
            either derivative, so its dz is known only to within A_da; that
            uncertainty propagates like A.
    Returns ([(A_dW, A_db, U_dW, U_db) per layer], A_dx0, U_dx0); a GPU value
    passes where |got - ref| <= c * A + U."""
    acts, zs = cache
    n_layers = len(layers)
    S = [np.abs(acts[0])]
    live = []
    for k in range(n_layers):
        W, b = layers[k]
        sc = S[-1] @ np.abs(_id(W)).T + np.abs(_id(b))[None, :]
        if k < n_layers - 1:
            z = zs[k]
            amb = np.abs(z) <= tau * sc
            lv = (z > 0.0) | amb
            live.append((lv, amb))
            S.append(sc * lv)
        else:
            S_y = sc[:, 0]
    A_dz = (2.0 * (S_y + np.abs(_id(target))) / n_global)[:, None]
    U_dz = np.zeros_like(A_dz)
    out = [None] * n_layers
    A_dx0 = U_dx0 = None
    for k in range(n_layers - 1, -1, -1):
        aW = np.abs(_id(layers[k][0]))
        out[k] = (A_dz.T @ S[k], A_dz.sum(axis=0), U_dz.T @ S[k], U_dz.sum(axis=0))
        A_da = A_dz @ aW
        U_da = U_dz @ aW
        if k > 0:
            lv, amb = live[k - 1]
            A_dz = A_da * lv
            # the derivative of an ambiguous unit is 0 or 1: its dz is unknown up to A_da
            U_dz = U_da * lv + amb * A_da
        else:
            A_dx0, U_dx0 = A_da, U_da
    return out, A_dx0, U_dx0


def adam_step(p: np.ndarray, g: np.ndarray, m: np.ndarray, v: np.ndarray, step: int,
              lr: float = 0.01, b1: float = 0.9, b2: float = 0.999, eps: float = 1e-8):
    """Bias-corrected Adam (Kingma & Ba; P:489 lr; S:384 betas/eps), fp64.
    step counts from 1.  Returns new (p, m, v)."""
    p, g, m, v = _id(p), _id(g), _id(m), _id(v)
    m = b1 * m + (1.0 - b1) * g
    v = b2 * v + (1.0 - b2) * g * g
    mhat = m / (1.0 - b1 ** step)
    vhat = v / (1.0 - b2 ** step)
    p = p - lr * mhat / (np.sqrt(vhat) + eps)
    return p, m, v
