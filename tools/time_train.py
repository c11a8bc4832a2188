"""Train-step timing helper for optimisation / ncu (not the bench).

    python tools/time_train.py [cfg3|cfg4] [iters] [batch_log2]

Builds the synthetic field, a trainer, and times sample + fwd_bwd + apply
per step with CUDA events (L2 not flushed: consecutive steps).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2507_03836_b200 import fhash as fh  # noqa: E402


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    if which == "cfg3":
        field = fh.field_gaussian_blobs(256, 32, W.gaussian_blob_params(W.rng(0)))
        cfg, mlp, N = W.CFG3, W.MLP3, W.N_CFG3
    else:
        field = fh.field_value_noise(640, 256, 256, 100, seed=0)
        cfg, mlp, N = W.CFG4, W.MLP4, W.N_CFG4
    if len(sys.argv) > 3:
        N = 1 << int(sys.argv[3])
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    gen = torch.Generator("cuda").manual_seed(0)
    table0 = (torch.rand((enc.entries, cfg.F), device="cuda", generator=gen) * 2 - 1) * 1e-4
    tr = fh.Trainer(enc, table0, W.draw_mlp(W.rng(0), mlp), N)
    coords = torch.empty((N, 4), device="cuda")
    target = torch.empty((N,), device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    acc = [0.0, 0.0, 0.0]
    for k in range(iters + 3):
        ev[0].record()
        fh.sample_voxels(field, N, 1234, 0, k, coords, target)
        ev[1].record()
        tr.fwd_bwd(coords, target, N)
        ev[2].record()
        tr.apply()
        ev[3].record()
        torch.cuda.synchronize()
        if k >= 3:
            for i in range(3):
                acc[i] += ev[i].elapsed_time(ev[i + 1])
    s, fb, ad = (a / iters for a in acc)
    print(f"{which} N={N}: sample {s:.3f} ms  fwd_bwd {fb:.3f} ms  adam {ad:.3f} ms  "
          f"-> {N / ((s + fb + ad) / 1e3) / 1e6:.1f} M samples/s  loss {tr.loss.item():.5f}")


if __name__ == "__main__":
    main()
