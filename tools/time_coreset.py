"""Coreset timing helper (NEXT-4 optimisation experiments, not the bench).

    python tools/time_coreset.py [iters]

fh_coreset_build + fh_coreset_emit on 8 key frames of the cfg3 field (256^3
Gaussian blobs), segmentation >= 0.5, L2 flushed between iterations."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2507_03836_b200 import fhash as fh  # noqa: E402


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    field = fh.field_gaussian_blobs(256, 32, W.gaussian_blob_params(W.rng(0)))
    keys = field[::4].contiguous()
    del field
    cs = fh.Coreset(keys, fh.FH_FEAT_SEGMENTATION, 0.5)
    M = cs.count
    coords = torch.empty((M, 4), device="cuda")
    vals = torch.empty((M,), device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tb = te = 0.0
    for it in range(iters + 2):
        flush.fill_(it & 255)
        e[0].record()
        c2 = fh.Coreset(keys, fh.FH_FEAT_SEGMENTATION, 0.5)
        e[1].record()
        torch.cuda._sleep(0)
        fh._check(fh._coreset_lib().fh_coreset_emit(fh._ptr(keys), c2.dims, c2.n, fh._ptr(c2.workspace),
                                                    c2.workspace.numel(), fh._ptr(coords), fh._ptr(vals), M,
                                                    fh._stream(None)))
        e[2].record()
        torch.cuda.synchronize()
        if it >= 2:
            tb += e[0].elapsed_time(e[1])
            te += e[1].elapsed_time(e[2])
    n, V = keys.shape[0], keys[0].numel()
    print(f"coreset: {n} x {V} vertices, M = {M}: build {tb / iters:.3f} ms  emit {te / iters:.3f} ms  "
          f"({n * V / ((tb + te) / iters / 1e3) / 1e9:.2f} G vertices/s)")


if __name__ == "__main__":
    main()
