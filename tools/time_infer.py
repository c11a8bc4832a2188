"""fh_infer (NEXT-1 fused encode + MLP) latency / throughput -- experiments,
not the bench.

    python tools/time_infer.py [cfg3|cfg5] [reps]

Prints, per batch size, the eager and CUDA-graph-replayed time of one call.
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
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    cfg, mlp = (W.CFG3, W.MLP3) if which == "cfg3" else (W.CFG4, W.MLP4)
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    g = torch.Generator("cuda").manual_seed(0)
    table0 = (torch.rand((enc.entries, cfg.F), device="cuda", generator=g) * 2 - 1) * 1e-4
    nmax = 1 << 20
    tr = fh.Trainer(enc, table0, W.draw_mlp(W.rng(0), mlp), nmax)
    coords = torch.rand((nmax, 4), device="cuda", generator=g)
    y = torch.empty(nmax, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for nb in (1 << 7, 1 << 10, 1 << 12, 1 << 16, 1 << 20):
        cs, ys = coords[:nb], y[:nb]
        r = reps if nb <= 1 << 16 else 20
        for _ in range(3):
            tr.infer(cs, ys)
        e0.record()
        for _ in range(r):
            tr.infer(cs, ys)
        e1.record()
        torch.cuda.synchronize()
        eager = e0.elapsed_time(e1) / r * 1e3
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            tr.infer(cs, ys, stream=s)
            with torch.cuda.graph(graph, stream=s):
                tr.infer(cs, ys, stream=s)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(r):
            graph.replay()
        e1.record()
        torch.cuda.synchronize()
        gus = e0.elapsed_time(e1) / r * 1e3
        print(f"{which} N={nb}: eager {eager:.2f} us  graph {gus:.2f} us  ({nb / (gus * 1e-6) / 1e9:.3f} G samples/s)")


if __name__ == "__main__":
    main()
