"""fh_infer latency at renderer-sized batches: eager vs CUDA graph (probe)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2507_03836_b200 import fhash as fh  # noqa: E402

cfg, mlp = W.CFG3, W.MLP3
enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
table0 = (torch.rand((enc.entries, cfg.F), device="cuda") * 2 - 1) * 1e-4
tr = fh.Trainer(enc, table0, W.draw_mlp(W.rng(0), mlp), 1 << 16)
for n in (1 << 10, 1 << 12, 1 << 14, 1 << 16):
    coords = torch.rand((n, 4), device="cuda")
    y = torch.empty(n, device="cuda")
    for _ in range(5):
        tr.infer(coords, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 200
    e0.record()
    for _ in range(reps):
        tr.infer(coords, y)
    e1.record()
    torch.cuda.synchronize()
    eager = e0.elapsed_time(e1) / reps
    t0 = time.perf_counter()
    for _ in range(reps):
        tr.infer(coords, y)
    torch.cuda.synchronize()
    host = (time.perf_counter() - t0) / reps * 1e3
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        tr.infer(coords, y, stream=s)
        with torch.cuda.graph(g, stream=s):
            tr.infer(coords, y, stream=s)
    torch.cuda.synchronize()
    ref = y.clone()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(ref, y)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    graph = e0.elapsed_time(e1) / reps
    print(f"N={n}: eager {eager * 1e3:.1f} us/call (host loop {host * 1e3:.1f} us), graph {graph * 1e3:.1f} us/call")
