"""Probe: encode fwd and bwd on two streams concurrently vs back to back
(cfg2 / cfg4 shapes, independent inputs).  Experiment only."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2507_03836_b200 import fhash as fh  # noqa: E402


def run(name, iters=10):
    cfg = {"cfg2": W.CFG2, "cfg4": W.CFG4}[name]
    N = {"cfg2": W.N_CFG2, "cfg4": W.N_CFG4}[name]
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    g = torch.Generator("cuda").manual_seed(0)
    tdt = torch.float32 if cfg.table_dtype == "f32" else torch.float16
    table = ((torch.rand((enc.entries, cfg.F), device="cuda", generator=g) - 0.5) * 2e-4).to(tdt)
    c1 = torch.rand((N, 4), device="cuda", generator=g)
    c2 = torch.rand((N, 4), device="cuda", generator=g)
    out = torch.empty((N, cfg.L * cfg.F), device="cuda", dtype=torch.float32 if name == "cfg2" else torch.bfloat16)
    dout = torch.randn((N, cfg.L * cfg.F), device="cuda", generator=g)
    dt = torch.zeros((enc.entries, cfg.F), device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    od = "f32" if name == "cfg2" else "bf16"
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    res = {}
    for mode in ("serial", "concurrent"):
        tot = 0.0
        for it in range(iters + 2):
            flush.fill_(it & 255)
            torch.cuda.synchronize()
            e0.record()
            if mode == "serial":
                enc.fwd(c1, table, out, out_dtype=od)
                enc.bwd(c2, dout, dt)
            else:
                ev = torch.cuda.Event()
                ev.record()
                s1.wait_event(ev)
                s2.wait_event(ev)
                enc.fwd(c1, table, out, out_dtype=od, stream=s1)
                enc.bwd(c2, dout, dt, stream=s2)
                a, b = torch.cuda.Event(), torch.cuda.Event()
                a.record(s1)
                b.record(s2)
                torch.cuda.current_stream().wait_event(a)
                torch.cuda.current_stream().wait_event(b)
            e1.record()
            torch.cuda.synchronize()
            if it >= 2:
                tot += e0.elapsed_time(e1)
        res[mode] = tot / iters
        print(f"{name} {mode}: {tot / iters:.3f} ms")


for n in sys.argv[1:] or ["cfg2", "cfg4"]:
    run(n)
