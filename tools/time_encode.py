"""Kernel timing helper for optimisation experiments (not the bench).

    FHASH_LIB=path/to/lib.so python tools/time_encode.py [cfg2|cfg4|cfg3] [iters]

Prints the average CUDA-event time of encode fwd and bwd on the config's
full batch, L2 flushed before each launch.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2507_03836_b200 import fhash as fh  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    pc = W.EncoderConfig("pc", tuple(fh.fold_schedule((200, 110, 54), 10, 2)), F=2, cap=0, table_dtype="f32")
    cfg = {"cfg2": W.CFG2, "cfg3": W.CFG3, "cfg4": W.CFG4, "pc": pc}[name]
    N = {"cfg2": W.N_CFG2, "cfg3": W.N_CFG3, "cfg4": W.N_CFG4, "pc": 1 << 21}[name]
    enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap, lin=int(os.environ.get("FH_LIN", "0")))
    g = torch.Generator("cuda").manual_seed(0)
    coords = torch.rand((N, 4), device="cuda", generator=g)
    tdt = torch.float32 if cfg.table_dtype == "f32" else torch.float16
    table = ((torch.rand((enc.entries, cfg.F), device="cuda", generator=g) - 0.5) * 2e-4).to(tdt)
    dout = torch.randn((N, cfg.L * cfg.F), device="cuda", generator=g)
    out = torch.empty((N, cfg.L * cfg.F), device="cuda")
    dtab = torch.zeros((enc.entries, cfg.F), device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    tf = tb = 0.0
    overwrite = os.environ.get("FH_OVERWRITE", "0") == "1"   # bwd overwrites dtable (no separate zero_grad)
    lm = os.environ.get("FH_LM", "0") == "1"                 # level-major dout (FH_BWD_DOUT_LEVEL_MAJOR)
    if lm:
        dout = dout.view(N, cfg.L, cfg.F).permute(1, 0, 2).contiguous()
    for it in range(iters + 3):
        flush.fill_(it & 255)
        if not overwrite:
            enc.zero_grad(dtab)
        e[1].record()
        enc.fwd(coords, table, out)
        e[2].record()
        enc.bwd(coords, dout, dtab, overwrite=overwrite, level_major=lm)
        e[3].record()
        torch.cuda.synchronize()
        if it >= 3:
            tf += e[1].elapsed_time(e[2])
            tb += e[2].elapsed_time(e[3])
    tot = (tf + tb) / iters
    print(f"{os.path.basename(fh.LIB_PATH)} {name} lin={enc.lin} lm={int(lm)}: "
          f"fwd {tf / iters:.4f} ms  bwd {tb / iters:.4f} ms  ({N / (tot / 1e3) / 1e6:.1f} M samples/s)")


if __name__ == "__main__":
    main()
