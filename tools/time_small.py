"""Backward timing of the few-cell levels alone (the coarse end of the
Combustion fold-2 schedule) -- bwd_small_kernel experiments, not the bench.

    python tools/time_small.py [iters]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2507_03836_b200 import fhash as fh  # noqa: E402


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 10
    full = fh.fold_schedule((200, 110, 54), 10, 2)
    sets = [("l4-7", full[4:]), ("l4", full[4:5]), ("l5", full[5:6]), ("l6-7", full[6:])]
    if "--all" in sys.argv:
        sets += [("l1-3", full[1:4]), ("l1", full[1:2]), ("l2", full[2:3]), ("l3", full[3:4]), ("l0", full[0:1])]
    for name, lv in sets:
        enc = fh.Encoder(lv, 2)
        N = 1 << 21
        g = torch.Generator("cuda").manual_seed(0)
        c = torch.rand((N, 4), device="cuda", generator=g)
        dout = torch.randn((N, enc.L * 2), device="cuda", generator=g)
        dt = torch.zeros((enc.entries, 2), device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(3):
            enc.bwd(c, dout, dt, overwrite=True)
        e0.record()
        for _ in range(iters):
            enc.bwd(c, dout, dt, overwrite=True)
        e1.record()
        torch.cuda.synchronize()
        print(f"{name} {[tuple(x) for x in lv]} bwd {e0.elapsed_time(e1) / iters * 1e3:.1f} us")


if __name__ == "__main__":
    main()
