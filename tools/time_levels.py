"""Per-level encode timing (optimisation experiments, not the bench).

    python tools/time_levels.py [cfg2|cfg4] [iters]

For every level l of the config, builds a one-level encoder (same
resolution, cap and table dtype) and times, on the config's full batch with
L2 flushed before each launch: the direct fwd / bwd (natural order) and the
ordered fwd / bwd (fh_spatial_sort order, tiled fwd / warp-aggregated bwd
where the planner picks them).  Prints one line per level.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2507_03836_b200 import fhash as fh  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    cfg = {"cfg2": W.CFG2, "cfg4": W.CFG4}[name]
    N = {"cfg2": W.N_CFG2, "cfg4": W.N_CFG4}[name]
    full = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
    g = torch.Generator("cuda").manual_seed(0)
    coords = torch.rand((N, 4), device="cuda", generator=g)
    tdt = torch.float32 if cfg.table_dtype == "f32" else torch.float16
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    so = fh.SpatialOrder(full, N)
    order = so(coords)  # the full encoder's key (what the real path uses)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timeit(fn):
        tot = 0.0
        for it in range(iters + 2):
            flush.fill_(it & 255)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            if it >= 2:
                tot += e0.elapsed_time(e1)
        return tot / iters * 1e3  # us

    print(f"{name}: N={N}  per level, us: fwd direct / ordered   bwd direct / ordered")
    sums = [0.0] * 4
    for l, res in enumerate(cfg.levels):
        enc = fh.Encoder([res], cfg.F, cfg.table_dtype, cfg.cap)
        table = ((torch.rand((enc.entries, cfg.F), device="cuda", generator=g) - 0.5) * 2e-4).to(tdt)
        out = torch.empty((N, cfg.F), device="cuda")
        dout = torch.randn((N, cfg.F), device="cuda", generator=g)
        dt = torch.zeros((enc.entries, cfg.F), device="cuda")
        t = [timeit(lambda: enc.fwd(coords, table, out)),
             timeit(lambda: enc.fwd_ordered(coords, order, table, out)),
             timeit(lambda: enc.bwd(coords, dout, dt)),
             timeit(lambda: enc.bwd_ordered(coords, order, dout, dt))]
        sums = [a + b for a, b in zip(sums, t)]
        info = enc.level_info(0)
        print(f"  l={l:2d} R={res} T={info['table_size']:>8d} {'hash' if info['hashed'] else 'mphf'}  "
              f"fwd {t[0]:7.1f} / {t[1]:7.1f}   bwd {t[2]:7.1f} / {t[3]:7.1f}")
    print(f"  sum: fwd {sums[0]:.1f} / {sums[1]:.1f}   bwd {sums[2]:.1f} / {sums[3]:.1f}")


if __name__ == "__main__":
    main()
