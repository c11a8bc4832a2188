"""A few fh_infer calls at one batch size (for ncu launch timing) -- experiments."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import workloads as W  # noqa: E402
from paper_2507_03836_b200 import fhash as fh  # noqa: E402
which, N = sys.argv[1], int(sys.argv[2])
cfg, mlp = (W.CFG3, W.MLP3) if which == "cfg3" else (W.CFG4, W.MLP4)
enc = fh.Encoder(cfg.levels, cfg.F, cfg.table_dtype, cfg.cap)
g = torch.Generator("cuda").manual_seed(0)
tr = fh.Trainer(enc, (torch.rand((enc.entries, cfg.F), device="cuda", generator=g) * 2 - 1) * 1e-4,
                W.draw_mlp(W.rng(0), mlp), max(N, 4096))
c = torch.rand((N, 4), device="cuda", generator=g)
for _ in range(6):
    tr.infer(c)
torch.cuda.synchronize()
print("ok")
