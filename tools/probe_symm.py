"""Probe: torch symmetric memory / NVLS multicast on this box (1 rank)."""
import os
import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as sm

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29555")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
t = sm.empty(1 << 20, dtype=torch.float32, device="cuda")
h = sm.rendezvous(t, dist.group.WORLD)
print("attrs", [a for a in dir(h) if not a.startswith("_")])
for a in ("multicast_ptr", "has_multicast_support", "world_size", "rank", "buffer_ptrs", "signal_pad_ptrs"):
    try:
        v = getattr(h, a)
        print(a, v() if callable(v) else v)
    except Exception as e:
        print(a, "ERR", e)
print("backend", sm.get_backend(torch.device("cuda", 0)) if hasattr(sm, "get_backend") else None)
dist.destroy_process_group()
