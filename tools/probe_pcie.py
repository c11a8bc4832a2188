"""PCIe probe: pinned host <-> device copy bandwidth, one direction and both
at once (the e2e figure's ceiling).  Not the bench."""
import torch

n = 184 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn in [("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))]:
    fn(); torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        fn()
    e1.record(); torch.cuda.synchronize()
    print(name, round(5 * n / (e0.elapsed_time(e1) / 1e3) / 1e9, 1), "GB/s")
torch.cuda.synchronize()
e0.record()
for _ in range(5):
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
torch.cuda.current_stream().wait_stream(s1)
torch.cuda.current_stream().wait_stream(s2)
e1.record(); torch.cuda.synchronize()
print("both", round(5 * n / (e0.elapsed_time(e1) / 1e3) / 1e9, 1), "GB/s per direction")
