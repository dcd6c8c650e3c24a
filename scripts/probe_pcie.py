"""Raw pinned D2H / H2D copy rates of the bench's e2e byte counts (445.6 MB obs+reward+done down, 17.8 MB up)."""
import torch

d = torch.empty(445644800, dtype=torch.uint8, device="cuda")
h = torch.empty(445644800, dtype=torch.uint8).pin_memory()
u = torch.empty(17825792, dtype=torch.uint8).pin_memory()
du = torch.empty(17825792, dtype=torch.uint8, device="cuda")
s2 = torch.cuda.Stream()
for name, fn in (("D2H", lambda: h.copy_(d, non_blocking=True)), ("H2D", lambda: d.copy_(h, non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        fn()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    print(f"{name} 445.6 MB: {ms:.2f} ms  {445.6e6 / ms / 1e6:.1f} GB/s")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    h.copy_(d, non_blocking=True)
    with torch.cuda.stream(s2):
        du.copy_(u, non_blocking=True)
torch.cuda.current_stream().wait_stream(s2)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 5
print(f"D2H 445.6 MB + concurrent H2D 17.8 MB: {ms:.2f} ms per step -> {2**20 / ms * 1e3:.3e} env-steps/s bound")
