"""Pinned host -> device copy bandwidth for the bench's per-step feature block (562 MB)."""
import time
import torch
x = torch.empty((232965, 604), dtype=torch.float32).pin_memory()
d = torch.empty_like(x, device="cuda")
for _ in range(2):
    d.copy_(x, non_blocking=True)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    d.copy_(x, non_blocking=True)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 5
print(f"H2D {x.numel() * 4 / 1e6:.0f} MB in {ms:.2f} ms = {x.numel() * 4 / ms / 1e6:.1f} GB/s")
