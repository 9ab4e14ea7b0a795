"""Diagnostic: pinned H2D bandwidth on this box (18 MB chunks, like the e2e leg)."""
import time
import torch
dev = torch.device("cuda", 0)
for mb in (2, 18, 64):
    h = torch.empty(mb << 20, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(mb << 20, dtype=torch.uint8, device=dev)
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        d.copy_(h, non_blocking=True)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    print(f"{mb} MB pinned H2D: {ms*1e3:.1f} us -> {(mb<<20)/(ms*1e-3)/1e9:.1f} GB/s")
# many fresh pinned tensors (like the e2e leg: one per step and node)
hs = [torch.empty(4 << 20, dtype=torch.uint8, pin_memory=True) for _ in range(200)]
d = torch.empty(4 << 20, dtype=torch.uint8, device=dev)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for h in hs:
    d.copy_(h, non_blocking=True)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / len(hs)
print(f"200 distinct 4 MB pinned buffers: {ms*1e3:.1f} us each -> {(4<<20)/(ms*1e-3)/1e9:.1f} GB/s")
