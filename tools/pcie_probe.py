"""Pinned host->device copy bandwidth on the box (the e2e ceiling): gpurun -- python tools/pcie_probe.py"""
import torch, time
x = torch.empty(2_080_000_000, dtype=torch.uint8).pin_memory()
d = torch.empty_like(x, device="cuda")
y = torch.empty(160_000_000, dtype=torch.uint8, device="cuda"); yh = torch.empty(160_000_000, dtype=torch.uint8).pin_memory()
for i in range(2): d.copy_(x, non_blocking=True)
torch.cuda.synchronize()
a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
a.record(); 
for i in range(3): d.copy_(x, non_blocking=True)
b.record(); b.synchronize(); print("H2D GB/s", 3*x.numel()/a.elapsed_time(b)/1e6)
s2 = torch.cuda.Stream()
a.record()
for i in range(3):
    d.copy_(x, non_blocking=True)
    with torch.cuda.stream(s2): yh.copy_(y, non_blocking=True)
torch.cuda.synchronize(); b.record(); b.synchronize(); print("H2D + concurrent D2H GB/s (H2D bytes)", 3*x.numel()/a.elapsed_time(b)/1e6)
