"""Pinned host -> device bandwidth on this box (context for the e2e number)."""
import torch, time
x = torch.empty(1 << 27, dtype=torch.float64).pin_memory()  # 1 GiB
y = torch.empty_like(x, device="cuda")
for _ in range(2):
    y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    y.copy_(x, non_blocking=True)
e1.record()
torch.cuda.synchronize()
print(f"H2D pinned 1 GiB: {5 * x.numel() * 8 / (e0.elapsed_time(e1) / 1e3) / 1e9:.1f} GB/s")
