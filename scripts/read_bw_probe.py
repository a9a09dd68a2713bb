"""Diagnostic: read-only HBM bandwidth (torch sum over a 16 GiB fp32 tensor) vs
the copy figure in MEASURED_PEAKS.json."""
import torch

x = torch.empty(4 << 30, dtype=torch.float32, device="cuda").fill_(1.0)
for _ in range(2):
    x.sum()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    x.sum()
e1.record()
torch.cuda.synchronize()
print(f"read-only sum: {x.numel() * 4 * 5 / (e0.elapsed_time(e1) / 1e3) / 1e9:.0f} GB/s")
y = torch.empty_like(x)
y.copy_(x)
torch.cuda.synchronize()
e0.record()
for _ in range(5):
    y.copy_(x)
e1.record()
torch.cuda.synchronize()
print(f"copy (read + write): {2 * x.numel() * 4 * 5 / (e0.elapsed_time(e1) / 1e3) / 1e9:.0f} GB/s")
