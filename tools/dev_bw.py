"""Box calibration: device-to-device copy bandwidth (read + write bytes)."""
import torch
a = torch.empty(2**29, dtype=torch.float64, device="cuda")  # 4.3 GB
b = torch.empty_like(a)
a.fill_(1.0)
for _ in range(3):
    b.copy_(a)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); b.copy_(a); e.record(); torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e))
print("copy %.1f GB/s (best of 10, 2x%.2f GB)" % (2 * a.numel() * 8 / best / 1e6, a.numel() * 8 / 1e9))
