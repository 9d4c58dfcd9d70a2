"""Pure-write and pure-read HBM ceilings on this B200 (fill_, sum) for 7.2 GB."""
import torch
n = 7_200_000_000 // 4
x = torch.empty(n, dtype=torch.float32, device="cuda")
for _ in range(2): x.fill_(1.0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(5): x.fill_(0.5)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"fill (write-only) {n * 4 / ms / 1e9:.1f} TB/s  ({ms:.3f} ms per 7.2 GB)")
e0.record()
for _ in range(5): s = x.sum()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"sum (read-only) {n * 4 / ms / 1e9:.1f} TB/s")
y = torch.empty_like(x)
e0.record()
for _ in range(5): y.copy_(x)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"copy (read+write) {2 * n * 4 / ms / 1e9:.1f} TB/s")
