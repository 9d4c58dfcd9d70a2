"""B200 HBM stream ceilings (context for the K1 read / K5 write rooflines):
read-only, write-only and copy bandwidth on multi-GB buffers, CUDA events."""
import json
import torch

n = 7 * 1024 ** 3 // 4                      # ~7 GB of float32
a = torch.rand(n, device="cuda")
b = torch.empty_like(a)


def t(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


r = t(lambda: a.sum())
w = t(lambda: b.fill_(0.5))
c = t(lambda: b.copy_(a))
nb = n * 4
print(json.dumps({"bytes": nb, "read_GBps": round(nb / r / 1e6, 1),
                  "write_GBps": round(nb / w / 1e6, 1),
                  "copy_GBps_read_plus_write": round(2 * nb / c / 1e6, 1)}))
