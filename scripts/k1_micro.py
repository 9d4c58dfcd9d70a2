import sys; sys.path.insert(0, ".")
import torch
from paper_2602_03529_b200 import _dev, _lib
G, H, W = 32, 1080, 1920
dev = _dev.device()
fr = torch.rand((G, 9, H, W, 3), device=dev)
for s in (3, 2):
    h, w = -(-H // s), -(-W // s); Ht, Wt = -(-h // 8), -(-w // 8)
    tok = torch.empty((G, 2, Ht, Wt, 12), dtype=torch.float64, device=dev)
    sim = torch.empty((G, Ht, Wt), dtype=torch.float64, device=dev)
    run = lambda: _lib.call("sst_encode", fr.data_ptr(), G, H, W, s, tok.data_ptr(), sim.data_ptr(), _dev.stream())
    for _ in range(3): run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10): run()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"s={s}: {ms:.3f} ms  {fr.numel() * 4 / ms / 1e6:.0f} GB/s")
