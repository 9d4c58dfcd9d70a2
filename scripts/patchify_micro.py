"""k_lt_patchify alone: 32 x 1080p GoPs -> I / P patch tensors (s=3)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2602_03529_b200 import _dev, _lib
G, H, W, s = 32, 1080, 1920, 3
dev = _dev.device()
fr = torch.rand((G, 9, H, W, 3), device=dev)
h, w = -(-H // s), -(-W // s)
Ht, Wt = -(-h // 8), -(-w // 8)
pI = torch.empty((G, Ht, Wt, 192), dtype=torch.bfloat16, device=dev)
pP = torch.empty((G, Ht, Wt, 1536), dtype=torch.bfloat16, device=dev)
run = lambda: _lib.call("sst_lt_patchify", fr.data_ptr(), G, H, W, s, pI.data_ptr(), pP.data_ptr(),
                        _dev.stream())
for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(10):
    run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"patchify s={s}: {ms:.3f} ms  {fr.numel() * 4 / ms / 1e6:.0f} GB/s (frame reads)")
