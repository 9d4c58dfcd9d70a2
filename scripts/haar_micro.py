"""Int8 patchify alone, 32 x 1080p GoPs at s=1 and s=3: plain
(sst_lt8_patchify) vs the integer 3-D Haar front end (sst_lt8_patchify_haar).
Both read the f32 frames once (224 MB per GoP) and write the int8 patches."""
import os
import sys
sys.path.insert(0, ".")
import torch
from paper_2602_03529_b200 import _dev, _lib
G, H, W = 32, 1080, 1920
dev = _dev.device()
fr = torch.rand((G, 9, H, W, 3), device=dev)
for s in (1, 3):
    h, w = -(-H // s), -(-W // s)
    Ht, Wt = -(-h // 8), -(-w // 8)
    pI = torch.empty((G, Ht, Wt, 256), dtype=torch.int8, device=dev)
    pP = torch.empty((G, Ht, Wt, 1536), dtype=torch.int8, device=dev)
    for fn, env in (("sst_lt8_patchify", ""), ("sst_lt8_patchify", "band"),
                    ("sst_lt8_patchify_haar", "")):
        os.environ["SST_LT8_PATCHIFY"] = env
        def run():
            _lib.call(fn, fr.data_ptr(), G, H, W, s, pI.data_ptr(), pP.data_ptr(), _dev.stream())
        for _ in range(2):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(5):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        gb = (fr.numel() * 4 + pI.numel() + pP.numel()) / 1e9
        print(f"s={s} {fn} {env}: {ms:.3f} ms per launch, {gb / ms:.2f} TB/s")
