"""K5-9 over uint8 working frames (the int8 learned codec's path) vs float32:
back-to-back sst_upscale_blend9_u8 / sst_upscale_blend9 launches (G x 1080p)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2602_03529_b200 import _dev, _lib
G = 32; H, W = 1080, 1920
dev = _dev.device()
out = torch.empty((G, 9, H, W, 3), device=dev)
for s in (3, 2):
    h, w = -(-H // s), -(-W // s)
    for dt, fn in ((torch.uint8, "sst_upscale_blend9_u8"), (torch.float32, "sst_upscale_blend9")):
        img = (torch.rand((G, 9, h, w, 3), device=dev) * (255 if dt == torch.uint8 else 1)).to(dt)
        prv = (torch.rand((G, 9, h, w, 3), device=dev) * (255 if dt == torch.uint8 else 1)).to(dt)
        d = np.zeros(G, dtype=_lib.PREV_DTYPE)
        d["p_img"] = prv.data_ptr() + np.arange(G, dtype=np.uint64) * np.uint64(prv[0].numel() * prv.element_size())
        d["h"], d["w"], d["s"] = h, w, s
        prev = torch.from_numpy(d.view(np.uint8).copy()).to(dev)
        for pv in (None, prev):
            def run():
                _lib.call(fn, img.data_ptr(), G, h, w, s, H, W,
                          None if pv is None else pv.data_ptr(), 2, out.data_ptr(), _dev.stream())
            for _ in range(3): run()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            n = 10
            e0.record()
            for _ in range(n): run()
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / n
            print(f"s={s} {str(dt):14s} prev={'y' if pv is not None else 'n'}: {ms:.3f} ms")
