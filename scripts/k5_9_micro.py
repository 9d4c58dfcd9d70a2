"""K5-9 alone: back-to-back sst_upscale_blend9 launches (G x 1080p GoPs)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2602_03529_b200 import _dev, _lib
G = 32; H, W = 1080, 1920
dev = _dev.device()
out = torch.empty((G, 9, H, W, 3), device=dev)
for s in (3, 2):
    h, w = -(-H // s), -(-W // s)
    img = torch.rand((G, 9, h, w, 3), device=dev)
    prv = torch.rand((G, 9, h, w, 3), device=dev)
    d = np.zeros(G, dtype=_lib.PREV_DTYPE)
    d["p_img"] = prv.data_ptr() + np.arange(G, dtype=np.uint64) * np.uint64(9 * h * w * 3 * 4)
    d["h"], d["w"], d["s"] = h, w, s
    prev = torch.from_numpy(d.view(np.uint8).copy()).to(dev)
    for pv in (None, prev):
        def run():
            _lib.call("sst_upscale_blend9", img.data_ptr(), G, h, w, s, H, W,
                      None if pv is None else pv.data_ptr(), 2, out.data_ptr(), _dev.stream())
        for _ in range(3): run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        n = 10
        e0.record()
        for _ in range(n): run()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        byts = G * 9 * H * W * 3 * 4
        print(f"s={s} prev={'y' if pv is not None else 'n'}: {ms:.3f} ms  {byts / ms / 1e6:.0f} GB/s (writes only)")
