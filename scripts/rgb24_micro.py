"""K1 and K5 alone over raw-rgb24 (uint8) vs float32 frames: back-to-back
launches of 32 x 1080p GoPs (sst_encode_u8 vs sst_encode_work;
sst_upscale_blend_u8 vs sst_upscale_blend, blend n=2)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2602_03529_b200 import _dev, _lib
G, H, W = 32, 1080, 1920
dev = _dev.device()


def timed(fn, n=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


f32 = torch.rand((G, 9, H, W, 3), device=dev)
u8 = (f32 * 255).to(torch.uint8)
for s in (3, 2):
    h, w = -(-H // s), -(-W // s)
    Ht, Wt = -(-h // 8), -(-w // 8)
    tok = torch.empty((G, 2, Ht, Wt, 12), dtype=torch.float64, device=dev)
    sim = torch.empty((G, Ht, Wt), dtype=torch.float64, device=dev)
    for nm, fr, fn in (("f32", f32, "sst_encode_work"), ("u8 ", u8, "sst_encode_u8")):
        ms = timed(lambda: _lib.call(fn, fr.data_ptr(), G, H, W, s, tok.data_ptr(), sim.data_ptr(), None,
                                     _dev.stream()))
        print(f"K1 s={s} {nm}: {ms:.3f} ms  {fr.numel() * fr.element_size() / ms / 1e6:.0f} GB/s read")
    img = torch.rand((G, 2, h, w, 3), device=dev)
    d = np.zeros(G, dtype=_lib.PREV_DTYPE)
    d["p_img"] = img.data_ptr() + np.arange(G, dtype=np.uint64) * np.uint64(2 * h * w * 3 * 4) + np.uint64(h * w * 3 * 4)
    d["h"], d["w"], d["s"] = h, w, s
    prev = torch.from_numpy(d.view(np.uint8).copy()).to(dev)
    for nm, out, fn in (("f32", f32, "sst_upscale_blend"), ("u8 ", u8, "sst_upscale_blend_u8")):
        ms = timed(lambda: _lib.call(fn, img.data_ptr(), G, h, w, s, H, W, prev.data_ptr(), 2, out.data_ptr(),
                                     _dev.stream()))
        print(f"K5 s={s} {nm}: {ms:.3f} ms  {out.numel() * out.element_size() / ms / 1e6:.0f} GB/s written")
