"""ncu target: one raw-rgb24 K1 (sst_encode_u8) and K5 (sst_upscale_blend_u8)
launch over 32 x 1080p GoPs at s = argv[1] (3)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2602_03529_b200 import _dev, _lib
G, H, W = 32, 1080, 1920
s = int(sys.argv[1]) if len(sys.argv) > 1 else 3
dev = _dev.device()
u8 = (torch.rand((G, 9, H, W, 3), device=dev) * 255).to(torch.uint8)
h, w = -(-H // s), -(-W // s)
Ht, Wt = -(-h // 8), -(-w // 8)
tok = torch.empty((G, 2, Ht, Wt, 12), dtype=torch.float64, device=dev)
sim = torch.empty((G, Ht, Wt), dtype=torch.float64, device=dev)
img = torch.rand((G, 2, h, w, 3), device=dev)
d = np.zeros(G, dtype=_lib.PREV_DTYPE)
d["p_img"] = img.data_ptr() + np.arange(G, dtype=np.uint64) * np.uint64(2 * h * w * 3 * 4) + np.uint64(h * w * 3 * 4)
d["h"], d["w"], d["s"] = h, w, s
prev = torch.from_numpy(d.view(np.uint8).copy()).to(dev)
for _ in range(3):
    _lib.call("sst_encode_u8", u8.data_ptr(), G, H, W, s, tok.data_ptr(), sim.data_ptr(), None, _dev.stream())
    _lib.call("sst_upscale_blend_u8", img.data_ptr(), G, h, w, s, H, W, prev.data_ptr(), 2, u8.data_ptr(),
              _dev.stream())
torch.cuda.synchronize()
