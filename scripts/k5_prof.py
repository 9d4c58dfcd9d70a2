"""K5 (main path) alone, one configuration launched a few times: the ncu
target (32 x 1080p GoPs, s = argv[1] (3), blend n=2 against a previous GoP)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2602_03529_b200 import _dev, _lib
G, H, W = 32, 1080, 1920
s = int(sys.argv[1]) if len(sys.argv) > 1 else 3
dev = _dev.device()
out = torch.empty((G, 9, H, W, 3), device=dev)
h, w = -(-H // s), -(-W // s)
img = torch.rand((G, 2, h, w, 3), device=dev)
d = np.zeros(G, dtype=_lib.PREV_DTYPE)
d["p_img"] = img.data_ptr() + np.arange(G, dtype=np.uint64) * np.uint64(2 * h * w * 3 * 4) + np.uint64(h * w * 3 * 4)
d["h"], d["w"], d["s"] = h, w, s
prev = torch.from_numpy(d.view(np.uint8).copy()).to(dev)
for _ in range(5):
    _lib.call("sst_upscale_blend", img.data_ptr(), G, h, w, s, H, W, prev.data_ptr(), 2,
              out.data_ptr(), _dev.stream())
torch.cuda.synchronize()
