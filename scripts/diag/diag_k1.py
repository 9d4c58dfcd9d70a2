import sys
sys.path.insert(0, ".")
import numpy as np, torch
from oracle import semstream_oracle as O
from oracle.synth import make_clip
from paper_2602_03529_b200 import _dev, _lib
for (H, W, s, kind, sd) in [(60, 56, 3, "static-detail", 85), (60, 57, 3, "static-detail", 85), (60, 56, 3, "noisy-motion", 1), (64, 64, 3, "static-detail", 85)]:
    src = make_clip(kind, W, H, 9, seed=sd).gop(0)
    work = O.downscale(src, s)
    iv, pv = O.encode(work)
    Ht, Wt = iv.shape[:2]
    fr = torch.from_numpy(src[None].copy()).cuda()
    tok = torch.empty((1, 2, Ht, Wt, 12), dtype=torch.float64, device="cuda")
    sim = torch.empty((1, Ht, Wt), dtype=torch.float64, device="cuda")
    _lib.call("sst_encode", fr.data_ptr(), 1, H, W, s, tok.data_ptr(), sim.data_ptr(), _dev.stream())
    torch.cuda.synchronize()
    t = tok.cpu().numpy()[0]
    di = np.abs(t[0] - iv); dp = np.abs(t[1] - pv)
    bad = np.argwhere(di > 0)
    print((H, W, s, kind), "I maxdiff", di.max(), "P maxdiff", dp.max(), "bad I positions", bad[:6].tolist())
    # downscale alone
    ds = torch.empty((9, -(-H // s), -(-W // s), 3), dtype=torch.float32, device="cuda")
    _lib.call("sst_downscale", fr.data_ptr(), 9, H, W, s, ds.data_ptr(), _dev.stream())
    torch.cuda.synchronize()
    print("   downscale equal", np.array_equal(ds.cpu().numpy(), work))
