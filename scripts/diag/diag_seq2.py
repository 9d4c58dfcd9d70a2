import sys
sys.path.insert(0, ".")
import numpy as np, torch
from oracle import semstream_oracle as O
from oracle.synth import make_clip
from paper_2602_03529_b200 import _dev, _lib
def run(H, W, s, kind, sd, fill=None):
    src = make_clip(kind, W, H, 9, seed=sd).gop(0)
    iv, pv = O.encode(O.downscale(src, s))
    Ht, Wt = iv.shape[:2]
    fr = torch.from_numpy(src[None].copy()).cuda()
    tok = torch.empty((1, 2, Ht, Wt, 12), dtype=torch.float64, device="cuda")
    if fill is not None: tok.fill_(fill)
    sim = torch.empty((1, Ht, Wt), dtype=torch.float64, device="cuda")
    _lib.call("sst_encode", fr.data_ptr(), 1, H, W, s, tok.data_ptr(), sim.data_ptr(), _dev.stream())
    torch.cuda.synchronize()
    t = tok.cpu().numpy()[0]
    bad = np.argwhere(np.abs(t[0] - iv).max(-1) > 0)
    badp = np.argwhere(np.abs(t[1] - pv).max(-1) > 0)
    print((H, W, s, kind, sd, fill), "I bad", bad.tolist()[:8], "P bad", badp.tolist()[:8])
    if len(bad):
        y, x = bad[0]
        print("   got", t[0, y, x, :4], "want", iv[y, x, :4])
run(60, 56, 3, "static-detail", 85)
run(60, 56, 3, "static-detail", 85, fill=7.0)
run(113, 104, 3, "noisy-motion", 5)
run(60, 56, 3, "static-detail", 85)
run(60, 56, 3, "static-detail", 85, fill=float("nan"))
