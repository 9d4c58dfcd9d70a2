import sys
sys.path.insert(0, ".")
import numpy as np, torch
from oracle import semstream_oracle as O
from oracle.synth import make_clip
from paper_2602_03529_b200 import _dev, _lib
def enc(H, W, s, srcs, label):
    g = len(srcs)
    fr = torch.from_numpy(np.stack(srcs)).cuda()
    Ht, Wt = -(-(-(-H // s)) // 8), -(-(-(-W // s)) // 8)
    tok = torch.full((g, 2, Ht, Wt, 12), 7.0, dtype=torch.float64, device="cuda")
    sim = torch.empty((g, Ht, Wt), dtype=torch.float64, device="cuda")
    _lib.call("sst_encode", fr.data_ptr(), g, H, W, s, tok.data_ptr(), sim.data_ptr(), _dev.stream())
    torch.cuda.synchronize()
    t = tok.cpu().numpy()
    res = []
    for i in range(g):
        iv, pv = O.encode(O.downscale(srcs[i], s))
        res.append(bool(np.array_equal(t[i, 0], iv) and np.array_equal(t[i, 1], pv)))
    print(label, (H, W, s, g), res, "frames ptr", hex(fr.data_ptr()))
    return fr
a = [make_clip("noise-field", 104, 113, 9, seed=60).gop(0), make_clip("noisy-motion", 104, 113, 9, seed=75).gop(0)]
b = [make_clip("static-detail", 56, 60, 9, seed=85).gop(0)]
enc(60, 56, 3, b, "b first")
enc(113, 104, 3, a, "a")
enc(60, 56, 3, b, "b after a")
enc(60, 56, 3, b, "b again")
keep = enc(113, 104, 3, a, "a (kept)")
enc(60, 56, 3, b, "b after a kept")
