import sys
sys.path.insert(0, ".")
import numpy as np, torch
from oracle import semstream_oracle as O
from oracle.synth import make_clip
from paper_2602_03529_b200 import _dev, _lib
np.set_printoptions(precision=5, linewidth=150)
b = make_clip("static-detail", 56, 60, 9, seed=85).gop(0)
fr = torch.from_numpy(b[None].copy()).cuda()
tok = torch.full((1, 2, 3, 3, 12), 7.0, dtype=torch.float64, device="cuda")
sim = torch.empty((1, 3, 3), dtype=torch.float64, device="cuda")
_lib.call("sst_encode", fr.data_ptr(), 1, 60, 56, 3, tok.data_ptr(), sim.data_ptr(), _dev.stream())
torch.cuda.synchronize()
t = tok.cpu().numpy()[0]
iv, pv = O.encode(O.downscale(b, 3))
print("nan in gpu", np.isnan(t).any(), "nan in oracle", np.isnan(iv).any(), np.isnan(pv).any())
print("gpu I[0,0]", t[0, 0, 0], "\nora I[0,0]", iv[0, 0])
print("frames min/max", b.min(), b.max(), "nan in frames", np.isnan(b).any())
w = O.downscale(b, 3)
print("working nan", np.isnan(w).any(), w.shape)
d = t[0] - iv
print("I maxdiff", np.abs(d).max(), "n diff", (d != 0).sum(), "of", d.size)
d = t[1] - pv
print("P maxdiff", np.abs(d).max(), "n diff", (d != 0).sum())
idx = np.argwhere(t[0] != iv)[:5]
for y, x, c in idx: print(y, x, c, repr(t[0, y, x, c]), repr(iv[y, x, c]))
# check the GPU downscale too and the oracle pieces
ds = torch.empty((9, 20, 19, 3), dtype=torch.float32, device="cuda")
_lib.call("sst_downscale", fr.data_ptr(), 9, 60, 56, 3, ds.data_ptr(), _dev.stream())
torch.cuda.synchronize()
print("downscale equal", np.array_equal(ds.cpu().numpy(), w), "max", np.abs(ds.cpu().numpy() - w).max())
