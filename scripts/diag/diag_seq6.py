import sys
sys.path.insert(0, ".")
import numpy as np, torch
from oracle import semstream_oracle as O
from oracle.synth import make_clip
from paper_2602_03529_b200 import _dev, _lib
b0 = make_clip("static-detail", 56, 60, 9, seed=85).gop(0)
a = [make_clip("noise-field", 104, 113, 9, seed=60).gop(0), make_clip("noisy-motion", 104, 113, 9, seed=75).gop(0)]
b = make_clip("static-detail", 56, 60, 9, seed=85).gop(0)
print("b same as b0:", np.array_equal(b, b0))
np.save("gpurun_out/b_seq.npy", b)
fr = torch.from_numpy(b[None].copy()).cuda()
tok = torch.full((1, 2, 3, 3, 12), 7.0, dtype=torch.float64, device="cuda")
sim = torch.empty((1, 3, 3), dtype=torch.float64, device="cuda")
_lib.call("sst_encode", fr.data_ptr(), 1, 60, 56, 3, tok.data_ptr(), sim.data_ptr(), _dev.stream())
ds = torch.empty((9, 20, 19, 3), dtype=torch.float32, device="cuda")
_lib.call("sst_downscale", fr.data_ptr(), 9, 60, 56, 3, ds.data_ptr(), _dev.stream())
torch.cuda.synchronize()
np.save("gpurun_out/b_tok.npy", tok.cpu().numpy())
w = O.downscale(b, 3)
print("downscale equal", np.array_equal(ds.cpu().numpy(), w))
iv, pv = O.encode(w)
t = tok.cpu().numpy()[0]
print("I diffs", (t[0] != iv).sum(), "P diffs", (t[1] != pv).sum(), "max", np.abs(t[0]-iv).max(), np.abs(t[1]-pv).max())
