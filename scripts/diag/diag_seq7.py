import sys
sys.path.insert(0, ".")
import numpy as np, torch
from oracle import semstream_oracle as O
from oracle.synth import make_clip
from paper_2602_03529_b200 import _dev, _lib
a = [make_clip("noise-field", 104, 113, 9, seed=60).gop(0), make_clip("noisy-motion", 104, 113, 9, seed=75).gop(0)]
b = [make_clip("static-detail", 56, 60, 9, seed=85).gop(0)]
fr = torch.from_numpy(np.stack(b)).cuda()
tok = torch.full((1, 2, 3, 3, 12), 7.0, dtype=torch.float64, device="cuda")
sim = torch.empty((1, 3, 3), dtype=torch.float64, device="cuda")
_lib.call("sst_encode", fr.data_ptr(), 1, 60, 56, 3, tok.data_ptr(), sim.data_ptr(), _dev.stream())
torch.cuda.synchronize()
t = tok.cpu().numpy()[0]
for rep in range(2):
    w = O.downscale(b[0], 3)
    iv, pv = O.encode(w)
    print("rep", rep, "I diffs", (t[0] != iv).sum(), "P diffs", (t[1] != pv).sum(), "max", np.abs(t[0]-iv).max())
w2 = O.downscale(np.ascontiguousarray(b[0].copy()), 3)
print("oracle downscale stable", np.array_equal(w, w2))
iv2, pv2 = O.encode(w2.copy())
print("oracle encode stable", np.array_equal(iv, iv2), np.array_equal(pv, pv2))
print("flags", b[0].flags['C_CONTIGUOUS'], b[0].dtype, b[0].shape, b[0].strides)
