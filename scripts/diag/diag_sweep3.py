import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
from oracle import semstream_oracle as O
from oracle.synth import make_clip
from paper_2602_03529_b200.pipeline import GopCodec
H, W, s = 60, 56, 3
src = make_clip("static-detail", W, H, 9, seed=85).gop(0)
for gid in (0, 0xa929a2af):
    for dk in (0, 1):
        c = GopCodec(1, H, W, s)
        c.set_gop_ids([gid])
        frames = torch.from_numpy(src[None].copy()).cuda()
        c.tokenize(frames, 1)
        torch.cuda.synchronize()
        t0 = c.tok[0].cpu().numpy().copy()
        c.select_and_pack(1, dk)
        torch.cuda.synchronize()
        t1 = c.tok[0].cpu().numpy()
        iv, pv = O.encode(O.downscale(src, s))
        arena, lengths = c.arena.cpu().numpy(), c.lengths.cpu().numpy()
        ref = O.pipeline_gop(src, s, gop_id=gid, drop_rate=0.05)
        print(hex(gid), "drop_k", dk, "tok I ok", np.array_equal(t0[0], iv), "P ok", np.array_equal(t0[1], pv),
              "after pack I ok", np.array_equal(t1[0], iv), "pkt0 eq", arena[0, :lengths[0]].tobytes() == ref["wire"][0],
              "k used", c.drop_k(0.05))
