import sys
sys.path.insert(0, ".")
import numpy as np, torch
from oracle import semstream_oracle as O
from oracle.synth import make_clip
from paper_2602_03529_b200.pipeline import GopCodec
kinds = ["moving-square", "noisy-motion", "static-detail", "noise-field", "static-gradient"]
for seed in range(4):
    rng = np.random.default_rng(1000 + seed)
    H, W = int(rng.integers(9, 181)), int(rng.integers(9, 261))
    s = int(rng.choice([2, 3])); g = int(rng.integers(1, 4))
    drop = float(rng.choice([0.0, 0.05, 0.1, 0.25, 0.3]))
    ks = []
    srcs = []
    for _ in range(g):
        k = kinds[int(rng.integers(len(kinds)))]; sd = int(rng.integers(99)); ks.append((k, sd))
        srcs.append(make_clip(k, W, H, 9, seed=sd).gop(0))
    print(seed, H, W, s, g, ks)
    c = GopCodec(g, H, W, s)
    frames = torch.from_numpy(np.stack(srcs)).cuda()
    c.tokenize(frames, g)
    torch.cuda.synchronize()
    tok = c.tok[:g].cpu().numpy().copy()
    print("   frames intact", np.array_equal(frames.cpu().numpy(), np.stack(srcs)))
    for i in range(g):
        iv, pv = O.encode(O.downscale(srcs[i], s))
        src2 = make_clip(*ks[i][:1], W, H, 9, seed=ks[i][1]).gop(0)
        print("   src regenerated equal", np.array_equal(src2, srcs[i]))
        bad = np.argwhere(np.abs(tok[i, 0] - iv).max(-1) > 0)
        print("   I bad", bad.tolist()[:6], "P bad", np.argwhere(np.abs(tok[i, 1] - pv).max(-1) > 0).tolist()[:6])
