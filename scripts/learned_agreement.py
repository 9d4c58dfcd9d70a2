"""End-to-end FSQ index agreement GPU vs oracle for the default learned config."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from oracle import learned_oracle as LO
from oracle.synth import make_clip
from paper_2602_03529_b200 import _dev
from paper_2602_03529_b200.learned import LearnedConfig, LearnedTokenizer, make_weights
cfg = LearnedConfig()
w = make_weights(cfg)
m = LearnedTokenizer(cfg, w)
for name, seed in (("moving-square", 1), ("noisy-motion", 2)):
    fr = np.stack([make_clip(name, 1920, 1080, 9, seed=seed).gop(0)])
    codes, idx, mask, hw = m.encode_frames(torch.from_numpy(fr).to(_dev.device()), 3)
    oc, oi, _, z = LO.encode(fr, 3, w, cfg.blocks)
    tok = (idx.cpu().numpy() == oi).all(-1).mean()
    per_idx = (idx.cpu().numpy() == oi).mean()
    print(f"{name}: tokens {oi.shape[1:4]} token agreement {tok:.5f} index agreement {per_idx:.5f}")
