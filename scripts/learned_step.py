"""Driver for ncu: warm-up + N steps of the learned codec (G x 1080p, s=3).
argv: G steps [i8|bf16]"""
import sys
sys.path.insert(0, ".")
import torch
from paper_2602_03529_b200 import _dev
G = int(sys.argv[1]) if len(sys.argv) > 1 else 32
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
prec = sys.argv[3] if len(sys.argv) > 3 else "i8"
if prec == "i8":
    from paper_2602_03529_b200.learned_i8 import LearnedI8Config as Cfg, LearnedI8GopCodec as Codec
else:
    from paper_2602_03529_b200.learned import LearnedConfig as Cfg, LearnedGopCodec as Codec
dev = _dev.device()
codec = Codec(G, 1080, 1920, 3, cfg=Cfg())
fr = torch.rand((G, 9, 1080, 1920, 3), device=dev)
out = torch.empty_like(fr)
for _ in range(steps):
    codec.step(fr, out, G, drop_k=codec.drop_k(0.1))
torch.cuda.synchronize()
print("done")
