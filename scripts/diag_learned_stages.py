import sys
sys.path.insert(0, ".")
import torch
from paper_2602_03529_b200 import _dev
from paper_2602_03529_b200.pipeline import StageTimer
from paper_2602_03529_b200.learned import LearnedConfig, LearnedGopCodec
G, H, W, s = 32, 1080, 1920, 3
dev = _dev.device()
codec = LearnedGopCodec(G, H, W, s, cfg=LearnedConfig())
fr = torch.rand((G, 9, H, W, 3), device=dev)
out = torch.empty_like(fr); prev = torch.empty_like(fr)
for _ in range(2):
    codec.step(fr, out, G, drop_k=codec.drop_k(0.1))
torch.cuda.synchronize()
t = StageTimer(); codec.timer = t
for _ in range(3):
    codec.step(fr, out, G, drop_k=codec.drop_k(0.1))
torch.cuda.synchronize()
for k, (ms, n) in t.summary().items():
    print(f"{k:20s} {ms / n:8.3f} ms")
