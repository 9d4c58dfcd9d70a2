"""Driver for ncu: warm-up + N steps of LearnedGopCodec (G x 1080p, s=3)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2602_03529_b200 import _dev
from paper_2602_03529_b200.learned import LearnedConfig, LearnedGopCodec
G = int(sys.argv[1]) if len(sys.argv) > 1 else 32
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = _dev.device()
codec = LearnedGopCodec(G, 1080, 1920, 3, cfg=LearnedConfig())
fr = torch.rand((G, 9, 1080, 1920, 3), device=dev)
out = torch.empty_like(fr)
for _ in range(steps):
    codec.step(fr, out, G, drop_k=codec.drop_k(0.1))
torch.cuda.synchronize()
print("done")
