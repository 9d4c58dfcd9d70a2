"""LearnedGopCodec at G x 1080p GoPs per step: eager steps vs CUDA-graph
replay (GraphedLearnedGopCodec), CUDA-event timed."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2602_03529_b200.learned import (GraphedLearnedGopCodec, LearnedConfig,
                                           LearnedGopCodec, LearnedTokenizer)
G = int(sys.argv[1]) if len(sys.argv) > 1 else 32
H, W, s = 1080, 1920, 3
dev = torch.device("cuda")
model = LearnedTokenizer(LearnedConfig())
frames = torch.rand((G, 9, H, W, 3), device=dev)
out = torch.empty_like(frames)


def timed(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


c = LearnedGopCodec(G, H, W, s, model=model)
c.set_gop_ids(list(range(G)))
k = c.drop_k(0.1)
eager = timed(lambda: c.step(frames, out, G, drop_k=k))
del c
cg = LearnedGopCodec(G, H, W, s, model=model)
gr = GraphedLearnedGopCodec(cg, G, frames, out, drop_k=k)
graph = timed(lambda: gr.step(list(range(G))))
print(f"G={G}: eager {eager:.3f} ms  graph {graph:.3f} ms  ({G * 9 / graph * 1e3:.0f} frames/s graphed)")
