import sys; sys.path.insert(0, ".")
import torch
from paper_2602_03529_b200 import _lib
from paper_2602_03529_b200.learned import LearnedTokenizer, LearnedConfig, TAPS_233
m = LearnedTokenizer(LearnedConfig())
G, Ht, Wt, D = 32, 45, 80, 256
dev = torch.device("cuda")
x = (torch.randn((G, 2, Ht, Wt, 64), device=dev) * 0.3).to(torch.bfloat16)
h = torch.empty((G, 2, Ht, Wt, D), dtype=torch.bfloat16, device=dev)
TAPS_23 = [(kt - 1, ky - 1, 0) for kt in range(2) for ky in range(3)]
m.W["p6"] = (torch.randn((D, 6 * 64), device=dev) * 0.05).to(torch.bfloat16)
m.b["p6"] = torch.zeros(D, device=dev)
def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
a = t(lambda: m._conv("dec_in", x, (G, 2, Ht, Wt, 64), (Ht, Wt), TAPS_233, 0, 2, _lib.LT_EPI_STORE, act=1, out=h))
b = t(lambda: m._conv("p6", x, (G, 2, Ht, Wt, 64), (Ht, Wt), TAPS_23, 0, 2, _lib.LT_EPI_STORE, act=1, out=h))
print(f"dec_in 18 taps: {a:.3f} ms   packed 6 taps: {b:.3f} ms")
