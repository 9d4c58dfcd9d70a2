"""Driver for ncu / timing: one 1080p stream through StreamBank, one GoP in
flight, scales 3,3,2,2 (the bench's single_stream leg).  argv: steps"""
import sys
sys.path.insert(0, ".")
import torch
from paper_2602_03529_b200.pipeline import StreamBank
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
H, W = 1080, 1920
bank = StreamBank(1, H, W)
fr = torch.rand((1, 9, H, W, 3), device="cuda")
out = torch.empty_like(fr)
for k in range(steps):
    s = (3, 3, 2, 2)[k % 4]
    bank.step({s: fr}, {s: out}, {s: [0]}, {s: [k]}, drop_rate=0.1)
    torch.cuda.synchronize()
print("done")
