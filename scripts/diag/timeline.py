"""Timeline of one bench step (2 lanes x 32 x 1080p): CUDA-event timestamps of
every stage on its own stream, relative to the step start."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import bench
from paper_2602_03529_b200.pipeline import StreamBank

class EvTimer:
    def __init__(self, tag): self.tag, self.ev = tag, []
    def begin(self, name):
        e = torch.cuda.Event(enable_timing=True); e.record(); self.ev.append((self.tag, name, "b", e))
    def end(self, name):
        e = torch.cuda.Event(enable_timing=True); e.record(); self.ev.append((self.tag, name, "e", e))

dev = torch.device("cuda", 0)
S, H, W = 64, 1080, 1920
inputs = bench.make_inputs(list(range(S)), H, W, dev)
out = torch.empty_like(inputs[0])
even, odd = list(range(0, S, 2)), list(range(1, S, 2))
lanes = []
for ph, ids in enumerate((even, odd)):
    lanes.append(dict(sl=slice(ph * 32, ph * 32 + 32), phase=ph, bank=StreamBank(32, H, W, concurrent_groups=False),
                      stream=torch.cuda.Stream()))
def step(k, timers=None):
    fr = inputs[k % 2]
    for i, ln in enumerate(lanes):
        s = bench.scale_of(ln["phase"], k)
        if timers: ln["bank"].set_timer(timers[i])
        with torch.cuda.stream(ln["stream"]):
            ln["bank"].step({s: fr[ln["sl"]]}, {s: out[ln["sl"]]}, {s: list(range(32))}, {s: [k] * 32}, drop_rate=0.1)
for k in range(4): step(k)
torch.cuda.synchronize()
t0 = torch.cuda.Event(enable_timing=True)
timers = [EvTimer("A"), EvTimer("B")]
main = torch.cuda.current_stream()
t0.record()
for ln in lanes: ln["stream"].wait_stream(main)
step(4, timers)
for ln in lanes: main.wait_stream(ln["stream"])
t1 = torch.cuda.Event(enable_timing=True); t1.record()
torch.cuda.synchronize()
print("step ms", t0.elapsed_time(t1))
rows = []
for tm in timers:
    for tag, name, be, e in tm.ev:
        rows.append((t0.elapsed_time(e), tag, name, be))
for r in sorted(rows): print(f"{r[0]:8.3f} {r[1]} {r[2]:18s} {r[3]}")
