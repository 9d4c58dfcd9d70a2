"""Learned-tokenizer throughput at 1080p (encode + FSQ + decode), per-layer
tensor-core rates.  Usage: python scripts/bench_learned.py [G] [s] [dim] [blocks]"""
import json, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2602_03529_b200 import _dev
from paper_2602_03529_b200.learned import LearnedConfig, LearnedTokenizer, TAPS_233

G = int(sys.argv[1]) if len(sys.argv) > 1 else 16
s = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dim = int(sys.argv[3]) if len(sys.argv) > 3 else 256
blocks = int(sys.argv[4]) if len(sys.argv) > 4 else 2
dev = _dev.device()
m = LearnedTokenizer(LearnedConfig(dim=dim, blocks=blocks))
H, W = 1080, 1920
frames = torch.rand((G, 9, H, W, 3), device=dev)
codes, idx, mask, hw = m.encode_frames(frames, s)
out = m.decode_tokens(codes, mask, hw)
torch.cuda.synchronize()
Ht, Wt = codes.shape[2], codes.shape[3]
# per-layer timing (serialised)
times = {}
orig = m._conv
def timed(name, x, in_shape, out_grid, taps, t_lo, t_cnt, epi, **k):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); orig(name, x, in_shape, out_grid, taps, t_lo, t_cnt, epi, **k); e1.record()
    torch.cuda.synchronize()
    N, K = m.W[name].shape
    flops = 2 * in_shape[0] * t_cnt * Ht * Wt * N * K
    times.setdefault(name, []).append((e0.elapsed_time(e1), flops))
m._conv = timed
for _ in range(3):
    codes, idx, mask, hw = m.encode_frames(frames, s)
    out = m.decode_tokens(codes, mask, hw)
m._conv = orig
rows = []
for k, v in times.items():
    ms = np.median([a for a, _ in v]); fl = v[0][1]
    rows.append((k, ms, fl / ms / 1e9))
for k, ms, tf in rows:
    print(f"{k:10s} {ms:8.3f} ms  {tf:7.1f} TFLOP/s")
# whole path, pipelined
for _ in range(2):
    codes, idx, mask, hw = m.encode_frames(frames, s); out = m.decode_tokens(codes, mask, hw)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
n = 5
e0.record()
for _ in range(n):
    codes, idx, mask, hw = m.encode_frames(frames, s); out = m.decode_tokens(codes, mask, hw)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
fl = m.flops_per_gop(Ht, Wt) * G
print(json.dumps({"G": G, "s": s, "dim": dim, "blocks": blocks, "ms_per_step": ms,
                  "fps": G * 9 / ms * 1e3, "tflops": fl / ms / 1e9, "gflop_per_gop": m.flops_per_gop(Ht, Wt) / 1e9}))
