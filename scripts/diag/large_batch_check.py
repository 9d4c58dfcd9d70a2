"""Large-batch index safety: one LearnedGopCodec step over G = 64 1080p GoPs
(3.6 G floats of frames: > 2^31 elements) must equal the same GoPs run as two
G = 32 halves, bit for bit (second step, blend on)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2602_03529_b200.learned import LearnedConfig, LearnedGopCodec, LearnedTokenizer
G, H, W, s = 64, 1080, 1920, 3
dev = torch.device("cuda")
model = LearnedTokenizer(LearnedConfig())
gen = torch.Generator(device=dev).manual_seed(1)
f0 = torch.rand((G, 9, H, W, 3), generator=gen, device=dev)
f1 = torch.rand((G, 9, H, W, 3), generator=gen, device=dev)
big = LearnedGopCodec(G, H, W, s, model=model)
big.set_gop_ids(list(range(G)))
out = torch.empty_like(f0)
k = big.drop_k(0.1)
big.step(f0, out, G, drop_k=k)
big.step(f1, out, G, drop_k=k)
torch.cuda.synchronize()
ok = True
for half in range(2):
    sl = slice(half * 32, half * 32 + 32)
    c = LearnedGopCodec(32, H, W, s, model=model)
    c.set_gop_ids(list(range(half * 32, half * 32 + 32)))
    o = torch.empty((32, 9, H, W, 3), device=dev)
    c.step(f0[sl].contiguous(), o, 32, drop_k=k)
    c.step(f1[sl].contiguous(), o, 32, drop_k=k)
    torch.cuda.synchronize()
    same = torch.equal(o, out[sl])
    print(f"half {half}: bit-identical {same}")
    ok &= same
    del c, o
print("OK" if ok else "MISMATCH")

# main path: StreamBank with 64 streams at one scale vs two banks of 32
from paper_2602_03529_b200.pipeline import StreamBank
del big, out, model
torch.cuda.empty_cache()
outs = torch.empty_like(f0)
bank = StreamBank(G, H, W, scales=(s,))
for kk, f in enumerate((f0, f1)):
    bank.step({s: f}, {s: outs}, {s: list(range(G))}, {s: [kk] * G}, drop_rate=0.1)
torch.cuda.synchronize()
ok2 = True
for half in range(2):
    sl = slice(half * 32, half * 32 + 32)
    b = StreamBank(32, H, W, scales=(s,))
    o = torch.empty((32, 9, H, W, 3), device=dev)
    for kk, f in enumerate((f0, f1)):
        b.step({s: f[sl].contiguous()}, {s: o}, {s: list(range(32))}, {s: [kk] * 32}, drop_rate=0.1)
    torch.cuda.synchronize()
    same = torch.equal(o, outs[sl])
    print(f"main path half {half}: bit-identical {same}")
    ok2 &= same
    del b, o
print("MAIN OK" if ok2 else "MAIN MISMATCH")
