"""Library baseline for the learned tokenizer: the same network
(weights from learned.make_weights, same layer order as oracle/learned_oracle.py)
in plain PyTorch on the GPU -- bf16 cuDNN conv3d (channels-last), cuBLAS
linears, SDPA window attention -- timed with CUDA events at the bench shape
(G x 1080p GoPs, s=3, D=256, 2 blocks per side), next to this repository's
tcgen05 tokenizer on the same inputs (LearnedTokenizer.encode_frames +
decode_tokens).  A comparison, not a parity check (the library path rounds
differently).

    python scripts/torch_baseline_learned.py [G]
"""
import json
import sys

sys.path.insert(0, ".")
import numpy as np
import torch
import torch.nn.functional as F

from paper_2602_03529_b200.learned import (FSQ_LEVELS, LearnedConfig, LearnedTokenizer,
                                           make_weights)

G = int(sys.argv[1]) if len(sys.argv) > 1 else 32
H, W, s = 1080, 1920, 3
dev = torch.device("cuda")
cfg = LearnedConfig()
D = cfg.dim
wts = make_weights(cfg)
Wt_ = {k: torch.from_numpy(v).to(dev, torch.bfloat16) for k, v in wts["W"].items()}
Bt_ = {k: torch.from_numpy(v).to(dev, torch.bfloat16) for k, v in wts["b"].items()}
conv_w = {}
for k, v in Wt_.items():
    if v.shape[1] == 18 * D or k == "dec_in":
        cin = v.shape[1] // 18
        conv_w[k] = (v.reshape(v.shape[0], 2, 3, 3, cin).permute(0, 4, 1, 2, 3)
                     .contiguous(memory_format=torch.channels_last_3d))
lv = torch.tensor(FSQ_LEVELS, device=dev, dtype=torch.float32)


def conv(x, name, act=False, res=None):
    """x [G][C][T=2][H][W] channels-last-3d bf16, causal (2,3,3) conv."""
    y = F.conv3d(F.pad(x, (1, 1, 1, 1, 1, 0)), conv_w[name], Bt_[name])
    if act:
        y = F.silu(y)
    if res is not None:
        y = y + res
    return y.contiguous(memory_format=torch.channels_last_3d)


def attention(x, part):
    """x [G][D][2][Ht][Wt] -> x + proj(window attention(qkv(x)))."""
    G_, D_, T, Ht, Wt = x.shape
    Hp, Wp = -(-Ht // 8) * 8, -(-Wt // 8) * 8
    t = x.permute(0, 2, 3, 4, 1)                                       # [G][2][Ht][Wt][D]
    t = F.pad(t, (0, 0, 0, Wp - Wt, 0, Hp - Ht))
    t = t.reshape(G_, 2, Hp // 8, 8, Wp // 8, 8, D_).permute(0, 2, 4, 1, 3, 5, 6)
    t = t.reshape(-1, 128, D_)                                         # [B][2*64][D]
    qkv = F.linear(t, Wt_[f"{part}_qkv"], Bt_[f"{part}_qkv"]).view(t.shape[0], 128, 3, D_ // 64, 64)
    q, k, v = qkv.permute(2, 0, 3, 1, 4)                               # [B][heads][128][64]
    o = F.scaled_dot_product_attention(q, k, v, attn_mask=mask_cache[(Ht, Wt)])
    o = o.permute(0, 2, 1, 3).reshape(-1, 128, D_)
    o = F.linear(o, Wt_[f"{part}_proj"], Bt_[f"{part}_proj"])
    o = o.view(G_, Hp // 8, Wp // 8, 2, 8, 8, D_).permute(0, 3, 1, 4, 2, 5, 6)
    o = o.reshape(G_, 2, Hp, Wp, D_)[:, :, :Ht, :Wt].permute(0, 4, 1, 2, 3)
    return (x + o).contiguous(memory_format=torch.channels_last_3d)


def window_mask(Ht, Wt):
    """[B][1][128][128] bool: key inside the frame and of a frame <= the query's."""
    Hp, Wp = -(-Ht // 8) * 8, -(-Wt // 8) * 8
    yy = torch.arange(Hp, device=dev).view(Hp // 8, 1, 8, 1)
    xx = torch.arange(Wp, device=dev).view(1, Wp // 8, 1, 8)
    inside = ((yy < Ht) & (xx < Wt)).reshape(Hp // 8 * (Wp // 8), 64)  # [nwin][64]
    kval = inside.repeat(1, 2)                                         # [nwin][128]
    ft = torch.arange(128, device=dev) // 64
    causal = ft.view(128, 1) >= ft.view(1, 128)
    m = causal.view(1, 128, 128) & kval.view(-1, 1, 128)
    return m.repeat(G, 1, 1).view(-1, 1, 128, 128)


def encode(frames):
    fr = F.avg_pool2d(frames.view(G * 9, H, W, 3).permute(0, 3, 1, 2), s)  # box downscale
    h_, w_ = fr.shape[2], fr.shape[3]
    Ht, Wt = -(-h_ // 8), -(-w_ // 8)
    fr = F.pad(fr, (0, Wt * 8 - w_, 0, Ht * 8 - h_), mode="replicate")
    t = fr.view(G, 9, 3, Ht, 8, Wt, 8).permute(0, 3, 5, 1, 4, 6, 2).to(torch.bfloat16)
    pI = t[:, :, :, 0].reshape(G, Ht, Wt, 192)
    pP = t[:, :, :, 1:].reshape(G, Ht, Wt, 1536)
    h = torch.stack([F.linear(pI, Wt_["pe_i"], Bt_["pe_i"]),
                     F.linear(pP, Wt_["pe_p"], Bt_["pe_p"])], 1)       # [G][2][Ht][Wt][D]
    x = h.permute(0, 4, 1, 2, 3).contiguous(memory_format=torch.channels_last_3d)
    for i in range(cfg.blocks):
        u = conv(x, f"enc{i}_c1", act=True)
        x = conv(u, f"enc{i}_c2", res=x)
    x = attention(x, "enc")
    z = F.linear(x.permute(0, 2, 3, 4, 1), Wt_["head"], Bt_["head"])[..., :12].float()
    half_l = (lv - 1) * (1 - 1e-3) / 2
    off = torch.where(lv % 2 == 0, 0.5, 0.0)
    codes = torch.round(torch.tanh(z + torch.atanh(off / half_l)) * half_l - off) / (lv // 2)
    return codes, (Ht, Wt)


def decode(codes, hw):
    Ht, Wt = hw
    x = F.pad(codes.to(torch.bfloat16), (0, 64 - 12)).permute(0, 4, 1, 2, 3)
    x = conv(x.contiguous(memory_format=torch.channels_last_3d), "dec_in", act=True)
    x = attention(x, "dec")
    for i in range(cfg.blocks):
        u = conv(x, f"dec{i}_c1", act=True)
        x = conv(u, f"dec{i}_c2", res=x)
    h = x.permute(0, 2, 3, 4, 1)
    oi = F.linear(h[:, 0], Wt_["out_i"], Bt_["out_i"]).clamp(0, 1).float()
    op = F.linear(h[:, 1], Wt_["out_p"], Bt_["out_p"]).clamp(0, 1).float()
    f = torch.cat([oi.view(G, Ht, Wt, 1, 8, 8, 3), op.view(G, Ht, Wt, 8, 8, 8, 3)], 3)
    return f.permute(0, 3, 1, 4, 2, 5, 6).reshape(G, 9, Ht * 8, Wt * 8, 3)


def timed(fn, n=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


frames = torch.rand((G, 9, H, W, 3), device=dev)
hw_tok = (-(-(-(-H // s)) // 8), -(-(-(-W // s)) // 8))
mask_cache = {hw_tok: window_mask(*hw_tok)}
torch.backends.cudnn.benchmark = True
with torch.no_grad():
    lib_ms = timed(lambda: decode(*encode(frames)))
    # one causal (2,3,3) D -> D conv alone (cuDNN) at the latent shape
    xc = torch.randn((G, D, 2, hw_tok[0], hw_tok[1]), device=dev, dtype=torch.bfloat16)
    xc = xc.contiguous(memory_format=torch.channels_last_3d)
    conv_ms = timed(lambda: conv(xc, "enc0_c1", act=True), n=10)
model = LearnedTokenizer(cfg)


def ours():
    codes, idx, mask, hw = model.encode_frames(frames, s)
    model.decode_tokens(codes, mask, hw)


our_ms = timed(ours)
print(json.dumps({"G": G, "shape": "1080p, s=3, D=256, 2 blocks per side + attention",
                  "torch_cudnn_bf16_ms": round(lib_ms, 3), "tcgen05_ms": round(our_ms, 3),
                  "speedup": round(lib_ms / our_ms, 2),
                  "cudnn_conv233_ms": round(conv_ms, 3),
                  "cudnn_conv233_tflops": round(2 * G * 2 * hw_tok[0] * hw_tok[1] * D * 18 * D
                                                / conv_ms / 1e9, 1),
                  "frames_per_s": {"torch": round(G * 9 / lib_ms * 1e3),
                                   "tcgen05": round(G * 9 / our_ms * 1e3)}}))
